"""The reference package running on the B200 backend (SURVEY §8b plugin point, §8f row 4).

A scratch copy of the installed reference (baseline/_ref/tsnmf, tools/install_reference.sh) gets the 6-line
maintainer patch from paper_1402_6964_b200.refbackend; with TSNMF_BACKEND=b200 the reference's own
``kernels.py`` selects the device block kernels and its ``__init__`` routes ``stream_pass`` / ``factor_chunk``
/ ``combine`` / ``sketch_chunk`` onto the device.  Then, unchanged reference code runs:
  * the reference's own tests/test_kernels.py (backend contract, reference tests/test_kernels.py:10-69);
  * the reference's ``pipeline.run_factorize`` / ``run_sweep`` on BASELINE config C1, which must reproduce the
    live reference's K, residual and H (tests/golden/c1.npz, made by tests/golden/make_golden.py).
CPU tests: the patch applies, is inert for the stock backends, and TSNMF_BACKEND=b200 without a GPU fails
loudly (no CPU fallback).
"""

from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "tsnmf")
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "ref_tests")

needs_ref = pytest.mark.skipif(not os.path.isdir(REF_PKG),
                               reason="reference not installed (bash tools/install_reference.sh)")


def _scratch_reference(tmp_path):
    from paper_1402_6964_b200.refbackend import patch_reference_tree

    dst = tmp_path / "ref"
    shutil.copytree(REF_PKG, dst / "tsnmf", ignore=shutil.ignore_patterns("__pycache__"))
    patch_reference_tree(dst / "tsnmf")
    return dst


def _env(scratch, backend):
    env = dict(os.environ)
    env["TSNMF_BACKEND"] = backend
    env["PYTHONPATH"] = os.pathsep.join([str(scratch), ROOT] + [p for p in [env.get("PYTHONPATH")] if p])
    return env


def _run(args, scratch, backend, timeout=600):
    return subprocess.run([sys.executable, *args], env=_env(scratch, backend), capture_output=True, text=True,
                          timeout=timeout, cwd=str(scratch))


@needs_ref
def test_patch_is_small_and_inert_for_stock_backends(tmp_path):
    scratch = _scratch_reference(tmp_path)
    orig = open(os.path.join(REF_PKG, "kernels.py")).read().splitlines()
    new = (scratch / "tsnmf" / "kernels.py").read_text().splitlines()
    assert len(new) - len(orig) == 2
    init_added = len((scratch / "tsnmf" / "__init__.py").read_text().splitlines()) - len(
        open(os.path.join(REF_PKG, "__init__.py")).read().splitlines())
    assert init_added <= 6
    for backend in ("compiled", "python"):
        p = _run([os.path.join(ROOT, "tests", "refbackend_run.py"), "backend"], scratch, backend)
        assert p.returncode == 0, p.stderr
        out = json.loads(p.stdout.strip().splitlines()[-1])
        assert out == {"backend": backend, "impl": out["impl"], "installed": False}
    # patching twice is a no-op
    from paper_1402_6964_b200.refbackend import patch_reference_tree

    before = (scratch / "tsnmf" / "kernels.py").read_text()
    patch_reference_tree(scratch / "tsnmf")
    assert (scratch / "tsnmf" / "kernels.py").read_text() == before


@needs_ref
def test_b200_backend_without_gpu_fails_loudly(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    scratch = _scratch_reference(tmp_path)
    p = _run(["-c", "import tsnmf"], scratch, "b200")
    assert p.returncode != 0
    assert "no CUDA device" in p.stderr or "libtsnmf_b200" in p.stderr


@pytest.mark.gpu
@needs_ref
def test_reference_kernel_tests_on_b200_backend(tmp_path):
    """The reference's own backend tests with TSNMF_BACKEND=b200.  test_backend_reported pins the backend name
    to the two stock backends ("compiled", "python") and is the one expected deviation: it is run separately
    and must fail on exactly that name."""
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference tests not copied (tools/install_reference.sh)")
    scratch = _scratch_reference(tmp_path)
    shutil.copytree(REF_TESTS, scratch / "ref_tests")
    p = _run(["-m", "pytest", "-q", "-p", "no:cacheprovider", str(scratch / "ref_tests" / "test_kernels.py"),
              "-k", "not test_backend_reported"], scratch, "b200")
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout and "failed" not in p.stdout
    p = _run(["-m", "pytest", "-q", "-p", "no:cacheprovider", str(scratch / "ref_tests" / "test_kernels.py"),
              "-k", "test_backend_reported"], scratch, "b200")
    assert p.returncode == 1 and "'b200' in ('compiled', 'python')" in p.stdout, p.stdout[-2000:]
    p = _run([os.path.join(ROOT, "tests", "refbackend_run.py"), "backend"], scratch, "b200")
    assert p.returncode == 0, p.stderr
    assert json.loads(p.stdout.strip().splitlines()[-1]) == {
        "backend": "b200", "impl": "paper_1402_6964_b200.refbackend", "installed": True}


@pytest.mark.gpu
@needs_ref
def test_reference_pipeline_c1_on_b200_backend(tmp_path, oracle, golden_c1):
    """reference pipeline.run_factorize (pipeline.py:252-298) and run_sweep (:301-331) on C1, unchanged, with
    the pass on the device: K, GP K and the residual equal the live reference's; H within 1e-8."""
    from paper_1402_6964_b200.matio import write_matrix

    spec = oracle.config_spec("C1")
    x = oracle.config_rows(spec, 0, spec.m)
    path = tmp_path / "c1.tsm"
    write_matrix(path, x)
    scratch = _scratch_reference(tmp_path)
    out = tmp_path / "run"
    p = _run([os.path.join(ROOT, "tests", "refbackend_run.py"), "pipeline", str(path), str(out)], scratch, "b200")
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    s1, s2, sx = res["first"], res["second"], res["xray"]
    assert res["backend"] == "b200" and s1["backend"] == "b200"
    assert res["stream_pass_module"] == "paper_1402_6964_b200.refbackend"
    assert s1["results"]["spa"]["indices"] == list(golden_c1["k_spa"])
    assert s1["results"]["gp"]["indices"] == list(golden_c1["k_gp"])
    assert abs(s1["results"]["spa"]["relative_residual"] - float(golden_c1["resid_spa"][0])) <= 1e-10
    assert np.abs(np.array(res["h_spa"]) - golden_c1["h_spa"]).max() <= 1e-8
    assert (s1["m"], s1["n"], s1["cache_hit"]) == (spec.m, spec.n, False)
    assert s1["reader"]["rows_read"] == spec.m and s1["reader"]["bytes_read"] == path.stat().st_size
    # second run: the reference's artifact cache, no read
    assert s2["cache_hit"] and s2["reader"]["rows_read"] == 0
    assert s2["results"]["spa"]["indices"] == s1["results"]["spa"]["indices"]
    # XRAY with the refits on the device NNLS
    assert sx["results"]["xray"]["indices"] == list(golden_c1["k_xray"])
    assert res["sweep_cells"] == 3 and res["sweep_cache_hit"]
    for f in ("spa.extremes.json", "spa.H.tsm", "spa.residual.json", "gp.extremes.json", "run_summary.json",
              "timings.json", "sweep.csv"):
        assert f in res["files"], f
