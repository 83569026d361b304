"""Run orchestration on the B200 backend (reference pkg/src/tsnmf/pipeline.py): flag validation on CPU,
factorize / sweep / artifact cache on the GPU against the live reference's C1 results (golden)."""
import json

import numpy as np
import pytest

from paper_1402_6964_b200.errors import UsageError
from paper_1402_6964_b200.matio import write_matrix
from paper_1402_6964_b200.pipeline import RunConfig, run_factorize, run_sweep


@pytest.mark.parametrize("kw,msg", [
    (dict(algorithms=("foo",)), "unknown algorithms"),
    (dict(algorithms=()), "at least one algorithm"),
    (dict(r_values=(0,)), "separation ranks must be >= 1"),
    (dict(reduction="lu"), "reduction must be qr or svd"),
    (dict(threads=0), "threads must be >= 1"),
    (dict(sketch_k=0), "sketch rows must be >= 1"),
    (dict(algorithms=("xray",), normalization="l1"), "xray forbids normalization"),
    (dict(algorithms=("gp",), normalization="none"), "gp requires l1 normalization"),
    (dict(normalization="l2"), "normalization must be l1 or none"),
])
def test_run_config_validation(tmp_path, kw, msg):
    with pytest.raises(UsageError, match=msg):
        RunConfig(input=tmp_path / "x.bin", outdir=tmp_path / "out", **kw).validate()


def test_run_config_defaults(tmp_path):
    cfg = RunConfig(input=tmp_path / "x.bin", outdir=tmp_path, algorithms=("spa", "gp"), r_values=(20,)).validate()
    assert cfg.normalization == "l1" and cfg.resolve_sketch_k() == 120
    assert RunConfig(input="a", outdir="b", algorithms=("xray",)).validate().normalization == "none"


@pytest.mark.gpu
def test_factorize_c1_matches_reference(tmp_path, oracle, golden_c1):
    spec = oracle.config_spec("C1")
    x = oracle.config_rows(spec, 0, spec.m)
    path = tmp_path / "c1.bin"
    write_matrix(path, x)
    out = tmp_path / "run"
    s = run_factorize(RunConfig(input=path, outdir=out, algorithms=("spa", "gp"), r_values=(20,)))
    assert s["results"]["spa"]["indices"] == list(golden_c1["k_spa"])
    assert s["results"]["gp"]["indices"] == list(golden_c1["k_gp"])
    assert abs(s["results"]["spa"]["relative_residual"] - float(golden_c1["resid_spa"][0])) <= 1e-10
    assert (s["m"], s["n"], s["cache_hit"]) == (spec.m, spec.n, False)
    assert s["reader"]["rows_read"] == spec.m and s["reader"]["bytes_read"] == path.stat().st_size
    for f in ("spa.extremes.json", "spa.H.tsm", "spa.residual.json", "gp.extremes.json", "run_summary.json",
              "timings.json"):
        assert (out / f).exists(), f
    assert json.loads((out / "spa.extremes.json").read_text())["indices"] == list(golden_c1["k_spa"])
    # second run: artifacts from the cache, no read
    s2 = run_factorize(RunConfig(input=path, outdir=out, algorithms=("spa", "gp"), r_values=(20,)))
    assert s2["cache_hit"] and s2["reader"]["rows_read"] == 0
    assert s2["results"]["spa"]["indices"] == s["results"]["spa"]["indices"]
    # xray (no normalisation), host and device selection agree with the reference
    sx = run_factorize(RunConfig(input=path, outdir=tmp_path / "rx", algorithms=("xray",), r_values=(20,),
                                 device_select=True))
    assert sx["results"]["xray"]["indices"] == list(golden_c1["k_xray"])
    sw = run_sweep(RunConfig(input=path, outdir=out, algorithms=("spa",), r_values=(5, 10, 20)))
    assert sw["cells"] == 3 and (out / "sweep.csv").exists() and sw["cache_hit"]
