"""Run the REFERENCE package with the B200 backend selected — TEST INFRASTRUCTURE (subprocess target of
tests/test_refbackend.py).

The reference tree is a scratch copy of the installed reference (baseline/_ref/tsnmf, built by
tools/install_reference.sh) with the 6-line maintainer patch of paper_1402_6964_b200.refbackend applied; this
script is started with ``TSNMF_BACKEND=b200`` and PYTHONPATH = <scratch>:<repo>, so ``import tsnmf`` is the
reference's own code with its hot path on the device.

    python tests/refbackend_run.py pipeline <x.tsm> <outdir>   # reference pipeline.run_factorize / run_sweep
    python tests/refbackend_run.py backend                      # which backend the reference reports

Prints one JSON object on stdout.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path


def pipeline(x_path: str, outdir: str) -> dict:
    import tsnmf
    from tsnmf import pipeline as pl

    assert getattr(tsnmf, "__b200_installed__", False), "the B200 backend was not installed by the patch"
    out = Path(outdir)
    cfg = pl.RunConfig(input=Path(x_path), outdir=out, algorithms=("spa", "gp"), r_values=(20,))
    s1 = pl.run_factorize(cfg)
    s2 = pl.run_factorize(pl.RunConfig(input=Path(x_path), outdir=out, algorithms=("spa", "gp"), r_values=(20,)))
    # XRAY refits and compute_h through the device batched NNLS
    from paper_1402_6964_b200 import refbackend

    refbackend.install(tsnmf, select=True)
    sx = pl.run_factorize(pl.RunConfig(input=Path(x_path), outdir=out / "xray", algorithms=("xray",),
                                       r_values=(20,)))
    sw = pl.run_sweep(pl.RunConfig(input=Path(x_path), outdir=out, algorithms=("spa",), r_values=(5, 10, 20)))
    files = sorted(p.name for p in out.iterdir() if p.is_file())
    h = tsnmf.CoefficientMatrix.load(out / "spa.H.tsm")
    return {"first": s1, "second": s2, "xray": sx, "sweep_cells": sw["cells"], "sweep_cache_hit": sw["cache_hit"],
            "files": files, "h_spa": h.entries.tolist(), "backend": tsnmf.get_backend(),
            "stream_pass_module": tsnmf.tsqr.stream_pass.__module__}


def backend() -> dict:
    import tsnmf
    from tsnmf import kernels

    return {"backend": tsnmf.get_backend(), "impl": kernels._impl.__name__,
            "installed": getattr(tsnmf, "__b200_installed__", False)}


if __name__ == "__main__":
    what = sys.argv[1]
    res = pipeline(sys.argv[2], sys.argv[3]) if what == "pipeline" else backend()
    print(json.dumps(res, default=str))
