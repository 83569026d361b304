"""Parity of the whole device path against the oracle on the BASELINE configs' generators through the
full-size harness (tests/parity_full.py): R, stats, sketch, Gram, SPA / XRAY / GP selections and H.

By default each config runs at 1/64 of its m (C2 2^20 x 200, C5 2^22 x 64, C4 shard 6.25e6 x 25) so the
-m gpu suite stays short; TSNMF_PARITY_FULL=1 runs the configs at their own m (C2 2^26, C5 2^28, C4 shard
4e8 rows: ~10 min of host-core oracle time; the committed run is profiles/r02_parity_full.json)."""

import os

import pytest

pytestmark = pytest.mark.gpu


def test_configs_match_oracle(tmp_path):
    import parity_full as pf

    full = os.environ.get("TSNMF_PARITY_FULL") == "1"
    procs = min(len(os.sched_getaffinity(0)), 16)
    rep = pf.main(["--configs", "C2,C3,C5,C4s", "--scale", "1" if full else str(1 / 64), "--procs", str(procs),
                   "--out", str(tmp_path / "parity.json")])
    bad = [c["case"] for c in rep["cases"] if not c["pass"]]
    assert not bad, {c["case"]: (c["errors"], c["selection"]) for c in rep["cases"] if c["case"] in bad}
