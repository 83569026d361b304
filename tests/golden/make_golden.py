"""Generate the golden fixtures under tests/golden/ by running the LIVE reference.

Run in the build container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py            # builds /tmp/tsnmf_ref from /root/reference if needed

The reference package is copied to a writable scratch dir and its Cython RNG
is compiled there (reference pkg/setup.py); nothing from the reference is
written into this repository except these small output vectors.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = os.environ.get("TSNMF_REFERENCE", "/root/reference/pkg")
REF_BUILD = os.environ.get("TSNMF_REF_BUILD", "/tmp/tsnmf_ref")


def load_reference():
    if not os.path.isdir(os.path.join(REF_BUILD, "src", "tsnmf")):
        shutil.copytree(REF_SRC, REF_BUILD)
        subprocess.run(["chmod", "-R", "u+w", REF_BUILD], check=True)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=REF_BUILD,
                       check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(REF_BUILD, "src"))
    import tsnmf  # noqa: E402

    assert tsnmf.get_backend() == "compiled", tsnmf.get_backend()
    return tsnmf


def rng_fixture(ts):
    from tsnmf import kernels, rng

    seeds_tags = [(0, 0), (0, 1), (1, 0), (7, 3), (2**63 + 17, 2), (987654321, 0), (2**64 - 1, 5)]
    streams = np.array([rng.derive_stream(s, t) for s, t in seeds_tags], dtype=np.uint64)
    blocks = [(123, 0, 4096), (9, 10, 1000), (2**63 + 5, 2**40, 777), (0x48218226FF3CD4BF, 2**64 - 300, 600)]
    out = {
        "seeds_tags": np.array(seeds_tags, dtype=np.uint64),
        "streams": streams,
        "blocks": np.array(blocks, dtype=np.uint64),
    }
    for i, (s, start, cnt) in enumerate(blocks):
        out[f"uniform_{i}"] = kernels.uniform_block(s, start, cnt)
        out[f"normal_{i}"] = kernels.normal_block(s, start % 2**63, cnt)
    out["gaussian_rows_5_0_10_4"] = rng.gaussian_rows(5, 0, 10, 4)
    out["gaussian_rows_3_1000_16_9"] = rng.gaussian_rows(3, 1000, 16, 9)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def small_cases():
    g = np.random.default_rng(20140227)
    cases = {}
    cases["tall_40x5"] = g.standard_normal((40, 5))
    cases["tall_300x17"] = g.uniform(0, 1, (300, 17))
    cases["tall_1000x64"] = g.standard_normal((1000, 64)) * np.logspace(0, -3, 64)
    x = g.uniform(0, 1, (257, 25))
    x[:, 7] = 0.0
    cases["zerocol_257x25"] = x
    cases["square_30x30"] = g.standard_normal((30, 30))
    cases["ill_500x12"] = g.standard_normal((500, 12)) @ np.diag(np.logspace(0, -7, 12))
    return cases


def tsqr_fixture(ts):
    from tsnmf import RowChunk, tsqr

    out = {}
    for name, x in small_cases().items():
        out[f"{name}__x"] = x
        for size in (1, 7, 64, x.shape[0]):
            # "first-come" with threads=1 takes the reference's ordered tree branch (tsqr.py:315-333)
            for order in ("tree", "sequential", "first-come"):
                chunks = [RowChunk(o, x[o:o + size]) for o in range(0, x.shape[0], size)]
                res = tsqr.stream_pass(chunks, sketch_rows=6, seed=11, combine_order=order)
                key = f"{name}__c{size}__{order}"
                out[key + "__r"] = np.asarray(res.factor.entries)
                out[key + "__l1"] = np.asarray(res.stats.l1)
                out[key + "__l2"] = np.asarray(res.stats.l2)
                out[key + "__sketch"] = np.asarray(res.sketch.entries)
                out[key + "__meta"] = np.array([res.rows, res.chunks, res.tree_depth])
    # factor_chunk / combine known answers and edge shapes
    out["fc_345"] = np.asarray(tsqr.factor_chunk(np.array([[3.0, 0], [4, 0], [0, 5]])).entries)
    out["fc_row"] = np.asarray(tsqr.factor_chunk(np.array([[1.0, 2, 2]])).entries)
    out["fc_negrow"] = np.asarray(tsqr.factor_chunk(np.array([[-1.0, 2, -2]])).entries)
    w = np.random.default_rng(5).standard_normal((3, 6))
    out["fc_wide_in"] = w
    out["fc_wide"] = np.asarray(tsqr.factor_chunk(w).entries)
    d34 = tsqr.TriangularFactor(np.diag([3.0, 4.0]))
    d43 = tsqr.TriangularFactor(np.diag([4.0, 3.0]))
    out["comb_diag"] = np.asarray(tsqr.combine(d34, d43).entries)
    np.savez_compressed(os.path.join(HERE, "tsqr_small.npz"), **out)


def c1_fixture(ts):
    """BASELINE config C1 (m=1e4, n=200, r=20): X from the oracle's config
    generator, reduced by the reference; selection + NNLS by the reference."""
    sys.path.insert(0, REPO)
    from oracle import tsnmf_oracle as orc
    from tsnmf import RowChunk, compute_h, gp_select, relative_residual, scale_columns
    from tsnmf import spa, stream_pass, xray_greedy, rsvd

    spec = orc.config_spec("C1", seed=0)
    mix, planted, perm = orc.config_mixing(spec)
    x = orc.config_rows(spec, 0, spec.m, mix)
    k = orc.default_sketch_rows(spec.r)
    chunks = [RowChunk(o, x[o:o + 8192]) for o in range(0, spec.m, 8192)]
    res = stream_pass(chunks, sketch_rows=k, seed=0)
    red = rsvd(res.factor)
    k_spa = spa(red, spec.r, normalize=True, stats=res.stats)
    k_xray = xray_greedy(red, spec.r)
    k_gp = gp_select(scale_columns(res.sketch, res.stats), spec.r)
    h = compute_h(red, k_spa)
    resid = relative_residual(red, k_spa, h)
    h_r = compute_h(res.factor, k_spa)
    np.savez_compressed(
        os.path.join(HERE, "c1.npz"),
        x_checksum=np.array([x.sum(), (x * x).sum(), x[123, 45], x[9999, 199]]),
        planted=np.array(planted), perm=perm, mix=mix,
        r=np.asarray(res.factor.entries), l1=np.asarray(res.stats.l1), l2=np.asarray(res.stats.l2),
        sketch=np.asarray(res.sketch.entries), meta=np.array([res.rows, res.chunks, res.tree_depth, k]),
        k_spa=np.array(k_spa.indices), k_xray=np.array(k_xray.indices), k_gp=np.array(k_gp.indices),
        h_spa=np.asarray(h.entries), h_spa_on_r=np.asarray(h_r.entries), resid_spa=np.array([resid]),
        sigma=np.asarray(red.singular_values),
    )


def select_fixture(ts):
    """Selection / NNLS known answers and random reduced
    matrices run through the reference host algorithms."""
    from tsnmf import compute_h, gp_select, nnls_solve, relative_residual, spa, xray_greedy
    from tsnmf import SketchResult, ColumnStats

    g = np.random.default_rng(31)
    out = {}
    for i in range(4):
        n, r = (12, 4) if i < 2 else (40, 8)
        w = g.uniform(0, 1, (3 * n, r))
        hp = g.uniform(0, 1, (r, n - r))
        x = w @ np.hstack([np.eye(r), hp / hp.sum(0)])
        x = x[:, g.permutation(n)]
        rr = np.linalg.qr(x, mode="r")
        rr[np.diagonal(rr) < 0] *= -1
        stats = ColumnStats(l1=np.abs(x).sum(0), l2=np.sqrt((x * x).sum(0)))
        out[f"m{i}"] = rr
        out[f"m{i}_l1"] = np.asarray(stats.l1)
        out[f"m{i}_spa"] = np.array(spa(rr, r, normalize=True, stats=stats).indices)
        out[f"m{i}_spa_raw"] = np.array(spa(rr, r).indices)
        kx = xray_greedy(rr, r)
        out[f"m{i}_xray"] = np.array(kx.indices)
        h = compute_h(rr, kx)
        out[f"m{i}_h_xray"] = np.asarray(h.entries)
        out[f"m{i}_res_xray"] = np.array([relative_residual(rr, kx, h)])
        sk = SketchResult(entries=g.standard_normal((7, n)), seed=0)
        out[f"m{i}_sk"] = np.asarray(sk.entries)
        gp = gp_select(sk, r)
        out[f"m{i}_gp"] = np.array(gp.indices)
        out[f"m{i}_gp_short"] = np.array([gp.shortfall])
    a = g.standard_normal((20, 6))
    b = g.standard_normal(20)
    out["nnls_a"], out["nnls_b"] = a, b
    out["nnls_y"] = nnls_solve(a, b)
    np.savez_compressed(os.path.join(HERE, "select.npz"), **out)


def main():
    ts = load_reference()
    rng_fixture(ts)
    tsqr_fixture(ts)
    select_fixture(ts)
    c1_fixture(ts)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
