"""BASELINE.json configurations generated straight into HBM.

X = max(W [I_r H'] Pi + sigma N, 0), every random value addressed by
(seed, tag, counter) through the reference's counter scheme (reference
rng.py:26-55) with new tags >= 4, so any row range can be regenerated
independently on the host (oracle) or the device (``tsnmf_generate``):

  C1  m=1e4,   n=200, r=20, W ~ U[0,1], H' ~ U[0,1] columns scaled to sum 1, sigma 1e-3
  C2  m=2^26,  n=200, r=20, as C1                                  (107 GB)
  C3  C2 row-sharded over 1/2/4/8 GPUs, sigma in {1e-3, 1e-2}
  C4  m=1.6e9, n=25,  r=10, W lognormal(0,1), H' Dirichlet(1), sigma 1e-2   (320 GB)
  C5  m=2^28,  n=64,  r=16, W = sums of 4 Gaussian bumps, H' U[0,1] normalised, sigma 5e-3 (137 GB)

The small r x n mixing matrix and bump parameters are computed on the host
(host numpy, O(r n)); the m-sized work is the device generator.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _native
from . import device as dv
from . import streams

TAG_W, TAG_H, TAG_PERM, TAG_NOISE, TAG_BUMPS = 4, 5, 6, 7, 8
_W_KIND = {"uniform": 0, "lognormal": 1, "bumps": 2}


@dataclass(frozen=True)
class ConfigSpec:
    m: int
    n: int
    r: int
    sigma: float
    seed: int = 0
    w_kind: str = "uniform"
    h_kind: str = "uniform"


CONFIGS = {
    "C1": ConfigSpec(10_000, 200, 20, 1e-3),
    "C2": ConfigSpec(1 << 26, 200, 20, 1e-3),
    "C3": ConfigSpec(1 << 26, 200, 20, 1e-3),
    "C4": ConfigSpec(1_600_000_000, 25, 10, 1e-2, 0, "lognormal", "dirichlet"),
    "C5": ConfigSpec(1 << 28, 64, 16, 5e-3, 0, "bumps", "uniform"),
}


def config(name: str, **overrides) -> ConfigSpec:
    return replace(CONFIGS[name], **overrides)


def mixing(spec: ConfigSpec):
    """(M = [I H'] Pi as r x n, planted positions, permutation)."""
    r, n = spec.r, spec.n
    hu = streams.uniforms(spec.seed, TAG_H, 0, r * (n - r)).reshape(r, n - r)
    if spec.h_kind == "dirichlet":
        hu = -np.log1p(-hu)
    hp = hu / hu.sum(axis=0, keepdims=True)
    base = np.hstack([np.eye(r), hp])
    perm = np.argsort(streams.uniforms(spec.seed, TAG_PERM, 0, n), kind="stable")
    mix = np.ascontiguousarray(base[:, perm])
    planted = [int(np.flatnonzero(perm == t)[0]) for t in range(r)]
    return mix, planted, perm


def bump_params(spec: ConfigSpec) -> np.ndarray:
    u = streams.uniforms(spec.seed, TAG_BUMPS, 0, spec.r * 12).reshape(spec.r, 4, 3)
    p = u.copy()
    p[..., 2] = 0.02 + 0.18 * u[..., 2]
    return p


def generate_into(out, spec: ConfigSpec, row0: int = 0, mix=None, bumps=None):
    """Fill the device tensor ``out`` (rows x n, float64) with rows
    [row0, row0 + rows) of the configuration."""
    t = dv.torch()
    dev = out.device
    if mix is None:
        mix = mixing(spec)[0]
    mix_d = t.as_tensor(np.ascontiguousarray(mix), dtype=t.float64, device=dev)
    bumps_d = None
    if spec.w_kind == "bumps":
        bumps_d = t.as_tensor(bump_params(spec) if bumps is None else bumps, dtype=t.float64, device=dev)
    rows = int(out.shape[0])
    step = 1 << 22
    for a in range(0, rows, step):
        b = min(rows, a + step)
        view = out[a:b]
        _native.call("tsnmf_generate", view.data_ptr(), int(out.stride(0)), int(row0 + a), int(b - a), spec.n,
                     spec.r, mix_d.data_ptr(), _W_KIND[spec.w_kind],
                     bumps_d.data_ptr() if bumps_d is not None else None, int(spec.m), float(spec.sigma),
                     int(spec.seed), dv.stream_ptr(dev), device=dev, stage="generate")
    return out


def generate(spec: ConfigSpec, row0: int = 0, rows: int | None = None, device=None):
    t = dv.torch()
    dev = dv.require_device(device)
    rows = spec.m - row0 if rows is None else rows
    out = t.empty((rows, spec.n), dtype=t.float64, device=dev)
    return generate_into(out, spec, row0)
