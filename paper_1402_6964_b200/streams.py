"""Counter-based random streams on the device — the backend contract of
reference pkg/src/tsnmf/kernels.py:13-31 (``uniform_block``, ``normal_block``,
``get_backend``) and the stream helpers of reference rng.py:20-55.

Values are addressed by (stream, counter): the integer part (splitmix64) is
bit-exact with the reference; normals use CUDA's log/cos/sqrt and agree with
the reference's libm to a few ulp (the reference's own compiled-vs-python
contract is rtol 1e-12, reference tests/test_kernels.py:40-49).
Block functions return numpy arrays like the reference; ``*_device``
variants return torch CUDA tensors.
"""

from __future__ import annotations

import numpy as np

from . import device as dv

BACKEND = "cuda-sm100a"

TAG_SKETCH = 0
TAG_BASIS = 1
TAG_COEFF = 2
TAG_NOISE = 3

_MASK = (1 << 64) - 1


def get_backend() -> str:
    dv.require_device()
    return BACKEND


def derive_stream(seed: int, tag: int) -> int:
    """mix(seed ^ mix(tag + gamma)) (reference rng.py:33-35), computed by the library."""
    return dv.derive_stream(seed, tag)


def uniform_block_device(stream: int, start: int, count: int):
    return dv.uniform_block(stream, start & _MASK, count)


def normal_block_device(stream: int, start: int, count: int):
    return dv.normal_block(stream, start & _MASK, count)


def uniform_block(stream: int, start: int, count: int) -> np.ndarray:
    """Uniform [0, 1) doubles at counters start .. start+count-1."""
    return uniform_block_device(stream, start, count).cpu().numpy()


def normal_block(stream: int, start: int, count: int) -> np.ndarray:
    """Standard normals at indices start .. start+count-1 (Box-Muller, cosine branch)."""
    return normal_block_device(stream, start, count).cpu().numpy()


def uniforms(seed: int, tag: int, start: int, count: int) -> np.ndarray:
    return uniform_block(derive_stream(seed, tag), start & _MASK, count)


def normals(seed: int, tag: int, start: int, count: int) -> np.ndarray:
    return normal_block(derive_stream(seed, tag), start & _MASK, count)


def gaussian_rows_device(seed: int, row_offset: int, rows: int, k: int):
    return dv.gaussian_rows(seed, row_offset, rows, k)


def gaussian_rows(seed: int, row_offset: int, rows: int, k: int) -> np.ndarray:
    """rows x k: entry (i, t) is normal #((row_offset + i) * k + t) of the
    sketch stream (reference rng.py:48-55)."""
    return gaussian_rows_device(seed, row_offset, rows, k).cpu().numpy()
