"""The streaming unit (reference pkg/src/tsnmf/matio.py:65-78).

``data`` is a rows x n float64 block: a numpy array (host, streamed over PCIe)
or a torch CUDA tensor (device-resident, reduced in place).  ``row_offset`` is
the global index of its first row, which keys the sketch's Gaussian rows.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class RowChunk:
    row_offset: int
    data: object

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    @property
    def cols(self) -> int:
        return int(self.data.shape[1])
