"""Learned sort-join (reference lsj.py) -- GPU pipeline under construction."""

from __future__ import annotations

from dataclasses import dataclass


class ModelMismatchError(ValueError):
    """A sorted relation was joined under a model/scale it was not built with."""


@dataclass(frozen=True)
class LsjConfig:
    """lsj.py:30-68."""

    workers: int = 1
    sample_rate: float = 0.01
    fanout: int = 10000
    swwc: bool = True
    swwc_buf_len: int = 64
    overalloc: float = 0.02
    model_fanout: int | None = None
    seed: int = 0x1D5EED

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if not 0.0 < self.sample_rate <= 1.0:
            raise ValueError("sample_rate must be in (0, 1]")
        if self.fanout < self.workers:
            raise ValueError("fanout must be >= workers")
        if self.swwc_buf_len < 1:
            raise ValueError("swwc_buf_len must be >= 1")
        if self.overalloc < 0.0:
            raise ValueError("overalloc must be >= 0")

    def effective_fanout(self) -> int:
        return -(-self.fanout // self.workers) * self.workers


def lsj_join(r, s, config: LsjConfig | None = None, materialize: bool = False):
    raise NotImplementedError("LSJ GPU pipeline not built yet")
