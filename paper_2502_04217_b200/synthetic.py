"""Synthetic test problems (reference synthetic.py:1-63), host-side inputs."""

from __future__ import annotations

from dataclasses import dataclass

from .fourier import GridShape
from .masking import Mask
from .workloads import harmonics

__all__ = ["SyntheticSpec", "generate_synthetic"]


@dataclass(frozen=True)
class SyntheticSpec:
    """Recipe for a reproducible noisy problem with missing samples."""

    dims: tuple[int, ...]
    noise_seed: int = 0
    missing_fraction: float = 0.15
    missing_seed: int = 1

    def __post_init__(self):
        if not 0.0 <= self.missing_fraction < 1.0:
            raise ValueError("missing_fraction must lie in [0, 1)")


def generate_synthetic(spec: SyntheticSpec):
    """(noisy signal, mask, truth) -- deterministic in the seeds."""
    shape = GridShape(spec.dims)
    noisy, flags, truth = harmonics(shape.dims, spec.noise_seed, spec.missing_fraction,
                                    spec.missing_seed)
    return noisy, Mask.from_bool(flags, shape), truth
