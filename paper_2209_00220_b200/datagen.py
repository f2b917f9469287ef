"""Seeded synthetic columns (mirror of reference datagen.py:20-56).

Uniform draws come from numpy's PCG64 on the host (so a seed yields the same
column as the reference); the inverse-CDF search runs on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import device, stream

__all__ = ["ZipfSpec", "zipf_pmf", "gen_zipf", "gen_zipf_device", "PRNG_NAME"]

PRNG_NAME = "pcg64"


@dataclass(frozen=True)
class ZipfSpec:
    s: float
    domain_bits: int
    n_rows: int
    seed: int = 0

    def __post_init__(self):
        if self.s < 0:
            raise ValueError("skew must be >= 0")
        if not 4 <= self.domain_bits <= 24:
            raise ValueError("domain_bits must be 4..24")
        if self.n_rows < 1:
            raise ValueError("n_rows must be positive")

    @property
    def domain(self) -> int:
        return 1 << self.domain_bits


def zipf_pmf(s: float, domain: int) -> np.ndarray:
    """P(value v) for v = 0..domain-1, rank v+1 weighted (v+1)^-s."""
    w = np.arange(1, domain + 1, dtype=np.float64) ** -float(s)
    return w / w.sum()


def _cdf(spec: ZipfSpec) -> np.ndarray:
    c = np.cumsum(zipf_pmf(spec.s, spec.domain))
    c[-1] = 1.0
    return c


def gen_zipf_device(spec: ZipfSpec, chunk: int = 1 << 26) -> torch.Tensor:
    """int64 CUDA tensor of the spec's values (identical to the reference)."""
    cdf = torch.from_numpy(_cdf(spec)).to(device())
    rng = np.random.default_rng(spec.seed)
    out = torch.empty(spec.n_rows, dtype=torch.int64, device=cdf.device)
    lib = _lib.load()
    done = 0
    while done < spec.n_rows:
        m = min(chunk, spec.n_rows - done)
        u = torch.from_numpy(rng.random(m)).to(cdf.device)  # PCG64 stream, in order
        _lib.check(lib.bsb_zipf_from_uniform(u.data_ptr(), m, cdf.data_ptr(), spec.domain,
                                             out[done:].data_ptr(), stream()), "gen_zipf")
        done += m
    return out


def gen_zipf(spec: ZipfSpec) -> np.ndarray:
    """Deterministic int64 values for the spec (datagen.py:50-56)."""
    return gen_zipf_device(spec).cpu().numpy()
