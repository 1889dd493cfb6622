"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no hashing, no sketching, no
peeling): it only draws sparse fp32 gradients with the shapes, densities and
support structures of the paper's workloads (Table 1, resized to
BASELINE.json's configs).  Recipe:

* numpy ``PCG64`` seeded with ``base_seed + 1000 * config_index + worker``;
* exactly ``nnz_w = round(rho * d)`` nonzeros per worker, supports independent
  across workers (reading R19);
* support structure ``uniform`` (positions without replacement) or ``runs``
  (aligned runs of ``run`` consecutive coordinates: embedding rows / LSTM rows);
* value law ``dyadic`` (v = +-q * 2^-12, q uniform in [1, 2^12): every fp32 partial
  sum of such values is exact, so sums are order-independent) or ``gauss``
  (N(0, sigma^2), zeros redrawn as sigma).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 240207529


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def support(rng: np.random.Generator, d: int, nnz: int, structure: str = "uniform",
            run: int = 64) -> np.ndarray:
    """Sorted uint32 positions of exactly ``nnz`` distinct coordinates in [0, d)."""
    if nnz <= 0:
        return np.zeros(0, np.uint32)
    if nnz > d:
        raise ValueError("nnz > d")
    if structure == "uniform":
        pos = rng.choice(d, nnz, replace=False)
    elif structure == "runs":
        n_slots = d // run
        full, rem = divmod(nnz, run)
        need = full + (1 if rem else 0)
        if need > n_slots:
            raise ValueError("too many runs for d")
        slots = rng.choice(n_slots, need, replace=False)
        starts = slots.astype(np.int64) * run
        pos = (starts[:, None] + np.arange(run)[None, :]).reshape(-1)
        if rem:
            pos = np.concatenate([pos[: full * run], starts[-1] + np.arange(rem)])
    else:
        raise ValueError(structure)
    pos = np.sort(pos.astype(np.uint32))
    return pos


def values(rng: np.random.Generator, n: int, law: str = "gauss", sigma: float = 1e-3) -> np.ndarray:
    if law == "dyadic":
        q = rng.integers(1, 1 << 12, n)
        s = rng.integers(0, 2, n) * 2 - 1
        return (s * q).astype(np.float32) * np.float32(2.0 ** -12)
    if law == "gauss":
        v = (rng.standard_normal(n) * sigma).astype(np.float32)
        v[v == 0] = np.float32(sigma)
        return v
    if law == "ones":
        return np.ones(n, np.float32)
    raise ValueError(law)


@dataclass
class Workload:
    """One synthetic configuration (BASELINE.json configs)."""

    name: str
    d: int
    density: float
    workers: int
    structure: str = "uniform"
    run: int = 64
    law: str = "gauss"
    sigma: float = 1e-3
    index: int = 0  # config index for the seed recipe
    extra: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(round(self.density * self.d))

    def seed(self, worker: int) -> int:
        return BASE_SEED + 1000 * self.index + worker

    def coo(self, worker: int):
        rng = rng_for(self.seed(worker))
        idx = support(rng, self.d, self.nnz, self.structure, self.run)
        val = values(rng, len(idx), self.law, self.sigma)
        return idx, val

    def dense(self, worker: int, out: np.ndarray | None = None) -> np.ndarray:
        idx, val = self.coo(worker)
        x = np.zeros(self.d, np.float32) if out is None else out
        if out is not None:
            x[:] = 0
        x[idx] = val
        return x


# BASELINE.json configs: name -> Workload
CONFIGS = {
    "tiny": Workload("tiny", 10_000, 0.01, 2, "uniform", index=0),
    "ncf": Workload("ncf", 32_000_000, 0.01, 8, "runs", run=64, index=1),
    "lstm": Workload("lstm", 66_000_000, 0.05, 8, "runs", run=256, index=2),
    "bert": Workload("bert", 110_000_000, 0.01, 8, "uniform", index=3),
    "vgg": Workload("vgg", 143_000_000, 0.01, 8, "uniform", index=4),
}


def config(name: str, **over) -> Workload:
    base = CONFIGS[name]
    kw = dict(base.__dict__)
    kw.update(over)
    return Workload(**kw)
