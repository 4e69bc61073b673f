"""Seeded synthetic molecule batches for BASELINE.json configs 0-4.

No public dataset is used: the paper's MOSES / PCQM4Mv2 corpora are not in
the image. Each config restates BASELINE.json's distribution (SURVEY.md
§8(d)): atom counts, element probabilities, coordinate law, minimum pair
distance (sequential rejection), grid shape and box. Molecule ``i`` of
config ``k`` is drawn from its own generator ``default_rng([1000 + k, i])``,
so any subset (a rank's shard, a strided parity sample) is generated
directly and identically on every host.

Channel integers follow the reference's atomic-number order
(H0 C1 N2 O3 F4 / H0 C1 N2 O3 P4 S5 Fe6 Zn7, reference io.py:69-85).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["SynthConfig", "CONFIGS", "atom_counts", "molecule", "packed_batch", "PackedBatch"]

_SMALL_P = (0.5, 0.35, 0.07, 0.07, 0.01)                     # H C N O F
# BASELINE lists (H,C,N,O,S,P,Fe,Zn) p=(.49,.31,.08,.09,.01,.005,.0025,.0025),
# summing to 0.99; reordered to atomic-number channels (P before S), renormalised.
_LARGE_P = tuple(v / 0.99 for v in (0.49, 0.31, 0.08, 0.09, 0.005, 0.01, 0.0025, 0.0025))


@dataclass(frozen=True)
class SynthConfig:
    index: int
    name: str
    n_molecules: int
    atoms: tuple          # ("uniform", lo, hi) inclusive | ("loguniform", lo, hi)
    element_p: tuple
    coords: tuple         # ("uniform", lo, hi) | ("gaussian", center, std)
    min_dist: float
    shape: tuple          # (H, W, D)
    box_origin: tuple
    box_extents: tuple
    sigma: float = 0.5    # GaussianVoxelizer default, reference estimator.py:55

    @property
    def channels(self) -> int:
        return len(self.element_p)

    @property
    def seed(self) -> int:
        return 1000 + self.index

    @property
    def grid_bytes(self) -> int:
        H, W, D = self.shape
        return self.channels * H * W * D * 4


CONFIGS = {
    0: SynthConfig(0, "cfg0-small-batch", 64, ("uniform", 9, 29), _SMALL_P,
                   ("uniform", 0.0, 10.0), 0.9, (32, 32, 32), (0.0, 0.0, 0.0), (10.0, 10.0, 10.0)),
    1: SynthConfig(1, "cfg1-1024x64^3", 1024, ("uniform", 9, 29), _SMALL_P,
                   ("uniform", 0.0, 10.0), 0.9, (64, 64, 64), (-1.0, -1.0, -1.0),
                   (12.0, 12.0, 12.0)),
    2: SynthConfig(2, "cfg2-65536x32^3", 65536, ("uniform", 9, 29), _SMALL_P,
                   ("uniform", 0.0, 10.0), 0.9, (32, 32, 32), (0.0, 0.0, 0.0), (10.0, 10.0, 10.0)),
    3: SynthConfig(3, "cfg3-32x128^3-clusters", 32, ("uniform", 1500, 3000), _LARGE_P,
                   ("gaussian", 32.0, 12.0), 1.0, (128, 128, 128), (0.0, 0.0, 0.0),
                   (64.0, 64.0, 64.0)),
    4: SynthConfig(4, "cfg4-4096x48^3-skewed", 4096, ("loguniform", 5, 200), _SMALL_P,
                   ("uniform", 0.0, 16.0), 0.9, (48, 48, 48), (0.0, 0.0, 0.0), (16.0, 16.0, 16.0)),
}


def _atom_count(cfg: SynthConfig, rng) -> int:
    kind, lo, hi = cfg.atoms
    if kind == "uniform":
        return int(rng.integers(lo, hi + 1))
    return int(np.rint(np.exp(rng.uniform(math.log(lo), math.log(hi)))))


def _draw(cfg: SynthConfig, rng, m: int) -> np.ndarray:
    kind, a, b = cfg.coords
    if kind == "uniform":
        return rng.uniform(a, b, size=(m, 3))
    return rng.normal(a, b, size=(m, 3))


def atom_counts(cfg: SynthConfig, indices) -> np.ndarray:
    """Atom count of each molecule in ``indices`` without drawing its atoms
    (the count is the first draw of the molecule's generator), for
    cost-balanced sharding."""
    return np.array([_atom_count(cfg, np.random.default_rng([cfg.seed, int(i)]))
                     for i in indices], dtype=np.int64)


def molecule(cfg: SynthConfig, index: int):
    """(channels int32 (n,), xyz float64 (n, 3)) of molecule ``index``."""
    rng = np.random.default_rng([cfg.seed, int(index)])
    n = _atom_count(cfg, rng)
    channels = rng.choice(cfg.channels, size=n, p=np.asarray(cfg.element_p)).astype(np.int32)
    xyz = np.empty((n, 3), dtype=np.float64)
    r2 = cfg.min_dist * cfg.min_dist
    k = 0
    while k < n:
        for cand in _draw(cfg, rng, 8 + 2 * (n - k)):
            if k == 0 or float(np.min(((xyz[:k] - cand) ** 2).sum(axis=1))) >= r2:
                xyz[k] = cand
                k += 1
                if k == n:
                    break
    return channels, xyz


@dataclass
class PackedBatch:
    """CSR batch: molecule b owns atoms offsets[b]:offsets[b+1]."""

    offsets: np.ndarray   # int64 (B+1,)
    channels: np.ndarray  # int32 (n,)
    xyz: np.ndarray       # float64 (n, 3)

    @property
    def n_molecules(self) -> int:
        return len(self.offsets) - 1

    def molecule(self, b: int):
        lo, hi = self.offsets[b], self.offsets[b + 1]
        return self.channels[lo:hi], self.xyz[lo:hi]


def packed_batch(cfg: SynthConfig, indices=None) -> PackedBatch:
    """Pack molecules ``indices`` (default: the whole config) into CSR arrays."""
    if indices is None:
        indices = range(cfg.n_molecules)
    mols = [molecule(cfg, i) for i in indices]
    counts = np.array([len(c) for c, _ in mols], dtype=np.int64)
    offsets = np.zeros(len(mols) + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    channels = np.concatenate([c for c, _ in mols]) if mols else np.zeros(0, np.int32)
    xyz = np.concatenate([x for _, x in mols]) if mols else np.zeros((0, 3))
    return PackedBatch(offsets, channels.astype(np.int32), np.ascontiguousarray(xyz))
