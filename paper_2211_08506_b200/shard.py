"""Molecule sharding across GPUs (one process per GPU, no collective).

Each molecule's grid depends only on its own atoms (reference gridgen.py:
192-201; SPEC "batch parallelism is across grids only"), so a batch splits
into contiguous molecule ranges, one per rank, with no exchange step. Ranges
are balanced by an estimated per-molecule cost: output bytes dominate
(every voxel is written once), plus a term for the atoms' pair work.
"""

from __future__ import annotations

import numpy as np

__all__ = ["BYTES_PER_ATOM", "molecule_costs", "plan_shards", "shard_range", "rank_world",
           "rank_shard"]


# K3 cost of one atom in output-byte equivalents, from per-CTA timing of
# cfg4 on a B200 (5-20 atom molecules: 174 CTA-us for 2.2 MB of grid;
# 150-200 atoms: 461 CTA-us): ~1.76 us per atom ~ 22 KB of writes.
BYTES_PER_ATOM = 22_000.0


def molecule_costs(atom_counts, grid_bytes: int, bytes_per_atom: float = 0.0) -> np.ndarray:
    """Relative cost of each molecule: grid bytes + ``bytes_per_atom`` x atoms."""
    counts = np.asarray(atom_counts, dtype=np.float64)
    return float(grid_bytes) + bytes_per_atom * counts


def plan_shards(costs, world_size: int) -> list:
    """Split molecules into ``world_size`` contiguous ``(start, stop)`` ranges
    whose summed costs are as equal as prefix sums allow. Deterministic: every
    rank computes the same plan from the same costs."""
    if world_size < 1:
        raise ValueError(f"world_size must be >= 1, got {world_size}")
    costs = np.asarray(costs, dtype=np.float64).reshape(-1)
    n = len(costs)
    if n == 0:
        return [(0, 0)] * world_size
    prefix = np.concatenate([[0.0], np.cumsum(costs)])
    total = prefix[-1]
    cuts = [0]
    for r in range(1, world_size):
        target = total * r / world_size
        k = int(np.searchsorted(prefix, target, side="left"))
        # pick the closer of the two neighbouring cut points
        if k > 0 and abs(prefix[k - 1] - target) <= abs(prefix[min(k, n)] - target):
            k -= 1
        cuts.append(min(max(k, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world_size)]


def shard_range(n_molecules: int, rank: int, world_size: int, costs=None) -> range:
    """This rank's molecule indices (equal counts unless ``costs`` is given)."""
    if not 0 <= rank < world_size:
        raise ValueError(f"rank {rank} outside world of {world_size}")
    if costs is None:
        costs = np.ones(n_molecules)
    start, stop = plan_shards(costs, world_size)[rank]
    return range(start, stop)


def rank_world(group=None) -> tuple:
    """``(rank, world_size)`` of this process: from torch.distributed when it
    is initialised (``group`` optional), else from the launcher's RANK /
    WORLD_SIZE environment (torchrun), else ``(0, 1)``."""
    import os

    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(group), dist.get_world_size(group)
    except ImportError:  # pragma: no cover - torch is in the image
        pass
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def rank_shard(n_molecules: int, atom_counts=None, grid_bytes: int = 0, group=None) -> range:
    """This process's contiguous molecule range of a batch sharded over the
    job's ranks (one process per GPU, no collective: reference
    gridgen.py:206-219 fans molecules out the same way inside one process).
    With ``atom_counts`` and ``grid_bytes`` the cut balances the estimated
    K3 cost (grid bytes + BYTES_PER_ATOM x atoms) instead of the counts;
    every rank computes the same plan."""
    rank, world = rank_world(group)
    costs = None
    if atom_counts is not None:
        costs = molecule_costs(atom_counts, grid_bytes, BYTES_PER_ATOM)
    return shard_range(n_molecules, rank, world, costs)
