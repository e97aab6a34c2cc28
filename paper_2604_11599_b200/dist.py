"""Multi-GPU sharding of independent units: one process per GPU.

* trajectories (cfg 1/2): each rank runs a contiguous range of GLOBAL shot indices --
  the same split rule as the reference's process pool (`np.linspace` bounds,
  sim.py:382-391) -- and the per-shot RNG stream `for_shot(seed, global_shot)`
  (sim.py:54-57) makes the merged histogram identical for any number of ranks.
  No collective touches the data path; the histogram merge is one host-side gather.
* parameter points (cfg 3): contiguous point ranges per rank; energies gathered.

The per-rank executor defaults to this package's GPU path; tests inject the CPU
oracle to check the protocol under `gloo` with world size 2 (no GPU needed).
"""

from __future__ import annotations

from collections import Counter

import numpy as np


def shard_bounds(total: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) ranges, np.linspace rule of sim.py:382."""
    b = np.linspace(0, total, world + 1, dtype=int)
    return [(int(b[i]), int(b[i + 1])) for i in range(world)]


def _world(group=None):
    """(module, rank, world size) of `group` (default: the default process group)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_rank(group), dist.get_world_size(group)
    return None, 0, 1


def _gpu_counts(bound, shots, seed, shot_begin, precision, device):
    from . import sim

    if shots <= 0:
        return Counter()
    tape = sim.compile_tape(bound.kernel, device)
    if tape.nwords == 1:  # histogram built on the device; only distinct outcomes come back
        uniq, counts = sim.sample_counts(bound, shots, seed, shot_begin=shot_begin, precision=precision, device=device)
        keys = tape.keys(uniq) if tape.nbits else [""] * len(uniq)
        return Counter({k: int(c) for k, c in zip(keys, counts)})
    words, tape = sim.sample_words(bound, shots, seed, shot_begin=shot_begin, precision=precision, device=device)
    return Counter(sim.histogram_from_words(tape, words, shots).counts)


def sample_sharded(bound, shots: int, seed: int, *, executor=None, precision=None, device=None, group=None):
    """`sample` over all ranks of the default process group; every rank returns the
    same ShotHistogram.  executor(bound, n, seed, shot_begin) -> Counter runs one
    rank's contiguous global-shot range."""
    from .errors import SimError
    from .sim import ShotHistogram

    if shots < 1:
        raise SimError("shots must be >= 1")
    dist, rank, world = _world(group)
    lo, hi = shard_bounds(shots, world)[rank]
    if executor is None:
        local = _gpu_counts(bound, hi - lo, seed, lo, precision, device)
    else:
        local = executor(bound, hi - lo, seed, lo)
    if dist is None:
        return ShotHistogram(dict(local), shots)
    parts = [None] * world
    dist.all_gather_object(parts, dict(local), group=group)
    merged: Counter = Counter()
    for p in parts:  # fixed rank order
        merged.update(p)
    return ShotHistogram(dict(merged), shots)


def observe_sharded(kernel, hamiltonian, points, *, executor=None, precision=None, device=None, group=None):
    """Energies of all points, computed as contiguous point ranges per rank and
    gathered in rank order (every rank returns the full array)."""
    pts = np.asarray(points, dtype=np.float64).reshape(len(points), -1)
    dist, rank, world = _world(group)
    lo, hi = shard_bounds(len(pts), world)[rank]
    if hi > lo:
        if executor is None:
            from . import sim

            local = np.asarray(sim.observe(kernel, hamiltonian, pts[lo:hi], precision=precision, device=device))
        else:
            local = np.asarray(executor(kernel, hamiltonian, pts[lo:hi]))
    else:
        local = np.zeros(0)
    if dist is None:
        return local
    parts = [None] * world
    dist.all_gather_object(parts, local.tolist(), group=group)
    return np.array([e for p in parts for e in p], dtype=np.float64)
