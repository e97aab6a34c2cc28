"""Multi-process sharding protocol under gloo, world size 2, on CPU.

The per-rank executor is the CPU oracle (test-only), so these tests check the host
side of the multi-GPU path: contiguous global-shot ranges, per-shot RNG streams and
the rank-ordered merge give the single-process histogram exactly; point sharding
gathers energies in order.
"""

import os
import socket
from collections import Counter

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_11599_b200 import dist as qdist
from paper_2604_11599_b200 import ir, workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_counts(bound, n, seed, shot_begin):
    from oracle import sim_port as P

    if n <= 0:
        return Counter()
    if P.is_dynamic(bound.kernel):
        return Counter(P.trajectory_keys(bound, seed, shot_begin, n))
    keys = P.static_keys(bound, n, seed, shot_begin)
    return Counter(keys)


def _oracle_energies(kernel, ham, pts):
    from oracle import sim_port as P

    return [P.observe(ir.bind(kernel, list(p)), ham) for p in pts]


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, k = workloads.dyn_circuit(n=6, layers=6, every=3, nmeas=2, seed=3)
        h = qdist.sample_sharded(ir.bind(k, []), 37, 11, executor=_oracle_counts)
        _, kv = workloads.vqe_ansatz(4, 1)
        ham = workloads.vqe_hamiltonian(4, 6, seed=2)
        pts = workloads.vqe_points(5, kv.total_params, seed=3)
        e = qdist.observe_sharded(kv, ham, pts, executor=_oracle_energies)
        out_q.put((rank, h.counts, h.total_shots, list(e)))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_match_reference_rule():
    assert qdist.shard_bounds(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert sum(hi - lo for lo, hi in qdist.shard_bounds(12345, 8)) == 12345


@pytest.mark.timeout(300)
def test_world_size_2_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    _, k = workloads.dyn_circuit(n=6, layers=6, every=3, nmeas=2, seed=3)
    want = _oracle_counts(ir.bind(k, []), 37, 11, 0)
    _, kv = workloads.vqe_ansatz(4, 1)
    ham = workloads.vqe_hamiltonian(4, 6, seed=2)
    pts = workloads.vqe_points(5, kv.total_params, seed=3)
    want_e = _oracle_energies(kv, ham, pts)
    for rank, counts, total, e in res:
        assert counts == dict(want) and total == 37
        np.testing.assert_array_equal(e, want_e)
