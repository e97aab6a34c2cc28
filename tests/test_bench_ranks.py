"""bench.py's multi-rank logic on CPU (gloo, world size 2): disjoint global-shot
ranges per (step, rank), MAX-over-ranks timing, SUM-over-ranks counters, and the
`--gpus N` launcher refusing to run with fewer than N GPUs (no silent 1-rank run)."""

import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402


def test_step_ranges_disjoint_and_complete():
    B, world, steps = 5, 4, 3
    seen = []
    for step in range(steps):
        for rank in range(world):
            lo = bench.step_shot_begin(step, rank, world, B)
            seen.extend(range(lo, lo + B))
    assert sorted(seen) == list(range(steps * world * B))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sim_port as P
        from paper_2604_11599_b200 import ir, workloads

        _, k = workloads.dyn_circuit(n=6, layers=5, every=5, nmeas=2, seed=5)
        b = ir.bind(k, [])
        B, steps = 3, 2
        keys = {}
        for step in range(steps):
            lo = bench.step_shot_begin(step, rank, world, B)
            for s in range(lo, lo + B):
                keys[s] = P.trajectory(b, P.PortRng.for_shot(1234, s))[0].key()
        times, counts = bench.reduce_over_ranks([10.0 + rank, 1.0 - rank * 0.5], [len(keys), 1.0], "cpu")
        parts = [None] * world
        dist.all_gather_object(parts, keys)
        q.put((rank, times, counts, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world_size_2_rank_logic():
    from oracle import sim_port as P
    from paper_2604_11599_b200 import ir, workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    _, k = workloads.dyn_circuit(n=6, layers=5, every=5, nmeas=2, seed=5)
    b = ir.bind(k, [])
    want = {s: P.trajectory(b, P.PortRng.for_shot(1234, s))[0].key() for s in range(12)}
    for rank, times, counts, parts in res:
        assert times == [11.0, 1.0]  # max over ranks
        assert counts == [12.0, 2.0]  # sum over ranks
        merged = {}
        for p in parts:
            assert not (set(p) & set(merged))  # disjoint ranges
            merged.update(p)
        assert merged == want


def test_gpus_flag_refuses_without_enough_gpus():
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("a multi-GPU host would really launch")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "GPU(s) visible" in r.stderr
