"""Global-qubit slicing (cfg 5 path) vs the CPU oracle.

* CPU: the sliced executor with a numpy slice backend (test-only stand-in for the
  device kernels) and the in-process transport -- exchanges, qubit relabeling, the
  global Pauli frame and slice-summed measurement give the oracle's trajectories.
* CPU, gloo world size 2: one slice per rank, half-buffer exchanges over
  torch.distributed send/recv, rank-ordered probability sums.
* GPU: the product backend (C-ABI kernels) with the single-device transport.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import sim_port as P
from paper_2604_11599_b200 import ir, sim, sliced, workloads


class NumpyBackend:
    def new_slice(self, L, one):
        a = np.zeros(1 << L, dtype=np.complex128)
        if one:
            a[0] = 1.0
        return a

    def apply(self, a, base, m, t, ctrl):
        idx = np.arange(a.size)
        cm = sum(1 << q for q, _ in ctrl)
        cv = sum((1 << q) for q, pol in ctrl if pol)
        sel = (((idx >> t) & 1) == 0) & ((idx & cm) == cv)
        i0 = idx[sel]
        i1 = i0 | (1 << t)
        a0, a1 = a[i0].copy(), a[i1].copy()
        a[i0] = m[0, 0] * a0 + m[0, 1] * a1
        a[i1] = m[1, 0] * a0 + m[1, 1] * a1

    def scale(self, a, c):
        a *= c

    def prob1(self, a, q):
        if q < 0:
            return float(np.sum(a.real**2 + a.imag**2))
        ones = (np.arange(a.size) >> q) & 1 == 1
        return float(np.sum(a.real[ones] ** 2 + a.imag[ones] ** 2))

    def collapse(self, a, q, outcome, scale, flip):
        idx = np.arange(a.size)
        i0 = idx[((idx >> q) & 1) == 0]
        i1 = i0 | (1 << q)
        keep = (a[i1] if outcome else a[i0]) * scale
        a[i0] = 0
        a[i1] = 0
        if outcome and not flip:
            a[i1] = keep
        else:
            a[i0] = keep

    def view(self, a):
        import torch

        return torch.from_numpy(a.view(np.float64))

    def sync_after_transport(self, a):
        pass

    def to_numpy(self, a):
        return a.copy()


def _circuits():
    out = []
    for seed in range(3):
        _, k = workloads.rdc_circuit(n=7, depth=12, every=4, seed=50 + seed)
        out.append(k)
    out.append(workloads.random_dynamic(6, 40, seed=5))
    out.append(workloads.random_static(6, 60, seed=6, max_controls=2))
    _, k = workloads.dyn_circuit(n=6, layers=6, every=3, nmeas=2, seed=4)
    out.append(k)
    return out


@pytest.mark.parametrize("G", [1, 2, 3])
def test_sliced_numpy_matches_oracle(G):
    for k in _circuits():
        b = ir.bind(k, [])
        for shot in range(3):
            try:
                rs, ref = P.trajectory(b, P.PortRng.for_shot(9, shot))
            except P.DegenerateBranch:
                continue
            store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(9, shot), G,
                                                     backend=NumpyBackend(),
                                                     transport=sliced.LocalTransport(2**G))
            assert store.key() == rs.key()
            np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        res = []
        for k in _circuits()[:3]:
            b = ir.bind(k, [])
            store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(9, 1), 1, backend=NumpyBackend(),
                                                     transport=sliced.DistTransport())
            res.append((store.key(), st.perm, st.gframe, st.slices[rank].tolist()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sliced_gloo_world_size_2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for ci, k in enumerate(_circuits()[:3]):
        b = ir.bind(k, [])
        rs, ref = P.trajectory(b, P.PortRng.for_shot(9, 1))
        key0, perm, gframe, s0 = got[0][ci]
        key1, _, _, s1 = got[1][ci]
        assert key0 == key1 == rs.key()
        # reassemble the logical vector from the two ranks' slices
        st = sliced.SlicedState.__new__(sliced.SlicedState)
        st.n, st.G, st.L, st.perm, st.gframe = k.qubit_count, 1, k.qubit_count - 1, perm, gframe
        st.backend = NumpyBackend()
        st.slices = {0: np.array(s0), 1: np.array(s1)}
        np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 3])
def test_sliced_gpu_matches_oracle(G):
    for k in _circuits():
        b = ir.bind(k, [])
        rs, ref = P.trajectory(b, P.PortRng.for_shot(9, 0))
        store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(9, 0), G)
        assert store.key() == rs.key()
        np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-10)
    # a 16-qubit RDC with 3 global qubits (8 slices of 2^13)
    _, k = workloads.rdc_circuit(n=16, depth=20, every=10, seed=16)
    b = ir.bind(k, [])
    rs, ref = P.trajectory(b, P.PortRng.for_shot(1234, 0))
    store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(1234, 0), 3)
    assert store.key() == rs.key()
    np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-10)
    assert st.exchanges > 0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [6, 14])
def test_apply_tape_in_place(n):
    """qsb_apply_tape runs a gates-only tape on an arbitrary existing state (the fused
    path of the sliced executor): equal to the oracle's gate-by-gate application."""
    import ctypes

    from paper_2604_11599_b200 import _lib

    k = workloads.random_static(n, 120, seed=n, max_controls=2)
    rng = np.random.default_rng(n)
    a0 = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    a0 /= np.linalg.norm(a0)
    st = sim.StateVector(n, a0)
    ctx = st._ctx
    recs = sim.tape_records(k)
    tape = ctypes.c_void_p()
    _lib.check(ctx.lib.qsb_tape_create(ctx.handle, _lib.ptr(recs), len(recs), n, 0, 0, ctypes.byref(tape)))
    try:
        _lib.check(ctx.lib.qsb_apply_tape(tape, None, st._device()))
    finally:
        ctx.lib.qsb_tape_destroy(tape)
    ref = P.PortState(n, a0.copy())
    for op in k.body:
        P.gate_pass(ref, op)
    np.testing.assert_allclose(st.amps, ref.amps, atol=1e-10)


@pytest.mark.gpu
def test_sliced_fused_equals_per_op():
    _, k = workloads.rdc_circuit(n=16, depth=20, every=10, seed=16)
    b = ir.bind(k, [])
    out = []
    for fuse in (False, True):
        store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(1234, 0), 3,
                                                 backend=sliced.GpuSliceBackend(fuse=fuse))
        out.append((store.key(), st.gather()))
    assert out[0][0] == out[1][0]
    np.testing.assert_allclose(out[0][1], out[1][1], atol=1e-12)
