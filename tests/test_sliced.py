"""Global-qubit slicing (cfg 5 path) vs the CPU oracle.

* CPU: the sliced executor with a numpy slice backend (test-only stand-in for the
  device kernels) and the in-process transport -- exchanges, qubit relabeling, the
  global Pauli frame and slice-summed measurement give the oracle's trajectories.
* CPU, gloo world size 2 / 4 / 8: one slice per rank, remaps of 1-3 positions as
  packed region send/recv among each group of ranks over torch.distributed,
  rank-ordered probability sums.
* GPU: the product backend (C-ABI kernels) with the single-device transport, the remap
  kernels against the numpy restatement, the NCCL data plane through a 1-rank
  communicator.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import sim_port as P
from paper_2604_11599_b200 import ir, sim, sliced, workloads


class _NpCtl:
    """Host model of the device SliceCtl (test-only): reference arithmetic of
    sim.py:230-276 on the guard stack, the classical store and the RNG words."""

    def __init__(self, nslices, nbits, words):
        self.rng = sim.RngStream(0)
        self.rng.s0, self.rng.s1, self.rng.s2, self.rng.s3 = (int(w) for w in words)
        self.bits = [0] * max(1, (nbits + 63) // 64)
        self.partials = np.zeros(nslices)
        self.depth = self.active = self.status = self.draws = 0
        self.outcome, self.scale = -1, 1.0

    def live(self):
        return self.status == 0 and self.active == self.depth


def _pred(bits, rec):
    v = 0
    for j in range(int(rec["pred_width"])):
        f = int(rec["pred_bit"]) + j
        v = (v << 1) | ((bits[f >> 6] >> (f & 63)) & 1)
    rhs, cmp = int(rec["pred_rhs"]), int(rec["pred_cmp"])
    return [v == rhs, v != rhs, v < rhs, v <= rhs, v > rhs, v >= rhs, v != 0][cmp]


class NumpyBackend:
    """numpy stand-in for GpuSliceBackend's primitives (test-only)."""

    def new_slice(self, L, one):
        a = np.zeros(1 << L, dtype=np.complex128)
        if one:
            a[0] = 1.0
        return a

    def new_ctl(self, nslices, nbits, words):
        return _NpCtl(nslices, nbits, words)

    def gate(self, a, ctl, base, m, t, ctrl, guarded):
        if not ctl.live():
            return
        idx = np.arange(a.size)
        cm = sum(1 << q for q, _ in ctrl)
        cv = sum((1 << q) for q, pol in ctrl if pol)
        sel = (((idx >> t) & 1) == 0) & ((idx & cm) == cv)
        i0 = idx[sel]
        i1 = i0 | (1 << t)
        a0, a1 = a[i0].copy(), a[i1].copy()
        a[i0] = m[0, 0] * a0 + m[0, 1] * a1
        a[i1] = m[1, 0] * a0 + m[1, 1] * a1

    def scale(self, a, ctl, c):
        if ctl.live():
            a *= c

    def guard(self, ctl, kind, rec=None):
        if kind == "if":
            act = ctl.active == ctl.depth
            taken = act and _pred(ctl.bits, rec[0])
            ctl.depth += 1
            if taken:
                ctl.active = ctl.depth
        elif kind == "else":
            if ctl.active == ctl.depth:
                ctl.active = ctl.depth - 1
            elif ctl.active == ctl.depth - 1:
                ctl.active = ctl.depth
        else:
            if ctl.active == ctl.depth:
                ctl.active -= 1
            ctl.depth -= 1

    def prob1(self, a, ctl, q, select, index):
        if not select:
            ctl.partials[index] = 0.0
        elif q < 0:
            ctl.partials[index] = float(np.sum(a.real**2 + a.imag**2))
        else:
            ones = (np.arange(a.size) >> q) & 1 == 1
            ctl.partials[index] = float(np.sum(a.real[ones] ** 2 + a.imag[ones] ** 2))

    def decide(self, ctl, reset, bit):
        if not ctl.live():
            ctl.outcome = -1
            return
        p1 = 0.0
        for v in ctl.partials:
            p1 += v
        u = ctl.rng.uniform()
        ctl.draws += 1
        o = 1 if u < p1 else 0
        pout = p1 if o else 1.0 - p1
        ctl.outcome = o
        if pout < 1e-15:
            ctl.status = 3
            return
        ctl.scale = 1.0 / np.sqrt(pout)
        if not reset:
            ctl.bits[bit >> 6] = (ctl.bits[bit >> 6] & ~(1 << (bit & 63))) | (o << (bit & 63))

    def collapse(self, a, ctl, q, gbit, flip):
        if ctl.outcome < 0 or ctl.status:
            return
        o, s = ctl.outcome, ctl.scale
        if q < 0:
            a *= s if gbit == o else 0.0
            return
        idx = np.arange(a.size)
        i0 = idx[((idx >> q) & 1) == 0]
        i1 = i0 | (1 << q)
        keep = (a[i1] if o else a[i0]) * s
        a[i0] = 0
        a[i1] = 0
        if o and not flip:
            a[i1] = keep
        else:
            a[i0] = keep

    def remap_local(self, group, lposs):
        """(slice y, local bits x at lposs) -> (slice x, local bits y), in place."""
        old = [a.copy() for a in group]
        for y, a in enumerate(old):
            for x in range(len(group)):
                group[x][self._region(a, lposs, y)] = a[self._region(a, lposs, x)]

    @staticmethod
    def _spread(lposs, x):
        return sum(((x >> i) & 1) << p for i, p in enumerate(lposs))

    def _region(self, a, lposs, x):
        idx = np.arange(a.size)
        mask = self._spread(lposs, (1 << len(lposs)) - 1)
        return idx[(idx & mask) == self._spread(lposs, x)]

    def pack_sub(self, a, lposs, x):
        return a[self._region(a, lposs, x)].copy()

    def unpack_sub(self, a, lposs, x, data):
        a[self._region(a, lposs, x)] = data

    def partials(self, ctl):
        return ctl.partials

    def read_ctl(self, ctl, nwords):
        r = ctl.rng
        return (np.array(ctl.bits, dtype=np.uint64), ctl.status, ctl.draws,
                np.array([r.s0, r.s1, r.s2, r.s3], dtype=np.uint64))

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


@pytest.mark.parametrize("G,group", [(1, None), (2, None), (3, None), (3, 1), (3, 2)])
def test_sliced_numpy_matches_oracle(G, group):
    for k in _circuits():
        b = ir.bind(k, [])
        for shot in range(3):
            prng = P.PortRng.for_shot(9, shot)
            try:
                rs, ref = P.trajectory(b, prng)
            except P.DegenerateBranch:
                continue
            rng = sim.RngStream.for_shot(9, shot)
            store, st = sliced.run_trajectory_sliced(b, rng, G, backend=NumpyBackend(),
                                                     transport=sliced.LocalTransport(2**G), group=group)
            assert store.key() == rs.key()
            assert rng.next_u64() == prng.next_u64()  # advanced by exactly the uniforms consumed
            np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        G = world.bit_length() - 1
        for k in _circuits()[:4]:
            b = ir.bind(k, [])
            try:
                store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(9, 1), G, backend=NumpyBackend(),
                                                         transport=sliced.DistTransport())
                res.append((store.key(), st.perm, st.slices[rank].tolist(), st.exchanges))
            except Exception as e:  # DegenerateNorm must agree on every rank
                res.append((type(e).__name__, None, None, None))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sliced_gloo_ranks(world):
    """One slice per rank (world 2: 1 global qubit, world 4: 2, world 8: 3), remaps of
    up to G positions as packed send/recv to every peer of the rank's group, the
    partials all-gathered and summed in slice order on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    G = world.bit_length() - 1
    for ci, k in enumerate(_circuits()[:4]):
        b = ir.bind(k, [])
        try:
            rs, ref = P.trajectory(b, P.PortRng.for_shot(9, 1))
        except P.DegenerateBranch:
            assert all(got[r][ci][0] == "DegenerateNorm" for r in range(world))
            continue
        keys = {got[r][ci][0] for r in range(world)}
        assert keys == {rs.key()}
        perm = got[0][ci][1]
        # reassemble the logical vector from the ranks' slices
        st = sliced.SlicedState.__new__(sliced.SlicedState)
        st.n, st.G, st.L, st.perm = k.qubit_count, G, k.qubit_count - G, perm
        st.backend = NumpyBackend()
        st.slices = {r: np.array(got[r][ci][2]) for r in range(world)}
        np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-12)


def test_lookahead_plan_fewer_exchanges():
    """Belady eviction (farthest next local use) against the round-1 rule (always the
    top local position) on RDC26 depth 40 with 3 global qubits: fewer exchanges; grouped
    remaps of up to 3 positions: fewer steps and < 80 % of the pairwise volume; the same
    trajectory every way (numpy backend, RDC10 twin)."""
    _, k = workloads.rdc_circuit(n=26, depth=40, every=20, seed=30200)
    b = ir.bind(k, [])
    old = sliced.plan_slices(k, b.values, 3, lookahead=False).exchanges
    new = sliced.plan_slices(k, b.values, 3, lookahead=True, group=1).exchanges
    assert new < old, (new, old)
    # grouped remaps (up to 3 positions per all-to-all): fewer steps and less volume
    pair = sliced.plan_slices(k, b.values, 3, group=1)
    grp = sliced.plan_slices(k, b.values, 3)
    assert pair.exchanges == new and pair.volume == 0.5 * new
    assert grp.exchanges < pair.exchanges and grp.volume < 0.8 * pair.volume, (grp.exchanges, grp.volume, pair.volume)
    assert any(len(s[1]) == 3 for s in grp.steps if s[0] == "xchg")
    _, k = workloads.rdc_circuit(n=10, depth=40, every=20, seed=10)
    b = ir.bind(k, [])
    out = []
    for la, group in ((False, None), (True, 1), (True, None)):
        store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(5, 0), 3, backend=NumpyBackend(),
                                                 transport=sliced.LocalTransport(8), lookahead=la, group=group)
        out.append((store.key(), st.gather()))
    for key, amps in out[1:]:
        assert key == out[0][0]
        np.testing.assert_allclose(amps, out[0][1], atol=1e-12)


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


@pytest.mark.gpu
def test_nccl_exchange_and_allgather_single_gpu():
    """The NCCL data plane of the sliced engine on one GPU: a 1-rank communicator whose
    exchange with a self-peer swaps the halves of two slices exactly like the in-place
    single-device kernel (pack -> chunked ncclSend / ncclRecv -> unpack, small chunks so
    several are in flight), and an in-place all-gather of the partial slot."""
    import ctypes

    from paper_2604_11599_b200 import _lib

    ctx = _lib.context()
    uid = np.zeros(128, dtype=np.uint8)
    _lib.check(ctx.lib.qsb_comm_unique_id(_lib.ptr(uid)))
    comm = ctypes.c_void_p()
    _lib.check(ctx.lib.qsb_comm_init(ctx.handle, _lib.ptr(uid), 0, 1, ctypes.byref(comm)))
    try:
        _lib.check(ctx.lib.qsb_comm_set_chunk(comm, 64 << 10))
        rng = np.random.default_rng(3)
        L = 16
        for prec in ("c128", "c64"):
            for pos in (0, 7, L - 1):
                a0 = rng.normal(size=1 << L) + 1j * rng.normal(size=1 << L)
                b0 = rng.normal(size=1 << L) + 1j * rng.normal(size=1 << L)
                ref_a, ref_b = sim.StateVector(L, a0, precision=prec), sim.StateVector(L, b0, precision=prec)
                _lib.check(ctx.lib.qsb_slice_exchange_local(ref_a._device(), ref_b._device(), pos))
                a, b = sim.StateVector(L, a0, precision=prec), sim.StateVector(L, b0, precision=prec)
                a2, b2 = sim.StateVector(L, a0, precision=prec), sim.StateVector(L, b0, precision=prec)
                # a (global bit 0) -> b2's half, b (global bit 1) -> a2's half, through the self-peer
                _lib.check(ctx.lib.qsb_comm_exchange(comm, a._device(), 0, b2._device(), 1, pos, 0))
                _lib.check(ctx.lib.qsb_comm_exchange(comm, b._device(), 1, a2._device(), 0, pos, 0))
                np.testing.assert_array_equal(a2.amps, ref_a.amps)
                np.testing.assert_array_equal(b2.amps, ref_b.amps)
        out = np.zeros(3, dtype=np.int64)
        ms = ctypes.c_double()
        _lib.check(ctx.lib.qsb_comm_stats(comm, _lib.ptr(out), ctypes.byref(ms)))
        assert out[1] == 12 and out[0] == 6 * (16 + 8) * (1 << (L - 1))
        # partial slot all-gather (1 rank: in place, unchanged)
        ctl = sliced.GpuSliceBackend().new_ctl(1, 4, np.array([1, 2, 3, 4], dtype=np.uint64))
        st = sim.StateVector(L, rng.normal(size=1 << L) + 0j)
        _lib.check(ctx.lib.qsb_slice_prob1(st._device(), ctl.h, 3, 1, 0))
        _lib.check(ctx.lib.qsb_comm_allgather_partials(comm, ctl.h))
        _lib.check(ctx.lib.qsb_slice_decide(ctl.h, _lib.OP_MEASURE, 2))
        bits, status, draws, _ = sliced.GpuSliceBackend().read_ctl(ctl, 1)
        assert status == 0 and draws == 1
    finally:
        ctx.lib.qsb_comm_destroy(comm)


@pytest.mark.gpu
def test_sliced_device_decisions_match_oracle_with_branches():
    """Dynamic circuits with nested if/else, register predicates and resets on the
    sliced device path (decisions, guards and the classical store on the device), all
    slice counts, vs the oracle; the RNG advances by exactly the draws."""
    for seed in range(4):
        k = workloads.random_dynamic(7, 50, seed=70 + seed)
        b = ir.bind(k, [])
        for G in (1, 2, 3):
            prng = P.PortRng.for_shot(3, seed)
            try:
                rs, ref = P.trajectory(b, prng)
            except P.DegenerateBranch:
                with pytest.raises(sim.DegenerateNorm):
                    sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(3, seed), G)
                continue
            rng = sim.RngStream.for_shot(3, seed)
            store, st = sliced.run_trajectory_sliced(b, rng, G)
            assert store.key() == rs.key()
            np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-10)
            assert rng.next_u64() == prng.next_u64()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_remap_kernels_match_numpy(prec):
    """qsb_slice_remap_local (k = 1, 2, 3; positions in pairing order, low and high) and
    the region staging qsb_slice_read_sub / write_sub against the numpy restatement."""
    from paper_2604_11599_b200.errors import BackendError

    be, nb = sliced.GpuSliceBackend(precision=prec), NumpyBackend()
    rng = np.random.default_rng(11)
    L = 12
    dt = np.complex64 if prec == "c64" else np.complex128
    for lposs in ((5,), (0, 11), (7, 1), (3, 0, 9), (11, 6, 2)):
        k = len(lposs)
        host = [(rng.normal(size=1 << L) + 1j * rng.normal(size=1 << L)).astype(dt) for _ in range(1 << k)]
        dev = [sim.StateVector(L, h.astype(np.complex128), precision=prec) for h in host]
        be.remap_local(dev, lposs)
        ref = [h.copy() for h in host]
        nb.remap_local(ref, lposs)
        for d, r in zip(dev, ref):
            np.testing.assert_array_equal(np.asarray(d.amps).astype(dt), r)
        for x in range(1 << k):
            np.testing.assert_array_equal(be.pack_sub(dev[0], lposs, x), nb.pack_sub(ref[0], lposs, x))
        data = (rng.normal(size=1 << (L - k)) + 1j * rng.normal(size=1 << (L - k))).astype(dt)
        be.unpack_sub(dev[1], lposs, (1 << k) - 1, data)
        nb.unpack_sub(ref[1], lposs, (1 << k) - 1, data)
        np.testing.assert_array_equal(np.asarray(dev[1].amps).astype(dt), ref[1])
    with pytest.raises(BackendError):
        be.remap_local(dev[:4], (4, 4))  # repeated local position


@pytest.mark.gpu
def test_nccl_remap_self_peers_and_grouped_sliced_run():
    """qsb_comm_remap through a 1-rank communicator (every peer = this rank: each region
    goes out and comes back through NCCL, chunked, all peers in one group), and a sliced
    RDC16 run with grouped 3-position remaps on one device vs the oracle."""
    import ctypes

    from paper_2604_11599_b200 import _lib

    ctx = _lib.context()
    uid = np.zeros(128, dtype=np.uint8)
    _lib.check(ctx.lib.qsb_comm_unique_id(_lib.ptr(uid)))
    comm = ctypes.c_void_p()
    _lib.check(ctx.lib.qsb_comm_init(ctx.handle, _lib.ptr(uid), 0, 1, ctypes.byref(comm)))
    try:
        _lib.check(ctx.lib.qsb_comm_set_chunk(comm, 16 << 10))
        L = 14
        a0 = np.random.default_rng(4).normal(size=1 << L) + 0j
        st = sim.StateVector(L, a0)
        lp = np.array([2, 13, 7], dtype=np.int32)
        peers = np.zeros(8, dtype=np.int32)
        _lib.check(ctx.lib.qsb_comm_remap(comm, st._device(), 3, _lib.ptr(lp), _lib.ptr(peers), 0))
        np.testing.assert_array_equal(st.amps, a0)
        out = np.zeros(3, dtype=np.int64)
        _lib.check(ctx.lib.qsb_comm_stats(comm, _lib.ptr(out), None))
        assert out[0] == 7 * (1 << (L - 3)) * 16 and out[1] == 1
        bad = np.array([0, 1, 0, 0, 0, 0, 0, 0], dtype=np.int32)  # peer 1 does not exist
        assert ctx.lib.qsb_comm_remap(comm, st._device(), 3, _lib.ptr(lp), _lib.ptr(bad), 0) != 0
    finally:
        ctx.lib.qsb_comm_destroy(comm)
    _, k = workloads.rdc_circuit(n=16, depth=20, every=10, seed=16)
    b = ir.bind(k, [])
    plan = sliced.plan_slices(k, b.values, 3)
    assert any(len(s[1]) == 3 for s in plan.steps if s[0] == "xchg")
    rs, ref = P.trajectory(b, P.PortRng.for_shot(1234, 0))
    store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(1234, 0), 3, plan=plan)
    assert store.key() == rs.key()
    np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-10)


def _gpu_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        G = world.bit_length() - 1
        for k in _circuits()[:4]:
            b = ir.bind(k, [])
            try:
                store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(9, 1), G,
                                                         backend=sliced.GpuSliceBackend(),
                                                         transport=sliced.DistTransport())
                res.append((store.key(), st.perm, np.asarray(st.slices[rank].amps).tolist()))
            except Exception as e:  # DegenerateNorm must agree on every rank
                res.append((type(e).__name__, None, None))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 4])
def test_sliced_device_backend_over_ranks(world):
    """The device slice backend under the multi-rank protocol: one slice per process
    (all on this GPU; the transport stages remap regions and partial slots through the
    host with gloo, so no kernel waits on another rank), remaps of 1-2 positions, device
    decisions from rank-ordered partial sums -- every rank's key and the reassembled
    state vs the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=500) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    G = world.bit_length() - 1
    for ci, k in enumerate(_circuits()[:4]):
        b = ir.bind(k, [])
        try:
            rs, ref = P.trajectory(b, P.PortRng.for_shot(9, 1))
        except P.DegenerateBranch:
            assert all(got[r][ci][0] == "DegenerateNorm" for r in range(world))
            continue
        assert {got[r][ci][0] for r in range(world)} == {rs.key()}
        st = sliced.SlicedState.__new__(sliced.SlicedState)
        st.n, st.G, st.L, st.perm = k.qubit_count, G, k.qubit_count - G, got[0][ci][1]
        st.backend = NumpyBackend()
        st.slices = {r: np.array(got[r][ci][2]) for r in range(world)}
        np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-10)


@pytest.mark.gpu
def test_sliced_complex64_matches_oracle():
    """complex64 slices (grouped remaps, device decisions) vs the complex128 oracle
    within 1e-5 wherever the key agrees; keys agree on these circuits."""
    for k in _circuits()[:4]:
        b = ir.bind(k, [])
        try:
            rs, ref = P.trajectory(b, P.PortRng.for_shot(9, 2))
        except P.DegenerateBranch:
            continue
        store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(9, 2), 3,
                                                 backend=sliced.GpuSliceBackend(precision="c64"))
        assert store.key() == rs.key()
        np.testing.assert_allclose(st.gather(), ref.amps, atol=1e-5)
