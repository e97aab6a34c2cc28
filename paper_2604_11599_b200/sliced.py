"""Global-qubit slicing of one state vector over 2^G slices (BASELINE cfg 5: 34 qubits
complex128 over 8 B200s).

Layout.  The top G *physical* qubit positions are global: slice s holds the 2^L
amplitudes (L = n - G) whose global physical bits equal s.  Logical qubit q lives at
physical position perm[q].  One slice per rank (one GPU per process, NCCL between them)
in production; all slices in one process for the single-device emulation.

Plan (host, static, `plan_slices`).  The kernel IR is flattened (CondBlock -> IF / ELSE /
ENDIF, sim.py:296-301) and the data movement is decided once, before anything runs:
* a gate whose target is local runs on every slice (controls on global positions select
  slices, local controls go to the kernel); a diagonal gate on a global target is a
  per-slice phase;
* a non-diagonal gate (or a reset) on a global position first REMAPS that global
  position with a local one -- together with every other global qubit needed locally
  before the local qubit it would evict (up to G positions in one remap): within each
  group of 2^k slices that differ only in the remapped global bits, the amplitude at
  (slice y, local bits x) moves to (slice x, local bits y) -- grouped NCCL send/recv to
  the 2^k - 1 peers across GPUs, an in-place kernel on one GPU; (1 - 2^-k) of a slice
  per rank instead of k/2 for k pairwise exchanges.  The local positions evicted are the
  ones whose qubits are next needed locally FARTHEST in the future (Belady look-ahead
  over the whole flattened program, branches included) -- not a fixed position;
* swap gates are relabelings of `perm` (no data movement).
Because the plan does not depend on outcomes (a gate in an untaken branch still gets its
exchange -- a relabeling that changes nothing logically), the host never has to wait for
the device.

Execution.  Every classical decision is made on the device (qsb_slice_*: SliceCtl with
the RNG stream, the classical store and the if/else guards): a measurement writes each
slice's partial p1 into a slot of a partials array, the transport all-gathers the slots
(one 8-byte NCCL all-gather per measurement across ranks; nothing on one GPU), the decide
kernel sums them IN SLICE ORDER on every rank, draws u from the shared stream and applies
sim.py:230-259 (u < p1, p0 = 1 - p1, 1e-15, 1/sqrt); the collapse kernels read the
decision.  The host reads the classical store back once, at the end.

Backends: `GpuSliceBackend` (C ABI kernels).  Transports: `LocalTransport` (all slices in
this process), `NcclTransport` (C ABI NCCL communicator: qsb_comm_*), `DistTransport`
(torch.distributed: the protocol tests run it under gloo with a numpy backend).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from .errors import DegenerateNorm
from .ir import op_kind

_DIAG = frozenset(("z", "s", "t", "rz", "p"))


# ---------------------------------------------------------------------------
# static plan
# ---------------------------------------------------------------------------


@dataclass
class SlicePlan:
    n: int
    G: int
    steps: list = field(default_factory=list)  # see plan_slices
    exchanges: int = 0    # remap steps
    volume: float = 0.0   # slices sent per rank over all remaps (sum of 1 - 2^-k)
    final_perm: list = field(default_factory=list)

    @property
    def L(self) -> int:
        return self.n - self.G


def _flatten(ops, out: list, offsets: dict, params) -> None:
    from .sim import gate_matrix

    for op in ops:
        k = op_kind(op)
        if k == "gate":
            if op.base == "swap":
                a, b = op.targets
                if not op.controls:
                    out.append(("swap", a, b))
                    continue
                # Fredkin = CX(b->a) . CCX(ctrls + a -> b) . CX(b->a)
                x = np.array([[0, 1], [1, 0]], dtype=np.complex128)
                out.append(("gate", "x", x, a, ((b, 1),)))
                out.append(("gate", "x", x, b, tuple(op.controls) + ((a, 1),)))
                out.append(("gate", "x", x, a, ((b, 1),)))
                continue
            out.append(("gate", op.base, gate_matrix(op, params), op.targets[0], tuple(op.controls)))
        elif k == "measure":
            base, _ = offsets[op.bit[0]]
            out.append(("measure", op.qubit, base + op.bit[1]))
        elif k == "reset":
            out.append(("reset", op.qubit))
        elif k == "nop":
            continue
        else:
            out.append(("if", op.predicate))
            _flatten(op.then_body, out, offsets, params)
            if op.else_body:
                out.append(("else",))
                _flatten(op.else_body, out, offsets, params)
            out.append(("endif",))


def _needs_local(item) -> int | None:
    """Logical qubit the item needs at a local position, if any."""
    if item[0] == "gate" and item[1] not in _DIAG:
        return item[3]
    if item[0] == "reset":
        return item[1]
    return None


def plan_slices(kernel, params, G: int, lookahead: bool = True, group: int | None = None) -> SlicePlan:
    """Static schedule of a sliced trajectory.  Steps (physical positions):
        ("xchg", gposs, lposs)                       remap: global position gposs[i] <-> local
                                                     position lposs[i], all at once
        ("gate", base, m, tpos, ctrls, guarded)      ctrls: ((pos, pol), ...)
        ("measure", pos, bit) / ("reset", pos)       reset positions are always local
        ("if", pred_record) / ("else",) / ("endif",)
    `lookahead=False` evicts the top local position every time (the round-1 rule).
    `group` = most global positions one remap moves (default G): when a gate needs a
    global qubit, every other global qubit that is needed locally BEFORE the local qubit
    it would evict comes along in the same remap -- one all-to-all among 2^k ranks moves
    (1 - 2^-k) of a slice per rank, against k/2 for k separate pairwise exchanges."""
    from . import _lib
    from .sim import _classical_offsets, _pred_record

    n = int(kernel.qubit_count)
    if not 0 <= G < n:
        raise ValueError("need 0 <= G < n")
    L = n - G
    kmax = G if group is None else max(1, min(int(group), G))
    if not lookahead:
        kmax = 1
    offsets = _classical_offsets([(nm, int(w)) for nm, w in kernel.classical_layout])
    items: list = []
    _flatten(kernel.body, items, offsets, params)
    # next index at which each logical qubit must be local (Belady distances)
    INF = len(items) + 1
    next_need = [[INF] * n for _ in range(len(items) + 1)] if lookahead else None
    if lookahead:
        cur = [INF] * n
        for i in range(len(items) - 1, -1, -1):
            q = _needs_local(items[i])
            if q is not None:
                cur[q] = i
            next_need[i] = list(cur)
    perm = list(range(n))  # logical -> physical
    where = list(range(n))  # physical -> logical
    plan = SlicePlan(n, G)
    depth = 0
    for i, it in enumerate(items):
        kind = it[0]
        if kind == "swap":
            a, b = it[1], it[2]
            perm[a], perm[b] = perm[b], perm[a]
            where[perm[a]], where[perm[b]] = a, b
            continue
        if kind == "if":
            rec = np.zeros(1, dtype=_lib.OP_DTYPE)
            _pred_record(rec[0], it[1], offsets)
            plan.steps.append(("if", rec))
            depth += 1
            continue
        if kind == "else":
            plan.steps.append(("else",))
            continue
        if kind == "endif":
            plan.steps.append(("endif",))
            depth -= 1
            continue
        q = _needs_local(it)
        if q is not None and perm[q] >= L:
            busy = set()
            if kind == "gate":
                busy = {perm[c] for c, _ in it[4]}  # keep the gate's own controls local if possible
            if lookahead:
                nxt = next_need[i + 1] if i + 1 < len(items) else [INF] * n
                cands = sorted(range(L), key=lambda p: (nxt[where[p]], p not in busy, p), reverse=True)
                # the other global qubits, soonest needed first, each paired with the next
                # eviction candidate if it is needed before that candidate
                others = sorted((nxt[where[g]], g) for g in range(L, n) if g != perm[q])
                gposs, lposs = [perm[q]], [cands[0]]
                for need, g in others:
                    if len(gposs) >= kmax or need >= INF:
                        break
                    c = cands[len(lposs)]
                    if need < nxt[where[c]]:
                        gposs.append(g)
                        lposs.append(c)
            else:
                gposs, lposs = [perm[q]], [L - 1]
            plan.steps.append(("xchg", tuple(gposs), tuple(lposs)))
            plan.exchanges += 1
            plan.volume += 1.0 - 0.5 ** len(gposs)
            for g, lp in zip(gposs, lposs):
                qg, ql = where[g], where[lp]
                perm[qg], perm[ql] = lp, g
                where[lp], where[g] = qg, ql
        if kind == "gate":
            _, base, m, t, ctrls = it
            plan.steps.append(("gate", base, m, perm[t], tuple((perm[c], pol) for c, pol in ctrls), depth > 0))
        elif kind == "measure":
            plan.steps.append(("measure", perm[it[1]], it[2]))
        else:
            plan.steps.append(("reset", perm[it[1]]))
    plan.final_perm = perm
    return plan


# ---------------------------------------------------------------------------
# device backend (C ABI)
# ---------------------------------------------------------------------------


class GpuSliceBackend:
    """Slices are device StateVectors; every primitive is an asynchronous C-ABI call on
    the context's stream.  Unguarded local gates between two other steps are queued per
    slice and run as ONE fused tape (`qsb_apply_tape`: the streaming engine's
    register-blocked passes, in place) for slices of >= FUSE_MIN_LOCAL qubits; guarded
    gates (inside an if/else) run one by one with the device guard check."""

    FUSE_MIN_LOCAL = 24  # below: a slice pass is cheaper than building a fused tape

    def __init__(self, precision=None, device=None, fuse: bool | None = None):
        self.precision = precision
        self.device = device
        self.fuse = fuse
        self._queue: dict = {}  # id(slice) -> (slice, [qsb_op records])

    @staticmethod
    def _lib():
        from . import _lib

        return _lib

    def new_slice(self, L: int, initial_one: bool):
        from . import sim

        st = sim.StateVector.zero(L, precision=self.precision, device=self.device)
        if not initial_one:
            _l = self._lib()
            _l.check(st._ctx.lib.qsb_state_scale(st._device(), 0.0, 0.0))
        return st

    def new_ctl(self, nslices: int, nbits: int, rng_words, device_ctx=None):
        _l = self._lib()
        ctx = _l.context(self.device)
        h = ctypes.c_void_p()
        w = np.ascontiguousarray(rng_words, dtype=np.uint64)
        _l.check(ctx.lib.qsb_slice_ctl_create(ctx.handle, nslices, nbits, 0, 0, _l.ptr(w), ctypes.byref(h)))
        return _Ctl(ctx, h, nslices)

    def flush(self, st=None) -> None:
        _l = self._lib()
        keys = [id(st)] if st is not None else list(self._queue)
        for key in keys:
            item = self._queue.pop(key, None)
            if item is None:
                continue
            sl, recs = item
            ops = np.concatenate(recs)
            ctx = sl._ctx
            tape = ctypes.c_void_p()
            ctx.set_option("jit", 0)
            try:
                _l.check(ctx.lib.qsb_tape_create(ctx.handle, _l.ptr(ops), len(ops), sl.n, 0, 0, ctypes.byref(tape)))
                try:
                    _l.check(ctx.lib.qsb_apply_tape(tape, None, sl._device()))
                finally:
                    ctx.lib.qsb_tape_destroy(tape)
            finally:
                ctx.set_option("jit", 1)

    @staticmethod
    def _record(base, m, t, ctrl_local):
        from . import _lib

        rec = np.zeros(1, dtype=_lib.OP_DTYPE)
        r = rec[0]
        r["kind"] = _lib.OP_GATE
        r["base"] = _lib.BASES[base]  # selects the update class (perm / anti / diag / dense)
        r["ntargets"] = 1
        r["target"][0] = t
        cm = cv = 0
        for q, pol in ctrl_local:
            cm |= 1 << q
            cv |= (1 << q) if pol else 0
        r["ctrl_mask"], r["ctrl_val"] = cm, cv
        r["angle_slot"][:] = -1
        rec["mat"][0][:] = [m[0, 0].real, m[0, 0].imag, m[0, 1].real, m[0, 1].imag,
                            m[1, 0].real, m[1, 0].imag, m[1, 1].real, m[1, 1].imag]
        rec["has_matrix"] = 1
        return rec

    def gate(self, st, ctl, base, m, t, ctrl_local, guarded: bool):
        rec = self._record(base, m, t, ctrl_local)
        if not guarded and (self.fuse or (self.fuse is None and st.n >= self.FUSE_MIN_LOCAL)):
            self._queue.setdefault(id(st), (st, []))[1].append(rec)
            return
        self.flush(st)
        _l = self._lib()
        _l.check(st._ctx.lib.qsb_slice_gate(st._device(), ctl.h, _l.ptr(rec)))

    def scale(self, st, ctl, c: complex):
        self.flush(st)
        c = complex(c)
        self._lib().check(st._ctx.lib.qsb_slice_scale(st._device(), ctl.h, c.real, c.imag))

    def guard(self, ctl, kind: str, rec=None):
        _l = self._lib()
        if rec is None:
            rec = np.zeros(1, dtype=_l.OP_DTYPE)
            rec["kind"] = _l.OP_ELSE if kind == "else" else _l.OP_ENDIF
        _l.check(ctl.ctx.lib.qsb_slice_guard(ctl.h, _l.ptr(rec)))

    def prob1(self, st, ctl, q: int, select: bool, index: int):
        self.flush(st)
        self._lib().check(st._ctx.lib.qsb_slice_prob1(st._device(), ctl.h, int(q), 1 if select else 0, int(index)))

    def decide(self, ctl, reset: bool, bit: int):
        _l = self._lib()
        _l.check(ctl.ctx.lib.qsb_slice_decide(ctl.h, _l.OP_RESET if reset else _l.OP_MEASURE, int(bit)))

    def collapse(self, st, ctl, q: int, gbit: int, flip: bool):
        self.flush(st)
        self._lib().check(st._ctx.lib.qsb_slice_collapse(st._device(), ctl.h, int(q), int(gbit), 1 if flip else 0))

    def exchange_local(self, a, b, pos: int):
        self.flush(a)
        self.flush(b)
        self._lib().check(a._ctx.lib.qsb_slice_exchange_local(a._device(), b._device(), int(pos)))

    def remap_local(self, group, lposs):
        """Remap len(lposs) global positions across the 2^k slices `group` (index = the
        remapped global bits) in one in-place kernel."""
        for sl in group:
            self.flush(sl)
        _l = self._lib()
        hs = (ctypes.c_void_p * len(group))(*[sl._device().value for sl in group])
        lp = np.array(lposs, dtype=np.int32)
        _l.check(group[0]._ctx.lib.qsb_slice_remap_local(hs, len(lposs), _l.ptr(lp)))

    def pack_sub(self, st, lposs, x: int) -> np.ndarray:
        self.flush(st)
        _l = self._lib()
        out = np.empty(1 << (st.n - len(lposs)), dtype=np.complex64 if st.precision == "c64" else np.complex128)
        lp = np.array(lposs, dtype=np.int32)
        _l.check(st._ctx.lib.qsb_slice_read_sub(st._device(), len(lposs), _l.ptr(lp), int(x), _l.ptr(out)))
        return out

    def unpack_sub(self, st, lposs, x: int, data) -> None:
        self.flush(st)
        _l = self._lib()
        d = np.ascontiguousarray(data, dtype=np.complex64 if st.precision == "c64" else np.complex128)
        lp = np.array(lposs, dtype=np.int32)
        _l.check(st._ctx.lib.qsb_slice_write_sub(st._device(), len(lposs), _l.ptr(lp), int(x), _l.ptr(d)))

    def partials(self, ctl) -> np.ndarray:
        """Host copy of the partial slots (DistTransport stages the all-gather through
        the host; `set_partials` writes them back)."""
        _l = self._lib()
        out = np.zeros(ctl.nslices, dtype=np.float64)
        _l.check(ctl.ctx.lib.qsb_slice_partials(ctl.h, _l.ptr(out), None))
        return out

    def set_partials(self, ctl, values) -> None:
        _l = self._lib()
        v = np.ascontiguousarray(values, dtype=np.float64)
        _l.check(ctl.ctx.lib.qsb_slice_partials(ctl.h, None, _l.ptr(v)))

    def read_ctl(self, ctl, nwords: int):
        _l = self._lib()
        bits = np.zeros(max(1, nwords), dtype=np.uint64)
        rng = np.zeros(4, dtype=np.uint64)
        status, draws = ctypes.c_int32(), ctypes.c_int32()
        _l.check(ctl.ctx.lib.qsb_slice_ctl_read(ctl.h, _l.ptr(bits), ctypes.byref(status), ctypes.byref(draws),
                                                _l.ptr(rng)))
        return bits, int(status.value), int(draws.value), rng

    def to_numpy(self, st) -> np.ndarray:
        self.flush(st)
        return np.array(st.amps)


class _Ctl:
    """Device SliceCtl handle (destroyed with the object)."""

    def __init__(self, ctx, h, nslices: int = 1):
        import weakref

        self.ctx, self.h, self.nslices = ctx, h, nslices
        self._fin = weakref.finalize(self, ctx.lib.qsb_slice_ctl_destroy, h)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------


class LocalTransport:
    """All slices in this process (single-device emulation of 2^G ranks): the partial
    slots are already side by side, a remap is one in-place kernel per group of 2^k
    slices."""

    def __init__(self, nslices: int):
        self.nslices = nslices
        self.owned = list(range(nslices))

    def allgather(self, backend, ctl) -> None:
        return None

    def exchange(self, backend, slices, groups, lposs):
        for g in groups:
            backend.remap_local([slices[m] for m in g], lposs)


class NcclTransport:
    """One slice per rank; the C-ABI NCCL communicator (qsb_comm_*) on the context's
    stream: a remap is chunked, grouped ncclSend/ncclRecv of the packed regions to the
    2^k - 1 peers of this rank's group, the partials an in-place ncclAllGather.  The
    unique id is broadcast over the default torch.distributed group (the only host-side
    collective, once)."""

    def __init__(self, device=None, chunk_bytes: int | None = None):
        import torch.distributed as dist

        from . import _lib

        self.rank, self.nslices = dist.get_rank(), dist.get_world_size()
        self.owned = [self.rank]
        self.ctx = _lib.context(device)
        uid = np.zeros(128, dtype=np.uint8)
        if self.rank == 0:
            _lib.check(self.ctx.lib.qsb_comm_unique_id(_lib.ptr(uid)))
        obj = [uid.tobytes()]
        dist.broadcast_object_list(obj, src=0)
        uid = np.frombuffer(obj[0], dtype=np.uint8).copy()
        h = ctypes.c_void_p()
        _lib.check(self.ctx.lib.qsb_comm_init(self.ctx.handle, _lib.ptr(uid), self.rank, self.nslices, ctypes.byref(h)))
        self.h = h
        if chunk_bytes:
            _lib.check(self.ctx.lib.qsb_comm_set_chunk(h, int(chunk_bytes)))

    def allgather(self, backend, ctl) -> None:
        from . import _lib

        _lib.check(self.ctx.lib.qsb_comm_allgather_partials(self.h, ctl.h))

    def exchange(self, backend, slices, groups, lposs):
        from . import _lib

        for g in groups:
            if self.rank not in g:
                continue
            st = slices[self.rank]
            backend.flush(st)
            peers = np.array(g, dtype=np.int32)
            lp = np.array(lposs, dtype=np.int32)
            _lib.check(self.ctx.lib.qsb_comm_remap(self.h, st._device(), len(lposs), _lib.ptr(lp), _lib.ptr(peers),
                                                   g.index(self.rank)))

    def stats(self) -> dict:
        from . import _lib

        out = np.zeros(3, dtype=np.int64)
        ms = ctypes.c_double()
        _lib.check(self.ctx.lib.qsb_comm_stats(self.h, _lib.ptr(out), ctypes.byref(ms)))
        return {"bytes_sent": int(out[0]), "exchanges": int(out[1]), "allgathers": int(out[2]),
                "last_exchange_ms": ms.value}

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.qsb_comm_destroy(self.h)
            self.h = None


class DistTransport:
    """One slice per rank over torch.distributed (the protocol of NcclTransport with
    host tensors: gloo in the CPU tests, and the device backend staged through the
    host).  The backend provides `partials(ctl)` (+ `set_partials` for device slots) and
    `pack_sub` / `unpack_sub` of a slice's remap regions."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.nslices = dist.get_world_size()
        self.owned = [self.rank]

    def allgather(self, backend, ctl) -> None:
        import torch

        part = backend.partials(ctl)
        out = [torch.zeros(1, dtype=torch.float64) for _ in range(self.nslices)]
        self.dist.all_gather(out, torch.tensor([float(part[self.rank])], dtype=torch.float64))
        for s in range(self.nslices):
            part[s] = float(out[s][0])
        if hasattr(backend, "set_partials"):  # device slots: write the gathered values back
            backend.set_partials(ctl, part)

    def exchange(self, backend, slices, groups, lposs):
        import torch

        dist = self.dist
        for g in groups:
            if self.rank not in g:
                continue
            st = slices[self.rank]
            me = g.index(self.rank)
            sends, recvs, ops = {}, {}, []
            dtype = None
            for x, peer in enumerate(g):
                if x == me:
                    continue
                data = np.ascontiguousarray(backend.pack_sub(st, lposs, x))
                dtype = data.dtype  # the slice's precision travels as raw bytes
                sends[x] = torch.from_numpy(data.view(np.uint8).copy())
                recvs[x] = torch.empty_like(sends[x])
                ops += [dist.P2POp(dist.isend, sends[x], peer), dist.P2POp(dist.irecv, recvs[x], peer)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            for x, buf in recvs.items():
                backend.unpack_sub(st, lposs, x, buf.numpy().view(dtype))


# ---------------------------------------------------------------------------
# the sliced executor
# ---------------------------------------------------------------------------


class SlicedState:
    """The slices owned by this process plus the layout (`perm`: logical qubit ->
    physical position)."""

    def __init__(self, n: int, G: int, backend, transport):
        self.n, self.G, self.L = n, G, n - G
        self.backend, self.transport = backend, transport
        self.perm = list(range(n))
        self.slices = {s: backend.new_slice(self.L, s == 0) for s in transport.owned}
        self.exchanges = 0

    def gbit(self, s: int, pos: int) -> int:
        return (s >> (pos - self.L)) & 1

    def gather(self) -> np.ndarray:
        """Logical amplitude vector (all slices must be local to this process)."""
        out = np.zeros(1 << self.n, dtype=np.complex128)
        local_idx = np.arange(1 << self.L)
        for s, st in self.slices.items():
            a = self.backend.to_numpy(st)
            phys = (s << self.L) | local_idx
            logical = np.zeros_like(phys)
            for q in range(self.n):
                logical |= ((phys >> self.perm[q]) & 1) << q
            out[logical] = a
        return out


def execute(plan: SlicePlan, st: SlicedState, ctl) -> None:
    """Enqueue a planned trajectory (nothing is read back)."""
    be, tr, L = st.backend, st.transport, st.L
    for step in plan.steps:
        kind = step[0]
        if kind == "gate":
            _, base, m, t, ctrls, guarded = step
            local = [(p, pol) for p, pol in ctrls if p < L]
            glob = [(p, pol) for p, pol in ctrls if p >= L]
            for s, sl in st.slices.items():
                if any(st.gbit(s, p) != pol for p, pol in glob):
                    continue
                if t < L:
                    be.gate(sl, ctl, base, m, t, local, guarded)
                    continue
                d = m[1, 1] if st.gbit(s, t) else m[0, 0]  # diagonal on a global target
                if d == 1:
                    continue
                if not local:
                    be.scale(sl, ctl, d)
                else:  # a phase on the first local control, the rest stay controls
                    (c, pol), rest = local[0], local[1:]
                    dm = np.array([[1, 0], [0, d]] if pol else [[d, 0], [0, 1]], dtype=np.complex128)
                    be.gate(sl, ctl, "rz", dm, c, rest, guarded)
        elif kind in ("measure", "reset"):
            p = step[1]
            for s, sl in st.slices.items():
                if p < L:
                    be.prob1(sl, ctl, p, True, s)
                else:
                    be.prob1(sl, ctl, -1, st.gbit(s, p) == 1, s)
            tr.allgather(be, ctl)
            be.decide(ctl, kind == "reset", step[2] if kind == "measure" else 0)
            for s, sl in st.slices.items():
                if p < L:
                    be.collapse(sl, ctl, p, 0, kind == "reset")
                else:
                    be.collapse(sl, ctl, -1, st.gbit(s, p), False)
        elif kind == "xchg":
            _, gposs, lposs = step
            bits = [1 << (g - L) for g in gposs]
            mask = sum(bits)
            # groups of 2^k slices that differ only in the remapped global bits, member
            # y = the slice whose remapped bits are y
            groups = [[s0 | sum(b for i, b in enumerate(bits) if y >> i & 1) for y in range(1 << len(bits))]
                      for s0 in range(1 << st.G) if not s0 & mask]
            tr.exchange(be, st.slices, groups, lposs)
            st.exchanges += 1
        elif kind == "if":
            be.guard(ctl, "if", step[1])
        else:
            be.guard(ctl, kind)
    if hasattr(be, "flush"):
        be.flush()
    st.perm = list(plan.final_perm)


def run_trajectory_sliced(bound, rng, global_qubits: int, *, backend=None, transport=None, lookahead: bool = True,
                          plan: SlicePlan | None = None, group: int | None = None):
    """run_trajectory (sim.py:306-314) on a state sliced over 2^global_qubits slices.
    `rng` must be an xoshiro stream (RngStream, ours or the reference's); it is advanced
    by exactly the uniforms consumed.  `group`: most global positions per remap (default
    G; 1 = pairwise exchanges only).  Returns (ClassicalStore, SlicedState)."""
    from .sim import ClassicalStore, _rng_words

    k = bound.kernel
    n = int(k.qubit_count)
    backend = backend or GpuSliceBackend()
    transport = transport or LocalTransport(2**global_qubits)
    if plan is None:
        plan = plan_slices(k, bound.values, global_qubits, lookahead=lookahead, group=group)
    words = _rng_words(rng)
    if words is None:
        raise ValueError("the sliced engine draws on the device: pass an RngStream")
    layout = [(nm, int(w)) for nm, w in k.classical_layout]
    nbits = sum(w for _, w in layout)
    st = SlicedState(n, global_qubits, backend, transport)
    ctl = backend.new_ctl(2**global_qubits, nbits, words)
    execute(plan, st, ctl)
    bits, status, _draws, rng_words = backend.read_ctl(ctl, max(1, (nbits + 63) // 64))
    rng.s0, rng.s1, rng.s2, rng.s3 = (int(w) for w in rng_words)
    if status:
        raise DegenerateNorm("selected measurement branch has probability < 1e-15")
    return ClassicalStore._from_words(layout, bits), st
