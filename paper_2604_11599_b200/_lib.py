"""ctypes binding of the sm_100a library `libqsb.so` (C ABI: include/qsb.h).

There is no CPU fallback: if the library is missing or no B200 is visible, every
entry point raises `NativeLibraryMissing` / `BackendError`.
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading

import numpy as np

from .errors import (
    BackendError,
    BadPauliString,
    DegenerateNorm,
    DimensionMismatch,
    DynamicCircuit,
    NativeLibraryMissing,
    SimError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSB_LIBRARY", os.path.join(HERE, "libqsb.so"))

# qsb_status (qsb.h)
OK, ERR_SIM, ERR_DYNAMIC, ERR_DEGENERATE, ERR_BAD_PAULI, ERR_DIMENSION = 0, 1, 2, 3, 4, 5
ERR_OOM, ERR_CUDA, ERR_ARG, ERR_UNSUPPORTED, ERR_PREDRAWN = 6, 7, 8, 9, 10
C128, C64 = 0, 1
OP_GATE, OP_MEASURE, OP_RESET, OP_IF, OP_ELSE, OP_ENDIF = 0, 1, 2, 3, 4, 5
BASES = {b: i for i, b in enumerate("x y z h s t sx rx ry rz p u swap".split())}
CMP = {"==": 0, "!=": 1, "<": 2, "<=": 3, ">": 4, ">=": 5, "truthy": 6}

# numpy mirror of `qsb_op` (176 bytes, natural alignment)
OP_DTYPE = np.dtype(
    {
        "names": ["kind", "base", "adjoint", "ntargets", "target", "qubit", "bit", "ctrl_mask", "ctrl_val",
                  "angle_slot", "has_matrix", "angle", "mat", "pred_cmp", "pred_bit", "pred_width", "reserved",
                  "pred_rhs"],
        "formats": ["<i4", "<i4", "<i4", "<i4", ("<i4", 2), "<i4", "<i4", "<u8", "<u8", ("<i4", 3), "<i4",
                    ("<f8", 3), ("<f8", 8), "<i4", "<i4", "<i4", "<i4", "<u8"],
        "offsets": [0, 4, 8, 12, 16, 24, 28, 32, 40, 48, 60, 64, 88, 152, 156, 160, 164, 168],
        "itemsize": 176,
    }
)


class Stats(ctypes.Structure):
    _fields_ = [
        ("kernel_launches", ctypes.c_int64),
        ("passes", ctypes.c_int64),
        ("decides", ctypes.c_int64),
        ("pass_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("pass_bytes", ctypes.c_double),
        ("gate_updates", ctypes.c_int64),
        ("tie_band", ctypes.c_int64),
        ("engine", ctypes.c_int32),
        ("tile_qubits", ctypes.c_int32),
        ("jit_passes", ctypes.c_int32),
        ("jit_compiled", ctypes.c_int32),
        ("jit_compile_ms", ctypes.c_double),
        ("pass_flops", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_D = ctypes.c_double
_PD = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "qsb_last_error": (ctypes.c_char_p, []),
    "qsb_abi_version": (_I32, []),
    "qsb_device_count": (_I32, [ctypes.POINTER(_I32)]),
    "qsb_ctx_create": (_I32, [_I32, ctypes.POINTER(_P)]),
    "qsb_ctx_destroy": (_I32, [_P]),
    "qsb_ctx_synchronize": (_I32, [_P]),
    "qsb_ctx_set_option": (_I32, [_P, ctypes.c_char_p, _I64]),
    "qsb_ctx_last_stats": (_I32, [_P, ctypes.POINTER(Stats)]),
    "qsb_state_create": (_I32, [_P, _I32, _I32, ctypes.POINTER(_P)]),
    "qsb_state_destroy": (_I32, [_P]),
    "qsb_state_set": (_I32, [_P, _P]),
    "qsb_state_get": (_I32, [_P, _P]),
    "qsb_state_copy": (_I32, [_P, _P]),
    "qsb_state_norm": (_I32, [_P, _PD]),
    "qsb_state_device_ptr": (_I32, [_P, ctypes.POINTER(_P)]),
    "qsb_apply_gate": (_I32, [_P, _P, _P, _I32]),
    "qsb_measure": (_I32, [_P, _I32, _D, ctypes.POINTER(_I32), _PD]),
    "qsb_reset": (_I32, [_P, _I32, _D, ctypes.POINTER(_I32)]),
    "qsb_expval_pauli": (_I32, [_P, _U64, _U64, _I32, _PD]),
    "qsb_tape_create": (_I32, [_P, _P, _I32, _I32, _I32, _I32, ctypes.POINTER(_P)]),
    "qsb_tape_destroy": (_I32, [_P]),
    "qsb_tape_is_dynamic": (_I32, [_P, ctypes.POINTER(_I32)]),
    "qsb_sample_trajectories": (_I32, [_P, _I32, _P, _U64, _I64, _I64, _P, _I32, _P, _P]),
    "qsb_sample_trajectories_states": (_I32, [_P, _I32, _P, _U64, _I64, _I64, _P, _P, _I32, _P]),
    "qsb_run_trajectory": (_I32, [_P, _I32, _P, _P, _U64, _I64, _P, _I32, _P, _P, _P, _I32, ctypes.POINTER(_I32),
                                  ctypes.POINTER(_I32)]),
    "qsb_statevector": (_I32, [_P, _P, _P]),
    "qsb_apply_tape": (_I32, [_P, _P, _P]),
    "qsb_sample_static": (_I32, [_P, _I32, _P, _U64, _I64, _I64, _P]),
    "qsb_sample_counts": (_I32, [_P, _I32, _P, _U64, _I64, _I64, _P, _P, _I64, ctypes.POINTER(_I64)]),
    "qsb_observe": (_I32, [_P, _I32, _P, _I64, _P, _P, _P, _P, _I32, _P, _P]),
    "qsb_debug_rng": (_I32, [_P, _U64, _I64, _I32, _P]),
    "qsb_plan_summary": (_I32, [_P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P]),
    "qsb_plan_passes": (_I32, [_P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _I32, ctypes.POINTER(_I32)]),
    "qsb_jit_selftest": (_I32, [_P, _I32, _I32, _I32, _I32, _I32, _I32, _P]),
    "qsb_jit_nvrtc_version": (_I32, [_P, _P]),
    "qsb_fusion_stats": (_I32, [_P, _I32, _I32, _I32, _I32, _I32, _I32, _P]),
    "qsb_debug_fma_peak": (_I32, [_P, _I32, _PD]),
    "qsb_state_prob1": (_I32, [_P, _I32, _PD]),
    "qsb_state_collapse": (_I32, [_P, _I32, _I32, _D, _I32]),
    "qsb_state_scale": (_I32, [_P, _D, _D]),
    "qsb_slice_ctl_create": (_I32, [_P, _I32, _I32, _U64, _I64, _P, ctypes.POINTER(_P)]),
    "qsb_slice_ctl_destroy": (_I32, [_P]),
    "qsb_slice_ctl_read": (_I32, [_P, _P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), _P]),
    "qsb_slice_guard": (_I32, [_P, _P]),
    "qsb_slice_gate": (_I32, [_P, _P, _P]),
    "qsb_slice_scale": (_I32, [_P, _P, _D, _D]),
    "qsb_slice_prob1": (_I32, [_P, _P, _I32, _I32, _I32]),
    "qsb_slice_decide": (_I32, [_P, _I32, _I32]),
    "qsb_slice_collapse": (_I32, [_P, _P, _I32, _I32, _I32]),
    "qsb_slice_exchange_local": (_I32, [_P, _P, _I32]),
    "qsb_slice_remap_local": (_I32, [_P, _I32, _P]),
    "qsb_slice_partials": (_I32, [_P, _P, _P]),
    "qsb_slice_read_sub": (_I32, [_P, _I32, _P, _I32, _P]),
    "qsb_slice_write_sub": (_I32, [_P, _I32, _P, _I32, _P]),
    "qsb_comm_unique_id": (_I32, [_P]),
    "qsb_comm_init": (_I32, [_P, _P, _I32, _I32, ctypes.POINTER(_P)]),
    "qsb_comm_destroy": (_I32, [_P]),
    "qsb_comm_set_chunk": (_I32, [_P, _I64]),
    "qsb_comm_allgather_partials": (_I32, [_P, _P]),
    "qsb_comm_exchange": (_I32, [_P, _P, _I32, _P, _I32, _I32, _I32]),
    "qsb_comm_remap": (_I32, [_P, _P, _I32, _P, _P, _I32]),
    "qsb_comm_stats": (_I32, [_P, _P, _PD]),
    "qsb_comm_nccl_version": (_I32, [ctypes.POINTER(_I32)]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lib_error: str | None = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the ctypes library; raise NativeLibraryMissing if absent."""
    global _lib, _lib_error
    with _lock:
        if _lib is not None:
            return _lib
        p = path or os.environ.get("QSB_LIB") or LIB_PATH  # QSB_LIB: A/B builds (experiments)
        if not os.path.exists(p):
            _lib_error = f"{p} not built (run `python -c 'import __graft_entry__ as g; g.build()'`)"
            raise NativeLibraryMissing(_lib_error)
        try:
            lib = ctypes.CDLL(p)
        except OSError as e:  # pragma: no cover
            _lib_error = str(e)
            raise NativeLibraryMissing(f"cannot load {p}: {e}") from e
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def ptr(a: np.ndarray | None):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


_ERRS = {
    ERR_SIM: SimError,
    ERR_DYNAMIC: DynamicCircuit,
    ERR_DEGENERATE: DegenerateNorm,
    ERR_BAD_PAULI: BadPauliString,
    ERR_DIMENSION: DimensionMismatch,
}


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = (_lib.qsb_last_error() or b"").decode(errors="replace")
    cls = _ERRS.get(rc, BackendError)
    raise cls(msg or f"qsb status {rc}")


class Context:
    """One device, one CUDA stream (qsb_ctx)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.qsb_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device
        self.lib = lib
        # QSB_OPTIONS="reg_bits=3,dedup=0": engine tuning knobs for experiments
        for kv in filter(None, os.environ.get("QSB_OPTIONS", "").split(",")):
            key, _, val = kv.partition("=")
            self.set_option(key.strip(), int(val))

    def set_option(self, key: str, value: int) -> None:
        check(self.lib.qsb_ctx_set_option(self.handle, key.encode(), int(value)))

    def stats(self) -> dict:
        s = Stats()
        check(self.lib.qsb_ctx_last_stats(self.handle, ctypes.byref(s)))
        return s.as_dict()

    def synchronize(self) -> None:
        check(self.lib.qsb_ctx_synchronize(self.handle))

    def close(self) -> None:
        if self.handle:
            self.lib.qsb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def default_device() -> int:
    """Device of a call that names none: $QSB_DEVICE, else the device torch was pointed
    at (torch.cuda.set_device), else the launcher's LOCAL_RANK (one process per GPU under
    torchrun), else 0.  Keeps `dist.sample_sharded(...)` without `device=` on its own
    GPU per rank instead of piling every rank onto GPU 0."""
    env = os.environ.get("QSB_DEVICE")
    if env is not None:
        return int(env)
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized() and torch.cuda.current_device() != 0:
                return int(torch.cuda.current_device())
        except Exception:  # pragma: no cover
            pass
    local = os.environ.get("LOCAL_RANK")
    if local is not None:
        n = device_count()
        return int(local) % n if n > 0 else int(local)
    return 0


def context(device: int | None = None) -> Context:
    """Per-device default context (created lazily)."""
    if device is None:
        device = default_device()
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx


def device_count() -> int:
    lib = load()
    c = _I32()
    check(lib.qsb_device_count(ctypes.byref(c)))
    return c.value
