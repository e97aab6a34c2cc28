"""HBM rate of the single-device remap kernel (k_slice_remap_local) over 8 slices of
2^L complex128 amplitudes: bytes moved = 2 x (1 - 2^-k) x the group's bytes (every
off-diagonal block element read and written once).  python experiments/remap_bw.py [L]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_11599_b200 import sim, sliced

L = int(sys.argv[1]) if len(sys.argv) > 1 else 27
be = sliced.GpuSliceBackend()
sl = [sim.StateVector.zero(L) for _ in range(8)]
for lposs in ((L - 1,), (0,), (L - 1, L - 2), (0, 1), (L - 1, L - 2, L - 3), (0, 1, 2), (0, 13, L - 1)):
    k = len(lposs)
    groups = [[s0 | sum(1 << i for i in range(k) if y >> i & 1) for y in range(1 << k)] for s0 in range(8) if not s0 & ((1 << k) - 1)]
    def run():
        for g in groups:
            be.remap_local([sl[m] for m in g], lposs)
    run(); sl[0]._ctx.synchronize()
    import time
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        run()
    sl[0]._ctx.synchronize()
    dt = (time.perf_counter() - t0) / reps
    moved = 2 * (1 - 0.5 ** k) * 8 * (16 << L)
    print(json.dumps({"k": k, "lpos": lposs, "ms": round(dt * 1e3, 2), "GBs": round(moved / dt / 1e9, 1)}), flush=True)
