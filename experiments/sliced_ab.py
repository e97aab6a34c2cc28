"""A/B: sliced RDC30 (8 emulated slices) per-op vs fused, with the package at argv[1]."""
import sys, time
sys.path.insert(0, sys.argv[1])
from paper_2604_11599_b200 import ir, sim, sliced, workloads
_, k = workloads.rdc_circuit(n=30, depth=20, every=10, seed=34)
b = ir.bind(k, [])
for fuse in (False, True):
    for rep in range(2):
        t0 = time.perf_counter()
        store, st = sliced.run_trajectory_sliced(b, sim.RngStream.for_shot(1234, 0), 3, backend=sliced.GpuSliceBackend(fuse=fuse))
        dt = time.perf_counter() - t0
        del st
    print(sys.argv[1], "fuse" if fuse else "per-op", round(dt, 3), store.key())
