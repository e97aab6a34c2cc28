"""RDC30 / VQE24 device time vs the contiguous low qubits of a tile (experiment)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_11599_b200 import _lib, ir, sim, workloads
ctx = _lib.context()
lowq = int(sys.argv[1])
ctx.set_option("low_qubits", lowq)
for prec in ("c128", "c64"):
    _, k = workloads.rdc_circuit(n=30, depth=40, every=20, seed=30200)
    b = ir.bind(k, [])
    sim.sample_words(b, 1, 1234, precision=prec)
    words, tape = sim.sample_words(b, 1, 1234, precision=prec)
    st = sim.last_stats()
    print(f"lowq {lowq} RDC30d40 {prec} passes {st['passes']} device_ms {st['total_ms']:.1f} key {tape.keys(words)[0]}")
k = workloads.vqe_ansatz()
k = k[1] if isinstance(k, tuple) else k
H = workloads.vqe_hamiltonian()
pts = workloads.vqe_points(32)
for prec in ("c128", "c64"):
    sim.observe(k, H, pts, precision=prec)
    e = sim.observe(k, H, pts, precision=prec)
    st = sim.last_stats()
    print(f"lowq {lowq} VQE24 {prec} 32 points device_ms {st['total_ms']:.1f} E0 {e[0]:.15f}")
