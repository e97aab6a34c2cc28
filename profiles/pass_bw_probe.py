"""Streaming-pass bandwidth probe: a 28-qubit static circuit of x / z layers (no FP64
work to speak of), so the fused pass kernel is pure HBM streaming; prints the pass
bandwidth (algorithmic bytes / pass time) per precision."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2604_11599_b200 import ir, sim
import os
for prec in ("c128", "c64"):
    n = 28
    body = []
    for layer in range(4):
        for q in range(n):
            body.append(ir.Gate("x" if layer % 2 == 0 else "z", (), (q,), ()))
    k = ir.Kernel(n, [("q", n)], [], [], body)
    b = ir.bind(k, [])
    for rep in range(3):
        st = sim.statevector(b, precision=prec)
        s = sim.last_stats()
    print(prec, "passes", s["passes"], "pass_ms", round(s["pass_ms"], 2), "GB/s", round(s["pass_bytes"] / (s["pass_ms"] / 1e3) / 1e9, 1))
    del st
