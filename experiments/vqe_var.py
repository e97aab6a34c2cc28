"""VQE24 observe timing stability (experiment): repeated calls, pass vs total device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, sim, workloads
_, k = workloads.vqe_ansatz()
H = workloads.vqe_hamiltonian()
pts = workloads.vqe_points(32)
for prec in ("c128", "c64", "c128"):
    for rep in range(3):
        sim.observe(k, H, pts, precision=prec)
        st = sim.last_stats()
        print(prec, rep, f"total_ms {st['total_ms']:.1f} pass_ms {st['pass_ms']:.1f} passes {st['passes']} launches {st['kernel_launches']}")
