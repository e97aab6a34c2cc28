"""VQE24 observe, complex64, 32 points x 3 (experiment: run-to-run variance)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import sim, workloads
_, k = workloads.vqe_ansatz()
H = workloads.vqe_hamiltonian()
pts = workloads.vqe_points(32)
for rep in range(3):
    sim.observe(k, H, pts, precision="c64")
    st = sim.last_stats()
    print(rep, f"total_ms {st['total_ms']:.1f} pass_ms {st['pass_ms']:.1f}")
