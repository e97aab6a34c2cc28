"""VQE24 observe over a few points (profiling target): python experiments/vqe_one.py [points] [c128|c64]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import sim, workloads
npts = int(sys.argv[1]) if len(sys.argv) > 1 else 8
prec = sys.argv[2] if len(sys.argv) > 2 else "c128"
_, k = workloads.vqe_ansatz()
H = workloads.vqe_hamiltonian()
pts = workloads.vqe_points(npts)
reds = []
for rep in range(6):
    e = sim.observe(k, H, pts, precision=prec)
    st = sim.last_stats()
    reds.append(st['total_ms'] - st['pass_ms'])
    print(prec, rep, f"E0 {e[0]:.12f} total_ms {st['total_ms']:.1f} pass_ms {st['pass_ms']:.1f} passes {st['passes']}")
print(prec, f"reducer ms min {min(reds[1:]):.1f} median {sorted(reds[1:])[len(reds[1:]) // 2]:.1f}", os.environ.get("QSB_LIB", ""))
