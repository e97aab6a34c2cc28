"""RDC30 depth 20 (one measurement round), one trajectory, complex128 (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import ir, sim, workloads
_, k = workloads.rdc_circuit(n=30, depth=20, every=20, seed=30200)
b = ir.bind(k, [])
words, tape = sim.sample_words(b, 1, 1234)
st = sim.last_stats()
print("passes", st["passes"], "pass_ms", st["pass_ms"], "key", tape.keys(words)[0])
