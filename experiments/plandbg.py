import sys
sys.path.insert(0, '/root/repo')
from paper_2604_11599_b200 import ir, sim, workloads
_, k = workloads.dyn_circuit()
sim.sample_words(ir.bind(k, []), 2, 1)
