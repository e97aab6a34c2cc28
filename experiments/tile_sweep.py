"""DYN20 pass time per step vs tile size / CTAs per SM (experiment; env QSB_JIT_MINBLOCKS)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_11599_b200 import _lib, ir, sim, workloads
tile = int(sys.argv[1]); prec = sys.argv[2] if len(sys.argv) > 2 else "c128"
_, k = workloads.dyn_circuit()
b = ir.bind(k, [])
ctx = _lib.context()
ctx.set_option("tile_qubits", tile)
ctx.set_option("reg_bits", int(os.environ.get("RB", "4")))
ctx.set_option("low_qubits", int(os.environ.get("LOWQ", "0")))
B = 2048
for rep in range(3):
    sim.sample_words(b, B, 1234, shot_begin=rep * B, precision=prec)
    st = sim.last_stats()
print(f"lowq {os.environ.get('LOWQ', 0)} rb {os.environ.get('RB', 4)} tile {tile} {prec} minblocks {os.environ.get('QSB_JIT_MINBLOCKS')} passes/step {st['passes']} pass_ms {st['pass_ms']:.1f} total_ms {st['total_ms']:.1f} shots/s {B / st['total_ms'] * 1e3:.0f}")
