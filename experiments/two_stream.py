"""DYN20: one context over B trajectories vs two contexts (two streams) over B/2 each,
running concurrently so that one context's heavy (FP64-bound) passes can share the SMs
with the other's light (HBM-bound) passes.  Experiment; pair with
QSB_JIT_CTAS_PER_SM=1 so that each context's persistent grid leaves room for the other.

    python experiments/two_stream.py one|two [B] [c128|c64]
"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_11599_b200 import _lib, ir, sim, workloads

mode = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
prec = sys.argv[3] if len(sys.argv) > 3 else "c128"
_, k = workloads.dyn_circuit()
b = ir.bind(k, [])
P = sim._prec(prec)


def run(tape, begin, shots, out):
    status = np.zeros(shots, dtype=np.int32)
    _lib.check(tape.ctx.lib.qsb_sample_trajectories(tape.handle, P, None, 1234, begin, shots, None, 0,
                                                    _lib.ptr(out), _lib.ptr(status)))


if mode == "one":
    tapes = [sim.compile_tape(k, 0)]
else:
    tapes = [sim.compile_tape(k, 0), sim.Tape(k, _lib.Context(0))]
per = B // len(tapes)
outs = [np.zeros((per, tapes[0].nwords), dtype=np.uint64) for _ in tapes]
for rep in range(4):
    base = rep * B
    t0 = time.perf_counter()
    th = [threading.Thread(target=run, args=(t, base + i * per, per, outs[i])) for i, t in enumerate(tapes)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t0
    ms = [t.ctx.stats()["total_ms"] for t in tapes]
    print(f"{mode} {prec} B={B} ctas/sm={os.environ.get('QSB_JIT_CTAS_PER_SM')} rep {rep}: wall {dt * 1e3:.0f} ms "
          f"device ms {['%.0f' % m for m in ms]} shots/s {B / dt:.0f}", flush=True)
np.save(f"gpurun_out/two_stream_{mode}_{prec}.npy", np.concatenate(outs))
