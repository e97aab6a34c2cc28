"""Time the reference's own CPU simulator against the oracle port on DYN20 shots.

Build-container only (imports `/root/reference`, which does not travel to the GPU box):
bench.py's reference arm runs the oracle port (oracle/sim_port.py) because the Python
reference cannot travel; this script checks that the port is a fair stand-in -- same
classical outcomes per shot and comparable single-core speed.

    OPENBLAS_NUM_THREADS=1 python experiments/ref_vs_port_speed.py [shots]
"""
from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests", "golden"))

import make_goldens as G  # noqa: E402  (reference imports + mirror -> reference IR)
from oracle import sim_port as P  # noqa: E402

SEED = 1234  # bench.py's seed


def main(shots: int = 3) -> None:
    _, k = G.workloads.dyn_circuit()
    bound_port = G.ir.bind(k, [])
    bound_ref = G.rkir.bind(G.to_ref(G.ir.kernel_to_json(k)), [])
    t_ref = t_port = 0.0
    for s in range(shots):
        t0 = time.perf_counter()
        rstore, _ = G.rsim.run_trajectory(bound_ref, G.rsim.RngStream.for_shot(SEED, s))
        t1 = time.perf_counter()
        pstore, _ = P.trajectory(bound_port, P.PortRng.for_shot(SEED, s))
        t2 = time.perf_counter()
        t_ref += t1 - t0
        t_port += t2 - t1
        rkey, pkey = rstore.key(), pstore.key()
        assert rkey == pkey, (s, rkey, pkey)
        print(f"shot {s}: {rkey}  reference {t1 - t0:.2f} s  port {t2 - t1:.2f} s", flush=True)
    print(f"DYN20 single core: reference {shots / t_ref:.4f} shots/s, port {shots / t_port:.4f} shots/s, "
          f"identical outcomes on {shots} shots")


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(HERE))
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
