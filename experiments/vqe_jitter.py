"""Run-to-run spread of VQE24 observe (64 points): per call the device total / gate-pass /
reducer time, the host wall time and the SM clock range + throttle reasons sampled with
NVML every 2 ms during the call.  python experiments/vqe_jitter.py [c128|c64] [calls]"""
import os, sys, json, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
from paper_2604_11599_b200 import sim, workloads
prec = sys.argv[1] if len(sys.argv) > 1 else "c128"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 20
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
_, kv = workloads.vqe_ansatz(); ham = workloads.vqe_hamiltonian(); pts = workloads.vqe_points(64)
sim.observe(kv, ham, pts, precision=prec)
if len(sys.argv) > 3:  # warm the GPU first (a DYN20 batch) to see whether the slow calls follow the power ramp
    from paper_2604_11599_b200 import ir
    _, kd = workloads.dyn_circuit(); sim.sample_words(ir.bind(kd, []), 4096, 1234)
for i in range(calls):
    samples, stop = [], threading.Event()
    def poll():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h),
                            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.002)
    th = threading.Thread(target=poll); th.start()
    t0 = time.perf_counter()
    sim.observe(kv, ham, pts, precision=prec)
    wall = (time.perf_counter() - t0) * 1e3
    stop.set(); th.join()
    st = sim.last_stats()
    reasons = 0
    for s_ in samples: reasons |= s_[1]
    print(json.dumps({"call": i, "total_ms": round(st["total_ms"], 1), "pass_ms": round(st["pass_ms"], 1),
                      "reducer_ms": round(st["total_ms"] - st["pass_ms"], 1), "wall_ms": round(wall, 1),
                      "sm_mhz_min": min(s[0] for s in samples), "sm_mhz_max": max(s[0] for s in samples),
                      "throttle_mask": hex(reasons),
                      "mem_mhz_min": min(s_[2] for s_ in samples), "power_w_max": round(max(s_[3] for s_ in samples))}), flush=True)
