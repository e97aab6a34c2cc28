"""Benchmark: BASELINE.json configs[1] -- DYN20 dynamic circuit, batched trajectories.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one batch of B trajectories of DYN20 (20 qubits, 40 layers of u + cx,
8 rounds of 4 x {measure, conditional x, reset}: 1180 gates + 64 draws per shot),
each shot its own RNG stream RngStream.for_shot(1234, global_shot).  N ranks
(torchrun, one process per GPU) run disjoint shot ranges -- no collective on the
data path ("scaling": "weak"); the histogram merge is host-side.

value  : shots/s over all ranks, device time (CUDA events on the library's stream,
         max over ranks), states resident in HBM (B x 16 MiB >> 126 MB L2).
e2e    : the same shots through the public API `sim.sample(bound, B, seed)`
         (host wall clock, includes parameter upload, key download, histogram).
roofline: the fused pass kernel (k_pass): algorithmic bytes 2 * 2^n * 16 B per state
         per pass (1x for the first, write-only pass) / its CUDA-event time.
--impl reference: the UNMODIFIED reference simulator installed in baseline/_ref
         (`pip install --target baseline/_ref`) through its public API
         (`qasm2cudaq.suites.compile_source` -> `kir.bind` -> `sim.run_trajectory` with
         `RngStream.for_shot`, the unit of work of `sim.sample`'s process pool,
         sim.py:346-391) on all host cores, one shot per process per step; the pinned
         oracle port (oracle/sim_port.py) only when baseline/_ref is absent.
--gpus N: without a launcher-provided WORLD_SIZE, bench.py re-launches itself under
         `torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL); it exits
         non-zero when fewer than N GPUs are visible.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

SEED = 1234
METRIC = "shots/s on the DYN20 dynamic circuit (20q, 1180 gates + 32 measure + 32 reset per shot, batched trajectories)"
WORKLOAD = "DYN20: BASELINE configs[1], 20-qubit dynamic circuit, 10^5 batched trajectories"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows: list = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in self.rows if (num(r[7]) or 0) > 0] or self.rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        reasons = set()
        for r in self.rows:
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(self.rows[0][1]),
                "reasons": sorted(reasons), "samples": len(self.rows), "samples_under_load": len(loaded),
                "power_w_max": max((num(r[2]) or 0) for r in self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port, one shot per worker process
# ---------------------------------------------------------------------------


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "qasm2cudaq"))


def host_info() -> dict:
    """nproc / CPU model / RAM of the host the CPU arm ran on."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    info["ram_gib"] = round(int(line.split()[1]) / 2**20, 1)
                    break
    except OSError:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keep = ("Socket(s)", "Core(s) per socket", "Thread(s) per core", "NUMA node(s)")
        info["lscpu"] = {k.strip(): v.strip() for k, _, v in (ln.partition(":") for ln in out.splitlines())
                         if k.strip() in keep}
    except Exception:
        pass
    return info


_REF_BOUND = {}


def _ref_shot(args):
    """One DYN20 shot through the UNMODIFIED reference (baseline/_ref)."""
    shot, kind = args
    if not _REF_BOUND:
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        sys.path.insert(0, REPO)
        from paper_2604_11599_b200 import workloads

        src, k = workloads.dyn_circuit()
        if kind == "reference":
            sys.path.insert(0, REF_DIR)
            from qasm2cudaq import kir, sim, suites

            _REF_BOUND["run"] = lambda s: sim.run_trajectory(kir.bind(_REF_BOUND["k"], []),
                                                             sim.RngStream.for_shot(SEED, s))[0].key()
            _REF_BOUND["k"] = suites.compile_source(src)
        else:
            from oracle import sim_port as P
            from paper_2604_11599_b200 import ir

            b = ir.bind(k, [])
            _REF_BOUND["run"] = lambda s: P.trajectory(b, P.PortRng.for_shot(SEED, s))[0].key()
    t0 = time.perf_counter()
    key = _REF_BOUND["run"](shot)
    return key, time.perf_counter() - t0


def cpu_baseline(steps: int, warmup: int, shots_per_step: int | None = None) -> dict:
    """The reference CPU path on all host cores: a process pool (1 BLAS thread per
    process, the reference's own recipe for linear scaling), one
    DYN20 shot per process per step, global shots continuing across steps."""
    import multiprocessing as mp

    kind = "reference" if reference_available() else "port"
    cores = os.cpu_count() or 1
    per = shots_per_step or cores
    ctx = mp.get_context("spawn")
    env_before = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    times = []
    shot = 0
    with ctx.Pool(processes=min(cores, per)) as pool:
        for step in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_ref_shot, [(shot + i, kind) for i in range(per)], chunksize=1)
            dt = time.perf_counter() - t0
            shot += per
            if step >= warmup:
                times.append(dt)
    if env_before is None:
        os.environ.pop("OPENBLAS_NUM_THREADS", None)
    total = sum(times)
    what = ("the unmodified reference qasm2cudaq (baseline/_ref) sim.run_trajectory" if kind == "reference"
            else "the numpy oracle port oracle/sim_port.py")
    return {"value": per * len(times) / total, "unit": "shots/s", "cores": min(cores, per), "kind": kind,
            "sample": f"{per * len(times)} DYN20 shots ({per} per step, one per process, {what}, "
                      f"OPENBLAS_NUM_THREADS=1), {total:.1f} s",
            "host": host_info(), "ms_per_step": 1000 * total / len(times)}


def base_config(batch: int, world: int, prec: str) -> dict:
    """The workload description shared by both arms (same keys, so the driver's
    same-config check compares like with like)."""
    return {"workload": WORKLOAD, "qubits": 20, "batch_per_gpu": batch, "shots_per_step": batch * world,
            "precision": "complex128" if prec == "c128" else "complex64", "seed": SEED,
            "l2": f"inputs larger than L2: {batch} x {16 if prec == 'c128' else 8} MiB states per GPU"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(args.steps, args.warmup)
    cfg = base_config(args.batch, args.gpus, args.precision)  # identical keys and values to our arm's
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "shots/s",
            "engine": "CPU: " + ("reference qasm2cudaq sim (baseline/_ref)" if cb["kind"] == "reference"
                                 else "oracle port of the reference sim"),
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "host")},
            "e2e": {"value": cb["value"], "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < (local + 1):
        sys.exit(f"bench.py: rank {rank} needs GPU {local}, {torch.cuda.device_count()} visible")
    comm = {"backend": None, "world_size": world}
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version()),
                "data_path_collectives": 0,
                "collectives": "barrier + all_reduce(MAX) of the device times + all_gather of the e2e histogram"}

    from paper_2604_11599_b200 import _lib, ir, sim, workloads
    from paper_2604_11599_b200 import dist as qdist

    ctx = _lib.context(local)
    _, kernel = workloads.dyn_circuit()
    bound = ir.bind(kernel, [])
    B = args.batch
    prec = args.precision
    tape = sim.compile_tape(kernel, local)  # compile once (excluded from timing, like lower())
    h2d_bytes = 8  # the step's seed / shot offset; DYN20 has no parameters

    def step_shots(step):  # disjoint global shot ranges per (step, rank)
        return step_shot_begin(step, rank, world, B)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(local)

    # warm-up
    for w in range(args.warmup):
        sim.sample_words(bound, B, SEED, shot_begin=step_shots(w), precision=prec, device=local)
    # timed device region
    barrier()
    dev_ms, pass_ms, pass_bytes, launches, gate_updates, ties, passes = 0.0, 0.0, 0.0, 0, 0, 0, 0
    flops, jit_passes = 0.0, 0
    fma_peak = ctypes.c_double()
    _lib.check(ctx.lib.qsb_debug_fma_peak(ctx.handle, _lib.C64 if prec == "c64" else _lib.C128,
                                          ctypes.byref(fma_peak)))
    with ClockSampler(local) as clocks:
        for s in range(args.steps):
            sim.sample_words(bound, B, SEED, shot_begin=step_shots(args.warmup + s), precision=prec, device=local)
            st = ctx.stats()
            dev_ms += st["total_ms"]
            pass_ms += st["pass_ms"]
            pass_bytes += st["pass_bytes"]
            launches += st["kernel_launches"]
            gate_updates += st["gate_updates"]
            ties += st["tie_band"]
            passes += st["passes"]
            flops += st["pass_flops"]
            jit_passes = st["jit_passes"]
        barrier()
    # e2e through the public API (host wall clock)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    hists = []
    for s in range(e2e_steps):
        if world > 1:  # one job of B x world shots, contiguous shot ranges per rank, merged histogram
            hists.append(qdist.sample_sharded(bound, B * world, SEED, precision=prec, device=local))
        else:
            hists.append(sim.sample(bound, B, SEED, precision=prec, device=local))
    torch.cuda.synchronize(local)
    e2e_s = time.perf_counter() - t0
    # sim.sample histograms on the device: per-shot status words + the distinct outcomes
    # (8-byte word + 4-byte count each) + the distinct count come back
    d2h_bytes = B * 4 + 4 + 12 * len(hists[-1].counts)

    (dev_ms_max, e2e_max), (gate_updates_all, ties_all, launches_all) = reduce_over_ranks(
        [dev_ms, e2e_s], [gate_updates, ties, launches], f"cuda:{local}")
    shots_total = B * args.steps * world
    value = shots_total / (dev_ms_max / 1000.0)
    e2e_value = B * e2e_steps * world / e2e_max
    if rank == 0:
        peaks, which = _peaks()
        achieved = pass_bytes / (pass_ms / 1000.0) / 1e9 if pass_ms > 0 else None
        traffic = None
        prof = os.path.join(REPO, "profiles", "pass_kernel_traffic.json")
        if os.path.exists(prof):
            try:
                # ncu dram bytes / algorithmic bytes per state-pass, applied to this run's
                # algorithmic bytes per pass launch (physical: dedup'd states excluded)
                prof_d = json.load(open(prof))
                ratio = prof_d["traffic_bytes_per_state_pass"] / prof_d["algorithmic_bytes_per_state_pass"]
                traffic = ratio * pass_bytes / passes if (passes and prec == "c128") else None
            except Exception:
                traffic = None
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "shots/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": dev_ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64" if prec == "c128" else "f32",
            "data": "synthetic",
            "config": base_config(B, world, prec),
            "engine": "streaming (fused passes + decide)",
            "tile_qubits": ctx.stats()["tile_qubits"],
            "comm": comm,
            "gate_updates_per_s": gate_updates_all / (dev_ms_max / 1000.0),
            "tie_band_decisions": int(ties_all),
            "passes_per_step": passes / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                         "frac": (achieved / peaks["hbm_gbs"]) if achieved else None, "traffic": traffic,
                         "kernel": "k_pass (fused gate pass)", "peak_kind": which,
                         "algorithmic_bytes_per_step": pass_bytes / args.steps,
                         "pass_ms_per_step": pass_ms / args.steps,
                         "note": "bytes the passes must move: amplitudes known to be zero (untouched "
                                 "qubits, rejected by the last collapse) are neither read nor stored; "
                                 "the binding roof of the complex128 passes is FP64 (compute_roofline)"},
            # the pass kernel's binding roof for complex128 is the FP64 FMA pipe, not HBM:
            # executed floating-point work (FMA = 2) vs the FMA throughput probed on this GPU
            "compute_roofline": {"bound": "fp64" if prec == "c128" else "fp32",
                                 "achieved": flops / (pass_ms / 1000.0) / 1e12 if pass_ms > 0 else None,
                                 "peak": fma_peak.value, "unit": "TFLOP/s",
                                 "frac": (flops / (pass_ms / 1000.0) / 1e12 / fma_peak.value)
                                 if pass_ms > 0 and fma_peak.value > 0 else None,
                                 "peak_kind": "measured on this GPU (qsb_debug_fma_peak)",
                                 "flops_per_step": flops / args.steps},
            "jit_passes": jit_passes,
            "e2e": {"value": e2e_value, "unit": "shots/s", "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": d2h_bytes, "api": "paper_2604_11599_b200.sim.sample" if world == 1
                    else "paper_2604_11599_b200.dist.sample_sharded"},
            "gpu_launches": int(launches_all),
            "clocks": clocks.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(1, 0)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "host")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def step_shot_begin(step: int, rank: int, world: int, batch: int) -> int:
    """First global shot of `rank`'s batch in `step`: every (step, rank) pair gets a
    disjoint contiguous range, so each shot keeps its own for_shot(seed, shot) stream
    (sim.py:54-57) and the union over ranks is [0, steps * world * batch)."""
    return (step * world + rank) * batch


def reduce_over_ranks(times: list, counts: list, device: str) -> tuple[list, list]:
    """Times -> MAX over ranks (the job ends when the slowest rank does), counters ->
    SUM over ranks; identity without a process group."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(times, dtype=torch.float64, device=device)
    g = torch.tensor(counts, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(g, op=dist.ReduceOp.SUM)
    return t.tolist(), g.tolist()


def relaunch(args, argv) -> int:
    """`--gpus N` without a launcher: start N ranks (one per GPU) under torchrun."""
    import socket

    try:
        import torch

        visible = torch.cuda.device_count()
    except Exception:  # pragma: no cover
        visible = 0
    if visible < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {visible} GPU(s) visible", file=sys.stderr)
        return 1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=8192,
                    help="trajectories per GPU per step (8192 x 16 MiB = 128 GiB of complex128 states)")
    ap.add_argument("--precision", choices=["c128", "c64"], default="c128")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args, sys.argv[1:]))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
