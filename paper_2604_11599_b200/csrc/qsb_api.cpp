// C ABI of the B200 state-vector backend (include/qsb.h): contexts, state objects,
// tapes, and the orchestration of the resident / streaming engines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <chrono>
#include <future>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "qsb_jit.h"
#include "qsb_launch.h"
#include "qsb_plan.h"
#include "qsb_objects.h"

using namespace qsb;

namespace {
thread_local std::string g_err;
}  // namespace

int qsb::fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace {

struct PlanDev {
  StreamPlan plan;
  std::future<JitJobs> pending;  // jit_async: NVRTC running in the background
  DevBuf gates, rops, guard_gates, phases, phase_gates;
  std::vector<JitKernel> jit;  // NVRTC-specialised kernel per pass (empty: generic kernel)
  std::vector<double> pflops;  // floating-point operations per state of each pass
  std::string jit_error;
  int jit_compiled = 0, jit_cached = 0;
  double jit_ms = 0;
};

}  // namespace

struct qsb_tape_s {
  qsb_ctx ctx = nullptr;
  TapeInfo info;
  DevBuf d_dev, d_matsrc, d_mats;  // d_mats: literal-only matrix table (no ParamRef angles)
  std::map<std::pair<int, uint64_t>, std::unique_ptr<PlanDev>> plans;  // (geometry, engine options)
  std::unique_ptr<qsb_tape_s> gates_only;          // static sampling view
  std::unique_ptr<qsb_tape_s> phase_free;          // observe() view: global phases dropped
};

namespace {


size_t amp_bytes(int c64) { return c64 ? 8 : 16; }

int tile_qubits(qsb_ctx ctx, int c64, bool staged = false) {
  if (ctx->opt_tile > 0) return (int)std::min<int64_t>(ctx->opt_tile, kMaxTile);
  // 64 KiB (complex128) / 32 KiB (complex64) of amplitudes per CTA.  (11-qubit tiles for
  // complex128 observe passes -- 4 CTAs per SM for the per-slot gate staging -- won 7 % on
  // VQE24 until the |0...0>-start planning (init_aware) made the 12-qubit plan mostly
  // known-zero passes: 844 vs 639 points/s with 12.)
  (void)staged;
  (void)c64;
  return 12;
}
// contiguous low qubits of every tile: 3 (runs of 8 amplitudes: 128 B complex128, 64 B
// complex64) by default -- measured on B200 with the beam-search tiling (round 2), the tile
// covering one more qubit of the light cones beats the longer runs: DYN20 c128 3443 -> 3518
// shots/s, c64 4951 -> 5286, RDC30 d40 c128 698 -> 681 ms, VQE24 c128 267 -> 271 points/s
// (round 1's 256-byte runs: lowq 4 / 5).  Option low_qubits overrides.
int low_qubits(qsb_ctx ctx, int c64) { return ctx->opt_lowq > 0 ? (int)ctx->opt_lowq : 3; }

// Blocking copy ordered on the context's stream.  ctx->stream is non-blocking, so a plain
// cudaMemcpy (legacy stream) neither waits for work queued on it nor -- for pageable
// host-to-device copies -- guarantees the bytes have landed when it returns; a kernel
// launched next on ctx->stream could read the destination early.
cudaError_t copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

int upload_tape_device(qsb_tape tp) {
  TapeInfo& t = tp->info;
  QSB_CUDA(tp->d_dev.ensure(std::max<size_t>(1, t.dev.size()) * sizeof(DevOp)));
  if (!t.dev.empty())
    QSB_CUDA(copy_sync(tp->d_dev.p, t.dev.data(), t.dev.size() * sizeof(DevOp), cudaMemcpyHostToDevice, tp->ctx->stream));
  QSB_CUDA(tp->d_matsrc.ensure(std::max<size_t>(1, t.mats.size()) * sizeof(MatSrc)));
  if (!t.mats.empty())
    QSB_CUDA(copy_sync(tp->d_matsrc.p, t.mats.data(), t.mats.size() * sizeof(MatSrc), cudaMemcpyHostToDevice, tp->ctx->stream));
  QSB_CUDA(tp->d_mats.ensure(std::max<size_t>(1, t.mats.size()) * 8 * sizeof(double)));
  if (!t.mats.empty() && !t.has_param_angles) {
    launch_mats_prep(tp->d_matsrc.as<MatSrc>(), (int)t.mats.size(), nullptr, 0, 1, tp->d_mats.as<double>(),
                     tp->ctx->stream);
    QSB_CUDA(cudaGetLastError());
    QSB_CUDA(cudaStreamSynchronize(tp->ctx->stream));
  }
  return QSB_OK;
}

int reg_bits(qsb_ctx ctx) { return (int)ctx->opt_reg_bits; }  // amplitudes per thread = 2^reg_bits

// jit_async: the background NVRTC compile of a plan finished -> load its kernels (this thread)
void finish_async_jit(qsb_tape tp, PlanDev* pd, int c64) {
  if (!pd->pending.valid() || pd->pending.wait_for(std::chrono::seconds(0)) != std::future_status::ready) return;
  JitJobs J = pd->pending.get();
  pd->jit_error = jit_load(tp->info, pd->plan, c64, J, pd->jit, &pd->jit_ms, &pd->jit_compiled, &pd->jit_cached);
  if (!pd->jit_error.empty()) pd->jit.clear();
}

int get_plan(qsb_tape tp, int c64, int k, int lowq, int rb, PlanDev** out) {
  const bool want_jit = tp->ctx->opt_jit && tp->info.n >= tp->ctx->opt_jit_min;
  // jit_async: the generic kernel runs until the specialised kernels are compiled; fusion is
  // off for such plans so both kernels give bit-identical results (deterministic whichever ran)
  const bool async = want_jit && tp->ctx->opt_jit_async != 0;
  const bool fuse = tp->ctx->opt_fuse != 0 && !async;
  int key = (((((k * 64 + lowq) * 8 + rb) * 2 + (want_jit ? 1 : 0)) * 2 + (fuse ? 1 : 0)) * 2 + c64) * 2 + (async ? 1 : 0);
  const std::pair<int, uint64_t> pkey(key, tp->ctx->eopt.key());
  auto it = tp->plans.find(pkey);
  if (it != tp->plans.end()) {
    if (async) finish_async_jit(tp, it->second.get(), c64);
    *out = it->second.get();
    return QSB_OK;
  }
  auto pd = std::make_unique<PlanDev>();
  std::string e = build_stream_plan(tp->info, k, lowq, rb, swizzle_bits(c64), pd->plan, tp->ctx->eopt);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  StreamPlan& P = pd->plan;
  QSB_CUDA(pd->gates.ensure(std::max<size_t>(1, P.gates.size()) * sizeof(PassGate)));
  if (!P.gates.empty())
    QSB_CUDA(copy_sync(pd->gates.p, P.gates.data(), P.gates.size() * sizeof(PassGate), cudaMemcpyHostToDevice, tp->ctx->stream));
  QSB_CUDA(pd->rops.ensure(std::max<size_t>(1, P.region_ops.size()) * sizeof(DevOp)));
  if (!P.region_ops.empty())
    QSB_CUDA(copy_sync(pd->rops.p, P.region_ops.data(), P.region_ops.size() * sizeof(DevOp), cudaMemcpyHostToDevice, tp->ctx->stream));
  QSB_CUDA(pd->guard_gates.ensure(std::max<size_t>(1, P.guard_gates.size()) * sizeof(int32_t)));
  QSB_CUDA(copy_sync(pd->guard_gates.p, P.guard_gates.data(), P.guard_gates.size() * sizeof(int32_t),
                      cudaMemcpyHostToDevice, tp->ctx->stream));
  QSB_CUDA(pd->phases.ensure(std::max<size_t>(1, P.phases.size()) * sizeof(PhaseDesc)));
  if (!P.phases.empty())
    QSB_CUDA(copy_sync(pd->phases.p, P.phases.data(), P.phases.size() * sizeof(PhaseDesc), cudaMemcpyHostToDevice, tp->ctx->stream));
  QSB_CUDA(pd->phase_gates.ensure(std::max<size_t>(1, P.phase_gates.size()) * sizeof(PhaseGate)));
  if (!P.phase_gates.empty())
    QSB_CUDA(copy_sync(pd->phase_gates.p, P.phase_gates.data(), P.phase_gates.size() * sizeof(PhaseGate),
                        cudaMemcpyHostToDevice, tp->ctx->stream));
  pd->pflops.assign(P.passes.size(), 0.0);
  for (size_t i = 0; i < P.passes.size(); ++i)
    if (P.passes[i].phase_count) pd->pflops[i] = pass_flops(tp->info, P, (int)i);
  if (want_jit && P.rb && async) {
    pd->pending = std::async(std::launch::async, [info = tp->info, plan = P, c64] {
      return jit_prepare(info, plan, c64, false);
    });
  } else if (want_jit && P.rb) {
    pd->jit_error = jit_build(tp->info, P, c64, fuse, pd->jit, &pd->jit_ms, &pd->jit_compiled, &pd->jit_cached);
    if (!pd->jit_error.empty()) pd->jit.clear();  // generic kernel for every pass
  }
  if (fuse && !pd->jit.empty())  // executed flops of the fused NVRTC kernels
    for (size_t i = 0; i < P.passes.size(); ++i)
      if (P.passes[i].phase_count && pd->jit[i].kern) pd->pflops[i] = pass_flops_fused(tp->info, P, (int)i);
  if (getenv("QSB_PLAN_DEBUG"))
    for (size_t i = 0; i < P.passes.size(); ++i) {
      fprintf(stderr, "pass %zu: k %d gates %d phases %d flops/state %.4g (unfused %.4g) epi %d last-phase tpos", i,
              P.passes[i].k, P.passes[i].pgate_count, P.passes[i].phase_count, pd->pflops[i],
              pass_flops(tp->info, P, (int)i), P.passes[i].epi);
      if (P.passes[i].phase_count) {
        const PhaseDesc& ph = P.phases[P.passes[i].phase_begin + P.passes[i].phase_count - 1];
        for (int b = 0; b < ph.nt && b < 16; ++b) fprintf(stderr, " %d", ph.tpos[b]);
      }
      fprintf(stderr, "\n");
    }
  *out = pd.get();
  tp->plans[pkey] = std::move(pd);
  return QSB_OK;
}

// matrix table for a run: shared literal table, or per-slot tables built from params
int prepare_mats(qsb_tape tp, const double* params_dev, int64_t slots, const double** mats, int64_t* stride) {
  qsb_ctx ctx = tp->ctx;
  const TapeInfo& t = tp->info;
  if (!t.has_param_angles || t.mats.empty()) {
    *mats = tp->d_mats.as<double>();
    *stride = 0;
    return QSB_OK;
  }
  size_t per = t.mats.size() * 8;
  QSB_CUDA(ctx->mats.ensure(per * sizeof(double) * slots));
  launch_mats_prep(tp->d_matsrc.as<MatSrc>(), (int)t.mats.size(), params_dev, t.nparams, slots,
                   ctx->mats.as<double>(), ctx->stream);
  QSB_CUDA(cudaGetLastError());
  *mats = ctx->mats.as<double>();
  *stride = slots > 1 ? (int64_t)per : 0;
  return QSB_OK;
}

int upload_params(qsb_tape tp, const double* params, int64_t rows, const double** out) {
  qsb_ctx ctx = tp->ctx;
  int np = tp->info.nparams;
  if (np == 0) {
    *out = nullptr;
    return QSB_OK;
  }
  if (!params) return fail(QSB_ERR_ARG, "parameters required");
  QSB_CUDA(ctx->params.ensure(sizeof(double) * np * rows));
  QSB_CUDA(cudaMemcpyAsync(ctx->params.p, params, sizeof(double) * np * rows, cudaMemcpyHostToDevice, ctx->stream));
  *out = ctx->params.as<double>();
  return QSB_OK;
}

bool use_resident(qsb_ctx ctx, const TapeInfo& t, int c64) {
  if (ctx->opt_engine == 0) return true;
  if (ctx->opt_engine == 1) return false;
  int lim = ctx->opt_resident_max >= 0 ? (int)ctx->opt_resident_max : resident_max_qubits(c64);
  lim = std::min(lim, resident_max_qubits(c64));
  return t.n <= lim && t.nwords <= kResMaxWords;
}

struct RunTimer {
  qsb_ctx ctx;
  explicit RunTimer(qsb_ctx c) : ctx(c) { cudaEventRecord(ctx->ev_a, ctx->stream); }
  float stop() {
    cudaEventRecord(ctx->ev_b, ctx->stream);
    cudaEventSynchronize(ctx->ev_b);
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b);
    return ms;
  }
};

// Executes the streaming plan for `slots` states already allocated at `state`.
// Control blocks / bits / guards / partials live in the context scratch.
struct StreamRun {
  qsb_tape tp;
  PlanDev* pd;
  int c64;
  int64_t slots;
  void* state;
  const double* mats;
  int64_t mat_stride;
  uint64_t seed;
  int64_t shot_begin;
  const double* predrawn;
  int predrawn_stride;
  int64_t predrawn_slot0;
  int64_t* trace;
  int max_trace;
  int32_t* ntrace;
  const uint64_t* rng_init = nullptr;
  bool physical_counted = false;
  uint64_t final_clear = 0;
  int final_consumed = 0;
  double pass_bytes = 0;
  int64_t passes = 0, decides = 0, launches = 0;
  std::vector<std::pair<int, int>> pass_event_idx;
  bool in_place = false;  // apply to the state already in `state` (no |0...0> initialisation)
};

int alloc_stream_scratch(qsb_ctx ctx, const TapeInfo& t, const StreamPlan& P, int64_t slots) {
  QSB_CUDA(ctx->ctl.ensure(sizeof(TrajCtl) * slots));
  QSB_CUDA(ctx->bits.ensure(sizeof(uint64_t) * t.nwords * slots));
  QSB_CUDA(ctx->guards.ensure(sizeof(uint32_t) * t.gwords * slots));
  int64_t pstride = ((int64_t)1 << P.ntiles_log2) * P.max_local_bins;
  QSB_CUDA(ctx->partial.ensure(sizeof(double) * pstride * slots));
  QSB_CUDA(ctx->dedup.ensure(sizeof(int32_t) * (5 * slots + 8)));
  return QSB_OK;
}

int run_stream(qsb_ctx ctx, StreamRun& r) {
  const TapeInfo& t = r.tp->info;
  const StreamPlan& P = r.pd->plan;
  int rc = alloc_stream_scratch(ctx, t, P, r.slots);
  if (rc) return rc;
  StreamArgs a{};
  a.state = r.state;
  a.n = t.n;
  a.c64 = r.c64;
  a.gates = r.pd->gates.as<PassGate>();
  a.phases = P.rb ? r.pd->phases.as<PhaseDesc>() : nullptr;
  a.phase_gates = r.pd->phase_gates.as<PhaseGate>();
  a.mats = r.mats;
  a.mat_stride = r.mat_stride;
  a.ctl = ctx->ctl.as<TrajCtl>();
  a.bits = ctx->bits.as<uint64_t>();
  a.nwords = t.nwords;
  a.gwords = t.gwords;
  a.guards = ctx->guards.as<uint32_t>();
  a.partial = ctx->partial.as<double>();
  a.partial_stride = ((int64_t)1 << P.ntiles_log2) * P.max_local_bins;
  a.slots = r.slots;
  a.region_ops = r.pd->rops.as<DevOp>();
  a.predrawn = r.predrawn;
  a.predrawn_stride = r.predrawn_stride;
  a.ntiles_log2 = P.ntiles_log2;
  a.predrawn_slot0 = r.predrawn_slot0;
  a.tie_count = ctx->counters.as<unsigned long long>();
  a.trace_out = r.trace;
  a.max_trace = r.max_trace;
  a.ntrace_out = r.ntrace;
  // dedup is valid only when every slot runs the same circuit (shared matrices): it is
  // off for observe(), whose slots are different parameter points
  const bool dedup = ctx->opt_dedup && r.slots > 1 && r.mat_stride == 0;
  int32_t* d_new_rep = ctx->dedup.as<int32_t>();
  int32_t* d_copy_src = d_new_rep + r.slots;
  int32_t* d_active = d_copy_src + r.slots;
  int32_t* d_nactive = d_active + r.slots;
  int32_t* d_split = d_nactive + 4;  // [branches | others | 2 counts] (launch_dedup)
  double* d_phys = reinterpret_cast<double*>(ctx->counters.as<char>() + 16);  // [bytes, flops] physical
  if (dedup) {  // outcome-history rows: one bit per draw (measure / reset ops bound the draws)
    int ndraw_ops = 0;
    for (const DevOp& d : t.dev) ndraw_ops += (d.kind == QSB_OP_MEASURE || d.kind == QSB_OP_RESET) ? 1 : 0;
    a.hwords = std::max(1, (ndraw_ops + 63) / 64);
    QSB_CUDA(ctx->histbits.ensure(sizeof(uint64_t) * a.hwords * r.slots));
    QSB_CUDA(cudaMemsetAsync(ctx->histbits.p, 0, sizeof(uint64_t) * a.hwords * r.slots, ctx->stream));
    a.hbits = ctx->histbits.as<uint64_t>();
  }
  launch_ctl_init(a.ctl, a.bits, t.nwords, a.guards, t.gwords, r.slots, r.seed, r.shot_begin, r.rng_init, dedup ? 1 : 0,
                  ctx->stream);
  r.launches++;
  if (dedup) {
    a.active = d_active;
    a.nactive = d_nactive;
    launch_dedup(a, d_new_rep, d_copy_src, d_active, d_nactive, r.c64, false, nullptr, ctx->stream);
    r.launches += 2;
  }
  r.physical_counted = dedup;
  if (dedup) ctx->run_physical = true;
  if (P.passes.empty() && !r.in_place) {
    launch_init_zero(r.c64, r.state, t.n, r.slots, ctx->stream);
    r.launches++;
  }
  size_t need_events = 2 * P.passes.size();
  while (ctx->pass_events.size() < need_events) {
    cudaEvent_t e;
    QSB_CUDA(cudaEventCreate(&e));
    ctx->pass_events.push_back(e);
  }
  uint64_t acc = 0;
  int consumed = 0;
  const double state_bytes = (double)amp_bytes(r.c64) * (double)((int64_t)1 << t.n) * (double)r.slots;
  bool split_next = false;  // the next pass starts the branches of the last regroup
  // qubits still |0> since the |0...0> start (none for an in-place run)
  uint64_t untouched = r.in_place ? 0 : ((t.n >= 64) ? ~0ull : ((1ull << t.n) - 1));
  bool zeroed = false;  // states zeroed before the first pass (the skipped items hold zeros)
  uint64_t proj_next = 0;  // qubits the last region's unguarded measure / reset ops project
  uint64_t zero_known = 0; // projected qubits whose rejected amplitudes no pass has stored yet
  for (size_t si = 0; si < P.steps.size(); ++si) {
    const Step& s = P.steps[si];
    if (s.type == 0) {
      PassDesc pd = P.passes[s.index];
      if (r.in_place) pd.init_zero = 0;
      // From the |0...0> start until the first decide, qubits no non-diagonal gate has
      // touched are still |0>: the states are zeroed once before the first pass, and every
      // register-phase pass then runs only the items whose tile id has none of those
      // qubits set (the first pass: the tile holding index 0; gates act inside a tile, so
      // the other items stay exactly zero).  Not for passes with an epilogue (their
      // marginal partials cover every tile).
      pd.zero_tid = 0;
      const bool skippable = a.phases && pd.rb > 0 && !pd.epi && untouched;
      if (pd.init_zero) {
        if (skippable) {
          launch_zero_slots(a, r.c64, 0, ctx->stream);
          r.launches++;
          zeroed = true;
        }
      }
      if (skippable && zeroed) {
        int j = 0;
        for (int q = 0; q < t.n; ++q) {
          if (pd.smask >> q & 1) continue;
          if (untouched >> q & 1) pd.zero_tid |= 1ull << j;
          ++j;
        }
      }
      // After a measurement, the amplitudes the collapse rejects on the qubits every live
      // trajectory projected (the region's unguarded measure / reset ops) are zero.  The
      // first pass runs only the items the collapse keeps on its out-of-tile qubits (tile-
      // id bits fixed to the slot's projection values) and stores nothing for the others;
      // those qubits stay "known zero" (zero_known) until a pass holds them in its tile:
      // its gather makes the rejected amplitudes zero instead of reading the stale buffer,
      // and it skips the items rejected on its own out-of-tile known-zero qubits.
      // (Items rejected on qubits some trajectories did not project take the per-item
      // zero-store path, PassItem::zero.)
      const bool driver = a.phases && pd.rb > 0;
      uint64_t zo = 0;  // known-zero qubits outside this pass's tile whose rejected items it skips
      pd.zk_mask = 0;
      if (driver && ctx->opt_zero_fill) {
        if (pd.prologue && !pd.epi) zero_known = proj_next & ~pd.smask & ~1ull;  // (qubit 0: always in the low run)
        if (!pd.prologue) pd.zk_mask = zero_known;
        zo = pd.epi ? 0 : (zero_known & ~pd.smask);
        int j = 0;
        for (int q = 0; q < t.n; ++q) {
          if (pd.smask >> q & 1) continue;
          if (zo >> q & 1) pd.zero_tid |= 1ull << j;
          ++j;
        }
        pd.zero_from_vp = zo ? 1 : 0;
      } else if (zero_known) {  // a pass that reads every amplitude: store the zeros first
        launch_zero_projected(a, r.c64, zero_known, ctx->stream);
        r.launches++;
        zero_known = 0;
      }
      const double pass_frac = std::ldexp(1.0, -__builtin_popcountll(pd.zero_tid));  // share of the items run
      // per-item zero stores: the executed share, for the accounting only
      const bool item_zero = !zo && pd.prologue && driver && !pd.epi;  // per-item zero stores only
      const double flop_frac = item_zero ? std::ldexp(1.0, -__builtin_popcountll(proj_next & ~pd.smask)) : 1.0;
      const double read_frac = flop_frac * std::ldexp(1.0, -__builtin_popcountll(pd.zk_mask & pd.smask));
      proj_next = 0;
      for (int g = pd.gate_begin; g < pd.gate_begin + pd.gate_count; ++g) {  // qubits this pass can move
        const PassGate& q = P.gates[g];
        if (q.gclass == GC_DIAG || q.gclass == GC_DIAG_GLOBAL) continue;
        if (q.lt >= 0) untouched &= ~(1ull << pd.sq[q.lt]);
        if (q.gclass == GC_SWAP && q.lt2 >= 0) untouched &= ~(1ull << pd.sq[q.lt2]);
      }
      cudaEventRecord(ctx->pass_events[2 * s.index], ctx->stream);
      auto launch = [&](const StreamArgs& x) -> cudaError_t {
        if (s.index < (int)r.pd->jit.size() && r.pd->jit[s.index].kern) return jit_launch(r.pd->jit[s.index], x, pd, ctx->stream);
        return launch_pass(x, pd, ctx->stream);
      };
      if (split_next) {
        // branches first (gather from the old representative's buffer, write their own),
        // then the other representatives in place -- every read of a buffer precedes its
        // overwrite by the stream order of the two launches
        StreamArgs b = a;
        b.active = d_split;
        b.nactive = d_split + 2 * r.slots;
        b.read_src = d_copy_src;
        QSB_CUDA(launch(b));
        b.active = d_split + r.slots;
        b.nactive = d_split + 2 * r.slots + 1;
        b.read_src = nullptr;
        QSB_CUDA(launch(b));
        r.launches++;
        split_next = false;
      } else {
        QSB_CUDA(launch(a));
      }
      cudaEventRecord(ctx->pass_events[2 * s.index + 1], ctx->stream);
      // the pass stored every amplitude of its items: its tile qubits are materialised; with
      // no item skipped, all of them
      zero_known = pd.zero_tid ? (zero_known & ~pd.smask) : 0;
      if (!driver) zero_known = 0;
      // writes + reads of the items run
      const double byte_frac = pass_frac * (pd.init_zero ? 1.0 : 1.0 + read_frac);
      r.pass_bytes += byte_frac * state_bytes;
      ctx->run_flops += r.pd->pflops[s.index] * pass_frac * flop_frac * (double)r.slots;
      if (dedup) {  // the kernels touched only the representatives
        launch_accum_physical(d_nactive, r.pd->pflops[s.index] * pass_frac * flop_frac,
                              byte_frac * state_bytes / (double)r.slots, d_phys, ctx->stream);
        r.launches++;
      }
      r.passes++;
      r.launches++;
      acc |= pd.smask;
      if (pd.prologue) consumed = 1;
    } else {
      const RegionDesc& rd = P.regions[s.index];
      QSB_CUDA(launch_decide(a, rd, ctx->stream));
      r.decides++;
      r.launches++;
      if (dedup) {
        // a pass next: it reads the old buffers itself (no state copies); else copy now
        // (register-phase passes only: the shared-memory fallback kernel walks every slot)
        split_next = ctx->opt_defer_copy && si + 1 < P.steps.size() && P.steps[si + 1].type == 0 && !r.in_place &&
                     a.phases && P.passes[P.steps[si + 1].index].rb > 0;
        launch_dedup(a, d_new_rep, d_copy_src, d_active, d_nactive, r.c64, true, split_next ? d_split : nullptr,
                     ctx->stream);
        r.launches += split_next ? 2 : 3;  // regroup (+ copy) + commit
      }
      acc = 0;
      consumed = 0;
      if (rd.op_end > rd.op_begin) untouched = 0;  // after a measurement: no known-zero qubits
      for (int oi = rd.op_begin; oi < rd.op_end; ++oi) {
        const DevOp& op = P.region_ops[oi];
        if ((op.kind == QSB_OP_MEASURE || op.kind == QSB_OP_RESET) && op.guard < 0) proj_next |= 1ull << op.qubit;
      }
    }
  }
  if (zero_known) {  // the run ends with rejected amplitudes never stored: store the zeros
    launch_zero_projected(a, r.c64, zero_known, ctx->stream);
    r.launches++;
  }
  r.final_clear = acc;
  r.final_consumed = consumed;
  launch_count_gates(a, r.pd->guard_gates.as<int32_t>(), t.nguards, P.unguarded_gates,
                     ctx->counters.as<unsigned long long>() + 1, ctx->stream);
  r.launches++;
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

double pass_ms_sum(qsb_ctx ctx, size_t npasses) {
  double tot = 0;
  for (size_t i = 0; i < npasses; ++i) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ctx->pass_events[2 * i], ctx->pass_events[2 * i + 1]) == cudaSuccess) tot += ms;
  }
  return tot;
}

int64_t pick_batch(qsb_ctx ctx, const TapeInfo& t, const StreamPlan& P, int c64, int64_t count) {
  if (ctx->opt_batch > 0) return std::min<int64_t>(ctx->opt_batch, count);
  // the whole job already fits the buffers this context holds: no driver query
  // (cudaMemGetInfo takes 0.1 to tens of ms -- GPU idle time inside a timed call)
  if ((double)ctx->state.bytes >= (double)amp_bytes(c64) * std::ldexp(1.0, t.n) * (double)count &&
      (double)ctx->partial.bytes >= 8.0 * std::ldexp(1.0, P.ntiles_log2) * P.max_local_bins * (double)count)
    return count;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  // already-held scratch counts as available
  size_t held = ctx->state.bytes + ctx->partial.bytes;
  double per = (double)amp_bytes(c64) * std::ldexp(1.0, t.n) +
               8.0 * std::ldexp(1.0, P.ntiles_log2) * P.max_local_bins + sizeof(TrajCtl) + 8.0 * t.nwords +
               4.0 * t.gwords;
  double budget = 0.85 * (double)(free_b + held) - 256.0 * 1024 * 1024;
  int64_t b = (int64_t)(budget / per);
  b = std::max<int64_t>(1, std::min<int64_t>(b, 65535));
  return std::min<int64_t>(b, count);
}

int finish_stats(qsb_ctx ctx, float total_ms, double pass_ms, double pass_bytes, int64_t passes, int64_t decides,
                 int64_t launches, int engine, int k) {
  unsigned long long cnt[4] = {0, 0, 0, 0};
  QSB_CUDA(copy_sync(cnt, ctx->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->run_physical) {  // history dedup: what the kernels actually moved / computed
    double phys[2];
    std::memcpy(phys, &cnt[2], sizeof(phys));
    pass_bytes = phys[0];
    ctx->run_flops = phys[1];
  }
  ctx->last.kernel_launches = launches;
  ctx->last.passes = passes;
  ctx->last.decides = decides;
  ctx->last.pass_ms = pass_ms;
  ctx->last.total_ms = total_ms;
  ctx->last.pass_bytes = pass_bytes;
  ctx->last.pass_flops = ctx->run_flops;
  ctx->last.gate_updates = (int64_t)cnt[1];
  ctx->last.tie_band = (int64_t)cnt[0];
  ctx->last.engine = engine;
  ctx->last.tile_qubits = k;
  return QSB_OK;
}

void note_jit(qsb_ctx ctx, const PlanDev* pd) {
  int n = 0;
  for (const JitKernel& k : pd->jit) n += k.kern ? 1 : 0;
  ctx->last.jit_passes = n;
  ctx->last.jit_compiled = pd->jit_compiled;
  ctx->last.jit_compile_ms = pd->jit_ms;
}

int check_sticky() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(QSB_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
  return QSB_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* qsb_last_error(void) { return g_err.c_str(); }
int32_t qsb_abi_version(void) { return QSB_ABI_VERSION; }

int32_t qsb_device_count(int32_t* count) {
  int c = 0;
  QSB_CUDA(cudaGetDeviceCount(&c));
  *count = c;
  return QSB_OK;
}

int32_t qsb_ctx_create(int32_t device, qsb_ctx* out) {
  if (!out) return fail(QSB_ERR_ARG, "null out");
  int cnt = 0;
  QSB_CUDA(cudaGetDeviceCount(&cnt));
  if (device < 0 || device >= cnt) return fail(QSB_ERR_ARG, "device index out of range");
  DeviceGuard g(device);
  QSB_CUDA(cudaSetDevice(device));
  auto* c = new qsb_ctx_s();
  c->device = device;
  cudaDeviceProp prop;
  QSB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    delete c;
    return fail(QSB_ERR_UNSUPPORTED, std::string("needs an sm_100 (B200) device, found ") + prop.name);
  }
  c->num_sms = prop.multiProcessorCount;
  QSB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  QSB_CUDA(cudaEventCreate(&c->ev_a));
  QSB_CUDA(cudaEventCreate(&c->ev_b));
  QSB_CUDA(c->counters.ensure(64));
  *out = c;
  return QSB_OK;
}

int32_t qsb_ctx_destroy(qsb_ctx ctx) {
  if (!ctx) return QSB_OK;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->state, &ctx->partial, &ctx->ctl, &ctx->bits, &ctx->guards, &ctx->mats, &ctx->params,
                    &ctx->predrawn, &ctx->status, &ctx->counters, &ctx->misc, &ctx->misc2, &ctx->trace,
                    &ctx->dedup, &ctx->histbits, &ctx->shotwords, &ctx->histo})
    b->release();
  for (auto& kv : ctx->ev_jit) cudaLibraryUnload((cudaLibrary_t)kv.second.first);
  for (auto e : ctx->pass_events) cudaEventDestroy(e);
  cudaEventDestroy(ctx->ev_a);
  cudaEventDestroy(ctx->ev_b);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return QSB_OK;
}

int32_t qsb_ctx_synchronize(qsb_ctx ctx) {
  DeviceGuard g(ctx->device);
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QSB_OK;
}

int32_t qsb_ctx_set_option(qsb_ctx ctx, const char* key, int64_t value) {
  std::string k = key ? key : "";
  if (k == "tile_qubits") ctx->opt_tile = value;
  else if (k == "batch") ctx->opt_batch = value;
  else if (k == "resident_max_qubits") ctx->opt_resident_max = value;
  else if (k == "engine") ctx->opt_engine = value;  // -1 auto, 0 resident, 1 streaming
  else if (k == "jit") ctx->opt_jit = value;        // NVRTC per-pass kernels (1) or generic kernel (0)
  else if (k == "jit_min_qubits") ctx->opt_jit_min = value;
  else if (k == "dedup") ctx->opt_dedup = value;
  else if (k == "fuse") ctx->opt_fuse = value;
  else if (k == "jit_async") ctx->opt_jit_async = value;    // NVRTC in the background, generic kernel meanwhile
  else if (k == "defer_copy") ctx->opt_defer_copy = value;  // dedup: branches read the old buffer in their first pass
  else if (k == "zero_fill") ctx->opt_zero_fill = value;    // known-zero amplitudes after a measurement stay lazy
  else if (k == "expval_low_qubits") ctx->opt_ev_lowq = value;  // contiguous run of the Pauli reducer's tiles
  else if (k == "expval_jit") ctx->opt_ev_jit = value;          // NVRTC-specialised Pauli reducer
  else if (k == "expval_jit_terms") ctx->opt_ev_jit_terms = value;  // its terms per launch (<= 32)
  else if (k == "low_qubits") ctx->opt_lowq = value;   // 0: default (3)
  else if (k == "reg_bits") {                       // register-blocked phases: 3..5 register qubits
    if (value < 3 || value > 5) return fail(QSB_ERR_ARG, "reg_bits must be 3, 4 or 5");
    ctx->opt_reg_bits = value;
  }
  else if (k == "release_scratch") {
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf* b : {&ctx->state, &ctx->partial, &ctx->ctl, &ctx->bits, &ctx->guards, &ctx->mats, &ctx->params,
                      &ctx->predrawn, &ctx->status, &ctx->misc, &ctx->misc2, &ctx->trace, &ctx->dedup,
                      &ctx->histbits})
      b->release();
  } else if (!ctx->eopt.set(k, value)) return fail(QSB_ERR_ARG, "unknown option " + k);
  return QSB_OK;
}

int32_t qsb_ctx_last_stats(qsb_ctx ctx, qsb_stats* out) {
  *out = ctx->last;
  return QSB_OK;
}

// ---- states ------------------------------------------------------------------
int32_t qsb_state_create(qsb_ctx ctx, int32_t nqubits, int32_t precision, qsb_state* out) {
  if (nqubits < 0 || nqubits > 40) return fail(QSB_ERR_UNSUPPORTED, "qubit count outside [0, 40] for one state");
  DeviceGuard g(ctx->device);
  auto* s = new qsb_state_s();
  s->ctx = ctx;
  s->n = nqubits;
  s->c64 = precision == QSB_C64 ? 1 : 0;
  cudaError_t e = s->amps.ensure(amp_bytes(s->c64) << nqubits);
  if (e == cudaSuccess) e = s->scratch.ensure(sizeof(double) * (prob_scratch_len(nqubits) + 8));
  if (e != cudaSuccess) {
    s->amps.release();
    s->scratch.release();
    delete s;
    return fail(e == cudaErrorMemoryAllocation ? QSB_ERR_OOM : QSB_ERR_CUDA, cudaGetErrorString(e));
  }
  launch_init_zero(s->c64, s->amps.p, nqubits, 1, ctx->stream);
  QSB_CUDA(cudaGetLastError());
  *out = s;
  return QSB_OK;
}

int32_t qsb_state_destroy(qsb_state st) {
  if (!st) return QSB_OK;
  DeviceGuard g(st->ctx->device);
  cudaStreamSynchronize(st->ctx->stream);
  st->amps.release();
  st->scratch.release();
  st->tmp.release();
  delete st;
  return QSB_OK;
}

int32_t qsb_state_set(qsb_state st, const double* amps) {
  DeviceGuard g(st->ctx->device);
  size_t N = (size_t)1 << st->n;
  if (!st->c64) {
    QSB_CUDA(cudaMemcpyAsync(st->amps.p, amps, 16 * N, cudaMemcpyHostToDevice, st->ctx->stream));
  } else {
    QSB_CUDA(st->tmp.ensure(16 * N));
    QSB_CUDA(cudaMemcpyAsync(st->tmp.p, amps, 16 * N, cudaMemcpyHostToDevice, st->ctx->stream));
    launch_c128_to_c64(st->tmp.as<double>(), st->amps.as<float>(), (int64_t)N, st->ctx->stream);
  }
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  return QSB_OK;
}

int32_t qsb_state_get(qsb_state st, double* amps) {
  DeviceGuard g(st->ctx->device);
  size_t N = (size_t)1 << st->n;
  if (!st->c64) {
    QSB_CUDA(cudaMemcpyAsync(amps, st->amps.p, 16 * N, cudaMemcpyDeviceToHost, st->ctx->stream));
  } else {
    QSB_CUDA(st->tmp.ensure(16 * N));
    launch_c64_to_c128(st->amps.as<float>(), st->tmp.as<double>(), (int64_t)N, st->ctx->stream);
    QSB_CUDA(cudaMemcpyAsync(amps, st->tmp.p, 16 * N, cudaMemcpyDeviceToHost, st->ctx->stream));
  }
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  return QSB_OK;
}

int32_t qsb_state_copy(qsb_state dst, qsb_state src) {
  if (dst->n != src->n || dst->c64 != src->c64) return fail(QSB_ERR_DIMENSION, "state shape / precision mismatch");
  DeviceGuard g(dst->ctx->device);
  QSB_CUDA(cudaMemcpyAsync(dst->amps.p, src->amps.p, amp_bytes(src->c64) << src->n, cudaMemcpyDeviceToDevice,
                           dst->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(dst->ctx->stream));
  return QSB_OK;
}

int32_t qsb_state_norm(qsb_state st, double* out) {
  DeviceGuard g(st->ctx->device);
  double* sc = st->scratch.as<double>();
  launch_prob(st->c64, st->amps.p, st->n, -1, sc + 8, sc, st->ctx->stream);
  double v = 0;
  QSB_CUDA(cudaMemcpyAsync(&v, sc, sizeof(double), cudaMemcpyDeviceToHost, st->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  *out = std::sqrt(v);
  return QSB_OK;
}

int32_t qsb_state_device_ptr(qsb_state st, void** out) {
  *out = st->amps.p;
  return QSB_OK;
}

int32_t qsb_apply_gate(qsb_state st, const qsb_op* op, const double* params, int32_t nparams) {
  if (!op || op->kind != QSB_OP_GATE) return fail(QSB_ERR_ARG, "not a gate op");
  TapeInfo ti;
  std::string e = analyze_tape(op, 1, st->n, 0, nparams, ti);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  DeviceGuard g(st->ctx->device);
  const DevOp& d = ti.dev[0];
  double m[8];
  if (ti.mats[0].has_matrix) {
    std::memcpy(m, ti.mats[0].mat, sizeof(m));
  } else {  // ParamRef / literal angles: build on the device, bring the 2x2 back
    double* sc = st->scratch.as<double>();
    QSB_CUDA(st->tmp.ensure(sizeof(MatSrc) + sizeof(double) * (nparams + 1)));
    char* tb = st->tmp.as<char>();
    QSB_CUDA(cudaMemcpyAsync(tb, &ti.mats[0], sizeof(MatSrc), cudaMemcpyHostToDevice, st->ctx->stream));
    if (nparams > 0)
      QSB_CUDA(cudaMemcpyAsync(tb + sizeof(MatSrc), params, sizeof(double) * nparams, cudaMemcpyHostToDevice,
                               st->ctx->stream));
    launch_mats_prep(reinterpret_cast<MatSrc*>(tb), 1, nparams > 0 ? reinterpret_cast<double*>(tb + sizeof(MatSrc)) : nullptr,
                     nparams, 1, sc, st->ctx->stream);
    QSB_CUDA(cudaMemcpyAsync(m, sc, sizeof(m), cudaMemcpyDeviceToHost, st->ctx->stream));
    QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  }
  if (d.gclass == GC_SWAP) launch_apply_swap(st->c64, st->amps.p, st->n, d.t0, d.t1, d.cm, d.cv, st->ctx->stream);
  else launch_apply_1q(st->c64, st->amps.p, st->n, d.t0, d.cm, d.cv, d.gclass, m, st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_measure(qsb_state st, int32_t qubit, double u, int32_t* outcome, double* p1_out) {
  if (qubit < 0 || qubit >= st->n) return fail(QSB_ERR_ARG, "qubit out of range");
  DeviceGuard g(st->ctx->device);
  double* sc = st->scratch.as<double>();
  launch_prob(st->c64, st->amps.p, st->n, qubit, sc + 8, sc, st->ctx->stream);
  double p1 = 0;
  QSB_CUDA(cudaMemcpyAsync(&p1, sc, sizeof(double), cudaMemcpyDeviceToHost, st->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  int o = u < p1 ? 1 : 0;
  double pout = o ? p1 : 1.0 - p1;
  if (p1_out) *p1_out = p1;
  if (outcome) *outcome = o;
  if (pout < 1e-15) {
    char buf[160];
    snprintf(buf, sizeof(buf), "selected measurement branch %d on qubit %d has probability %.17g", o, qubit, pout);
    return fail(QSB_ERR_DEGENERATE, buf);
  }
  launch_collapse(st->c64, st->amps.p, st->n, qubit, o, 1.0 / std::sqrt(pout), 0, st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_state_prob1(qsb_state st, int32_t qubit, double* p1) {
  if (qubit >= st->n) return fail(QSB_ERR_ARG, "qubit out of range");
  DeviceGuard g(st->ctx->device);
  double* sc = st->scratch.as<double>();
  launch_prob(st->c64, st->amps.p, st->n, qubit < 0 ? -1 : qubit, sc + 8, sc, st->ctx->stream);
  QSB_CUDA(cudaMemcpyAsync(p1, sc, sizeof(double), cudaMemcpyDeviceToHost, st->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  return QSB_OK;
}

int32_t qsb_state_collapse(qsb_state st, int32_t qubit, int32_t outcome, double scale, int32_t flip) {
  if (qubit < 0 || qubit >= st->n) return fail(QSB_ERR_ARG, "qubit out of range");
  DeviceGuard g(st->ctx->device);
  launch_collapse(st->c64, st->amps.p, st->n, qubit, outcome ? 1 : 0, scale, flip ? 1 : 0, st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_state_scale(qsb_state st, double re, double im) {
  DeviceGuard g(st->ctx->device);
  double m[8] = {re, im, 0, 0, 0, 0, re, im};  // diag(c, c) on qubit 0 == global scale
  if (st->n == 0) return fail(QSB_ERR_ARG, "qsb_state_scale needs at least one qubit");
  launch_apply_1q(st->c64, st->amps.p, st->n, 0, 0, 0, GC_DIAG, m, st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_reset(qsb_state st, int32_t qubit, double u, int32_t* outcome) {
  if (qubit < 0 || qubit >= st->n) return fail(QSB_ERR_ARG, "qubit out of range");
  DeviceGuard g(st->ctx->device);
  double* sc = st->scratch.as<double>();
  launch_prob(st->c64, st->amps.p, st->n, qubit, sc + 8, sc, st->ctx->stream);
  double p1 = 0;
  QSB_CUDA(cudaMemcpyAsync(&p1, sc, sizeof(double), cudaMemcpyDeviceToHost, st->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  int o = u < p1 ? 1 : 0;
  double pout = o ? p1 : 1.0 - p1;
  if (outcome) *outcome = o;
  if (pout < 1e-15) {
    char buf[160];
    snprintf(buf, sizeof(buf), "selected measurement branch %d on qubit %d has probability %.17g", o, qubit, pout);
    return fail(QSB_ERR_DEGENERATE, buf);
  }
  launch_collapse(st->c64, st->amps.p, st->n, qubit, o, 1.0 / std::sqrt(pout), 1, st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

}  // extern "C"

// ---- Pauli expectation (shared by qsb_expval_pauli and qsb_observe) -----------------
namespace {

// Tile-fused reducer: group terms so that each group's X supports fit in one k-qubit
// tile set (greedy first fit, larger supports first); Z-only terms join the first group.
int expval_terms_tiled(qsb_ctx ctx, int c64, const void* amps, int n, int64_t slots, const uint64_t* xm,
                       const uint64_t* zm, const int32_t* ny, int nterm, double* out_host) {
  const int k = std::min(12, n), lowq = std::min((int)(ctx->opt_ev_lowq > 0 ? ctx->opt_ev_lowq : 2), k);
  const uint64_t lowmask = (1ull << lowq) - 1;
  struct Grp { uint64_t S; std::vector<int> terms; };
  std::vector<Grp> groups;
  // Tile sets (each launch reads every state once, whatever its term count, so the
  // number of launches is the cost): greedy maximum coverage -- grow a k-qubit set from
  // the low run one qubit at a time, each time the qubit that completes the most
  // uncovered X-supports (ties: the most support bits inside), until every term is
  // covered; then every term goes to one set that contains its X-support, single-choice
  // terms first, the others where the current launch of cap terms has room.  VQE24's 200
  // terms: 12 -> 9 launches per state (first-fit by X weight before).
  // (the NVRTC launch size, also when the generic kernel runs: the grouping -- and so the
  // per-term arithmetic -- must not depend on which kernel evaluates it)
  const int cap = (int)std::max<int64_t>(1, std::min<int64_t>(32, ctx->opt_ev_jit_terms));
  std::vector<int> left, diag, wide_sup;
  for (int t = 0; t < nterm; ++t) {
    if (xm[t] == 0) diag.push_back(t);
    else if (__builtin_popcountll(xm[t] | lowmask) > k) wide_sup.push_back(t);  // fits no tile
    else left.push_back(t);
  }
  while (!left.empty()) {
    uint64_t S = lowmask;
    while (__builtin_popcountll(S) < k) {
      int best_q = -1;
      long best_cov = -1, best_part = -1;
      for (int q = 0; q < n; ++q) {
        if (S >> q & 1) continue;
        const uint64_t T = S | (1ull << q);
        long cov = 0, part = 0;
        for (int t : left) {
          if ((xm[t] & ~T) == 0) ++cov;
          else part += __builtin_popcountll(xm[t] & T);
        }
        if (cov > best_cov || (cov == best_cov && part > best_part)) {
          best_q = q;
          best_cov = cov;
          best_part = part;
        }
      }
      if (best_q < 0) break;
      S |= 1ull << best_q;
    }
    std::vector<int> rest;
    bool any = false;
    for (int t : left) {
      if ((xm[t] & ~S) == 0) any = true;
      else rest.push_back(t);
    }
    if (!any) {  // cannot happen (the first support fits a tile), but never loop forever
      S = lowmask | xm[left[0]];
      for (int q = 0; q < n && __builtin_popcountll(S) < k; ++q) S |= 1ull << q;
      rest.clear();
      for (int t : left)
        if ((xm[t] & ~S) != 0) rest.push_back(t);
    }
    groups.push_back({S, {}});
    left.swap(rest);
  }
  if (groups.empty()) {
    uint64_t S = lowmask;
    for (int q = 0; q < n && __builtin_popcountll(S) < k; ++q) S |= 1ull << q;
    groups.push_back({S, {}});
  }
  {
    std::vector<int> cnt(groups.size(), 0), flex;
    std::vector<std::vector<int>> feas(nterm);
    for (int t = 0; t < nterm; ++t) {
      if (__builtin_popcountll(xm[t] | lowmask) > k) continue;
      for (size_t i = 0; i < groups.size(); ++i)
        if ((xm[t] & ~groups[i].S) == 0) feas[t].push_back((int)i);
      if (feas[t].size() == 1) {
        groups[feas[t][0]].terms.push_back(t);
        cnt[feas[t][0]]++;
      } else if (!feas[t].empty()) {
        flex.push_back(t);
      }
    }
    std::stable_sort(flex.begin(), flex.end(), [&](int a, int b) { return feas[a].size() < feas[b].size(); });
    for (int t : flex) {
      int best = feas[t][0];
      auto score = [&](int i) {  // prefer a launch with room (most terms already in it), not a fresh one
        const int r = cnt[i] % cap;
        return (cnt[i] > 0 && r == 0) ? -1 : r;
      };
      for (int i : feas[t])
        if (score(i) > score(best)) best = i;
      groups[best].terms.push_back(t);
      cnt[best]++;
    }
    // keep each group's terms in the historical order (by X weight, descending)
    for (Grp& g : groups)
      std::stable_sort(g.terms.begin(), g.terms.end(), [&](int a, int b) {
        return __builtin_popcountll(xm[a]) > __builtin_popcountll(xm[b]);
      });
    std::vector<Grp> kept;
    for (Grp& g : groups)
      if (!g.terms.empty()) kept.push_back(std::move(g));
    groups.swap(kept);
  }
  for (int t : wide_sup) groups.push_back({lowmask | xm[t], {t}});  // > k support bits: pair-loop path
  std::vector<ExpvalTerm> dev_terms, by_out(nterm);
  std::vector<ExpvalGroup> dev_groups;  // pair-loop launches (path 1)
  std::vector<ExpvalGroup> acc_groups;  // accumulating launches (path 0, k = 12)
  std::vector<EvClass> dev_classes;
  // NVRTC-specialised reducer for observe-sized jobs: register accumulators allow larger
  // launches (fewer reads of the states); the generic kernel keeps kEvAccTerms
  const bool use_ev_jit = ctx->opt_jit && ctx->opt_ev_jit && n >= 16 && nterm >= 8 && jit_available();
  const int ev_jit_terms = use_ev_jit ? (int)std::max<int64_t>(1, std::min<int64_t>(32, ctx->opt_ev_jit_terms)) : kEvAccTerms;
  std::vector<EvMap> dev_maps;
  const int sb = c64 ? 4 : 3;
  for (Grp& g : groups) {
    for (int q = 0; q < n && __builtin_popcountll(g.S) < k; ++q) g.S |= 1ull << q;
    ExpvalGroup eg{};
    eg.smask = g.S;
    eg.k = k;
    eg.lowq = lowq;
    eg.term_begin = (int)dev_terms.size();
    eg.nterm = (int)g.terms.size();
    auto compress = [&](uint64_t m) {
      uint32_t out = 0;
      int j = 0;
      for (uint64_t s = g.S; s; s &= s - 1, ++j)
        if (m & (s & (~s + 1))) out |= 1u << j;
      return out;
    };
    auto make_term = [&](int t) {
      ExpvalTerm e{};
      e.xl = compress(xm[t]);
      e.zl = compress(zm[t] & g.S);
      e.xg = xm[t] & ~g.S;
      e.zg = zm[t] & ~g.S;
      e.ny = ny[t];
      e.out = t;
      return e;
    };
    if (k == 12) {
      // register mappings: first-fit of each term's X support (tile positions) into
      // sets of <= 4 positions; per mapping, the 16 registers span those positions
      struct Map { uint32_t U; std::vector<int> terms; };
      std::vector<Map> maps;
      std::vector<int> wide;  // > 4 X letters in the tile: pair-loop kernel
      for (int t : g.terms) {
        const uint32_t xl = compress(xm[t]);
        if (__builtin_popcount(xl) > 4) {
          wide.push_back(t);
          continue;
        }
        bool placed = false;
        for (Map& m : maps)
          if (__builtin_popcount(m.U | xl) <= 4) {
            m.U |= xl;
            m.terms.push_back(t);
            placed = true;
            break;
          }
        if (!placed) maps.push_back({xl, {t}});
      }
      // per mapping: the terms sorted by (register X pattern, Re / Im) so that each class
      // of equal patterns is one run (its pair products are formed once), then cut into
      // launches of <= kEvAccTerms terms (the per-thread accumulators of one launch live
      // in shared memory: kEvAccTerms x 256 doubles)
      const int cap = ev_jit_terms;
      auto flush_launch = [&](ExpvalGroup& cur) {
        if (cur.nterm) {  // its classes: runs of equal xr per mapping part (Re before Im)
          cur.cls_begin = (int)dev_classes.size();
          for (int mi = 0; mi < cur.nmap; ++mi) {
            const EvMap& m = dev_maps[cur.map_begin + mi];
            const int tb = m.term_begin - cur.term_begin, te = tb + m.nterm;
            for (int t = tb; t < te;) {
              const uint32_t xr = dev_terms[cur.term_begin + t].xr;
              int e = t, im0 = -1;
              while (e < te && dev_terms[cur.term_begin + e].xr == xr) {
                if (im0 < 0 && (dev_terms[cur.term_begin + e].ny & 1)) im0 = e;
                ++e;
              }
              dev_classes.push_back(EvClass{(int16_t)mi, (int16_t)xr, (int16_t)t, (int16_t)(im0 < 0 ? e : im0),
                                            (int16_t)e, 0});
              t = e;
            }
          }
          cur.ncls = (int)dev_classes.size() - cur.cls_begin;
          acc_groups.push_back(cur);
        }
        cur = ExpvalGroup{};
        cur.smask = g.S;
        cur.k = k;
        cur.lowq = lowq;
        cur.term_begin = (int)dev_terms.size();
        cur.map_begin = (int)dev_maps.size();
      };
      ExpvalGroup cur{};
      flush_launch(cur);
      for (Map& m : maps) {
        int rpos[4], nr = 0;
        for (int p = 0; p < k && nr < 4; ++p)
          if (m.U >> p & 1) rpos[nr++] = p;
        for (int p = 0; p < k && nr < 4; ++p)
          if (!(m.U >> p & 1)) rpos[nr++] = p;
        EvMap em{};
        tile_mapping(rpos, 4, k, sb, em.tpos, em.soff);
        std::vector<ExpvalTerm> mts;
        for (int t : m.terms) {
          ExpvalTerm e = make_term(t);
          for (int b = 0; b < 4; ++b)
            if (e.xl >> rpos[b] & 1) e.xr |= 1u << b;
          for (int j = 0; j < 16; ++j) {
            uint32_t pos = 0;
            for (int b = 0; b < 4; ++b)
              if (j >> b & 1) pos |= 1u << rpos[b];
            if (__builtin_popcount(pos & e.zl) & 1) e.zsig |= 1u << j;
          }
          e.path = 0;
          mts.push_back(e);
        }
        std::stable_sort(mts.begin(), mts.end(), [](const ExpvalTerm& x, const ExpvalTerm& y) {
          return x.xr != y.xr ? x.xr < y.xr : (x.ny & 1) < (y.ny & 1);
        });
        size_t i = 0;
        while (i < mts.size()) {
          if (cur.nterm == cap) flush_launch(cur);
          const size_t take = std::min<size_t>(mts.size() - i, (size_t)(cap - cur.nterm));
          EvMap part = em;
          part.term_begin = (int)dev_terms.size();
          part.nterm = (int)take;
          for (size_t j = 0; j < take; ++j) {
            dev_terms.push_back(mts[i + j]);
            by_out[mts[i + j].out] = mts[i + j];
          }
          dev_maps.push_back(part);
          cur.nterm += (int)take;
          cur.nmap++;
          i += take;
        }
      }
      flush_launch(cur);
      eg = ExpvalGroup{};
      eg.smask = g.S;
      eg.k = k;
      eg.lowq = lowq;
      eg.term_begin = (int)dev_terms.size();
      eg.nterm = (int)wide.size();
      for (int t : wide) {
        ExpvalTerm e = make_term(t);
        e.path = 1;
        dev_terms.push_back(e);
        by_out[t] = e;
      }
      if (eg.nterm) dev_groups.push_back(eg);
    } else {
      for (int t : g.terms) {
        ExpvalTerm e = make_term(t);
        e.path = 1;
        dev_terms.push_back(e);
        by_out[t] = e;
      }
      dev_groups.push_back(eg);
    }
  }
  const int ntl = n - k;
  const int nchunks = expval_acc_chunks(n);
  const bool any_tile = !dev_groups.empty();
  // partials: [slot][chunk][term] of the accumulating kernel, then (pair-loop terms only)
  // [slot][tile][term]
  const size_t acc_words = (size_t)slots * nterm * nchunks;
  const size_t pbytes = sizeof(double) * (acc_words + (any_tile ? (size_t)slots * nterm * ((size_t)1 << ntl) : 0));
  QSB_CUDA(ctx->misc.ensure(pbytes + 64));
  QSB_CUDA(ctx->misc2.ensure(sizeof(ExpvalTerm) * 2 * (nterm + 1) + sizeof(double) * nterm * slots +
                              sizeof(EvMap) * (dev_maps.size() + 1) + sizeof(EvClass) * (dev_classes.size() + 1) +
                              64));
  char* base = ctx->misc2.as<char>();
  ExpvalTerm* d_terms = reinterpret_cast<ExpvalTerm*>(base);
  ExpvalTerm* d_byout = d_terms + (nterm + 1);
  double* d_out = reinterpret_cast<double*>(d_byout + (nterm + 1));
  EvMap* d_maps = reinterpret_cast<EvMap*>(d_out + nterm * slots);
  EvClass* d_classes = reinterpret_cast<EvClass*>(d_maps + dev_maps.size() + 1);
  if (!dev_classes.empty())
    QSB_CUDA(cudaMemcpyAsync(d_classes, dev_classes.data(), sizeof(EvClass) * dev_classes.size(),
                             cudaMemcpyHostToDevice, ctx->stream));
  if (!dev_maps.empty())
    QSB_CUDA(cudaMemcpyAsync(d_maps, dev_maps.data(), sizeof(EvMap) * dev_maps.size(), cudaMemcpyHostToDevice,
                             ctx->stream));
  if (nterm) {
    QSB_CUDA(cudaMemcpyAsync(d_terms, dev_terms.data(), sizeof(ExpvalTerm) * nterm, cudaMemcpyHostToDevice,
                             ctx->stream));
    QSB_CUDA(cudaMemcpyAsync(d_byout, by_out.data(), sizeof(ExpvalTerm) * nterm, cudaMemcpyHostToDevice, ctx->stream));
  }
  double* p_acc = ctx->misc.as<double>();
  double* p_tile = p_acc + acc_words;
  // NVRTC-specialised reducer per launch group (observe-sized jobs; compiled once per
  // Hamiltonian grouping and cached per context and on disk), else the generic kernel
  std::vector<void*> jk(acc_groups.size(), nullptr);
  if (use_ev_jit && !acc_groups.empty()) {
    std::vector<std::string> srcs(acc_groups.size());
    std::vector<size_t> keys(acc_groups.size());
    std::vector<size_t> missing;
    for (size_t gi = 0; gi < acc_groups.size(); ++gi) {
      const ExpvalGroup& g = acc_groups[gi];
      EvJitSpec sp;
      sp.c64 = c64;
      sp.lowq = lowq;
      for (int mi = 0; mi < g.nmap; ++mi) {
        const EvMap& em = dev_maps[g.map_begin + mi];
        EvJitMap m{};
        for (int b = 0; b < 8; ++b) m.tpos[b] = em.tpos[b];
        for (int j = 0; j < 16; ++j) m.soff[j] = em.soff[j];
        m.t0 = em.term_begin - g.term_begin;
        m.nt = em.nterm;
        sp.maps.push_back(m);
      }
      for (int t = 0; t < g.nterm; ++t) {
        const ExpvalTerm& e = dev_terms[g.term_begin + t];
        sp.terms.push_back(EvJitTerm{e.xr, e.zsig, e.zl, e.zg, e.ny, e.out});
      }
      srcs[gi] = ev_jit_source(sp);  // smask is a kernel argument: one kernel per structure
      keys[gi] = std::hash<std::string>()(srcs[gi]);
      auto it = ctx->ev_jit.find(keys[gi]);
      if (it != ctx->ev_jit.end()) jk[gi] = it->second.second;
      else missing.push_back(gi);
    }
    if (!missing.empty()) {
      std::vector<std::string> ms;
      for (size_t gi : missing) ms.push_back(srcs[gi]);
      std::vector<JitKernel> built;
      ev_jit_build(ms, built);  // failures leave kern null: the generic kernel runs
      for (size_t i = 0; i < missing.size(); ++i)
        if (built[i].kern) {
          ctx->ev_jit[keys[missing[i]]] = {built[i].lib, built[i].kern};
          jk[missing[i]] = built[i].kern;
        }
    }
  }
  for (size_t gi = 0; gi < acc_groups.size(); ++gi) {
    const ExpvalGroup& g = acc_groups[gi];
    if (!jk[gi]) {
      launch_expval_acc(c64, amps, n, slots, g, d_terms, d_maps, d_classes, p_acc, nterm, ctx->stream);
      continue;
    }
    const size_t amp = c64 ? 8 : 16;
    auto up = [](size_t b) { return (b + 15) & ~(size_t)15; };
    const size_t smem = up((c64 ? 2 : 1) * amp * 4096) +
                        up(sizeof(uint64_t) * (4096 >> lowq)) + up(sizeof(uint32_t) * (4096 >> (c64 ? 4 : 3))) +
                        up(sizeof(uint64_t) * 32) + up(sizeof(uint32_t) * 2) + 16;
    const int nchunks_i = nchunks;
    const void* st_p = amps;
    int n_i = n;
    unsigned long long sm = g.smask;
    int nt_i = nterm;
    void* args[] = {(void*)&st_p, (void*)&n_i, (void*)&sm, (void*)&p_acc, (void*)&nt_i, (void*)&nchunks_i};
    QSB_CUDA(cudaLaunchKernel(jk[gi], dim3((unsigned)(slots * nchunks)), dim3(256), args, smem, ctx->stream));
  }
  for (const ExpvalGroup& g : dev_groups)
    if (g.nterm)
      launch_expval_tile(c64, amps, n, slots, g, d_terms, d_maps, p_tile, nterm, ctx->stream);
  QSB_CUDA(cudaGetLastError());
  launch_expval_tile_finish(p_acc, nchunks, p_tile, 1 << ntl, slots, nterm, d_byout, d_out, ctx->stream);
  QSB_CUDA(cudaMemcpyAsync(out_host, d_out, sizeof(double) * nterm * slots, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return check_sticky();
}

int expval_terms(qsb_ctx ctx, int c64, const void* amps, int n, int64_t slots, const uint64_t* xm,
                 const uint64_t* zm, const int32_t* ny, int nterm, double* out_host /*[slots][nterm]*/) {
  if (n >= 1 && nterm > 0) return expval_terms_tiled(ctx, c64, amps, n, slots, xm, zm, ny, nterm, out_host);
  std::map<uint64_t, std::vector<int>> groups;
  for (int t = 0; t < nterm; ++t) groups[xm[t]].push_back(t);
  int blocks = expval_blocks(n);
  QSB_CUDA(ctx->misc.ensure(sizeof(double) * blocks * nterm * slots));
  QSB_CUDA(ctx->misc2.ensure((sizeof(double) + sizeof(uint64_t) + sizeof(int32_t)) * nterm * slots + 64));
  // term order for the kernels: grouped, then mapped back
  std::vector<int> order;
  for (auto& kv : groups)
    for (int t : kv.second) order.push_back(t);
  std::vector<uint64_t> gx(nterm);
  std::vector<int32_t> gny(nterm);
  for (int i = 0; i < nterm; ++i) {
    gx[i] = xm[order[i]];
    gny[i] = ny[order[i]];
  }
  int pos = 0;
  for (auto& kv : groups) {
    const std::vector<int>& ts = kv.second;
    for (size_t c = 0; c < ts.size(); c += 8) {
      PauliGroup g{};
      g.xmask = kv.first;
      g.nterm = (int)std::min<size_t>(8, ts.size() - c);
      g.term0 = pos;
      for (int j = 0; j < g.nterm; ++j) {
        g.zy[j] = zm[ts[c + j]];
        g.ny[j] = ny[ts[c + j]];
      }
      launch_expval_group(c64, amps, n, slots, g, ctx->misc.as<double>(), nterm, ctx->stream);
      pos += g.nterm;
    }
  }
  char* base = ctx->misc2.as<char>();
  double* d_out = reinterpret_cast<double*>(base);
  uint64_t* d_x = reinterpret_cast<uint64_t*>(base + sizeof(double) * nterm * slots);
  int32_t* d_ny = reinterpret_cast<int32_t*>(d_x + nterm);
  QSB_CUDA(cudaMemcpyAsync(d_x, gx.data(), sizeof(uint64_t) * nterm, cudaMemcpyHostToDevice, ctx->stream));
  QSB_CUDA(cudaMemcpyAsync(d_ny, gny.data(), sizeof(int32_t) * nterm, cudaMemcpyHostToDevice, ctx->stream));
  launch_expval_finish(ctx->misc.as<double>(), slots, nterm, blocks, d_x, d_ny, d_out, ctx->stream);
  std::vector<double> tmp((size_t)nterm * slots);
  QSB_CUDA(cudaMemcpyAsync(tmp.data(), d_out, sizeof(double) * nterm * slots, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t s = 0; s < slots; ++s)
    for (int i = 0; i < nterm; ++i) out_host[s * nterm + order[i]] = tmp[s * nterm + i];
  return QSB_OK;
}

}  // namespace

extern "C" {

int32_t qsb_expval_pauli(qsb_state st, uint64_t xmask, uint64_t zmask, int32_t ny, double* out) {
  uint64_t qm = st->n >= 64 ? ~0ull : ((1ull << st->n) - 1);
  if ((xmask & ~qm) || (zmask & ~qm)) return fail(QSB_ERR_BAD_PAULI, "pauli mask outside the register");
  DeviceGuard g(st->ctx->device);
  return expval_terms(st->ctx, st->c64, st->amps.p, st->n, 1, &xmask, &zmask, &ny, 1, out);
}

// ---- tapes ------------------------------------------------------------------
int32_t qsb_tape_create(qsb_ctx ctx, const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                        qsb_tape* out) {
  auto* tp = new qsb_tape_s();
  tp->ctx = ctx;
  std::string e = analyze_tape(ops, nops, nqubits, nbits, nparams, tp->info);
  if (!e.empty()) {
    delete tp;
    return fail(QSB_ERR_ARG, e);
  }
  DeviceGuard g(ctx->device);
  int rc = upload_tape_device(tp);
  if (rc) {
    delete tp;
    return rc;
  }
  // gates-only view for static sampling (_gates_only_state, sim.py:338-343)
  std::vector<qsb_op> gops;
  for (int i = 0; i < nops; ++i)
    if (ops[i].kind == QSB_OP_GATE) gops.push_back(ops[i]);
  if ((int)gops.size() != nops) {
    auto* go = new qsb_tape_s();
    go->ctx = ctx;
    analyze_tape(gops.data(), (int)gops.size(), nqubits, nbits, nparams, go->info);
    rc = upload_tape_device(go);
    if (rc) {
      delete go;
      delete tp;
      return rc;
    }
    tp->gates_only.reset(go);
  }
  *out = tp;
  return QSB_OK;
}

int32_t qsb_tape_destroy(qsb_tape tp) {
  if (!tp) return QSB_OK;
  DeviceGuard g(tp->ctx->device);
  cudaStreamSynchronize(tp->ctx->stream);
  std::vector<qsb_tape> all = {tp};
  if (tp->gates_only) all.push_back(tp->gates_only.get());
  if (tp->phase_free) all.push_back(tp->phase_free.get());
  for (qsb_tape t : all) {
    t->d_dev.release();
    t->d_matsrc.release();
    t->d_mats.release();
    for (auto& kv : t->plans) {
      kv.second->gates.release();
      kv.second->rops.release();
      kv.second->guard_gates.release();
      kv.second->phases.release();
      kv.second->phase_gates.release();
      jit_release(kv.second->jit);
    }
  }
  delete tp;
  return QSB_OK;
}

int32_t qsb_tape_is_dynamic(qsb_tape tp, int32_t* out) {
  *out = tp->info.needs_trajectories ? 1 : 0;
  return QSB_OK;
}

}  // extern "C"

namespace {

// Per-shot classical words of `shot_count` trajectories: into host memory (bits_out) or
// left on the device (dev_out, [shot_count][nwords]) for the device-side histogram.
int sample_traj_impl(qsb_tape tp, int32_t precision, const double* params, uint64_t seed, int64_t shot_begin,
                     int64_t shot_count, const double* predrawn, int32_t predrawn_stride, uint64_t* bits_out,
                     uint64_t* dev_out, int32_t* shot_status, int32_t nstates = 0, qsb_state* states = nullptr) {
  if (shot_count < 1) return fail(QSB_ERR_SIM, "shots must be >= 1");
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  const TapeInfo& t = tp->info;
  const int c64 = precision == QSB_C64 ? 1 : 0;
  if (nstates < 0 || nstates > shot_count || (nstates && !states)) return fail(QSB_ERR_ARG, "bad nstates");
  for (int32_t i = 0; i < nstates; ++i)
    if (!states[i] || states[i]->n != t.n || states[i]->c64 != c64)
      return fail(QSB_ERR_DIMENSION, "states_out shape / precision mismatch");
  QSB_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 32, ctx->stream));
  ctx->run_flops = 0;
  ctx->run_physical = false;
  RunTimer timer(ctx);
  const double* d_params = nullptr;
  int rc = upload_params(tp, params, 1, &d_params);
  if (rc) return rc;
  const double* mats;
  int64_t mstride;
  rc = prepare_mats(tp, d_params, 1, &mats, &mstride);
  if (rc) return rc;
  const double* d_pre = nullptr;
  if (predrawn) {
    if (predrawn_stride < 0) return fail(QSB_ERR_ARG, "bad predrawn stride");
    QSB_CUDA(ctx->predrawn.ensure(sizeof(double) * std::max<int64_t>(1, (int64_t)predrawn_stride * shot_count)));
    QSB_CUDA(cudaMemcpyAsync(ctx->predrawn.p, predrawn, sizeof(double) * predrawn_stride * shot_count,
                             cudaMemcpyHostToDevice, ctx->stream));
    d_pre = ctx->predrawn.as<double>();
  }
  std::vector<int32_t> status((size_t)shot_count, 0);
  if (use_resident(ctx, t, c64)) {
    if (nstates) return fail(QSB_ERR_UNSUPPORTED, "final states of a batch: streaming engine only (engine=1)");
    QSB_CUDA(ctx->bits.ensure(sizeof(uint64_t) * t.nwords * shot_count));
    QSB_CUDA(ctx->status.ensure(sizeof(int32_t) * shot_count));
    ResidentArgs a{};
    a.ops = tp->d_dev.as<DevOp>();
    a.nops = (int)t.dev.size();
    a.n = t.n;
    a.nwords = t.nwords;
    a.predrawn_stride = predrawn_stride;
    a.mats = mats;
    a.mat_stride = 0;
    a.seed = seed;
    a.shot_begin = shot_begin;
    a.count = shot_count;
    a.predrawn = d_pre;
    a.bits_out = dev_out ? dev_out : ctx->bits.as<uint64_t>();
    a.status_out = ctx->status.as<int32_t>();
    a.tie_count = ctx->counters.as<unsigned long long>();
    a.gate_count = ctx->counters.as<unsigned long long>() + 1;
    a.c64 = c64;
    QSB_CUDA(launch_resident(a, ctx->num_sms, ctx->stream));
    if (!dev_out)
      QSB_CUDA(cudaMemcpyAsync(bits_out, ctx->bits.p, sizeof(uint64_t) * t.nwords * shot_count, cudaMemcpyDeviceToHost,
                               ctx->stream));
    QSB_CUDA(cudaMemcpyAsync(status.data(), ctx->status.p, sizeof(int32_t) * shot_count, cudaMemcpyDeviceToHost,
                             ctx->stream));
    float ms = timer.stop();
    rc = check_sticky();
    if (rc) return rc;
    finish_stats(ctx, ms, 0, 0, 0, 0, 1, 0, t.n);
  } else {
    PlanDev* pd;
    rc = get_plan(tp, c64, tile_qubits(ctx, c64), low_qubits(ctx, c64), reg_bits(ctx), &pd);
    if (rc) return rc;
    int64_t B = pick_batch(ctx, t, pd->plan, c64, shot_count);
    QSB_CUDA(ctx->state.ensure((amp_bytes(c64) << t.n) * B));
    double pass_ms = 0, pass_bytes = 0;
    int64_t passes = 0, decides = 0, launches = 0;
    for (int64_t off = 0; off < shot_count; off += B) {
      int64_t b = std::min(B, shot_count - off);
      StreamRun r{tp, pd, c64, b, ctx->state.p, mats, mstride, seed, shot_begin + off, d_pre, predrawn_stride, off,
                  nullptr, 0, nullptr};
      rc = run_stream(ctx, r);
      if (rc) return rc;
      if (off == 0 && nstates) {  // the batch's first slots as the engine left them
        StreamArgs a{};
        a.state = ctx->state.p;
        a.n = t.n;
        a.c64 = c64;
        a.ctl = ctx->ctl.as<TrajCtl>();
        for (int32_t i = 0; i < nstates; ++i)
          launch_finalize(a, states[i]->amps.p, r.final_clear, r.final_consumed, ctx->stream, i);
      }
      QSB_CUDA(cudaMemcpyAsync(dev_out ? dev_out + off * t.nwords : bits_out + off * t.nwords, ctx->bits.p,
                               sizeof(uint64_t) * t.nwords * b,
                               dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
      // only the 4-byte status field of each control block crosses PCIe (strided copy)
      QSB_CUDA(cudaMemcpy2DAsync(status.data() + off, sizeof(int32_t),
                                 ctx->ctl.as<char>() + offsetof(TrajCtl, status), sizeof(TrajCtl), sizeof(int32_t),
                                 (size_t)b, cudaMemcpyDeviceToHost, ctx->stream));
      QSB_CUDA(cudaStreamSynchronize(ctx->stream));
      pass_ms += pass_ms_sum(ctx, pd->plan.passes.size());
      pass_bytes += r.pass_bytes;
      passes += r.passes;
      decides += r.decides;
      launches += r.launches;
    }
    float ms = timer.stop();
    rc = check_sticky();
    if (rc) return rc;
    finish_stats(ctx, ms, pass_ms, pass_bytes, passes, decides, launches, 1, pd->plan.k);
    note_jit(ctx, pd);
  }
  int worst = QSB_OK;
  for (int64_t i = 0; i < shot_count; ++i) {
    if (shot_status) shot_status[i] = status[i];
    if (status[i] != QSB_OK && worst == QSB_OK) worst = status[i];
  }
  if (worst == QSB_ERR_DEGENERATE) return fail(worst, "selected measurement branch has probability < 1e-15");
  if (worst == QSB_ERR_PREDRAWN) return fail(worst, "pre-drawn uniform stream exhausted");
  if (worst != QSB_OK) return fail(worst, "trajectory failed");
  return QSB_OK;
}

}  // namespace

extern "C" {

int32_t qsb_sample_trajectories(qsb_tape tp, int32_t precision, const double* params, uint64_t seed,
                                int64_t shot_begin, int64_t shot_count, const double* predrawn,
                                int32_t predrawn_stride, uint64_t* bits_out, int32_t* shot_status) {
  return sample_traj_impl(tp, precision, params, seed, shot_begin, shot_count, predrawn, predrawn_stride, bits_out,
                          nullptr, shot_status);
}

int32_t qsb_sample_trajectories_states(qsb_tape tp, int32_t precision, const double* params, uint64_t seed,
                                       int64_t shot_begin, int64_t shot_count, uint64_t* bits_out,
                                       int32_t* shot_status, int32_t nstates, qsb_state* states_out) {
  return sample_traj_impl(tp, precision, params, seed, shot_begin, shot_count, nullptr, 0, bits_out, nullptr,
                          shot_status, nstates, states_out);
}

int32_t qsb_run_trajectory(qsb_tape tp, int32_t precision, const double* params, uint64_t* rng_state, uint64_t seed,
                           int64_t shot, const double* predrawn, int32_t npredrawn, uint64_t* bits_out,
                           qsb_state state_out, int64_t* trace_out, int32_t max_trace, int32_t* ntrace,
                           int32_t* ndraws) {
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  const TapeInfo& t = tp->info;
  const int c64 = precision == QSB_C64 ? 1 : 0;
  if (state_out && (state_out->n != t.n || state_out->c64 != c64))
    return fail(QSB_ERR_DIMENSION, "state_out shape / precision mismatch");
  QSB_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 32, ctx->stream));
  ctx->run_flops = 0;
  ctx->run_physical = false;
  RunTimer timer(ctx);
  const double* d_params = nullptr;
  int rc = upload_params(tp, params, 1, &d_params);
  if (rc) return rc;
  const double* mats;
  int64_t mstride;
  rc = prepare_mats(tp, d_params, 1, &mats, &mstride);
  if (rc) return rc;
  const double* d_pre = nullptr;
  if (predrawn) {
    QSB_CUDA(ctx->predrawn.ensure(sizeof(double) * std::max(1, npredrawn)));
    if (npredrawn > 0)
      QSB_CUDA(cudaMemcpyAsync(ctx->predrawn.p, predrawn, sizeof(double) * npredrawn, cudaMemcpyHostToDevice,
                               ctx->stream));
    d_pre = ctx->predrawn.as<double>();
  }
  int64_t* d_trace = nullptr;
  int32_t* d_ntrace = nullptr;
  size_t trace_bytes = trace_out ? sizeof(int64_t) * (size_t)std::max(1, max_trace) * (2 + t.nwords) : 0;
  QSB_CUDA(ctx->trace.ensure(trace_bytes + 128));
  d_ntrace = reinterpret_cast<int32_t*>(ctx->trace.as<char>());
  int32_t* d_draws = d_ntrace + 1;
  uint64_t* d_rng = reinterpret_cast<uint64_t*>(ctx->trace.as<char>() + 64);
  QSB_CUDA(cudaMemsetAsync(d_ntrace, 0, 2 * sizeof(int32_t), ctx->stream));
  if (rng_state)
    QSB_CUDA(cudaMemcpyAsync(d_rng, rng_state, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  if (trace_out) d_trace = reinterpret_cast<int64_t*>(ctx->trace.as<char>() + 128);
  int32_t status = 0;
  if (use_resident(ctx, t, c64)) {
    QSB_CUDA(ctx->bits.ensure(sizeof(uint64_t) * t.nwords));
    QSB_CUDA(ctx->status.ensure(sizeof(int32_t)));
    ResidentArgs a{};
    a.ops = tp->d_dev.as<DevOp>();
    a.nops = (int)t.dev.size();
    a.n = t.n;
    a.nwords = t.nwords;
    a.predrawn_stride = npredrawn;
    a.mats = mats;
    a.seed = seed;
    a.shot_begin = shot;
    a.count = 1;
    a.predrawn = d_pre;
    a.bits_out = ctx->bits.as<uint64_t>();
    a.status_out = ctx->status.as<int32_t>();
    a.state_out = state_out ? state_out->amps.p : nullptr;
    a.trace_out = d_trace;
    a.max_trace = max_trace;
    a.ntrace_out = d_ntrace;
    a.tie_count = ctx->counters.as<unsigned long long>();
    a.gate_count = ctx->counters.as<unsigned long long>() + 1;
    a.rng_init = rng_state ? d_rng : nullptr;
    a.rng_final = d_rng;
    a.draws_out = d_draws;
    a.c64 = c64;
    QSB_CUDA(launch_resident(a, ctx->num_sms, ctx->stream));
    QSB_CUDA(cudaMemcpyAsync(&status, ctx->status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    float ms = timer.stop();
    rc = check_sticky();
    if (rc) return rc;
    finish_stats(ctx, ms, 0, 0, 0, 0, 1, 0, t.n);
  } else {
    PlanDev* pd;
    rc = get_plan(tp, c64, tile_qubits(ctx, c64), low_qubits(ctx, c64), reg_bits(ctx), &pd);
    if (rc) return rc;
    QSB_CUDA(ctx->state.ensure(amp_bytes(c64) << t.n));
    StreamRun r{tp, pd, c64, 1, ctx->state.p, mats, mstride, seed, shot, d_pre, npredrawn, 0, d_trace, max_trace,
                d_ntrace};
    r.rng_init = rng_state ? d_rng : nullptr;
    rc = run_stream(ctx, r);
    if (rc) return rc;
    StreamArgs a{};
    a.state = ctx->state.p;
    a.n = t.n;
    a.c64 = c64;
    a.ctl = ctx->ctl.as<TrajCtl>();
    if (state_out) launch_finalize(a, state_out->amps.p, r.final_clear, r.final_consumed, ctx->stream);
    TrajCtl c;
    QSB_CUDA(cudaMemcpyAsync(&c, ctx->ctl.p, sizeof(TrajCtl), cudaMemcpyDeviceToHost, ctx->stream));
    float ms = timer.stop();
    rc = check_sticky();
    if (rc) return rc;
    status = c.status;
    QSB_CUDA(copy_sync(d_rng, c.rng, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    QSB_CUDA(copy_sync(d_draws, &c.draws, sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    finish_stats(ctx, ms, pass_ms_sum(ctx, pd->plan.passes.size()), r.pass_bytes, r.passes, r.decides, r.launches + 1,
                 1, pd->plan.k);
    note_jit(ctx, pd);
  }
  QSB_CUDA(copy_sync(bits_out, ctx->bits.p, sizeof(uint64_t) * t.nwords, cudaMemcpyDeviceToHost, ctx->stream));
  int32_t nt2[2] = {0, 0};
  QSB_CUDA(copy_sync(nt2, d_ntrace, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  int32_t nt = nt2[0];
  if (ntrace) *ntrace = nt;
  if (ndraws) *ndraws = nt2[1];
  if (rng_state) QSB_CUDA(copy_sync(rng_state, d_rng, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  if (trace_out && nt > 0)
    QSB_CUDA(copy_sync(trace_out, d_trace, sizeof(int64_t) * std::min(nt, max_trace) * (2 + t.nwords),
                        cudaMemcpyDeviceToHost, ctx->stream));
  if (status == QSB_ERR_DEGENERATE) return fail(status, "selected measurement branch has probability < 1e-15");
  if (status == QSB_ERR_PREDRAWN) return fail(status, "pre-drawn uniform stream exhausted");
  if (status != QSB_OK) return fail(status, "trajectory failed");
  return QSB_OK;
}

int32_t qsb_apply_tape(qsb_tape tp, const double* params, qsb_state st) {
  const TapeInfo& t = tp->info;
  if (t.top_level_dynamic) return fail(QSB_ERR_DYNAMIC, "apply_tape needs a gates-only tape");
  if (st->n != t.n) return fail(QSB_ERR_DIMENSION, "state has the wrong qubit count");
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  const int c64 = st->c64;
  QSB_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 32, ctx->stream));
  ctx->run_flops = 0;
  ctx->run_physical = false;
  RunTimer timer(ctx);
  const double* d_params = nullptr;
  int rc = upload_params(tp, params, 1, &d_params);
  if (rc) return rc;
  const double* mats;
  int64_t mstride;
  rc = prepare_mats(tp, d_params, 1, &mats, &mstride);
  if (rc) return rc;
  PlanDev* pd;
  rc = get_plan(tp, c64, tile_qubits(ctx, c64), low_qubits(ctx, c64), reg_bits(ctx), &pd);
  if (rc) return rc;
  StreamRun r{tp, pd, c64, 1, st->amps.p, mats, mstride, 0, 0, nullptr, 0, 0, nullptr, 0, nullptr};
  r.in_place = true;
  rc = run_stream(ctx, r);
  if (rc) return rc;
  float ms = timer.stop();
  rc = check_sticky();
  if (rc) return rc;
  finish_stats(ctx, ms, pass_ms_sum(ctx, pd->plan.passes.size()), r.pass_bytes, r.passes, r.decides, r.launches, 1,
               pd->plan.k);
  note_jit(ctx, pd);
  return QSB_OK;
}

int32_t qsb_statevector(qsb_tape tp, const double* params, qsb_state out) {
  const TapeInfo& t = tp->info;
  if (t.top_level_dynamic) return fail(QSB_ERR_DYNAMIC, "Measure/CondBlock/Reset requires trajectory sampling; use sample()");
  if (out->n != t.n) return fail(QSB_ERR_DIMENSION, "output state has the wrong qubit count");
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  const int c64 = out->c64;
  QSB_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 32, ctx->stream));
  ctx->run_flops = 0;
  ctx->run_physical = false;
  RunTimer timer(ctx);
  const double* d_params = nullptr;
  int rc = upload_params(tp, params, 1, &d_params);
  if (rc) return rc;
  const double* mats;
  int64_t mstride;
  rc = prepare_mats(tp, d_params, 1, &mats, &mstride);
  if (rc) return rc;
  if (use_resident(ctx, t, c64)) {
    QSB_CUDA(ctx->bits.ensure(sizeof(uint64_t) * t.nwords));
    QSB_CUDA(ctx->status.ensure(sizeof(int32_t)));
    ResidentArgs a{};
    a.ops = tp->d_dev.as<DevOp>();
    a.nops = (int)t.dev.size();
    a.n = t.n;
    a.nwords = t.nwords;
    a.mats = mats;
    a.count = 1;
    a.bits_out = ctx->bits.as<uint64_t>();
    a.status_out = ctx->status.as<int32_t>();
    a.state_out = out->amps.p;
    a.gate_count = ctx->counters.as<unsigned long long>() + 1;
    a.c64 = c64;
    QSB_CUDA(launch_resident(a, ctx->num_sms, ctx->stream));
    float ms = timer.stop();
    rc = check_sticky();
    if (rc) return rc;
    finish_stats(ctx, ms, 0, 0, 0, 0, 1, 0, t.n);
    return QSB_OK;
  }
  PlanDev* pd;
  rc = get_plan(tp, c64, tile_qubits(ctx, c64), low_qubits(ctx, c64), reg_bits(ctx), &pd);
  if (rc) return rc;
  StreamRun r{tp, pd, c64, 1, out->amps.p, mats, mstride, 0, 0, nullptr, 0, 0, nullptr, 0, nullptr};
  rc = run_stream(ctx, r);
  if (rc) return rc;
  float ms = timer.stop();
  rc = check_sticky();
  if (rc) return rc;
  finish_stats(ctx, ms, pass_ms_sum(ctx, pd->plan.passes.size()), r.pass_bytes, r.passes, r.decides, r.launches, 1,
               pd->plan.k);
    note_jit(ctx, pd);
  return QSB_OK;
}

}  // extern "C"

namespace {

int sample_static_impl(qsb_tape tp, int32_t precision, const double* params, uint64_t seed, int64_t shot_begin,
                       int64_t shot_count, uint64_t* bits_out, uint64_t* dev_out) {
  if (shot_count < 1) return fail(QSB_ERR_SIM, "shots must be >= 1");
  const TapeInfo& t = tp->info;
  if (t.needs_trajectories) return fail(QSB_ERR_ARG, "tape needs trajectories");
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  qsb_tape view = tp->gates_only ? tp->gates_only.get() : tp;
  qsb_state st = nullptr;
  int rc = qsb_state_create(ctx, t.n, precision, &st);
  if (rc) return rc;
  rc = qsb_statevector(view, params, st);
  if (rc) {
    qsb_state_destroy(st);
    return rc;
  }
  std::vector<int32_t> mq, mb;
  for (int idx : t.top_measures) {
    mq.push_back(t.dev[idx].qubit);
    mb.push_back(t.dev[idx].bit);
  }
  cudaError_t e = ctx->misc.ensure(sizeof(double) * (size_t)cdf_blocks(t.n) + 64);
  if (e == cudaSuccess) e = ctx->misc2.ensure(sizeof(int32_t) * 2 * (mq.size() + 1) + sizeof(uint64_t) * t.nwords * shot_count);
  if (e != cudaSuccess) {
    qsb_state_destroy(st);
    return fail(QSB_ERR_OOM, cudaGetErrorString(e));
  }
  int32_t* d_mq = ctx->misc2.as<int32_t>();
  int32_t* d_mb = d_mq + mq.size() + 1;
  uint64_t* d_bits = reinterpret_cast<uint64_t*>(ctx->misc2.as<char>() + sizeof(int32_t) * 2 * (mq.size() + 1));
  d_bits = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(d_bits) + 7) & ~uintptr_t(7));
  if (!mq.empty()) {
    QSB_CUDA(cudaMemcpyAsync(d_mq, mq.data(), sizeof(int32_t) * mq.size(), cudaMemcpyHostToDevice, ctx->stream));
    QSB_CUDA(cudaMemcpyAsync(d_mb, mb.data(), sizeof(int32_t) * mb.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  launch_cumsum_seq(st->c64, st->amps.p, t.n, ctx->misc.as<double>(), ctx->stream);
  launch_static_search(st->c64, st->amps.p, ctx->misc.as<double>(), t.n, seed, shot_begin, shot_count, d_mq, d_mb,
                       (int)mq.size(), t.nwords, dev_out ? dev_out : d_bits, ctx->stream);
  e = cudaSuccess;
  if (!dev_out)
    e = cudaMemcpyAsync(bits_out, d_bits, sizeof(uint64_t) * t.nwords * shot_count, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  qsb_state_destroy(st);
  if (e != cudaSuccess) return fail(QSB_ERR_CUDA, cudaGetErrorString(e));
  return check_sticky();
}

}  // namespace

extern "C" {

int32_t qsb_sample_static(qsb_tape tp, int32_t precision, const double* params, uint64_t seed, int64_t shot_begin,
                          int64_t shot_count, uint64_t* bits_out) {
  return sample_static_impl(tp, precision, params, seed, shot_begin, shot_count, bits_out, nullptr);
}

int32_t qsb_sample_counts(qsb_tape tp, int32_t precision, const double* params, uint64_t seed, int64_t shot_begin,
                          int64_t shot_count, uint64_t* words_out, int64_t* counts_out, int64_t max_unique,
                          int64_t* nunique_out) {
  if (shot_count < 1) return fail(QSB_ERR_SIM, "shots must be >= 1");
  const TapeInfo& t = tp->info;
  if (t.nwords != 1) return fail(QSB_ERR_UNSUPPORTED, "device histogram needs <= 64 classical bits");
  if (shot_count > INT32_MAX) return fail(QSB_ERR_ARG, "device histogram: at most 2^31-1 shots per call");
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  const size_t n = (size_t)shot_count;
  const size_t scratch = hist_scratch_bytes(n);
  QSB_CUDA(ctx->shotwords.ensure(sizeof(uint64_t) * n));
  QSB_CUDA(ctx->histo.ensure(sizeof(uint64_t) * n + sizeof(int32_t) * n + sizeof(uint64_t) * n + 64 + scratch));
  uint64_t* d_words = ctx->shotwords.as<uint64_t>();
  int rc = t.needs_trajectories
               ? sample_traj_impl(tp, precision, params, seed, shot_begin, shot_count, nullptr, 0, nullptr, d_words,
                                  nullptr)
               : sample_static_impl(tp, precision, params, seed, shot_begin, shot_count, nullptr, d_words);
  if (rc) return rc;
  char* hb = ctx->histo.as<char>();
  uint64_t* d_uniq = reinterpret_cast<uint64_t*>(hb);
  int32_t* d_counts = reinterpret_cast<int32_t*>(d_uniq + n);
  uint64_t* d_sorted = reinterpret_cast<uint64_t*>(d_counts + n + (n & 1));
  int32_t* d_nruns = reinterpret_cast<int32_t*>(d_sorted + n);
  void* d_scratch = reinterpret_cast<char*>(d_nruns) + 64;
  QSB_CUDA(launch_histogram(d_words, d_sorted, n, std::max(1, t.nbits), d_uniq, d_counts, d_nruns, d_scratch, scratch,
                            ctx->stream));
  int32_t nr = 0;
  QSB_CUDA(cudaMemcpyAsync(&nr, d_nruns, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  *nunique_out = nr;
  if (nr > max_unique) return fail(QSB_ERR_ARG, "more distinct outcomes than max_unique (see nunique_out)");
  std::vector<int32_t> c32((size_t)nr);
  QSB_CUDA(cudaMemcpyAsync(words_out, d_uniq, sizeof(uint64_t) * nr, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaMemcpyAsync(c32.data(), d_counts, sizeof(int32_t) * nr, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int32_t i = 0; i < nr; ++i) counts_out[i] = c32[i];
  return check_sticky();
}

namespace {
// observe() only needs <psi|P|psi>, which a global phase of psi does not change: the
// ParamRef rz(theta) = e^{-i theta/2} diag(1, e^{i theta}) of the view is p(theta) (its
// adjoint p(-theta)), a diagonal with a unit |0> entry that the pass kernels apply as one
// complex scale of the |1> amplitude instead of two (VQE24: 192 of the 568 gates).
int phase_free_view(qsb_tape tp, qsb_tape* out) {
  if (tp->phase_free) {
    *out = tp->phase_free.get();
    return QSB_OK;
  }
  auto* v = new qsb_tape_s();
  v->ctx = tp->ctx;
  v->info = tp->info;
  // only UNcontrolled rz: under a control the phase e^{-i theta/2} is relative, not global
  std::vector<int> uses(v->info.mats.size(), 0);
  for (const DevOp& d : v->info.dev)
    if (d.kind == QSB_OP_GATE && d.mat >= 0) uses[d.mat]++;
  bool changed = false;
  for (DevOp& d : v->info.dev) {
    if (d.kind != QSB_OP_GATE || d.gclass != GC_DIAG || d.cm != 0 || d.mat < 0 || uses[d.mat] != 1) continue;
    MatSrc& m = v->info.mats[d.mat];
    if (m.base == QSB_G_RZ && !m.has_matrix) {
      m.base = QSB_G_P;
      d.diag_one0 = 1;
      changed = true;
    }
  }
  if (!changed) {
    delete v;
    *out = tp;
    return QSB_OK;
  }
  int rc = upload_tape_device(v);
  if (rc) {
    delete v;
    return rc;
  }
  tp->phase_free.reset(v);
  *out = v;
  return QSB_OK;
}
}  // namespace

int32_t qsb_observe(qsb_tape tp_in, int32_t precision, const double* params, int64_t npoints, const uint64_t* xmask,
                    const uint64_t* zmask, const int32_t* ny, const double* coef, int32_t nterms, double* energies_out,
                    double* term_out) {
  if (tp_in->info.top_level_dynamic) return fail(QSB_ERR_DYNAMIC, "observe needs a static kernel");
  qsb_tape tp = tp_in;
  {
    DeviceGuard g0(tp_in->ctx->device);
    int rc0 = phase_free_view(tp_in, &tp);
    if (rc0) return rc0;
  }
  const TapeInfo& t = tp->info;
  if (t.top_level_dynamic) return fail(QSB_ERR_DYNAMIC, "observe needs a static kernel");
  if (npoints < 1) return fail(QSB_ERR_ARG, "npoints must be >= 1");
  uint64_t qm = t.n >= 64 ? ~0ull : ((1ull << t.n) - 1);
  for (int i = 0; i < nterms; ++i)
    if ((xmask[i] & ~qm) || (zmask[i] & ~qm)) return fail(QSB_ERR_BAD_PAULI, "pauli mask outside the register");
  qsb_ctx ctx = tp->ctx;
  DeviceGuard g(ctx->device);
  const int c64 = precision == QSB_C64 ? 1 : 0;
  QSB_CUDA(cudaMemsetAsync(ctx->counters.p, 0, 32, ctx->stream));
  ctx->run_flops = 0;
  ctx->run_physical = false;
  RunTimer timer(ctx);
  PlanDev* pd;
  int rc = get_plan(tp, c64, tile_qubits(ctx, c64, t.has_param_angles), low_qubits(ctx, c64), reg_bits(ctx), &pd);
  if (rc) return rc;
  int64_t B = pick_batch(ctx, t, pd->plan, c64, npoints);
  QSB_CUDA(ctx->state.ensure((amp_bytes(c64) << t.n) * B));
  std::vector<double> terms((size_t)std::max(1, nterms) * B);
  double pass_ms = 0, pass_bytes = 0;
  int64_t passes = 0, decides = 0, launches = 0;
  for (int64_t off = 0; off < npoints; off += B) {
    int64_t b = std::min(B, npoints - off);
    const double* d_params = nullptr;
    rc = upload_params(tp, t.nparams ? params + off * t.nparams : nullptr, b, &d_params);
    if (rc) return rc;
    const double* mats;
    int64_t mstride;
    if (t.has_param_angles && !t.mats.empty()) {
      size_t per = t.mats.size() * 8;
      QSB_CUDA(ctx->mats.ensure(per * sizeof(double) * b));
      launch_mats_prep(tp->d_matsrc.as<MatSrc>(), (int)t.mats.size(), d_params, t.nparams, b, ctx->mats.as<double>(),
                       ctx->stream);
      mats = ctx->mats.as<double>();
      mstride = (int64_t)per;
    } else {
      mats = tp->d_mats.as<double>();
      mstride = 0;
    }
    StreamRun r{tp, pd, c64, b, ctx->state.p, mats, mstride, 0, 0, nullptr, 0, 0, nullptr, 0, nullptr};
    rc = run_stream(ctx, r);
    if (rc) return rc;
    pass_bytes += r.pass_bytes;
    passes += r.passes;
    decides += r.decides;
    launches += r.launches;
    if (nterms > 0) {
      rc = expval_terms(ctx, c64, ctx->state.p, t.n, b, xmask, zmask, ny, nterms, terms.data());
      if (rc) return rc;
    }
    pass_ms += pass_ms_sum(ctx, pd->plan.passes.size());
    for (int64_t p = 0; p < b; ++p) {
      double e = 0.0;
      for (int i = 0; i < nterms; ++i) e += coef[i] * terms[p * nterms + i];
      energies_out[off + p] = e;
      if (term_out)
        for (int i = 0; i < nterms; ++i) term_out[(off + p) * nterms + i] = terms[p * nterms + i];
    }
  }
  float ms = timer.stop();
  rc = check_sticky();
  if (rc) return rc;
  finish_stats(ctx, ms, pass_ms, pass_bytes, passes, decides, launches, 1, pd->plan.k);
    note_jit(ctx, pd);
  return QSB_OK;
}

}  // extern "C"

namespace qsb {
void launch_debug_rng(uint64_t seed, int64_t shot, int count, double* out, cudaStream_t s);
double measure_fma_peak(int c64, int num_sms, cudaStream_t s);
}

extern "C" int32_t qsb_debug_fma_peak(qsb_ctx ctx, int32_t precision, double* tflops) {
  DeviceGuard g(ctx->device);
  *tflops = qsb::measure_fma_peak(precision == QSB_C64 ? 1 : 0, ctx->num_sms, ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

extern "C" int32_t qsb_debug_rng(qsb_ctx ctx, uint64_t seed, int64_t shot, int32_t count, double* out) {
  if (count < 0) return fail(QSB_ERR_ARG, "negative count");
  DeviceGuard g(ctx->device);
  QSB_CUDA(ctx->misc.ensure(sizeof(double) * (count + 1)));
  qsb::launch_debug_rng(seed, shot, count, ctx->misc.as<double>(), ctx->stream);
  QSB_CUDA(cudaMemcpyAsync(out, ctx->misc.p, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));
  return QSB_OK;
}

extern "C" int32_t qsb_plan_summary(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                                    int32_t tile_qubits, int32_t low_qubits, int32_t reg_bits, int64_t* out) {
  TapeInfo t;
  std::string e = analyze_tape(ops, nops, nqubits, nbits, nparams, t);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  StreamPlan P;
  e = build_stream_plan(t, tile_qubits, low_qubits, reg_bits, swizzle_bits(low_qubits == 5), P);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  int64_t epi = 0, maxph = 0;
  for (const PassDesc& pd : P.passes) {
    epi += pd.epi;
    maxph = std::max<int64_t>(maxph, pd.phase_count);
  }
  out[0] = (int64_t)P.passes.size();
  out[1] = (int64_t)P.phases.size();
  out[2] = (int64_t)P.gates.size();
  out[3] = (int64_t)P.regions.size();
  out[4] = P.descriptor_gates;
  out[5] = epi;
  out[6] = maxph;
  out[7] = P.rb ? 1 : 0;
  return QSB_OK;
}

extern "C" int32_t qsb_plan_passes(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                                   int32_t tile_qubits, int32_t low_qubits, int32_t reg_bits, int32_t defer_gates,
                                   int64_t* gates_out, int32_t* epi_out, int32_t max_passes, int32_t* npasses) {
  TapeInfo t;
  std::string e = analyze_tape(ops, nops, nqubits, nbits, nparams, t);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  StreamPlan P;
  EngineOptions o;
  o.defer_gates = defer_gates;
  e = build_stream_plan(t, tile_qubits, low_qubits, reg_bits, swizzle_bits(low_qubits == 5), P, o);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  *npasses = (int32_t)P.passes.size();
  for (int i = 0; i < (int)P.passes.size() && i < max_passes; ++i) {
    gates_out[i] = P.passes[i].gate_count;
    epi_out[i] = P.passes[i].epi;
  }
  return QSB_OK;
}

extern "C" int32_t qsb_jit_selftest(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits,
                                    int32_t nparams, int32_t precision, int32_t reg_bits, double* out) {
  const int c64 = precision == QSB_C64 ? 1 : 0;
  if (reg_bits < 3 || reg_bits > 5) return fail(QSB_ERR_ARG, "reg_bits must be 3, 4 or 5");
  TapeInfo t;
  std::string e = analyze_tape(ops, nops, nqubits, nbits, nparams, t);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  StreamPlan P;
  e = build_stream_plan(t, 12, 3, reg_bits, swizzle_bits(c64), P);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  int nk = 0;
  double ms = 0;
  e = jit_compile_only(t, P, c64, true, &nk, &ms);
  out[0] = nk;
  out[1] = ms;
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  return QSB_OK;
}

extern "C" int32_t qsb_jit_nvrtc_version(int32_t* major, int32_t* minor) {
  if (!major || !minor) return fail(QSB_ERR_ARG, "null output");
  int a = 0, b = 0;
  jit_nvrtc_version(&a, &b);
  *major = a;
  *minor = b;
  if (!jit_available()) return fail(QSB_ERR_ARG, "libnvrtc not loadable");
  return QSB_OK;
}

extern "C" int32_t qsb_fusion_stats(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits,
                                    int32_t nparams, int32_t precision, int32_t reg_bits, double* out) {
  const int c64 = precision == QSB_C64 ? 1 : 0;
  if (reg_bits < 3 || reg_bits > 5) return fail(QSB_ERR_ARG, "reg_bits must be 3, 4 or 5");
  TapeInfo t;
  std::string e = analyze_tape(ops, nops, nqubits, nbits, nparams, t);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  StreamPlan P;
  e = build_stream_plan(t, 12, 3, reg_bits, swizzle_bits(c64), P);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  const int fail0 = fuse_check_failures();
  double st[6] = {0, 0, 0, 0, 0, 0};
  for (size_t ph = 0; ph < P.phases.size(); ++ph) {
    if (P.phases[ph].nt < 0) continue;
    st[0] += 1;
    for (const FuseItem& f : fuse_phase(t, P, (int)ph, true))
      if (f.gate < 0) {
        st[1] += 1;
        st[2] += f.ngates;
      }
  }
  for (size_t i = 0; i < P.passes.size(); ++i)
    if (P.passes[i].phase_count) {
      st[4] += pass_flops(t, P, (int)i);
      st[5] += pass_flops_fused(t, P, (int)i);
    }
  st[3] = fuse_check_failures() - fail0;
  for (int i = 0; i < 6; ++i) out[i] = st[i];
  return QSB_OK;
}
