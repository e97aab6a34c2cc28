// Resident engine: one CTA per trajectory, the whole 2^n state in shared memory
// (n <= 12 in complex128, <= 13 in complex64), the full flattened program
// interpreted on chip -- gates, measure / reset with a deterministic block
// reduction, and IF/ELSE/ENDIF guards with the predicate evaluated once at entry
// (sim.py:297).  Nothing but the final classical bits (and optionally the final
// state / branch trace of slot 0) ever touches HBM.  This is the engine for
// BASELINE cfg 1 (<= 5 qubits) and every small-n parity case.
//
// Reference semantics reproduced exactly (sim.py:230-259):
//   p1 = sum |a|^2 over bit q == 1; outcome = (u < p1); p_out = p1 or 1.0 - p1;
//   DegenerateNorm if p_out < 1e-15; other branch zeroed; a *= 1.0 / sqrt(p_out);
//   reset = the same projection (no store write) followed by x when the outcome is 1.
//   One uniform per executed Measure / Reset, none for gates or predicates.
#include <cuda_runtime.h>

#include "qsb_device.cuh"
#include "qsb_launch.h"

namespace qsb {

namespace {

template <int T> __device__ __forceinline__ double block_sum_r(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < T / 32; ++w) tot += sh[w];
  return tot;
}

template <typename R, int T>
__global__ void __launch_bounds__(T) k_resident(ResidentArgs a) {
  using A = typename Amp<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* amps = reinterpret_cast<A*>(smem_raw);
  __shared__ uint64_t sbits[kResMaxWords];
  __shared__ double sred[T / 32];
  __shared__ int s_outcome, s_dead;
  __shared__ double s_scale;

  const int n = a.n;
  const int64_t N = 1ll << n;
  const int tid = threadIdx.x;
  for (int64_t slot = blockIdx.x; slot < a.count; slot += gridDim.x) {
    for (int64_t i = tid; i < N; i += T) amps[i] = mk<R>(i == 0 ? (R)1 : (R)0, (R)0);
    for (int w = tid; w < a.nwords; w += T) sbits[w] = 0;
    uint64_t rs[4] = {0, 0, 0, 0};
    int draws = 0, ntrace = 0, status = 0;
    int64_t gates = 0;
    if (tid == 0) {
      if (a.rng_init && slot == 0) {
        for (int w = 0; w < 4; ++w) rs[w] = a.rng_init[w];
      } else {
        rng_for_shot(rs, a.seed, (uint64_t)(a.shot_begin + slot));
      }
    }
    int depth = 0, active = 0;
    const double* mats = a.mats + slot * a.mat_stride;
    __syncthreads();
    for (int oi = 0; oi < a.nops; ++oi) {
      const DevOp& op = a.ops[oi];
      const int kind = op.kind;
      if (kind == QSB_OP_IF) {
        bool act = active == depth;
        bool taken = act && pred_eval(sbits, op.pred_bit, op.pred_width, op.pred_cmp, op.pred_rhs);
        if (act && tid == 0) {
          if (a.trace_out && slot == 0 && ntrace < a.max_trace) {
            int64_t* e = a.trace_out + (int64_t)ntrace * (2 + a.nwords);
            e[0] = op.op_index;
            e[1] = taken ? 1 : 0;
            for (int w = 0; w < a.nwords; ++w) e[2 + w] = (int64_t)sbits[w];
          }
          ntrace++;
        }
        depth++;
        if (taken) active = depth;
        continue;
      }
      if (kind == QSB_OP_ELSE) {
        if (active == depth) active = depth - 1;
        else if (active == depth - 1) active = depth;
        continue;
      }
      if (kind == QSB_OP_ENDIF) {
        if (active == depth) active--;
        depth--;
        continue;
      }
      if (active != depth) continue;
      if (kind == QSB_OP_GATE) {
        double m[8];
        const double* src = mats + (int64_t)op.mat * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = src[j];
        if (op.gclass == GC_SWAP) {
          int lo = op.t0 < op.t1 ? op.t0 : op.t1, hi = op.t0 < op.t1 ? op.t1 : op.t0;
          for (int64_t p = tid; p < (N >> 2); p += T) {
            uint64_t base = insert_zero(insert_zero((uint64_t)p, lo), hi);
            if ((base & op.cm) != op.cv) continue;
            uint64_t ia = base | (1ull << op.t0), ib = base | (1ull << op.t1);
            A x = amps[ia];
            amps[ia] = amps[ib];
            amps[ib] = x;
          }
        } else {
          const int t = op.t0;
          for (int64_t p = tid; p < (N >> 1); p += T) {
            uint64_t i0 = insert_zero((uint64_t)p, t);
            if ((i0 & op.cm) != op.cv) continue;
            uint64_t i1 = i0 | (1ull << t);
            A a0 = amps[i0], a1 = amps[i1];
            apply_pair<R>(op.gclass, m, a0, a1);
            amps[i0] = a0;
            amps[i1] = a1;
          }
        }
        gates++;
        __syncthreads();
        continue;
      }
      // MEASURE / RESET
      const int q = op.qubit;
      double part = 0.0;
      for (int64_t p = tid; p < (N >> 1); p += T) part += norm2<R>(amps[insert_zero((uint64_t)p, q) | (1ull << q)]);
      double p1 = block_sum_r<T>(part, sred);
      if (tid == 0) {
        int dead = 0, outcome = 0;
        double u = 0.0, scale = 1.0;
        if (a.predrawn) {
          if (draws >= a.predrawn_stride) {
            status = QSB_ERR_PREDRAWN;
            dead = 1;
          } else {
            u = a.predrawn[slot * a.predrawn_stride + draws];
          }
        } else {
          u = rng_uniform(rs);
        }
        draws++;
        if (!dead) {
          outcome = u < p1 ? 1 : 0;
          double pout = outcome ? p1 : 1.0 - p1;
          double tol = a.c64 ? 1e-6 : 1e-12;
          if (fabs(u - p1) < tol && a.tie_count) atomicAdd(a.tie_count, 1ull);
          if (pout < 1e-15) {
            status = QSB_ERR_DEGENERATE;
            dead = 1;
          } else {
            scale = 1.0 / sqrt(pout);
          }
          if (kind == QSB_OP_MEASURE) {
            int f = op.bit;
            sbits[f >> 6] = (sbits[f >> 6] & ~(1ull << (f & 63))) | ((uint64_t)outcome << (f & 63));
          }
        }
        s_outcome = outcome;
        s_scale = scale;
        s_dead = dead;
      }
      __syncthreads();
      if (s_dead) break;
      {
        const int outcome = s_outcome;
        const R sc = (R)s_scale;
        const bool flip = kind == QSB_OP_RESET && outcome;
        for (int64_t p = tid; p < (N >> 1); p += T) {
          uint64_t i0 = insert_zero((uint64_t)p, q), i1 = i0 | (1ull << q);
          A keep = outcome ? amps[i1] : amps[i0];
          keep = mk<R>(keep.x * sc, keep.y * sc);
          A z = mk<R>(0, 0);
          if (flip || !outcome) {
            amps[i0] = keep;
            amps[i1] = z;
          } else {
            amps[i0] = z;
            amps[i1] = keep;
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();
    for (int w = tid; w < a.nwords; w += T) a.bits_out[slot * a.nwords + w] = sbits[w];
    if (tid == 0) {
      a.status_out[slot] = status;
      if (a.gate_count) atomicAdd(a.gate_count, (unsigned long long)gates);
      if (slot == 0 && a.ntrace_out) *a.ntrace_out = ntrace;
      if (slot == 0 && a.rng_final)
        for (int w = 0; w < 4; ++w) a.rng_final[w] = rs[w];
      if (slot == 0 && a.draws_out) *a.draws_out = draws;
    }
    if (slot == 0 && a.state_out) {
      A* out = reinterpret_cast<A*>(a.state_out);
      for (int64_t i = tid; i < N; i += T) out[i] = amps[i];
    }
    __syncthreads();
  }
}

template <typename R, int T> cudaError_t launch_t(const ResidentArgs& a, int num_sms, cudaStream_t s) {
  size_t smem = sizeof(typename Amp<R>::T) << a.n;
  auto fn = k_resident<R, T>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, T, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)per_sm * num_sms;
  if (grid > a.count) grid = a.count;
  if (grid < 1) grid = 1;
  fn<<<(unsigned)grid, T, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename R> cudaError_t launch_r(const ResidentArgs& a, int num_sms, cudaStream_t s) {
  if (a.n <= 6) return launch_t<R, 32>(a, num_sms, s);
  if (a.n == 7) return launch_t<R, 64>(a, num_sms, s);
  if (a.n == 8) return launch_t<R, 128>(a, num_sms, s);
  return launch_t<R, 256>(a, num_sms, s);
}

}  // namespace

int resident_max_qubits(int c64) { return c64 ? 13 : 12; }

cudaError_t launch_resident(const ResidentArgs& a, int num_sms, cudaStream_t s) {
  return a.c64 ? launch_r<float>(a, num_sms, s) : launch_r<double>(a, num_sms, s);
}

}  // namespace qsb
