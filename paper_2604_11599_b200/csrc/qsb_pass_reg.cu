// Generic register-blocked fused-pass kernel (the streaming engine's hot kernel when
// no NVRTC-specialised kernel is available for the pass; see qsb_jit.cpp).
//
// One CTA owns one 2^k-amplitude tile of one state (k = 12: 64 KiB complex128 /
// 32 KiB complex64).  The tile is gathered from HBM once (pass_begin: Pauli-X frame,
// pending collapse), kept in XOR-swizzled shared memory, and run through the pass's
// phases: in a phase every thread holds the 16 amplitudes that differ only in the 4
// "register" tile positions of that phase and applies all of the phase's gates in
// registers; a phase boundary is one shared-memory round trip that re-maps which
// tile positions live in registers.  pass_end accumulates the marginal of the next
// measurement region and scatters the tile back -- one HBM read + one HBM write per
// pass regardless of how many gates it carries.
#include <cuda_runtime.h>

#include <algorithm>

#include "qsb_launch.h"
#include "qsb_pass_common.cuh"

namespace qsb {

namespace {

template <typename R, int NR, int JT, int KIND, bool CTRL>
__device__ __forceinline__ void ph_pair(typename Amp<R>::T* v, const R* m, uint32_t cmR, uint32_t cvR) {
  using A = typename Amp<R>::T;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (j & (1 << JT)) continue;
    if (CTRL && (((uint32_t)j & cmR) != cvR)) continue;
    const A a0 = v[j], a1 = v[j | (1 << JT)];
    A b0, b1;
    if (KIND == PK_XPERM) {
      b0 = a1;
      b1 = a0;
    } else if (KIND == PK_ANTI) {
      b0 = cmul<R>(m[2], m[3], a1);
      b1 = cmul<R>(m[4], m[5], a0);
    } else if (KIND == PK_DIAG_R) {
      b0 = cmul<R>(m[0], m[1], a0);
      b1 = cmul<R>(m[6], m[7], a1);
    } else if (KIND == PK_DENSE_REAL) {
      b0 = mk<R>(fma(m[0], a0.x, m[2] * a1.x), fma(m[0], a0.y, m[2] * a1.y));
      b1 = mk<R>(fma(m[4], a0.x, m[6] * a1.x), fma(m[4], a0.y, m[6] * a1.y));
    } else if (KIND == PK_DENSE_RX) {  // [[c, i m3], [i m5, d]]
      b0 = mk<R>(fma(m[0], a0.x, -m[3] * a1.y), fma(m[0], a0.y, m[3] * a1.x));
      b1 = mk<R>(fma(m[6], a1.x, -m[5] * a0.y), fma(m[6], a1.y, m[5] * a0.x));
    } else {
      b0 = cmac2<R>(m[0], m[1], a0, m[2], m[3], a1);
      b1 = cmac2<R>(m[4], m[5], a0, m[6], m[7], a1);
    }
    v[j] = b0;
    v[j | (1 << JT)] = b1;
  }
}

template <typename R, int NR, int KIND, bool CTRL>
__device__ __forceinline__ void ph_jt(int jt, typename Amp<R>::T* v, const R* m, uint32_t cmR, uint32_t cvR) {
  switch (jt) {
    case 0: ph_pair<R, NR, 0, KIND, CTRL>(v, m, cmR, cvR); break;
    case 1: ph_pair<R, NR, 1, KIND, CTRL>(v, m, cmR, cvR); break;
    case 2: ph_pair<R, NR, 2, KIND, CTRL>(v, m, cmR, cvR); break;
    case 3:
      if constexpr (NR > 8) ph_pair<R, NR, 3, KIND, CTRL>(v, m, cmR, cvR);
      break;
    default:
      if constexpr (NR > 16) ph_pair<R, NR, 4, KIND, CTRL>(v, m, cmR, cvR);
      break;
  }
}

template <typename R, int NR, int KIND>
__device__ __forceinline__ void ph_kind(int jt, typename Amp<R>::T* v, const R* m, uint32_t cmR, uint32_t cvR) {
  if (cmR) ph_jt<R, NR, KIND, true>(jt, v, m, cmR, cvR);
  else ph_jt<R, NR, KIND, false>(jt, v, m, 0, 0);
}

template <typename R, int NR, bool CTRL>
__device__ __forceinline__ void ph_scale(typename Amp<R>::T* v, R dr, R di, uint32_t cmR, uint32_t cvR) {
#pragma unroll
  for (int j = 0; j < NR; ++j)
    if (!CTRL || (((uint32_t)j & cmR) == cvR)) v[j] = cmul<R>(dr, di, v[j]);
}

template <typename R, int RB>
__global__ void __launch_bounds__((1 << (12 - RB)), 2) k_pass_reg(StreamArgs a, PassDesc pd) {
  using A = typename Amp<R>::T;
  constexpr int NR = 1 << RB;
  constexpr int SB = sizeof(R) == 8 ? 3 : 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pass_persistent<R, RB>(a, pd, smem_raw, [&](const PassCtx<R>& cx) {
    const int tid = cx.tid;
    for (int ph = 0; ph < pd.phase_count; ++ph) {
      const PhaseDesc* P = a.phases + pd.phase_begin + ph;
      const int nt = P->nt;
      if (nt < 0) {
        pass_swap<R, SB>(cx, cx.sg[P->gate_begin - pd.pgate_begin]);
        cx.sync();
        continue;
      }
      uint32_t base = 0;
      for (int i = 0; i < nt; ++i) base |= (uint32_t)((tid >> i) & 1) << P->tpos[i];
      const uint32_t sbase = swz_slot<SB>(cx.swz, base);
      A v[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) v[j] = cx.tile[sbase ^ P->soff[j]];
      const int g0 = P->gate_begin - pd.pgate_begin, g1 = g0 + P->gate_count;
      for (int gi = g0; gi < g1; ++gi) {
        const SGate<R>& g = cx.sg[gi];
        const int kind = g.kind;
        if (kind == PK_SKIP) continue;
        if ((base & g.cmT) != g.cvT) continue;
        R m[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = g.m[j];
        switch (kind) {
          case PK_DENSE: ph_kind<R, NR, PK_DENSE>(g.jt, v, m, g.cmR, g.cvR); break;
          case PK_DENSE_REAL: ph_kind<R, NR, PK_DENSE_REAL>(g.jt, v, m, g.cmR, g.cvR); break;
          case PK_DENSE_RX: ph_kind<R, NR, PK_DENSE_RX>(g.jt, v, m, g.cmR, g.cvR); break;
          case PK_XPERM: ph_kind<R, NR, PK_XPERM>(g.jt, v, m, g.cmR, g.cvR); break;
          case PK_ANTI: ph_kind<R, NR, PK_ANTI>(g.jt, v, m, g.cmR, g.cvR); break;
          case PK_DIAG_R: ph_kind<R, NR, PK_DIAG_R>(g.jt, v, m, g.cmR, g.cvR); break;
          default: {  // PK_DIAG_T (per-thread factor) / PK_DIAG_G (per-CTA factor, resolved at staging)
            R dr = m[0], di = m[1];
            if (g.tp >= 0) {
              const int b = (int)((base >> g.tp) & 1);
              if (!b && g.jt) break;  // jt carries diag_one0
              if (b) {
                dr = m[6];
                di = m[7];
              }
            }
            if (g.cmR) ph_scale<R, NR, true>(v, dr, di, g.cmR, g.cvR);
            else ph_scale<R, NR, false>(v, dr, di, 0, 0);
          } break;
        }
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) cx.tile[sbase ^ P->soff[j]] = v[j];
      cx.sync();
    }
  });
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename R, int RB> cudaError_t launch_t(const StreamArgs& a, const PassDesc& pd, cudaStream_t s) {
  const int T = 1 << (pd.k - RB);
  const size_t sm = pass_reg_smem(a.c64, pd, RB, a.n, true);
  cudaError_t e = cudaFuncSetAttribute(k_pass_reg<R, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_reg<R, RB>, T, sm);
  if (per_sm < 1) per_sm = 1;
  const int64_t W = (int64_t)a.slots << (a.n - pd.k);
  const int64_t grid = std::min<int64_t>(W, (int64_t)per_sm * num_sms());
  k_pass_reg<R, RB><<<(unsigned)grid, T, sm, s>>>(a, pd);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_pass_reg(const StreamArgs& a, const PassDesc& pd, cudaStream_t s) {
  if (pd.rb == 3) return a.c64 ? launch_t<float, 3>(a, pd, s) : launch_t<double, 3>(a, pd, s);
  if (pd.rb == 5) return a.c64 ? launch_t<float, 5>(a, pd, s) : launch_t<double, 5>(a, pd, s);
  return a.c64 ? launch_t<float, 4>(a, pd, s) : launch_t<double, 4>(a, pd, s);
}

}  // namespace qsb
