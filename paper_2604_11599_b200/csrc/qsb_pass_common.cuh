// Pass prologue / epilogue shared by the generic register-blocked kernel
// (qsb_pass_reg.cu) and the NVRTC-specialised per-pass kernels (qsb_jit.cpp), so both
// execute the identical load / collapse / marginal / store sequence.
#pragma once
#include "qsb_device.cuh"

namespace qsb {

__constant__ uint8_t c_swz3[16] = {1, 2, 4, 3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7, 1, 2};
__constant__ uint8_t c_swz4[16] = {1, 2, 4, 8, 3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 1};

// a pass gate staged in shared memory with its CTA-uniform decisions resolved
template <typename R> struct SGate {
  int32_t kind, jt, jt2, tp;
  uint32_t cmR, cvR, cmT, cvT;
  R m[8];
};

template <typename R> struct PassCtx {
  typename Amp<R>::T* tile;
  SGate<R>* sg;
  uint64_t* hi_off;
  uint32_t* swz;
  double* red;
  int tid, T, TL, n;
  int64_t slot;
  uint64_t S, qmask, base_phys, base_log;
};

__device__ __forceinline__ uint64_t pext64(uint64_t v, uint64_t mask) {
  uint64_t out = 0;
  int j = 0;
  for (uint64_t m = mask; m; m &= m - 1, ++j)
    if (v & (m & (~m + 1))) out |= 1ull << j;
  return out;
}

template <int SB> __device__ __forceinline__ uint32_t swz_slot(const uint32_t* swz, uint32_t l) {
  return l ^ swz[l >> SB];
}

// Shared-memory layout, tables, gate staging, gather of the tile (frame + pending
// collapse).  Returns false when the trajectory is dead (DegenerateNorm earlier).
template <typename R, int RB>
__device__ __forceinline__ bool pass_begin(const StreamArgs& a, const PassDesc& pd, unsigned char* smem_raw,
                                           PassCtx<R>& cx) {
  using A = typename Amp<R>::T;
  constexpr int SB = sizeof(R) == 8 ? 3 : 4;
  const int k = pd.k;
  cx.TL = 1 << k;
  cx.T = cx.TL >> RB;
  cx.tile = reinterpret_cast<A*>(smem_raw);
  cx.sg = reinterpret_cast<SGate<R>*>(smem_raw + sizeof(A) * cx.TL);
  cx.hi_off = reinterpret_cast<uint64_t*>(cx.sg + pd.pgate_count);
  cx.swz = reinterpret_cast<uint32_t*>(cx.hi_off + (cx.TL >> pd.lowq));
  cx.red = reinterpret_cast<double*>(cx.swz + (cx.TL >> SB));
  cx.tid = threadIdx.x;
  cx.slot = blockIdx.y;
  const TrajCtl* c = a.ctl + cx.slot;
  if (c->status) return false;
  cx.n = a.n;
  cx.qmask = (a.n >= 64) ? ~0ull : ((1ull << a.n) - 1);
  cx.S = pd.smask;
  const uint64_t F = c->frame & ~pd.clear_before;
  const bool pending = pd.prologue && c->pending;
  const uint64_t Kp = c->kmask, Vp = c->kval;
  const R sre = (R)c->sre, sim = (R)c->sim;
  cx.base_phys = pdep64((uint64_t)blockIdx.x, ~cx.S & cx.qmask);
  cx.base_log = cx.base_phys ^ (F & ~cx.S);
  uint32_t fl = 0;
  for (int j = 0; j < k; ++j)
    if ((F >> pd.sq[j]) & 1) fl |= 1u << j;
  const uint64_t lowm = (1ull << pd.lowq) - 1;
  const uint64_t shi = cx.S & ~lowm;
  const int tid = cx.tid, T = cx.T, TL = cx.TL;
  for (int h = tid; h < (TL >> pd.lowq); h += T) cx.hi_off[h] = pdep64((uint64_t)h, shi);
  const uint8_t* V = SB == 3 ? c_swz3 : c_swz4;
  for (int h = tid; h < (TL >> SB); h += T) {
    uint32_t s = 0;
    for (int p = SB, hh = h; hh; ++p, hh >>= 1)
      if (hh & 1) s ^= V[p];
    cx.swz[h] = s;
  }
  {  // stage the pass's gates: guards, out-of-tile controls, per-CTA diagonal factors
    const uint32_t* gw = a.guards + cx.slot * a.gwords;
    const double* mats = a.mats + cx.slot * a.mat_stride;
    for (int i = tid; i < pd.pgate_count; i += T) {
      const PhaseGate g = a.phase_gates[pd.pgate_begin + i];
      SGate<R> s;
      double m[8];
      const double* src = mats + (int64_t)g.mat * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) m[j] = src[j];
      int kind = g.kind;
      bool skip = (g.guard >= 0 && !((gw[g.guard >> 5] >> (g.guard & 31)) & 1u)) || ((cx.base_log & g.gcm) != g.gcv);
      if (kind == PK_DIAG_G) kind = PK_DIAG_T;  // same code path, tp = -1
      if (kind == PK_DENSE) {
        if (m[1] == 0.0 && m[3] == 0.0 && m[5] == 0.0 && m[7] == 0.0) kind = PK_DENSE_REAL;
        else if (m[1] == 0.0 && m[7] == 0.0 && m[2] == 0.0 && m[4] == 0.0) kind = PK_DENSE_RX;
      } else if (g.kind == PK_DIAG_G) {
        int b = (int)((cx.base_log >> g.tp) & 1);
        if (!b && g.diag_one0) skip = true;
        if (b) {
          m[0] = m[6];
          m[1] = m[7];
        }
      }
      s.kind = skip ? PK_SKIP : kind;
      s.jt = g.kind == PK_DIAG_T ? g.diag_one0 : g.jt;
      s.jt2 = g.jt2;
      s.tp = (g.kind == PK_DIAG_T || g.kind == PK_SWAP_R) ? g.tp : -1;
      s.cmR = g.cmR;
      s.cvR = g.cvR;
      s.cmT = g.cmT;
      s.cvT = g.cvT;
#pragma unroll
      for (int j = 0; j < 8; ++j) s.m[j] = (R)m[j];
      cx.sg[i] = s;
    }
  }
  __syncthreads();
  const A* st = reinterpret_cast<const A*>(a.state) + (cx.slot << cx.n);
  for (int l = tid; l < TL; l += T) {
    uint64_t p = cx.base_phys | ((uint64_t)l & lowm) | cx.hi_off[l >> pd.lowq];
    A v = pd.init_zero ? mk<R>(p == 0 ? (R)1 : (R)0, (R)0) : st[p];
    if (pending) {
      if ((p & Kp) != Vp) v = mk<R>(0, 0);
      else v = mk<R>(fma(sre, v.x, -sim * v.y), fma(sre, v.y, sim * v.x));
    }
    cx.tile[swz_slot<SB>(cx.swz, (uint32_t)l ^ fl)] = v;
  }
  __syncthreads();
  return true;
}

// swap-only phase: tile positions tp, jt2; controls on the full tile index
template <typename R, int SB> __device__ __forceinline__ void pass_swap(PassCtx<R>& cx, const SGate<R>& g) {
  using A = typename Amp<R>::T;
  if (g.kind != PK_SKIP) {
    const int lo = g.tp < g.jt2 ? g.tp : g.jt2, hi = g.tp < g.jt2 ? g.jt2 : g.tp;
    for (int qd = cx.tid; qd < (cx.TL >> 2); qd += cx.T) {
      uint32_t b = (uint32_t)insert_zero(insert_zero((uint64_t)qd, lo), hi);
      if ((b & g.cmT) != g.cvT) continue;
      uint32_t la = swz_slot<SB>(cx.swz, b | (1u << g.tp)), lb = swz_slot<SB>(cx.swz, b | (1u << g.jt2));
      A x = cx.tile[la];
      cx.tile[la] = cx.tile[lb];
      cx.tile[lb] = x;
    }
  }
}

// epilogue: per-tile marginal of the next region's measured qubits (fixed order), scatter
template <typename R, int SB>
__device__ __forceinline__ void pass_end(const StreamArgs& a, const PassDesc& pd, PassCtx<R>& cx) {
  using A = typename Amp<R>::T;
  const int tid = cx.tid, T = cx.T, TL = cx.TL;
  if (pd.epi) {
    const int ml = pd.m_local;
    const int nb = 1 << ml;
    uint32_t mlm = 0;
    for (int j = 0; j < ml; ++j) mlm |= 1u << pd.mloc[j];
    const uint32_t free_mask = ((uint32_t)TL - 1) & ~mlm;
    const int members = TL >> ml;
    const uint64_t t_log = pext64(cx.base_log, ~cx.S & cx.qmask);
    double* out = a.partial + cx.slot * a.partial_stride + (int64_t)t_log * nb;
    if (nb <= T) {
      const int tp = T / nb;
      const int b = tid / tp, j = tid % tp;
      uint32_t bpos = 0;
      for (int jj = 0; jj < ml; ++jj)
        if ((b >> jj) & 1) bpos |= 1u << pd.mloc[jj];
      double s = 0.0;
      for (int r = j; r < members; r += tp) {
        uint32_t l = (uint32_t)pdep64((uint64_t)r, free_mask) | bpos;
        s += norm2<R>(cx.tile[swz_slot<SB>(cx.swz, l)]);
      }
      cx.red[tid] = s;
      __syncthreads();
      if (j == 0) {
        double tot = 0.0;
        for (int jj = 0; jj < tp; ++jj) tot += cx.red[b * tp + jj];
        out[b] = tot;
      }
    } else {
      for (int b = tid; b < nb; b += T) {
        uint32_t bpos = 0;
        for (int jj = 0; jj < ml; ++jj)
          if ((b >> jj) & 1) bpos |= 1u << pd.mloc[jj];
        double s = 0.0;
        for (int r = 0; r < members; ++r) {
          uint32_t l = (uint32_t)pdep64((uint64_t)r, free_mask) | bpos;
          s += norm2<R>(cx.tile[swz_slot<SB>(cx.swz, l)]);
        }
        out[b] = s;
      }
    }
  }
  A* st = reinterpret_cast<A*>(a.state) + (cx.slot << cx.n);
  const uint64_t lowm = (1ull << pd.lowq) - 1;
  for (int l = tid; l < TL; l += T) {
    uint64_t p = cx.base_phys | ((uint64_t)l & lowm) | cx.hi_off[l >> pd.lowq];
    st[p] = cx.tile[swz_slot<SB>(cx.swz, (uint32_t)l)];
  }
}

// dynamic shared memory of a register-blocked pass
__host__ __device__ inline size_t pass_reg_smem(int c64, const PassDesc& pd, int rb) {
  const int sb = c64 ? 4 : 3;
  const size_t amp = c64 ? 8 : 16;
  const size_t sgate = c64 ? 64 : 96;
  return (amp << pd.k) + sgate * pd.pgate_count + (sizeof(uint64_t) << (pd.k - pd.lowq)) +
         (sizeof(uint32_t) << (pd.k - sb)) + sizeof(double) * (1u << (pd.k - rb));
}

}  // namespace qsb
