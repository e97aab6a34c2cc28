// Tile-fused Pauli expectation reducer (observe(), BASELINE cfg 3).
//
// <P> = Re[(-i)^ny * sum_i (-1)^popc(i & zy) conj(psi_i) psi_{i ^ x}]
//
// The terms are grouped on the host so that each group's X supports fit in one tile
// qubit set S (k qubits, always containing the low qubits for 32-byte runs); one launch
// per group reads every tile of every state exactly once and evaluates all of the
// group's terms on chip: pairs (l, l ^ x_local) stay inside the tile, Z/Y signs of the
// out-of-tile qubits are one per-tile sign.  Diagonal (Z-only) terms ride along with
// the first group.
//
// Full 12-qubit tiles use the register-mapped kernel: the group's terms are split into
// mappings whose X supports together fit in 4 tile positions; per mapping every thread
// loads the 16 amplitudes that differ only in those positions from the (swizzled,
// conflict-free) shared tile into registers, and every term of the mapping is then a
// compile-time pair pattern over those registers (its X letters in register space,
// its register Z signs a 16-bit mask) -- a few FP64 ops per pair, no shared-memory
// traffic or index arithmetic per pair.  Smaller tiles (n < 12) use the pair loop.
//
// The reduction is fixed-order (warp shfl_down, warp partials summed in order, tiles
// summed in order) -- deterministic, no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "qsb_device.cuh"
#include "qsb_launch.h"
#include "qsb_pass_common.cuh"

namespace qsb {

namespace {

constexpr int kET = 256;
#ifndef QSB_EV_L2_PREFETCH
#define QSB_EV_L2_PREFETCH 0
#endif
// L2 prefetch of the next item's runs in the register-mapped reducer: measured on B200 to
// make run-to-run times unstable (complex64 VQE24 reducer 53 - 130 ms per 32 points across
// processes) for no gain in the good case; off
constexpr bool kEvL2Prefetch = QSB_EV_L2_PREFETCH != 0;

__device__ __forceinline__ void prefetch_line_l2(const void* gmem) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(gmem));
}

// ---- pair-loop kernel (any tile size) -------------------------------------------

template <typename R>
__global__ void __launch_bounds__(kET) k_expval_tile(const typename Amp<R>::T* __restrict__ states, int n,
                                                    ExpvalGroup g, const ExpvalTerm* __restrict__ terms,
                                                    double* __restrict__ partial, int nterm_total) {
  using A = typename Amp<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int k = g.k, TL = 1 << k;
  A* tile = reinterpret_cast<A*>(smem_raw);
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(tile + TL);                      // [TL >> lowq]
  double* wsum = reinterpret_cast<double*>(hi_off + (TL >> g.lowq));              // [nterm][8 warps]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t slot = blockIdx.y;
  const uint64_t qmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t base = pdep64((uint64_t)blockIdx.x, ~g.smask & qmask);
  const A* st = states + (slot << n);
  const uint64_t lowm = (1ull << g.lowq) - 1;
  const uint64_t shi = g.smask & ~lowm;
  for (int h = tid; h < (TL >> g.lowq); h += kET) hi_off[h] = pdep64((uint64_t)h, shi);
  __syncthreads();
  for (int l = tid; l < TL; l += kET) tile[l] = st[base | ((uint64_t)l & lowm) | hi_off[l >> g.lowq]];
  __syncthreads();
  for (int t = 0; t < g.nterm; ++t) {
    const ExpvalTerm tm = terms[g.term_begin + t];
    double acc = 0.0;
    if (tm.xl == 0) {
      for (int l = tid; l < TL; l += kET) {
        const double w = norm2<R>(tile[l]);
        acc += (__popc((uint32_t)l & tm.zl) & 1) ? -w : w;
      }
    } else {
      const int h = 31 - __clz(tm.xl);
      for (int pi = tid; pi < (TL >> 1); pi += kET) {
        const uint32_t l = (uint32_t)insert_zero((uint64_t)pi, h);
        const A u = tile[l], v = tile[l ^ tm.xl];
        const double ur = u.x, ui = u.y, vr = v.x, vi = v.y;
        const double val = (tm.ny & 1) ? fma(ur, vi, -ui * vr) : fma(ur, vr, ui * vi);
        acc += (__popc(l & tm.zl) & 1) ? -val : val;
      }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) wsum[t * (kET / 32) + warp] = acc;
  }
  __syncthreads();
  for (int t = tid; t < g.nterm; t += kET) {  // fixed warp order per term
    const ExpvalTerm tm = terms[g.term_begin + t];
    double s = 0.0;
    for (int w = 0; w < kET / 32; ++w) s += wsum[t * (kET / 32) + w];
    if (__popcll(base & tm.zg) & 1) s = -s;
    partial[((int64_t)slot * gridDim.x + blockIdx.x) * nterm_total + tm.out] = s;
  }
}

// ---- register-mapped kernel (k = 12: 256 threads x 16 registers) -----------------

// (-1)^(bit j of zsig) * x as one integer op on the sign bit
__device__ __forceinline__ double flip_sign(double x, uint32_t zsig, int j) {
  const int hi = __double2hiint(x) ^ (int)((zsig << (31 - j)) & 0x80000000u);
  return __hiloint2double(hi, __double2loint(x));
}

__device__ __forceinline__ float flip_sign(float x, uint32_t zsig, int j) {
  return __int_as_float(__float_as_int(x) ^ (int)((zsig << (31 - j)) & 0x80000000u));
}

// sum over the 8 register pairs (j, j ^ XR), j without XR's top bit, of the signed
// Re / Im part of conj(v_j) v_{j ^ XR}; zsig bit j = Z sign of register j.  The products
// and the 8-term per-thread sum are in the state's precision (complex64: FP32, well inside
// the 1e-5 tolerance -- no conversions, half the FP work); everything after (warp, tile and
// state sums) is FP64.
template <typename R, int XR>
__device__ __forceinline__ double ev_pairs(const typename Amp<R>::T* v, uint32_t zsig, bool im) {
  constexpr int TOP = 1 << (31 - __builtin_clz(XR));
  R acc = (R)0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j & TOP) continue;
    const R ur = v[j].x, ui = v[j].y, vr = v[j ^ XR].x, vi = v[j ^ XR].y;
    const R val = im ? fma(ur, vi, -ui * vr) : fma(ur, vr, ui * vi);
    acc += flip_sign(val, zsig, j);
  }
  return (double)acc;
}

// empty asm with the amplitudes as in/out operands: the products of a term are not
// loop-invariant for the compiler, so it cannot hoist all 15 pair patterns' products
// out of the term loop (which spilled ~1.7 KB per thread)
__device__ __forceinline__ void opaque(double2& a) { asm volatile("" : "+d"(a.x), "+d"(a.y)); }
__device__ __forceinline__ void opaque(float2& a) { asm volatile("" : "+f"(a.x), "+f"(a.y)); }

template <typename R>
__device__ __forceinline__ double ev_term(const typename Amp<R>::T* v, uint32_t xr, uint32_t zsig, bool im) {
  switch (xr) {
    case 0: {
      if (sizeof(R) == 8) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += flip_sign(norm2<R>(v[j]), zsig, j);
        return acc;
      }
      R acc = (R)0;
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += flip_sign(fma(v[j].x, v[j].x, v[j].y * v[j].y), zsig, j);
      return (double)acc;
    }
#define QSB_EV_CASE(X) \
  case X: return ev_pairs<R, X>(v, zsig, im);
    QSB_EV_CASE(1) QSB_EV_CASE(2) QSB_EV_CASE(3) QSB_EV_CASE(4) QSB_EV_CASE(5) QSB_EV_CASE(6) QSB_EV_CASE(7)
    QSB_EV_CASE(8) QSB_EV_CASE(9) QSB_EV_CASE(10) QSB_EV_CASE(11) QSB_EV_CASE(12) QSB_EV_CASE(13) QSB_EV_CASE(14)
    QSB_EV_CASE(15)
#undef QSB_EV_CASE
    default: return 0.0;
  }
}

template <typename R>
__global__ void __launch_bounds__(kET, 2) k_expval_reg(const typename Amp<R>::T* __restrict__ states, int n,
                                                      int64_t slots, ExpvalGroup g,
                                                      const ExpvalTerm* __restrict__ terms,
                                                      const EvMap* __restrict__ maps, double* __restrict__ partial,
                                                      int nterm_total) {
  // persistent: the per-CTA tables are built once, then the CTA walks (slot, tile)
  // items with a grid stride (the L2 prefetch of the next item's runs is compiled out:
  // kEvL2Prefetch)
  using A = typename Amp<R>::T;
  constexpr int SB = sizeof(R) == 8 ? 3 : 4;
  constexpr int K = 12, TL = 1 << K, NT = K - 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* tile = reinterpret_cast<A*>(smem_raw);
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(tile + TL);       // [TL >> lowq]
  uint32_t* swz = reinterpret_cast<uint32_t*>(hi_off + (TL >> g.lowq));  // [TL >> SB]
  double* wsum = reinterpret_cast<double*>(swz + (TL >> SB));        // [nterm][8 warps]
  ExpvalTerm* sterm = reinterpret_cast<ExpvalTerm*>(wsum + (kET / 32) * g.nterm);  // [nterm]
  EvMap* smap = reinterpret_cast<EvMap*>(sterm + g.nterm);                       // [nmap]
  double* wred = reinterpret_cast<double*>(
      (reinterpret_cast<size_t>(smap + g.nmap) + 15) & ~(size_t)15);             // [8 warps][8][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t qmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t lowm = (1ull << g.lowq) - 1;
  const uint64_t shi = g.smask & ~lowm;
  for (int h = tid; h < (TL >> g.lowq); h += kET) hi_off[h] = pdep64((uint64_t)h, shi);
  const uint8_t* V = SB == 3 ? c_swz3 : c_swz4;
  for (int h = tid; h < (TL >> SB); h += kET) {
    uint32_t s = 0;
    for (int p = SB, hh = h; hh; ++p, hh >>= 1)
      if (hh & 1) s ^= V[p];
    swz[h] = s;
  }
  for (int t = tid; t < g.nterm; t += kET) sterm[t] = terms[g.term_begin + t];
  for (int m = tid; m < g.nmap; m += kET) smap[m] = maps[g.map_begin + m];
  __syncthreads();
  const int ntl = n - K;
  const int64_t tiles = (int64_t)1 << ntl, W = slots * tiles;
  const uint64_t outmask = ~g.smask & qmask;
  // per-thread constant parts of the gather (pdep / swizzle linear over disjoint bits)
  const uint64_t Pt = ((uint64_t)tid & lowm) | hi_off[tid >> g.lowq];
  const uint32_t St = swz_slot<SB>(swz, (uint32_t)tid);
  const int hstep = kET >> g.lowq;
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    const int64_t slot = w >> ntl;
    const uint64_t base = pdep64((uint64_t)(w & (tiles - 1)), outmask);
    const A* st = states + (slot << n);
    if (kEvL2Prefetch) {  // next item's runs into L2
      const int64_t wn = w + gridDim.x;
      if (wn < W) {
        const A* sn = states + ((wn >> ntl) << n) + pdep64((uint64_t)(wn & (tiles - 1)), outmask);
        for (int h = tid; h < (TL >> g.lowq); h += kET) prefetch_line_l2(sn + hi_off[h]);
      }
    }
#pragma unroll
    for (int i = 0; i < TL / kET; ++i) {  // all 16 loads of a thread in flight at once
      const A* src = st + (base | Pt | hi_off[i * hstep]);
      A* dst = tile + (St ^ swz_slot<SB>(swz, (uint32_t)(i * kET)));
      if (sizeof(A) == 16) cp_async16(dst, src);
      else cp_async8(dst, src);
    }
    cp_async_commit();
    cp_async_wait0();
    __syncthreads();
    for (int mi = 0; mi < g.nmap; ++mi) {
      const EvMap& m = smap[mi];
      uint32_t tb = 0;
#pragma unroll
      for (int i = 0; i < NT; ++i) tb |= (uint32_t)((tid >> i) & 1) << m.tpos[i];
      const uint32_t sbase = swz_slot<SB>(swz, tb);
      A v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tile[sbase ^ m.soff[j]];
      // terms in chunks of 8: each lane parks its per-term value in the warp's slice of
      // shared memory, then lane l sums the 8 entries (l & 3) * 8 .. + 7 of chunk term l >> 2
      // and two shuffles finish the warp sum -- one short dependency chain per chunk
      // instead of five dependent shuffles per term (fixed order: deterministic)
      // (complex64 only: measured -6 % there, +15 % for complex128, whose register budget
      // this loop shape strains)
      const int tend = m.term_begin + m.nterm;
      double* red = wred + warp * 256;
      if (sizeof(R) == 8) {
        for (int t = m.term_begin; t < tend; ++t) {
#pragma unroll
          for (int j = 0; j < 16; ++j) opaque(v[j]);
          const ExpvalTerm& tm = sterm[t - g.term_begin];
          double acc = ev_term<R>(v, tm.xr, tm.zsig, tm.ny & 1);
          acc = flip_sign(acc, __popc(tb & tm.zl), 0);
          for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
          if (lane == 0) wsum[(t - g.term_begin) * (kET / 32) + warp] = acc;
        }
        continue;
      }
      for (int t0 = m.term_begin; t0 < tend; t0 += 8) {
        const int cnt = tend - t0 < 8 ? tend - t0 : 8;
        for (int c = 0; c < cnt; ++c) {
#pragma unroll
          for (int j = 0; j < 16; ++j) opaque(v[j]);
          const ExpvalTerm& tm = sterm[t0 + c - g.term_begin];
          double acc = ev_term<R>(v, tm.xr, tm.zsig, tm.ny & 1);
          red[c * 32 + lane] = flip_sign(acc, __popc(tb & tm.zl), 0);
        }
        __syncwarp();
        const int c = lane >> 2, q = lane & 3;
        double s = 0.0;
        if (c < cnt) {
#pragma unroll
          for (int i = 0; i < 8; ++i) s += red[c * 32 + q * 8 + i];
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (q == 0 && c < cnt) wsum[(t0 + c - g.term_begin) * (kET / 32) + warp] = s;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int t = tid; t < g.nterm; t += kET) {  // fixed warp order per term
      const ExpvalTerm& tm = sterm[t];
      double s = 0.0;
      for (int w2 = 0; w2 < kET / 32; ++w2) s += wsum[t * (kET / 32) + w2];
      if (__popcll(base & tm.zg) & 1) s = -s;
      partial[w * nterm_total + tm.out] = s;
    }
    __syncthreads();
  }
}

// partials: the accumulating kernel's [slot][chunk][term] (path 0) or the pair-loop
// kernel's [slot][tile][term] (path 1); consecutive threads (terms) read consecutive
// words; chunks / tiles summed in order (deterministic)
__global__ void k_expval_tile_finish(const double* pacc, int nchunks, const double* ptile, int ntiles, int64_t slots,
                                     int nterm, const ExpvalTerm* terms_by_out, double* out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= slots * nterm) return;
  const int t = (int)(idx % nterm);
  const int64_t slot = idx / nterm;
  const ExpvalTerm tm = terms_by_out[t];
  const int cnt = tm.path ? ntiles : nchunks;
  const double* p = (tm.path ? ptile : pacc) + slot * cnt * nterm + t;
  double s = 0.0;
  for (int64_t b = 0; b < cnt; ++b) s += p[b * nterm];
  if (tm.xg | tm.xl) s *= 2.0;
  out[idx] = ((tm.ny & 3) >= 2) ? -s : s;
}

// ---- per-thread accumulating kernel (k = 12; the cfg 3 hot path) ---------------------
//
// One CTA = one (state, chunk of consecutive tiles).  Tiles are double-buffered with
// cp.async; per register mapping every thread loads its 16 amplitudes, and per CLASS of
// terms (same register X pattern XR) it forms the 8 pair products conj(v_j) v_{j^XR}
// once; each term of the class is then 8 signed adds of their real or imaginary parts
// (16 for the diagonal class, of |v_j|^2), signed by the thread's and the tile's Z
// parity, and ADDED TO THE THREAD'S OWN ACCUMULATOR for that term in shared memory.  No
// cross-thread reduction happens per tile: one fixed-order reduction per CTA at the end.
// Partials [state][chunk][term] are summed over chunks in order by the finish kernel --
// deterministic, and independent of how many states a launch holds.

template <typename R, int XR>
__device__ __forceinline__ void ev_class(const typename Amp<R>::T* v, const ExpvalTerm* st, int t0, int t1,
                                         double* acc, int tid, uint32_t tb, uint64_t base) {
  constexpr int TOP = XR ? 1 << (31 - __builtin_clz(XR)) : 0;
  if (XR == 0) {
    R nv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) nv[j] = fma(v[j].x, v[j].x, v[j].y * v[j].y);
    for (int t = t0; t < t1; ++t) {
      const ExpvalTerm& tm = st[t];
      R s = (R)0;
#pragma unroll
      for (int j = 0; j < 16; ++j) s += flip_sign(nv[j], tm.zsig, j);
      const uint32_t par = (__popc(tb & tm.zl) + __popcll(base & tm.zg)) & 1;
      acc[t * kET + tid] += flip_sign((double)s, par, 0);
    }
    return;
  }
  R pr[8], pi[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = ((k & ~(TOP - 1)) << 1) | (k & (TOP - 1));  // k with a 0 inserted at TOP
    const R ur = v[j].x, ui = v[j].y, vr = v[j ^ XR].x, vi = v[j ^ XR].y;
    pr[k] = fma(ur, vr, ui * vi);
    pi[k] = fma(ur, vi, -ui * vr);
  }
  for (int t = t0; t < t1; ++t) {
    const ExpvalTerm& tm = st[t];
    R s = (R)0;
    if (tm.ny & 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) s += flip_sign(pi[k], tm.zsig, ((k & ~(TOP - 1)) << 1) | (k & (TOP - 1)));
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) s += flip_sign(pr[k], tm.zsig, ((k & ~(TOP - 1)) << 1) | (k & (TOP - 1)));
    }
    const uint32_t par = (__popc(tb & tm.zl) + __popcll(base & tm.zg)) & 1;
    acc[t * kET + tid] += flip_sign((double)s, par, 0);
  }
}

template <typename R>
__device__ __forceinline__ void ev_class_dispatch(int xr, const typename Amp<R>::T* v, const ExpvalTerm* st, int t0,
                                                  int t1, double* acc, int tid, uint32_t tb, uint64_t base) {
  switch (xr) {
#define QSB_EV_CLS(X) \
  case X: ev_class<R, X>(v, st, t0, t1, acc, tid, tb, base); break;
    QSB_EV_CLS(0) QSB_EV_CLS(1) QSB_EV_CLS(2) QSB_EV_CLS(3) QSB_EV_CLS(4) QSB_EV_CLS(5) QSB_EV_CLS(6) QSB_EV_CLS(7)
    QSB_EV_CLS(8) QSB_EV_CLS(9) QSB_EV_CLS(10) QSB_EV_CLS(11) QSB_EV_CLS(12) QSB_EV_CLS(13) QSB_EV_CLS(14)
    QSB_EV_CLS(15)
#undef QSB_EV_CLS
    default: break;
  }
}

template <typename R>
__global__ void __launch_bounds__(kET, 1) k_expval_acc(const typename Amp<R>::T* __restrict__ states, int n,
                                                      ExpvalGroup g, const ExpvalTerm* __restrict__ terms,
                                                      const EvMap* __restrict__ maps, double* __restrict__ partial,
                                                      int nterm_total, int nchunks) {
  using A = typename Amp<R>::T;
  constexpr int SB = sizeof(R) == 8 ? 3 : 4;
  constexpr int K = 12, TL = 1 << K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* tiles = reinterpret_cast<A*>(smem_raw);                              // [2][TL]
  double* acc = reinterpret_cast<double*>(tiles + 2 * TL);                // [nterm][kET]
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(acc + g.nterm * kET);    // [TL >> lowq]
  uint32_t* swz = reinterpret_cast<uint32_t*>(hi_off + (TL >> g.lowq));   // [TL >> SB]
  ExpvalTerm* sterm = reinterpret_cast<ExpvalTerm*>(
      (reinterpret_cast<size_t>(swz + (TL >> SB)) + 15) & ~(size_t)15);  // [nterm]
  EvMap* smap = reinterpret_cast<EvMap*>(sterm + g.nterm);                // [nmap]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t qmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t lowm = (1ull << g.lowq) - 1;
  const uint64_t shi = g.smask & ~lowm;
  for (int h = tid; h < (TL >> g.lowq); h += kET) hi_off[h] = pdep64((uint64_t)h, shi);
  const uint8_t* V = SB == 3 ? c_swz3 : c_swz4;
  for (int h = tid; h < (TL >> SB); h += kET) {
    uint32_t sw = 0;
    for (int p = SB, hh = h; hh; ++p, hh >>= 1)
      if (hh & 1) sw ^= V[p];
    swz[h] = sw;
  }
  for (int t = tid; t < g.nterm; t += kET) sterm[t] = terms[g.term_begin + t];
  for (int m = tid; m < g.nmap; m += kET) smap[m] = maps[g.map_begin + m];
  for (int i = tid; i < g.nterm * kET; i += kET) acc[i] = 0.0;
  __syncthreads();
  const int ntl = n - K;
  const int64_t ntiles = (int64_t)1 << ntl;
  const int64_t slot = blockIdx.x / nchunks, chunk = blockIdx.x % nchunks;
  const int64_t tpc = ntiles / nchunks, w0 = chunk * tpc;
  const uint64_t outmask = ~g.smask & qmask;
  const A* st = states + (slot << n);
  const uint64_t Pt = ((uint64_t)tid & lowm) | hi_off[tid >> g.lowq];
  const uint32_t St = swz_slot<SB>(swz, (uint32_t)tid);
  const int hstep = kET >> g.lowq;
  auto load = [&](int64_t w, A* dst_tile) {
    const uint64_t base = pdep64((uint64_t)w, outmask);
#pragma unroll
    for (int i = 0; i < TL / kET; ++i) {
      const A* src = st + (base | Pt | hi_off[i * hstep]);
      A* dst = dst_tile + (St ^ swz_slot<SB>(swz, (uint32_t)(i * kET)));
      if (sizeof(A) == 16) cp_async16(dst, src);
      else cp_async8(dst, src);
    }
    cp_async_commit();
  };
  load(w0, tiles);
  for (int64_t i = 0; i < tpc; ++i) {
    if (i + 1 < tpc) {
      load(w0 + i + 1, tiles + ((i + 1) & 1) * TL);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
    const A* tile = tiles + (i & 1) * TL;
    const uint64_t base = pdep64((uint64_t)(w0 + i), outmask);
    for (int mi = 0; mi < g.nmap; ++mi) {
      const EvMap& m = smap[mi];
      uint32_t tb = 0;
#pragma unroll
      for (int b = 0; b < K - 4; ++b) tb |= (uint32_t)((tid >> b) & 1) << m.tpos[b];
      const uint32_t sbase = swz_slot<SB>(swz, tb);
      A v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = tile[sbase ^ m.soff[j]];
      const int tend = m.term_begin - g.term_begin + m.nterm;
      for (int t = m.term_begin - g.term_begin; t < tend;) {  // classes: runs of equal xr
        const uint32_t xr = sterm[t].xr;
        int e = t + 1;
        while (e < tend && sterm[e].xr == xr) ++e;
#pragma unroll
        for (int j = 0; j < 16; ++j) opaque(v[j]);  // no hoisting of every class's products
        ev_class_dispatch<R>((int)xr, v, sterm, t, e, acc, tid, tb, base);
        t = e;
      }
    }
    __syncthreads();  // the buffer is refilled by the load issued next iteration
  }
  // one fixed-order reduction per CTA: warp w sums terms w, w + 8, ...; lane l adds the
  // accumulators of threads l, l + 32, ... in order, then a fixed shuffle tree
  for (int t = warp; t < g.nterm; t += kET / 32) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kET / 32; ++r) s += acc[t * kET + r * 32 + lane];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) partial[(slot * nchunks + chunk) * nterm_total + sterm[t].out] = s;
  }
}

}  // namespace

void launch_expval_tile(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                        const ExpvalTerm* terms, const EvMap* maps, double* partial, int nterm_total,
                        cudaStream_t s) {
  dim3 grid((unsigned)(1ull << (n - g.k)), (unsigned)slots);
  const size_t amp = c64 ? 8 : 16;
  if (g.nmap > 0) {
    const size_t smem = amp * ((size_t)1 << g.k) + sizeof(uint64_t) * ((size_t)1 << (g.k - g.lowq)) +
                        sizeof(uint32_t) * ((size_t)1 << (g.k - (c64 ? 4 : 3))) +
                        sizeof(double) * (kET / 32) * (size_t)g.nterm + sizeof(ExpvalTerm) * (size_t)g.nterm +
                        sizeof(EvMap) * (size_t)g.nmap + 16 + sizeof(double) * 8 * kET;
    // driver queries cached per (device, precision, smem): a group launch stays a pure
    // enqueue (no attribute / occupancy calls between the kernels of an observe)
    struct OccKey { int dev, c64; size_t smem; };
    static thread_local std::vector<std::pair<OccKey, int>> occ;  // -> resident CTAs on the device
    int dev = 0;
    cudaGetDevice(&dev);
    int resident = 0;
    for (const auto& e : occ)
      if (e.first.dev == dev && e.first.c64 == c64 && e.first.smem == smem) resident = e.second;
    if (!resident) {
      // the attribute is a ceiling: set it to the device's opt-in maximum once, so that
      // cached launches of any group size stay valid
      int sms = 148, per_sm = 1, optin = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      const int cap = std::max(optin, (int)smem);
      if (c64) {
        cudaFuncSetAttribute(k_expval_reg<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_expval_reg<float>, kET, smem);
      } else {
        cudaFuncSetAttribute(k_expval_reg<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_expval_reg<double>, kET, smem);
      }
      resident = std::max(1, per_sm) * sms;
      occ.push_back({OccKey{dev, c64, smem}, resident});
    }
    const int64_t W = (int64_t)grid.x * slots;
    const unsigned pg = (unsigned)std::min<int64_t>(W, (int64_t)resident);
    if (c64)
      k_expval_reg<float><<<pg, kET, smem, s>>>((const float2*)states, n, slots, g, terms, maps, partial,
                                                nterm_total);
    else
      k_expval_reg<double><<<pg, kET, smem, s>>>((const double2*)states, n, slots, g, terms, maps, partial,
                                                 nterm_total);
    return;
  }
  const size_t smem = amp * ((size_t)1 << g.k) + sizeof(uint64_t) * ((size_t)1 << (g.k - g.lowq)) +
                      sizeof(double) * (kET / 32) * (size_t)g.nterm;
  if (c64) {
    cudaFuncSetAttribute(k_expval_tile<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_expval_tile<float><<<grid, kET, smem, s>>>((const float2*)states, n, g, terms, partial, nterm_total);
  } else {
    cudaFuncSetAttribute(k_expval_tile<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_expval_tile<double><<<grid, kET, smem, s>>>((const double2*)states, n, g, terms, partial, nterm_total);
  }
}

void launch_expval_tile_finish(const double* partial_acc, int nchunks, const double* partial_tile, int ntiles,
                               int64_t slots, int nterm, const ExpvalTerm* terms_by_out, double* out, cudaStream_t s) {
  const int64_t items = slots * nterm;
  k_expval_tile_finish<<<(unsigned)((items + 127) / 128), 128, 0, s>>>(partial_acc, nchunks, partial_tile, ntiles,
                                                                      slots, nterm, terms_by_out, out);
}

// chunks per state: a function of n only (results do not depend on the batch); 128
// chunks of 32 tiles at 24 qubits
int expval_acc_chunks(int n) {
  const int64_t ntiles = n >= 12 ? (1ll << (n - 12)) : 1;
  return (int)std::min<int64_t>(ntiles, 128);
}

void launch_expval_acc(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                       const ExpvalTerm* terms, const EvMap* maps, double* partial, int nterm_total, cudaStream_t s) {
  const size_t amp = c64 ? 8 : 16;
  const size_t smem = 2 * amp * 4096 + sizeof(double) * kET * (size_t)g.nterm + sizeof(uint64_t) * (4096 >> g.lowq) +
                      sizeof(uint32_t) * (4096 >> (c64 ? 4 : 3)) + 16 + sizeof(ExpvalTerm) * (size_t)g.nterm +
                      sizeof(EvMap) * (size_t)g.nmap;
  static thread_local int set_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev != dev) {  // the attribute is a ceiling: the device's opt-in maximum, once
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_expval_acc<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaFuncSetAttribute(k_expval_acc<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    set_dev = dev;
  }
  const int nchunks = expval_acc_chunks(n);
  const unsigned grid = (unsigned)(slots * nchunks);
  if (c64)
    k_expval_acc<float><<<grid, kET, smem, s>>>((const float2*)states, n, g, terms, maps, partial, nterm_total, nchunks);
  else
    k_expval_acc<double><<<grid, kET, smem, s>>>((const double2*)states, n, g, terms, maps, partial, nterm_total,
                                                 nchunks);
}

}  // namespace qsb
