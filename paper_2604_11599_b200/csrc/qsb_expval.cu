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
// Full 12-qubit tiles use the ACCUMULATING kernel (k_expval_acc, below): the group's
// terms are split into mappings whose X supports together fit in 4 tile positions; per
// mapping every thread loads the 16 amplitudes that differ only in those positions from
// the (swizzled, conflict-free) shared tile into registers; per class of terms with the
// same register X pattern it forms the 8 pair products once, and each term is then a
// 3-level signed butterfly (7 FMA) added to the thread's own accumulator -- no
// cross-thread reduction per tile.  Terms with more than 4 X letters inside a tile, and
// tiles of n < 12 qubits, use the pair loop (k_expval_tile).
//
// Every reduction is fixed-order (per-thread accumulators summed in thread order, warp
// shfl_down trees, chunks / tiles summed in order) -- deterministic, no atomics, and
// independent of how many states one launch holds.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "qsb_device.cuh"
#include "qsb_launch.h"
#include "qsb_pass_common.cuh"

namespace qsb {

namespace {

constexpr int kET = 256;
constexpr int kEvTilesPerCta = 32;  // upper bound of the accumulating kernel's tiles per CTA
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

// empty asm with the amplitudes as in/out operands: the products of a class are not
// loop-invariant for the compiler, so it cannot hoist every class's products out of the
// class loop (register spills)
__device__ __forceinline__ void opaque(double2& a) { asm volatile("" : "+d"(a.x), "+d"(a.y)); }
__device__ __forceinline__ void opaque(float2& a) { asm volatile("" : "+f"(a.x), "+f"(a.y)); }

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

// x with its sign bit XORed with bit 31 of m (one LOP3 on the high word)
__device__ __forceinline__ double sgn(double x, uint32_t m) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((unsigned long long)m << 32));
}
__device__ __forceinline__ float sgn(float x, uint32_t m) { return __int_as_float(__float_as_int(x) ^ (int)m); }

// per term of the accumulating kernel (shared memory): the Z sign (+1 / -1) of register
// bit b, so that every butterfly step below is one FMA (no sign-bit integer ops)
template <typename R> struct AccTerm {
  R s[4];
};

// sum_j (-1)^{j . zr} x_j over the register subspace spanned by bits B0 < B1 < B2 (< B3):
// a butterfly whose level over bit b adds or subtracts with the term's sign of bit b
template <typename R, int B0, int B1, int B2>
__device__ __forceinline__ R signed_sum8(const R* x, const AccTerm<R>& a) {
  const R q0 = fma(a.s[B0], x[1], x[0]), q1 = fma(a.s[B0], x[3], x[2]);
  const R q2 = fma(a.s[B0], x[5], x[4]), q3 = fma(a.s[B0], x[7], x[6]);
  const R r0 = fma(a.s[B1], q1, q0), r1 = fma(a.s[B1], q3, q2);
  return fma(a.s[B2], r1, r0);
}

template <typename R, int XR>
__device__ __forceinline__ void ev_class(const typename Amp<R>::T* v, const AccTerm<R>* __restrict__ at, int t0, int t1,
                                         int im0, double* __restrict__ acc, int tid, uint32_t pw) {
  if (XR == 0) {  // diagonal terms: sum_j (-1)^{j . zr} |v_j|^2 over all 16 registers
    R nv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) nv[j] = fma(v[j].x, v[j].x, v[j].y * v[j].y);
    for (int t = t0; t < t1; ++t) {
      const AccTerm<R> a = at[t];
      const R lo = signed_sum8<R, 0, 1, 2>(nv, a), hi = signed_sum8<R, 0, 1, 2>(nv + 8, a);
      const R s = fma(a.s[3], hi, lo);
      acc[t * kET + tid] += sgn((double)s, (pw << (31 - t)) & 0x80000000u);
    }
    return;
  }
  constexpr int TOP = 31 - __builtin_clz(XR);  // the pair partner differs in XR; j has TOP clear
  constexpr int B0 = TOP == 0 ? 1 : 0;
  constexpr int B1 = (TOP <= 1) ? 2 : 1;
  constexpr int B2 = (TOP <= 2) ? 3 : 2;
  R pr[8], pi[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = (((k >> 2) & 1) << B2) | (((k >> 1) & 1) << B1) | ((k & 1) << B0);
    const R ur = v[j].x, ui = v[j].y, vr = v[j ^ XR].x, vi = v[j ^ XR].y;
    pr[k] = fma(ur, vr, ui * vi);
    pi[k] = fma(ur, vi, -ui * vr);
  }
#pragma unroll 2
  for (int t = t0; t < im0; ++t) {  // Re terms (even number of Y letters)
    const AccTerm<R> a = at[t];
    const R s = signed_sum8<R, B0, B1, B2>(pr, a);
    acc[t * kET + tid] += sgn((double)s, (pw << (31 - t)) & 0x80000000u);
  }
#pragma unroll 2
  for (int t = im0; t < t1; ++t) {  // Im terms
    const AccTerm<R> a = at[t];
    const R s = signed_sum8<R, B0, B1, B2>(pi, a);
    acc[t * kET + tid] += sgn((double)s, (pw << (31 - t)) & 0x80000000u);
  }
}

template <typename R>
__device__ __forceinline__ void ev_class_dispatch(int xr, const typename Amp<R>::T* v, const AccTerm<R>* at, int t0,
                                                  int t1, int im0, double* acc, int tid, uint32_t pw) {
  switch (xr) {
#define QSB_EV_CLS(X) \
  case X: ev_class<R, X>(v, at, t0, t1, im0, acc, tid, pw); break;
    QSB_EV_CLS(0) QSB_EV_CLS(1) QSB_EV_CLS(2) QSB_EV_CLS(3) QSB_EV_CLS(4) QSB_EV_CLS(5) QSB_EV_CLS(6) QSB_EV_CLS(7)
    QSB_EV_CLS(8) QSB_EV_CLS(9) QSB_EV_CLS(10) QSB_EV_CLS(11) QSB_EV_CLS(12) QSB_EV_CLS(13) QSB_EV_CLS(14)
    QSB_EV_CLS(15)
#undef QSB_EV_CLS
    default: break;
  }
}


// NBUF tile buffers: 2 (complex64, 32 KiB tiles) double-buffers the loads; complex128 (64
// KiB tiles) keeps one so that two CTAs fit an SM and each hides the other's loads
template <typename R, int NBUF>
__global__ void __launch_bounds__(kET, 2) k_expval_acc(const typename Amp<R>::T* __restrict__ states, int n,
                                                      ExpvalGroup g, const ExpvalTerm* __restrict__ terms,
                                                      const EvMap* __restrict__ maps, const EvClass* __restrict__ classes,
                                                      double* __restrict__ partial, int nterm_total, int nchunks) {
  using A = typename Amp<R>::T;
  constexpr int SB = sizeof(R) == 8 ? 3 : 4;
  constexpr int K = 12, TL = 1 << K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // layout as byte offsets from smem_raw (pointer arithmetic keeps the shared address space:
  // no generic loads)
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    unsigned char* p = smem_raw + off;
    off = (off + bytes + 15) & ~(size_t)15;
    return p;
  };
  A* tiles = reinterpret_cast<A*>(carve(sizeof(A) * NBUF * TL));                    // [NBUF][TL]
  double* acc = reinterpret_cast<double*>(carve(sizeof(double) * g.nterm * kET));   // [nterm][kET]
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * (TL >> g.lowq)));
  uint32_t* swz = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * (TL >> SB)));
  AccTerm<R>* at = reinterpret_cast<AccTerm<R>*>(carve(sizeof(AccTerm<R>) * g.nterm));
  EvClass* cls = reinterpret_cast<EvClass*>(carve(sizeof(EvClass) * g.ncls));
  EvMap* smap = reinterpret_cast<EvMap*>(carve(sizeof(EvMap) * g.nmap));
  uint32_t* szl = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * g.nterm));
  uint64_t* ibase = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * kEvTilesPerCta));  // pdep(i) of the chunk's tiles
  uint32_t* tword = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * 2));       // tile parity words
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
  for (int m = tid; m < g.nmap; m += kET) smap[m] = maps[g.map_begin + m];
  for (int t = tid; t < g.nterm; t += kET) {
    const ExpvalTerm e = terms[g.term_begin + t];
    AccTerm<R> a;
    // register bit b's Z sign: zsig bit (1 << b) = parity of that register's tile position
    for (int b = 0; b < 4; ++b) a.s[b] = ((e.zsig >> (1u << b)) & 1u) ? (R)-1 : (R)1;
    at[t] = a;
    szl[t] = e.zl;
  }
  for (int c = tid; c < g.ncls; c += kET) cls[c] = classes[g.cls_begin + c];
  const uint64_t outmask0 = ~g.smask & ((n >= 64) ? ~0ull : ((1ull << n) - 1));
  for (int i = tid; i < kEvTilesPerCta; i += kET) ibase[i] = pdep64((uint64_t)i, outmask0);
  for (int i = tid; i < g.nterm * kET; i += kET) acc[i] = 0.0;
  __syncthreads();
  const int nc = g.ncls;
  // this thread's Z parity per term (tile positions on thread bits, fixed for the CTA)
  uint32_t pthread = 0;
  for (int mi = 0; mi < g.nmap; ++mi) {
    const EvMap& m = smap[mi];
    uint32_t tb = 0;
    for (int b = 0; b < K - 4; ++b) tb |= (uint32_t)((tid >> b) & 1) << m.tpos[b];
    for (int t = m.term_begin - g.term_begin; t < m.term_begin - g.term_begin + m.nterm; ++t)
      pthread |= (uint32_t)(__popc(tb & szl[t]) & 1) << t;
  }
  const int ntl = n - K;
  const int64_t ntiles = (int64_t)1 << ntl;
  const int64_t slot = blockIdx.x / nchunks, chunk = blockIdx.x % nchunks;
  const int64_t tpc = ntiles / nchunks, w0 = chunk * tpc;
  const uint64_t outmask = ~g.smask & qmask;
  const A* st = states + (slot << n);
  const uint64_t Pt = ((uint64_t)tid & lowm) | hi_off[tid >> g.lowq];
  const uint32_t St = swz_slot<SB>(swz, (uint32_t)tid);
  const int hstep = kET >> g.lowq;
  const uint64_t my_zg = lane < g.nterm ? terms[g.term_begin + lane].zg : 0;
  // tiles w0 + i, w0 a multiple of tpc (a power of two): pdep is linear over disjoint bits
  const uint64_t base0 = pdep64((uint64_t)w0, outmask);
  auto load = [&](int64_t i, A* dst_tile) {
    const uint64_t base = base0 | ibase[i];
#pragma unroll
    for (int i = 0; i < TL / kET; ++i) {
      const A* src = st + (base | Pt | hi_off[i * hstep]);
      A* dst = dst_tile + (St ^ swz_slot<SB>(swz, (uint32_t)(i * kET)));
      if (sizeof(A) == 16) cp_async16(dst, src);
      else cp_async8(dst, src);
    }
    cp_async_commit();
  };
  load(0, tiles);
  for (int64_t i = 0; i < tpc; ++i) {
    if (NBUF == 2 && i + 1 < tpc) {
      load(i + 1, tiles + ((i + 1) & 1) * TL);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    if (warp == 0) {  // the tile's out-of-tile Z parity of every term, one bit per term
      const uint64_t base = base0 | ibase[i];
      const uint32_t word = __ballot_sync(0xffffffffu, lane < g.nterm && (__popcll(base & my_zg) & 1));
      if (lane == 0) tword[i & 1] = word;
    }
    __syncthreads();
    const A* tile = tiles + (NBUF == 2 ? (i & 1) * TL : 0);
    const uint32_t pw = pthread ^ tword[i & 1];
    int cur_map = -1;
    A v[16];
    for (int c = 0; c < nc; ++c) {
      const EvClass k = cls[c];
      if (k.map != cur_map) {
        cur_map = k.map;
        const EvMap& m = smap[cur_map];
        uint32_t tb = 0;
#pragma unroll
        for (int b = 0; b < K - 4; ++b) tb |= (uint32_t)((tid >> b) & 1) << m.tpos[b];
        const uint32_t sbase = swz_slot<SB>(swz, tb);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = tile[sbase ^ m.soff[j]];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) opaque(v[j]);  // no hoisting of every class's products
      ev_class_dispatch<R>(k.xr, v, at, k.t0, k.t1, k.im0, acc, tid, pw);
    }
    __syncthreads();  // the buffer is refilled by the load issued next iteration
    if (NBUF == 1 && i + 1 < tpc) load(i + 1, tiles);
  }
  // one fixed-order reduction per CTA: warp w sums terms w, w + 8, ...; lane l adds the
  // accumulators of threads l, l + 32, ... in order, then a fixed shuffle tree
  for (int t = warp; t < g.nterm; t += kET / 32) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kET / 32; ++r) s += acc[t * kET + r * 32 + lane];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) partial[(slot * nchunks + chunk) * nterm_total + terms[g.term_begin + t].out] = s;
  }
}

}  // namespace

void launch_expval_tile(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                        const ExpvalTerm* terms, const EvMap* maps, double* partial, int nterm_total,
                        cudaStream_t s) {
  dim3 grid((unsigned)(1ull << (n - g.k)), (unsigned)slots);
  const size_t amp = c64 ? 8 : 16;
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
  return (int)std::max<int64_t>(std::min<int64_t>(ntiles, 128), ntiles / kEvTilesPerCta);
}

void launch_expval_acc(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                       const ExpvalTerm* terms, const EvMap* maps, const EvClass* classes, double* partial,
                       int nterm_total, cudaStream_t s) {
  const size_t amp = c64 ? 8 : 16;
  auto up = [](size_t b) { return (b + 15) & ~(size_t)15; };
  const int nbuf = c64 ? 2 : 1;
  const size_t smem = up(nbuf * amp * 4096) + up(sizeof(double) * kET * (size_t)g.nterm) +
                      up(sizeof(uint64_t) * (4096 >> g.lowq)) + up(sizeof(uint32_t) * (4096 >> (c64 ? 4 : 3))) +
                      up(sizeof(AccTerm<double>) * (size_t)g.nterm) + up(sizeof(EvClass) * (size_t)g.ncls) +
                      up(sizeof(EvMap) * (size_t)g.nmap) + up(sizeof(uint32_t) * (size_t)g.nterm) +
                      up(sizeof(uint64_t) * kEvTilesPerCta) + 16;
  static thread_local int set_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev != dev) {  // the attribute is a ceiling: the device's opt-in maximum, once
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_expval_acc<float, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    cudaFuncSetAttribute(k_expval_acc<double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    set_dev = dev;
  }
  const int nchunks = expval_acc_chunks(n);
  const unsigned grid = (unsigned)(slots * nchunks);
  if (c64)
    k_expval_acc<float, 2><<<grid, kET, smem, s>>>((const float2*)states, n, g, terms, maps, classes, partial,
                                                nterm_total, nchunks);
  else
    k_expval_acc<double, 1><<<grid, kET, smem, s>>>((const double2*)states, n, g, terms, maps, classes, partial,
                                                 nterm_total, nchunks);
}

}  // namespace qsb
