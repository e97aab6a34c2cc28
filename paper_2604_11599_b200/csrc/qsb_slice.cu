// Kernels of the global-qubit-sliced engine (BASELINE cfg 5; sliced.py, qsb.h qsb_slice_*).
//
// One slice = the 2^L amplitudes of one value of the G global (rank) qubits.  Every
// classical decision of the trajectory -- measure / reset outcomes, the classical store,
// if/else guards, the degenerate-branch status -- is made on the device from a SliceCtl
// (qsb_internal.h), so the host enqueues a whole trajectory without reading anything back
// (north_star: "no host round-trip"):
//   * gate / scale kernels are guarded: they return at once when the innermost branch is
//     not taken (or the trajectory already hit a degenerate branch);
//   * a measurement is p1 partial per slice (deterministic block reduction) -> the
//     partials of all slices side by side (one device array; NCCL all-gather across ranks)
//     -> k_slice_decide sums them IN SLICE ORDER, draws u from the shared RNG stream and
//     applies the reference's arithmetic (sim.py:230-251: u < p1, p0 = 1 - p1, 1e-15,
//     1/sqrt) -> the collapse kernel reads the decision;
//   * a swap of a global position with local position `pos` moves the amplitudes whose
//     local bit `pos` differs from the slice's global bit to the partner slice: in place
//     on one device (k_slice_exchange_local), or packed / NCCL send-recv / unpacked in
//     chunks across ranks (k_slice_pack / k_slice_unpack, qsb_slice_api.cpp);
//   * a remap of k = 2..3 global positions at once is a transpose of 2^k x 2^k blocks
//     across a group of 2^k slices (k_slice_remap_local on one device; k_slice_pack_sub /
//     grouped NCCL send-recv to the 2^k - 1 peers / k_slice_unpack_sub across ranks).
#include <cuda_runtime.h>

#include <utility>

#include "qsb_device.cuh"
#include "qsb_launch.h"

namespace qsb {

struct MatArg {  // a 2x2 matrix by value (kernel parameter space, no device copy)
  double m[8];
};

namespace {

constexpr int kST = 256;

__device__ __forceinline__ bool slice_live(const SliceCtl* c) { return c->status == 0 && c->active == c->depth; }

int sgrid(int64_t items) {
  int64_t g = (items + kST - 1) / kST;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

__global__ void k_slice_init(SliceCtl* c, uint64_t seed, int64_t shot, const uint64_t* rng_init, int nwords) {
  SliceCtl x;
  if (rng_init)
    for (int w = 0; w < 4; ++w) x.rng[w] = rng_init[w];
  else
    rng_for_shot(x.rng, seed, (uint64_t)shot);
  x.status = 0;
  x.depth = 0;
  x.active = 0;
  x.draws = 0;
  x.outcome = -1;
  x.nwords = nwords;
  x.scale = 1.0;
  x.p1 = 0.0;
  for (int w = 0; w < kSliceWords; ++w) x.bits[w] = 0;
  *c = x;
}

__global__ void k_slice_guard(SliceCtl* c, int kind, int pred_bit, int pred_width, int pred_cmp, uint64_t rhs) {
  if (kind == QSB_OP_IF) {  // evaluated once at entry (sim.py:296-301)
    const bool act = c->active == c->depth;
    const bool taken = act && pred_eval(c->bits, pred_bit, pred_width, pred_cmp, rhs);
    c->depth++;
    if (taken) c->active = c->depth;
  } else if (kind == QSB_OP_ELSE) {
    if (c->active == c->depth) c->active = c->depth - 1;
    else if (c->active == c->depth - 1) c->active = c->depth;
  } else {  // ENDIF
    if (c->active == c->depth) c->active--;
    c->depth--;
  }
}

template <typename R>
__global__ void __launch_bounds__(kST) k_slice_gate(typename Amp<R>::T* amps, int n, int t, uint64_t cm, uint64_t cv,
                                                    int gc, MatArg m8, const SliceCtl* ctl) {
  if (!slice_live(ctl)) return;
  const int64_t pairs = 1ll << (n - 1);
  for (int64_t p = blockIdx.x * (int64_t)kST + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * kST) {
    const uint64_t i0 = insert_zero((uint64_t)p, t);
    if ((i0 & cm) != cv) continue;
    const uint64_t i1 = i0 | (1ull << t);
    auto a0 = amps[i0], a1 = amps[i1];
    apply_pair<R>(gc, m8.m, a0, a1);
    amps[i0] = a0;
    amps[i1] = a1;
  }
}

template <typename R>
__global__ void __launch_bounds__(kST) k_slice_scale(typename Amp<R>::T* amps, int64_t N, double re, double im,
                                                     const SliceCtl* ctl) {
  if (!slice_live(ctl)) return;
  const R sr = (R)re, si = (R)im;
  for (int64_t i = blockIdx.x * (int64_t)kST + threadIdx.x; i < N; i += (int64_t)gridDim.x * kST) {
    const auto a = amps[i];
    amps[i] = mk<R>(sr * a.x - si * a.y, sr * a.y + si * a.x);
  }
}

// this slice's partial p1 into partials[index]: the fixed-order sum of the block sums
// (select = 0: the slice holds no amplitude with the measured bit set -> exactly 0)
__global__ void k_slice_put(const double* blocks, int nblocks, int select, double* partials, int index) {
  double s = 0.0;
  if (select)
    for (int b = 0; b < nblocks; ++b) s += blocks[b];
  partials[index] = s;
}

__global__ void k_slice_decide(SliceCtl* c, const double* partials, int nslices, int kind, int bit) {
  SliceCtl x = *c;
  if (!(x.status == 0 && x.active == x.depth)) {
    c->outcome = -1;
    return;
  }
  double p1 = 0.0;
  for (int s = 0; s < nslices; ++s) p1 += partials[s];  // slice order on every rank
  const double u = rng_uniform(x.rng);
  x.draws++;
  const int outcome = u < p1 ? 1 : 0;
  const double pout = outcome ? p1 : 1.0 - p1;
  x.p1 = p1;
  x.outcome = outcome;
  if (pout < 1e-15) {
    x.status = QSB_ERR_DEGENERATE;
    x.scale = 0.0;
  } else {
    x.scale = 1.0 / sqrt(pout);
    if (kind == QSB_OP_MEASURE)
      x.bits[bit >> 6] = (x.bits[bit >> 6] & ~(1ull << (bit & 63))) | ((uint64_t)outcome << (bit & 63));
  }
  *c = x;
}

// q >= 0: projection of local qubit q onto the decided outcome, scaled; flip (reset) moves
// the surviving |1> half to |0> (sim.py:254-259).  q < 0: the measured qubit is global --
// the whole slice is kept (scaled) iff its global bit `gbit` equals the outcome.
template <typename R>
__global__ void __launch_bounds__(kST) k_slice_collapse(typename Amp<R>::T* amps, int n, int q, int gbit, int flip,
                                                        const SliceCtl* ctl) {
  const int outcome = ctl->outcome;
  if (outcome < 0 || ctl->status) return;
  const R s = (R)ctl->scale;
  const auto z = mk<R>(0, 0);
  if (q < 0) {
    const R f = gbit == outcome ? s : (R)0;
    const int64_t N = 1ll << n;
    for (int64_t i = blockIdx.x * (int64_t)kST + threadIdx.x; i < N; i += (int64_t)gridDim.x * kST) {
      const auto a = amps[i];
      amps[i] = mk<R>(a.x * f, a.y * f);
    }
    return;
  }
  const int64_t pairs = 1ll << (n - 1);
  for (int64_t p = blockIdx.x * (int64_t)kST + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * kST) {
    const uint64_t i0 = insert_zero((uint64_t)p, q), i1 = i0 | (1ull << q);
    if (outcome) {
      auto a1 = amps[i1];
      a1 = mk<R>(a1.x * s, a1.y * s);
      amps[i0] = flip ? a1 : z;
      amps[i1] = flip ? z : a1;
    } else {
      auto a0 = amps[i0];
      amps[i0] = mk<R>(a0.x * s, a0.y * s);
      amps[i1] = z;
    }
  }
}

// a holds global bit 0, b global bit 1: a[i | bit] <-> b[i] for every i with bit `pos` clear
template <typename R>
__global__ void __launch_bounds__(kST) k_slice_exchange_local(typename Amp<R>::T* a, typename Amp<R>::T* b, int n,
                                                              int pos) {
  const int64_t pairs = 1ll << (n - 1);
  for (int64_t p = blockIdx.x * (int64_t)kST + threadIdx.x; p < pairs; p += (int64_t)gridDim.x * kST) {
    const uint64_t i = insert_zero((uint64_t)p, pos);
    const auto x = a[i | (1ull << pos)];
    a[i | (1ull << pos)] = b[i];
    b[i] = x;
  }
}

// region of a slice with global bit c: local indices whose bit `pos` is !c, in index order
template <typename R>
__global__ void __launch_bounds__(kST) k_slice_pack(const typename Amp<R>::T* amps, int pos, int c, int64_t first,
                                                    int64_t count, typename Amp<R>::T* out) {
  const uint64_t set = c ? 0ull : (1ull << pos);
  for (int64_t k = blockIdx.x * (int64_t)kST + threadIdx.x; k < count; k += (int64_t)gridDim.x * kST)
    out[k] = amps[insert_zero((uint64_t)(first + k), pos) | set];
}

template <typename R>
__global__ void __launch_bounds__(kST) k_slice_unpack(typename Amp<R>::T* amps, int pos, int c, int64_t first,
                                                      int64_t count, const typename Amp<R>::T* in) {
  const uint64_t set = c ? 0ull : (1ull << pos);
  for (int64_t k = blockIdx.x * (int64_t)kST + threadIdx.x; k < count; k += (int64_t)gridDim.x * kST)
    amps[insert_zero((uint64_t)(first + k), pos) | set] = in[k];
}

// k-position remaps (1 <= k <= 3).  A group of 2^k slices differing only in the k global
// bits being swapped is indexed by y (bit i <-> global position i of the remap); local
// positions lpos[i] pair with them.  Swapping global position i with lpos[i] for all i at
// once moves the amplitude at (slice y, local bits x at lpos, rest r) to (slice x, local
// bits y, rest r): a transpose of the 2^k x 2^k blocks, one per r.
struct RemapArg {
  int k;
  int lpos[3];   // pairing order
  int sorted[3]; // ascending (zero insertion)
};

__device__ __forceinline__ uint64_t remap_base(uint64_t r, const RemapArg& a) {
  for (int i = 0; i < a.k; ++i) r = insert_zero(r, a.sorted[i]);
  return r;
}

__device__ __forceinline__ uint64_t remap_spread(int x, const RemapArg& a) {
  uint64_t v = 0;
  for (int i = 0; i < a.k; ++i) v |= (uint64_t)((x >> i) & 1) << a.lpos[i];
  return v;
}

template <typename R>
struct GroupPtrs {
  typename Amp<R>::T* p[8];
};

// in place on one device: every off-diagonal pair (x < y) of every block swapped once
template <typename R>
__global__ void __launch_bounds__(kST) k_slice_remap_local(GroupPtrs<R> g, int n, RemapArg a) {
  const int64_t rows = 1ll << (n - a.k);
  const int m = 1 << a.k;
  for (int64_t r = blockIdx.x * (int64_t)kST + threadIdx.x; r < rows; r += (int64_t)gridDim.x * kST) {
    const uint64_t base = remap_base((uint64_t)r, a);
    for (int y = 1; y < m; ++y)
      for (int x = 0; x < y; ++x) {
        typename Amp<R>::T* py = g.p[y] + (base | remap_spread(x, a));
        typename Amp<R>::T* px = g.p[x] + (base | remap_spread(y, a));
        const auto t = *py;
        *py = *px;
        *px = t;
      }
  }
}

// the rows of one slice whose local bits at lpos equal x, in increasing order of the rest
template <typename R>
__global__ void __launch_bounds__(kST) k_slice_pack_sub(const typename Amp<R>::T* amps, RemapArg a, int x,
                                                        int64_t first, int64_t count, typename Amp<R>::T* out) {
  const uint64_t set = remap_spread(x, a);
  for (int64_t j = blockIdx.x * (int64_t)kST + threadIdx.x; j < count; j += (int64_t)gridDim.x * kST)
    out[j] = amps[remap_base((uint64_t)(first + j), a) | set];
}

template <typename R>
__global__ void __launch_bounds__(kST) k_slice_unpack_sub(typename Amp<R>::T* amps, RemapArg a, int x, int64_t first,
                                                          int64_t count, const typename Amp<R>::T* in) {
  const uint64_t set = remap_spread(x, a);
  for (int64_t j = blockIdx.x * (int64_t)kST + threadIdx.x; j < count; j += (int64_t)gridDim.x * kST)
    amps[remap_base((uint64_t)(first + j), a) | set] = in[j];
}

RemapArg remap_arg(int k, const int* lpos) {
  RemapArg a{};
  a.k = k;
  for (int i = 0; i < k; ++i) a.lpos[i] = a.sorted[i] = lpos[i];
  for (int i = 0; i < k; ++i)
    for (int j = i + 1; j < k; ++j)
      if (a.sorted[j] < a.sorted[i]) std::swap(a.sorted[i], a.sorted[j]);
  return a;
}

}  // namespace

void launch_slice_remap_local(int c64, void* const* group, int n, int k, const int* lpos, cudaStream_t s) {
  const RemapArg a = remap_arg(k, lpos);
  const int g = sgrid(1ll << (n - k));
  if (c64) {
    GroupPtrs<float> p{};
    for (int i = 0; i < (1 << k); ++i) p.p[i] = (float2*)group[i];
    k_slice_remap_local<float><<<g, kST, 0, s>>>(p, n, a);
  } else {
    GroupPtrs<double> p{};
    for (int i = 0; i < (1 << k); ++i) p.p[i] = (double2*)group[i];
    k_slice_remap_local<double><<<g, kST, 0, s>>>(p, n, a);
  }
}

void launch_slice_pack_sub(int c64, const void* amps, int k, const int* lpos, int x, int64_t first, int64_t count,
                           void* out, cudaStream_t s) {
  const RemapArg a = remap_arg(k, lpos);
  if (c64) k_slice_pack_sub<float><<<sgrid(count), kST, 0, s>>>((const float2*)amps, a, x, first, count, (float2*)out);
  else k_slice_pack_sub<double><<<sgrid(count), kST, 0, s>>>((const double2*)amps, a, x, first, count, (double2*)out);
}

void launch_slice_unpack_sub(int c64, void* amps, int k, const int* lpos, int x, int64_t first, int64_t count,
                             const void* in, cudaStream_t s) {
  const RemapArg a = remap_arg(k, lpos);
  if (c64) k_slice_unpack_sub<float><<<sgrid(count), kST, 0, s>>>((float2*)amps, a, x, first, count, (const float2*)in);
  else k_slice_unpack_sub<double><<<sgrid(count), kST, 0, s>>>((double2*)amps, a, x, first, count, (const double2*)in);
}

void launch_slice_init(SliceCtl* c, uint64_t seed, int64_t shot, const uint64_t* rng_init, int nwords,
                       cudaStream_t s) {
  k_slice_init<<<1, 1, 0, s>>>(c, seed, shot, rng_init, nwords);
}

void launch_slice_guard(SliceCtl* c, int kind, int pred_bit, int pred_width, int pred_cmp, uint64_t rhs,
                        cudaStream_t s) {
  k_slice_guard<<<1, 1, 0, s>>>(c, kind, pred_bit, pred_width, pred_cmp, rhs);
}

void launch_slice_gate(int c64, void* amps, int n, int t, uint64_t cm, uint64_t cv, int gc, const double* m,
                       const SliceCtl* ctl, cudaStream_t s) {
  MatArg a;
  for (int i = 0; i < 8; ++i) a.m[i] = m[i];
  const int g = sgrid(1ll << (n - 1));
  if (c64) k_slice_gate<float><<<g, kST, 0, s>>>((float2*)amps, n, t, cm, cv, gc, a, ctl);
  else k_slice_gate<double><<<g, kST, 0, s>>>((double2*)amps, n, t, cm, cv, gc, a, ctl);
}

void launch_slice_scale(int c64, void* amps, int n, double re, double im, const SliceCtl* ctl, cudaStream_t s) {
  const int64_t N = 1ll << n;
  if (c64) k_slice_scale<float><<<sgrid(N), kST, 0, s>>>((float2*)amps, N, re, im, ctl);
  else k_slice_scale<double><<<sgrid(N), kST, 0, s>>>((double2*)amps, N, re, im, ctl);
}

void launch_slice_put(const double* blocks, int nblocks, int select, double* partials, int index, cudaStream_t s) {
  k_slice_put<<<1, 1, 0, s>>>(blocks, nblocks, select, partials, index);
}

void launch_slice_decide(SliceCtl* c, const double* partials, int nslices, int kind, int bit, cudaStream_t s) {
  k_slice_decide<<<1, 1, 0, s>>>(c, partials, nslices, kind, bit);
}

void launch_slice_collapse(int c64, void* amps, int n, int q, int gbit, int flip, const SliceCtl* ctl,
                           cudaStream_t s) {
  const int g = sgrid(1ll << (n - (q < 0 ? 0 : 1)));
  if (c64) k_slice_collapse<float><<<g, kST, 0, s>>>((float2*)amps, n, q, gbit, flip, ctl);
  else k_slice_collapse<double><<<g, kST, 0, s>>>((double2*)amps, n, q, gbit, flip, ctl);
}

void launch_slice_exchange_local(int c64, void* a, void* b, int n, int pos, cudaStream_t s) {
  const int g = sgrid(1ll << (n - 1));
  if (c64) k_slice_exchange_local<float><<<g, kST, 0, s>>>((float2*)a, (float2*)b, n, pos);
  else k_slice_exchange_local<double><<<g, kST, 0, s>>>((double2*)a, (double2*)b, n, pos);
}

void launch_slice_pack(int c64, const void* amps, int pos, int c, int64_t first, int64_t count, void* out,
                       cudaStream_t s) {
  if (c64) k_slice_pack<float><<<sgrid(count), kST, 0, s>>>((const float2*)amps, pos, c, first, count, (float2*)out);
  else k_slice_pack<double><<<sgrid(count), kST, 0, s>>>((const double2*)amps, pos, c, first, count, (double2*)out);
}

void launch_slice_unpack(int c64, void* amps, int pos, int c, int64_t first, int64_t count, const void* in,
                         cudaStream_t s) {
  if (c64) k_slice_unpack<float><<<sgrid(count), kST, 0, s>>>((float2*)amps, pos, c, first, count, (const float2*)in);
  else k_slice_unpack<double><<<sgrid(count), kST, 0, s>>>((double2*)amps, pos, c, first, count, (const double2*)in);
}

}  // namespace qsb
