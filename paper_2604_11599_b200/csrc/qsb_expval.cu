// Tile-fused Pauli expectation reducer (observe(), BASELINE cfg 3).
//
// <P> = Re[(-i)^ny * sum_i (-1)^popc(i & zy) conj(psi_i) psi_{i ^ x}]
//
// The terms are grouped on the host so that each group's X supports fit in one tile
// qubit set S (k qubits, always containing the low qubits for 32-byte runs); one launch
// per group reads every tile of every state exactly once and evaluates all of the
// group's terms from shared memory: pairs (l, l ^ x_local) stay inside the tile, Z/Y
// signs of the out-of-tile qubits are one per-tile sign.  Diagonal (Z-only) terms ride
// along with the first group.  The per-grid reduction is fixed-order (warp shfl_down,
// warp partials summed in order, tiles summed in order) -- deterministic.
#include <cuda_runtime.h>

#include "qsb_device.cuh"
#include "qsb_launch.h"

namespace qsb {

namespace {

constexpr int kET = 256;

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
  const int ntiles_log2 = n - k;
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
    partial[((int64_t)slot * nterm_total + tm.out) * ((int64_t)1 << ntiles_log2) + blockIdx.x] = s;
  }
}

__global__ void k_expval_tile_finish(const double* partial, int64_t slots, int nterm, int ntiles_log2,
                                     const ExpvalTerm* terms_by_out, double* out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= slots * nterm) return;
  const int t = (int)(idx % nterm);
  const double* p = partial + idx * ((int64_t)1 << ntiles_log2);
  double s = 0.0;
  for (int64_t b = 0; b < ((int64_t)1 << ntiles_log2); ++b) s += p[b];
  const ExpvalTerm tm = terms_by_out[t];
  if (tm.xg | tm.xl) s *= 2.0;
  out[idx] = ((tm.ny & 3) >= 2) ? -s : s;
}

}  // namespace

void launch_expval_tile(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                        const ExpvalTerm* terms, double* partial, int nterm_total, cudaStream_t s) {
  const size_t smem = (size_t)(c64 ? 8 : 16) * ((size_t)1 << g.k) + sizeof(uint64_t) * ((size_t)1 << (g.k - g.lowq)) +
                      sizeof(double) * (kET / 32) * (size_t)g.nterm;
  dim3 grid((unsigned)(1ull << (n - g.k)), (unsigned)slots);
  if (c64) {
    cudaFuncSetAttribute(k_expval_tile<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_expval_tile<float><<<grid, kET, smem, s>>>((const float2*)states, n, g, terms, partial, nterm_total);
  } else {
    cudaFuncSetAttribute(k_expval_tile<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_expval_tile<double><<<grid, kET, smem, s>>>((const double2*)states, n, g, terms, partial, nterm_total);
  }
}

void launch_expval_tile_finish(const double* partial, int64_t slots, int nterm, int ntiles_log2,
                               const ExpvalTerm* terms_by_out, double* out, cudaStream_t s) {
  const int64_t items = slots * nterm;
  k_expval_tile_finish<<<(unsigned)((items + 127) / 128), 128, 0, s>>>(partial, slots, nterm, ntiles_log2,
                                                                      terms_by_out, out);
}

}  // namespace qsb
