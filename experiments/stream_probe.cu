// Streaming micro-benchmark for the fused-pass driver: gather a 2^12-amplitude
// complex128 tile (low 4 qubits contiguous = 256 B runs, 8 further tile qubits),
// hold it in shared memory, scatter it back.  No gate work: this bounds the pass
// driver's HBM rate for each load/store mechanism.
//   A: per-thread cp.async 16 B (swizzled slots) + LDS/STG scatter, 1 buffer, 2 CTAs/SM
//   C: bulk copies (cp.async.bulk, 256 B runs, mbarrier) in and out, 1 buffer, 2 CTAs/SM
//   D: bulk copies, 1 CTA/SM, NBUF-buffer ring, loads issued NBUF-1 items ahead
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int K = 12, TL = 1 << K, LOWQ = 4, RUNS = TL >> LOWQ, RUNB = 16 << LOWQ;

struct Args {
  double2* st;
  int n;
  uint64_t hi_off[RUNS];  // physical offset of run r (tile high bits)
  uint64_t outmask;       // qubits outside the tile
};

__device__ __forceinline__ uint64_t pdep(uint64_t v, uint64_t m) {
  uint64_t r = 0;
  for (uint64_t b = 1; m; b <<= 1) {
    uint64_t low = m & (~m + 1);
    if (v & b) r |= low;
    m &= m - 1;
  }
  return r;
}

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}

__global__ void __launch_bounds__(256, 2) kA(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* tile = (double2*)sm;
  const int tid = threadIdx.x;
  const int64_t W = 1ll << (a.n - K);
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    const uint64_t base = pdep((uint64_t)w, a.outmask);
    double2* st = a.st;
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
      int l = tid + j * 256;
      uint64_t p = base | a.hi_off[l >> LOWQ] | (l & 15);
      int s = l ^ ((l >> 3) & 7);
      cp16(tile + s, st + p);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
      int l = tid + j * 256;
      uint64_t p = base | a.hi_off[l >> LOWQ] | (l & 15);
      int s = l ^ ((l >> 3) & 7);
      st[p] = tile[s];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(a),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* s, const void* g, uint32_t bytes, uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s), m = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(a),
               "l"(g), "r"(bytes), "r"(m)
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* g, const void* s, uint32_t bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g), "r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// C: 2 CTAs/SM, one buffer, one 256 B run per thread in and out
__global__ void __launch_bounds__(256, 2) kC(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* tile = (double2*)sm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  const int64_t W = 1ll << (a.n - K);
  uint32_t ph = 0;
  for (int64_t w = blockIdx.x; w < W; w += gridDim.x) {
    const uint64_t base = pdep((uint64_t)w, a.outmask);
    if (tid == 0) {
      bulk_wait_read<0>();  // previous stores have read the buffer
      mbar_expect(&bar, TL * 16);
    }
    __syncthreads();
    bulk_load(tile + tid * 16, a.st + (base | a.hi_off[tid]), RUNB, &bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    // (gates would run here)
    fence_async();
    bulk_store(a.st + (base | a.hi_off[tid]), tile + tid * 16, RUNB);
    bulk_commit();
    bulk_wait_read<0>();
    __syncthreads();
  }
  bulk_wait<0>();
}

// D: 1 CTA/SM, ring of NB buffers; the loads of item i+NB-1 are issued while item i is processed
template <int NB> __global__ void __launch_bounds__(256, 1) kD(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* bufs = (double2*)sm;
  __shared__ __align__(8) uint64_t bar[NB];
  const int tid = threadIdx.x;
  if (tid < NB) mbar_init(&bar[tid], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  const int64_t W = 1ll << (a.n - K);
  auto issue = [&](int64_t w, int b) {
    const uint64_t base = pdep((uint64_t)w, a.outmask);
    if (tid == 0) mbar_expect(&bar[b], TL * 16);
    __syncthreads();
    bulk_load(bufs + b * TL + tid * 16, a.st + (base | a.hi_off[tid]), RUNB, &bar[b]);
  };
  int64_t w = blockIdx.x;
  for (int i = 0; i < NB - 1; ++i)
    if (w + (int64_t)i * gridDim.x < W) issue(w + (int64_t)i * gridDim.x, i);
  uint32_t phs = 0;
  int b = 0;
  for (int i = 0; w < W; w += gridDim.x, ++i) {
    // next load into buffer (b + NB - 1) % NB: its last store must have read out
    const int64_t wn = w + (int64_t)(NB - 1) * gridDim.x;
    const int bn = (b + NB - 1) % NB;
    bulk_wait_read<0>();
    if (wn < W) issue(wn, bn);
    mbar_wait(&bar[b], (phs >> b) & 1);
    phs ^= 1u << b;
    double2* tile = bufs + b * TL;
    const uint64_t base = pdep((uint64_t)w, a.outmask);
    fence_async();
    bulk_store(a.st + (base | a.hi_off[tid]), tile + tid * 16, RUNB);
    bulk_commit();
    b = (b + 1) % NB;
  }
  bulk_wait<0>();
}

__global__ void kcopy(const double2* __restrict__ x, double2* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

int main() {
  const int n = 28;
  double2* st;
  CK(cudaMalloc(&st, (16ull << n)));
  CK(cudaMemset(st, 0, 16ull << n));
  double2* st2;
  CK(cudaMalloc(&st2, (16ull << n)));
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 2.0 * (16ull << n);
  {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      kcopy<<<nsm * 8, 512>>>(st, st2, 1ll << n);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("plain copy kernel: %.1f GB/s\n", bytes / ms / 1e6);
  }
  std::vector<std::vector<int>> pats = {
      {4, 5, 6, 7, 8, 9, 10, 11}, {20, 21, 22, 23, 24, 25, 26, 27}, {4, 7, 10, 13, 16, 19, 22, 25}, {12, 13, 14, 15, 24, 25, 26, 27}};
  for (auto& hp : pats) {
    Args a;
    a.st = st;
    a.n = n;
    uint64_t smask = 15;
    for (int q : hp) smask |= 1ull << q;
    a.outmask = ((1ull << n) - 1) & ~smask;
    for (int r = 0; r < RUNS; ++r) {
      uint64_t o = 0;
      for (int j = 0; j < 8; ++j)
        if ((r >> j) & 1) o |= 1ull << hp[j];
      a.hi_off[r] = o;
    }
    printf("tile hi bits:");
    for (int q : hp) printf(" %d", q);
    printf("\n");
    auto run = [&](const char* name, auto kern, int grid, int threads, size_t smem) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, threads, smem>>>(a);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("  %-34s %.1f GB/s\n", name, bytes / best / 1e6);
    };
    run("A cp.async16 2CTA/SM 1buf", kA, 2 * nsm, 256, 64 * 1024);
    run("C bulk 2CTA/SM 1buf", kC, 2 * nsm, 256, 64 * 1024);
    run("C bulk 3CTA/SM 1buf", kC, 3 * nsm, 256, 64 * 1024);
    run("D bulk 1CTA/SM 2buf", kD<2>, nsm, 256, 2 * 64 * 1024);
    run("D bulk 1CTA/SM 3buf", kD<3>, nsm, 256, 3 * 64 * 1024);
  }
  return 0;
}
