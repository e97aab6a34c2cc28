// Does FP64 mma.sync (DMMA) run on a pipe separate from DFMA on B200?
// Measures TFLOP/s of: DFMA only, DMMA only, and both interleaved in every warp.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_probe dmma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int iters, double s) {
  double f[16];
  double c[8][2];
  for (int i = 0; i < 16; ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
  const double a = s + threadIdx.x * 1e-6, b = s * 0.5;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    }
  }
  double acc = 0;
  for (int i = 0; i < 16; ++i) acc += f[i];
  for (int i = 0; i < 8; ++i) acc += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * nsm * 8 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, grid = nsm * 4, threads = 256;
  const char* names[3] = {"DFMA only", "DMMA only", "DFMA + DMMA"};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<grid, threads>>>(out, iters, 1.0000001);
      if (mode == 1) k<1><<<grid, threads>>>(out, iters, 1.0000001);
      if (mode == 2) k<2><<<grid, threads>>>(out, iters, 1.0000001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double warps = (double)grid * threads / 32;
    const double fma_flops = mode != 1 ? (double)grid * threads * iters * 64 * 2 : 0;
    const double mma_flops = mode != 0 ? warps * iters * 8 * (8.0 * 8 * 4 * 2) : 0;
    printf("%-12s %.3f ms  DFMA %.1f TF  DMMA %.1f TF  total %.1f TF  (%s)\n", names[mode], best,
           fma_flops / best / 1e9, mma_flops / best / 1e9, (fma_flops + mma_flops) / best / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
