// Shared-memory bank behaviour of 8-byte (float2) and 16-byte (double2) loads on B200:
// which lanes are serviced together?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// bank_probe.cu -o bank_probe; ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum ./bank_probe
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t swz4(uint32_t l) {
  const uint32_t V[16] = {1, 2, 4, 8, 3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 1};
  uint32_t s = 0, h = l >> 4;
  for (int p = 4; h; ++p, h >>= 1)
    if (h & 1) s ^= V[p];
  return l ^ s;
}

template <typename T>
__global__ void probe(T* out, int pattern, int iters) {
  __shared__ T t[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) t[i] = T{};
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t slot;
  switch (pattern) {
    case 0: slot = lane; break;                               // consecutive
    case 1: {  // DYN20 c64 pass3/ph0 thread positions 4,5,7,8,6 (+swizzle)
      const int tp[5] = {4, 5, 7, 8, 6};
      uint32_t b = 0;
      for (int i = 0; i < 5; ++i) b |= ((lane >> i) & 1u) << tp[i];
      slot = swz4(b);
    } break;
    case 2: slot = (lane & 15) * 16 + (lane >> 4); break;     // lanes 0-15 distinct rows, same bank pair
    case 3: slot = ((lane & 15) ^ ((lane >> 4) * 8)) ; break; // 0..15 then 8..15,0..7
    case 4: slot = (lane & 15) + 16 * (lane >> 4) + 8 * ((lane >> 3) & 1) * 0; break;
    case 5: { // lanes L and L+16 -> same bank pair, different row; L<16 distinct
      slot = (lane & 15) + 16 * (lane >> 4);
    } break;
    case 6: { // lanes 0-7 and 16-23 distinct mod 16 (quarter pairs), 8-15 / 24-31 repeat 0-7
      slot = (lane & 7) + 8 * (lane >> 4) + 32 * ((lane >> 3) & 1);
    } break;
    default: slot = lane * 2;
  }
  T acc{};
  for (int it = 0; it < iters; ++it) {
    T v = t[(slot + it * 64) & 2047];
    acc.x += v.x;
    acc.y += v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float2* o;
  cudaMalloc(&o, 1 << 20);
  for (int p = 0; p <= 7; ++p) {
    probe<float2><<<1, 32>>>(o, p, 64);
    cudaDeviceSynchronize();
  }
  for (int p = 0; p <= 7; ++p) {
    probe<double2><<<1, 32>>>((double2*)o, p, 64);
    cudaDeviceSynchronize();
  }
  printf("done\n");
  return 0;
}
