// Device-side shot histogram: the per-shot classical words of
// a sample stay in HBM; they are radix-sorted on their low `nbits` bits and run-length
// encoded, so only the distinct outcomes and their counts cross PCIe.  The host then
// formats ShotHistogram keys (sim.py:118-131) for the distinct words only.
//
// Integer-only and order-independent, so the counts are exact and deterministic; CUB
// (CUDA toolkit, header-only) provides the sort and the run-length encoder -- this is
// result formatting next to the hot path, not the hot path itself.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include "qsb_launch.h"

namespace qsb {

size_t hist_scratch_bytes(size_t n) {
  size_t a = 0, b = 0;
  const int ni = (int)n;
  cub::DeviceRadixSort::SortKeys(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, ni, 0, 64);
  cub::DeviceRunLengthEncode::Encode(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                     (int32_t*)nullptr, ni);
  return (a > b ? a : b) + 256;
}

cudaError_t launch_histogram(const uint64_t* words, uint64_t* sorted, size_t n, int nbits, uint64_t* uniq,
                             int32_t* counts, int32_t* nruns, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const int ni = (int)n;
  size_t bytes = scratch_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(scratch, bytes, words, sorted, ni, 0, nbits, s);
  if (e != cudaSuccess) return e;
  bytes = scratch_bytes;
  return cub::DeviceRunLengthEncode::Encode(scratch, bytes, sorted, uniq, counts, nruns, ni, s);
}

}  // namespace qsb
