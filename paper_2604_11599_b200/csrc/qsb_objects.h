// Host-side objects shared by the C-ABI translation units (qsb_api.cpp, qsb_slice_api.cpp):
// the error slot, the CUDA-check macro, device buffers, contexts and state objects.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/qsb.h"
#include "qsb_plan.h"

namespace qsb {
// record `msg` as qsb_last_error() and return `code`
int fail(int code, const std::string& msg);
}  // namespace qsb


#define QSB_CUDA(call)                                                                         \
  do {                                                                                         \
    cudaError_t _e = (call);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      int _code = (_e == cudaErrorMemoryAllocation) ? QSB_ERR_OOM : QSB_ERR_CUDA;              \
      return ::qsb::fail(_code, std::string(#call) + ": " + cudaGetErrorString(_e));                  \
    }                                                                                          \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want ? want : 16);
    if (e == cudaSuccess) bytes = want ? want : 16;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};


// makes `dev` current for the scope of a C-ABI call, restores the caller's device
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct qsb_ctx_s {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  std::vector<cudaEvent_t> pass_events;
  int64_t opt_tile = 0, opt_batch = 0, opt_resident_max = -1, opt_engine = -1, opt_jit = 1, opt_jit_min = 13;
  int64_t opt_dedup = 1, opt_reg_bits = 4, opt_fuse = 1, opt_lowq = 0, opt_jit_async = 0, opt_ev_lowq = 0, opt_ev_jit = 1, opt_ev_jit_terms = 32, opt_defer_copy = 1, opt_zero_fill = 1;
  qsb::EngineOptions eopt;  // planner / NVRTC generator options (qsb_plan.h)
  DevBuf state, partial, ctl, bits, guards, mats, params, predrawn, status, counters, misc, misc2, trace, dedup;
  DevBuf shotwords, histo;  // device-side shot histogram (qsb_sample_counts)
  DevBuf histbits;          // exact outcome histories of the dedup'd batch
  std::map<size_t, std::pair<void*, void*>> ev_jit;  // reducer source hash -> (library, kernel)
  qsb_stats last{};
  double run_flops = 0;  // floating-point work of the pass kernels in the current run
  bool run_physical = false;  // dedup ran: bytes / flops come from the device counters
};

struct qsb_state_s {
  qsb_ctx ctx = nullptr;
  int n = 0;
  int c64 = 0;
  DevBuf amps, scratch, tmp;
};

