// Per-pass specialised kernels, generated at tape-compile time and built with NVRTC
// for sm_100a (see qsb_jit.cpp).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "qsb_plan.h"

namespace qsb {

struct JitKernel {
  void* lib = nullptr;   // cudaLibrary_t
  void* kern = nullptr;  // cudaKernel_t
  size_t smem = 0;
  int64_t max_grid = 148;  // resident CTAs (persistent kernel)
  int threads = 256;       // 2^(k - register bits)
};

// true if libnvrtc could be loaded
bool jit_available();
// the loaded NVRTC's version (0.0 when none)
void jit_nvrtc_version(int* major, int* minor);

// true if a phase of the pass reads the per-item staged gates (see pass_persistent)
bool pass_needs_stage(const TapeInfo& t, const StreamPlan& P, int pass);

// one pass kernel's source / cubin (jit_prepare) before it is loaded (jit_load)
struct JitJob {
  int pass = -1;
  std::string src, path;
  std::vector<char> cubin;
  std::string log;
  bool ok = false, from_cache = false;
};
struct JitJobs {
  std::vector<JitJob> jobs;
  std::string error;
  double ms = 0;
};
// host half (no CUDA calls; background-thread safe): sources, cache, parallel NVRTC
JitJobs jit_prepare(const TapeInfo& t, const StreamPlan& P, int c64, bool fuse);
// device half: load the cubins into modules / kernels
std::string jit_load(const TapeInfo& t, const StreamPlan& P, int c64, JitJobs& jobs, std::vector<JitKernel>& out,
                     double* compile_ms, int* compiled, int* cached);

// Generates, compiles (parallel, cached by source hash in $QSB_JIT_CACHE or
// /tmp/qsb_jit_cache) and loads one kernel per register-blocked pass of `P`.
// out[i] stays empty for passes without phases.  Returns "" or an error.
std::string jit_build(const TapeInfo& t, const StreamPlan& P, int c64, bool fuse, std::vector<JitKernel>& out,
                      double* compile_ms, int* compiled, int* cached);

// compile every pass kernel without loading it (host-only self test)
std::string jit_compile_only(const TapeInfo& t, const StreamPlan& P, int c64, bool fuse, int* kernels, double* ms);

// the generated CUDA source of pass `pass` (debug / tests)
std::string jit_source(const TapeInfo& t, const StreamPlan& P, int pass, int c64, bool fuse);

cudaError_t jit_launch(const JitKernel& jk, const StreamArgs& a, const PassDesc& pd, cudaStream_t s);

// ---- NVRTC-specialised Pauli reducer (one launch group of k_expval_acc) ---------------
struct EvJitMap {
  int tpos[8];         // thread bit i -> tile position
  uint16_t soff[16];   // swizzled slot offset of register j
  int t0, nt;          // its terms [t0, t0 + nt) (launch-relative)
};
struct EvJitTerm {
  uint32_t xr, zsig, zl;
  uint64_t zg;
  int ny, out;
};
struct EvJitSpec {
  int c64 = 0, lowq = 2;
  bool regacc = true;            // per-term accumulators in registers (else shared memory)
  std::vector<EvJitMap> maps;
  std::vector<EvJitTerm> terms;  // sorted by (map, xr, Re/Im) like the generic launch
};
std::string ev_jit_source(const EvJitSpec& s);
// compile (parallel, disk-cached) and load one kernel per source; out[i] receives the kernel
// of srcs[i] (kern == nullptr on failure, then the caller runs the generic kernel)
std::string ev_jit_build(const std::vector<std::string>& srcs, std::vector<JitKernel>& out);
void jit_release(std::vector<JitKernel>& ks);

}  // namespace qsb
