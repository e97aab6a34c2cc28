// NVRTC specialisation of the fused passes.
//
// The generic register-blocked kernel (qsb_pass_reg.cu) dispatches every gate through
// a switch on (kind, target register bit, controls).  Each switch join forces the
// compiler to shuffle the 16 register amplitudes back into canonical registers:
// measured on B200, IMAD/MOV made up ~44% of the issued instructions against ~25%
// FP64.  Here every pass of a compiled tape becomes its own kernel whose phases are
// straight-line code: targets and register-bit controls are compile-time constants
// (an x is a register renaming, a controlled gate touches only the matching pairs),
// thread-bit controls become selects, and only guarded gates keep a (CTA-uniform)
// branch.  Matrices still come from the per-CTA shared-memory staging, so ParamRef
// tapes (one matrix set per VQE point) use the same kernels.  Each phase is a
// __noinline__ function (phases communicate through shared memory only), which keeps
// ptxas time linear in the number of phases.
//
// Kernels are compiled once per tape (compile-once, like the reference's kir.lower),
// in parallel, and cached on disk by source hash.
#include "qsb_jit.h"

#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <thread>

#include "qsb_pass_common.cuh"

namespace qsb {

#include "jit_prelude.inc"

namespace {

struct Nvrtc {
  void* h = nullptr;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  int major = 0, minor = 0;  // nvrtcVersion (part of the cubin cache key)
  bool ok = false;
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    // the toolkit's NVRTC first, by path: a process that imported torch already has the
    // wheel's libnvrtc.so.12 (12.8) mapped, which a soname lookup would return, and its
    // ptxas materialises the swapped FFMA2 operands of the complex64 blocks as MOV pairs
    // (measured on B200: 20 % of a DYN20 c64 pass's instructions) where 12.9 uses the
    // free LO_HI operand swizzle.  $QSB_NVRTC overrides.
    const char* env = getenv("QSB_NVRTC");
    for (const char* name : {env && *env ? env : "", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                             "libnvrtc.so"}) {
      if (!*name) continue;
      n.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) return;
    auto ver = (nvrtcResult(*)(int*, int*))dlsym(n.h, "nvrtcVersion");
    if (ver) ver(&n.major, &n.minor);
    n.create = (decltype(n.create))dlsym(n.h, "nvrtcCreateProgram");
    n.compile = (decltype(n.compile))dlsym(n.h, "nvrtcCompileProgram");
    n.cubin_size = (decltype(n.cubin_size))dlsym(n.h, "nvrtcGetCUBINSize");
    n.cubin = (decltype(n.cubin))dlsym(n.h, "nvrtcGetCUBIN");
    n.log_size = (decltype(n.log_size))dlsym(n.h, "nvrtcGetProgramLogSize");
    n.log = (decltype(n.log))dlsym(n.h, "nvrtcGetProgramLog");
    n.destroy = (decltype(n.destroy))dlsym(n.h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size && n.log && n.destroy;
  });
  return n;
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// cubin cache: $QSB_JIT_CACHE, else a per-user directory ($XDG_CACHE_HOME or ~/.cache, then
// /tmp/qsb_jit_cache-<uid>) created 0700 -- never a shared, predictable world-writable path
std::string cache_dir() {
  const char* e = getenv("QSB_JIT_CACHE");
  std::string d;
  if (e && *e) {
    d = e;
  } else if (const char* x = getenv("XDG_CACHE_HOME"); x && *x) {
    d = std::string(x) + "/qsb_jit";
  } else if (const char* h = getenv("HOME"); h && *h) {
    mkdir((std::string(h) + "/.cache").c_str(), 0700);
    d = std::string(h) + "/.cache/qsb_jit";
  } else {
    d = "/tmp/qsb_jit_cache-" + std::to_string((unsigned)getuid());
  }
  mkdir(d.c_str(), 0700);
  return d;
}

const char* kOpts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-DQSB_JIT=1"};

bool compile_one(const std::string& src, std::vector<char>& cubin, std::string& log) {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    log = "libnvrtc not available";
    return false;
  }
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "qsb_pass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return false;
  }
  nvrtcResult rc = nv.compile(prog, (int)(sizeof(kOpts) / sizeof(kOpts[0])), kOpts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  if (ls > 1) {
    log.resize(ls);
    nv.log(prog, &log[0]);
  }
  bool ok = rc == NVRTC_SUCCESS;
  if (ok) {
    size_t n = 0;
    nv.cubin_size(prog, &n);
    cubin.resize(n);
    nv.cubin(prog, cubin.data());
  }
  nv.destroy(&prog);
  return ok;
}

// ---------------------------------------------------------------------------
// code generation
// ---------------------------------------------------------------------------


const char* kHelpers = R"(
__device__ __forceinline__ A CM(R mr, R mi, A a) { return qsb::cmul<R>(mr, mi, a); }
__device__ __forceinline__ void G_GEN(A& a0, A& a1, const R* m) {
  A b0 = qsb::cmac2<R>(m[0], m[1], a0, m[2], m[3], a1);
  A b1 = qsb::cmac2<R>(m[4], m[5], a0, m[6], m[7], a1);
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_REAL(A& a0, A& a1, const R* m) {
  A b0 = qsb::mk<R>(fma(m[0], a0.x, m[2] * a1.x), fma(m[0], a0.y, m[2] * a1.y));
  A b1 = qsb::mk<R>(fma(m[4], a0.x, m[6] * a1.x), fma(m[4], a0.y, m[6] * a1.y));
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_RX(A& a0, A& a1, const R* m) {
  A b0 = qsb::mk<R>(fma(m[0], a0.x, -m[3] * a1.y), fma(m[0], a0.y, m[3] * a1.x));
  A b1 = qsb::mk<R>(fma(m[6], a1.x, -m[5] * a0.y), fma(m[6], a1.y, m[5] * a0.x));
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_ANTI(A& a0, A& a1, const R* m) {
  A b0 = qsb::cmul<R>(m[2], m[3], a1);
  A b1 = qsb::cmul<R>(m[4], m[5], a0);
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_DIAG(A& a0, A& a1, const R* m) {
  a0 = qsb::cmul<R>(m[0], m[1], a0);
  a1 = qsb::cmul<R>(m[6], m[7], a1);
}
)";

// complex64: the same helpers on packed FP32 pairs (fma.rn.f32x2 / mul.rn.f32x2).  Each
// lane runs exactly the scalar chain above (same terms, same order: the re lane is the
// scalar re chain, the im lane the scalar im chain), so results are bit-identical to the
// scalar helpers and to the generic kernel, with half the FP32 instructions.
const char* kPackedHelpers = R"(
__device__ __forceinline__ unsigned long long U(A a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ A F(unsigned long long d) { return *reinterpret_cast<A*>(&d); }
__device__ __forceinline__ A ffma2(A a, A b, A c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(U(a)), "l"(U(b)), "l"(U(c)));
  return F(d);
}
__device__ __forceinline__ A fmul2(A a, A b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(U(a)), "l"(U(b)));
  return F(d);
}
__device__ __forceinline__ A PR(R m) { return qsb::mk<R>(m, m); }    // real part, both lanes
__device__ __forceinline__ A PI(R m) { return qsb::mk<R>(-m, m); }   // imaginary part: (-mi, +mi)
__device__ __forceinline__ A SW(A a) { return qsb::mk<R>(a.y, a.x); }
__device__ __forceinline__ A CM(R mr, R mi, A a) { return ffma2(PR(mr), a, fmul2(PI(mi), SW(a))); }
__device__ __forceinline__ A MAC2(const R* m, int o, A a0, A a1) {  // cmac2(m[o..o+1], a0, m[o+2..o+3], a1)
  return ffma2(PR(m[o]), a0, ffma2(PI(m[o + 1]), SW(a0), ffma2(PR(m[o + 2]), a1, fmul2(PI(m[o + 3]), SW(a1)))));
}
__device__ __forceinline__ void G_GEN(A& a0, A& a1, const R* m) {
  A b0 = MAC2(m, 0, a0, a1), b1 = MAC2(m, 4, a0, a1);
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_REAL(A& a0, A& a1, const R* m) {
  A b0 = ffma2(PR(m[0]), a0, fmul2(PR(m[2]), a1));
  A b1 = ffma2(PR(m[4]), a0, fmul2(PR(m[6]), a1));
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_RX(A& a0, A& a1, const R* m) {
  A b0 = ffma2(PR(m[0]), a0, fmul2(PI(m[3]), SW(a1)));
  A b1 = ffma2(PR(m[6]), a1, fmul2(PI(m[5]), SW(a0)));
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_ANTI(A& a0, A& a1, const R* m) {
  A b0 = CM(m[2], m[3], a1);
  A b1 = CM(m[4], m[5], a0);
  a0 = b0; a1 = b1;
}
__device__ __forceinline__ void G_DIAG(A& a0, A& a1, const R* m) {
  a0 = CM(m[0], m[1], a0);
  a1 = CM(m[6], m[7], a1);
}
)";

// packed sparse helper: the scalar G_S<z> chain on f32x2 pairs (bit-identical)
std::string sparse_helper_packed(uint32_t z) {
  std::ostringstream o;
  o << "__device__ __forceinline__ void G_S" << z << "(A& a0, A& a1, const R* m) {\n  A b0, b1;\n";
  for (int r = 0; r < 2; ++r) {
    const int o0 = 4 * r;
    // innermost first: m[o0+3] (imag, a1), m[o0+2] (real, a1), m[o0+1] (imag, a0), m[o0] (real, a0)
    const int ci[4] = {o0 + 3, o0 + 2, o0 + 1, o0 + 0};
    const char* xv[4] = {"SW(a1)", "a1", "SW(a0)", "a0"};
    const bool im[4] = {true, false, true, false};
    std::string acc;
    for (int i = 0; i < 4; ++i) {
      if (z >> ci[i] & 1) continue;
      const std::string coef = std::string(im[i] ? "PI" : "PR") + "(m[" + std::to_string(ci[i]) + "])";
      acc = acc.empty() ? "fmul2(" + coef + ", " + xv[i] + ")" : "ffma2(" + coef + ", " + xv[i] + ", " + acc + ")";
    }
    if (acc.empty()) acc = "qsb::mk<R>(0.f, 0.f)";
    o << "  " << (r ? "b1" : "b0") << " = " << acc << ";\n";
  }
  o << "  a0 = b0; a1 = b1;\n}\n";
  return o.str();
}

// A dense 2x2 with statically-zero components dropped from cmac2's FMA chain.  The
// chain keeps cmac2's association order, and the dropped terms are exact zeros, so
// the result is bit-identical to the generic kernel's cmac2.
std::string sparse_helper(uint32_t z) {
  std::ostringstream o;
  auto chain = [&](const char* out, const int* c, const char** x, const bool* neg) {
    // terms innermost first: (c[i], x[i], neg[i])
    std::string acc;
    for (int i = 0; i < 4; ++i) {
      if (z >> c[i] & 1) continue;
      std::string coef = std::string(neg[i] ? "-" : "") + "m[" + std::to_string(c[i]) + "]";
      if (acc.empty()) acc = coef + " * " + x[i];
      else acc = "fma(" + coef + ", " + x[i] + ", " + acc + ")";
    }
    if (acc.empty()) acc = "(R)0";
    o << "  " << out << " = " << acc << ";\n";
  };
  o << "__device__ __forceinline__ void G_S" << z << "(A& a0, A& a1, const R* m) {\n  A b0, b1;\n";
  for (int r = 0; r < 2; ++r) {
    const int o0 = 4 * r;  // m00 m01 (row 0) or m10 m11 (row 1)
    int cre[4] = {o0 + 3, o0 + 2, o0 + 1, o0 + 0};
    const char* xre[4] = {"a1.y", "a1.x", "a0.y", "a0.x"};
    bool nre[4] = {true, false, true, false};
    int cim[4] = {o0 + 3, o0 + 2, o0 + 1, o0 + 0};
    const char* xim[4] = {"a1.x", "a1.y", "a0.x", "a0.y"};
    bool nim[4] = {false, false, false, false};
    chain(r ? "b1.x" : "b0.x", cre, xre, nre);
    chain(r ? "b1.y" : "b0.y", cim, xim, nim);
  }
  o << "  a0 = b0; a1 = b1;\n}\n";
  return o.str();
}

// one fused block (qsb_plan.h fuse_phase): a dense 2x2 / 4x4 over register bits qa (matrix
// bit 0) and qb (bit 1) with its entries at qsb_cf[cf ...]; exact-zero parts dropped
// complex64 fused blocks as packed FFMA2 (fma.rn.f32x2): one instruction per complex
// coefficient part instead of two FFMA -- (mr, mr) * (xr, xi) and (-mi, mi) * (xi, xr), the
// swapped operand being a free LO_HI operand modifier.  Halves the FP32 instructions of a
// block (complex64 passes are issue / instruction-fetch bound).  $QSB_JIT_FFMA2=0 disables.
bool packed_blocks(const StreamPlan& P, int c64) { return c64 && P.opt.ffma2 == 1; }

void emit_block(std::ostringstream& o, const FuseItem& f, int cf, int nr, bool packed) {
  const int d = f.qb < 0 ? 2 : 4;
  const int A = 1 << f.qa, B = f.qb < 0 ? 0 : 1 << f.qb;
  o << "  {  // fused block of " << f.ngates << " gates on register bits " << f.qa;
  if (f.qb >= 0) o << ", " << f.qb;
  o << "\n";
  for (int j = 0; j < nr; ++j) {
    if ((j & A) || (j & B)) continue;
    const int idx[4] = {j, j | A, j | B, j | A | B};
    o << "  { const A";
    for (int c = 0; c < d; ++c) o << (c ? ", " : " ") << "x" << c << " = v" << idx[c];
    o << ";\n";
    if (packed) {
      for (int r = 0; r < d; ++r) {
        std::string acc;
        for (int c = 0; c < d; ++c) {
          const int e = 2 * (r * d + c);
          for (int part = 0; part < 2; ++part) {  // 0: real part (mr, mr) * x; 1: (-mi, mi) * swap(x)
            if (f.m[e + part] == 0.0) continue;
            const std::string x = part ? "qsb::mk<R>(x" + std::to_string(c) + ".y, x" + std::to_string(c) + ".x)"
                                       : "x" + std::to_string(c);
            const std::string k = "qsb_cf2[" + std::to_string(cf + e + part) + "]";
            acc = "ffma2(" + k + ", " + x + ", " + (acc.empty() ? std::string("qsb::mk<R>(0.f, 0.f)") : acc) + ")";
          }
        }
        o << "    v" << idx[r] << " = " << (acc.empty() ? std::string("qsb::mk<R>(0.f, 0.f)") : acc) << ";\n";
      }
      o << "  }\n";
      continue;
    }
    for (int r = 0; r < d; ++r) {
      auto chain = [&](bool im) {
        std::string acc;
        for (int c = d - 1; c >= 0; --c) {
          const int e = 2 * (r * d + c);
          // re: mr*x.x - mi*x.y ; im: mr*x.y + mi*x.x
          const struct { int k; const char* x; bool neg; } terms[2] = {
              {e + 1, im ? ".x" : ".y", !im}, {e, im ? ".y" : ".x", false}};
          for (const auto& tm : terms) {
            if (f.m[tm.k] == 0.0) continue;
            const std::string coef = std::string(tm.neg ? "-" : "") + "qsb_cf[" + std::to_string(cf + tm.k) + "]";
            const std::string x = "x" + std::to_string(c) + tm.x;
            acc = acc.empty() ? coef + " * " + x : "fma(" + coef + ", " + x + ", " + acc + ")";
          }
        }
        return acc.empty() ? std::string("(R)0") : acc;
      };
      o << "    v" << idx[r] << " = qsb::mk<R>(" << chain(false) << ", " << chain(true) << ");\n";
    }
    o << "  }\n";
  }
  o << "  }\n";
}

bool edge_x_disabled(const StreamPlan& P) { return P.opt.edge_x == 0; }

// Phases are separate __noinline__ functions (ptxas time linear in the phases) except for
// complex128, where inlining them into the pass kernel measured 2.2 % faster on B200 (DYN20
// pass time 607.8 -> 594.5 ms per 2048 shots; no callee-saved spills at phase boundaries)
// for ~1.7x the NVRTC time; complex64 measured 7 % slower inlined.  $QSB_JIT_INLINE_PHASES
// = 0 / 1 overrides.
bool inline_phases(const StreamPlan& P, int c64, const PassDesc& pd) {
  if (P.opt.inline_phases >= 0) return P.opt.inline_phases == 1;
  if (P.opt.inline_max_phases > 0 && pd.phase_count > P.opt.inline_max_phases) return false;
  return !c64 && pd.pgate_count >= P.opt.inline_min_gates;
}

void emit_phase(std::ostringstream& o, const TapeInfo& t, const StreamPlan& P, const PassDesc& pd, int ph_index,
                const PhaseDesc& ph, int sb, const std::vector<FuseItem>& items, int cf0, bool direct = false) {
  const int c64 = sb == 4;
  const int nr = 1 << P.rb;  // amplitudes per thread
  if (direct) {  // last phase of a DIRECT pass (qsb_pass_common.cuh): inlined, stores to HBM
    o << "template <typename MID> __device__ __forceinline__ void phL"
      << "(A* __restrict__ tile, const uint32_t* __restrict__ swz, const qsb::SGate<R>* __restrict__ sg, "
         "const int tid, A* __restrict__ dst, const uint64_t* __restrict__ hi_off, MID mid) {\n";
  } else {
    o << (inline_phases(P, c64, pd) ? "__device__ __forceinline__ void ph" : "__device__ __noinline__ void ph") << ph_index
      << "(A* __restrict__ tile, const uint32_t* __restrict__ swz, const qsb::SGate<R>* __restrict__ sg, "
         "const int tid) {\n";
  }
  o << "  const uint32_t base = 0u";
  for (int i = 0; i < ph.nt; ++i) o << " | ((((uint32_t)tid >> " << i << ") & 1u) << " << (int)ph.tpos[i] << ")";
  o << ";\n  const uint32_t sb = base ^ swz[base >> " << sb << "];\n";
  // X gates with a per-item condition (control outside the tile, or an if-guard) that
  // commute to the start or the end of the phase become a conditional XOR of the thread's
  // slot base at the phase's loads / stores (the slot map is XOR-linear in the register
  // index) instead of a branch whose join needs 2 x 16 register moves
  std::vector<int> edge(items.size(), 0);  // 1: at the loads, 2: at the stores
  if (!edge_x_disabled(P)) {
    auto bits_of = [&](const FuseItem& it) -> uint32_t {
      if (it.gate < 0) return (1u << it.qa) | (it.qb >= 0 ? 1u << it.qb : 0u);
      const PhaseGate& q = P.phase_gates[it.gate];
      switch (q.kind) {
        case PK_DENSE: case PK_XPERM: case PK_ANTI: case PK_DIAG_R: return q.cmR | (1u << q.jt);
        case PK_DIAG_T: case PK_DIAG_G: return q.cmR;
        default: return ~0u;
      }
    };
    for (size_t i = 0; i < items.size(); ++i) {
      if (items[i].gate < 0) continue;
      const PhaseGate& q = P.phase_gates[items[i].gate];
      // per-item (guard / out-of-tile control) or per-thread (control on a thread
      // position) condition; an unconditional X is a free register renaming anyway
      if (q.kind != PK_XPERM || q.cmR || !(q.guard >= 0 || q.gcm != 0 || q.cmT != 0)) continue;
      bool front = true, back = !direct;
      for (size_t j = 0; j < items.size(); ++j) {
        if (j == i || edge[j] == 1) continue;  // earlier front-moved X gates commute with it
        if (!(bits_of(items[j]) >> q.jt & 1)) continue;
        if (j < i) front = false;
        else back = false;
      }
      if (front) edge[i] = 1;
      else if (back) edge[i] = 2;
    }
  }
  auto edge_flip = [&](int which, const char* name) {
    o << "  uint32_t " << name << " = 0u;\n";
    for (size_t i = 0; i < items.size(); ++i)
      if (edge[i] == which) {
        const PhaseGate& q = P.phase_gates[items[i].gate];
        std::string cond;
        if (q.guard >= 0 || q.gcm != 0)
          cond = "sg[" + std::to_string(items[i].gate - pd.pgate_begin) + "].kind != " + std::to_string((int)PK_SKIP);
        if (q.cmT)
          cond += std::string(cond.empty() ? "" : " && ") + "(base & " + std::to_string(q.cmT) + "u) == " +
                  std::to_string(q.cvT) + "u";
        o << "  if (" << cond << ") " << name << " ^= " << ph.soff[1 << q.jt] << "u;\n";
      }
  };
  edge_flip(1, "fl_in");
  for (int j = 0; j < nr; ++j) o << "  A v" << j << " = tile[(sb ^ fl_in) ^ " << ph.soff[j] << "u];\n";
  if (direct) o << "  mid();\n";
  int cf = cf0;
  for (size_t ii = 0; ii < items.size(); ++ii) {
    const FuseItem& item = items[ii];
    if (edge[ii]) continue;
    if (item.gate < 0) {
      emit_block(o, item, cf, nr, packed_blocks(P, c64));
      cf += item.qb < 0 ? 8 : 32;
      continue;
    }
    const int gidx = item.gate;
    const PhaseGate& q = P.phase_gates[gidx];
    const int gi = gidx - pd.pgate_begin;
    const MatSrc& ms = t.mats[q.mat];
    const bool need_skip = q.guard >= 0 || q.gcm != 0 || q.kind == PK_DIAG_G;
    o << "  {  // gate " << gi << " kind " << q.kind << "\n";
    if (need_skip) o << "  if (sg[" << gi << "].kind != " << (int)PK_SKIP << ") {\n";
    // literal matrices live in the module's constant bank (FMA operands straight from the
    // constant cache, no registers / shared loads); ParamRef and per-CTA factors use staging
    if (ms.has_matrix && q.kind != PK_DIAG_G) o << "  const R* m = qsb_cm + " << 8 * gi << ";\n";
    else o << "  const R* m = sg[" << gi << "].m;\n";
    const bool thr = q.cmT != 0;
    if (thr) o << "  const bool c = (base & " << q.cmT << "u) == " << q.cvT << "u;\n";
    auto sel_pair = [&](int j0, int j1, const char* fn) {
      if (!thr) {
        o << "  " << fn << "(v" << j0 << ", v" << j1 << ", m);\n";
      } else {
        o << "  { A t0 = v" << j0 << ", t1 = v" << j1 << "; " << fn << "(t0, t1, m); v" << j0 << " = c ? t0 : v" << j0
          << "; v" << j1 << " = c ? t1 : v" << j1 << "; }\n";
      }
    };
    auto scale = [&](int j, const char* dr, const char* di) {
      if (!thr) o << "  v" << j << " = CM(" << dr << ", " << di << ", v" << j << ");\n";
      else o << "  v" << j << " = c ? CM(" << dr << ", " << di << ", v" << j << ") : v" << j << ";\n";
    };
    switch (q.kind) {
      case PK_DENSE:
      case PK_XPERM:
      case PK_ANTI:
      case PK_DIAG_R: {
        const int b = 1 << q.jt;
        std::string fname = "G_GEN";
        if (q.kind == PK_DENSE) {
          DenseVariant dv = dense_variant(ms);
          const uint32_t z = zero_mask(ms);
          fname = dv == DV_REAL ? "G_REAL" : dv == DV_RX ? "G_RX" : z ? "G_S" + std::to_string(z) : "G_GEN";
        }
        const char* fn = fname.c_str();
        if (q.kind == PK_DENSE) {
        } else if (q.kind == PK_ANTI) {
          fn = "G_ANTI";
        } else if (q.kind == PK_DIAG_R) {
          fn = "G_DIAG";
        }
        for (int j = 0; j < nr; ++j) {
          if (j & b) continue;
          if (((uint32_t)j & q.cmR) != q.cvR) continue;
          const int j1 = j | b;
          if (q.kind == PK_XPERM) {
            if (!thr) o << "  { A x = v" << j << "; v" << j << " = v" << j1 << "; v" << j1 << " = x; }\n";
            else
              o << "  { A x = v" << j << "; v" << j << " = c ? v" << j1 << " : v" << j << "; v" << j1 << " = c ? x : v"
                << j1 << "; }\n";
          } else if (q.kind == PK_DIAG_R && q.diag_one0) {
            scale(j1, "m[6]", "m[7]");
          } else {
            sel_pair(j, j1, fn);
          }
        }
      } break;
      case PK_DIAG_T: {
        o << "  const bool bt = (base >> " << q.tp << ") & 1u;\n";
        o << "  const R dr = bt ? m[6] : m[0], di = bt ? m[7] : m[1];\n";
        for (int j = 0; j < nr; ++j)
          if (((uint32_t)j & q.cmR) == q.cvR) scale(j, "dr", "di");
      } break;
      case PK_DIAG_G: {
        for (int j = 0; j < nr; ++j)
          if (((uint32_t)j & q.cmR) == q.cvR) scale(j, "m[0]", "m[1]");
      } break;
      default:
        o << "  // unsupported kind\n";
        break;
    }
    if (need_skip) o << "  }\n";
    o << "  }\n";
  }
  if (direct) {
    // HBM offset of register j: pdep over the tile qubits is linear over disjoint bits, so
    // it is the thread's part (hi_off table) OR a compile-time constant per register
    uint32_t tmask = 0;
    for (int i = 0; i < ph.nt; ++i) tmask |= 1u << ph.tpos[i];
    int rpos[kMaxRegBits], nrb = 0;
    for (int p = 0; p < pd.k; ++p)
      if (!(tmask >> p & 1)) rpos[nrb++] = p;
    o << "  const uint64_t tof = (uint64_t)(base & " << ((1u << pd.lowq) - 1) << "u) | hi_off[base >> " << pd.lowq
      << "];\n";
    for (int j = 0; j < nr; ++j) {
      uint64_t l = 0;
      for (int b = 0; b < nrb; ++b)
        if (j >> b & 1) l |= 1ull << rpos[b];
      // tile element l -> qubit offsets (local bit p <-> p-th qubit of S)
      uint64_t off = 0;
      int p = 0;
      for (int q = 0; q < 64 && p < pd.k; ++q)
        if (pd.smask >> q & 1) {
          if (l >> p & 1) off |= 1ull << q;
          ++p;
        }
      o << "  dst[tof | " << off << "ull] = v" << j << ";\n";
    }
  } else {
    edge_flip(2, "fl_out");
    for (int j = 0; j < nr; ++j) o << "  tile[(sb ^ fl_out) ^ " << ph.soff[j] << "u] = v" << j << ";\n";
  }
  o << "}\n";
}

}  // namespace

bool jit_available() { return nvrtc().ok; }

void jit_nvrtc_version(int* major, int* minor) {
  *major = nvrtc().major;
  *minor = nvrtc().minor;
}

// staging is needed only if a phase reads the staged gates: per-item skips (guards,
// out-of-tile controls, per-tile diagonal factors), non-literal matrices, swap phases
bool pass_needs_stage(const TapeInfo& t, const StreamPlan& P, int pass) {
  const PassDesc& pd = P.passes[pass];
  for (int g = pd.pgate_begin; g < pd.pgate_begin + pd.pgate_count; ++g) {
    const PhaseGate& q = P.phase_gates[g];
    if (q.guard >= 0 || q.gcm != 0 || q.kind == PK_DIAG_G || !t.mats[q.mat].has_matrix) return true;
  }
  for (int i = 0; i < pd.phase_count; ++i)
    if (P.phases[pd.phase_begin + i].nt < 0) return true;
  return false;
}

// buffering mode of a pass kernel (qsb_pass_common.cuh): one thread group per CTA, two
// CTAs per SM.  (Round 1 also shipped a two-group / three-tile-ring mode, measured 6-20 %
// slower on B200 -- the per-item context loads and mbarrier waits sat on each group's
// critical path -- and it was removed.)
int jit_pass_mode(const TapeInfo&, const StreamPlan&, int, int) { return 0; }

// DIRECT last phase (qsb_pass_common.cuh): complex128 MODE 0 passes without an epilogue
// and without per-item gate staging whose last phase is a register phase with coalesced
// stores.  Measured on B200: streaming probe 4.46 -> 4.75 TB/s, RDC30 neutral, no DYN20
// pass qualifies (its last phases hold qubits 0-3 in registers, which would make the
// stores uncoalesced); staged passes (ParamRef, VQE24) measured slower, so they are
// excluded.  $QSB_LAST_DIRECT=0 disables, =2 also allows staged passes.
bool jit_pass_direct(const TapeInfo& t, const StreamPlan& P, int pass, int c64, int mode) {
  const int lvl = P.opt.last_direct;
  if (lvl == 0) return false;
  const PassDesc& pd = P.passes[pass];
  if (c64 || mode != 0 || pd.epi || pd.phase_count < 1) return false;
  if (lvl < 2 && pass_needs_stage(t, P, pass)) return false;
  const PhaseDesc& ph = P.phases[pd.phase_begin + pd.phase_count - 1];
  if (ph.nt < 3) return false;
  // store coalescing: with s of the tile positions 0..s-1 in registers (each thread owns
  // 2^s consecutive amplitudes), lanes advance by 2^s amplitudes and a warp store covers
  // 16-byte pieces of 2^s * 16-byte runs that the thread's other registers complete
  // (merged in L2).  s <= $QSB_LAST_DIRECT_MAXLOW (default 0: lanes 0..7 cover 128 B).
  const int maxlow = P.opt.last_direct_maxlow;
  uint32_t tmask = 0;
  for (int i = 0; i < ph.nt; ++i) tmask |= 1u << ph.tpos[i];
  int s = 0;
  while (s < pd.k && !(tmask >> s & 1)) ++s;  // low positions held in registers
  if (s > maxlow) return false;
  for (int i = 0; i < 3; ++i)  // the next three tile positions are the lanes' low bits
    if (ph.tpos[i] != s + i) return false;
  return true;
}

std::string jit_source(const TapeInfo& t, const StreamPlan& P, int pass, int c64, bool fuse) {
  const PassDesc& pd = P.passes[pass];
  const int sb = c64 ? 4 : 3;
  std::vector<std::vector<FuseItem>> items(pd.phase_count);
  std::vector<int> cf0(pd.phase_count, 0);
  std::vector<double> cfv;  // fused-block matrices of the pass
  for (int i = 0; i < pd.phase_count; ++i) {
    items[i] = fuse_phase(t, P, pd.phase_begin + i, fuse);
    cf0[i] = (int)cfv.size();
    for (const FuseItem& f : items[i])
      if (f.gate < 0) cfv.insert(cfv.end(), f.m, f.m + (f.qb < 0 ? 8 : 32));
  }
  std::ostringstream o;
  for (const char* part : kJitPreludeParts) o << part;
  o << "\ntypedef " << (c64 ? "float" : "double") << " R;\ntypedef " << (c64 ? "float2" : "double2") << " A;\n";
  // packed f32x2 arithmetic pays in the fused complex64 blocks (-6 % DYN20 pass time); the
  // packed versions of the single-gate helpers (kPackedHelpers, bit-identical) measured no
  // gain on DYN20 and a loss on RDC30 / VQE24 ($QSB_JIT_PACKED_GATES=1 selects them)
  const bool packed = packed_blocks(P, c64);
  const bool packed_gates = packed && P.opt.packed_gates == 1;
  o << (packed_gates ? kPackedHelpers : kHelpers);
  if (packed && !packed_gates)
    o << "__device__ __forceinline__ A ffma2(A a, A b, A c) {\n  unsigned long long d;\n"
         "  asm(\"fma.rn.f32x2 %0, %1, %2, %3;\" : \"=l\"(d) : \"l\"(*reinterpret_cast<unsigned long long*>(&a)), "
         "\"l\"(*reinterpret_cast<unsigned long long*>(&b)), \"l\"(*reinterpret_cast<unsigned long long*>(&c)));\n"
         "  return *reinterpret_cast<A*>(&d);\n}\n";
  {  // sparse dense-gate helpers used by this pass
    std::vector<uint32_t> seen;
    for (int g = pd.pgate_begin; g < pd.pgate_begin + pd.pgate_count; ++g) {
      const PhaseGate& q = P.phase_gates[g];
      if (q.kind != PK_DENSE) continue;
      const MatSrc& ms = t.mats[q.mat];
      if (dense_variant(ms) != DV_GEN) continue;
      const uint32_t z = zero_mask(ms);
      if (!z || std::find(seen.begin(), seen.end(), z) != seen.end()) continue;
      seen.push_back(z);
      o << (packed_gates ? sparse_helper_packed(z) : sparse_helper(z));
    }
  }
  {  // literal matrices of the pass, indexed by pass-relative gate (exact hex literals)
    o << "__constant__ R qsb_cm[" << 8 * std::max(1, pd.pgate_count) << "] = {";
    for (int g = 0; g < pd.pgate_count; ++g) {
      const MatSrc& ms = t.mats[P.phase_gates[pd.pgate_begin + g].mat];
      for (int i = 0; i < 8; ++i) {
        char buf[64];
        if (c64) snprintf(buf, sizeof(buf), "%af", (double)(float)ms.mat[i]);
        else snprintf(buf, sizeof(buf), "%a", ms.mat[i]);
        o << (g || i ? ", " : "") << buf;
      }
    }
    if (!pd.pgate_count) o << "0";
    o << "};\n";
  }
  if (!cfv.empty() && packed_blocks(P, c64)) {  // (mr, mr), (-mi, mi) per complex entry, same indices
    o << "__constant__ float2 qsb_cf2[" << cfv.size() << "] = {";
    for (size_t i = 0; i + 1 < cfv.size(); i += 2) {
      char buf[160];
      const float mr = (float)cfv[i], mi = (float)cfv[i + 1];
      snprintf(buf, sizeof(buf), "%s{%af, %af}, {%af, %af}", i ? ", " : "", (double)mr, (double)mr, (double)-mi,
               (double)mi);
      o << buf;
    }
    o << "};\n";
  }
  if (!cfv.empty()) {
    o << "__constant__ R qsb_cf[" << cfv.size() << "] = {";
    for (size_t i = 0; i < cfv.size(); ++i) {
      char buf[64];
      if (c64) snprintf(buf, sizeof(buf), "%af", (double)(float)cfv[i]);
      else snprintf(buf, sizeof(buf), "%a", cfv[i]);
      o << (i ? ", " : "") << buf;
    }
    o << "};\n";
  }
  const int mode = jit_pass_mode(t, P, pass, c64);
  const bool direct = jit_pass_direct(t, P, pass, c64, mode);
  for (int i = 0; i < pd.phase_count; ++i) {
    const PhaseDesc& ph = P.phases[pd.phase_begin + i];
    if (ph.nt >= 0) emit_phase(o, t, P, pd, i, ph, sb, items[i], cf0[i], direct && i == pd.phase_count - 1);
  }
  const bool stage = pass_needs_stage(t, P, pass);
  const int threads = pass_groups(mode) << (pd.k - P.rb);
  if (direct)
    o << "struct LastPhase {\n  template <typename MID> __device__ void operator()(const qsb::PassCtx<R>& cx, A* dst, "
         "const uint64_t* hi_off, MID mid) const {\n    phL(cx.tile, cx.swz, cx.sg, cx.tid, dst, hi_off, mid);\n  }\n};\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << std::max(1, P.opt.minblocks)
    << ") qsb_jit_pass(qsb::StreamArgs a, qsb::PassDesc pd) {\n";
  o << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n";
  o << "  qsb::pass_persistent<R, " << P.rb << ", " << (stage ? "true" : "false") << ", " << mode << ", "
    << (direct ? "true" : "false") << ">(a, pd, smem_raw, [&](const qsb::PassCtx<R>& cx) {\n";
  for (int i = 0; i < pd.phase_count - (direct ? 1 : 0); ++i) {
    const PhaseDesc& ph = P.phases[pd.phase_begin + i];
    if (ph.nt >= 0) o << "    ph" << i << "(cx.tile, cx.swz, cx.sg, cx.tid);\n";
    else o << "    qsb::pass_swap<R, " << sb << ">(cx, cx.sg[" << (ph.gate_begin - pd.pgate_begin) << "]);\n";
    o << "    cx.sync();\n";
  }
  if (direct) o << "  }, LastPhase());\n}\n";
  else o << "  });\n}\n";
  return o.str();
}

namespace {
// write-then-rename with a name unique per process and thread: concurrent ranks compiling
// the same pass never expose a partially written file under the final name
void write_cache(const std::string& path, const std::vector<char>& cubin) {
  const std::string tmp = path + ".tmp." + std::to_string((long)getpid()) + "." +
                          std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
  std::ofstream f(tmp, std::ios::binary);
  f.write(cubin.data(), (std::streamsize)cubin.size());
  f.close();
  if (!f || rename(tmp.c_str(), path.c_str()) != 0) unlink(tmp.c_str());
}
}  // namespace

// host half of jit_build: generate every pass's source, read the cubin cache, NVRTC-compile
// the misses in parallel and write them back.  No CUDA calls: safe on a background thread.
JitJobs jit_prepare(const TapeInfo& t, const StreamPlan& P, int c64, bool fuse) {
  JitJobs out;
  auto t0 = std::chrono::steady_clock::now();
  if (!P.rb) return out;
  if (!jit_available()) {
    out.error = "libnvrtc not available";
    return out;
  }
  const std::string dir = cache_dir();
  std::vector<JitJob>& jobs = out.jobs;
  for (int i = 0; i < (int)P.passes.size(); ++i) {
    if (P.passes[i].phase_count == 0) continue;
    JitJob j;
    j.pass = i;
    j.src = jit_source(t, P, i, c64, fuse);
    std::string key = j.src;
    for (const char* opt : kOpts) key += opt;
    key += "nvrtc " + std::to_string(nvrtc().major) + "." + std::to_string(nvrtc().minor);
    char name[64];
    snprintf(name, sizeof(name), "/%016llx.cubin", (unsigned long long)fnv1a(key));
    j.path = dir + name;
    std::ifstream f(j.path, std::ios::binary);
    if (f) {
      j.cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
      j.ok = j.from_cache = !j.cubin.empty();
    }
    jobs.push_back(std::move(j));
  }
  std::atomic<size_t> next(0);
  unsigned nthreads = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < nthreads; ++w)
    pool.emplace_back([&] {
      for (size_t i = next++; i < jobs.size(); i = next++) {
        JitJob& j = jobs[i];
        if (j.ok) continue;
        j.ok = compile_one(j.src, j.cubin, j.log);
        if (j.ok) write_cache(j.path, j.cubin);
      }
    });
  for (auto& th : pool) th.join();
  out.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

// device half: load the cubins (on the calling thread; a damaged cache entry is recompiled)
std::string jit_load(const TapeInfo& t, const StreamPlan& P, int c64, JitJobs& J, std::vector<JitKernel>& out,
                     double* compile_ms, int* compiled, int* cached) {
  auto t0 = std::chrono::steady_clock::now();
  out.assign(P.passes.size(), JitKernel());
  *compiled = *cached = 0;
  if (!J.error.empty()) return J.error;
  std::vector<JitJob>& jobs = J.jobs;
  for (JitJob& j : jobs) {
    if (!j.ok) {
      jit_release(out);
      return "NVRTC failed for pass " + std::to_string(j.pass) + ": " + j.log.substr(0, 2000);
    }
    cudaLibrary_t lib;
    cudaError_t e = cudaLibraryLoadData(&lib, j.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess && j.from_cache) {  // a damaged cache entry: drop it, compile afresh
      cudaGetLastError();
      unlink(j.path.c_str());
      j.from_cache = false;
      j.ok = compile_one(j.src, j.cubin, j.log);
      if (!j.ok) {
        jit_release(out);
        return "NVRTC failed for pass " + std::to_string(j.pass) + ": " + j.log.substr(0, 2000);
      }
      write_cache(j.path, j.cubin);
      e = cudaLibraryLoadData(&lib, j.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    }
    if (e != cudaSuccess) {
      jit_release(out);
      return std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e);
    }
    cudaKernel_t k;
    e = cudaLibraryGetKernel(&k, lib, "qsb_jit_pass");
    if (e != cudaSuccess) {
      cudaLibraryUnload(lib);
      jit_release(out);
      return std::string("cudaLibraryGetKernel: ") + cudaGetErrorString(e);
    }
    JitKernel& jk = out[j.pass];
    jk.lib = (void*)lib;
    jk.kern = (void*)k;
    const int mode = jit_pass_mode(t, P, j.pass, c64);
    jk.smem = pass_reg_smem(c64, P.passes[j.pass], P.rb, t.n, pass_needs_stage(t, P, j.pass), mode);
    jk.threads = pass_groups(mode) << (P.passes[j.pass].k - P.rb);
    e = cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jk.smem);
    if (e != cudaSuccess) {
      jit_release(out);
      return std::string("cudaFuncSetAttribute (jit): ") + cudaGetErrorString(e);
    }
    int per_sm = 1, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k, jk.threads, jk.smem);
    // option ctas_per_sm caps the persistent grid (experiment: two contexts on two
    // streams sharing the SMs, experiments/two_stream.py)
    if (P.opt.ctas_per_sm > 0) per_sm = std::min(per_sm, P.opt.ctas_per_sm);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    jk.max_grid = (int64_t)std::max(1, per_sm) * sms;
    if (j.from_cache) (*cached)++;
    else (*compiled)++;
  }
  *compile_ms = J.ms + std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return "";
}

std::string jit_build(const TapeInfo& t, const StreamPlan& P, int c64, bool fuse, std::vector<JitKernel>& out,
                      double* compile_ms, int* compiled, int* cached) {
  JitJobs J = jit_prepare(t, P, c64, fuse);
  return jit_load(t, P, c64, J, out, compile_ms, compiled, cached);
}


std::string jit_compile_only(const TapeInfo& t, const StreamPlan& P, int c64, bool fuse, int* kernels, double* ms) {
  auto t0 = std::chrono::steady_clock::now();
  *kernels = 0;
  for (int i = 0; i < (int)P.passes.size(); ++i) {
    if (P.passes[i].phase_count == 0) continue;
    std::vector<char> cubin;
    std::string log;
    const std::string src = jit_source(t, P, i, c64, fuse);
    if (const char* d = getenv("QSB_JIT_DUMP")) {  // debug: keep the generated sources
      std::ofstream f(std::string(d) + "/pass" + std::to_string(i) + ".cu");
      f << src;
    }
    if (!compile_one(src, cubin, log)) return "pass " + std::to_string(i) + ": " + log;
    (*kernels)++;
  }
  *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return "";
}


// ---------------------------------------------------------------------------
// NVRTC-specialised Pauli reducer: the generic k_expval_acc (qsb_expval.cu) with every
// structural quantity a compile-time constant -- mapping thread positions and swizzled
// register offsets, each class's register X pattern (only the product parts its terms
// use), each term's register Z signs (add / subtract in the butterfly, no sign factors),
// its thread-parity mask, out-of-tile Z mask and output index.  Per term and tile a thread
// does 7 (diagonal: 15) add / subtract, one sign flip and one accumulator update.
// ---------------------------------------------------------------------------

std::string ev_jit_source(const EvJitSpec& S) {
  const int T = (int)S.terms.size();
  const int sbits = S.c64 ? 4 : 3;
  std::ostringstream o;
  for (const char* part : kJitPreludeParts) o << part;
  o << "\ntypedef " << (S.c64 ? "float" : "double") << " R;\ntypedef " << (S.c64 ? "float2" : "double2") << " A;\n";
  o << "__device__ __forceinline__ double sgnd(double x, uint32_t m) {\n"
       "  return __longlong_as_double(__double_as_longlong(x) ^ ((unsigned long long)m << 32));\n}\n";
  o << "__constant__ unsigned long long qsb_ev_zg[" << std::max(1, T) << "] = {";
  for (int t = 0; t < T; ++t) o << (t ? ", " : "") << S.terms[t].zg << "ull";
  if (!T) o << "0ull";
  o << "};\n";
  const int nbuf = S.c64 ? 2 : 1;
  o << "extern \"C\" __global__ void __launch_bounds__(256, 2) qsb_ev_jit(const A* __restrict__ states, int n, "
       "unsigned long long smask, double* __restrict__ partial, int nterm_total, int nchunks) {\n";
  o << "  constexpr int SB = " << sbits << ", K = 12, TL = 4096, LOWQ = " << S.lowq << ", NT = " << T
    << ", NBUF = " << nbuf << ", TPC_MAX = 32;\n  constexpr bool REGACC = " << (S.regacc ? "true" : "false") << ";\n";
  o << R"(  extern __shared__ __align__(16) unsigned char smem_raw[];
  size_t off = 0;
  auto carve = [&](size_t bytes) { unsigned char* p = smem_raw + off; off = (off + bytes + 15) & ~(size_t)15; return p; };
  A* tiles = reinterpret_cast<A*>(carve(sizeof(A) * NBUF * TL));
  double* acc = reinterpret_cast<double*>(carve(sizeof(double) * (REGACC ? 0 : NT) * 256));
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * (TL >> LOWQ)));
  uint32_t* swz = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * (TL >> SB)));
  uint64_t* ibase = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * TPC_MAX));
  uint32_t* tword = reinterpret_cast<uint32_t*>(carve(sizeof(uint32_t) * 2));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t qmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t lowm = (1ull << LOWQ) - 1;
  const uint64_t shi = smask & ~lowm;
  for (int h = tid; h < (TL >> LOWQ); h += 256) hi_off[h] = qsb::pdep64((uint64_t)h, shi);
  const uint8_t* V = SB == 3 ? qsb::c_swz3 : qsb::c_swz4;
  for (int h = tid; h < (TL >> SB); h += 256) {
    uint32_t sw = 0;
    for (int p = SB, hh = h; hh; ++p, hh >>= 1)
      if (hh & 1) sw ^= V[p];
    swz[h] = sw;
  }
  const uint64_t outmask = ~smask & qmask;
  for (int i = tid; i < TPC_MAX; i += 256) ibase[i] = qsb::pdep64((uint64_t)i, outmask);
  for (int i = tid; i < (REGACC ? 0 : NT) * 256; i += 256) acc[i] = 0.0;
  __syncthreads();
)";
  if (S.regacc)
    for (int t = 0; t < T; ++t) o << "  double acc" << t << " = 0.0;\n";
  // per-thread parity word: bit t = parity(thread's tile bits of t's mapping & zl_t) = parity(tid & TM_t)
  o << "  const uint32_t pthread = 0u";
  for (const EvJitMap& m : S.maps)
    for (int t = m.t0; t < m.t0 + m.nt; ++t) {
      uint32_t tm = 0;
      for (int b = 0; b < 8; ++b)
        if (S.terms[t].zl >> m.tpos[b] & 1) tm |= 1u << b;
      if (tm) o << " | ((uint32_t)(__popc((uint32_t)tid & " << tm << "u) & 1) << " << t << ")";
    }
  o << ";\n";
  o << R"(  const int ntl = n - K;
  const int64_t ntiles = (int64_t)1 << ntl;
  const int64_t slot = blockIdx.x / nchunks, chunk = blockIdx.x % nchunks;
  const int64_t tpc = ntiles / nchunks, w0 = chunk * tpc;
  const A* st = states + (slot << n);
  const uint64_t Pt = ((uint64_t)tid & lowm) | hi_off[tid >> LOWQ];
  const uint32_t St = qsb::swz_slot<SB>(swz, (uint32_t)tid);
  const int hstep = 256 >> LOWQ;
  const uint64_t my_zg = lane < NT ? qsb_ev_zg[lane < NT ? lane : 0] : 0ull;
  const uint64_t base0 = qsb::pdep64((uint64_t)w0, outmask);
  auto load = [&](int64_t i, A* dst_tile) {
    const uint64_t base = base0 | ibase[i];
#pragma unroll
    for (int r = 0; r < TL / 256; ++r) {
      const A* src = st + (base | Pt | hi_off[r * hstep]);
      A* dst = dst_tile + (St ^ qsb::swz_slot<SB>(swz, (uint32_t)(r * 256)));
      if (sizeof(A) == 16) qsb::cp_async16(dst, src);
      else qsb::cp_async8(dst, src);
    }
    qsb::cp_async_commit();
  };
  load(0, tiles);
  for (int64_t i = 0; i < tpc; ++i) {
    if (NBUF == 2 && i + 1 < tpc) {
      load(i + 1, tiles + ((i + 1) & 1) * TL);
      qsb::cp_async_wait1();
    } else {
      qsb::cp_async_wait0();
    }
    if (warp == 0) {
      const uint64_t base = base0 | ibase[i];
      const uint32_t word = __ballot_sync(0xffffffffu, lane < NT && (__popcll(base & my_zg) & 1));
      if (lane == 0) tword[i & 1] = word;
    }
    __syncthreads();
    const A* tile = tiles + (NBUF == 2 ? (i & 1) * TL : 0);
    const uint32_t pw = pthread ^ tword[i & 1];
)";
  auto acc_line = [&](int t, const std::string& s) {
    if (S.regacc)
      o << "      acc" << t << " += sgnd((double)(" << s << "), (pw << " << (31 - t) << ") & 0x80000000u);\n";
    else
      o << "      acc[" << t << " * 256 + tid] += sgnd((double)(" << s << "), (pw << " << (31 - t) << ") & 0x80000000u);\n";
  };
  for (size_t mi = 0; mi < S.maps.size(); ++mi) {
    const EvJitMap& m = S.maps[mi];
    o << "    {  // mapping " << mi << "\n      const uint32_t tb = 0u";
    for (int b = 0; b < 8; ++b) o << " | ((((uint32_t)tid >> " << b << ") & 1u) << " << m.tpos[b] << ")";
    o << ";\n      const uint32_t sb = qsb::swz_slot<SB>(swz, tb);\n";
    for (int j = 0; j < 16; ++j) o << "      const A v" << j << " = tile[sb ^ " << m.soff[j] << "u];\n";
    // classes: runs of equal xr
    int t = m.t0;
    while (t < m.t0 + m.nt) {
      const uint32_t xr = S.terms[t].xr;
      int e = t;
      bool need_re = false, need_im = false;
      while (e < m.t0 + m.nt && S.terms[e].xr == xr) {
        if (S.terms[e].ny & 1) need_im = true;
        else need_re = true;
        ++e;
      }
      o << "      {  // class xr " << xr << "\n";
      if (xr == 0) {
        for (int j = 0; j < 16; ++j)
          o << "      const R q" << j << " = fma(v" << j << ".x, v" << j << ".x, v" << j << ".y * v" << j << ".y);\n";
        for (int tt = t; tt < e; ++tt) {
          // butterfly over the 4 register bits with the term's signs (zsig bit (1 << b))
          std::vector<std::string> x(16);
          for (int j = 0; j < 16; ++j) x[j] = "q" + std::to_string(j);
          for (int b = 0; b < 4; ++b) {
            const bool neg = S.terms[tt].zsig >> (1u << b) & 1;
            std::vector<std::string> y;
            for (size_t j = 0; j < x.size(); j += 2) y.push_back("(" + x[j] + (neg ? " - " : " + ") + x[j + 1] + ")");
            x.swap(y);
          }
          acc_line(tt, x[0]);
        }
      } else {
        const int top = 31 - __builtin_clz(xr);
        int bits[3], nb = 0;
        for (int b = 0; b < 4; ++b)
          if (b != top) bits[nb++] = b;
        for (int k = 0; k < 8; ++k) {
          const int j = ((k & 1) << bits[0]) | (((k >> 1) & 1) << bits[1]) | (((k >> 2) & 1) << bits[2]);
          const int jx = j ^ (int)xr;
          if (need_re)
            o << "      const R pr" << k << " = fma(v" << j << ".x, v" << jx << ".x, v" << j << ".y * v" << jx << ".y);\n";
          if (need_im)
            o << "      const R pi" << k << " = fma(v" << j << ".x, v" << jx << ".y, -v" << j << ".y * v" << jx << ".x);\n";
        }
        for (int tt = t; tt < e; ++tt) {
          const char* pre = (S.terms[tt].ny & 1) ? "pi" : "pr";
          std::vector<std::string> x(8);
          for (int k = 0; k < 8; ++k) x[k] = std::string(pre) + std::to_string(k);
          for (int lv = 0; lv < 3; ++lv) {
            const bool neg = S.terms[tt].zsig >> (1u << bits[lv]) & 1;
            std::vector<std::string> y;
            for (size_t j = 0; j < x.size(); j += 2) y.push_back("(" + x[j] + (neg ? " - " : " + ") + x[j + 1] + ")");
            x.swap(y);
          }
          acc_line(tt, x[0]);
        }
      }
      o << "      }\n";
      t = e;
    }
    o << "    }\n";
  }
  o << R"(    __syncthreads();
    if (NBUF == 1 && i + 1 < tpc) load(i + 1, tiles);
  }
)";
  if (S.regacc) {  // the register accumulators -> shared memory (the tile buffer is free now)
    o << "  double* red = reinterpret_cast<double*>(tiles);\n";
    for (int t = 0; t < T; ++t) o << "  red[" << t << " * 256 + tid] = acc" << t << ";\n";
    o << "  __syncthreads();\n  acc = red;\n";
  }
  o << "  const int outs[" << std::max(1, T) << "] = {";
  for (int t = 0; t < T; ++t) o << (t ? ", " : "") << S.terms[t].out;
  if (!T) o << "0";
  o << "};\n";
  o << R"(  for (int t = warp; t < NT; t += 8) {
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) s += acc[t * 256 + r * 32 + lane];
    for (int o2 = 16; o2; o2 >>= 1) s += __shfl_down_sync(0xffffffffu, s, o2);
    if (lane == 0) partial[(slot * nchunks + chunk) * nterm_total + outs[t]] = s;
  }
}
)";
  return o.str();
}

std::string ev_jit_build(const std::vector<std::string>& srcs, std::vector<JitKernel>& out) {
  out.assign(srcs.size(), JitKernel());
  if (!jit_available()) return "libnvrtc not available";
  const std::string dir = cache_dir();
  std::vector<JitJob> jobs(srcs.size());
  for (size_t i = 0; i < srcs.size(); ++i) {
    JitJob& j = jobs[i];
    j.pass = (int)i;
    j.src = srcs[i];
    std::string key = j.src;
    for (const char* opt : kOpts) key += opt;
    key += "nvrtc " + std::to_string(nvrtc().major) + "." + std::to_string(nvrtc().minor);
    char name[64];
    snprintf(name, sizeof(name), "/ev%016llx.cubin", (unsigned long long)fnv1a(key));
    j.path = dir + name;
    std::ifstream f(j.path, std::ios::binary);
    if (f) {
      j.cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
      j.ok = j.from_cache = !j.cubin.empty();
    }
  }
  std::atomic<size_t> next(0);
  unsigned nthreads = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  std::vector<std::thread> pool;
  for (unsigned w = 0; w < nthreads; ++w)
    pool.emplace_back([&] {
      for (size_t i = next++; i < jobs.size(); i = next++) {
        JitJob& j = jobs[i];
        if (j.ok) continue;
        j.ok = compile_one(j.src, j.cubin, j.log);
        if (j.ok) write_cache(j.path, j.cubin);
      }
    });
  for (auto& th : pool) th.join();
  std::string err;
  for (size_t i = 0; i < jobs.size(); ++i) {
    JitJob& j = jobs[i];
    if (!j.ok) {
      err = "NVRTC failed for reducer kernel: " + j.log.substr(0, 2000);
      continue;
    }
    cudaLibrary_t lib;
    if (cudaLibraryLoadData(&lib, j.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
      cudaGetLastError();
      unlink(j.path.c_str());
      err = "cudaLibraryLoadData failed for a reducer kernel";
      continue;
    }
    cudaKernel_t k;
    if (cudaLibraryGetKernel(&k, lib, "qsb_ev_jit") != cudaSuccess) {
      cudaGetLastError();
      cudaLibraryUnload(lib);
      err = "cudaLibraryGetKernel failed for a reducer kernel";
      continue;
    }
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    out[i].lib = (void*)lib;
    out[i].kern = (void*)k;
  }
  return err;
}

cudaError_t jit_launch(const JitKernel& jk, const StreamArgs& a, const PassDesc& pd, cudaStream_t s) {
  StreamArgs aa = a;
  PassDesc pp = pd;
  void* args[] = {(void*)&aa, (void*)&pp};
  const int64_t W = (int64_t)a.slots << (a.n - pd.k);
  dim3 grid((unsigned)std::min<int64_t>(W, jk.max_grid));
  dim3 block((unsigned)jk.threads);
  return cudaLaunchKernel((const void*)jk.kern, grid, block, args, jk.smem, s);
}

void jit_release(std::vector<JitKernel>& ks) {
  for (JitKernel& k : ks)
    if (k.lib) cudaLibraryUnload((cudaLibrary_t)k.lib);
  ks.clear();
}

}  // namespace qsb
