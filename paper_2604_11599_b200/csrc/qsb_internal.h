// Internal types of the B200 state-vector backend (host + device).
//
// Layout in HBM:
//   state  : [slots][2^n] interleaved complex (double2 for c128, float2 for c64);
//            physical index p holds logical amplitude p ^ frame (lazy Pauli-X frame,
//            cleared bit-by-bit as fused passes cover the qubits).
//   ctl    : [slots] TrajCtl (RNG words, frame, pending collapse, guard stack, status)
//   bits   : [slots][nwords] packed classical store (ClassicalStore, sim.py:98-119)
//   guards : [slots][gwords] one bit per IF branch (then / else), snapshot at entry
//   partial: [slots][tiles][2^|M∩S|] per-tile marginal of the measured qubits
//   mats   : [slots or 1][nmat][8] 2x2 gate matrices (host-built for literal angles,
//            device-built from params for ParamRef angles)
#pragma once
#ifndef QSB_JIT  // the NVRTC prelude (gen_prelude.py) inlines these files without system headers
#include <cstdint>
#include <cstddef>

#include "../../include/qsb.h"
#endif

#ifdef __CUDACC__
#define QSB_HD __host__ __device__ __forceinline__
#else
#define QSB_HD inline
#endif

namespace qsb {

constexpr int kMaxQubits = 63;
constexpr int kMaxMeasureRegion = 10;  // |M| cap of one decide region (2^10 marginal bins)
constexpr int kMaxTile = 13;           // largest fused-pass tile (2^13 amplitudes)

// gate classes decided on the host from the base (never from matrix values)
enum GateClass : int32_t {
  GC_DENSE = 0,  // h sx rx ry u
  GC_DIAG = 1,   // z s t rz p            b0 = m00 a0, b1 = m11 a1
  GC_XPERM = 2,  // x                     exact swap
  GC_ANTI = 3,   // y                     b0 = m01 a1, b1 = m10 a0
  GC_SWAP = 4,   // swap                  exchange |..1..0..> and |..0..1..>
  GC_DIAG_GLOBAL = 5,  // (pass only) diagonal gate whose target is outside the tile
};

// compact op consumed by the device interpreters (resident kernel, decide kernel)
struct DevOp {
  int32_t kind;    // qsb_op_kind
  int32_t gclass;  // GateClass
  int32_t t0, t1;  // targets (swap: both)
  int32_t qubit;   // measure / reset
  int32_t bit;     // measure: flat classical bit
  uint64_t cm, cv; // controls
  int32_t mat;     // matrix index (GATE)
  int32_t guard;   // innermost enclosing guard id (-1 = none)
  int32_t g_then, g_else;  // IF: guard ids it defines
  int32_t pred_cmp, pred_bit, pred_width;
  int32_t op_index;        // position in the caller's tape (trace)
  int32_t diag_one0;       // GC_DIAG with m00 == 1 exactly (z s t p)
  uint64_t pred_rhs;
  // decide-kernel view (measure regions): positions inside M
  int32_t mj;              // M-index of qubit / target
  int32_t pad;
  uint64_t mcm, mcv;       // controls as M-index masks
};

// matrix source used by the device prep kernel (one per GATE op)
struct MatSrc {
  int32_t base, adjoint, has_matrix, pad;
  int32_t slot[3];
  int32_t pad2;
  double angle[3];
  double mat[8];
};

// one gate inside a fused pass (tile-local coordinates)
struct PassGate {
  int32_t gclass;
  int32_t lt, lt2;     // local target bit positions
  int32_t gq;          // GC_DIAG_GLOBAL: global qubit
  uint32_t lcm, lcv;   // controls inside the tile (local positions)
  uint64_t gcm, gcv;   // controls outside the tile (logical qubit masks)
  int32_t guard;       // guard id or -1
  int32_t mat;         // matrix index
  int32_t diag_one0;
  int32_t pad;
};

// Register-blocked execution of one pass (k_pass_reg): the tile lives in swizzled
// shared memory; a phase maps r "register" tile positions R onto each thread's 2^r
// registers and the other k - r positions onto the thread index, applies every gate
// of the phase in registers, and writes back.  Phases change R (a remap through
// shared memory) only when the next gate targets a position outside R.
constexpr int kMaxRegBits = 5;
enum PhaseKind : int32_t {
  PK_DENSE = 0,   // target jt in R (2x2 general)
  PK_XPERM = 1,   // x on jt in R
  PK_ANTI = 2,    // y on jt in R
  PK_DIAG_R = 3,  // diagonal, target jt in R
  PK_DIAG_T = 4,  // diagonal, target tile position tp outside R (per-thread factor)
  PK_DIAG_G = 5,  // diagonal, target outside the tile (per-CTA factor)
  PK_SWAP_R = 6,  // swap of jt, jt2 both in R
  // assigned on the device when the gate is staged, from the matrix values:
  PK_DENSE_REAL = 7,  // all entries real (h, ry): 8 FMA per pair instead of 16
  PK_DENSE_RX = 8,    // real diagonal, imaginary off-diagonal (rx): 8 FMA per pair
  PK_SKIP = 9,        // guard off or out-of-tile control unsatisfied for this CTA
};
constexpr int kMaxPassGates = 256;  // gates staged in shared memory per pass

struct PhaseGate {
  int32_t kind;
  int32_t jt, jt2;     // register-index bits of the targets
  int32_t tp;          // PK_DIAG_T: tile position; PK_DIAG_G: global qubit
  uint32_t cmR, cvR;   // controls on register bits (j space)
  uint32_t cmT, cvT;   // controls on thread-mapped tile positions (checked on the thread base)
  uint64_t gcm, gcv;   // controls outside the tile (logical qubit masks)
  int32_t guard, mat;
  int32_t diag_one0, pad;
};

struct PhaseDesc {
  int32_t gate_begin, gate_count;
  int32_t nt;                      // thread bits (k - r)
  int32_t pad;
  int8_t tpos[16];                 // thread bit i -> tile position
  uint16_t soff[1 << kMaxRegBits]; // swizzled tile slot of register j (XOR with the thread base slot)
};

struct PassDesc {
  int32_t phase_begin, phase_count;  // register-blocked phases (k_pass_reg); 0 = shared-memory kernel
  int32_t pgate_begin, pgate_count;  // the phases' gates (contiguous in StreamPlan::phase_gates)
  uint64_t smask;       // tile qubits S (always includes the low `lowq` qubits)
  uint64_t clear_before;// frame bits cleared by earlier passes since the last decide
  uint64_t mmask;       // measured qubits of the next region (epilogue marginal)
  int32_t k;            // |S|
  int32_t lowq;         // qubits 0..lowq-1 are the contiguous low part of S
  int32_t sq[kMaxTile]; // local bit j -> qubit
  int32_t gate_begin, gate_count;
  int32_t prologue;     // apply the pending collapse of the previous decide
  int32_t init_zero;    // input is |0...0> (first pass): no read
  int32_t epi;          // compute the marginal of mmask in the epilogue
  int32_t m_local;      // |M ∩ S|
  int32_t mloc[kMaxMeasureRegion];   // local positions of M∩S, in M order
  int32_t region;       // decide region fed by the epilogue
  int32_t rb;           // register bits of the phases (0: no phases, shared-memory kernel)
  // tile-id bits of qubits still in |0> (no non-diagonal gate on them since the |0...0>
  // start; set by the host per run): every item with one of them set is zero before and
  // after the pass and its buffer already holds zeros -- only the others run
  uint64_t zero_tid;
  // 1: the known bits of zero_tid are the slot's projection values (after a measurement:
  // the items the collapse rejects are zero but not stored), 0: they are 0 (|0...0> start)
  int32_t zero_from_vp;
  int32_t pad_z;
  // qubits whose amplitudes the last collapse rejected (p & zk_mask != kval & zk_mask) and
  // that no pass has stored since: the gather makes those amplitudes zero instead of
  // reading them (the buffer still holds stale values there)
  uint64_t zk_mask;
};

struct RegionDesc {
  int32_t op_begin, op_end;  // control ops (DevOp list of the plan) executed in order
  int32_t mcount;            // |M|
  int32_t has_marginal;
  int32_t mq[kMaxMeasureRegion];  // M qubits; bin bit j <-> qubit mq[j]
  uint64_t mmask;
  uint64_t clear_mask;       // frame bits cleared by the passes since the previous decide
  int32_t m_local;           // |M ∩ S_epi|
  int32_t mloc_bit[kMaxMeasureRegion];   // for each j: local bin bit, or -1 if mq[j] is outside S
  int32_t mtile_bit[kMaxMeasureRegion];  // for each j outside S: bit of the tile id, else -1
  int32_t desc_gates;        // descriptor gates in this region (gate-update accounting)
  uint64_t epi_smask;        // S of the epilogue pass
};

// per-trajectory control block
struct TrajCtl {
  uint64_t rng[4];
  uint64_t frame;        // physical = logical ^ frame
  uint64_t kmask, kval;  // pending projection on PHYSICAL indices: keep iff (p & kmask) == kval
  double sre, sim;       // pending complex scale
  int32_t pending;       // projection / scale not yet applied
  int32_t status;        // qsb_status of this trajectory
  int32_t depth, active; // guard stack (counter form: active iff active == depth)
  int32_t draws;         // uniforms consumed (pre-drawn streams)
  int32_t pad;
  int64_t gates;         // executed Gate ops (logical gate updates)
  uint64_t hist;         // hash of the executed measure / reset outcomes so far
  int32_t rep;           // slot whose state buffer holds this trajectory's state (history dedup)
  int32_t pad2;
};

// classical control of one sliced trajectory (qsb_slice_*): everything a measurement,
// reset or if/else decides lives here, in device memory -- the host only enqueues
constexpr int kSliceWords = 16;  // classical bits of a sliced run: <= 1024
struct SliceCtl {
  uint64_t rng[4];
  int32_t status;      // qsb_status (QSB_ERR_DEGENERATE once a branch had p < 1e-15)
  int32_t depth, active;  // guard stack (counter form: active iff active == depth)
  int32_t draws;       // uniforms consumed
  int32_t outcome;     // last decision; -1: the measure / reset sat in an inactive branch
  int32_t nwords;
  double scale;        // 1 / sqrt(p_out) of the last decision
  double p1;           // p1 of the last decision (sum of the per-slice partials, slice order)
  uint64_t bits[kSliceWords];
};

// kernel arguments of the streaming engine (passed by value)
struct StreamArgs {
  void* state;
  int32_t n;
  int32_t c64;
  const PassGate* gates;
  const PhaseDesc* phases;
  const PhaseGate* phase_gates;
  const double* mats;
  int64_t mat_stride;
  TrajCtl* ctl;
  uint64_t* bits;
  int32_t nwords;
  int32_t gwords;
  uint32_t* guards;
  double* partial;
  int64_t partial_stride;   // doubles per slot
  int64_t slots;
  // decide
  const DevOp* region_ops;
  const double* predrawn;
  int32_t predrawn_stride;
  int32_t ntiles_log2;
  int64_t predrawn_slot0;   // global slot index of slot 0 (row of predrawn)
  unsigned long long* tie_count;
  int64_t* trace_out;
  int32_t max_trace;
  int32_t* ntrace_out;
  // branch-history deduplication: passes run only the representative slots listed in
  // active[0 .. *nactive) (null: every slot)
  const int32_t* active;
  const int32_t* nactive;
  // per slot: the slot whose buffer its gather reads (< 0 or null: its own)
  const int32_t* read_src;
  // ... whose keys are verified on the exact outcome history: bit d of slot s's row is
  // the outcome of its d-th draw (null: no dedup)
  uint64_t* hbits;
  int32_t hwords;
  int32_t pad_h;
};

QSB_HD uint64_t insert_zero(uint64_t v, int pos) {
  uint64_t lo = v & ((1ull << pos) - 1);
  return ((v >> pos) << (pos + 1)) | lo;
}

QSB_HD uint64_t pdep64(uint64_t v, uint64_t mask) {
  uint64_t out = 0;
  for (uint64_t m = mask; m; m &= m - 1) {
    uint64_t low = m & (~m + 1);
    if (v & 1) out |= low;
    v >>= 1;
  }
  return out;
}

// RNG: splitmix64-seeded xoshiro256++ (sim.py:26-72)
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
QSB_HD uint64_t splitmix_next(uint64_t& x) {
  x += kGolden;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
QSB_HD void rng_seed(uint64_t* s, uint64_t seed) {
  uint64_t x = seed;
  s[0] = splitmix_next(x);
  s[1] = splitmix_next(x);
  s[2] = splitmix_next(x);
  s[3] = splitmix_next(x);
}
// RngStream.for_shot(seed, shot) (sim.py:54-57)
QSB_HD void rng_for_shot(uint64_t* s, uint64_t seed, uint64_t shot) {
  uint64_t x = seed + (shot + 1ull) * kGolden;
  uint64_t derived = splitmix_next(x);
  rng_seed(s, derived);
}
QSB_HD uint64_t rotl64(uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }
QSB_HD uint64_t rng_next(uint64_t* s) {
  uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}
QSB_HD double rng_uniform(uint64_t* s) { return (double)(rng_next(s) >> 11) * 0x1.0p-53; }

// Predicate (sim.py:262-276): value is the MSB-first unsigned of `width` bits
QSB_HD bool pred_eval(const uint64_t* bits, int first, int width, int cmp, uint64_t rhs) {
  uint64_t v = 0;
  for (int j = 0; j < width; ++j) {
    int f = first + j;
    v = (v << 1) | ((bits[f >> 6] >> (f & 63)) & 1ull);
  }
  switch (cmp) {
    case QSB_CMP_EQ: return v == rhs;
    case QSB_CMP_NE: return v != rhs;
    case QSB_CMP_LT: return v < rhs;
    case QSB_CMP_LE: return v <= rhs;
    case QSB_CMP_GT: return v > rhs;
    case QSB_CMP_GE: return v >= rhs;
    default: return v != 0;  // truthy
  }
}

}  // namespace qsb
