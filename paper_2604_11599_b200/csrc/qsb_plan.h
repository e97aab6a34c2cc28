// Host-side tape analysis and the fused-pass planner.
#pragma once
#include <string>
#include <vector>

#include "qsb_internal.h"

namespace qsb {

struct TapeInfo {
  int n = 0, nbits = 0, nwords = 1, nparams = 0, nguards = 0, gwords = 1;
  bool needs_trajectories = false;  // sim.py:322-335
  bool top_level_dynamic = false;   // sim.py:394-399 (statevector refuses)
  bool has_param_angles = false;
  int draws_max = 0;                // upper bound on uniforms consumed by one shot
  std::vector<DevOp> dev;           // flattened program (all ops, program order)
  std::vector<MatSrc> mats;         // one per GATE op (DevOp.mat)
  std::vector<int> top_measures;    // dev indices of top-level MEASURE ops (static sampling)
};

// Validates caller ops and builds the flattened device program.  Returns an error
// message (empty on success).
std::string analyze_tape(const qsb_op* ops, int nops, int n, int nbits, int nparams, TapeInfo& out);

struct Step {
  int type;   // 0 = pass, 1 = decide
  int index;
};

// shared-memory swizzle of the register-blocked pass kernel: slot(l) = l ^ V(l >> sb),
// V linear; `sb` = 3 for 16-byte amplitudes, 4 for 8-byte ones.
int swizzle_bits(int c64);
uint32_t swizzle_hi(uint32_t hi, int sb);  // V applied to tile bits >= sb (hi = l >> sb)
// register / thread mapping of a swizzled k-position tile: register bit b <-> tile
// position rpos[b] (b < rb); writes the k - rb thread positions and the swizzled slot
// offset of each of the 2^rb registers
void tile_mapping(const int* rpos, int rb, int k, int sb, int8_t* tpos, uint16_t* soff, uint32_t avoid = 0);

// Engine options of the planner and the NVRTC generator, set per context
// (qsb_ctx_set_option); the defaults are the settings measured best on B200 (DESIGN.md
// §7b).  Part of the plan cache key.
struct EngineOptions {
  int pair_aware = 1;         // phase register sets follow two-qubit partners
  int phase_search = 1;       // per-phase register-set search (round 2: measured faster on every config)
  int block_condx = 0;        // a conditional X ends its target's use in a phase
  int inline_phases = -1;     // phases inlined into the pass kernel (-1: complex128 yes, complex64 no)
  int inline_min_gates = 0;   // ... only for passes with at least this many gates
  int inline_max_phases = 8;  // ... and at most this many phases (0: no limit; VQE24 +2 %, DYN20 / RDC30 neutral)
  int ffma2 = 1;              // complex64 fused blocks as packed fma.rn.f32x2
  int packed_gates = 0;       // complex64 single-gate helpers packed too (bit-identical)
  int last_direct = 1;        // last phase stores to HBM: 0 off, 1 unstaged passes, 2 also staged
  int last_direct_maxlow = 0; // ... with at most this many low tile positions in registers
  int minblocks = 2;          // CTAs per SM the register budget of a pass kernel targets
  int edge_x = 1;             // conditional X gates at a phase edge as slot-base XORs
  int ctas_per_sm = 0;        // cap of the persistent pass grid per SM (0: occupancy)
  int defer_gates = 0;        // gates commuting with a measurement region run after it (measured slower: off)
  int zero_aware = 2;         // after a measurement, the first (1) or first two (2) passes may avoid the projected qubits
  int zero_cost = 2;          // their cost model: 0 = 1 per full pass; gate-weighted 1 = everywhere, 2 = prefix searches, 3 = zero_aware only
  int zero_width = 4;         // first-pass candidates tried (and width / 2 per later avoiding pass)
  int zero_depth = 3;         // ... prefixes of up to zero_depth passes
  int zero_step = 1;          // after a measurement: also prefixes taking in <= zero_step projected qubits per pass
  int init_aware = 2;         // the region at the |0...0> start: prefixes of up to init_aware + 1 passes by known-zero cost
  uint64_t key() const {
    const int v[] = {pair_aware, phase_search, block_condx, inline_phases, inline_min_gates, ffma2, packed_gates,
                     last_direct, last_direct_maxlow, minblocks, edge_x, ctas_per_sm, defer_gates, inline_max_phases,
                     zero_aware, zero_cost, zero_width, init_aware, zero_step, zero_depth};
    uint64_t h = 1469598103934665603ull;
    for (int x : v) h = (h ^ (uint64_t)(uint32_t)x) * 1099511628211ull;
    return h;
  }
  // set a named option; false if `key` is not an engine option
  bool set(const std::string& key, int64_t value);
};

struct StreamPlan {
  EngineOptions opt;  // the options the plan (and its NVRTC kernels) were built with
  int k = 0, lowq = 0, ntiles_log2 = 0, rb = 0;
  std::vector<PassDesc> passes;
  std::vector<PassGate> gates;
  std::vector<PhaseDesc> phases;
  std::vector<PhaseGate> phase_gates;
  std::vector<RegionDesc> regions;
  std::vector<DevOp> region_ops;
  std::vector<Step> steps;
  int max_local_bins = 1;           // max 2^|M∩S| over epilogue passes
  std::vector<int32_t> guard_gates; // pass gates guarded directly by each guard id
  int64_t unguarded_gates = 0;
  int64_t descriptor_gates = 0;     // gates folded into decide regions
};

// Dense-matrix structure known before execution (literal matrices by value, ParamRef
// angles by base): shared by the JIT code generator and the FLOP accounting.
enum DenseVariant { DV_GEN, DV_REAL, DV_RX };
DenseVariant dense_variant(const MatSrc& m);
uint32_t zero_mask(const MatSrc& m);  // bit i: component m[i] is exactly zero
// floating-point operations (FMA = 2) the specialised kernels spend per affected pair
double phase_gate_flops(const PhaseGate& q, const MatSrc& m);
// flops per state of one pass (sum over its gates and affected pairs)
double pass_flops(const TapeInfo& t, const StreamPlan& P, int pass);

// rb = register bits of k_pass_reg (4 for complex128, 5 for complex64); phases are
// built when k - rb >= 5 (at least one warp per tile), else the shared-memory kernel runs.
std::string build_stream_plan(const TapeInfo& t, int k, int lowq, int rb, int swz_bits, StreamPlan& out,
                              const EngineOptions& opt = EngineOptions());

}  // namespace qsb

namespace qsb {

// ---------------------------------------------------------------------------
// Gate fusion inside a register phase (NVRTC kernels).  Literal, unguarded gates on
// register bits are collected into 1- and 2-qubit blocks (commutation on disjoint
// qubits); a block whose product matrix costs fewer FP operations per amplitude than
// its gates applied one by one is emitted as one dense 2x2 / 4x4 (e.g. the four `u`
// gates around a cx of a brick layer: 4 x 24 x 2 flops per 4 amplitudes -> 120).
// ---------------------------------------------------------------------------
struct FuseItem {
  int gate = -1;         // >= 0: emit phase gate P.phase_gates[gate] unchanged
  int qa = -1, qb = -1;  // fused block: register bits of matrix index bit 0 / bit 1 (qb = -1: 2x2)
  int ngates = 0;        // gates folded into the block
  double m[32];          // row-major complex entries (re, im); a 2x2 uses m[0..7]
};
// items of phase `phase` (index into P.phases) in emission order; `enable` = false
// returns the gates one by one.  Every fused phase is checked on the host against its
// gates on random register vectors; a mismatch falls back to the unfused list.
std::vector<FuseItem> fuse_phase(const TapeInfo& t, const StreamPlan& P, int phase, bool enable);
// flops of one fused block per group of 2 (2x2) or 4 (4x4) amplitudes, zero components dropped
double fuse_block_flops(const FuseItem& f);
// pass_flops with the fused blocks of the NVRTC kernels
double pass_flops_fused(const TapeInfo& t, const StreamPlan& P, int pass);
// number of fused phases whose host check failed (diagnostics; should stay 0)
int fuse_check_failures();

}  // namespace qsb
