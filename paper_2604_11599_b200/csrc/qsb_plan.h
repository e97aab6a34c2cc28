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
void tile_mapping(const int* rpos, int rb, int k, int sb, int8_t* tpos, uint16_t* soff);

struct StreamPlan {
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
std::string build_stream_plan(const TapeInfo& t, int k, int lowq, int rb, int swz_bits, StreamPlan& out);

}  // namespace qsb
