// Host-callable launchers for the sm_100a kernels (precision-dispatched).
#pragma once
#include <cuda_runtime.h>

#include "qsb_internal.h"

namespace qsb {

constexpr int kResMaxWords = 16;  // classical words kept in shared memory by the resident engine

// ---- single-state kernels (qsb_state.cu) -----------------------------------
void launch_init_zero(int c64, void* amps, int n, int64_t slots, cudaStream_t s);
void launch_apply_1q(int c64, void* amps, int n, int t, uint64_t cm, uint64_t cv, int gclass,
                     const double* m8, cudaStream_t s);
void launch_apply_swap(int c64, void* amps, int n, int t0, int t1, uint64_t cm, uint64_t cv, cudaStream_t s);
// deterministic sum of |a|^2 over indices with bit q == 1 (q < 0: all indices) -> *out_dev
void launch_prob(int c64, const void* amps, int n, int q, double* scratch, double* out_dev, cudaStream_t s);
int prob_scratch_len(int n);
void launch_collapse(int c64, void* amps, int n, int q, int outcome, double scale, int flip, cudaStream_t s);
void launch_c128_to_c64(const double* in, float* out, int64_t count, cudaStream_t s);
void launch_c64_to_c128(const float* in, double* out, int64_t count, cudaStream_t s);

// Pauli expectation over `slots` states: one launch per X-mask group of <= 8 terms.
struct PauliGroup {
  uint64_t xmask;
  int32_t nterm;
  int32_t term0;          // first output term index
  uint64_t zy[8];         // Z|Y masks
  int32_t ny[8];
};
int expval_blocks(int n);
void launch_expval_group(int c64, const void* amps, int n, int64_t slots, const PauliGroup& g,
                         double* partial /*[slots][nterm_total][blocks]*/, int nterm_total, cudaStream_t s);
void launch_expval_finish(const double* partial, int64_t slots, int nterm_total, int blocks,
                          const uint64_t* xmask, const int32_t* ny, double* out /*[slots][nterm]*/, cudaStream_t s);

// tile-fused Pauli reducer (qsb_expval.cu)
struct ExpvalTerm {
  uint32_t xl, zl;  // X|Y and Z|Y letters inside the tile (tile positions)
  uint64_t xg, zg;  // outside the tile (qubit masks; xg must be 0 for the tile path)
  int32_t ny, out;  // #Y, output index
  uint32_t xr;      // register path: X|Y letters in register-bit space of the term's mapping
  uint32_t zsig;    // register path: bit j = parity(tile positions of register j & zl)
  int32_t path;     // 0: per-thread accumulating kernel (partials [slot][chunk][term]);
                    // 1: pair-loop kernel (partials [slot][tile][term])
  int32_t pad;
};
// register mapping of a tile group (k = 12): register bit b <-> tile position rpos[b];
// the terms [term_begin, term_begin + nterm) of the group are evaluated with it
struct EvMap {
  int8_t tpos[16];    // thread bit i -> tile position (k - 4 entries)
  uint16_t soff[16];  // swizzled slot offset of register j
  int32_t term_begin, nterm;
};
struct ExpvalGroup {
  uint64_t smask;   // tile qubits
  int32_t k, lowq, term_begin, nterm;
  int32_t map_begin, nmap;  // register mappings of the accumulating kernel (k == 12)
  int32_t cls_begin, ncls;  // its classes (EvClass)
};
// a class of the accumulating kernel: a run of terms with equal register X pattern in one
// mapping (launch-relative indices), Re terms [t0, im0) before Im terms [im0, t1)
struct EvClass {
  int16_t map, xr, t0, im0, t1, pad;
};
void launch_expval_tile(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                        const ExpvalTerm* terms, const EvMap* maps,
                        double* partial /*[slots][tiles][nterm_total]*/, int nterm_total, cudaStream_t s);
void launch_expval_tile_finish(const double* partial_acc, int nchunks, const double* partial_tile, int ntiles,
                               int64_t slots, int nterm, const ExpvalTerm* terms_by_out, double* out, cudaStream_t s);
// per-thread accumulating Pauli reducer (k = 12 register mappings, <= kEvAccTerms terms per
// launch): partials [slot][chunk][nterm_total], chunks = expval_acc_chunks(n)
constexpr int kEvAccTerms = 16;
int expval_acc_chunks(int n);
void launch_expval_acc(int c64, const void* states, int n, int64_t slots, const ExpvalGroup& g,
                       const ExpvalTerm* terms, const EvMap* maps, const EvClass* classes, double* partial,
                       int nterm_total, cudaStream_t s);

// device-side shot histogram (qsb_hist.cu): sort the per-shot words on their low
// `nbits` bits and run-length encode -> ascending distinct words + counts
size_t hist_scratch_bytes(size_t n);
cudaError_t launch_histogram(const uint64_t* words, uint64_t* sorted, size_t n, int nbits, uint64_t* uniq,
                             int32_t* counts, int32_t* nruns, void* scratch, size_t scratch_bytes, cudaStream_t s);

// static sampling
// static sampling (sim.py:354-369), bit-exact: one sequential pass keeps the running sum
// at the end of every block (cdf_blocks(n) doubles); each shot searches the blocks and
// re-runs its block's left-to-right additions
int64_t cdf_blocks(int n);
void launch_cumsum_seq(int c64, const void* amps, int n, double* ends, cudaStream_t s);
void launch_static_search(int c64, const void* amps, const double* ends, int n, uint64_t seed, int64_t shot_begin,
                          int64_t count, const int32_t* mq, const int32_t* mb, int nmeas, int nwords, uint64_t* bits,
                          cudaStream_t s);

// ---- resident engine (qsb_resident.cu) -------------------------------------
struct ResidentArgs {
  const DevOp* ops;
  int32_t nops;
  int32_t n;
  int32_t nwords;
  int32_t predrawn_stride;
  const double* mats;
  int64_t mat_stride;     // doubles between slots' matrix tables (0 = shared)
  uint64_t seed;
  int64_t shot_begin;
  int64_t count;
  const double* predrawn; // [count][predrawn_stride] or null
  uint64_t* bits_out;     // [count][nwords]
  int32_t* status_out;    // [count]
  void* state_out;        // final state of slot 0 (or null)
  int64_t* trace_out;     // slot 0 trace (or null)
  int32_t max_trace;
  int32_t* ntrace_out;
  unsigned long long* tie_count;
  unsigned long long* gate_count;
  const uint64_t* rng_init;  // slot 0 starts from these words (or null: for_shot)
  uint64_t* rng_final;       // slot 0 RNG words after the run (or null)
  int32_t* draws_out;        // slot 0 uniforms consumed (or null)
  int32_t c64;
};
int resident_max_qubits(int c64);
cudaError_t launch_resident(const ResidentArgs& a, int num_sms, cudaStream_t s);

// ---- streaming engine (qsb_stream.cu) --------------------------------------
void launch_mats_prep(const MatSrc* src, int nmat, const double* params, int nparams, int64_t slots,
                      double* mats_out, cudaStream_t s);
void launch_ctl_init(TrajCtl* ctl, uint64_t* bits, int nwords, uint32_t* guards, int gwords, int64_t slots,
                     uint64_t seed, int64_t shot_begin, const uint64_t* rng_init, int dedup, cudaStream_t s);
// history dedup bookkeeping: regroup + copy (after a decide) or initial grouping, then
// the representative list the passes iterate.  split != null (regroup before a pass):
// no copies -- the new branches and the other representatives are listed apart
// (k_dedup_commit) and the next pass runs as two launches, the branches first, reading
// their old representatives' buffers (StreamArgs::read_src = copy_src)
void launch_dedup(const StreamArgs& a, int32_t* new_rep, int32_t* copy_src, int32_t* active, int32_t* nactive,
                  int c64, bool regroup, int32_t* split, cudaStream_t s);
// store the zeros of the amplitudes the pending collapse rejects on the qubits M (known-zero
// amplitudes no pass has stored: end of a run, or before a pass that reads everything)
void launch_zero_projected(const StreamArgs& a, int c64, uint64_t M, cudaStream_t s);
// zero the states (+ epilogue partials) of the active slots before a tile-0-only init pass
void launch_zero_slots(const StreamArgs& a, int c64, int zero_partials, cudaStream_t s);
// physical pass work under dedup: phys[0] += bytes_per_state * nactive, phys[1] += flops * nactive
void launch_accum_physical(const int32_t* nactive, double flops_per_state, double bytes_per_state, double* phys,
                           cudaStream_t s);

cudaError_t launch_pass(const StreamArgs& a, const PassDesc& pd, cudaStream_t s);
// register-blocked variant (qsb_pass_reg.cu), used when the pass has phases
cudaError_t launch_pass_reg(const StreamArgs& a, const PassDesc& pd, cudaStream_t s);
cudaError_t launch_decide(const StreamArgs& a, const RegionDesc& rd, cudaStream_t s);
void launch_count_gates(const StreamArgs& a, const int32_t* guard_gates, int nguards, int64_t unguarded,
                        unsigned long long* out, cudaStream_t s);
// out[i] = collapse(state[i ^ frame]) for slot 0; `clear` = frame bits already cleared by
// passes after the last decide, `consumed` = a pass already applied the pending collapse
void launch_finalize(const StreamArgs& a, void* out, uint64_t clear, int consumed, cudaStream_t s, int64_t slot = 0);

// ---- global-qubit-sliced engine (qsb_slice.cu) ---------------------------------------
void launch_slice_init(SliceCtl* c, uint64_t seed, int64_t shot, const uint64_t* rng_init, int nwords,
                       cudaStream_t s);
void launch_slice_guard(SliceCtl* c, int kind, int pred_bit, int pred_width, int pred_cmp, uint64_t rhs,
                        cudaStream_t s);
void launch_slice_gate(int c64, void* amps, int n, int t, uint64_t cm, uint64_t cv, int gc, const double* m,
                       const SliceCtl* ctl, cudaStream_t s);
void launch_slice_scale(int c64, void* amps, int n, double re, double im, const SliceCtl* ctl, cudaStream_t s);
void launch_slice_put(const double* blocks, int nblocks, int select, double* partials, int index, cudaStream_t s);
void launch_slice_decide(SliceCtl* c, const double* partials, int nslices, int kind, int bit, cudaStream_t s);
void launch_slice_collapse(int c64, void* amps, int n, int q, int gbit, int flip, const SliceCtl* ctl,
                           cudaStream_t s);
void launch_slice_remap_local(int c64, void* const* group, int n, int k, const int* lpos, cudaStream_t s);
void launch_slice_pack_sub(int c64, const void* amps, int k, const int* lpos, int x, int64_t first, int64_t count,
                           void* out, cudaStream_t s);
void launch_slice_unpack_sub(int c64, void* amps, int k, const int* lpos, int x, int64_t first, int64_t count,
                             const void* in, cudaStream_t s);
void launch_slice_exchange_local(int c64, void* a, void* b, int n, int pos, cudaStream_t s);
void launch_slice_pack(int c64, const void* amps, int pos, int c, int64_t first, int64_t count, void* out,
                       cudaStream_t s);
void launch_slice_unpack(int c64, void* amps, int pos, int c, int64_t first, int64_t count, const void* in,
                         cudaStream_t s);
// per-block partial sums of |a|^2 over the amplitudes with bit q set (q < 0: all); the
// block count is prob_blocks_for(n, q)
void launch_prob_blocks(int c64, const void* amps, int n, int q, double* blocks, cudaStream_t s);
int prob_blocks_for(int n, int q);

}  // namespace qsb
