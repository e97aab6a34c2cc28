/*
 * qsb.h -- C ABI of the B200-native state-vector backend ("qsb": qasm state-vector
 * backend) that replaces the CPU simulator target of qasm2cudaq.
 *
 * The reference has no native interface: its simulator target is the module-level
 * Python API of /root/reference/pkg/src/qasm2cudaq/sim.py.  Each entry point below
 * names the reference function it replaces (file:line).  The Python host mirror
 * (paper_2604_11599_b200/sim.py) binds these with ctypes; INTEGRATION.md shows the
 * binding a maintainer adds on the reference side.
 *
 * Conventions
 *  - plain C, no exceptions cross the ABI; every call returns a qsb_status and
 *    qsb_last_error() returns a thread-local message for the last failure.
 *  - amplitudes cross the ABI as interleaved complex128 (re, im) in HOST memory,
 *    little-endian qubit order: qubit k = bit k of the index (sim.py:3).
 *  - classical bits cross as packed uint64 words: flat bit f (registers in
 *    declaration order, bit 0 of each register first -- exactly the character
 *    order of ClassicalStore.key(), sim.py:118-119) is bit (f & 63) of word f >> 6.
 *  - one host thread per context; a context owns one device and one CUDA stream.
 *    The caller owns every host buffer; the context owns device memory.
 */
#ifndef QSB_H
#define QSB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB_ABI_VERSION 1

typedef enum {
  QSB_OK = 0,
  QSB_ERR_SIM = 1,          /* errors.SimError (e.g. shots < 1, sim.py:375-376)          */
  QSB_ERR_DYNAMIC = 2,      /* errors.DynamicCircuit (sim.py:394-399)                    */
  QSB_ERR_DEGENERATE = 3,   /* errors.DegenerateNorm (sim.py:243-246)                    */
  QSB_ERR_BAD_PAULI = 4,    /* errors.BadPauliString (sim.py:422-425)                    */
  QSB_ERR_DIMENSION = 5,    /* errors.DimensionMismatch                                  */
  QSB_ERR_OOM = 6,          /* device allocation failed                                  */
  QSB_ERR_CUDA = 7,         /* CUDA runtime / launch failure                             */
  QSB_ERR_ARG = 8,          /* malformed argument / tape                                 */
  QSB_ERR_UNSUPPORTED = 9,  /* outside this build's limits (e.g. > 64 qubits)            */
  QSB_ERR_PREDRAWN = 10     /* pre-drawn uniform stream exhausted                        */
} qsb_status;

typedef enum { QSB_C128 = 0, QSB_C64 = 1 } qsb_precision;

/* ---- kernel-IR tape (kir.py:41-106 flattened; CondBlock -> IF/ELSE/ENDIF) ---- */
typedef enum {
  QSB_OP_GATE = 0,
  QSB_OP_MEASURE = 1,
  QSB_OP_RESET = 2,
  QSB_OP_IF = 3,     /* evaluate predicate once at entry (sim.py:297), open then-branch */
  QSB_OP_ELSE = 4,   /* switch to the else-branch of the innermost IF                   */
  QSB_OP_ENDIF = 5
} qsb_op_kind;

/* canonical bases, kir.py:18 */
typedef enum {
  QSB_G_X = 0, QSB_G_Y, QSB_G_Z, QSB_G_H, QSB_G_S, QSB_G_T, QSB_G_SX,
  QSB_G_RX, QSB_G_RY, QSB_G_RZ, QSB_G_P, QSB_G_U, QSB_G_SWAP
} qsb_gate_base;

/* Predicate.comparator, kir.py:66-71 */
typedef enum {
  QSB_CMP_EQ = 0, QSB_CMP_NE, QSB_CMP_LT, QSB_CMP_LE, QSB_CMP_GT, QSB_CMP_GE, QSB_CMP_TRUTHY
} qsb_cmp;

typedef struct {
  int32_t kind;          /* qsb_op_kind                                                  */
  int32_t base;          /* qsb_gate_base (GATE)                                         */
  int32_t adjoint;       /* conjugate transpose (sim.py:198-199)                         */
  int32_t ntargets;      /* 1, or 2 for swap; targets[0] is the matrix high bit          */
  int32_t target[2];
  int32_t qubit;         /* MEASURE / RESET                                              */
  int32_t bit;           /* MEASURE: flat classical bit                                  */
  uint64_t ctrl_mask;    /* control qubits                                               */
  uint64_t ctrl_val;     /* required value per control (POS = 1, NEG = 0)                */
  int32_t angle_slot[3]; /* ParamRef slot, or -1 for a literal in angle[]                */
  int32_t has_matrix;    /* 1: mat[] holds the host-built matrix (literal angles)        */
  double angle[3];
  double mat[8];         /* 2x2 row-major, (re, im) pairs: m00 m01 m10 m11               */
  int32_t pred_cmp;      /* IF: qsb_cmp                                                  */
  int32_t pred_bit;      /* IF: first flat bit of the compared value                     */
  int32_t pred_width;    /* IF: bits compared, MSB-first (1 for a single bit)            */
  int32_t reserved;
  uint64_t pred_rhs;     /* IF: unsigned right-hand side                                 */
} qsb_op;

typedef struct qsb_ctx_s* qsb_ctx;
typedef struct qsb_state_s* qsb_state;
typedef struct qsb_tape_s* qsb_tape;
typedef struct qsb_slicectl_s* qsb_slicectl;  /* classical control of one sliced trajectory */
typedef struct qsb_comm_s* qsb_comm;          /* NCCL communicator of the sliced engine     */

typedef struct {
  int64_t kernel_launches;   /* device kernels launched by the last run                   */
  int64_t passes;            /* fused state passes launched                               */
  int64_t decides;           /* measurement-region decide launches                        */
  double pass_ms;            /* CUDA-event time of all pass kernels of the last run       */
  double total_ms;           /* CUDA-event time of the last run (device side)             */
  double pass_bytes;         /* algorithmic bytes moved by pass kernels (2 * 2^n * S per state pass) */
  int64_t gate_updates;      /* logical executed Gate ops summed over trajectories        */
  int64_t tie_band;          /* measure decisions with |u - p1| < 1e-12 (c128) / 1e-6 (c64) */
  int32_t engine;            /* 0 resident (state on chip), 1 streaming (state in HBM)    */
  int32_t tile_qubits;       /* k of the fused passes                                     */
  int32_t jit_passes;        /* passes run by NVRTC-specialised kernels                   */
  int32_t jit_compiled;      /* of those, compiled (not loaded from the cache) for this tape */
  double jit_compile_ms;     /* one-time specialisation cost of the tape's plan           */
  double pass_flops;         /* floating-point operations (FMA = 2) of the pass kernels   */
} qsb_stats;

#ifndef QSB_JIT /* the NVRTC prelude of the specialised kernels needs only the types */
/* ---- library / context ---------------------------------------------------- */
const char* qsb_last_error(void);
int32_t qsb_abi_version(void);
int32_t qsb_device_count(int32_t* count);
int32_t qsb_ctx_create(int32_t device, qsb_ctx* out);
int32_t qsb_ctx_destroy(qsb_ctx ctx);
int32_t qsb_ctx_synchronize(qsb_ctx ctx);
/* options: "tile_qubits", "batch", "resident_max_qubits", "threads" (0 = default)   */
int32_t qsb_ctx_set_option(qsb_ctx ctx, const char* key, int64_t value);
int32_t qsb_ctx_last_stats(qsb_ctx ctx, qsb_stats* out);

/* ---- StateVector objects (sim.py:80-95) ----------------------------------- */
int32_t qsb_state_create(qsb_ctx ctx, int32_t nqubits, int32_t precision, qsb_state* out); /* |0..0> (StateVector.zero, sim.py:86-89) */
int32_t qsb_state_destroy(qsb_state st);
int32_t qsb_state_set(qsb_state st, const double* amps);          /* host complex128[2^n] -> device */
int32_t qsb_state_get(qsb_state st, double* amps);                /* device -> host complex128[2^n] */
int32_t qsb_state_copy(qsb_state dst, qsb_state src);             /* StateVector.copy, sim.py:94-95 */
int32_t qsb_state_norm(qsb_state st, double* out);                /* StateVector.norm, sim.py:91-92 */
int32_t qsb_state_device_ptr(qsb_state st, void** out);           /* raw device amplitudes         */

/* apply_gate / _apply_unitary (sim.py:203-227); params = BoundKernel.values */
int32_t qsb_apply_gate(qsb_state st, const qsb_op* op, const double* params, int32_t nparams);
/* measure (sim.py:230-251): u is the caller's uniform draw; outcome = u < p1          */
int32_t qsb_measure(qsb_state st, int32_t qubit, double u, int32_t* outcome, double* p1);
/* reset (sim.py:254-259)                                                             */
int32_t qsb_reset(qsb_state st, int32_t qubit, double u, int32_t* outcome);

/* slice primitives of the global-qubit-sliced engine (sliced.py): the measurement of
 * sim.py:230-251 split into a deterministic partial p1 (summed across slices in rank
 * order by the host) and the collapse; a complex scale for diagonal gates and
 * projections on global qubits.                                                       */
int32_t qsb_state_prob1(qsb_state st, int32_t qubit, double* p1);  /* qubit < 0: sum of |a|^2 */
int32_t qsb_state_collapse(qsb_state st, int32_t qubit, int32_t outcome, double scale, int32_t flip);
int32_t qsb_state_scale(qsb_state st, double re, double im);
/* expval_pauli (sim.py:420-430): xmask = X|Y letters, zmask = Z|Y letters, ny = #Y   */
int32_t qsb_expval_pauli(qsb_state st, uint64_t xmask, uint64_t zmask, int32_t ny, double* out);

/* ---- tapes: a compiled Kernel, immutable, reused across binds (compile-once) ---- */
int32_t qsb_tape_create(qsb_ctx ctx, const qsb_op* ops, int32_t nops, int32_t nqubits,
                        int32_t nbits, int32_t nparams, qsb_tape* out);
int32_t qsb_tape_destroy(qsb_tape tp);
/* 1 if the reference's _needs_trajectories rule (sim.py:322-335) selects trajectories */
int32_t qsb_tape_is_dynamic(qsb_tape tp, int32_t* out);

/* sample's trajectory path (_trajectory_counts, sim.py:346-351 / 379-391): shots
 * [shot_begin, shot_begin + shot_count) of the per-shot RNG streams
 * RngStream.for_shot(seed, shot) (sim.py:54-57).  bits_out: [shot_count][nwords]
 * with nwords = ceil(nbits / 64).  predrawn (nullable): [shot_count][predrawn_stride]
 * uniforms consumed instead of the RNG.  shot_status (nullable): per-shot qsb_status.
 * Returns QSB_ERR_DEGENERATE if any shot hit a degenerate branch.                    */
int32_t qsb_sample_trajectories(qsb_tape tp, int32_t precision, const double* params,
                                uint64_t seed, int64_t shot_begin, int64_t shot_count,
                                const double* predrawn, int32_t predrawn_stride,
                                uint64_t* bits_out, int32_t* shot_status);

/* qsb_sample_trajectories (no pre-drawn stream) that also returns the final states of
 * the first nstates shots into states_out[0..nstates-1] (tape qubit count, same
 * precision), read from the batched streaming engine exactly as it left them (history
 * dedup, fused passes, pending collapse applied): the final StateVector that
 * run_trajectory (sim.py:306-314) returns for each of those shots.  Streaming engine
 * only (QSB_ERR_UNSUPPORTED under the resident engine).                              */
int32_t qsb_sample_trajectories_states(qsb_tape tp, int32_t precision, const double* params, uint64_t seed,
                                       int64_t shot_begin, int64_t shot_count, uint64_t* bits_out,
                                       int32_t* shot_status, int32_t nstates, qsb_state* states_out);

/* run_trajectory (sim.py:306-314) for one shot.  The RNG starts from `rng_state`
 * (4 xoshiro256++ words, updated in place with the words after the run, like the
 * reference mutating its RngStream) or, when rng_state is null, from
 * RngStream.for_shot(seed, shot).  Optionally returns the final state into
 * `state_out` (tape qubit count, same precision) and the CondBlock trace
 * (sim.py:296-301): per executed IF, [op_index, taken, bits words...] (2 + nwords
 * int64 per entry).  ndraws receives the number of uniforms consumed.               */
int32_t qsb_run_trajectory(qsb_tape tp, int32_t precision, const double* params, uint64_t* rng_state,
                           uint64_t seed, int64_t shot, const double* predrawn, int32_t npredrawn,
                           uint64_t* bits_out, qsb_state state_out, int64_t* trace_out,
                           int32_t max_trace, int32_t* ntrace, int32_t* ndraws);

/* statevector (sim.py:402-409): static tapes only (QSB_ERR_DYNAMIC otherwise).       */
int32_t qsb_statevector(qsb_tape tp, const double* params, qsb_state out);

/* apply a gates-only tape to a state IN PLACE (the fused streaming passes of
 * qsb_statevector without the |0...0> start): the sequence of apply_gate calls
 * (sim.py:224-227) it replaces, fused.  Used by the sliced executor to run the local
 * gates between two exchanges on each slice in a few passes.                         */
int32_t qsb_apply_tape(qsb_tape tp, const double* params, qsb_state st);

/* _sample_static (sim.py:354-369): one simulation, sequential fp64 cumsum, per-shot
 * searchsorted(side="right"), top-level measures written in program order.           */
int32_t qsb_sample_static(qsb_tape tp, int32_t precision, const double* params, uint64_t seed,
                          int64_t shot_begin, int64_t shot_count, uint64_t* bits_out);

/* sample (sim.py:372-391) with the shot histogram built on the device
 * (ShotHistogram.counts, sim.py:122-131): the per-shot words of shots
 * [shot_begin, shot_begin + shot_count) -- trajectory or static path, exactly as
 * qsb_sample_trajectories / qsb_sample_static produce them -- are sorted and
 * run-length encoded in HBM; words_out / counts_out receive the distinct words in
 * ascending order and their counts, *nunique_out their number.  Tapes with more than
 * 64 classical bits return QSB_ERR_UNSUPPORTED (use the per-shot words); more than
 * max_unique distinct outcomes returns QSB_ERR_ARG with *nunique_out set.            */
int32_t qsb_sample_counts(qsb_tape tp, int32_t precision, const double* params, uint64_t seed,
                          int64_t shot_begin, int64_t shot_count, uint64_t* words_out, int64_t* counts_out,
                          int64_t max_unique, int64_t* nunique_out);

/* observe(): E[p] = sum_t coef[t] * <psi(params[p])| P_t |psi(params[p])>, the caller-
 * side composition of statevector + expval_pauli (suites.py:319-323).  term_out
 * (nullable) receives [npoints][nterms] single-term expectations.                    */
int32_t qsb_observe(qsb_tape tp, int32_t precision, const double* params, int64_t npoints,
                    const uint64_t* xmask, const uint64_t* zmask, const int32_t* ny,
                    const double* coef, int32_t nterms, double* energies_out, double* term_out);

/* host-only planner summary (no device needed): builds the streaming plan of a tape
 * for tile_qubits / low_qubits / reg_bits and writes
 * out[0..7] = {passes, phases, pass gates, regions, descriptor gates, epilogue passes,
 *              max phases per pass, register-blocked (1) or shared-memory (0) kernel}.   */
int32_t qsb_plan_summary(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                         int32_t tile_qubits, int32_t low_qubits, int32_t reg_bits, int64_t* out);

/* host-only: the streaming plan's passes (gates per pass, epilogue flag) with gate
 * deferral past measurement regions on (1) or off (0); *npasses = number of passes.   */
int32_t qsb_plan_passes(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                        int32_t tile_qubits, int32_t low_qubits, int32_t reg_bits, int32_t defer_gates,
                        int64_t* gates_out, int32_t* epi_out, int32_t max_passes, int32_t* npasses);

/* host-only: generate and NVRTC-compile (no device needed, nothing loaded) the
 * specialised pass kernels of a tape's streaming plan; returns QSB_OK or QSB_ERR_ARG
 * with the compiler log in qsb_last_error().  reg_bits = 3, 4 or 5 amplitude-register
 * qubits per thread.  out[0] = kernels, out[1] = milliseconds. */
int32_t qsb_jit_selftest(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                         int32_t precision, int32_t reg_bits, double* out);

/* host-only: version of the NVRTC library the pass generator compiles with (opened on first
 * use: $QSB_NVRTC, then the toolkit's /usr/local/cuda/lib64/libnvrtc.so.12, then the
 * soname).  QSB_ERR_ARG when no NVRTC can be loaded.                                   */
int32_t qsb_jit_nvrtc_version(int32_t* major, int32_t* minor);

/* host-only: register-phase gate fusion of the NVRTC kernels (qsb_plan.h fuse_phase) over
 * a tape's streaming plan (tile 12).  out[0..5] = {phases, fused blocks, gates folded into
 * blocks, host-check failures, pass flops per state unfused, the same fused}.          */
int32_t qsb_fusion_stats(const qsb_op* ops, int32_t nops, int32_t nqubits, int32_t nbits, int32_t nparams,
                         int32_t precision, int32_t reg_bits, double* out);

/* ---- global-qubit-sliced engine (BASELINE cfg 5; sliced.py drives it) -----------------
 * A state of n qubits is split into 2^G slices of L = n - G qubits (one per rank/GPU, or
 * all on one GPU for the single-device emulation).  The host planner enqueues; every
 * classical decision is made on the device from the qsb_slicectl (RNG stream, classical
 * store, if/else guards, status), so a trajectory runs without host round-trips.
 * Reference semantics: run_trajectory / _exec_ops (sim.py:279-314), measure / reset
 * (sim.py:230-259), _eval_predicate (sim.py:262-276).                                  */
/* RNG = rng_state (4 words) or RngStream.for_shot(seed, shot); nslices partial slots   */
int32_t qsb_slice_ctl_create(qsb_ctx ctx, int32_t nslices, int32_t nbits, uint64_t seed, int64_t shot,
                             const uint64_t* rng_state, qsb_slicectl* out);
int32_t qsb_slice_ctl_destroy(qsb_slicectl c);
/* synchronising read-back: classical words, qsb_status, uniforms drawn, RNG words     */
int32_t qsb_slice_ctl_read(qsb_slicectl c, uint64_t* bits_out, int32_t* status, int32_t* draws, uint64_t* rng_out);
/* IF (predicate evaluated on the device store at entry) / ELSE / ENDIF records         */
int32_t qsb_slice_guard(qsb_slicectl c, const qsb_op* op);
/* guarded gate on LOCAL positions (matrix host-built, has_matrix = 1; no swap)         */
int32_t qsb_slice_gate(qsb_state st, qsb_slicectl c, const qsb_op* op);
/* guarded complex scale (a diagonal gate on a global target, per slice)               */
int32_t qsb_slice_scale(qsb_state st, qsb_slicectl c, double re, double im);
/* this slice's partial p1 of local qubit `qubit` (< 0: its whole norm; select = 0: the
 * slice holds none of the measured amplitudes) into partial slot `index`              */
int32_t qsb_slice_prob1(qsb_state st, qsb_slicectl c, int32_t qubit, int32_t select, int32_t index);
/* host read (host_out) and / or write (host_in) of the nslices partial slots, for a
 * transport that all-gathers them through the host (torch.distributed / gloo)         */
int32_t qsb_slice_partials(qsb_slicectl c, double* host_out, const double* host_in);
/* sum the partials in slice order, draw, decide (sim.py:236-248), write the bit       */
int32_t qsb_slice_decide(qsb_slicectl c, int32_t kind, int32_t bit);
/* apply the decision: local qubit (flip = reset) or, qubit < 0, a global qubit whose
 * value in this slice is gbit                                                         */
int32_t qsb_slice_collapse(qsb_state st, qsb_slicectl c, int32_t qubit, int32_t gbit, int32_t flip);
/* single device: swap global position <-> local position pos between the slice pair
 * (a: global bit 0, b: global bit 1) in place                                         */
int32_t qsb_slice_exchange_local(qsb_state a, qsb_state b, int32_t pos);
/* single device: remap k = 1..3 global positions with local positions lpos[0..k) across
 * the 2^k slices group[0 .. 2^k) (group[y]: remapped global bits y) -- the amplitude at
 * (slice y, local bits x at lpos) moves to (slice x, local bits y), in place            */
int32_t qsb_slice_remap_local(const qsb_state* group, int32_t k, const int32_t* lpos);
/* host copy of / into the region of a slice whose local bits at lpos equal x (2^(n-k)
 * amplitudes in the slice's precision, increasing order of the other bits)             */
int32_t qsb_slice_read_sub(qsb_state st, int32_t k, const int32_t* lpos, int32_t x, void* host_out);
int32_t qsb_slice_write_sub(qsb_state st, int32_t k, const int32_t* lpos, int32_t x, const void* host_in);

/* NCCL data plane (libnccl.so.2 opened at run time; QSB_ERR_UNSUPPORTED without it)    */
int32_t qsb_comm_unique_id(uint8_t* out128);                  /* rank 0, broadcast by the caller */
int32_t qsb_comm_init(qsb_ctx ctx, const uint8_t* id128, int32_t rank, int32_t nranks, qsb_comm* out);
int32_t qsb_comm_destroy(qsb_comm c);
int32_t qsb_comm_set_chunk(qsb_comm c, int64_t bytes);        /* exchange staging chunk (default 64 MiB) */
/* partial slot `rank` of every rank -> all slots on every rank (ncclAllGather, in place) */
int32_t qsb_comm_allgather_partials(qsb_comm c, qsb_slicectl s);
/* exchange with `peer`: send the packed half of `send` (global bit send_c: local bit pos
 * == !send_c) and unpack the peer's into the same half of `recv`; chunked ncclSend /
 * ncclRecv on the context stream.  Production: send == recv (in place).               */
int32_t qsb_comm_exchange(qsb_comm c, qsb_state send, int32_t send_c, qsb_state recv, int32_t recv_c, int32_t pos,
                          int32_t peer);
/* remap of k = 1..3 global positions among the ranks peers[0 .. 2^k) (this rank =
 * peers[self]): region x of this slice goes to peers[x], peers[x]'s region `self` comes
 * back into region x -- grouped ncclSend / ncclRecv to all 2^k - 1 peers per chunk      */
int32_t qsb_comm_remap(qsb_comm c, qsb_state st, int32_t k, const int32_t* lpos, const int32_t* peers, int32_t self);
/* out3 = {bytes sent, exchanges, all-gathers}; CUDA-event ms of the last exchange     */
int32_t qsb_comm_stats(qsb_comm c, int64_t* out3, double* last_exchange_ms);
int32_t qsb_comm_nccl_version(int32_t* version);

/* debug / known-answer hook: the first `count` uniforms of RngStream.for_shot(seed, shot)
 * drawn by the DEVICE generator (pins the on-device RNG to sim.py:54-72).              */
int32_t qsb_debug_rng(qsb_ctx ctx, uint64_t seed, int64_t shot, int32_t count, double* out);

/* measured FMA throughput of this device in TFLOP/s (fp64 for QSB_C128, fp32 for
 * QSB_C64): the compute roofline denominator of the pass kernels.                     */
int32_t qsb_debug_fma_peak(qsb_ctx ctx, int32_t precision, double* tflops);
#endif /* QSB_JIT */

#ifdef __cplusplus
}
#endif
#endif /* QSB_H */
