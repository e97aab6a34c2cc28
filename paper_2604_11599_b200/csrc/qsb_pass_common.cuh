// Persistent, double-buffered fused-pass driver shared by the generic register-blocked
// kernel (qsb_pass_reg.cu) and the NVRTC-specialised per-pass kernels (qsb_jit.cpp).
//
// A CTA walks work items w = (slot, tile) with a grid stride.  While the gates of
// item w run on one shared-memory buffer, the gather of item w + gridDim.x is in
// flight into the other buffer through cp.async (LDGSTS, 16 B per complex128
// amplitude straight into its swizzled slot, Pauli-X frame applied by the
// destination address), so HBM traffic overlaps the FP64 work instead of
// alternating with it.  The phase code is supplied by the caller (a functor), which
// is the only difference between the generic and the specialised kernels.
#pragma once
#include "qsb_device.cuh"

namespace qsb {

__constant__ uint8_t c_swz3[16] = {1, 2, 4, 3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7, 1, 2};
__constant__ uint8_t c_swz4[16] = {1, 2, 4, 8, 3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 1};

// a pass gate staged in shared memory with its CTA-uniform decisions resolved
// 112 B (complex128) / 80 B (complex64): strides of 28 / 20 banks, so the 16-byte stores
// of 8 consecutive staging threads hit distinct bank groups (96 / 64 B were 2- / 4-way)
template <typename R> struct SGate {
  int32_t kind, jt, jt2, tp;
  uint32_t cmR, cvR, cmT, cvT;
  R m[8];
  int32_t pad[4];
};

__device__ __forceinline__ uint64_t pext64(uint64_t v, uint64_t mask) {
  uint64_t out = 0;
  int j = 0;
  for (uint64_t m = mask; m; m &= m - 1, ++j)
    if (v & (m & (~m + 1))) out |= 1ull << j;
  return out;
}

template <int SB> __device__ __forceinline__ uint32_t swz_slot(const uint32_t* swz, uint32_t l) {
  return l ^ swz[l >> SB];
}

// named barrier of a thread group (0: __syncthreads of the whole CTA)
__device__ __forceinline__ void group_sync(int bar, int nthreads) {
  if (bar == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(nthreads) : "memory");
}

// the shared-memory context handed to the phase code
template <typename R> struct PassCtx {
  typename Amp<R>::T* tile;
  SGate<R>* sg;
  uint32_t* swz;
  int tid, T, TL;
  int bar;  // barrier of the thread group working on `tile`
  __device__ __forceinline__ void sync() const { group_sync(bar, T); }
};

// per work-item (slot, tile) view of the trajectory control block
struct PassItem {
  int64_t slot;
  int64_t src;  // slot whose buffer the gather reads (history dedup: a branch's first pass)
  bool zero;    // the pending projection zeroes the whole item: no gather, no gates, zeros stored
  uint64_t base_phys, base_log, Kp, Vp;
  uint32_t fl;
  bool alive, pending;
  double sre, sim;
};

// Per-CTA nibble tables for the per-item bit scatters / gathers (all linear over
// disjoint bit fields, so a 64-bit operand is the OR of one entry per 4-bit chunk):
//   pdt[c][v]: pdep of (v << 4c) into the out-of-tile qubits   (tile id -> base)
//   pxs[c][v]: tile positions of the qubits of (v << 4c)        (frame -> tile flip)
//   pxo[c][v]: pext of (v << 4c) over the out-of-tile qubits    (frame -> tile id flip)
struct ItemTables {
  uint64_t* pdt;
  uint32_t* pxs;
  uint64_t* pxo;
};
__host__ __device__ inline int item_chunks(int n) { return (n + 3) / 4; }  // 4-bit chunks of a qubit mask
__host__ __device__ inline size_t item_tables_bytes(int n) {
  return (2 * sizeof(uint64_t) + sizeof(uint32_t)) * item_chunks(n) * 16;
}

__device__ __forceinline__ void build_item_tables(const ItemTables& tb, const PassDesc& pd, int n, int tid, int T) {
  const uint64_t qmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t out = ~pd.smask & qmask;
  for (int e = tid; e < item_chunks(n) * 16; e += T) {
    const int c = e >> 4;
    const uint64_t v = (uint64_t)(e & 15) << (4 * c);
    tb.pdt[e] = pdep64(v, out);
    tb.pxo[e] = pext64(v & out, out);
    uint32_t f = 0;
    for (int j = 0; j < pd.k; ++j)
      if ((v >> pd.sq[j]) & 1) f |= 1u << j;
    tb.pxs[e] = f;
  }
}

__device__ __forceinline__ uint64_t tab64(const uint64_t* t, uint64_t x, int nbits) {
  uint64_t r = 0;
  for (int c = 0; c * 4 < nbits; ++c) r |= t[c * 16 + ((x >> (4 * c)) & 15)];
  return r;
}
__device__ __forceinline__ uint32_t tab32(const uint32_t* t, uint64_t x, int nbits) {
  uint32_t r = 0;
  for (int c = 0; c * 4 < nbits; ++c) r |= t[c * 16 + ((x >> (4 * c)) & 15)];
  return r;
}

// the per-state part of an item's context (one TrajCtl read)
struct SlotCtx {
  int64_t idx;  // active-list index (w >> ntl)
  int64_t slot, src;
  uint64_t F, Kp, Vp;
  double sre, sim;
  bool alive, pending;
};

__device__ __forceinline__ SlotCtx slot_ctx(const StreamArgs& a, const PassDesc& pd, int64_t idx) {
  SlotCtx s;
  s.idx = idx;
  s.slot = a.active ? a.active[idx] : idx;  // representative slots only (history dedup)
  // a branch that just split off its representative reads the representative's
  // (pre-collapse) buffer in its first pass instead of a copy of it
  const int32_t rs = a.read_src ? a.read_src[s.slot] : -1;
  s.src = rs >= 0 ? rs : s.slot;
  const TrajCtl* c = a.ctl + s.slot;
  s.alive = c->status == 0;
  s.F = c->frame & ~pd.clear_before;
  s.pending = pd.prologue && c->pending;
  s.Kp = c->kmask;
  s.Vp = c->kval;
  s.sre = c->sre;
  s.sim = c->sim;
  return s;
}

__device__ __forceinline__ PassItem item_of(const SlotCtx& s, const PassDesc& pd, uint64_t tile, int ntl, int n,
                                            const ItemTables& tb) {
  PassItem it;
  it.slot = s.slot;
  it.src = s.src;
  it.alive = s.alive;
  it.pending = s.pending;
  it.Kp = s.Kp;
  it.Vp = s.Vp;
  it.sre = s.sre;
  it.sim = s.sim;
  it.base_phys = tab64(tb.pdt, tile, ntl);
  // the collapse of the previous measurement keeps only (p & Kp) == Vp: when the item's
  // out-of-tile bits already disagree, every amplitude of it becomes zero
  it.zero = s.pending && ((it.base_phys ^ s.Vp) & s.Kp & ~pd.smask) != 0 && !pd.epi;
  it.base_log = it.base_phys ^ (s.F & ~pd.smask);
  it.fl = tab32(tb.pxs, s.F, n);
  return it;
}

__device__ __forceinline__ PassItem pass_item(const StreamArgs& a, const PassDesc& pd, int64_t w, int ntl,
                                              const ItemTables& tb) {
  return item_of(slot_ctx(a, pd, w >> ntl), pd, (uint64_t)w & ((1ull << ntl) - 1), ntl, a.n, tb);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {  // release: plain shared stores before it are visible
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* b) {  // fires when this thread's cp.async land
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nQSB_MBW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra QSB_MBW;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

// Buffering of the persistent driver: each CTA (2 per SM) walks its items alone;
// complex64 tiles (32 KiB) double-buffer, complex128 tiles (64 KiB) keep one buffer whose
// scatter overlaps the next gather, and the two CTAs of an SM overlap each other.  (A
// two-group / three-tile-ring mode with mbarrier hand-off was measured 6-20 % slower in
// round 1 and removed; `mode` stays in the signatures as 0.)
__host__ __device__ inline int pass_buffers(int c64, int mode) { return c64 ? 2 : 1; }
__host__ __device__ inline int pass_groups(int mode) { return 1; }

// dynamic shared memory of a register-blocked pass
__host__ __device__ inline size_t pass_reg_smem(int c64, const PassDesc& pd, int rb, int n, bool stage, int mode = 0) {
  const int sb = c64 ? 4 : 3;
  const size_t amp = c64 ? 8 : 16;
  const size_t sgate = c64 ? 80 : 112;  // sizeof(SGate<float / double>)
  const int G = pass_groups(mode);
  return pass_buffers(c64, mode) * (amp << pd.k) + G * (stage ? sgate * pd.pgate_count : 0) +
         (sizeof(uint64_t) << (pd.k - pd.lowq)) + (sizeof(uint32_t) << (pd.k - sb)) +
         G * sizeof(double) * (1u << (pd.k - rb)) + sizeof(uint32_t) * (1u << rb) + item_tables_bytes(n) + 16;
}


// STAGE: stage the pass gates into shared memory per item (guards, out-of-tile
// controls, per-tile diagonal factors, per-point matrices).  The NVRTC kernels pass
// false when none of their phases reads the staged gates (literal matrices from the
// constant bank, no per-item decisions), which removes a global-load round trip and a
// barrier from every item.
// DIRECT (NVRTC complex128 passes without an epilogue, MODE 0): `run` executes every
// phase but the last; `run_last(cx, dst, hi_off, mid)` loads the last phase's registers
// from the tile, calls mid() -- which releases the buffer and issues the next item's
// gather -- and then computes and stores its registers straight to HBM, so the gather
// overlaps the last phase's arithmetic and the tile makes one shared-memory round trip
// less.
struct NoLastPhase {
  template <typename... T> __device__ void operator()(T&&...) const {}
};

template <typename R, int RB, bool STAGE = true, int MODE = 0, bool DIRECT = false, typename PhaseRunner,
          typename LastRunner = NoLastPhase>
__device__ __forceinline__ void pass_persistent(const StreamArgs& a, const PassDesc& pd, unsigned char* smem_raw,
                                                PhaseRunner run, LastRunner run_last = LastRunner()) {
  static_assert(MODE == 0, "single-group driver");
  using A = typename Amp<R>::T;
  constexpr int SB = sizeof(R) == 8 ? 3 : 4;
  constexpr int G = 1;                             // thread groups
  constexpr int NB = sizeof(R) == 4 ? 2 : 1;       // pass_buffers()
  const int k = pd.k, TL = 1 << k, T = TL >> RB;
  const int grp = 0;
  const int tid = (int)threadIdx.x;
  const int ctid = threadIdx.x, CT = G * T;        // whole CTA (table set-up)
  const int bar = 0;
  A* bufs = reinterpret_cast<A*>(smem_raw);
  SGate<R>* sg0 = reinterpret_cast<SGate<R>*>(bufs + NB * TL);
  SGate<R>* sg = sg0 + (STAGE ? grp * pd.pgate_count : 0);
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(sg0 + (STAGE ? G * pd.pgate_count : 0));
  uint32_t* swz = reinterpret_cast<uint32_t*>(hi_off + (TL >> pd.lowq));
  double* red0 = reinterpret_cast<double*>(swz + (TL >> SB));
  double* red = red0 + grp * T;
  uint32_t* ujt = reinterpret_cast<uint32_t*>(red0 + G * T);  // [2^RB] swizzled slot of j*T
  ItemTables itb;
  itb.pdt = reinterpret_cast<uint64_t*>((reinterpret_cast<size_t>(ujt + (1 << RB)) + 15) & ~(size_t)15);
  itb.pxo = itb.pdt + item_chunks(a.n) * 16;
  itb.pxs = reinterpret_cast<uint32_t*>(itb.pxo + item_chunks(a.n) * 16);
  build_item_tables(itb, pd, a.n, ctid, CT);
  const uint64_t lowm = (1ull << pd.lowq) - 1;
  const uint64_t shi = pd.smask & ~lowm;
  for (int h = ctid; h < (TL >> pd.lowq); h += CT) hi_off[h] = pdep64((uint64_t)h, shi);
  const uint8_t* V = SB == 3 ? c_swz3 : c_swz4;
  for (int h = ctid; h < (TL >> SB); h += CT) {
    uint32_t s = 0;
    for (int p = SB, hh = h; hh; ++p, hh >>= 1)
      if (hh & 1) s ^= V[p];
    swz[h] = s;
  }
  __syncthreads();
  // Tile element l = tid + j*T (j < 2^RB; tid and j*T occupy disjoint bits, and
  // T is a multiple of 2^lowq and of 2^SB).  pdep and the swizzle are both linear
  // over disjoint bit fields, so
  //   physical offset  = base_phys | Pt | hi_off[j * (T >> lowq)]
  //   swizzled slot    = St ^ ujt[j]            (St = tid ^ swz[tid >> SB])
  // and with the Pauli-X frame flip fl of an item the slot of l ^ fl is
  //   (Ft ^ G) ^ ujt[j], Ft = swizzled slot of tid ^ (fl & (T-1)), G = that of fl & ~(T-1).
  // The loops below therefore cost a few integer ops per amplitude.
  if (ctid < (1 << RB)) ujt[ctid] = swz_slot<SB>(swz, (uint32_t)(ctid * T));
  const uint64_t Pt = ((uint64_t)tid & lowm) | hi_off[tid >> pd.lowq];
  const uint32_t St = swz_slot<SB>(swz, (uint32_t)tid);
  const int hstep = T >> pd.lowq;
  __syncthreads();
  const int ntl = a.n - k;
  // pd.zero_tid: the items whose tile id has one of these bits set are known zero (qubits
  // still in |0>, buffers pre-zeroed): enumerate only the others -- the tile id is the
  // item's free bits deposited around the zero ones (the init pass: tile 0 only)
  const uint64_t tid_all = (ntl >= 64) ? ~0ull : ((1ull << ntl) - 1);
  const uint64_t tid_free = tid_all & ~pd.zero_tid;
  const int ntl_run = __popcll(tid_free);
  const int64_t W = (int64_t)(a.active ? *a.nactive : a.slots) << ntl_run;
  auto item_at = [&](int64_t w) -> PassItem {
    if (!pd.zero_tid) return pass_item(a, pd, w, ntl, itb);
    const SlotCtx sc = slot_ctx(a, pd, w >> ntl_run);
    uint64_t tile = pdep64((uint64_t)w & ((1ull << ntl_run) - 1), tid_free);
    if (pd.zero_from_vp) tile |= tab64(itb.pxo, sc.Vp, a.n) & pd.zero_tid;  // the items the collapse keeps
    return item_of(sc, pd, tile, ntl, a.n, itb);
  };

  // swizzled-slot base of this thread for an item with frame flip fl
  auto flip_base = [&](uint32_t fl) -> uint32_t {
    return swz_slot<SB>(swz, (uint32_t)tid ^ (fl & (uint32_t)(T - 1))) ^ swz_slot<SB>(swz, fl & ~(uint32_t)(T - 1));
  };

  auto prefetch = [&](const PassItem& it, A* dst) {
    if (!it.alive || it.zero) return;
    const A* st = reinterpret_cast<const A*>(a.state) + (it.src << a.n);
    const uint64_t pb = it.base_phys | Pt;
    const uint32_t fb = flip_base(it.fl);
#pragma unroll 4
    for (int j = 0; j < (1 << RB); ++j) {
      A* d = dst + (fb ^ ujt[j]);
      const uint64_t p = pb | hi_off[j * hstep];
      if (pd.init_zero) {
        *d = mk<R>(p == 0 ? (R)1 : (R)0, (R)0);
      } else if (((p ^ it.Vp) & pd.zk_mask) != 0) {  // rejected by the last collapse, never stored since
        *d = mk<R>((R)0, (R)0);
      } else if (sizeof(A) == 16) {
        cp_async16(d, st + p);
      } else {
        cp_async8(d, st + p);
      }
    }
  };

  // One item on `tile` (gathered): pending collapse, gate staging, the phases, the
  // epilogue marginal; leaves the tile in the registers v.
  auto process = [&](const PassItem& it, A* tile, A* v) {
    if (it.pending) {  // collapse of the previous decide: projection + complex scale
      const R sre = (R)it.sre, sim = (R)it.sim;
      const uint64_t pb = it.base_phys | Pt;
      const uint32_t fb = flip_base(it.fl);
      for (int j = 0; j < (1 << RB); ++j) {
        const uint64_t p = pb | hi_off[j * hstep];
        A* d = tile + (fb ^ ujt[j]);
        A x = *d;
        if ((p & it.Kp) != it.Vp) x = mk<R>(0, 0);
        else x = mk<R>(fma(sre, x.x, -sim * x.y), fma(sre, x.y, sim * x.x));
        *d = x;
      }
    }
    if (STAGE) {  // stage the gates: guards, out-of-tile controls, per-CTA diagonal factors
      const uint32_t* gw = a.guards + it.slot * a.gwords;
      const double* mats = a.mats + it.slot * a.mat_stride;
      for (int i = tid; i < pd.pgate_count; i += T) {
        const PhaseGate g = a.phase_gates[pd.pgate_begin + i];
        SGate<R> s;
        double m[8];
        const double* src = mats + (int64_t)g.mat * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = src[j];
        int kind = g.kind;
        bool skip = (g.guard >= 0 && !((gw[g.guard >> 5] >> (g.guard & 31)) & 1u)) ||
                    ((it.base_log & g.gcm) != g.gcv);
        if (kind == PK_DIAG_G) kind = PK_DIAG_T;  // same code path, tp = -1
        if (kind == PK_DENSE) {
          if (m[1] == 0.0 && m[3] == 0.0 && m[5] == 0.0 && m[7] == 0.0) kind = PK_DENSE_REAL;
          else if (m[1] == 0.0 && m[7] == 0.0 && m[2] == 0.0 && m[4] == 0.0) kind = PK_DENSE_RX;
        } else if (g.kind == PK_DIAG_G) {
          int bb = (int)((it.base_log >> g.tp) & 1);
          if (!bb && g.diag_one0) skip = true;
          if (bb) {
            m[0] = m[6];
            m[1] = m[7];
          }
        }
        s.kind = skip ? PK_SKIP : kind;
        s.jt = g.kind == PK_DIAG_T ? g.diag_one0 : g.jt;
        s.jt2 = g.jt2;
        s.tp = (g.kind == PK_DIAG_T || g.kind == PK_SWAP_R) ? g.tp : -1;
        s.cmR = g.cmR;
        s.cvR = g.cvR;
        s.cmT = g.cmT;
        s.cvT = g.cvT;
#pragma unroll
        for (int j = 0; j < 8; ++j) s.m[j] = (R)m[j];
        sg[i] = s;
      }
    }
    if (STAGE || it.pending) group_sync(bar, T);
    PassCtx<R> cx{tile, sg, swz, tid, T, TL, bar};
    run(cx);  // the phases (each ends with cx.sync())
    if (DIRECT) return;
    if (pd.epi) {  // per-tile marginal of the next region's measured qubits (fixed order)
      const int ml = pd.m_local;
      const int nb = 1 << ml;
      uint32_t mlm = 0;
      for (int j = 0; j < ml; ++j) mlm |= 1u << pd.mloc[j];
      const uint32_t free_mask = ((uint32_t)TL - 1) & ~mlm;
      const int members = TL >> ml;
      const uint64_t t_log = tab64(itb.pxo, it.base_log, a.n);
      double* out = a.partial + it.slot * a.partial_stride + (int64_t)t_log * nb;
      if (nb <= T) {
        const int tp = T / nb;
        // bin fastest across the warp: neighbouring threads read neighbouring
        // amplitudes when the measured qubits are low tile positions (the common case)
        const int bb = tid % nb, j = tid / nb;
        uint32_t bpos = 0;
        for (int jj = 0; jj < ml; ++jj)
          if ((bb >> jj) & 1) bpos |= 1u << pd.mloc[jj];
        // members r = j, j + tp, ... deposited into free_mask by masked addition
        // (x | ~mask) + d carries across the holes), in increasing order
        const uint32_t inc = (uint32_t)pdep64((uint64_t)tp, free_mask);
        uint32_t f = (uint32_t)pdep64((uint64_t)j, free_mask);
        auto step = [&](uint32_t x) { return ((x | ~free_mask) + inc) & free_mask; };
        // four independent accumulators (fixed association): the shared loads and
        // FP64 adds of consecutive members overlap instead of forming one chain
        const int cnt = (members - j + tp - 1) / tp;
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        int i = 0;
        for (; i + 4 <= cnt; i += 4) {
          const uint32_t f1 = step(f), f2 = step(f1), f3 = step(f2);
          s4[0] += norm2<R>(tile[swz_slot<SB>(swz, f | bpos)]);
          s4[1] += norm2<R>(tile[swz_slot<SB>(swz, f1 | bpos)]);
          s4[2] += norm2<R>(tile[swz_slot<SB>(swz, f2 | bpos)]);
          s4[3] += norm2<R>(tile[swz_slot<SB>(swz, f3 | bpos)]);
          f = step(f3);
        }
        for (; i < cnt; ++i) {
          s4[0] += norm2<R>(tile[swz_slot<SB>(swz, f | bpos)]);
          f = step(f);
        }
        red[tid] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        group_sync(bar, T);
        if (j == 0) {
          double tot = 0.0;
          for (int jj = 0; jj < tp; ++jj) tot += red[bb + nb * jj];
          out[bb] = tot;
        }
      } else {
        for (int bb = tid; bb < nb; bb += T) {
          uint32_t bpos = 0;
          for (int jj = 0; jj < ml; ++jj)
            if ((bb >> jj) & 1) bpos |= 1u << pd.mloc[jj];
          double s = 0.0;
          uint32_t f = 0;
          for (int r = 0; r < members; ++r) {
            s += norm2<R>(tile[swz_slot<SB>(swz, f | bpos)]);
            f = ((f | ~free_mask) + 1u) & free_mask;
          }
          out[bb] = s;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) v[j] = tile[St ^ ujt[j]];
  };
  auto scatter = [&](const PassItem& it, const A* v) {
    A* st = reinterpret_cast<A*>(a.state) + (it.slot << a.n);
    const uint64_t pb = it.base_phys | Pt;
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) st[pb | hi_off[j * hstep]] = v[j];
  };

  int64_t w = blockIdx.x;
  PassItem cur;
  cur.alive = false;
  if (w < W) cur = item_at(w);
  if (w < W) prefetch(cur, bufs);
  cp_async_commit();
  int b = 0;
  for (; w < W; w += gridDim.x) {
    const int64_t wn = w + gridDim.x;
    PassItem nxt;
    nxt.alive = false;
    if (wn < W) nxt = item_at(wn);
    if (NB == 2) {
      if (wn < W) prefetch(nxt, bufs + (b ^ 1) * TL);
      cp_async_commit();
      cp_async_wait1();
    } else {
      // single buffer: this item's gather was issued at the end of the previous item,
      // concurrently with that item's scatter
      cp_async_wait0();
    }
    __syncthreads();
    const PassItem it = cur;
    cur = nxt;
    if (DIRECT && NB == 1) {
      auto mid = [&]() {
        __syncthreads();  // every thread holds its last-phase registers: the buffer is free
        if (wn < W) prefetch(cur, bufs);
        cp_async_commit();
      };
      if (it.alive && !it.zero) {
        A dummy[1];
        process(it, bufs, dummy);
        PassCtx<R> cx{bufs, sg, swz, tid, T, TL, bar};
        A* dst = reinterpret_cast<A*>(a.state) + (it.slot << a.n) + it.base_phys;
        run_last(cx, dst, hi_off, mid);
      } else {
        mid();
        if (it.alive) {  // projected away: store zeros
          A z[1 << RB];
#pragma unroll
          for (int j = 0; j < (1 << RB); ++j) z[j] = mk<R>((R)0, (R)0);
          scatter(it, z);
        }
      }
      continue;
    }
    A v[1 << RB];
    if (it.alive && !it.zero) {
      process(it, bufs + b * TL, v);
    } else {
#pragma unroll
      for (int j = 0; j < (1 << RB); ++j) v[j] = mk<R>((R)0, (R)0);
    }
    // single buffer: the tile is in registers -- release the buffer, start the next
    // item's gather, then store, so that the scatter and the next gather overlap
    __syncthreads();
    if (NB == 1) {
      if (wn < W) prefetch(cur, bufs);
      cp_async_commit();
    }
    if (it.alive) scatter(it, v);
    if (NB == 2) b ^= 1;
  }
  cp_async_wait0();
}

// swap-only phase: tile positions tp, jt2; controls on the full tile index
template <typename R, int SB> __device__ __forceinline__ void pass_swap(const PassCtx<R>& cx, const SGate<R>& g) {
  using A = typename Amp<R>::T;
  if (g.kind != PK_SKIP) {
    const int lo = g.tp < g.jt2 ? g.tp : g.jt2, hi = g.tp < g.jt2 ? g.jt2 : g.tp;
    for (int qd = cx.tid; qd < (cx.TL >> 2); qd += cx.T) {
      uint32_t b = (uint32_t)insert_zero(insert_zero((uint64_t)qd, lo), hi);
      if ((b & g.cmT) != g.cvT) continue;
      uint32_t la = swz_slot<SB>(cx.swz, b | (1u << g.tp)), lb = swz_slot<SB>(cx.swz, b | (1u << g.jt2));
      A x = cx.tile[la];
      cx.tile[la] = cx.tile[lb];
      cx.tile[lb] = x;
    }
  }
}

}  // namespace qsb
