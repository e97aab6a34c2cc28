// Streaming engine: states in HBM ([slots][2^n]), one fused pass = one read + one
// write of every amplitude.  See DESIGN.md "Streaming engine".
//
// pass kernel (grid = tiles x slots, one CTA per 2^k-amplitude tile of one state):
//   prologue  gather the tile (qubits S; the low `lowq` qubits are contiguous, so
//             every warp load is a >= 256 B run), undo the per-trajectory Pauli-X
//             frame on the tile's qubits, apply the pending collapse of the last
//             decide (projection + complex scale) -- no separate collapse pass;
//   body      every fused gate of the pass in shared memory (per-trajectory guard
//             bits and out-of-tile controls are CTA-uniform branches);
//   epilogue  per-tile marginal of the next region's measured qubits (fixed-order,
//             deterministic), scatter the tile back in logical order.
// decide kernel (grid = slots): sums the tile marginals in fixed order and walks the
//   region's control ops sequentially: measure / reset (u < p1, DegenerateNorm),
//   IF/ELSE/ENDIF guard bits, Pauli / phase gates on collapsed qubits.
#include <cuda_runtime.h>

#include "qsb_device.cuh"
#include "qsb_launch.h"

namespace qsb {

namespace {

constexpr int kPT = 256;  // pass threads
constexpr int kDT = 128;  // decide threads

__device__ __forceinline__ uint64_t pext64(uint64_t v, uint64_t mask) {
  uint64_t out = 0;
  int j = 0;
  for (uint64_t m = mask; m; m &= m - 1, ++j)
    if (v & (m & (~m + 1))) out |= 1ull << j;
  return out;
}

__global__ void k_mats_prep(const MatSrc* src, int nmat, const double* params, int nparams, double* out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t slot = blockIdx.y;
  if (j >= nmat) return;
  double m[8];
  build_matrix(src[j], params ? params + slot * nparams : nullptr, m);
  double* o = out + (slot * nmat + j) * 8;
  for (int i = 0; i < 8; ++i) o[i] = m[i];
}

__global__ void k_ctl_init(TrajCtl* ctl, uint64_t* bits, int nwords, uint32_t* guards, int gwords, int64_t slots,
                           uint64_t seed, int64_t shot_begin, const uint64_t* rng_init, int dedup) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= slots) return;
  TrajCtl c;
  if (rng_init && s == 0) {
    for (int w = 0; w < 4; ++w) c.rng[w] = rng_init[w];
  } else {
    rng_for_shot(c.rng, seed, (uint64_t)(shot_begin + s));
  }
  c.frame = 0;
  c.kmask = 0;
  c.kval = 0;
  c.sre = 1.0;
  c.sim = 0.0;
  c.pending = 0;
  c.status = 0;
  c.depth = 0;
  c.active = 0;
  c.draws = 0;
  c.pad = 0;
  c.gates = 0;
  c.hist = 0;
  c.rep = dedup ? 0 : (int32_t)s;  // identical (empty) histories share slot 0's state
  c.pad2 = 0;
  ctl[s] = c;
  for (int w = 0; w < nwords; ++w) bits[s * nwords + w] = 0;
  for (int w = 0; w < gwords; ++w) guards[s * gwords + w] = 0;
}

template <typename R>
__global__ void __launch_bounds__(kPT) k_pass(StreamArgs a, PassDesc pd) {
  using A = typename Amp<R>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int k = pd.k;
  const int TL = 1 << k;
  A* tile = reinterpret_cast<A*>(smem_raw);
  uint64_t* hi_off = reinterpret_cast<uint64_t*>(smem_raw + sizeof(A) * TL);
  double* red = reinterpret_cast<double*>(hi_off + (TL >> pd.lowq));

  const int tid = threadIdx.x;
  const int64_t slot = blockIdx.y;
  const TrajCtl* c = a.ctl + slot;
  if (c->status || c->rep != slot) return;  // dead, or its state lives in its representative
  const int n = a.n;
  const uint64_t qmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t S = pd.smask;
  const uint64_t F = c->frame & ~pd.clear_before;
  const bool pending = pd.prologue && c->pending;
  const uint64_t Kp = c->kmask, Vp = c->kval;
  const R sre = (R)c->sre, sim = (R)c->sim;

  const uint64_t base_phys = pdep64((uint64_t)blockIdx.x, ~S & qmask);
  const uint64_t base_log = base_phys ^ (F & ~S);
  uint32_t fl = 0;
  for (int j = 0; j < k; ++j)
    if ((F >> pd.sq[j]) & 1) fl |= 1u << j;
  const uint64_t lowm = (1ull << pd.lowq) - 1;
  const uint64_t shi = S & ~lowm;
  for (int h = tid; h < (TL >> pd.lowq); h += kPT) hi_off[h] = pdep64((uint64_t)h, shi);
  __syncthreads();

  A* st = reinterpret_cast<A*>(a.state) + (slot << n);
  // ---- prologue: gather ----
  for (int l = tid; l < TL; l += kPT) {
    uint64_t p = base_phys | ((uint64_t)l & lowm) | hi_off[l >> pd.lowq];
    A v;
    if (pd.init_zero) {
      v = mk<R>(p == 0 ? (R)1 : (R)0, (R)0);
    } else {
      v = st[p];
    }
    if (pending) {
      if ((p & Kp) != Vp) v = mk<R>(0, 0);
      else v = mk<R>(fma(sre, v.x, -sim * v.y), fma(sre, v.y, sim * v.x));
    }
    tile[l ^ fl] = v;
  }
  __syncthreads();

  // ---- body: fused gates ----
  const uint32_t* gw = a.guards + slot * a.gwords;
  const double* mats = a.mats + slot * a.mat_stride;
  for (int gi = 0; gi < pd.gate_count; ++gi) {
    const PassGate g = a.gates[pd.gate_begin + gi];
    if (g.guard >= 0 && !((gw[g.guard >> 5] >> (g.guard & 31)) & 1u)) continue;
    if ((base_log & g.gcm) != g.gcv) continue;
    double m[8];
    const double* src = mats + (int64_t)g.mat * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = src[j];
    switch (g.gclass) {
      case GC_DIAG_GLOBAL: {
        int b = (int)((base_log >> g.gq) & 1);
        if (!b && g.diag_one0) break;
        R dr = (R)(b ? m[6] : m[0]), di = (R)(b ? m[7] : m[1]);
        for (int l = tid; l < TL; l += kPT) {
          if (((uint32_t)l & g.lcm) != g.lcv) continue;
          A v = tile[l];
          tile[l] = cmul<R>(dr, di, v);
        }
      } break;
      case GC_DIAG: {
        for (int l = tid; l < TL; l += kPT) {
          if (((uint32_t)l & g.lcm) != g.lcv) continue;
          int b = (l >> g.lt) & 1;
          if (!b && g.diag_one0) continue;
          A v = tile[l];
          tile[l] = b ? cmul<R>((R)m[6], (R)m[7], v) : cmul<R>((R)m[0], (R)m[1], v);
        }
      } break;
      case GC_SWAP: {
        int lo = g.lt < g.lt2 ? g.lt : g.lt2, hi = g.lt < g.lt2 ? g.lt2 : g.lt;
        for (int qd = tid; qd < (TL >> 2); qd += kPT) {
          uint32_t base = (uint32_t)insert_zero(insert_zero((uint64_t)qd, lo), hi);
          if ((base & g.lcm) != g.lcv) continue;
          uint32_t la = base | (1u << g.lt), lb = base | (1u << g.lt2);
          A x = tile[la];
          tile[la] = tile[lb];
          tile[lb] = x;
        }
      } break;
      default: {
        for (int pi = tid; pi < (TL >> 1); pi += kPT) {
          uint32_t l0 = (uint32_t)insert_zero((uint64_t)pi, g.lt);
          if ((l0 & g.lcm) != g.lcv) continue;
          uint32_t l1 = l0 | (1u << g.lt);
          A a0 = tile[l0], a1 = tile[l1];
          apply_pair<R>(g.gclass, m, a0, a1);
          tile[l0] = a0;
          tile[l1] = a1;
        }
      } break;
    }
    __syncthreads();
  }

  // ---- epilogue: marginal of the measured qubits ----
  if (pd.epi) {
    const int ml = pd.m_local;
    const int nb = 1 << ml;
    uint32_t mlm = 0;
    for (int j = 0; j < ml; ++j) mlm |= 1u << pd.mloc[j];
    // bin bit j <-> local position mloc[j] (M order)
    const uint32_t free_mask = ((uint32_t)TL - 1) & ~mlm;
    const int members = TL >> ml;
    const uint64_t t_log = pext64(base_log, ~S & qmask);
    double* out = a.partial + slot * a.partial_stride + (int64_t)t_log * nb;
    if (nb <= kPT) {
      const int tp = kPT / nb;
      const int b = tid / tp, j = tid % tp;
      uint32_t bpos = 0;
      for (int jj = 0; jj < ml; ++jj)
        if ((b >> jj) & 1) bpos |= 1u << pd.mloc[jj];
      double s = 0.0;
      for (int r = j; r < members; r += tp) s += norm2<R>(tile[(uint32_t)pdep64((uint64_t)r, free_mask) | bpos]);
      red[tid] = s;
      __syncthreads();
      if (j == 0) {
        double tot = 0.0;
        for (int jj = 0; jj < tp; ++jj) tot += red[b * tp + jj];
        out[b] = tot;
      }
    } else {
      for (int b = tid; b < nb; b += kPT) {
        uint32_t bpos = 0;
        for (int jj = 0; jj < ml; ++jj)
          if ((b >> jj) & 1) bpos |= 1u << pd.mloc[jj];
        double s = 0.0;
        for (int r = 0; r < members; ++r) s += norm2<R>(tile[(uint32_t)pdep64((uint64_t)r, free_mask) | bpos]);
        out[b] = s;
      }
    }
  }

  // ---- scatter back (logical order on S: the frame on S is cleared) ----
  for (int l = tid; l < TL; l += kPT) {
    uint64_t p = base_phys | ((uint64_t)l & lowm) | hi_off[l >> pd.lowq];
    st[p] = tile[l];
  }
}


// complex helpers on (re, im) doubles for the decide kernel
struct Cd {
  double r, i;
};
__device__ __forceinline__ Cd cmuld(Cd a, Cd b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }

__global__ void __launch_bounds__(kDT) k_decide(StreamArgs a, RegionDesc rd) {
  __shared__ double marg[1 << kMaxMeasureRegion];
  const int64_t slot = blockIdx.x;
  TrajCtl* cp = a.ctl + slot;
  if (cp->status) return;
  const int tid = threadIdx.x;
  const int nbins = 1 << rd.mcount;
  if (rd.has_marginal) {
    const int nbl = 1 << rd.m_local;
    const int ntl = a.ntiles_log2;
    // the marginal of this trajectory's state was accumulated by its representative
    const double* part = a.partial + (int64_t)cp->rep * a.partial_stride;
    uint64_t gm = 0;
    for (int j = 0; j < rd.mcount; ++j)
      if (rd.mtile_bit[j] >= 0) gm |= 1ull << rd.mtile_bit[j];
    const uint64_t free_t = (((ntl >= 64) ? ~0ull : ((1ull << ntl) - 1))) & ~gm;
    const int64_t nfree = 1ll << (ntl - __popcll(gm));
    for (int b = tid; b < nbins; b += kDT) {
      int lb = 0;
      uint64_t gv = 0;
      for (int j = 0; j < rd.mcount; ++j) {
        int bit = (b >> j) & 1;
        if (rd.mloc_bit[j] >= 0) lb |= bit << rd.mloc_bit[j];
        else gv |= (uint64_t)bit << rd.mtile_bit[j];
      }
      // sum over the tiles in increasing tile order (fixed: run-to-run and batch
      // invariant); loads issued 8 ahead of the sequential adds
      double s = 0.0;
      int64_t tt = 0;
      if (gm == 0) {  // every measured qubit inside the tile: the tiles are 0 .. nfree-1
        const double* pp = part + lb;
        for (; tt + 8 <= nfree; tt += 8) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = pp[(tt + u) * nbl];
#pragma unroll
          for (int u = 0; u < 8; ++u) s += x[u];
        }
      } else {
        for (; tt + 8 <= nfree; tt += 8) {
          double x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = part[(int64_t)(pdep64((uint64_t)(tt + u), free_t) | gv) * nbl + lb];
#pragma unroll
          for (int u = 0; u < 8; ++u) s += x[u];
        }
      }
      for (; tt < nfree; ++tt) s += part[(int64_t)(pdep64((uint64_t)tt, free_t) | gv) * nbl + lb];
      marg[b] = s;
    }
  }
  __syncthreads();
  if (tid != 0) return;

  TrajCtl c = *cp;
  uint64_t* bits = a.bits + slot * a.nwords;
  uint32_t* gw = a.guards + slot * a.gwords;
  const uint64_t F = c.frame & ~rd.clear_mask;
  uint64_t K = 0, V = 0, Fp = 0;  // M-index space
  Cd S = {1.0, 0.0};
  bool collapsed = false;
  int depth = c.depth, active = c.active;
  const double* mats = a.mats + slot * a.mat_stride;
  const double tol = a.c64 ? 1e-6 : 1e-12;
  int ntrace = (slot == 0 && a.ntrace_out) ? *a.ntrace_out : 0;
  for (int oi = rd.op_begin; oi < rd.op_end; ++oi) {
    const DevOp& op = a.region_ops[oi];
    if (op.kind == QSB_OP_IF) {
      bool act = active == depth;
      bool taken = act && pred_eval(bits, op.pred_bit, op.pred_width, op.pred_cmp, op.pred_rhs);
      uint32_t tb = 1u << (op.g_then & 31), eb = 1u << (op.g_else & 31);
      gw[op.g_then >> 5] = (act && taken) ? (gw[op.g_then >> 5] | tb) : (gw[op.g_then >> 5] & ~tb);
      gw[op.g_else >> 5] = (act && !taken) ? (gw[op.g_else >> 5] | eb) : (gw[op.g_else >> 5] & ~eb);
      if (act && slot == 0 && a.trace_out) {
        if (ntrace < a.max_trace) {
          int64_t* e = a.trace_out + (int64_t)ntrace * (2 + a.nwords);
          e[0] = op.op_index;
          e[1] = taken ? 1 : 0;
          for (int w = 0; w < a.nwords; ++w) e[2 + w] = (int64_t)bits[w];
        }
        ntrace++;
      }
      depth++;
      if (taken) active = depth;
      continue;
    }
    if (op.kind == QSB_OP_ELSE) {
      if (active == depth) active = depth - 1;
      else if (active == depth - 1) active = depth;
      continue;
    }
    if (op.kind == QSB_OP_ENDIF) {
      if (active == depth) active--;
      depth--;
      continue;
    }
    if (active != depth) continue;
    const int j = op.mj;
    if (op.kind == QSB_OP_GATE) {  // Pauli / phase on collapsed qubits
      const uint64_t cur = V ^ Fp;
      if ((cur & op.mcm) != op.mcv) continue;
      const int cv = (int)((cur >> j) & 1);
      const double* m = mats + (int64_t)op.mat * 8;
      if (op.gclass == GC_XPERM) {
        Fp ^= 1ull << j;
      } else if (op.gclass == GC_ANTI) {
        Cd ph = cv ? Cd{m[2], m[3]} : Cd{m[4], m[5]};
        S = cmuld(S, ph);
        Fp ^= 1ull << j;
      } else {
        Cd ph = cv ? Cd{m[6], m[7]} : Cd{m[0], m[1]};
        S = cmuld(S, ph);
      }
      c.gates++;
      continue;
    }
    // MEASURE / RESET
    double p1 = 0.0;
    for (int b = 0; b < nbins; ++b)
      if ((((uint64_t)b & K) == V) && ((((uint64_t)b ^ Fp) >> j) & 1)) p1 += marg[b];
    p1 *= S.r * S.r + S.i * S.i;
    double u;
    if (a.predrawn) {
      if (c.draws >= a.predrawn_stride) {
        c.status = QSB_ERR_PREDRAWN;
        break;
      }
      u = a.predrawn[(a.predrawn_slot0 + slot) * a.predrawn_stride + c.draws];
    } else {
      u = rng_uniform(c.rng);
    }
    c.draws++;
    int outcome = u < p1 ? 1 : 0;
    if (a.hbits && c.draws <= 64 * a.hwords)  // exact outcome history (dedup verification)
      a.hbits[slot * a.hwords + ((c.draws - 1) >> 6)] |= (uint64_t)outcome << ((c.draws - 1) & 63);
    double pout = outcome ? p1 : 1.0 - p1;
    if (fabs(u - p1) < tol && a.tie_count) atomicAdd(a.tie_count, 1ull);
    if (pout < 1e-15) {
      c.status = QSB_ERR_DEGENERATE;
      break;
    }
    double s = 1.0 / sqrt(pout);
    {  // history hash: equal histories <=> equal states (deduplication key)
      uint64_t hx = c.hist + 0x9E3779B97F4A7C15ull * (uint64_t)(2 * op.op_index + outcome + 1);
      c.hist = splitmix_next(hx);
    }
    K |= 1ull << j;
    V = (V & ~(1ull << j)) | ((uint64_t)(outcome ^ (int)((Fp >> j) & 1)) << j);
    S.r *= s;
    S.i *= s;
    collapsed = true;
    if (op.kind == QSB_OP_MEASURE) {
      int f = op.bit;
      bits[f >> 6] = (bits[f >> 6] & ~(1ull << (f & 63))) | ((uint64_t)outcome << (f & 63));
    } else if (outcome) {
      Fp ^= 1ull << j;
    }
  }
  if (slot == 0 && a.ntrace_out) *a.ntrace_out = ntrace;
  // back to qubit masks; projection expressed on physical indices
  uint64_t Kq = 0, Vq = 0, Fq = 0;
  for (int j = 0; j < rd.mcount; ++j) {
    uint64_t qb = 1ull << rd.mq[j];
    if ((K >> j) & 1) Kq |= qb;
    if ((V >> j) & 1) Vq |= qb;
    if ((Fp >> j) & 1) Fq |= qb;
  }
  c.frame = F ^ Fq;
  c.kmask = Kq;
  c.kval = Vq ^ (F & Kq);
  c.sre = S.r;
  c.sim = S.i;
  c.pending = collapsed ? 1 : 0;
  c.depth = depth;
  c.active = active;
  *cp = c;
}

// ---- branch-history deduplication ------------------------
// The state is a deterministic function of the executed outcome history, so slots with
// equal histories share one state buffer.  After each decide: every slot's new
// representative is the lowest alive slot with the same history hash; a slot that
// becomes a representative while its state lived elsewhere copies the (pre-collapse)
// buffer of its old representative, then applies its own collapse in the next pass.
// The arithmetic per trajectory is unchanged, so results are bit-identical.
// One thread per slot scans the lower slots for the first one with its history; the
// candidates' keys (alive, draws, hash) are staged through shared memory a tile of
// kRegroupTile slots at a time (one coalesced load per tile for the whole block instead
// of three dependent global loads per candidate per thread), and the block stops as soon
// as every thread has its representative.  Same result as the plain scan: the lowest
// alive slot with the same exact history.
constexpr int kRegroupTile = 256;

__global__ void __launch_bounds__(kRegroupTile) k_dedup_regroup(StreamArgs a, int32_t* new_rep, int32_t* copy_src) {
  __shared__ uint64_t kh[kRegroupTile];
  __shared__ int32_t kd[kRegroupTile];
  const int64_t s = blockIdx.x * (int64_t)kRegroupTile + threadIdx.x;
  const bool valid = s < a.slots;
  uint64_t hist = 0;
  int32_t draws = 0, status = 1, rep = 0;
  if (valid) {
    const TrajCtl& c = a.ctl[s];
    hist = c.hist;
    draws = c.draws;
    status = c.status;
    rep = c.rep;
  }
  int32_t r = (int32_t)s;
  bool done = !valid || status != 0;
  const int64_t smax = blockIdx.x * (int64_t)kRegroupTile;  // candidates below the block (own tile: below)
  for (int64_t t0 = 0; t0 <= smax; t0 += kRegroupTile) {
    if (__syncthreads_and(done)) break;
    const int64_t t = t0 + threadIdx.x;
    const bool alive = t < a.slots && a.ctl[t].status == 0;
    kh[threadIdx.x] = alive ? a.ctl[t].hist : 0;
    kd[threadIdx.x] = alive ? a.ctl[t].draws : -1;  // draws >= 0: a dead slot never matches
    __syncthreads();
    if (!done) {
      const int64_t rem = s - t0;  // candidates t < s only
      const int lim = rem < kRegroupTile ? (int)rem : kRegroupTile;
      for (int j = 0; j < lim; ++j) {
        if (kd[j] != draws || kh[j] != hist) continue;
        // the 64-bit hash is only a filter: merge on the exact outcome history
        const int64_t u = t0 + j;
        bool same = true;
        for (int w = 0; w < a.hwords && same; ++w) same = a.hbits[u * a.hwords + w] == a.hbits[s * a.hwords + w];
        if (same) {
          r = (int32_t)u;
          done = true;
          break;
        }
      }
    }
    __syncthreads();
  }
  if (!valid) return;
  new_rep[s] = r;
  copy_src[s] = (r == s && rep != s && status == 0) ? rep : -1;
}

__global__ void k_dedup_copy(StreamArgs a, const int32_t* copy_src, int64_t amp_bytes) {
  const int64_t s = blockIdx.y;
  const int32_t src = copy_src[s];
  if (src < 0) return;
  const int64_t words = (amp_bytes << a.n) / 16;
  const int4* from = reinterpret_cast<const int4*>(reinterpret_cast<const char*>(a.state) + (int64_t)src * (amp_bytes << a.n));
  int4* to = reinterpret_cast<int4*>(reinterpret_cast<char*>(a.state) + s * (amp_bytes << a.n));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    to[i] = from[i];
}

__global__ void k_dedup_init_rep(StreamArgs a, int32_t* new_rep) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < a.slots) new_rep[s] = a.ctl[s].rep;
}

// split != null (deferred copies): the representatives are also listed apart -- split[0 ..)
// the new branches (copy_src >= 0: their first pass reads the old representative's
// buffer), split[slots ..) the rest, counts at split[2 slots], split[2 slots + 1]
__global__ void k_dedup_commit(StreamArgs a, const int32_t* new_rep, int32_t* active, int32_t* nactive,
                               const int32_t* copy_src, int32_t* split) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= a.slots) return;
  const int32_t r = new_rep[s];
  a.ctl[s].rep = r;
  if (r == s && a.ctl[s].status == 0) {
    active[atomicAdd(nactive, 1)] = (int32_t)s;  // order is irrelevant
    if (split) {
      const bool branch = copy_src[s] >= 0;
      int32_t* cnt = split + 2 * a.slots + (branch ? 0 : 1);
      split[(branch ? 0 : a.slots) + atomicAdd(cnt, 1)] = (int32_t)s;
    }
  }
}

__global__ void k_count(StreamArgs a, const int32_t* guard_gates, int nguards, int64_t unguarded,
                        unsigned long long* out) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= a.slots) return;
  int64_t tot = unguarded + a.ctl[s].gates;
  const uint32_t* gw = a.guards + s * a.gwords;
  for (int g = 0; g < nguards; ++g)
    if ((gw[g >> 5] >> (g & 31)) & 1u) tot += guard_gates[g];
  atomicAdd(out, (unsigned long long)tot);
}

template <typename R>
__global__ void k_finalize(StreamArgs a, typename Amp<R>::T* out, uint64_t clear, int consumed, int64_t slot) {
  using A = typename Amp<R>::T;
  TrajCtl c = a.ctl[slot];
  c.frame &= ~clear;
  if (consumed) c.pending = 0;
  const int64_t N = 1ll << a.n;
  // the slot's state lives in its representative's buffer (history dedup; rep == slot without)
  const A* st = reinterpret_cast<const A*>(a.state) + (int64_t)c.rep * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t p = (uint64_t)i ^ c.frame;
    A v = st[p];
    if (c.pending) {
      if ((p & c.kmask) != c.kval) v = mk<R>(0, 0);
      else v = mk<R>(fma((R)c.sre, v.x, -(R)c.sim * v.y), fma((R)c.sre, v.y, (R)c.sim * v.x));
    }
    out[i] = v;
  }
}

}  // namespace

void launch_mats_prep(const MatSrc* src, int nmat, const double* params, int nparams, int64_t slots, double* mats_out,
                      cudaStream_t s) {
  if (nmat <= 0 || slots <= 0) return;
  dim3 grid((unsigned)((nmat + 127) / 128), (unsigned)slots);
  k_mats_prep<<<grid, 128, 0, s>>>(src, nmat, params, nparams, mats_out);
}

void launch_ctl_init(TrajCtl* ctl, uint64_t* bits, int nwords, uint32_t* guards, int gwords, int64_t slots,
                     uint64_t seed, int64_t shot_begin, const uint64_t* rng_init, int dedup, cudaStream_t s) {
  k_ctl_init<<<(unsigned)((slots + 127) / 128), 128, 0, s>>>(ctl, bits, nwords, guards, gwords, slots, seed,
                                                            shot_begin, rng_init, dedup);
}

__global__ void k_accum_physical(const int32_t* nactive, double flops, double bytes, double* phys) {
  phys[0] += bytes * (double)*nactive;  // single thread: deterministic
  phys[1] += flops * (double)*nactive;
}

// zero the state (and the epilogue partials) of the active slots: the passes from the
// |0...0> start then run only the items not known to be zero (PassDesc::zero_tid)
__global__ void k_zero_slots(StreamArgs a, int64_t amp_words, int zero_partials) {
  const int64_t n_act = a.active ? *a.nactive : a.slots;
  for (int64_t si = blockIdx.y; si < n_act; si += gridDim.y) {
    const int64_t slot = a.active ? a.active[si] : si;
    int4* st = reinterpret_cast<int4*>(a.state) + slot * amp_words;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < amp_words; i += (int64_t)gridDim.x * blockDim.x)
      st[i] = make_int4(0, 0, 0, 0);
    if (zero_partials) {
      double* pp = a.partial + slot * a.partial_stride;
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.partial_stride;
           i += (int64_t)gridDim.x * blockDim.x)
        pp[i] = 0.0;
    }
  }
}

// the amplitudes the pending collapse rejects on the qubits M, per active slot: zero
// stores of the known-zero amplitudes no pass has stored (end of a run, or before a pass
// that reads every amplitude)
__global__ void k_zero_projected(StreamArgs a, uint64_t M, int64_t amp_words, int amps_per_word) {
  const int64_t n_act = a.active ? *a.nactive : a.slots;
  for (int64_t si = blockIdx.y; si < n_act; si += gridDim.y) {
    const int64_t slot = a.active ? a.active[si] : si;
    const TrajCtl& c = a.ctl[slot];
    if (c.status != 0 || !c.pending) continue;
    const uint64_t V = c.kval & M;
    int4* st = reinterpret_cast<int4*>(a.state) + slot * amp_words;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < amp_words; i += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t p = (uint64_t)i * (uint64_t)amps_per_word;  // M never holds bit 0 (low run in the tile)
      if ((p & M) != V) st[i] = make_int4(0, 0, 0, 0);
    }
  }
}

void launch_zero_projected(const StreamArgs& a, int c64, uint64_t M, cudaStream_t s) {
  const int64_t words = ((int64_t)(c64 ? 8 : 16) << a.n) / 16;
  const unsigned gx = (unsigned)std::min<int64_t>(std::max<int64_t>(1, words / 1024), 64);
  const unsigned gy = (unsigned)std::min<int64_t>(a.slots, 65535);
  k_zero_projected<<<dim3(gx, gy), 256, 0, s>>>(a, M, words, c64 ? 2 : 1);
}

void launch_zero_slots(const StreamArgs& a, int c64, int zero_partials, cudaStream_t s) {
  const int64_t words = ((int64_t)(c64 ? 8 : 16) << a.n) / 16;
  const unsigned gx = (unsigned)std::min<int64_t>(std::max<int64_t>(1, words / 1024), 64);
  const unsigned gy = (unsigned)std::min<int64_t>(a.slots, 65535);
  k_zero_slots<<<dim3(gx, gy), 256, 0, s>>>(a, words, zero_partials);
}

void launch_accum_physical(const int32_t* nactive, double flops_per_state, double bytes_per_state, double* phys,
                           cudaStream_t s) {
  k_accum_physical<<<1, 1, 0, s>>>(nactive, flops_per_state, bytes_per_state, phys);
}

void launch_dedup(const StreamArgs& a, int32_t* new_rep, int32_t* copy_src, int32_t* active, int32_t* nactive,
                  int c64, bool regroup, int32_t* split, cudaStream_t s) {
  const unsigned g = (unsigned)((a.slots + 127) / 128);
  if (regroup) {
    k_dedup_regroup<<<(unsigned)((a.slots + kRegroupTile - 1) / kRegroupTile), kRegroupTile, 0, s>>>(a, new_rep,
                                                                                                   copy_src);
    if (!split) {  // copies now (no pass follows that could read the old buffers)
      const int64_t amp = c64 ? 8 : 16;
      const int64_t words = (amp << a.n) / 16;
      unsigned chunks = (unsigned)std::min<int64_t>(std::max<int64_t>(1, words / 2048), 64);
      k_dedup_copy<<<dim3(chunks, (unsigned)a.slots), 256, 0, s>>>(a, copy_src, amp);
    }
  } else {  // initial grouping from ctl.rep
    k_dedup_init_rep<<<g, 128, 0, s>>>(a, new_rep);
    split = nullptr;
  }
  cudaMemsetAsync(nactive, 0, sizeof(int32_t), s);
  if (split) cudaMemsetAsync(split + 2 * a.slots, 0, 2 * sizeof(int32_t), s);
  k_dedup_commit<<<g, 128, 0, s>>>(a, new_rep, active, nactive, copy_src, split);
}

static size_t pass_smem(int c64, const PassDesc& pd) {
  size_t amp = c64 ? sizeof(float2) : sizeof(double2);
  return (amp << pd.k) + (sizeof(uint64_t) << (pd.k - pd.lowq)) + sizeof(double) * kPT;
}

cudaError_t launch_pass(const StreamArgs& a, const PassDesc& pd, cudaStream_t s) {
  size_t smem = pass_smem(a.c64, pd);
  dim3 grid((unsigned)(1ull << (a.n - pd.k)), (unsigned)a.slots);
  cudaError_t e;
  if (a.phases && pd.rb > 0)
    return launch_pass_reg(a, pd, s);
  if (a.c64) {
    e = cudaFuncSetAttribute(k_pass<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_pass<float><<<grid, kPT, smem, s>>>(a, pd);
  } else {
    e = cudaFuncSetAttribute(k_pass<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_pass<double><<<grid, kPT, smem, s>>>(a, pd);
  }
  return cudaGetLastError();
}

cudaError_t launch_decide(const StreamArgs& a, const RegionDesc& rd, cudaStream_t s) {
  k_decide<<<(unsigned)a.slots, kDT, 0, s>>>(a, rd);
  return cudaGetLastError();
}

void launch_count_gates(const StreamArgs& a, const int32_t* guard_gates, int nguards, int64_t unguarded,
                        unsigned long long* out, cudaStream_t s) {
  k_count<<<(unsigned)((a.slots + 127) / 128), 128, 0, s>>>(a, guard_gates, nguards, unguarded, out);
}

void launch_finalize(const StreamArgs& a, void* out, uint64_t clear, int consumed, cudaStream_t s, int64_t slot) {
  int64_t N = 1ll << a.n;
  unsigned g = (unsigned)((N + 255) / 256);
  if (g > 148 * 32) g = 148 * 32;
  if (a.c64) k_finalize<float><<<g, 256, 0, s>>>(a, (float2*)out, clear, consumed, slot);
  else k_finalize<double><<<g, 256, 0, s>>>(a, (double2*)out, clear, consumed, slot);
}

}  // namespace qsb
