// Tape analysis (Kernel IR -> flattened device program) and the fused-pass planner.
//
// Reference semantics preserved here:
//   * _needs_trajectories (sim.py:322-335): top-level scan only.
//   * _scan_static (sim.py:394-399): statevector refuses any top-level Measure /
//     CondBlock / Reset.
//   * CondBlock evaluates its predicate once at entry (sim.py:297): IF ops define a
//     then-guard and an else-guard bit per trajectory, evaluated once.
//
// Streaming plan (state in HBM):
//   gate region   -> greedy fused passes over k-qubit tiles (targets must be in the
//                    tile; controls and diagonal targets may live outside it)
//   measure region-> one "decide" step per trajectory that resolves every measure,
//                    reset, predicate and collapsed-qubit Pauli/phase gate of the
//                    region from the marginal of the measured qubits, computed by
//                    the epilogue of the preceding pass; the collapse itself is
//                    applied by the prologue of the next pass.
#include "qsb_plan.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <complex>
#include <map>
#include <cmath>
#include <functional>
#include <sstream>

namespace qsb {

static int popc(uint64_t v) { return __builtin_popcountll(v); }

// Swizzle vectors: tile position p >= sb contributes V[p] to the low sb slot bits.
// Every nonzero vector appears at most twice (sb = 3) / once (sb = 4), so any set of
// >= 7 (resp. >= 8) thread-mapped positions spans all sb dimensions and a phase can
// always give its 2^sb consecutive threads distinct bank groups.
static const uint32_t kV3[16] = {1, 2, 4, 3, 5, 6, 7, 1, 2, 4, 3, 5, 6, 7, 1, 2};
static const uint32_t kV4[16] = {1, 2, 4, 8, 3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 1};

int swizzle_bits(int c64) { return c64 ? 4 : 3; }

uint32_t swizzle_hi(uint32_t hi, int sb) {
  const uint32_t* V = sb == 3 ? kV3 : kV4;
  uint32_t s = 0;
  for (int p = sb; hi; ++p, hi >>= 1)
    if (hi & 1) s ^= V[p];
  return s;
}

static uint32_t swz_slot(uint32_t l, int sb) { return l ^ swizzle_hi(l >> sb, sb); }
static uint32_t swz_vec(int p, int sb) { return p < sb ? (1u << p) : (sb == 3 ? kV3[p] : kV4[p]); }

void tile_mapping(const int* rpos, int rb, int k, int sb, int8_t* tpos, uint16_t* soff, uint32_t avoid) {
  uint32_t R = 0;
  for (int b = 0; b < rb; ++b) R |= 1u << rpos[b];
  // thread positions: first sb positions with independent swizzle vectors, so that
  // 2^sb consecutive threads (the lanes one shared-memory wavefront serves: 8 for 16-byte,
  // 16 for 8-byte amplitudes) hit distinct bank groups.  Positions in `avoid` (thread
  // controls of the phase's X gates, which the generator folds into a per-thread XOR of
  // the slot: an XOR that differs inside a wavefront's lanes would break the distinctness)
  // are taken for those first sb slots only when nothing else is independent.
  std::vector<int> tp, others;
  uint32_t basis[8] = {0};
  auto reduce = [&](uint32_t v) {
    for (int b = sb - 1; b >= 0 && v; --b)
      if (v >> b & 1) {
        if (basis[b]) v ^= basis[b];
        else return v;
      }
    return v;
  };
  auto insert = [&](uint32_t v) {
    for (int b = sb - 1; b >= 0; --b)
      if (v >> b & 1) {
        basis[b] = v;
        return;
      }
  };
  std::vector<char> used(k, 0);
  for (int pass = 0; pass < 2; ++pass)
    for (int p = 0; p < k && (int)tp.size() < sb; ++p) {
      if ((R >> p & 1) || used[p] || ((avoid >> p & 1) && pass == 0)) continue;
      const uint32_t v = reduce(swz_vec(p, sb));
      if (v) {
        insert(v);
        tp.push_back(p);
        used[p] = 1;
      }
    }
  for (int p = 0; p < k; ++p)
    if (!(R >> p & 1) && !used[p]) others.push_back(p);
  for (int p : others) tp.push_back(p);
  for (int i = 0; i < k - rb; ++i) tpos[i] = (int8_t)tp[i];
  for (int j = 0; j < (1 << rb); ++j) {
    uint32_t off = 0;
    for (int b = 0; b < rb; ++b)
      if (j >> b & 1) off |= 1u << rpos[b];
    soff[j] = (uint16_t)swz_slot(off, sb);
  }
}

static int gate_class_of(int base) {
  switch (base) {
    case QSB_G_X: return GC_XPERM;
    case QSB_G_Y: return GC_ANTI;
    case QSB_G_Z: case QSB_G_S: case QSB_G_T: case QSB_G_RZ: case QSB_G_P: return GC_DIAG;
    case QSB_G_SWAP: return GC_SWAP;
    default: return GC_DENSE;
  }
}

std::string analyze_tape(const qsb_op* ops, int nops, int n, int nbits, int nparams, TapeInfo& out) {
  std::ostringstream err;
  if (n < 0 || n > kMaxQubits) {
    err << "qubit count " << n << " outside [0, " << kMaxQubits << "]";
    return err.str();
  }
  if (nbits < 0 || nparams < 0 || nops < 0) return "negative size";
  out = TapeInfo();
  out.n = n;
  out.nbits = nbits;
  out.nwords = std::max(1, (nbits + 63) / 64);
  out.nparams = nparams;
  const uint64_t qmask = n >= 64 ? ~0ull : ((1ull << n) - 1);
  struct Open { int g_then, g_else; bool else_seen; };
  std::vector<Open> stack;
  std::vector<int> path;
  int g = 0;
  uint64_t measured_top = 0;
  for (int i = 0; i < nops; ++i) {
    const qsb_op& o = ops[i];
    DevOp d{};
    d.kind = o.kind;
    d.op_index = i;
    d.guard = path.empty() ? -1 : path.back();
    d.mat = -1;
    d.mj = -1;
    const bool top = stack.empty();
    switch (o.kind) {
      case QSB_OP_GATE: {
        if (o.base < 0 || o.base > QSB_G_SWAP) { err << "op " << i << ": bad gate base " << o.base; return err.str(); }
        int nt = o.base == QSB_G_SWAP ? 2 : 1;
        if (o.ntargets != nt) { err << "op " << i << ": gate takes " << nt << " target(s)"; return err.str(); }
        uint64_t tm = 0;
        for (int j = 0; j < nt; ++j) {
          if (o.target[j] < 0 || o.target[j] >= n) { err << "op " << i << ": target out of range"; return err.str(); }
          if (tm & (1ull << o.target[j])) { err << "op " << i << ": repeated target"; return err.str(); }
          tm |= 1ull << o.target[j];
        }
        if ((o.ctrl_mask & ~qmask) || (o.ctrl_mask & tm) || (o.ctrl_val & ~o.ctrl_mask)) {
          err << "op " << i << ": bad control mask";
          return err.str();
        }
        d.gclass = gate_class_of(o.base);
        d.t0 = o.target[0];
        d.t1 = nt == 2 ? o.target[1] : -1;
        d.cm = o.ctrl_mask;
        d.cv = o.ctrl_val;
        d.diag_one0 = (o.base == QSB_G_Z || o.base == QSB_G_S || o.base == QSB_G_T || o.base == QSB_G_P) ? 1 : 0;
        MatSrc m{};
        m.base = o.base;
        m.adjoint = o.adjoint ? 1 : 0;
        m.has_matrix = o.has_matrix ? 1 : 0;
        for (int j = 0; j < 3; ++j) {
          m.slot[j] = o.angle_slot[j];
          m.angle[j] = o.angle[j];
          if (o.angle_slot[j] >= 0) {
            if (o.angle_slot[j] >= nparams) { err << "op " << i << ": parameter slot out of range"; return err.str(); }
            m.has_matrix = 0;
            out.has_param_angles = true;
          }
        }
        for (int j = 0; j < 8; ++j) m.mat[j] = o.mat[j];
        d.mat = (int)out.mats.size();
        out.mats.push_back(m);
        if (top && measured_top) out.needs_trajectories = true;
      } break;
      case QSB_OP_MEASURE:
      case QSB_OP_RESET: {
        if (o.qubit < 0 || o.qubit >= n) { err << "op " << i << ": qubit out of range"; return err.str(); }
        d.qubit = o.qubit;
        if (o.kind == QSB_OP_MEASURE) {
          if (o.bit < 0 || o.bit >= nbits) { err << "op " << i << ": classical bit out of range"; return err.str(); }
          d.bit = o.bit;
        }
        out.draws_max++;
        if (top) {
          out.top_level_dynamic = true;
          if (o.kind == QSB_OP_RESET) out.needs_trajectories = true;
          else {
            if (measured_top & (1ull << o.qubit)) out.needs_trajectories = true;
            measured_top |= 1ull << o.qubit;
            out.top_measures.push_back((int)out.dev.size());
          }
        }
      } break;
      case QSB_OP_IF: {
        if (o.pred_width < 1 || o.pred_width > 64 || o.pred_bit < 0 || o.pred_bit + o.pred_width > nbits ||
            o.pred_cmp < 0 || o.pred_cmp > QSB_CMP_TRUTHY) {
          err << "op " << i << ": bad predicate";
          return err.str();
        }
        if (top) { out.needs_trajectories = true; out.top_level_dynamic = true; }
        d.pred_cmp = o.pred_cmp;
        d.pred_bit = o.pred_bit;
        d.pred_width = o.pred_width;
        d.pred_rhs = o.pred_rhs;
        d.g_then = g++;
        d.g_else = g++;
        stack.push_back({d.g_then, d.g_else, false});
        path.push_back(d.g_then);
      } break;
      case QSB_OP_ELSE: {
        if (stack.empty() || stack.back().else_seen) { err << "op " << i << ": ELSE without IF"; return err.str(); }
        stack.back().else_seen = true;
        d.g_then = stack.back().g_then;
        d.g_else = stack.back().g_else;
        path.back() = d.g_else;
        d.guard = path.size() >= 2 ? path[path.size() - 2] : -1;
      } break;
      case QSB_OP_ENDIF: {
        if (stack.empty()) { err << "op " << i << ": ENDIF without IF"; return err.str(); }
        d.g_then = stack.back().g_then;
        d.g_else = stack.back().g_else;
        stack.pop_back();
        path.pop_back();
        d.guard = path.empty() ? -1 : path.back();
      } break;
      default:
        err << "op " << i << ": unknown kind " << o.kind;
        return err.str();
    }
    out.dev.push_back(d);
  }
  if (!stack.empty()) return "unterminated IF";
  out.nguards = g;
  out.gwords = std::max(1, (g + 31) / 32);
  return "";
}

// ---------------------------------------------------------------------------
// streaming plan
// ---------------------------------------------------------------------------

namespace {

struct RegionBuild {
  RegionDesc desc{};
  std::vector<DevOp> ops;
  std::vector<int> mq;
  std::map<int, std::vector<int>> collapsed_at;  // qubit -> guard path of its measure / reset
};

bool is_prefix(const std::vector<int>& a, const std::vector<int>& b) {
  if (a.size() > b.size()) return false;
  return std::equal(a.begin(), a.end(), b.begin());
}

struct Planner {
  const TapeInfo& t;
  int k, lowq, rb;
  int swz_bits_ = 3;
  StreamPlan& P;
  bool pair_aware_ = P.opt.pair_aware != 0;
  bool phase_search_ = P.opt.phase_search != 0;
  bool block_condx_ = P.opt.block_condx != 0;
  int defer_from_ = P.opt.defer_gates;  // 0: off; r: defer past measurement regions r, r+1, ...
  // qubits every trajectory projected in the measurement region just closed (unguarded
  // measure / reset): the next region's first pass runs only the items whose out-of-tile
  // projected bits match (the others store zeros) -- its tile set may avoid them
  uint64_t zero_next_ = 0;
  std::vector<RegionBuild> regions;

  Planner(const TapeInfo& t_, int k_, int lowq_, int rb_, StreamPlan& p) : t(t_), k(k_), lowq(lowq_), rb(rb_), P(p) {}

  // Split one pass's gates into register-blocked phases (greedy first fit: a gate
  // joins the phase if its non-diagonal targets fit in the rb register positions and
  // none of its tile positions is blocked by an earlier deferred gate).
  void build_phases(PassDesc& pd) {
    const int sb = swz_bits_;
    const int nt = k - rb;
    pd.phase_begin = (int)P.phases.size();
    pd.pgate_begin = (int)P.phase_gates.size();
    std::vector<int> rem;
    for (int i = 0; i < pd.gate_count; ++i) rem.push_back(pd.gate_begin + i);
    while (!rem.empty()) {
      if (P.gates[rem[0]].gclass == GC_SWAP) {  // swaps run as their own shared-memory phase
        const PassGate& g = P.gates[rem[0]];
        PhaseDesc ph{};
        ph.nt = -1;
        ph.gate_begin = (int)P.phase_gates.size();
        ph.gate_count = 1;
        PhaseGate q{};
        q.kind = PK_SWAP_R;
        q.tp = g.lt;
        q.jt2 = g.lt2;
        q.cmT = g.lcm;
        q.cvT = g.lcv;
        q.gcm = g.gcm;
        q.gcv = g.gcv;
        q.guard = g.guard;
        q.mat = g.mat;
        P.phase_gates.push_back(q);
        P.phases.push_back(ph);
        rem.erase(rem.begin());
        continue;
      }
      uint32_t R = 0, blocked = 0;
      std::vector<int> take, rest;
      if (phase_search_ && k > rb) {
        // choose the register set R (rb of the k tile positions, containing the target
        // of the first remaining non-diagonal gate) under which the in-order scan absorbs
        // the most gates -- fewer phases, i.e. fewer shared-memory round trips per pass;
        // ties prefer two-qubit gates with both qubits in R (register controls, 4x4 fusion)
        int first_t = -1;
        for (int gi : rem) {
          const PassGate& g = P.gates[gi];
          if (g.gclass == GC_DENSE || g.gclass == GC_XPERM || g.gclass == GC_ANTI) {
            first_t = g.lt;
            break;
          }
        }
        double best = -1.0;
        uint32_t bestR = 0;
        const uint32_t full = (k >= 32) ? ~0u : ((1u << k) - 1);
        for (uint32_t c = 0; c <= full; ++c) {
          if (popc(c) != rb || (first_t >= 0 && !(c >> first_t & 1))) continue;
          uint32_t bl = 0;
          double score = 0;
          for (int gi : rem) {
            const PassGate& g = P.gates[gi];
            uint32_t touched = g.lcm;
            if (g.gclass != GC_DIAG_GLOBAL) touched |= 1u << g.lt;
            if (g.gclass == GC_SWAP) touched |= 1u << g.lt2;
            const bool nd = g.gclass == GC_DENSE || g.gclass == GC_XPERM || g.gclass == GC_ANTI;
            if ((touched & bl) || g.gclass == GC_SWAP || (nd && !(c >> g.lt & 1))) {
              bl |= touched;
              continue;
            }
            // a control on a thread position costs per-pair selects and blocks fusion
            score += (g.lcm & ~c) ? 0.7 : 1.0;
          }
          if (score > best) {
            best = score;
            bestR = c;
          }
          if (first_t < 0) break;  // diagonal-only remainder: any R absorbs everything
        }
        R = bestR;
        for (const int& gi : rem) {
          const PassGate& g = P.gates[gi];
          uint32_t touched = g.lcm;
          if (g.gclass != GC_DIAG_GLOBAL) touched |= 1u << g.lt;
          if (g.gclass == GC_SWAP) touched |= 1u << g.lt2;
          const bool nd = g.gclass == GC_DENSE || g.gclass == GC_XPERM || g.gclass == GC_ANTI;
          if ((touched & blocked) || g.gclass == GC_SWAP || (nd && !(R >> g.lt & 1))) {
            rest.push_back(gi);
            blocked |= touched;
          } else {
            take.push_back(gi);
          }
        }
      } else
      for (const int& gi : rem) {
        const PassGate& g = P.gates[gi];
        uint32_t touched = g.lcm;
        if (g.gclass != GC_DIAG_GLOBAL) touched |= 1u << g.lt;
        if (g.gclass == GC_SWAP) touched |= 1u << g.lt2;
        if ((touched & blocked) || g.gclass == GC_SWAP) {
          rest.push_back(gi);
          blocked |= touched;
          continue;
        }
        uint32_t need = 0;
        if (g.gclass == GC_DENSE || g.gclass == GC_XPERM || g.gclass == GC_ANTI) need = 1u << g.lt;
        need &= ~R;
        // tile controls of a register-target gate: in the registers the controlled pairs
        // are chosen at compile time; on a thread position every pair costs selects
        uint32_t want = need ? (need | (g.lcm & ~R)) : 0;
        // a single-qubit gate brings the partner of its next two-qubit gate along, so that
        // the pair's gates can fuse into one 4x4 block (fuse_phase)
        if (pair_aware_ && need && !g.lcm) {
          for (size_t x = &gi - rem.data() + 1; x < rem.size(); ++x) {
            const PassGate& h = P.gates[rem[x]];
            const uint32_t ht = h.gclass == GC_DIAG_GLOBAL ? 0u : (1u << h.lt);
            if (!((ht | h.lcm) >> g.lt & 1)) continue;
            if (h.gclass != GC_DIAG_GLOBAL && h.gclass != GC_SWAP && popc(h.lcm) == 1)
              want |= (ht | h.lcm) & ~R;
            break;
          }
        }
        bool took = false;
        if (want && popc(R | want) <= rb) {
          R |= want;
          take.push_back(gi);
          took = true;
        } else if (popc(R | need) <= rb) {
          R |= need;
          take.push_back(gi);
          took = true;
        } else {
          rest.push_back(gi);
          blocked |= touched;
        }
        // an X whose condition is per item (out-of-tile control, guard) or per thread
        // (control on a thread position) ends its target's use in this phase, so that the
        // code generator can fold it into the phase's store addresses (edge X) instead of
        // a branch or per-pair selects
        if (took && block_condx_ && g.gclass == GC_XPERM && ((g.lcm & ~R) || g.gcm || g.guard >= 0))
          blocked |= 1u << g.lt;
      }
      for (int p = 0; p < k && popc(R) < rb; ++p) R |= 1u << p;
      PhaseDesc ph{};
      ph.nt = nt;
      int rpos[kMaxRegBits], rj[32];
      int nr = 0;
      for (int p = 0; p < k; ++p) {
        rj[p] = -1;
        if (R >> p & 1) {
          rpos[nr] = p;
          rj[p] = nr++;
        }
      }
      uint32_t avoid = 0;  // thread-position controls of X gates (edge-X slot flips)
      for (int gi : take) {
        const PassGate& g = P.gates[gi];
        if (g.gclass == GC_XPERM) avoid |= g.lcm & ~R;
      }
      tile_mapping(rpos, rb, k, sb, ph.tpos, ph.soff, avoid);
      ph.gate_begin = (int)P.phase_gates.size();
      for (int gi : take) {
        const PassGate& g = P.gates[gi];
        PhaseGate q{};
        q.guard = g.guard;
        q.mat = g.mat;
        q.diag_one0 = g.diag_one0;
        q.gcm = g.gcm;
        q.gcv = g.gcv;
        switch (g.gclass) {
          case GC_DENSE: q.kind = PK_DENSE; q.jt = rj[g.lt]; break;
          case GC_XPERM: q.kind = PK_XPERM; q.jt = rj[g.lt]; break;
          case GC_ANTI: q.kind = PK_ANTI; q.jt = rj[g.lt]; break;
          case GC_SWAP: q.kind = PK_SWAP_R; q.jt = rj[g.lt]; q.jt2 = rj[g.lt2]; break;
          case GC_DIAG:
            if (rj[g.lt] >= 0) { q.kind = PK_DIAG_R; q.jt = rj[g.lt]; }
            else { q.kind = PK_DIAG_T; q.tp = g.lt; }
            break;
          default: q.kind = PK_DIAG_G; q.tp = g.gq; break;
        }
        for (uint32_t m = g.lcm; m; m &= m - 1) {
          int p = __builtin_ctz(m);
          uint32_t v = (g.lcv >> p) & 1;
          if (rj[p] >= 0) {
            q.cmR |= 1u << rj[p];
            q.cvR |= v << rj[p];
          } else {
            q.cmT |= 1u << p;
            q.cvT |= v << p;
          }
        }
        P.phase_gates.push_back(q);
      }
      ph.gate_count = (int)take.size();
      P.phases.push_back(ph);
      rem.swap(rest);
    }
    pd.phase_count = (int)P.phases.size() - pd.phase_begin;
    pd.pgate_count = (int)P.phase_gates.size() - pd.pgate_begin;
  }

  uint64_t low_mask() const { return lowq >= 64 ? ~0ull : ((1ull << lowq) - 1); }

  void emit_pass(uint64_t S, const std::vector<int>& chosen, int epi_region) {
    // fill S up to k qubits with the lowest unused qubits (longest contiguous runs)
    for (int q = 0; q < t.n && popc(S) < k; ++q) S |= 1ull << q;
    PassDesc pd{};
    pd.smask = S;
    pd.k = popc(S);
    pd.lowq = lowq;
    int pos[64];
    int j = 0;
    for (int q = 0; q < t.n; ++q) {
      pos[q] = -1;
      if (S >> q & 1) { pd.sq[j] = q; pos[q] = j++; }
    }
    pd.gate_begin = (int)P.gates.size();
    for (int gi : chosen) {
      const DevOp& d = t.dev[gi];
      PassGate pg{};
      pg.gclass = d.gclass;
      pg.guard = d.guard;
      pg.mat = d.mat;
      pg.diag_one0 = d.diag_one0;
      if (d.gclass == GC_DIAG && pos[d.t0] < 0) {
        pg.gclass = GC_DIAG_GLOBAL;
        pg.gq = d.t0;
      } else {
        pg.lt = pos[d.t0];
        pg.lt2 = d.t1 >= 0 ? pos[d.t1] : -1;
      }
      for (uint64_t m = d.cm; m; m &= m - 1) {
        int q = __builtin_ctzll(m);
        uint64_t v = (d.cv >> q) & 1;
        if (pos[q] >= 0) {
          pg.lcm |= 1u << pos[q];
          pg.lcv |= (uint32_t)v << pos[q];
        } else {
          pg.gcm |= 1ull << q;
          pg.gcv |= v << q;
        }
      }
      if (d.guard >= 0) P.guard_gates[d.guard]++;
      else P.unguarded_gates++;
      P.gates.push_back(pg);
    }
    pd.gate_count = (int)chosen.size();
    pd.region = epi_region;
    pd.epi = epi_region >= 0 ? 1 : 0;
    pd.phase_begin = pd.phase_count = 0;
    pd.rb = 0;
    if (rb > 0 && pd.k - rb >= 5 && pd.k == k) {
      build_phases(pd);
      pd.rb = rb;
    }
    P.passes.push_back(pd);
    P.steps.push_back({0, (int)P.passes.size() - 1});
  }

  // gates of `remaining` (in order) that one pass over tile set S absorbs: a gate joins when
  // its targets are in S (diagonal gates anywhere) and no earlier rejected gate shares a
  // qubit with it; grow = true lets S grow (greedy first fit) up to k qubits
  int absorb(const std::vector<int>& remaining, uint64_t& S, bool grow, std::vector<int>* chosen,
             std::vector<int>* rest, uint64_t forbid = 0) const {
    uint64_t blocked = 0;
    int taken = 0;
    for (int gi : remaining) {
      const DevOp& d = t.dev[gi];
      if (taken == kMaxPassGates) {  // staging capacity of k_pass_reg
        if (rest) rest->push_back(gi);
        continue;
      }
      const uint64_t tm = (1ull << d.t0) | (d.t1 >= 0 ? (1ull << d.t1) : 0);
      const uint64_t touched = tm | d.cm;
      if (touched & blocked) {
        if (rest) rest->push_back(gi);
        blocked |= touched;
        continue;
      }
      const uint64_t need = d.gclass == GC_DIAG ? 0 : (tm & ~S);
      if (!need || (grow && popc(S | need) <= k && !(need & forbid))) {
        S |= need;
        if (chosen) chosen->push_back(gi);
        ++taken;
      } else {
        if (rest) rest->push_back(gi);
        blocked |= touched;
      }
    }
    return taken;
  }

  // candidate tile sets of the next pass over `remaining`: the greedy first-fit set and
  // every window of k - lowq consecutive qubits above the always-present low qubits (the
  // light-cone shape of nearest-neighbour layers), ranked by the gates they absorb
  std::vector<std::pair<int, uint64_t>> candidates(const std::vector<int>& remaining) const {
    std::vector<std::pair<int, uint64_t>> c;
    uint64_t g = low_mask();
    const int ng = absorb(remaining, g, true, nullptr, nullptr);
    c.push_back({ng, g});
    const int w = k - lowq;
    for (int a = lowq; w > 0 && a + w <= t.n; ++a) {
      uint64_t S = low_mask() | (((w >= 64) ? ~0ull : ((1ull << w) - 1)) << a);
      if (S == g) continue;
      const int nabs = absorb(remaining, S, false, nullptr, nullptr);
      if (nabs > 0) c.push_back({nabs, S});
    }
    std::stable_sort(c.begin(), c.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    return c;
  }

  // tile sets of the passes of `buf` by a beam search over the tile set of each pass (kBeam
  // partial schedules, kCand tile sets tried per step, ranked by the gates still left):
  // the fewest passes found -- each pass is a full read + write of every state
  std::vector<uint64_t> beam_sets(const std::vector<int>& buf, int max_beam = 64) const {
    if (buf.empty()) return {};
    // beam width scaled to the region so planning stays ~linear in the gate count (64 x 16
    // up to ~6k gates per region: DYN20 / RDC / VQE; a 100k-gate static region gets 4 x 8)
    const int kBeam = (int)std::max<size_t>(
        4, std::min<size_t>((size_t)max_beam, 400000 / std::max<size_t>(1, buf.size())));
    const int kCand = kBeam >= 16 ? 16 : 8;
    struct Sched {
      std::vector<uint64_t> sets;
      std::vector<int> remaining;
    };
    std::vector<Sched> beam{Sched{{}, buf}};
    while (true) {
      std::vector<Sched> next;
      for (const Sched& st : beam) {
        auto cands = candidates(st.remaining);
        for (int ci = 0; ci < (int)cands.size() && ci < kCand; ++ci) {
          Sched ns;
          ns.sets = st.sets;
          uint64_t S = cands[ci].second;
          std::vector<int> chosen;
          absorb(st.remaining, S, false, &chosen, &ns.remaining);
          if (chosen.empty()) continue;
          ns.sets.push_back(S);
          next.push_back(std::move(ns));
        }
      }
      if (next.empty()) return {};  // cannot happen: the first gate of a region always fits
      std::stable_sort(next.begin(), next.end(),
                       [](const Sched& a, const Sched& b) { return a.remaining.size() < b.remaining.size(); });
      if (next[0].remaining.empty()) return next[0].sets;
      if ((int)next.size() > kBeam) next.resize(kBeam);
      beam.swap(next);
    }
  }

  // relative cost of a region's schedule: 1 per pass, except the passes after a
  // measurement while projected qubits Z have not been in a tile yet: a pass that leaves u
  // of them outside runs 2^-u of its items (the rejected ones are neither read nor stored;
  // §4.2) -- not for the region's epilogue pass (its marginal needs every item)
  // (zero_cost = 1: a pass weighs max(0.45, gates / 70) -- the memory floor of a pass
  // against the compute of a ~70-gate DYN20 pass -- instead of 1)
  double sched_cost(const std::vector<uint64_t>& sets, uint64_t Z, const std::vector<int>* buf = nullptr) const {
    double c = 0;
    std::vector<int> remaining;
    if (buf) remaining = *buf;
    for (size_t i = 0; i < sets.size(); ++i) {
      const bool epi = i + 1 == sets.size();
      double w = 1.0;
      if (buf && (P.opt.zero_cost == 1 || P.opt.zero_cost == 3)) {
        uint64_t S = sets[i];
        std::vector<int> chosen, rest;
        absorb(remaining, S, false, &chosen, &rest);
        remaining.swap(rest);
        w = std::max(0.45, (double)chosen.size() / 70.0);
      }
      c += w * ((Z && !epi) ? std::ldexp(1.0, -popc(Z & ~sets[i])) : 1.0);
      Z &= ~sets[i];
    }
    return c;
  }

  // tile sets that avoid the qubits `avoid` (above the low run): the greedy first-fit set
  // with them forbidden and the windows without them, ranked by the gates they absorb
  std::vector<std::pair<int, uint64_t>> avoiding(const std::vector<int>& remaining, uint64_t avoid) const {
    std::vector<std::pair<int, uint64_t>> c1;
    uint64_t g = low_mask();
    c1.push_back({absorb(remaining, g, true, nullptr, nullptr, avoid), g});
    const int w = k - lowq;
    for (int a = lowq; w > 0 && a + w <= t.n; ++a) {
      uint64_t S = low_mask() | (((w >= 64) ? ~0ull : ((1ull << w) - 1)) << a);
      if (S & avoid) continue;
      c1.push_back({absorb(remaining, S, false, nullptr, nullptr), S});
    }
    std::stable_sort(c1.begin(), c1.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    return c1;
  }

  // beam width of the tails the zero-aware searches evaluate: full for small regions,
  // narrower for large ones so that planning stays ~1-2 s on RDC30 (a tail is adopted only
  // when its schedule is cheaper than the full-width default)
  static int tail_beam(size_t gates) { return gates <= 700 ? 64 : 8; }

  // compute weight of a pass's gates in dense-1q-gate units (a dense gate 1, a diagonal
  // 0.3, a permutation 0.1): the gate-weighted cost model's numerator
  double gate_work(const std::vector<int>& gates) const {
    double w = 0;
    for (int gi : gates) {
      const DevOp& d = t.dev[gi];
      w += d.gclass == GC_DENSE ? 1.0 : d.gclass == GC_DIAG ? 0.3 : 0.1;
    }
    return w;
  }

  // prefixes of up to `depth` passes, each from the ordinary candidates but adding at most
  // `max_new` known-zero qubits (of Z, not yet in a tile of the prefix; the first pass of
  // the |0...0> start is free), the rest by the beam search; keep the cheapest schedule
  void prefix_search(const std::vector<int>& buf, uint64_t Z, bool has_epi, int depth_max, int max_new,
                     std::vector<uint64_t>& sets) const {
    auto cost_of = [&](const std::vector<uint64_t>& ss) {
      uint64_t z = Z;
      double c = 0;
      std::vector<int> remaining = buf;
      for (size_t i = 0; i < ss.size(); ++i) {
        const bool epi = has_epi && i + 1 == ss.size();
        double w = 1.0;
        if (P.opt.zero_cost == 1 || P.opt.zero_cost == 2) {  // gate-weighted: max(memory floor, gates x per-gate compute)
          uint64_t S = ss[i];
          std::vector<int> chosen, rest;
          absorb(remaining, S, false, &chosen, &rest);
          remaining.swap(rest);
          w = std::max(0.45, gate_work(chosen) / 70.0);
        }
        c += w * (epi ? 1.0 : std::ldexp(1.0, -popc(z & ~ss[i])));
        z &= ~ss[i];
      }
      return c;
    };
    double best = cost_of(sets);
    const uint64_t all = (t.n >= 64) ? ~0ull : ((1ull << t.n) - 1);
    const bool init = Z == all;
    struct Pre {
      std::vector<uint64_t> sets;
      std::vector<int> remaining;
      uint64_t seen;
    };
    std::vector<Pre> level{Pre{{}, buf, 0}};
    for (int depth = 0; depth < depth_max; ++depth) {
      std::vector<Pre> next;
      for (const Pre& pr : level) {
        auto cands = candidates(pr.remaining);
        int taken = 0;
        for (const auto& c : cands) {
          if (taken >= 3) break;
          if (!(init && depth == 0) && popc(c.second & Z & ~pr.seen & ~low_mask()) > max_new) continue;
          Pre np;
          np.sets = pr.sets;
          np.sets.push_back(c.second);
          uint64_t S = c.second;
          std::vector<int> chosen;
          absorb(pr.remaining, S, false, &chosen, &np.remaining);
          if (chosen.empty()) continue;
          np.seen = pr.seen | c.second;
          ++taken;
          std::vector<uint64_t> alt = np.sets;
          const std::vector<uint64_t> tail = beam_sets(np.remaining, tail_beam(buf.size()));
          if (np.remaining.empty() || !tail.empty()) {
            alt.insert(alt.end(), tail.begin(), tail.end());
            const double cost = cost_of(alt);
            if (cost < best - 1e-9) {
              best = cost;
              sets = alt;
            }
          }
          if (!np.remaining.empty()) next.push_back(std::move(np));
        }
      }
      level.swap(next);
    }
  }

  void init_prefix_search(const std::vector<int>& buf, bool has_epi, std::vector<uint64_t>& sets) const {
    const uint64_t all = (t.n >= 64) ? ~0ull : ((1ull << t.n) - 1);
    prefix_search(buf, all, has_epi, P.opt.init_aware + 1, 6, sets);
  }

  void flush(std::vector<int>& buf, int epi_region) {
    const uint64_t Z = zero_next_;
    zero_next_ = 0;
    if (buf.empty()) {
      if (epi_region >= 0) emit_pass(low_mask(), {}, epi_region);
      return;
    }
    std::vector<uint64_t> sets = beam_sets(buf);
    // the region at the |0...0> start: qubits no tile has held yet are still |0>, so a pass
    // runs 2^-u of its items (u = such qubits outside its tile; §4.2 known-zero items).
    // Also try schedules whose first passes add few new qubits at a time, the rest by the
    // beam search; keep the cheapest
    if (P.opt.init_aware && P.passes.empty() && !Z && buf.size() <= 4000) init_prefix_search(buf, epi_region >= 0, sets);
    // after a measurement: also try one or two first passes whose tiles avoid the projected
    // qubits (above the always-present low run), the rest by the beam search; keep the
    // cheapest schedule
    const uint64_t avoid = Z & ~low_mask();
    if (P.opt.zero_aware && avoid && buf.size() <= 4000) {
      double best = sched_cost(sets, Z, &buf);
      std::vector<std::vector<uint64_t>> prefixes;
      for (const auto& c1 : avoiding(buf, avoid)) {
        if (c1.first == 0 || prefixes.size() >= (size_t)P.opt.zero_width) break;
        prefixes.push_back({c1.second});
      }
      // deeper prefixes: after each prefix, up to two more avoiding passes (zero_aware =
      // the most avoiding passes per region)
      for (size_t lo = 0, depth = 2; depth <= (size_t)P.opt.zero_aware; ++depth) {
        const size_t hi = prefixes.size();
        for (size_t i = lo; i < hi; ++i) {
          std::vector<int> remaining = buf;
          for (uint64_t S : prefixes[i]) {
            std::vector<int> chosen, rest;
            absorb(remaining, S, false, &chosen, &rest);
            remaining.swap(rest);
          }
          int taken = 0;
          for (const auto& c2 : avoiding(remaining, avoid)) {
            if (c2.first == 0 || taken >= P.opt.zero_width / 2) break;
            std::vector<uint64_t> pre = prefixes[i];
            pre.push_back(c2.second);
            prefixes.push_back(pre);
            ++taken;
          }
        }
        lo = hi;
      }
      for (const auto& pre : prefixes) {
        std::vector<int> remaining = buf;
        for (uint64_t S : pre) {
          std::vector<int> chosen, rest;
          absorb(remaining, S, false, &chosen, &rest);
          remaining.swap(rest);
        }
        std::vector<uint64_t> alt = pre;
        const std::vector<uint64_t> tail = beam_sets(remaining, tail_beam(buf.size()));
        if (!remaining.empty() && tail.empty()) continue;
        alt.insert(alt.end(), tail.begin(), tail.end());
        const double c = sched_cost(alt, Z, &buf);
        if (c < best - 1e-9) {
          best = c;
          sets = alt;
        }
      }
    }
    // after a measurement, prefixes that take in the projected qubits one or two at a time
    if (P.opt.zero_step > 0 && avoid && buf.size() <= 4000)
      prefix_search(buf, avoid, epi_region >= 0, P.opt.zero_depth, P.opt.zero_step, sets);
    // replay the chosen tile sets
    std::vector<int> remaining = buf;
    for (size_t i = 0; i < sets.size(); ++i) {
      uint64_t S = sets[i];
      std::vector<int> chosen, rest;
      absorb(remaining, S, false, &chosen, &rest);
      emit_pass(S, chosen, rest.empty() ? epi_region : -1);
      remaining.swap(rest);
    }
    buf.clear();
  }

  bool descriptor_ok(const DevOp& d, const RegionBuild& R, const std::vector<int>& path) const {
    if (d.gclass != GC_XPERM && d.gclass != GC_ANTI && d.gclass != GC_DIAG) return false;
    uint64_t qs = (1ull << d.t0) | d.cm;
    for (uint64_t m = qs; m; m &= m - 1) {
      int q = __builtin_ctzll(m);
      auto it = R.collapsed_at.find(q);
      if (it == R.collapsed_at.end() || !is_prefix(it->second, path)) return false;
    }
    return true;
  }

  // Gates of the region before a measurement region that touch none of its qubits (M:
  // measured / reset qubits, descriptor-gate qubits) commute with it: the projection, the
  // renormalisation, the lazy X frame and the marginal of M are all unchanged by a unitary
  // on the other qubits.  Such an unguarded gate is DEFERRED past the region into the next
  // gate region when it also commutes with every later gate that stays (disjoint
  // supports), so the epilogue pass carries only the measured qubits' light cone and the
  // deferred gates fill the next region's passes.  Option defer_gates (default off):
  // measured on B200 with the beam-search tiling, DYN20 c128 3378 -> 2907 shots/s and
  // RDC30 d40 696 -> 817 ms with it on (same pass counts, heavier epilogue passes).
  void split_deferred(const std::vector<int>& pre, uint64_t M, bool defer, std::vector<int>& kept,
                      std::vector<int>& deferred) {
    uint64_t after = M;  // supports of the region and of the kept gates later in order
    std::vector<char> keep(pre.size(), 1);
    for (int i = (int)pre.size() - 1; i >= 0; --i) {
      const DevOp& d = t.dev[pre[i]];
      const uint64_t sup = (1ull << d.t0) | (d.t1 >= 0 ? (1ull << d.t1) : 0) | d.cm;
      if (defer && d.guard < 0 && !(sup & after)) {
        keep[i] = 0;
        continue;
      }
      after |= sup;
    }
    kept.clear();
    deferred.clear();
    for (size_t i = 0; i < pre.size(); ++i) (keep[i] ? kept : deferred).push_back(pre[i]);
  }

  std::string run() {
    P.guard_gates.assign(std::max(1, t.nguards), 0);
    regions.emplace_back();  // R0: guards evaluated before the first measurement
    P.steps.push_back({1, 0});
    int cur = 0;
    bool meas_mode = false;
    std::vector<int> buf;   // gates since the last region
    std::vector<int> pre;   // gates before the open region (flushed when it closes)
    int open_region = -1;   // measurement region still collecting ops
    std::vector<int> path;
    auto close_region = [&]() {
      if (open_region < 0) return;
      const RegionBuild& R = regions[open_region];
      uint64_t M = 0;
      for (int q : R.mq) M |= 1ull << q;
      for (const DevOp& d : R.ops)
        if (d.kind == QSB_OP_GATE) M |= (1ull << d.t0) | d.cm;
      std::vector<int> kept, deferred;
      split_deferred(pre, M, defer_from_ > 0 && open_region >= defer_from_, kept, deferred);
      flush(kept, open_region);
      P.steps.push_back({1, open_region});
      zero_next_ = 0;
      for (const DevOp& d : R.ops)
        if ((d.kind == QSB_OP_MEASURE || d.kind == QSB_OP_RESET) && d.guard < 0) zero_next_ |= 1ull << d.qubit;
      // deferred gates run first in the next gate region (relative order kept)
      deferred.insert(deferred.end(), buf.begin(), buf.end());
      buf.swap(deferred);
      pre.clear();
      open_region = -1;
    };
    for (int i = 0; i < (int)t.dev.size(); ++i) {
      const DevOp& d = t.dev[i];
      switch (d.kind) {
        case QSB_OP_IF:
          regions[cur].ops.push_back(d);
          path.push_back(d.g_then);
          break;
        case QSB_OP_ELSE:
          regions[cur].ops.push_back(d);
          path.back() = d.g_else;
          break;
        case QSB_OP_ENDIF:
          regions[cur].ops.push_back(d);
          path.pop_back();
          break;
        case QSB_OP_MEASURE:
        case QSB_OP_RESET: {
          bool fresh = !meas_mode;
          if (meas_mode) {
            auto& mq = regions[cur].mq;
            bool known = std::find(mq.begin(), mq.end(), d.qubit) != mq.end();
            if (!known && (int)mq.size() == kMaxMeasureRegion) fresh = true;
          }
          if (fresh) {
            close_region();  // a previous region still open (back to back, full M)
            regions.emplace_back();
            int r = (int)regions.size() - 1;
            regions[r].desc.has_marginal = 1;
            pre.swap(buf);
            buf.clear();
            open_region = r;
            cur = r;
            meas_mode = true;
          }
          RegionBuild& R = regions[cur];
          if (std::find(R.mq.begin(), R.mq.end(), d.qubit) == R.mq.end()) R.mq.push_back(d.qubit);
          R.collapsed_at[d.qubit] = path;
          R.ops.push_back(d);
        } break;
        case QSB_OP_GATE:
          if (meas_mode && descriptor_ok(d, regions[cur], path)) {
            regions[cur].ops.push_back(d);
            regions[cur].desc.desc_gates++;
            break;
          }
          if (meas_mode) close_region();
          meas_mode = false;
          buf.push_back(i);
          break;
      }
    }
    close_region();
    flush(buf, -1);
    return finish();
  }

  std::string finish() {
    // regions: M ordering, M-index views of ops, epilogue bin maps
    for (int r = 0; r < (int)regions.size(); ++r) {
      RegionBuild& R = regions[r];
      RegionDesc& rd = R.desc;
      rd.mcount = (int)R.mq.size();
      rd.mmask = 0;
      for (int j = 0; j < rd.mcount; ++j) {
        rd.mq[j] = R.mq[j];
        rd.mmask |= 1ull << R.mq[j];
      }
      auto midx = [&](int q) {
        for (int j = 0; j < rd.mcount; ++j)
          if (rd.mq[j] == q) return j;
        return -1;
      };
      rd.op_begin = (int)P.region_ops.size();
      for (DevOp d : R.ops) {
        if (d.kind == QSB_OP_MEASURE || d.kind == QSB_OP_RESET) d.mj = midx(d.qubit);
        if (d.kind == QSB_OP_GATE) {
          d.mj = midx(d.t0);
          d.mcm = d.mcv = 0;
          for (uint64_t m = d.cm; m; m &= m - 1) {
            int q = __builtin_ctzll(m);
            int j = midx(q);
            if (j < 0) return "internal: descriptor control outside M";
            d.mcm |= 1ull << j;
            d.mcv |= ((d.cv >> q) & 1ull) << j;
          }
        }
        P.region_ops.push_back(d);
      }
      rd.op_end = (int)P.region_ops.size();
      for (int j = 0; j < kMaxMeasureRegion; ++j) rd.mloc_bit[j] = rd.mtile_bit[j] = -1;
    }
    // link epilogue passes to their regions
    for (PassDesc& pd : P.passes) {
      if (!pd.epi) continue;
      RegionDesc& rd = regions[pd.region].desc;
      rd.epi_smask = pd.smask;
      pd.mmask = rd.mmask;
      int ml = 0;
      for (int j = 0; j < rd.mcount; ++j) {
        int q = rd.mq[j];
        if (pd.smask >> q & 1) {
          int lp = popc(pd.smask & ((1ull << q) - 1));
          pd.mloc[ml] = lp;
          rd.mloc_bit[j] = ml++;
        } else {
          uint64_t nons = ~pd.smask & ((1ull << q) - 1);
          rd.mtile_bit[j] = popc(nons & (t.n >= 64 ? ~0ull : ((1ull << t.n) - 1)));
        }
      }
      pd.m_local = ml;
      rd.m_local = ml;
      P.max_local_bins = std::max(P.max_local_bins, 1 << ml);
    }
    // prologue / init / frame-clear bookkeeping in step order
    uint64_t acc = 0;
    bool pending = false, first_pass = true;
    for (const Step& s : P.steps) {
      if (s.type == 0) {
        PassDesc& pd = P.passes[s.index];
        pd.clear_before = acc;
        acc |= pd.smask;
        pd.prologue = pending ? 1 : 0;
        pending = false;
        pd.init_zero = first_pass ? 1 : 0;
        first_pass = false;
      } else {
        RegionDesc& rd = regions[s.index].desc;
        rd.clear_mask = acc;
        acc = 0;
        if (rd.has_marginal) pending = true;
      }
    }
    for (auto& R : regions) {
      P.regions.push_back(R.desc);
      P.descriptor_gates += R.desc.desc_gates;
    }
    return "";
  }
};

}  // namespace

bool EngineOptions::set(const std::string& key, int64_t value) {
  const int v = (int)value;
  if (key == "pair_aware") pair_aware = v;
  else if (key == "phase_search") phase_search = v;
  else if (key == "block_condx") block_condx = v;
  else if (key == "inline_phases") inline_phases = v;
  else if (key == "inline_min_gates") inline_min_gates = v;
  else if (key == "inline_max_phases") inline_max_phases = v;
  else if (key == "ffma2") ffma2 = v;
  else if (key == "packed_gates") packed_gates = v;
  else if (key == "last_direct") last_direct = v;
  else if (key == "last_direct_maxlow") last_direct_maxlow = v;
  else if (key == "minblocks") minblocks = v;
  else if (key == "edge_x") edge_x = v;
  else if (key == "ctas_per_sm") ctas_per_sm = v;
  else if (key == "defer_gates") defer_gates = v;
  else if (key == "zero_aware") zero_aware = v;
  else if (key == "zero_cost") zero_cost = v;
  else if (key == "zero_width") zero_width = v;
  else if (key == "init_aware") init_aware = v;
  else if (key == "zero_step") zero_step = v;
  else if (key == "zero_depth") zero_depth = v;
  else return false;
  return true;
}

std::string build_stream_plan(const TapeInfo& t, int k, int lowq, int rb, int swz, StreamPlan& out,
                              const EngineOptions& opt) {
  out = StreamPlan();
  out.opt = opt;
  k = std::max(1, std::min(k, std::min(t.n, kMaxTile)));
  lowq = std::max(0, std::min(lowq, k));
  out.k = k;
  out.lowq = lowq;
  // register-blocked kernels run 2^(k - rb) threads: one warp at least, 512 at most
  out.rb = (rb > 0 && k - rb >= 5 && k - rb <= 9) ? rb : 0;
  out.ntiles_log2 = t.n - k;
  Planner pl(t, k, lowq, out.rb, out);
  pl.swz_bits_ = swz;
  return pl.run();
}

DenseVariant dense_variant(const MatSrc& m) {
  if (m.has_matrix) {
    const double* x = m.mat;
    if (x[1] == 0.0 && x[3] == 0.0 && x[5] == 0.0 && x[7] == 0.0) return DV_REAL;
    if (x[1] == 0.0 && x[7] == 0.0 && x[2] == 0.0 && x[4] == 0.0) return DV_RX;
    return DV_GEN;
  }
  if (m.base == QSB_G_H || m.base == QSB_G_RY) return DV_REAL;
  if (m.base == QSB_G_RX) return DV_RX;
  return DV_GEN;
}

uint32_t zero_mask(const MatSrc& m) {
  uint32_t z = 0;
  if (m.has_matrix) {
    for (int i = 0; i < 8; ++i)
      if (m.mat[i] == 0.0) z |= 1u << i;
    return z;
  }
  if (m.base == QSB_G_U) return 1u << 1;  // m00 = cos(theta/2) is real
  return 0;
}

double phase_gate_flops(const PhaseGate& q, const MatSrc& m) {
  switch (q.kind) {
    case PK_XPERM:
    case PK_SWAP_R: return 0;
    case PK_DENSE: {
      DenseVariant dv = dense_variant(m);
      if (dv != DV_GEN) return 12;
      const uint32_t z = zero_mask(m);
      double f = 0;
      for (int r = 0; r < 2; ++r)
        for (int comp = 0; comp < 2; ++comp) {
          int terms = 0;
          for (int i = 0; i < 4; ++i) terms += (z >> (4 * r + i) & 1) ? 0 : 1;
          if (terms) f += 2.0 * (terms - 1) + 1.0;  // (terms-1) FMA + 1 MUL
        }
      return f;
    }
    case PK_DIAG_R: return q.diag_one0 ? 6 : 12;
    default: return 12;  // ANTI, DIAG_T, DIAG_G: two complex multiplies per pair
  }
}

double pass_flops(const TapeInfo& t, const StreamPlan& P, int pass) {
  const PassDesc& pd = P.passes[pass];
  double f = 0;
  for (int g = pd.pgate_begin; g < pd.pgate_begin + pd.pgate_count; ++g) {
    const PhaseGate& q = P.phase_gates[g];
    const int ctrl = popc(q.cmR) + popc(q.cmT) + popc(q.gcm);
    f += phase_gate_flops(q, t.mats[q.mat]) * std::ldexp(1.0, t.n - 1 - ctrl);
  }
  return f;
}


// ---------------------------------------------------------------------------
// register-phase gate fusion (see qsb_plan.h)
// ---------------------------------------------------------------------------
namespace {

using cd = std::complex<double>;
std::atomic<int> g_fuse_fail{0};

bool fusable(const TapeInfo& t, const PhaseGate& q) {
  if (q.kind != PK_DENSE && q.kind != PK_XPERM && q.kind != PK_ANTI && q.kind != PK_DIAG_R) return false;
  return q.guard < 0 && q.gcm == 0 && q.cmT == 0 && t.mats[q.mat].has_matrix && popc(q.cmR) <= 1 &&
         !(q.cmR >> q.jt & 1);
}

// the 2x2 a register-phase gate applies to its (bit jt = 0, 1) pairs, as the kernels compute it
void gate2x2(const TapeInfo& t, const PhaseGate& q, cd u[4]) {
  const double* m = t.mats[q.mat].mat;
  switch (q.kind) {
    case PK_XPERM: u[0] = 0.0; u[1] = 1.0; u[2] = 1.0; u[3] = 0.0; break;
    case PK_ANTI: u[0] = 0.0; u[1] = cd(m[2], m[3]); u[2] = cd(m[4], m[5]); u[3] = 0.0; break;
    case PK_DIAG_R:
      u[0] = q.diag_one0 ? cd(1.0, 0.0) : cd(m[0], m[1]);
      u[1] = 0.0; u[2] = 0.0; u[3] = cd(m[6], m[7]);
      break;
    default:
      for (int i = 0; i < 4; ++i) u[i] = cd(m[2 * i], m[2 * i + 1]);
  }
}

// register bits a phase gate reads or writes
uint32_t gate_bits(const PhaseGate& q) {
  switch (q.kind) {
    case PK_DENSE: case PK_XPERM: case PK_ANTI: case PK_DIAG_R: return q.cmR | (1u << q.jt);
    case PK_DIAG_T: case PK_DIAG_G: return q.cmR;
    default: return ~0u;
  }
}

// flops per pair of a gate applied on its own (the JIT kernels' zero-dropped chains)
double gate_pair_flops(const TapeInfo& t, const PhaseGate& q) { return phase_gate_flops(q, t.mats[q.mat]); }

double chain_flops(const cd* row, int nc) {  // one output amplitude: re and im chains
  int terms = 0;
  for (int c = 0; c < nc; ++c) terms += (row[c].real() != 0.0) + (row[c].imag() != 0.0);
  return terms ? 2.0 * (2.0 * (terms - 1) + 1.0) : 0.0;
}

struct Block {
  int qa = -1, qb = -1;       // register bits (qb = -1: single qubit)
  std::vector<int> gates;     // phase-gate indices in application order
};

// product matrix of a block: index bit 0 <-> qa, bit 1 <-> qb
void block_matrix(const TapeInfo& t, const StreamPlan& P, const Block& b, cd* M) {
  const int d = b.qb < 0 ? 2 : 4;
  for (int i = 0; i < d * d; ++i) M[i] = (i % (d + 1) == 0) ? 1.0 : 0.0;
  for (int gi : b.gates) {
    const PhaseGate& q = P.phase_gates[gi];
    cd u[4];
    gate2x2(t, q, u);
    const int tb = q.jt == b.qa ? 0 : 1;  // matrix bit of the target
    const int cb = q.cmR ? 1 - tb : -1;    // matrix bit of the control
    const int cval = q.cmR ? (q.cvR ? 1 : 0) : 0;
    cd G[16];
    for (int i = 0; i < d * d; ++i) G[i] = 0.0;
    for (int r = 0; r < d; ++r)
      for (int c = 0; c < d; ++c) {
        if ((r & ~(1 << tb)) != (c & ~(1 << tb))) continue;  // other bits unchanged
        if (cb >= 0 && ((r >> cb) & 1) != cval) {
          G[r * d + c] = r == c ? 1.0 : 0.0;
          continue;
        }
        G[r * d + c] = u[((r >> tb) & 1) * 2 + ((c >> tb) & 1)];
      }
    cd N[16];
    for (int r = 0; r < d; ++r)
      for (int c = 0; c < d; ++c) {
        cd s = 0.0;
        for (int x = 0; x < d; ++x) s += G[r * d + x] * M[x * d + c];
        N[r * d + c] = s;
      }
    for (int i = 0; i < d * d; ++i) M[i] = N[i];
  }
}

// host emulation of items on a register vector (check of the fusion)
void emulate(const TapeInfo& t, const StreamPlan& P, const std::vector<FuseItem>& items, int nr, cd* v) {
  for (const FuseItem& it : items) {
    if (it.gate >= 0) {
      const PhaseGate& q = P.phase_gates[it.gate];
      if (q.kind == PK_DIAG_T || q.kind == PK_DIAG_G) {
        const cd f(t.mats[q.mat].mat[0] + 0.25, t.mats[q.mat].mat[1] - 0.5);
        for (int j = 0; j < nr; ++j)
          if (((uint32_t)j & q.cmR) == q.cvR) v[j] *= f;
        continue;
      }
      cd u[4];
      gate2x2(t, q, u);
      const int b = 1 << q.jt;
      for (int j = 0; j < nr; ++j) {
        if ((j & b) || ((uint32_t)j & q.cmR) != q.cvR) continue;
        const cd a0 = v[j], a1 = v[j | b];
        v[j] = u[0] * a0 + u[1] * a1;
        v[j | b] = u[2] * a0 + u[3] * a1;
      }
      continue;
    }
    const int A = 1 << it.qa, B = it.qb < 0 ? 0 : 1 << it.qb, d = it.qb < 0 ? 2 : 4;
    for (int j = 0; j < nr; ++j) {
      if ((j & A) || (j & B)) continue;
      const int idx[4] = {j, j | A, j | B, j | A | B};
      cd x[4], y[4];
      for (int c = 0; c < d; ++c) x[c] = v[idx[c]];
      for (int r = 0; r < d; ++r) {
        y[r] = 0.0;
        for (int c = 0; c < d; ++c) y[r] += cd(it.m[2 * (r * d + c)], it.m[2 * (r * d + c) + 1]) * x[c];
      }
      for (int r = 0; r < d; ++r) v[idx[r]] = y[r];
    }
  }
}

}  // namespace

double fuse_block_flops(const FuseItem& f) {
  const int d = f.qb < 0 ? 2 : 4;
  double s = 0;
  for (int r = 0; r < d; ++r) {
    cd row[4];
    for (int c = 0; c < d; ++c) row[c] = cd(f.m[2 * (r * d + c)], f.m[2 * (r * d + c) + 1]);
    s += chain_flops(row, d);
  }
  return s;
}

int fuse_check_failures() { return g_fuse_fail.load(); }

std::vector<FuseItem> fuse_phase(const TapeInfo& t, const StreamPlan& P, int phase, bool enable) {
  const PhaseDesc& ph = P.phases[phase];
  std::vector<FuseItem> plain;
  for (int g = ph.gate_begin; g < ph.gate_begin + ph.gate_count; ++g) {
    FuseItem f;
    f.gate = g;
    plain.push_back(f);
  }
  if (!enable || ph.nt < 0 || ph.gate_count < 2) return plain;
  const int rb = P.rb;
  std::vector<FuseItem> out;
  std::vector<Block> blocks;       // open blocks (by id)
  std::vector<int> open(rb, -1);   // register bit -> open block id
  std::vector<bool> live;
  auto new_block = [&](int qa, int qb) {
    blocks.push_back(Block{qa, qb, {}});
    live.push_back(true);
    const int id = (int)blocks.size() - 1;
    open[qa] = id;
    if (qb >= 0) open[qb] = id;
    return id;
  };
  auto emit_gate = [&](int g) {
    FuseItem f;
    f.gate = g;
    out.push_back(f);
  };
  // close block id: fused if cheaper; otherwise its gates one by one, except that the
  // single-qubit gates after its last two-qubit gate stay open (keep_tail) so that a
  // later block can absorb them
  std::function<void(int, bool)> close = [&](int id, bool keep_tail) {
    if (!live[id]) return;
    live[id] = false;
    Block b = blocks[id];
    if (open[b.qa] == id) open[b.qa] = -1;
    if (b.qb >= 0 && open[b.qb] == id) open[b.qb] = -1;
    double sep = 0;
    for (int gi : b.gates) {
      const PhaseGate& q = P.phase_gates[gi];
      const double pairs = b.qb < 0 ? 1.0 : (q.cmR ? 1.0 : 2.0);  // pairs per group of the block
      sep += gate_pair_flops(t, q) * pairs;
    }
    if (b.gates.size() >= 2) {
      FuseItem f;
      f.qa = b.qa;
      f.qb = b.qb;
      f.ngates = (int)b.gates.size();
      cd M[16];
      block_matrix(t, P, b, M);
      const int d = b.qb < 0 ? 2 : 4;
      for (int i = 0; i < d * d; ++i) {
        f.m[2 * i] = M[i].real();
        f.m[2 * i + 1] = M[i].imag();
      }
      if (fuse_block_flops(f) < sep) {
        out.push_back(f);
        return;
      }
    }
    int last2 = -1;
    if (keep_tail && b.qb >= 0)
      for (int i = 0; i < (int)b.gates.size(); ++i)
        if (P.phase_gates[b.gates[i]].cmR) last2 = i;
    if (!keep_tail || b.qb < 0 || last2 < 0) {
      for (int gi : b.gates) emit_gate(gi);
      return;
    }
    for (int i = 0; i <= last2; ++i) emit_gate(b.gates[i]);
    for (int i = last2 + 1; i < (int)b.gates.size(); ++i) {
      const int gi = b.gates[i];
      const int q = P.phase_gates[gi].jt;
      if (open[q] < 0) new_block(q, -1);
      blocks[open[q]].gates.push_back(gi);
    }
  };
  for (int g = ph.gate_begin; g < ph.gate_begin + ph.gate_count; ++g) {
    const PhaseGate& q = P.phase_gates[g];
    if (!fusable(t, q)) {
      const uint32_t bits = gate_bits(q);
      for (int r = 0; r < rb; ++r)
        if ((bits >> r & 1) && open[r] >= 0) close(open[r], false);
      emit_gate(g);
      continue;
    }
    if (!q.cmR) {
      if (open[q.jt] < 0) new_block(q.jt, -1);
      blocks[open[q.jt]].gates.push_back(g);
      continue;
    }
    const int a = q.jt, c = __builtin_ctz(q.cmR);
    if (open[a] >= 0 && open[a] == open[c]) {
      blocks[open[a]].gates.push_back(g);
      continue;
    }
    for (int x : {a, c})
      if (open[x] >= 0 && blocks[open[x]].qb >= 0) close(open[x], true);
    std::vector<int> pre;
    for (int x : {a, c})
      if (open[x] >= 0) {
        const int id = open[x];
        pre.insert(pre.end(), blocks[id].gates.begin(), blocks[id].gates.end());
        live[id] = false;
        open[x] = -1;
      }
    const int id = new_block(std::min(a, c), std::max(a, c));
    blocks[id].gates = pre;
    blocks[id].gates.push_back(g);
  }
  for (int id = 0; id < (int)blocks.size(); ++id) close(id, false);
  if (getenv("QSB_FUSE_DEBUG")) {
    fprintf(stderr, "phase %d:", phase);
    for (const FuseItem& f : out) {
      if (f.gate >= 0) {
        const PhaseGate& q = P.phase_gates[f.gate];
        fprintf(stderr, " g%d(k%d t%d c%x)", f.gate - ph.gate_begin, q.kind, q.jt, q.cmR);
      } else fprintf(stderr, " [B%d,%d:%d]", f.qa, f.qb, f.ngates);
    }
    fprintf(stderr, "\n");
  }
  // host check: the items reproduce the gates on random register vectors
  const int nr = 1 << rb;
  uint64_t s = 0x9E3779B97F4A7C15ull ^ (uint64_t)phase;
  auto rnd = [&]() {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(s >> 11) * 0x1.0p-53 - 0.5;
  };
  for (int trial = 0; trial < 2; ++trial) {
    std::vector<cd> v(nr), w(nr);
    for (int j = 0; j < nr; ++j) v[j] = w[j] = cd(rnd(), rnd());
    emulate(t, P, plain, nr, v.data());
    emulate(t, P, out, nr, w.data());
    double err = 0, mag = 0;
    for (int j = 0; j < nr; ++j) {
      err = std::max(err, std::abs(v[j] - w[j]));
      mag = std::max(mag, std::abs(v[j]));
    }
    if (!(err <= 1e-12 * std::max(1.0, mag))) {
      ++g_fuse_fail;
      return plain;
    }
  }
  return out;
}

double pass_flops_fused(const TapeInfo& t, const StreamPlan& P, int pass) {
  const PassDesc& pd = P.passes[pass];
  double f = 0;
  for (int i = 0; i < pd.phase_count; ++i) {
    const int phase = pd.phase_begin + i;
    for (const FuseItem& it : fuse_phase(t, P, phase, true)) {
      if (it.gate >= 0) {
        const PhaseGate& q = P.phase_gates[it.gate];
        const int ctrl = popc(q.cmR) + popc(q.cmT) + popc(q.gcm);
        f += phase_gate_flops(q, t.mats[q.mat]) * std::ldexp(1.0, t.n - 1 - ctrl);
      } else {
        f += fuse_block_flops(it) * std::ldexp(1.0, t.n - (it.qb < 0 ? 1 : 2));
      }
    }
  }
  return f;
}

}  // namespace qsb
