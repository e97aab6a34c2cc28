// C ABI of the global-qubit-sliced engine and its NCCL data plane (qsb.h qsb_slice_* /
// qsb_comm_*; BASELINE cfg 5).
//
// A sliced trajectory is driven by the host planner (sliced.py: static schedule with
// look-ahead eviction) but DECIDED on the device: every call below only enqueues work on
// the context's stream, and the classical store / guards / RNG live in a device SliceCtl.
// The only data movement between GPUs is the exchange of a global position with a local
// one (ncclSend / ncclRecv of the packed half, in chunks) and the all-gather of one p1
// partial per rank per measurement (ncclAllGather of 8 bytes, in place).
//
// NCCL is opened with dlopen (libnccl.so.2: in a torch process the library torch already
// mapped), so the backend library has no link-time NCCL dependency and loads on hosts
// without it; qsb_comm_* return QSB_ERR_UNSUPPORTED there.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "qsb_launch.h"
#include "qsb_objects.h"
#include "qsb_plan.h"

using namespace qsb;

struct qsb_slicectl_s {
  qsb_ctx ctx = nullptr;
  int nslices = 1;
  int nwords = 1;
  DevBuf ctl, partials, blocks;
};

struct qsb_comm_s {
  qsb_ctx ctx = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t chunk_bytes = 64ll << 20;
  DevBuf sendbuf, recvbuf;
  int64_t bytes_sent = 0, exchanges = 0, allgathers = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  double exchange_ms = 0;
};

namespace {

struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.get_id = (decltype(n.get_id))dlsym(n.h, "ncclGetUniqueId");
    n.init = (decltype(n.init))dlsym(n.h, "ncclCommInitRank");
    n.destroy = (decltype(n.destroy))dlsym(n.h, "ncclCommDestroy");
    n.send = (decltype(n.send))dlsym(n.h, "ncclSend");
    n.recv = (decltype(n.recv))dlsym(n.h, "ncclRecv");
    n.allgather = (decltype(n.allgather))dlsym(n.h, "ncclAllGather");
    n.group_start = (decltype(n.group_start))dlsym(n.h, "ncclGroupStart");
    n.group_end = (decltype(n.group_end))dlsym(n.h, "ncclGroupEnd");
    n.errstr = (decltype(n.errstr))dlsym(n.h, "ncclGetErrorString");
    n.version = (decltype(n.version))dlsym(n.h, "ncclGetVersion");
    n.ok = n.get_id && n.init && n.destroy && n.send && n.recv && n.allgather && n.group_start && n.group_end &&
           n.errstr && n.version;
  });
  return n;
}

#define QSB_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t _r = (call);                                                                  \
    if (_r != ncclSuccess) return fail(QSB_ERR_CUDA, std::string(#call) + ": " + nccl().errstr(_r)); \
  } while (0)

int check_state(qsb_state st) {
  if (!st) return fail(QSB_ERR_ARG, "null state");
  return QSB_OK;
}

}  // namespace

extern "C" {

// ---- classical control of a sliced trajectory ---------------------------------------

int32_t qsb_slice_ctl_create(qsb_ctx ctx, int32_t nslices, int32_t nbits, uint64_t seed, int64_t shot,
                             const uint64_t* rng_state, qsb_slicectl* out) {
  if (!ctx || !out || nslices < 1) return fail(QSB_ERR_ARG, "bad slice control arguments");
  const int nwords = std::max(1, (nbits + 63) / 64);
  if (nwords > kSliceWords) return fail(QSB_ERR_UNSUPPORTED, "sliced runs hold at most 1024 classical bits");
  DeviceGuard g(ctx->device);
  auto* c = new qsb_slicectl_s();
  c->ctx = ctx;
  c->nslices = nslices;
  c->nwords = nwords;
  if (c->ctl.ensure(sizeof(SliceCtl) + 64) != cudaSuccess || c->partials.ensure(sizeof(double) * nslices) != cudaSuccess) {
    delete c;
    return fail(QSB_ERR_OOM, "slice control allocation failed");
  }
  uint64_t* d_rng = nullptr;
  if (rng_state) {
    d_rng = reinterpret_cast<uint64_t*>(c->ctl.as<char>() + sizeof(SliceCtl));
    QSB_CUDA(cudaMemcpyAsync(d_rng, rng_state, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  }
  launch_slice_init(c->ctl.as<SliceCtl>(), seed, shot, d_rng, nwords, ctx->stream);
  QSB_CUDA(cudaMemsetAsync(c->partials.p, 0, sizeof(double) * nslices, ctx->stream));
  QSB_CUDA(cudaGetLastError());
  *out = c;
  return QSB_OK;
}

int32_t qsb_slice_ctl_destroy(qsb_slicectl c) {
  if (!c) return QSB_OK;
  DeviceGuard g(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  c->ctl.release();
  c->partials.release();
  c->blocks.release();
  delete c;
  return QSB_OK;
}

int32_t qsb_slice_ctl_read(qsb_slicectl c, uint64_t* bits_out, int32_t* status, int32_t* draws, uint64_t* rng_out) {
  DeviceGuard g(c->ctx->device);
  SliceCtl x;
  QSB_CUDA(cudaMemcpyAsync(&x, c->ctl.p, sizeof(x), cudaMemcpyDeviceToHost, c->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(c->ctx->stream));
  if (bits_out) std::memcpy(bits_out, x.bits, sizeof(uint64_t) * c->nwords);
  if (status) *status = x.status;
  if (draws) *draws = x.draws;
  if (rng_out) std::memcpy(rng_out, x.rng, sizeof(x.rng));
  return QSB_OK;
}

// host access to the partial slots (a transport without a device collective: the
// torch.distributed / gloo path stages them through the host)
int32_t qsb_slice_partials(qsb_slicectl c, double* host_out, const double* host_in) {
  if (!c) return fail(QSB_ERR_ARG, "null slicectl");
  DeviceGuard g(c->ctx->device);
  const size_t bytes = sizeof(double) * c->nslices;
  if (host_out) {
    QSB_CUDA(cudaMemcpyAsync(host_out, c->partials.p, bytes, cudaMemcpyDeviceToHost, c->ctx->stream));
    QSB_CUDA(cudaStreamSynchronize(c->ctx->stream));
  }
  if (host_in) {
    QSB_CUDA(cudaMemcpyAsync(c->partials.p, host_in, bytes, cudaMemcpyHostToDevice, c->ctx->stream));
    QSB_CUDA(cudaStreamSynchronize(c->ctx->stream));
  }
  return QSB_OK;
}

int32_t qsb_slice_guard(qsb_slicectl c, const qsb_op* op) {
  if (!c || !op) return fail(QSB_ERR_ARG, "null argument");
  if (op->kind != QSB_OP_IF && op->kind != QSB_OP_ELSE && op->kind != QSB_OP_ENDIF)
    return fail(QSB_ERR_ARG, "qsb_slice_guard takes IF / ELSE / ENDIF records");
  if (op->kind == QSB_OP_IF && op->pred_bit + op->pred_width > 64 * c->nwords)
    return fail(QSB_ERR_ARG, "predicate reads bits outside the classical store");
  DeviceGuard g(c->ctx->device);
  launch_slice_guard(c->ctl.as<SliceCtl>(), op->kind, op->pred_bit, op->pred_width, op->pred_cmp, op->pred_rhs,
                     c->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_slice_gate(qsb_state st, qsb_slicectl c, const qsb_op* op) {
  if (check_state(st) || !c || !op) return fail(QSB_ERR_ARG, "null argument");
  if (op->kind != QSB_OP_GATE || !op->has_matrix) return fail(QSB_ERR_ARG, "slice gates need a host-built matrix");
  TapeInfo ti;
  std::string e = analyze_tape(op, 1, st->n, 0, 0, ti);
  if (!e.empty()) return fail(QSB_ERR_ARG, e);
  const DevOp& d = ti.dev[0];
  if (d.gclass == GC_SWAP) return fail(QSB_ERR_ARG, "swap is a relabeling in the sliced engine");
  DeviceGuard g(st->ctx->device);
  launch_slice_gate(st->c64, st->amps.p, st->n, d.t0, d.cm, d.cv, d.gclass, ti.mats[0].mat, c->ctl.as<SliceCtl>(),
                    st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_slice_scale(qsb_state st, qsb_slicectl c, double re, double im) {
  if (check_state(st) || !c) return fail(QSB_ERR_ARG, "null argument");
  DeviceGuard g(st->ctx->device);
  launch_slice_scale(st->c64, st->amps.p, st->n, re, im, c->ctl.as<SliceCtl>(), st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_slice_prob1(qsb_state st, qsb_slicectl c, int32_t qubit, int32_t select, int32_t index) {
  if (check_state(st) || !c) return fail(QSB_ERR_ARG, "null argument");
  if (qubit >= st->n || index < 0 || index >= c->nslices) return fail(QSB_ERR_ARG, "qubit / slice index out of range");
  DeviceGuard g(st->ctx->device);
  const int q = qubit < 0 ? -1 : qubit;
  const int nb = prob_blocks_for(st->n, q);
  QSB_CUDA(c->blocks.ensure(sizeof(double) * nb));
  if (select) launch_prob_blocks(st->c64, st->amps.p, st->n, q, c->blocks.as<double>(), st->ctx->stream);
  launch_slice_put(c->blocks.as<double>(), nb, select ? 1 : 0, c->partials.as<double>(), index, st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_slice_decide(qsb_slicectl c, int32_t kind, int32_t bit) {
  if (!c) return fail(QSB_ERR_ARG, "null argument");
  if (kind != QSB_OP_MEASURE && kind != QSB_OP_RESET) return fail(QSB_ERR_ARG, "decide takes MEASURE or RESET");
  if (kind == QSB_OP_MEASURE && (bit < 0 || bit >= 64 * c->nwords)) return fail(QSB_ERR_ARG, "bit out of range");
  DeviceGuard g(c->ctx->device);
  launch_slice_decide(c->ctl.as<SliceCtl>(), c->partials.as<double>(), c->nslices, kind, bit, c->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_slice_collapse(qsb_state st, qsb_slicectl c, int32_t qubit, int32_t gbit, int32_t flip) {
  if (check_state(st) || !c) return fail(QSB_ERR_ARG, "null argument");
  if (qubit >= st->n) return fail(QSB_ERR_ARG, "qubit out of range");
  if (qubit < 0 && flip) return fail(QSB_ERR_ARG, "reset of a global qubit: make it local first");
  DeviceGuard g(st->ctx->device);
  launch_slice_collapse(st->c64, st->amps.p, st->n, qubit < 0 ? -1 : qubit, gbit ? 1 : 0, flip ? 1 : 0,
                        c->ctl.as<SliceCtl>(), st->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

int32_t qsb_slice_exchange_local(qsb_state a, qsb_state b, int32_t pos) {
  if (check_state(a) || check_state(b)) return fail(QSB_ERR_ARG, "null state");
  if (a->n != b->n || a->c64 != b->c64 || a->ctx != b->ctx) return fail(QSB_ERR_DIMENSION, "slices differ");
  if (pos < 0 || pos >= a->n) return fail(QSB_ERR_ARG, "local position out of range");
  DeviceGuard g(a->ctx->device);
  launch_slice_exchange_local(a->c64, a->amps.p, b->amps.p, a->n, pos, a->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

namespace {
int check_remap(qsb_state st, int k, const int32_t* lpos) {
  if (k < 1 || k > 3 || !lpos) return fail(QSB_ERR_ARG, "remap of 1..3 positions expected");
  for (int i = 0; i < k; ++i) {
    if (lpos[i] < 0 || lpos[i] >= st->n) return fail(QSB_ERR_ARG, "local position out of range");
    for (int j = 0; j < i; ++j)
      if (lpos[j] == lpos[i]) return fail(QSB_ERR_ARG, "local positions must differ");
  }
  return QSB_OK;
}
}  // namespace

// single device: remap k global positions with local positions lpos[0..k) across the
// group of 2^k slices (group[y]: global bits y of the remapped positions)
int32_t qsb_slice_remap_local(const qsb_state* group, int32_t k, const int32_t* lpos) {
  if (!group || k < 1 || k > 3) return fail(QSB_ERR_ARG, "remap of 1..3 positions expected");
  void* ptrs[8];
  for (int i = 0; i < (1 << k); ++i) {
    if (check_state(group[i])) return fail(QSB_ERR_ARG, "null state");
    if (group[i]->n != group[0]->n || group[i]->c64 != group[0]->c64 || group[i]->ctx != group[0]->ctx)
      return fail(QSB_ERR_DIMENSION, "slices differ");
    for (int j = 0; j < i; ++j)
      if (group[j] == group[i]) return fail(QSB_ERR_ARG, "slices of a group must differ");
    ptrs[i] = group[i]->amps.p;
  }
  if (int rc = check_remap(group[0], k, lpos)) return rc;
  if (group[0]->n < k) return fail(QSB_ERR_ARG, "slice too small");
  int lp[3];
  for (int i = 0; i < k; ++i) lp[i] = lpos[i];
  DeviceGuard g(group[0]->ctx->device);
  launch_slice_remap_local(group[0]->c64, ptrs, group[0]->n, k, lp, group[0]->ctx->stream);
  QSB_CUDA(cudaGetLastError());
  return QSB_OK;
}

// host staging of one remap region (local bits at lpos == x, increasing order of the
// other bits; 2^(n-k) amplitudes in the slice's precision): the torch.distributed
// transport and the tests
int32_t qsb_slice_read_sub(qsb_state st, int32_t k, const int32_t* lpos, int32_t x, void* host_out) {
  if (check_state(st) || !host_out) return fail(QSB_ERR_ARG, "null argument");
  if (int rc = check_remap(st, k, lpos)) return rc;
  if (x < 0 || x >= (1 << k)) return fail(QSB_ERR_ARG, "region index out of range");
  DeviceGuard g(st->ctx->device);
  const int64_t cnt = 1ll << (st->n - k), amp = st->c64 ? 8 : 16;
  DevBuf tmp;
  QSB_CUDA(tmp.ensure(cnt * amp));
  int lp[3];
  for (int i = 0; i < k; ++i) lp[i] = lpos[i];
  launch_slice_pack_sub(st->c64, st->amps.p, k, lp, x, 0, cnt, tmp.p, st->ctx->stream);
  QSB_CUDA(cudaMemcpyAsync(host_out, tmp.p, cnt * amp, cudaMemcpyDeviceToHost, st->ctx->stream));
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  return QSB_OK;
}

int32_t qsb_slice_write_sub(qsb_state st, int32_t k, const int32_t* lpos, int32_t x, const void* host_in) {
  if (check_state(st) || !host_in) return fail(QSB_ERR_ARG, "null argument");
  if (int rc = check_remap(st, k, lpos)) return rc;
  if (x < 0 || x >= (1 << k)) return fail(QSB_ERR_ARG, "region index out of range");
  DeviceGuard g(st->ctx->device);
  const int64_t cnt = 1ll << (st->n - k), amp = st->c64 ? 8 : 16;
  DevBuf tmp;
  QSB_CUDA(tmp.ensure(cnt * amp));
  int lp[3];
  for (int i = 0; i < k; ++i) lp[i] = lpos[i];
  QSB_CUDA(cudaMemcpyAsync(tmp.p, host_in, cnt * amp, cudaMemcpyHostToDevice, st->ctx->stream));
  launch_slice_unpack_sub(st->c64, st->amps.p, k, lp, x, 0, cnt, tmp.p, st->ctx->stream);
  QSB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  return QSB_OK;
}

// ---- NCCL data plane ----------------------------------------------------------------

int32_t qsb_comm_unique_id(uint8_t* out128) {
  if (!nccl().ok) return fail(QSB_ERR_UNSUPPORTED, "libnccl.so.2 not available");
  ncclUniqueId id;
  QSB_NCCL(nccl().get_id(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return QSB_OK;
}

int32_t qsb_comm_init(qsb_ctx ctx, const uint8_t* id128, int32_t rank, int32_t nranks, qsb_comm* out) {
  if (!ctx || !id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(QSB_ERR_ARG, "bad comm arguments");
  if (!nccl().ok) return fail(QSB_ERR_UNSUPPORTED, "libnccl.so.2 not available");
  DeviceGuard g(ctx->device);
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto* c = new qsb_comm_s();
  c->ctx = ctx;
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = nccl().init(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(QSB_ERR_CUDA, std::string("ncclCommInitRank: ") + nccl().errstr(r));
  }
  cudaEventCreate(&c->e0);
  cudaEventCreate(&c->e1);
  *out = c;
  return QSB_OK;
}

int32_t qsb_comm_destroy(qsb_comm c) {
  if (!c) return QSB_OK;
  DeviceGuard g(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  if (c->comm) nccl().destroy(c->comm);
  c->sendbuf.release();
  c->recvbuf.release();
  if (c->e0) cudaEventDestroy(c->e0);
  if (c->e1) cudaEventDestroy(c->e1);
  delete c;
  return QSB_OK;
}

int32_t qsb_comm_set_chunk(qsb_comm c, int64_t bytes) {
  if (!c || bytes < 4096) return fail(QSB_ERR_ARG, "chunk must be >= 4 KiB");
  c->chunk_bytes = bytes;
  return QSB_OK;
}

// every rank's partials[rank] -> partials[0 .. nranks) on every rank (in place)
int32_t qsb_comm_allgather_partials(qsb_comm c, qsb_slicectl s) {
  if (!c || !s || s->nslices != c->nranks) return fail(QSB_ERR_ARG, "one slice per rank expected");
  DeviceGuard g(c->ctx->device);
  double* p = s->partials.as<double>();
  QSB_NCCL(nccl().allgather(p + c->rank, p, 1, ncclFloat64, c->comm, c->ctx->stream));
  c->allgathers++;
  return QSB_OK;
}

// The exchange of a global position with local position `pos`: this rank (global bit
// send_c) sends the amplitudes of `send` whose local bit `pos` is !send_c -- packed in
// index order, in chunks -- to `peer`, and unpacks what `peer` sends into the same region
// of `recv` (global bit recv_c).  Production passes the same slice twice (in place:
// chunk k is packed before chunk k is overwritten); a single-GPU test exchanges two
// slices through a self-peer.
int32_t qsb_comm_exchange(qsb_comm c, qsb_state send, int32_t send_c, qsb_state recv, int32_t recv_c, int32_t pos,
                          int32_t peer) {
  if (!c || check_state(send) || check_state(recv)) return fail(QSB_ERR_ARG, "null argument");
  if (send->n != recv->n || send->c64 != recv->c64) return fail(QSB_ERR_DIMENSION, "slices differ");
  if (pos < 0 || pos >= send->n || peer < 0 || peer >= c->nranks) return fail(QSB_ERR_ARG, "position / peer out of range");
  DeviceGuard g(c->ctx->device);
  const int64_t amp = send->c64 ? 8 : 16;
  const int64_t half = 1ll << (send->n - 1);
  const int64_t per = std::max<int64_t>(1, std::min<int64_t>(half, c->chunk_bytes / amp));
  QSB_CUDA(c->sendbuf.ensure(per * amp));
  QSB_CUDA(c->recvbuf.ensure(per * amp));
  cudaStream_t s = c->ctx->stream;
  cudaEventRecord(c->e0, s);
  for (int64_t first = 0; first < half; first += per) {
    const int64_t cnt = std::min(per, half - first);
    launch_slice_pack(send->c64, send->amps.p, pos, send_c ? 1 : 0, first, cnt, c->sendbuf.p, s);
    QSB_NCCL(nccl().group_start());
    QSB_NCCL(nccl().send(c->sendbuf.p, (size_t)(cnt * amp), ncclUint8, peer, c->comm, s));
    QSB_NCCL(nccl().recv(c->recvbuf.p, (size_t)(cnt * amp), ncclUint8, peer, c->comm, s));
    QSB_NCCL(nccl().group_end());
    launch_slice_unpack(recv->c64, recv->amps.p, pos, recv_c ? 1 : 0, first, cnt, c->recvbuf.p, s);
  }
  cudaEventRecord(c->e1, s);
  QSB_CUDA(cudaGetLastError());
  c->bytes_sent += half * amp;
  c->exchanges++;
  return QSB_OK;
}

// A remap of k global positions (1..3) with local positions lpos[0..k) among the 2^k
// ranks peers[0 .. 2^k) (peers[x]: the rank whose remapped global bits are x; this rank
// is peers[self]).  For every x != self this rank sends its region x (local bits at lpos
// == x) to peers[x] and receives peers[x]'s region `self` into its own region x: one
// grouped ncclSend / ncclRecv round per chunk, all 2^k - 1 peers in flight at once, in
// place (a chunk is packed before the same chunk is overwritten).  Moves (1 - 2^-k) of
// the slice per rank where k separate pairwise exchanges move k / 2.
int32_t qsb_comm_remap(qsb_comm c, qsb_state st, int32_t k, const int32_t* lpos, const int32_t* peers,
                       int32_t self) {
  if (!c || check_state(st) || !peers) return fail(QSB_ERR_ARG, "null argument");
  if (int rc = check_remap(st, k, lpos)) return rc;
  const int m = 1 << k;
  if (self < 0 || self >= m || peers[self] != c->rank) return fail(QSB_ERR_ARG, "peers[self] must be this rank");
  for (int x = 0; x < m; ++x)
    if (peers[x] < 0 || peers[x] >= c->nranks) return fail(QSB_ERR_ARG, "peer out of range");
  DeviceGuard g(c->ctx->device);
  int lp[3];
  for (int i = 0; i < k; ++i) lp[i] = lpos[i];
  const int64_t amp = st->c64 ? 8 : 16;
  const int64_t region = 1ll << (st->n - k);
  const int64_t per = std::max<int64_t>(1, std::min<int64_t>(region, c->chunk_bytes / amp));
  QSB_CUDA(c->sendbuf.ensure(per * amp * (m - 1)));
  QSB_CUDA(c->recvbuf.ensure(per * amp * (m - 1)));
  char* sb = (char*)c->sendbuf.p;
  char* rb = (char*)c->recvbuf.p;
  cudaStream_t s = c->ctx->stream;
  cudaEventRecord(c->e0, s);
  for (int64_t first = 0; first < region; first += per) {
    const int64_t cnt = std::min(per, region - first);
    for (int x = 0, j = 0; x < m; ++x)
      if (x != self) launch_slice_pack_sub(st->c64, st->amps.p, k, lp, x, first, cnt, sb + (j++) * per * amp, s);
    QSB_NCCL(nccl().group_start());
    for (int x = 0, j = 0; x < m; ++x) {
      if (x == self) continue;
      QSB_NCCL(nccl().send(sb + j * per * amp, (size_t)(cnt * amp), ncclUint8, peers[x], c->comm, s));
      QSB_NCCL(nccl().recv(rb + j * per * amp, (size_t)(cnt * amp), ncclUint8, peers[x], c->comm, s));
      ++j;
    }
    QSB_NCCL(nccl().group_end());
    for (int x = 0, j = 0; x < m; ++x)
      if (x != self) launch_slice_unpack_sub(st->c64, st->amps.p, k, lp, x, first, cnt, rb + (j++) * per * amp, s);
  }
  cudaEventRecord(c->e1, s);
  QSB_CUDA(cudaGetLastError());
  c->bytes_sent += (int64_t)(m - 1) * region * amp;
  c->exchanges++;
  return QSB_OK;
}

// bytes sent by this rank's exchanges, their number, all-gathers, and the CUDA-event time
// of the last exchange (synchronises the stream)
int32_t qsb_comm_stats(qsb_comm c, int64_t* out3, double* last_exchange_ms) {
  if (!c) return fail(QSB_ERR_ARG, "null comm");
  if (out3) {
    out3[0] = c->bytes_sent;
    out3[1] = c->exchanges;
    out3[2] = c->allgathers;
  }
  if (last_exchange_ms) {
    DeviceGuard g(c->ctx->device);
    QSB_CUDA(cudaStreamSynchronize(c->ctx->stream));
    float ms = 0;
    *last_exchange_ms = c->exchanges && cudaEventElapsedTime(&ms, c->e0, c->e1) == cudaSuccess ? ms : 0.0;
  }
  return QSB_OK;
}

int32_t qsb_comm_nccl_version(int32_t* version) {
  if (!nccl().ok) return fail(QSB_ERR_UNSUPPORTED, "libnccl.so.2 not available");
  int v = 0;
  QSB_NCCL(nccl().version(&v));
  *version = v;
  return QSB_OK;
}

}  // extern "C"
