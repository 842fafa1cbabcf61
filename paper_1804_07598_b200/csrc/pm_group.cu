// pm_group.cu -- multi-GPU groups behind the C-ABI: map() and ghost_get<>()
// (SURVEY §8(b) pm_map / pm_ghost_get / pm_nccl_unique_id / pm_create_dist;
// §8(e)).
//
// PAPER.md:62 (§3.1): the domain is split into sub-domains, each extended by
// a ghost layer of interaction width; PAPER.md:112-118 (§3.4): map() sends
// the particles that left a sub-domain to the processor that owns them and
// ghost_get() fills the ghost layers ("mappings that only communicate",
// non-blocking point-to-point messages); Listing 4.1 calls
// map() and ghost_get<>() every step.
//
// A group is the set of sub-domains of one px x py x pz cuboid decomposition
// (pm_set_decomposition).  Its members are pm_ctx contexts; a process owns
// one member per rank (pm_create_dist: one GPU per process, a library-owned
// NCCL communicator) or all of them (pm_create_dist_local: the in-process
// loopback group of SURVEY C2 -- P sub-domains on one GPU, messages as device
// copies, or through NCCL self-communication when asked).  Every group call
// is collective: each member calls it once, in the same order, and the last
// local member to call performs the work for all local members (so one host
// thread can drive a loopback group member by member, and a process with one
// member per rank just works).
//
// Message protocol (identical to the host reference in dist.py, which the
// gloo tests check): directions d = (ax+1) + 3 (ay+1) + 9 (az+1), d != 13;
// a direction exists when every nonzero component is along an axis with >= 2
// sub-domains; records are packed in the order "peer ascending, then
// direction"; per message round, first the record counts (int64 per peer),
// then one payload per (sender, receiver) pair, received concatenated in
// ascending sender order.  NCCL matches sends and receives between two ranks
// in issue order: both sides issue them in ascending (sender, receiver)
// sub-domain order inside one ncclGroupStart/End.
//
// The particle work (selection, packing, unpacking, cell lists, Verlet rows,
// forces, integration) is the single-context kernels behind pm_dist_*; this
// file only decides who talks to whom and moves bytes.  pm_dist_run enqueues
// its steps in batches: the rebuild flags are reduced on the device into
// State::hold (NCCL MAX across ranks, a one-thread kernel across local
// members), step kernels of held steps return at once, and the host
// synchronises once per batch (run_batched).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pm.h"

namespace pm {
cudaStream_t ctx_stream(pm_ctx c);
int ctx_device(pm_ctx c);
bool ctx_decomposed(pm_ctx c);
bool ctx_forces_valid(pm_ctx c);
bool ctx_list_valid(pm_ctx c);
bool ctx_ready(pm_ctx c);
pm_status ctx_error(pm_ctx c, pm_status code, const char *msg);
int *ctx_flag_ptr(pm_ctx c);
int *ctx_hold_ptr(pm_ctx c);
const long long *ctx_steps_ptr(pm_ctx c);
void launch_group_hold(pm_ctx const *cs, int m, cudaStream_t s);
bool ctx_profiling(pm_ctx c);
void ctx_add_force_profile(pm_ctx c, double ms, int64_t launches);
pm_status dist_plan_async(pm_ctx c, int32_t what, const int32_t order[26]);
pm_status dist_plan_complete(pm_ctx c, int64_t counts[27]);
pm_status dist_finish_async(pm_ctx c);
pm_status dist_finish_complete(pm_ctx c);
pm_status ctx_step_half(pm_ctx c, float dt, int final_step, int wphase, cudaStream_t s);
pm_status ctx_refresh_unpack_on(pm_ctx c, const void *recv, cudaStream_t s);
void group_detach(pm_ctx c);
}  // namespace pm

namespace {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time: the one torch already loaded when present
// (RTLD_NOLOAD), else the system library.  No link-time dependency, so the
// library loads on machines without NCCL (single-GPU use).
struct Nccl {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl &nccl() {
  static Nccl N;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (N.tried) return N;
  N.tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return N;
#define PM_SYM(field, name) N.field = reinterpret_cast<decltype(N.field)>(dlsym(h, name))
  PM_SYM(GetUniqueId, "ncclGetUniqueId");
  PM_SYM(CommInitRank, "ncclCommInitRank");
  PM_SYM(CommDestroy, "ncclCommDestroy");
  PM_SYM(GroupStart, "ncclGroupStart");
  PM_SYM(GroupEnd, "ncclGroupEnd");
  PM_SYM(Send, "ncclSend");
  PM_SYM(Recv, "ncclRecv");
  PM_SYM(AllReduce, "ncclAllReduce");
  PM_SYM(GetErrorString, "ncclGetErrorString");
#undef PM_SYM
  N.ok = N.GetUniqueId && N.CommInitRank && N.CommDestroy && N.GroupStart && N.GroupEnd &&
         N.Send && N.Recv && N.AllReduce && N.GetErrorString;
  return N;
}

// ---------------------------------------------------------------------------
constexpr int kSelf = 13;

struct Dirs {
  int a[27][3];
  Dirs() {
    for (int d = 0; d < 27; ++d) {
      a[d][0] = d % 3 - 1;
      a[d][1] = (d / 3) % 3 - 1;
      a[d][2] = d / 9 - 1;
    }
  }
};
const Dirs kDirs;

enum Op { kOpNone = 0, kOpMap, kOpGhost, kOpRun, kOpThermo };

struct Member {
  pm_ctx ctx = nullptr;
  int sd = -1;  // sub-domain index (cx + px (cy + py cz))
  std::vector<int> peers;               // ascending
  std::vector<int> order;               // 26 directions, send order
  std::vector<int64_t> seg_off, seg_n;  // send segment per peer (records)
  std::vector<int64_t> recv_n;          // records received per peer
  std::vector<int64_t> ghost_seg_n, ghost_recv_n;  // the last GHOST round (refresh)
  void *sbuf = nullptr, *rbuf = nullptr;
  size_t scap = 0, rcap = 0;
  int64_t *d_cnt = nullptr;  // [2][26] device: counts sent / received (NCCL)
  int64_t *h_cnt = nullptr;  // pinned mirror
  int flag = 0;              // last local rebuild flag
  // fused ghost refresh (the sweep's epilogue stores into the peers' ghost
  // slots): this member's ghost slots, per send entry (peer, receiver slot)
  int *d_slots = nullptr, *d_dst_peer = nullptr, *d_dst_slot = nullptr;
  size_t slots_cap = 0, dst_cap = 0, dst2_cap = 0;
  std::vector<uint8_t> peer_handles;  // IPC handles the peers' buffers were opened from
  std::vector<void *> peer_p0, peer_p1;
  pm_run_stats stats{};
  double thermo[5] = {0, 0, 0, 0, 0};
};

struct Group {
  int grid[3] = {1, 1, 1};
  int P = 1;
  int nranks = 1, rank = 0;
  std::vector<int> owner;  // sub-domain -> rank
  std::vector<Member> m;   // local members
  ncclComm_t comm = nullptr;
  bool via_nccl = false;   // local messages through NCCL self-communication (tests)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int device = 0;
  int op = kOpNone, entered = 0;
  float run_dt = 0.f;
  int64_t run_steps = 0;
  int *d_flag = nullptr;
  int *h_flag = nullptr;     // pinned: [0] flag, then (need_rebuild, abort) per member
  std::vector<cudaEvent_t> ev;  // sweep timing (profiling)
  double *d_red = nullptr;
  double *h_red = nullptr;
  int64_t rebuilds = 0;
  bool fused = false;       // fused ghost refresh enabled (PM_GROUP_FUSED, default 1)
  bool overlap = false;     // message refresh overlapped with interior forces (PM_GROUP_OVERLAP=1)
  int batch = 4;            // steps enqueued per host synchronisation (PM_GROUP_BATCH)
  unsigned char *h_bat = nullptr;  // pinned: per member (hold, need, abort, -, steps_done)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_unpacked = nullptr;
  bool fused_ready = false; // set up for the current ghost layout
  uint8_t *d_handles = nullptr;  // NCCL all-gather of the members' IPC handles
  uint8_t *h_handles = nullptr;

  int coord(int sd, int d) const {
    return d == 0 ? sd % grid[0] : d == 1 ? (sd / grid[0]) % grid[1] : sd / (grid[0] * grid[1]);
  }
  bool valid_dir(int d) const {
    if (d == kSelf) return false;
    for (int k = 0; k < 3; ++k)
      if (kDirs.a[d][k] != 0 && grid[k] < 2) return false;
    return true;
  }
  int peer(int sd, int d) const {
    int c[3];
    for (int k = 0; k < 3; ++k) {
      c[k] = coord(sd, k) + kDirs.a[d][k];
      c[k] = ((c[k] % grid[k]) + grid[k]) % grid[k];
    }
    return c[0] + grid[0] * (c[1] + grid[1] * c[2]);
  }
  bool local(int sd) const { return owner[sd] == rank; }
  Member *member_of(int sd) {
    for (auto &x : m)
      if (x.sd == sd) return &x;
    return nullptr;
  }
};

std::mutex g_mu;
std::map<pm_ctx, std::pair<Group *, int>> g_members;  // ctx -> (group, local index)

void setup_member_tables(Group &G, Member &M) {
  std::vector<int> valid;
  for (int d = 0; d < 27; ++d)
    if (G.valid_dir(d)) valid.push_back(d);
  std::vector<int> peers;
  for (int d : valid) peers.push_back(G.peer(M.sd, d));
  std::sort(peers.begin(), peers.end());
  peers.erase(std::unique(peers.begin(), peers.end()), peers.end());
  M.peers = peers;
  std::vector<int> order = valid;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const int pa = G.peer(M.sd, a), pb = G.peer(M.sd, b);
    return pa != pb ? pa < pb : a < b;
  });
  for (int d = 0; d < 27; ++d)
    if (d != kSelf && std::find(valid.begin(), valid.end(), d) == valid.end()) order.push_back(d);
  M.order = order;
  const size_t np = peers.size();
  M.seg_off.assign(np, 0);
  M.seg_n.assign(np, 0);
  M.recv_n.assign(np, 0);
  M.ghost_seg_n.assign(np, 0);
  M.ghost_recv_n.assign(np, 0);
}

int peer_index(const Member &M, int q) {
  for (size_t k = 0; k < M.peers.size(); ++k)
    if (M.peers[k] == q) return (int)k;
  return -1;
}

pm_status cuda_err(pm_ctx c, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return PM_OK;
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return pm::ctx_error(c, e == cudaErrorMemoryAllocation ? PM_E_NOMEM : PM_E_CUDA, buf);
}

pm_status nccl_err(pm_ctx c, ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return PM_OK;
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s: %s", what, nccl().GetErrorString(r));
  return pm::ctx_error(c, PM_E_NCCL, buf);
}

pm_status ensure_buf(pm_ctx c, void **p, size_t *cap, size_t need) {
  if (need <= *cap && *p) return PM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const size_t n = std::max<size_t>(need + need / 4, 256);
  pm_status s = cuda_err(c, cudaMalloc(p, n), "group buffer");
  if (!s) *cap = n;
  return s;
}

// Does a message between these two sub-domains go through NCCL?
bool via_nccl(const Group &G, int a, int b) {
  return G.comm && (!G.local(a) || !G.local(b) || G.via_nccl);
}

// Record counts of one round: every local sender's counts reach its peers.
pm_status exchange_counts(Group &G, std::vector<std::vector<int64_t>> &send_n) {
  // local pairs on the host
  for (auto &R : G.m)
    for (size_t k = 0; k < R.peers.size(); ++k) R.recv_n[k] = -1;
  for (size_t r = 0; r < G.m.size(); ++r) {
    Member &R = G.m[r];
    for (size_t k = 0; k < R.peers.size(); ++k) {
      const int q = R.peers[k];
      if (via_nccl(G, R.sd, q)) continue;
      Member *Q = G.member_of(q);
      Q->recv_n[peer_index(*Q, R.sd)] = send_n[r][k];
    }
  }
  if (!G.comm) return PM_OK;
  // the rest through NCCL (device int64 per pair), ascending (sender, receiver)
  bool any = false;
  for (size_t r = 0; r < G.m.size(); ++r) {
    Member &R = G.m[r];
    for (size_t k = 0; k < R.peers.size(); ++k) R.h_cnt[k] = send_n[r][k];
    cudaError_t e = cudaMemcpyAsync(R.d_cnt, R.h_cnt, sizeof(int64_t) * 26,
                                    cudaMemcpyHostToDevice, G.stream);
    if (e != cudaSuccess) return cuda_err(R.ctx, e, "counts");
  }
  Nccl &N = nccl();
  N.GroupStart();
  for (int a = 0; a < G.P; ++a) {    // sender a
    for (int b = 0; b < G.P; ++b) {  // receiver b
      if (!via_nccl(G, a, b)) continue;
      Member *A = G.local(a) ? G.member_of(a) : nullptr;
      Member *Bm = G.local(b) ? G.member_of(b) : nullptr;
      const int ka = A ? peer_index(*A, b) : -1;
      const int kb = Bm ? peer_index(*Bm, a) : -1;
      if (A && ka >= 0) {
        N.Send(A->d_cnt + ka, 1, ncclInt64, G.owner[b], G.comm, G.stream);
        any = true;
      }
      if (Bm && kb >= 0) {
        N.Recv(Bm->d_cnt + 26 + kb, 1, ncclInt64, G.owner[a], G.comm, G.stream);
        any = true;
      }
    }
  }
  pm_status s = nccl_err(G.m[0].ctx, N.GroupEnd(), "count exchange");
  if (s || !any) return s;
  for (auto &R : G.m) {
    cudaError_t e = cudaMemcpyAsync(R.h_cnt + 26, R.d_cnt + 26, sizeof(int64_t) * 26,
                                    cudaMemcpyDeviceToHost, G.stream);
    if (e != cudaSuccess) return cuda_err(R.ctx, e, "counts");
  }
  cudaError_t e = cudaStreamSynchronize(G.stream);
  if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "counts");
  for (auto &R : G.m)
    for (size_t k = 0; k < R.peers.size(); ++k)
      if (via_nccl(G, R.peers[k], R.sd)) R.recv_n[k] = R.h_cnt[26 + k];
  return PM_OK;
}

// Offset (records) of sender a's segment among receiver R's arrivals.
int64_t recv_offset(const Member &R, int a) {
  int64_t off = 0;
  for (size_t k = 0; k < R.peers.size(); ++k) {
    if (R.peers[k] == a) return off;
    off += R.recv_n[k];
  }
  return -1;
}

// Payloads: member r's segment for peer q -> q's receive buffer at r's offset
// (on stream s: the group stream, or the overlap's communication stream).
pm_status exchange_payload(Group &G, size_t rec, cudaStream_t s) {
  for (auto &R : G.m) {  // local pairs: device copies
    for (size_t k = 0; k < R.peers.size(); ++k) {
      const int q = R.peers[k];
      if (via_nccl(G, R.sd, q) || R.seg_n[k] == 0) continue;
      Member *Q = G.member_of(q);
      const int64_t off = recv_offset(*Q, R.sd);
      cudaError_t e = cudaMemcpyAsync(static_cast<char *>(Q->rbuf) + off * rec,
                                      static_cast<char *>(R.sbuf) + R.seg_off[k] * rec,
                                      R.seg_n[k] * rec, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return cuda_err(R.ctx, e, "payload copy");
    }
  }
  if (!G.comm) return PM_OK;
  Nccl &N = nccl();
  N.GroupStart();
  for (int a = 0; a < G.P; ++a) {
    for (int b = 0; b < G.P; ++b) {
      if (!via_nccl(G, a, b)) continue;
      Member *A = G.local(a) ? G.member_of(a) : nullptr;
      Member *Bm = G.local(b) ? G.member_of(b) : nullptr;
      const int ka = A ? peer_index(*A, b) : -1;
      const int kb = Bm ? peer_index(*Bm, a) : -1;
      if (A && ka >= 0 && A->seg_n[ka] > 0)
        N.Send(static_cast<char *>(A->sbuf) + A->seg_off[ka] * rec, A->seg_n[ka] * rec,
               ncclUint8, G.owner[b], G.comm, s);
      if (Bm && kb >= 0 && Bm->recv_n[kb] > 0)
        N.Recv(static_cast<char *>(Bm->rbuf) + recv_offset(*Bm, a) * rec, Bm->recv_n[kb] * rec,
               ncclUint8, G.owner[a], G.comm, s);
    }
  }
  return nccl_err(G.m[0].ctx, N.GroupEnd(), "payload exchange");
}

// plan -> pack -> counts -> payload -> unpack of one MIGRATE / GHOST round.
pm_status message_round(Group &G, int what) {
  const size_t rec = (size_t)pm_record_bytes(what);
  std::vector<std::vector<int64_t>> send_n(G.m.size());
  for (auto &R : G.m) {  // every member's plan, then one synchronisation
    pm_status s = pm::dist_plan_async(R.ctx, what, R.order.data());
    if (s) return s;
  }
  cudaError_t e = cudaStreamSynchronize(G.stream);
  if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "plan");
  for (size_t r = 0; r < G.m.size(); ++r) {
    Member &R = G.m[r];
    int64_t counts[27];
    pm_status s = pm::dist_plan_complete(R.ctx, counts);
    if (s) return s;
    int64_t off = 0;
    for (size_t k = 0; k < R.peers.size(); ++k) {
      R.seg_off[k] = off;
      R.seg_n[k] = 0;
      for (int d : R.order)
        if (G.valid_dir(d) && G.peer(R.sd, d) == R.peers[k]) R.seg_n[k] += counts[d];
      off += R.seg_n[k];
    }
    if ((s = ensure_buf(R.ctx, &R.sbuf, &R.scap, (size_t)off * rec))) return s;
    if ((s = pm_dist_pack(R.ctx, what, off ? R.sbuf : nullptr))) return s;
    send_n[r] = R.seg_n;
  }
  pm_status s = exchange_counts(G, send_n);
  if (s) return s;
  for (auto &R : G.m) {
    int64_t tot = 0;
    for (int64_t v : R.recv_n) tot += v;
    if ((s = ensure_buf(R.ctx, &R.rbuf, &R.rcap, (size_t)tot * rec))) return s;
  }
  if ((s = exchange_payload(G, rec, G.stream))) return s;
  for (auto &R : G.m) {
    int64_t tot = 0;
    for (int64_t v : R.recv_n) tot += v;
    if ((s = pm_dist_unpack(R.ctx, what, tot ? R.rbuf : nullptr, tot))) return s;
    if (what == PM_MSG_GHOST) {
      R.ghost_seg_n = R.seg_n;
      R.ghost_recv_n = R.recv_n;
    }
  }
  return PM_OK;
}

// Positions-only ghost refresh with the last GHOST round's layout (16 B per
// ghost, "only the properties that are needed").  pack on the
// group stream; with `overlap` the exchange and the unpack run on the
// communication stream (the caller runs the interior forces meanwhile and
// waits on ev_unpacked before the boundary forces).
pm_status refresh(Group &G, bool overlap = false) {
  const size_t rec = (size_t)pm_record_bytes(PM_MSG_REFRESH);
  pm_status s;
  for (auto &R : G.m) {
    int64_t off = 0;
    for (size_t k = 0; k < R.peers.size(); ++k) {
      R.seg_off[k] = off;
      R.seg_n[k] = R.ghost_seg_n[k];
      off += R.seg_n[k];
    }
    R.recv_n = R.ghost_recv_n;
    if ((s = ensure_buf(R.ctx, &R.sbuf, &R.scap, (size_t)off * rec))) return s;
    if ((s = pm_dist_refresh_pack(R.ctx, off ? R.sbuf : nullptr))) return s;
    int64_t tot = 0;
    for (int64_t v : R.recv_n) tot += v;
    if ((s = ensure_buf(R.ctx, &R.rbuf, &R.rcap, (size_t)tot * rec))) return s;
  }
  cudaStream_t cs = G.stream;
  if (overlap) {
    cudaEventRecord(G.ev_packed, G.stream);
    cudaStreamWaitEvent(G.comm_stream, G.ev_packed, 0);
    cs = G.comm_stream;
  }
  if ((s = exchange_payload(G, rec, cs))) return s;
  for (auto &R : G.m) {
    int64_t tot = 0;
    for (int64_t v : R.recv_n) tot += v;
    if ((s = overlap ? pm::ctx_refresh_unpack_on(R.ctx, tot ? R.rbuf : nullptr, cs)
                     : pm_dist_refresh_unpack(R.ctx, tot ? R.rbuf : nullptr)))
      return s;
  }
  if (overlap) cudaEventRecord(G.ev_unpacked, G.comm_stream);
  return PM_OK;
}

__global__ void k_fill_i32(int *p, int64_t n, int v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

pm_status ensure_i32(pm_ctx c, int **p, size_t *cap, size_t need) {
  if (need <= *cap && *p) return PM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const size_t n = std::max<size_t>(need + need / 4, 64);
  pm_status s = cuda_err(c, cudaMalloc((void **)p, n * sizeof(int)), "fused refresh tables");
  if (!s) *cap = n;
  return s;
}

// Fused ghost refresh ("the K6 epilogue ... stores straight
// into peer windows"): after a rebuild every member registers, per entry of
// its ghost send list, the receiving peer and the receiver's ghost slot (the
// receiver's arrival order: the ghost round reversed) and the peers' two
// position buffers -- same-process pointers for local peers, CUDA IPC
// mappings (handles all-gathered over NCCL) for peers in other processes.
// From then on the force sweep's velocity-Verlet epilogue writes x(s+1) of
// every sent particle into the peers' next position buffer: no pack, no
// message, no unpack per step; the per-step flag all-reduce orders it before
// the peers' next sweep.
pm_status setup_fused(Group &G) {
  pm_status s;
  for (auto &R : G.m) {  // ghost slots in arrival order
    int64_t ng = 0;
    for (int64_t v : R.ghost_recv_n) ng += v;
    if ((s = ensure_i32(R.ctx, &R.d_slots, &R.slots_cap, (size_t)ng + 1))) return s;
    if ((s = pm_dist_ghost_slots(R.ctx, ng ? R.d_slots : nullptr))) return s;
  }
  // peers' position buffers: local pointers, or IPC across processes
  const bool remote = G.comm && G.nranks > 1;
  if (remote) {
    Member &R = G.m[0];  // one member per rank
    uint8_t mine[128];
    if ((s = pm_dist_ipc_handles(R.ctx, mine))) return s;
    std::memcpy(G.h_handles + 128 * G.rank, mine, 128);
    cudaMemcpyAsync(G.d_handles + 128 * G.rank, mine, 128, cudaMemcpyHostToDevice, G.stream);
    Nccl &N = nccl();
    N.GroupStart();
    for (int r = 0; r < G.nranks; ++r)  // all-gather as point-to-point (no extra API)
      if (r != G.rank) {
        N.Send(G.d_handles + 128 * G.rank, 128, ncclUint8, r, G.comm, G.stream);
        N.Recv(G.d_handles + 128 * r, 128, ncclUint8, r, G.comm, G.stream);
      }
    if ((s = nccl_err(R.ctx, N.GroupEnd(), "IPC handle exchange"))) return s;
    cudaMemcpyAsync(G.h_handles, G.d_handles, 128 * (size_t)G.nranks, cudaMemcpyDeviceToHost,
                    G.stream);
    cudaError_t e = cudaStreamSynchronize(G.stream);
    if (e != cudaSuccess) return cuda_err(R.ctx, e, "IPC handle exchange");
    std::vector<uint8_t> all(G.h_handles, G.h_handles + 128 * (size_t)G.nranks);
    if (all != R.peer_handles) {  // (re)open when any rank reallocated
      if ((s = pm_dist_ipc_close_all(R.ctx))) return s;
      R.peer_p0.assign(R.peers.size(), nullptr);
      R.peer_p1.assign(R.peers.size(), nullptr);
      for (size_t k = 0; k < R.peers.size(); ++k)
        if ((s = pm_dist_ipc_open(R.ctx, G.h_handles + 128 * G.owner[R.peers[k]], &R.peer_p0[k],
                                  &R.peer_p1[k])))
          return s;
      R.peer_handles = all;
    }
  } else {
    for (auto &R : G.m) {
      R.peer_p0.assign(R.peers.size(), nullptr);
      R.peer_p1.assign(R.peers.size(), nullptr);
      for (size_t k = 0; k < R.peers.size(); ++k)
        if ((s = pm_dist_pos_buffers(G.member_of(R.peers[k])->ctx, &R.peer_p0[k],
                                     &R.peer_p1[k])))
          return s;
    }
  }
  // per send entry: peer index and the receiver's slot
  for (auto &R : G.m) {
    int64_t nsend = 0;
    for (int64_t v : R.ghost_seg_n) nsend += v;
    if ((s = ensure_i32(R.ctx, &R.d_dst_peer, &R.dst_cap, (size_t)nsend + 1))) return s;
    if ((s = ensure_i32(R.ctx, &R.d_dst_slot, &R.dst2_cap, (size_t)nsend + 1))) return s;
    int64_t off = 0;
    for (size_t k = 0; k < R.peers.size(); ++k) {
      const int64_t n = R.ghost_seg_n[k];
      if (n > 0) {
        k_fill_i32<<<(unsigned)((n + 255) / 256), 256, 0, G.stream>>>(R.d_dst_peer + off, n,
                                                                    (int)k);
        if (!remote) {
          Member *Q = G.member_of(R.peers[k]);
          const int64_t ro = recv_offset(*Q, R.sd);
          cudaMemcpyAsync(R.d_dst_slot + off, Q->d_slots + ro, n * sizeof(int),
                          cudaMemcpyDeviceToDevice, G.stream);
        }
      }
      off += n;
    }
  }
  if (remote) {  // the receivers hand their slot slices back (the ghost round reversed)
    Nccl &N = nccl();
    Member &R = G.m[0];
    N.GroupStart();
    int64_t off = 0;
    for (size_t k = 0; k < R.peers.size(); ++k) {
      const int q = R.peers[k];
      const int64_t n_out = R.ghost_recv_n[k], n_in = R.ghost_seg_n[k];
      if (n_out > 0)
        N.Send(R.d_slots + recv_offset(R, q), n_out, ncclInt32, G.owner[q], G.comm, G.stream);
      if (n_in > 0) N.Recv(R.d_dst_slot + off, n_in, ncclInt32, G.owner[q], G.comm, G.stream);
      off += n_in;
    }
    if ((s = nccl_err(R.ctx, N.GroupEnd(), "ghost slot exchange"))) return s;
  }
  for (auto &R : G.m) {
    std::vector<void *> p0 = R.peer_p0, p1 = R.peer_p1;
    if ((s = pm_dist_peer_setup(R.ctx, (int32_t)R.peers.size(), p0.data(), p1.data(),
                                R.d_dst_peer, R.d_dst_slot)))
      return s;
  }
  G.fused_ready = true;
  return PM_OK;
}

// Global MAX of the local rebuild flags (NCCL all-reduce across ranks).
pm_status allreduce_flag(Group &G, int *flag) {
  int f = 0;
  for (auto &R : G.m) f = std::max(f, R.flag);
  if (G.comm && G.nranks > 1) {
    *G.h_flag = f;
    cudaMemcpyAsync(G.d_flag, G.h_flag, sizeof(int), cudaMemcpyHostToDevice, G.stream);
    pm_status s = nccl_err(G.m[0].ctx,
                           nccl().AllReduce(G.d_flag, G.d_flag, 1, ncclInt32, ncclMax, G.comm,
                                            G.stream),
                           "flag all-reduce");
    if (s) return s;
    cudaMemcpyAsync(G.h_flag, G.d_flag, sizeof(int), cudaMemcpyDeviceToHost, G.stream);
    cudaError_t e = cudaStreamSynchronize(G.stream);
    if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "flag all-reduce");
    f = *G.h_flag;
  }
  *flag = f;
  return PM_OK;
}

// The per-step rebuild decision with ONE host synchronisation: the local
// flags (State::need_rebuild) are MAX-reduced in place across ranks by NCCL,
// then every member's (need_rebuild, abort) pair comes back in one copy each
// and the flags are cleared on the device.
pm_status step_flag(Group &G, int *flag) {
  if (G.comm && G.nranks > 1) {  // one member per rank
    pm_status s = nccl_err(G.m[0].ctx,
                           nccl().AllReduce(pm::ctx_flag_ptr(G.m[0].ctx),
                                            pm::ctx_flag_ptr(G.m[0].ctx), 1, ncclInt32, ncclMax,
                                            G.comm, G.stream),
                           "flag all-reduce");
    if (s) return s;
  }
  for (size_t k = 0; k < G.m.size(); ++k) {
    cudaError_t e = cudaMemcpyAsync(G.h_flag + 2 + 2 * k, pm::ctx_flag_ptr(G.m[k].ctx),
                                    2 * sizeof(int), cudaMemcpyDeviceToHost, G.stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(pm::ctx_flag_ptr(G.m[k].ctx), 0, sizeof(int),
                                              G.stream);
    if (e != cudaSuccess) return cuda_err(G.m[k].ctx, e, "rebuild flag");
  }
  cudaError_t e = cudaStreamSynchronize(G.stream);
  if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "rebuild flag");
  int f = 0;
  for (size_t k = 0; k < G.m.size(); ++k) {
    if (G.h_flag[3 + 2 * k]) {  // a device error: let the member report it
      int dummy = 0;
      pm_status s = pm_dist_read_flag(G.m[k].ctx, &dummy);
      return s ? s : pm::ctx_error(G.m[k].ctx, PM_E_CUDA, "device error in a group step");
    }
    f = std::max(f, G.h_flag[2 + 2 * k]);
  }
  *flag = f;
  return PM_OK;
}

pm_status ensure_decomposed(Group &G) {
  for (auto &R : G.m) {
    if (G.P > 1 && !pm::ctx_decomposed(R.ctx)) {
      if (!pm::ctx_ready(R.ctx))
        return pm::ctx_error(R.ctx, PM_E_STATE, "group member: pm_set_domain / pm_set_cutoff first");
      const int32_t c[3] = {G.coord(R.sd, 0), G.coord(R.sd, 1), G.coord(R.sd, 2)};
      pm_status s = pm_set_decomposition(R.ctx, G.grid, c);
      if (s) return s;
    }
  }
  return PM_OK;
}

pm_status do_map(Group &G) {
  pm_status s = ensure_decomposed(G);
  if (s || G.P == 1) return s;  // one sub-domain: nothing leaves it (the wrap is local)
  return message_round(G, PM_MSG_MIGRATE);
}

double g_t_map = 0, g_t_ghost = 0, g_t_finish = 0, g_t_fused = 0;  // PM_GROUP_TIMING

pm_status do_ghost_get(Group &G) {
  pm_status s = ensure_decomposed(G);
  if (s) return s;
  if (G.P == 1) return pm_build_verlet(G.m[0].ctx);
  G.fused_ready = false;  // new send lists and ghost slots
  static const bool timing = std::getenv("PM_GROUP_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  if ((s = message_round(G, PM_MSG_GHOST))) return s;
  if (timing) cudaStreamSynchronize(G.stream);
  auto t1 = std::chrono::steady_clock::now();
  for (auto &R : G.m)  // cell lists + Verlet rows of every member, one synchronisation
    if ((s = pm::dist_finish_async(R.ctx))) return s;
  cudaError_t e = cudaStreamSynchronize(G.stream);
  if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "finish");
  for (auto &R : G.m)
    if ((s = pm::dist_finish_complete(R.ctx))) return s;
  auto t2 = std::chrono::steady_clock::now();
  g_t_ghost += std::chrono::duration<double, std::milli>(t1 - t0).count();
  g_t_finish += std::chrono::duration<double, std::milli>(t2 - t1).count();
  return PM_OK;
}

pm_status rebuild(Group &G) {
  auto t0 = std::chrono::steady_clock::now();
  pm_status s = do_map(G);
  if (std::getenv("PM_GROUP_TIMING")) cudaStreamSynchronize(G.stream);
  g_t_map += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                 .count();
  if (!s) s = do_ghost_get(G);
  if (!s) ++G.rebuilds;
  return s;
}

// ---------------------------------------------------------------------------
// Batched steps of pm_dist_run: after each step the rebuild flags are reduced
// on the device into every member's State::hold (NCCL MAX across ranks, a
// one-thread kernel across this process's members); the next steps' kernels
// (sweep, refresh pack / unpack) do nothing while it is set.  The host
// enqueues `batch` steps, then reads (hold, abort, steps_done) once: the steps
// that ran, and whether a rebuild (map + ghost_get) comes next.
// ---------------------------------------------------------------------------
pm_status hold_update(Group &G) {
  if (G.comm && G.nranks > 1)  // one member per rank
    return nccl_err(G.m[0].ctx,
                    nccl().AllReduce(pm::ctx_flag_ptr(G.m[0].ctx), pm::ctx_hold_ptr(G.m[0].ctx),
                                     1, ncclInt32, ncclMax, G.comm, G.stream),
                    "flag all-reduce");
  std::vector<pm_ctx> cs;
  for (auto &R : G.m) cs.push_back(R.ctx);
  pm::launch_group_hold(cs.data(), (int)cs.size(), G.stream);
  return PM_OK;
}

pm_status clear_hold(Group &G) {
  for (auto &R : G.m) {
    cudaError_t e = cudaMemsetAsync(pm::ctx_flag_ptr(R.ctx), 0, sizeof(int), G.stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(pm::ctx_hold_ptr(R.ctx), 0, sizeof(int), G.stream);
    if (e != cudaSuccess) return cuda_err(R.ctx, e, "rebuild flag");
  }
  return PM_OK;
}

// (hold, steps_done) of member 0 after everything enqueued; a device error of
// any member is reported by that member
pm_status batch_status(Group &G, int *hold, long long *steps) {
  for (size_t k = 0; k < G.m.size(); ++k) {
    unsigned char *h = G.h_bat + 32 * k;
    cudaError_t e = cudaMemcpyAsync(h, pm::ctx_hold_ptr(G.m[k].ctx), sizeof(int),
                                    cudaMemcpyDeviceToHost, G.stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h + 4, pm::ctx_flag_ptr(G.m[k].ctx), 2 * sizeof(int),
                          cudaMemcpyDeviceToHost, G.stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(h + 16, pm::ctx_steps_ptr(G.m[k].ctx), sizeof(long long),
                          cudaMemcpyDeviceToHost, G.stream);
    if (e != cudaSuccess) return cuda_err(G.m[k].ctx, e, "batch status");
  }
  cudaError_t e = cudaStreamSynchronize(G.stream);
  if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "batch status");
  for (size_t k = 0; k < G.m.size(); ++k) {
    int ab;
    std::memcpy(&ab, G.h_bat + 32 * k + 8, sizeof(int));
    if (ab) {
      int dummy = 0;
      pm_status s = pm_dist_read_flag(G.m[k].ctx, &dummy);
      return s ? s : pm::ctx_error(G.m[k].ctx, PM_E_CUDA, "device error in a group step");
    }
  }
  std::memcpy(hold, G.h_bat, sizeof(int));
  std::memcpy(steps, G.h_bat + 16, sizeof(long long));
  return PM_OK;
}

// One step enqueued for every member: the refresh (message modes), the sweep
// with the fused kick/drift (or its interior / boundary halves), profiling
// events around the sweeps.
pm_status enqueue_step(Group &G, float dt, bool last, bool do_refresh, bool fused,
                       int64_t *ev_pair) {
  pm_status s;
  bool halves = false;
  if (do_refresh) {
    halves = G.overlap && !fused;
    if ((s = refresh(G, halves))) return s;
  }
  if (ev_pair) {
    const size_t need = 2 * (size_t)(*ev_pair + 1);
    while (G.ev.size() < need) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return PM_E_CUDA;
      G.ev.push_back(e);
    }
    cudaEventRecord(G.ev[2 * *ev_pair], G.stream);
  }
  if (halves) {
    for (auto &R : G.m)
      if ((s = pm::ctx_step_half(R.ctx, dt, last, 0, G.stream))) return s;
    cudaStreamWaitEvent(G.stream, G.ev_unpacked, 0);
    for (auto &R : G.m)
      if ((s = pm::ctx_step_half(R.ctx, dt, last, 1, G.stream))) return s;
  } else {
    for (auto &R : G.m)
      if ((s = pm_dist_step(R.ctx, dt, last ? PM_PHASE_FINAL : PM_PHASE_STEP, nullptr)))
        return s;
  }
  if (ev_pair) cudaEventRecord(G.ev[2 * *ev_pair + 1], G.stream);
  return PM_OK;
}

pm_status run_batched(Group &G, float dt, int64_t nsteps, int flag, bool prof,
                      double *prof_ms) {
  pm_status s;
  const bool fused = G.fused && G.P > 1;
  int hold = 0;
  long long steps0 = 0;
  if ((s = batch_status(G, &hold, &steps0))) return s;
  int64_t k = 0, npairs = 0;
  std::vector<int64_t> pairs;
  while (k < nsteps) {
    const bool rebuilt = flag != 0;
    if (rebuilt) {
      if ((s = clear_hold(G))) return s;
      if ((s = rebuild(G))) return s;
    }
    if (fused && !G.fused_ready && (s = setup_fused(G))) return s;
    const int64_t nb = std::min<int64_t>(G.batch, nsteps - k);
    pairs.clear();
    for (int64_t j = 0; j < nb; ++j) {
      const int64_t step = k + j;
      const bool last = step == nsteps - 1;
      // after a rebuild the ghosts are current; the fused refresh stores the
      // next positions from the sweep, except after the prologue's drift
      const bool do_refresh = !(j == 0 && rebuilt) && (!fused || step == 0);
      int64_t p = npairs;
      if ((s = enqueue_step(G, dt, last, do_refresh, fused, prof ? &p : nullptr))) return s;
      if (prof) pairs.push_back(npairs++);
      if (!last && (s = hold_update(G))) return s;
    }
    long long steps1 = 0;
    if ((s = batch_status(G, &hold, &steps1))) return s;
    const int64_t ran = steps1 - steps0;
    steps0 = steps1;
    if (ran < 0 || ran > nb || (ran < nb && !hold))
      return pm::ctx_error(G.m[0].ctx, PM_E_CUDA, "group batch: inconsistent step count");
    if (prof && prof_ms)
      for (int64_t q = 0; q < ran; ++q) {
        float t = 0.f;
        cudaEventElapsedTime(&t, G.ev[2 * pairs[q]], G.ev[2 * pairs[q] + 1]);
        *prof_ms += t;
      }
    k += ran;
    flag = hold;
  }
  return clear_hold(G);
}

// Velocity-Verlet steps of the whole group in lock step (Listing 4.1's loop,
// PAPER.md:282-320, with the Verlet skin: map + ghost_get only when a
// particle of any sub-domain moved more than skin/2; otherwise the
// positions-only ghost refresh).
pm_status do_run(Group &G, float dt, int64_t nsteps) {
  pm_status s;
  for (auto &R : G.m) std::memset(&R.stats, 0, sizeof R.stats);
  if (G.P == 1) return pm_step_vv(G.m[0].ctx, dt, nsteps, &G.m[0].stats);
  if (nsteps <= 0) return PM_OK;
  bool need_forces = false;
  for (auto &R : G.m) need_forces |= !pm::ctx_forces_valid(R.ctx) || !pm::ctx_list_valid(R.ctx);
  if (need_forces) {
    for (auto &R : G.m)
      if (!pm::ctx_list_valid(R.ctx)) {
        if ((s = rebuild(G))) return s;
        break;
      }
    for (auto &R : G.m)
      if ((s = pm_dist_step(R.ctx, dt, PM_PHASE_FORCES, nullptr))) return s;
  }
  const int64_t reb0 = G.rebuilds;
  for (auto &R : G.m)
    if ((s = pm_dist_step(R.ctx, dt, PM_PHASE_PROLOGUE, &R.flag))) return s;
  int flag = 0;
  if ((s = allreduce_flag(G, &flag))) return s;
  const bool prof = pm::ctx_profiling(G.m[0].ctx);
  // (PM_GROUP_TIMING times the synchronised phases of the per-step loop)
  if (G.batch > 1 && G.m.size() <= 64 && !std::getenv("PM_GROUP_TIMING")) {
    double ms = 0.0;
    if ((s = run_batched(G, dt, nsteps, flag, prof, &ms))) return s;
    if (prof) pm::ctx_add_force_profile(G.m[0].ctx, ms, nsteps);
    for (auto &R : G.m) {
      R.stats.steps = nsteps;
      R.stats.rebuilds = G.rebuilds - reb0;
    }
    return PM_OK;
  }
  if (prof) {
    while (G.ev.size() < 2 * (size_t)nsteps) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return PM_E_CUDA;
      G.ev.push_back(e);
    }
  }
  static const bool timing = std::getenv("PM_GROUP_TIMING") != nullptr;
  using clk = std::chrono::steady_clock;
  double t_reb = 0, t_ref = 0, t_step = 0, t_flag = 0;
  g_t_map = g_t_ghost = g_t_finish = g_t_fused = 0;
  const int64_t reb_start = G.rebuilds;
  const bool fused = G.fused && G.P > 1;
  for (int64_t k = 0; k < nsteps; ++k) {
    auto t0 = clk::now();
    if (timing) cudaStreamSynchronize(G.stream);
    // message refresh overlapped with the interior slices' forces (PAPER.md:128,
    // §3.6): the exchange and unpack run on the communication stream while the
    // interior half of the sweep runs; the boundary half waits for the unpack
    bool halves = false;
    if (flag) {
      if ((s = rebuild(G))) return s;
    } else if (!fused || k == 0) {  // k = 0: the prologue's drift has no fused stores
      halves = G.overlap && !fused;
      if ((s = refresh(G, halves))) return s;
    }
    if (fused && !G.fused_ready) {
      auto tf = clk::now();
      if ((s = setup_fused(G))) return s;
      if (timing) cudaStreamSynchronize(G.stream);
      g_t_fused += std::chrono::duration<double, std::milli>(clk::now() - tf).count();
    }
    if (timing) cudaStreamSynchronize(G.stream);
    auto t1 = clk::now();
    (flag ? t_reb : t_ref) += std::chrono::duration<double, std::milli>(t1 - t0).count();
    const bool last = k == nsteps - 1;
    if (prof) cudaEventRecord(G.ev[2 * k], G.stream);
    if (halves) {
      for (auto &R : G.m)
        if ((s = pm::ctx_step_half(R.ctx, dt, last, 0, G.stream))) return s;
      cudaStreamWaitEvent(G.stream, G.ev_unpacked, 0);
      for (auto &R : G.m)
        if ((s = pm::ctx_step_half(R.ctx, dt, last, 1, G.stream))) return s;
    } else {
      for (auto &R : G.m)
        if ((s = pm_dist_step(R.ctx, dt, last ? PM_PHASE_FINAL : PM_PHASE_STEP, nullptr)))
          return s;
    }
    if (prof) cudaEventRecord(G.ev[2 * k + 1], G.stream);
    if (timing) cudaStreamSynchronize(G.stream);
    auto t2 = clk::now();
    t_step += std::chrono::duration<double, std::milli>(t2 - t1).count();
    if (last) break;
    if ((s = step_flag(G, &flag))) return s;
    t_flag += std::chrono::duration<double, std::milli>(clk::now() - t2).count();
  }
  if (timing)
    std::fprintf(stderr, "pm_dist_run %lld steps: rebuild %.3f ms, refresh %.3f ms, step %.3f ms, "
                 "flag %.3f ms (synchronised phases); rebuilds: map %.3f, ghost round "
                 "%.3f, finish %.3f, fused setup %.3f ms (%lld rebuilds)\n", (long long)nsteps,
                 t_reb, t_ref, t_step, t_flag, g_t_map, g_t_ghost, g_t_finish, g_t_fused,
                 (long long)(G.rebuilds - reb_start));
  if (prof) {  // the force sweeps (+ fused kick/drift) of the local members, per step
    cudaStreamSynchronize(G.stream);
    double ms = 0.0;
    for (int64_t k = 0; k < nsteps; ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, G.ev[2 * k], G.ev[2 * k + 1]);
      ms += t;
    }
    pm::ctx_add_force_profile(G.m[0].ctx, ms, nsteps);
  }
  for (auto &R : G.m) {
    R.stats.steps = nsteps;
    R.stats.rebuilds = G.rebuilds - reb0;
  }
  return PM_OK;
}

pm_status do_thermo(Group &G) {
  for (auto &R : G.m) {
    double ke, pe, pes, vir;
    int64_t np;
    pm_status s = pm_thermo_compute(R.ctx);
    if (!s) s = pm_get_thermo(R.ctx, &ke, &pe, &pes, &vir, &np);
    if (s) return s;
    R.thermo[0] = ke;
    R.thermo[1] = pe;
    R.thermo[2] = pes;
    R.thermo[3] = vir;
    R.thermo[4] = (double)np;
  }
  double sum[5] = {0, 0, 0, 0, 0};
  for (auto &R : G.m)
    for (int k = 0; k < 5; ++k) sum[k] += R.thermo[k];
  if (G.comm && G.nranks > 1) {
    std::memcpy(G.h_red, sum, sizeof sum);
    cudaMemcpyAsync(G.d_red, G.h_red, sizeof sum, cudaMemcpyHostToDevice, G.stream);
    pm_status s = nccl_err(G.m[0].ctx,
                           nccl().AllReduce(G.d_red, G.d_red, 5, ncclFloat64, ncclSum, G.comm,
                                            G.stream),
                           "thermo all-reduce");
    if (s) return s;
    cudaMemcpyAsync(G.h_red, G.d_red, sizeof sum, cudaMemcpyDeviceToHost, G.stream);
    cudaError_t e = cudaStreamSynchronize(G.stream);
    if (e != cudaSuccess) return cuda_err(G.m[0].ctx, e, "thermo all-reduce");
    std::memcpy(sum, G.h_red, sizeof sum);
  }
  for (auto &R : G.m) std::memcpy(R.thermo, sum, sizeof sum);
  return PM_OK;
}

// Collective entry: the last local member to enter performs `op`.
pm_status enter(pm_ctx c, int op, Group **gout, int *idx, bool *perform) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_members.find(c);
  if (it == g_members.end()) return pm::ctx_error(c, PM_E_STATE, "not a group member");
  Group *G = it->second.first;
  if (G->op != kOpNone && G->op != op)
    return pm::ctx_error(c, PM_E_STATE, "group call order differs between members");
  G->op = op;
  G->entered += 1;
  *gout = G;
  *idx = it->second.second;
  *perform = G->entered == (int)G->m.size();
  if (*perform) {
    G->op = kOpNone;
    G->entered = 0;
  }
  return PM_OK;
}

Group *new_group(const int32_t grid[3], int nranks, int rank, int device, void *stream) {
  Group *G = new Group();
  for (int d = 0; d < 3; ++d) G->grid[d] = grid[d];
  G->P = grid[0] * grid[1] * grid[2];
  G->nranks = nranks;
  G->rank = rank;
  G->device = device;
  cudaSetDevice(device);
  if (stream) {
    G->stream = (cudaStream_t)stream;
  } else {
    cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking);
    G->own_stream = true;
  }
  cudaMalloc((void **)&G->d_flag, sizeof(int));
  cudaMallocHost((void **)&G->h_flag, sizeof(int) * (2 + 2 * G->P));
  cudaMalloc((void **)&G->d_red, 8 * sizeof(double));
  cudaMallocHost((void **)&G->h_red, 8 * sizeof(double));
  cudaMalloc((void **)&G->d_handles, 128 * (size_t)std::max(nranks, 1));
  cudaMallocHost((void **)&G->h_handles, 128 * (size_t)std::max(nranks, 1));
  // fused refresh: default on in-process (verified against one context on
  // the GPU); across processes (CUDA IPC over NVLink between ranks) opt-in
  // with PM_GROUP_FUSED=1 until it has run on more than one GPU
  const char *f = std::getenv("PM_GROUP_FUSED");
  G->fused = f ? f[0] != '0' : nranks == 1;
  // overlapped message refresh (§3.6): opt-in -- splitting the
  // sweep into an interior and a boundary launch measured +0.045 ms per member
  // per step on one B200, above the exchange latency it can hide
  const char *ov = std::getenv("PM_GROUP_OVERLAP");
  G->overlap = ov && ov[0] == '1';
  // steps per host synchronisation of pm_dist_run: the step kernels check the
  // device-side hold (the previous step's global rebuild flag), so the host
  // enqueues a batch and reads the flags once (1 = the per-step loop)
  const char *bt = std::getenv("PM_GROUP_BATCH");
  G->batch = bt ? std::max(1, std::atoi(bt)) : 4;
  cudaMallocHost((void **)&G->h_bat, 32 * (size_t)std::max(G->P, 1));
  cudaStreamCreateWithFlags(&G->comm_stream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&G->ev_packed, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&G->ev_unpacked, cudaEventDisableTiming);
  return G;
}

void free_group(Group *G) {
  cudaSetDevice(G->device);
  if (G->stream) cudaStreamSynchronize(G->stream);
  for (auto &R : G->m) {
    if (R.d_slots) cudaFree(R.d_slots);
    if (R.d_dst_peer) cudaFree(R.d_dst_peer);
    if (R.d_dst_slot) cudaFree(R.d_dst_slot);
    if (R.sbuf) cudaFree(R.sbuf);
    if (R.rbuf) cudaFree(R.rbuf);
    if (R.d_cnt) cudaFree(R.d_cnt);
    if (R.h_cnt) cudaFreeHost(R.h_cnt);
  }
  if (G->comm) nccl().CommDestroy(G->comm);
  cudaFree(G->d_flag);
  cudaFreeHost(G->h_flag);
  if (G->h_bat) cudaFreeHost(G->h_bat);
  for (cudaEvent_t e : G->ev) cudaEventDestroy(e);
  cudaFree(G->d_red);
  cudaFreeHost(G->h_red);
  if (G->d_handles) cudaFree(G->d_handles);
  if (G->h_handles) cudaFreeHost(G->h_handles);
  if (G->comm_stream) {
    cudaStreamSynchronize(G->comm_stream);
    cudaStreamDestroy(G->comm_stream);
  }
  if (G->ev_packed) cudaEventDestroy(G->ev_packed);
  if (G->ev_unpacked) cudaEventDestroy(G->ev_unpacked);
  if (G->own_stream) cudaStreamDestroy(G->stream);
  delete G;
}

pm_status add_member(Group *G, const pm_opts *opts, int sd, pm_ctx *out) {
  pm_opts o;
  pm_opts_default(&o);
  if (opts) o = *opts;
  o.cuda_stream = G->stream;  // every local member on the group stream
  pm_ctx c = nullptr;
  pm_status s = pm_create(&o, &c);
  if (s) return s;
  Member M;
  M.ctx = c;
  M.sd = sd;
  setup_member_tables(*G, M);
  if (cudaMalloc((void **)&M.d_cnt, sizeof(int64_t) * 52) != cudaSuccess ||
      cudaMallocHost((void **)&M.h_cnt, sizeof(int64_t) * 52) != cudaSuccess) {
    pm_destroy(c);
    return PM_E_NOMEM;
  }
  std::memset(M.h_cnt, 0, sizeof(int64_t) * 52);
  G->m.push_back(M);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_members[c] = {G, (int)G->m.size() - 1};
  }
  *out = c;
  return PM_OK;
}

pm_status check_grid(const int32_t grid[3]) {
  if (!grid) return PM_E_INVAL;
  for (int d = 0; d < 3; ++d)
    if (grid[d] < 1 || grid[d] > 64) return PM_E_INVAL;
  return PM_OK;
}

}  // namespace

namespace pm {
// pm_destroy of a member: the group (and its communicator) goes with its last
// member.
void group_detach(pm_ctx c) {
  Group *G = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_members.find(c);
    if (it == g_members.end()) return;
    G = it->second.first;
    g_members.erase(it);
    for (auto &R : G->m)
      if (R.ctx == c) R.ctx = nullptr;
    for (auto &R : G->m)
      if (R.ctx) return;
  }
  free_group(G);
}
}  // namespace pm

extern "C" {

pm_status pm_nccl_unique_id(uint8_t id[128]) {
  if (!id) return PM_E_INVAL;
  Nccl &N = nccl();
  if (!N.ok) return PM_E_NCCL;
  ncclUniqueId u;
  if (N.GetUniqueId(&u) != ncclSuccess) return PM_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return PM_OK;
}

pm_status pm_create_dist(const pm_opts *opts, int32_t rank, int32_t nranks, const uint8_t id[128],
                         const int32_t grid[3], pm_ctx *out) {
  if (!out || !id || check_grid(grid)) return PM_E_INVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || grid[0] * grid[1] * grid[2] != nranks)
    return PM_E_INVAL;
  Nccl &N = nccl();
  if (!N.ok) return PM_E_NCCL;
  pm_opts o;
  pm_opts_default(&o);
  if (opts) o = *opts;
  Group *G = new_group(grid, nranks, rank, o.device, o.cuda_stream);
  G->owner.resize(G->P);
  for (int s = 0; s < G->P; ++s) G->owner[s] = s;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  cudaSetDevice(o.device);
  if (N.CommInitRank(&G->comm, nranks, u, rank) != ncclSuccess) {
    G->comm = nullptr;
    free_group(G);
    return PM_E_NCCL;
  }
  pm_status s = add_member(G, &o, rank, out);
  if (s) free_group(G);
  return s;
}

pm_status pm_create_dist_local(const pm_opts *opts, const int32_t grid[3], int32_t via_nccl,
                               pm_ctx *out) {
  if (!out || check_grid(grid)) return PM_E_INVAL;
  pm_opts o;
  pm_opts_default(&o);
  if (opts) o = *opts;
  Group *G = new_group(grid, 1, 0, o.device, o.cuda_stream);
  G->owner.assign(G->P, 0);
  if (via_nccl) {
    Nccl &N = nccl();
    ncclUniqueId u;
    if (!N.ok || N.GetUniqueId(&u) != ncclSuccess ||
        N.CommInitRank(&G->comm, 1, u, 0) != ncclSuccess) {
      G->comm = nullptr;
      free_group(G);
      return PM_E_NCCL;
    }
    G->via_nccl = true;
  }
  for (int sd = 0; sd < G->P; ++sd) {
    pm_status s = add_member(G, &o, sd, &out[sd]);
    if (s) {
      for (int k = 0; k < sd; ++k) pm_destroy(out[k]);  // the last one frees the group
      if (sd == 0) free_group(G);
      return s;
    }
  }
  return PM_OK;
}

pm_status pm_dist_info(pm_ctx c, int32_t *sub_domain, int32_t *nsub, int32_t *rank,
                       int32_t *nranks) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_members.find(c);
  if (it == g_members.end()) return PM_E_STATE;
  const Group *G = it->second.first;
  if (sub_domain) *sub_domain = G->m[it->second.second].sd;
  if (nsub) *nsub = G->P;
  if (rank) *rank = G->rank;
  if (nranks) *nranks = G->nranks;
  return PM_OK;
}

pm_status pm_map(pm_ctx c) {
  Group *G;
  int idx;
  bool go;
  pm_status s = enter(c, kOpMap, &G, &idx, &go);
  if (s || !go) return s;
  cudaSetDevice(G->device);
  return do_map(*G);
}

pm_status pm_ghost_get(pm_ctx c) {
  Group *G;
  int idx;
  bool go;
  pm_status s = enter(c, kOpGhost, &G, &idx, &go);
  if (s || !go) return s;
  cudaSetDevice(G->device);
  return do_ghost_get(*G);
}

pm_status pm_dist_run(pm_ctx c, float dt, int64_t nsteps, pm_run_stats *out) {
  Group *G;
  int idx;
  bool go;
  if (!(dt > 0.f) || nsteps < 0) return PM_E_INVAL;
  pm_status s = enter(c, kOpRun, &G, &idx, &go);
  if (s) return s;
  if (go) {
    cudaSetDevice(G->device);
    s = do_run(*G, dt, nsteps);
  }
  if (go && out) *out = G->m[idx].stats;
  return s;
}

pm_status pm_dist_thermo(pm_ctx c, double *ke, double *pe_raw, double *pe_shift, double *virial,
                         int64_t *npairs) {
  Group *G;
  int idx;
  bool go;
  pm_status s = enter(c, kOpThermo, &G, &idx, &go);
  if (s || !go) return s;
  cudaSetDevice(G->device);
  if ((s = do_thermo(*G))) return s;
  const double *t = G->m[idx].thermo;
  if (ke) *ke = t[0];
  if (pe_raw) *pe_raw = t[1];
  if (pe_shift) *pe_shift = t[2];
  if (virial) *virial = t[3];
  if (npairs) *npairs = (int64_t)t[4];
  return PM_OK;
}

}  // extern "C"
