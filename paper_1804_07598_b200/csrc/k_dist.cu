// k_dist.cu -- domain decomposition kernels: migration (map),
// ghost-layer selection (ghost_get) and the per-step positions-only ghost
// refresh.
//
// PAPER.md:62 (§3.1): "sub-domains are extended by a ghost layer ... The width
// of the ghost layers is given by the particle interaction radius";
// PAPER.md:114-116 (§3.4): local map() "processors only communicate to their
// neighbors", ghost_get "populates the ghost layers"; a property
// subset can be mapped -- the per-step refresh moves positions only
// (Listing 4.1 ghost_get<>()).
//
// Every per-direction message is built by a STABLE partition of the owned
// particles (block counts -> scan -> ballot ranks), so message contents and
// order -- and therefore the receiver's storage order, its cell order and
// its force summation order -- are deterministic.
//
// Direction index d = (a_x+1) + 3 (a_y+1) + 9 (a_z+1), a in {-1,0,1};
// d = 13 is "stay / self".
#include "pm_internal.cuh"

namespace pm {

namespace {

constexpr int kDirBlock = 256;
constexpr int kDirItems = 8;  // particles per thread in mark / fill

// owner coordinate along a decomposed axis: the pinned fp32 rule (like R3)
// for equal cuboids, or the number of cut positions <= x for the
// load-balanced cuts of pm_set_decomposition_cuts (exact fp32 compares)
__device__ __forceinline__ int owner_coord(const Dist &D, int d, float x) {
  if (D.cuts) {
    int c = 0;
    for (int k = 0; k < D.p[d] - 1; ++k) c += (x >= D.cut[d][k]) ? 1 : 0;
    return c;
  }
  return cell_coord(x, D.glo[d], D.inv_s[d], D.p[d]);
}

// The direction mask of one owned particle (bit d = message direction d).
__device__ __forceinline__ uint32_t dist_mask_of(const Params &P, const Bufs &B, const Dist &D,
                                                 int i, int what) {
  State *st = B.st;
  // after a build owned particles and ghost copies are interleaved in cell
  // order: ghosts belong to no message (a migration drops them)
  if (B.kind[st->cur_id][i] & kGhostBit) return 0u;
  const float4 x4 = B.pos[st->cur_pv][i];
  const float x[3] = {x4.x, x4.y, x4.z};
  uint32_t m = 0;
  if (what == 0) {  // migration: the one direction towards the new owner
    int a[3] = {0, 0, 0};
    bool bad = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (D.p[d] < 2) continue;
      const int c = owner_coord(D, d, x[d]);
      if (c == D.c[d]) continue;
      const int delta = (c - D.c[d] + D.p[d]) % D.p[d];
      if (delta == 1) a[d] = 1;
      else if (delta == D.p[d] - 1) a[d] = -1;
      else bad = true;  // moved more than one sub-domain: impossible within skin/2
    }
    if (bad) raise_error(st, -6 /*PM_E_DOMAIN*/, (long long)B.gid[st->cur_id][i]);
    m = 1u << ((a[0] + 1) + 3 * (a[1] + 1) + 9 * (a[2] + 1));
  } else {  // ghosts: every direction whose face is within the ghost width
    int lo_f[3], hi_f[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo_f[d] = D.p[d] >= 2 && __fsub_rn(x[d], D.slo[d]) < D.rg;
      hi_f[d] = D.p[d] >= 2 && __fsub_rn(D.shi[d], x[d]) < D.rg;
    }
    for (int az = -1; az <= 1; ++az) {
      if ((az == -1 && !lo_f[2]) || (az == 1 && !hi_f[2])) continue;
      for (int ay = -1; ay <= 1; ++ay) {
        if ((ay == -1 && !lo_f[1]) || (ay == 1 && !hi_f[1])) continue;
        for (int ax = -1; ax <= 1; ++ax) {
          if ((ax == -1 && !lo_f[0]) || (ax == 1 && !hi_f[0])) continue;
          const int dd = (ax + 1) + 3 * (ay + 1) + 9 * (az + 1);
          if (dd != 13) m |= 1u << dd;
        }
      }
    }
  }
  return m;
}

// pass 1: direction masks of the block's kDirItems * kDirBlock particles and
// the block's counts per direction (warp-aggregated: one shared-memory add
// per direction present in a warp)
__global__ void __launch_bounds__(kDirBlock) k_dist_mark(Params P, Bufs B, Dist D, int n_owned,
                                                         int what, uint32_t *__restrict__ mask,
                                                         int *__restrict__ blk_counts) {
  __shared__ int cnt[27];
  if (threadIdx.x < 27) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int base = blockIdx.x * (kDirBlock * kDirItems);
  for (int it = 0; it < kDirItems; ++it) {
    const int i = base + it * kDirBlock + threadIdx.x;
    const uint32_t m = (i < n_owned) ? dist_mask_of(P, B, D, i, what) : 0u;
    if (i < n_owned) mask[i] = m;
    uint32_t wm = __reduce_or_sync(0xffffffffu, m);
    while (wm) {
      const int d = __ffs(wm) - 1;
      wm &= wm - 1;
      const unsigned b = __ballot_sync(0xffffffffu, (m >> d) & 1u);
      if (lane == 0) atomicAdd(&cnt[d], __popc(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < 27) blk_counts[blockIdx.x * 27 + threadIdx.x] = cnt[threadIdx.x];
}

// pass 2: per-direction exclusive scan over blocks (one 1024-thread block per
// direction, block-wide scan of the column); totals per direction.
__global__ void __launch_bounds__(1024) k_dist_scan(int *__restrict__ blk_counts, int nblk,
                                                    long long *__restrict__ totals) {
  __shared__ int wsum[32];
  const int d = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < nblk; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int c = (b < nblk) ? blk_counts[b * 27 + d] : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const int excl = carry + (w ? wsum[w - 1] : 0) + x - c;
    if (b < nblk) blk_counts[b * 27 + d] = excl;
    carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[d] = carry;
}

// pass 3: stable write of particle indices into the per-direction lists
// direction bases in the caller's packing order (order[0..25], then 13 last);
// the block's kDirItems chunks in index order, a running offset per direction
__global__ void __launch_bounds__(kDirBlock) k_dist_fill(const uint32_t *__restrict__ mask, int n,
                                                         const int *__restrict__ blk_off,
                                                         const long long *__restrict__ totals,
                                                         const int *__restrict__ order,
                                                         int *__restrict__ dir_base_out,
                                                         int *__restrict__ list) {
  __shared__ int wsum[27][kDirBlock / 32];
  __shared__ int dir_base[27];
  __shared__ int run[27];
  if (threadIdx.x == 0) {
    long long base = 0;
    for (int k = 0; k < 26; ++k) {
      dir_base[order[k]] = (int)base;
      base += totals[order[k]];
    }
    dir_base[13] = (int)base;
    if (blockIdx.x == 0)
      for (int k = 0; k < 27; ++k) dir_base_out[k] = dir_base[k];
  }
  if (threadIdx.x < 27) run[threadIdx.x] = blk_off[blockIdx.x * 27 + threadIdx.x];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int base = blockIdx.x * (kDirBlock * kDirItems);
  for (int it = 0; it < kDirItems; ++it) {
    const int i = base + it * kDirBlock + threadIdx.x;
    const uint32_t m = (i < n) ? mask[i] : 0u;
    // only the directions present in the warp (usually "stay" plus a face or
    // two) need a ballot; the others count zero
    if (lane < 27) wsum[lane][w] = 0;
    uint32_t wm = __reduce_or_sync(0xffffffffu, m);
    while (wm) {
      const int d = __ffs(wm) - 1;
      wm &= wm - 1;
      const unsigned b = __ballot_sync(0xffffffffu, (m >> d) & 1u);
      if (lane == 0) wsum[d][w] = __popc(b);
    }
    __syncthreads();
    if (threadIdx.x < 27) {  // exclusive scan over the block's warps, per direction
      int acc = run[threadIdx.x];
      for (int k = 0; k < kDirBlock / 32; ++k) {
        const int c = wsum[threadIdx.x][k];
        wsum[threadIdx.x][k] = acc;
        acc += c;
      }
      run[threadIdx.x] = acc;
    }
    __syncthreads();
    wm = __reduce_or_sync(0xffffffffu, m);
    while (wm) {
      const int d = __ffs(wm) - 1;
      wm &= wm - 1;
      const unsigned b = __ballot_sync(0xffffffffu, (m >> d) & 1u);
      if ((m >> d) & 1u) list[dir_base[d] + wsum[d][w] + __popc(b & lt)] = i;
    }
    __syncthreads();  // wsum is rewritten by the next chunk
  }
}

// migration record: pos, vel, aux, gid, kind (64 B; aux is the SPH stepping
// state v_old, or the DEM angular velocity, zero otherwise); ghost record:
// pos, gid, kind (32 B)
struct MigRec {
  float4 pos, vel, aux;
  long long gid;
  int kind, pad;
};
struct GhostRec {
  float4 pos;
  long long gid;
  int kind, pad;
};

__global__ void k_dist_pack(Bufs B, int what, const int *__restrict__ list, int nsend,
                            void *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nsend) return;
  State *st = B.st;
  const int i = list[e];
  PM_CHECK(i >= 0);
  const int cp = st->cur_pv, ci = st->cur_id;
  if (what == 0) {
    MigRec r;
    r.pos = B.pos[cp][i];
    r.vel = B.vel[cp][i];
    r.aux = B.vold[ci]    ? B.vold[ci][i]
            : B.omega[cp] ? B.omega[cp][i]
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    r.gid = B.gid[ci][i];
    r.kind = B.kind[ci][i];
    r.pad = 0;
    reinterpret_cast<MigRec *>(out)[e] = r;
  } else {
    GhostRec r;
    r.pos = B.pos[cp][i];
    r.gid = B.gid[ci][i];
    r.kind = B.kind[ci][i] & ~kGhostBit;
    r.pad = 0;
    reinterpret_cast<GhostRec *>(out)[e] = r;
  }
}

// stayers (direction-13 list, in index order) -> alternate buffers [0, n_stay)
__global__ void k_dist_compact(Bufs B, const int *__restrict__ stay, int n_stay) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_stay) return;
  State *st = B.st;
  const int cp = st->cur_pv, ci = st->cur_id;
  const int j = stay[k];
  B.pos[cp ^ 1][k] = B.pos[cp][j];
  B.vel[cp ^ 1][k] = B.vel[cp][j];
  B.gid[ci ^ 1][k] = B.gid[ci][j];
  B.kind[ci ^ 1][k] = B.kind[ci][j];
  B.rhoP[ci ^ 1][k] = B.rhoP[ci][j];
  if (B.vold[ci]) B.vold[ci ^ 1][k] = B.vold[ci][j];
  if (B.omega[cp]) B.omega[cp ^ 1][k] = B.omega[cp][j];
}

__global__ void k_dist_unpack(Bufs B, int what, const void *__restrict__ in, int nrecv, int base) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nrecv) return;
  State *st = B.st;
  const int cp = st->cur_pv, ci = st->cur_id;
  const int k = base + e;
  if (what == 0) {
    const MigRec r = reinterpret_cast<const MigRec *>(in)[e];
    B.pos[cp][k] = r.pos;
    B.vel[cp][k] = r.vel;
    B.gid[ci][k] = r.gid;
    B.kind[ci][k] = r.kind;
    B.rhoP[ci][k] = make_float2(r.vel.w, r.pos.w);  // an SPH run packs rho, P there
    if (B.vold[ci]) B.vold[ci][k] = r.aux;
    else if (B.omega[cp]) B.omega[cp][k] = r.aux;
  } else {
    const GhostRec r = reinterpret_cast<const GhostRec *>(in)[e];
    B.pos[cp][k] = r.pos;
    B.vel[cp][k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (B.omega[cp]) B.omega[cp][k] = make_float4(0.f, 0.f, 0.f, 0.f);
    B.gid[ci][k] = r.gid;
    B.kind[ci][k] = r.kind | kGhostBit;
  }
}

// after the cell sort: pre-sort indices -> sorted positions
__global__ void k_dist_remap(const int *__restrict__ invperm, int *__restrict__ send_idx,
                             int nsend, int *__restrict__ ghost_slot, int nghost, int n_owned) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nsend) {
    PM_CHECK(send_idx[e] >= 0 && send_idx[e] < n_owned);
    send_idx[e] = invperm[send_idx[e]];
  }
  if (e < nghost) ghost_slot[e] = invperm[n_owned + e];
}

__global__ void k_refresh_pack(Bufs B, const int *__restrict__ send_idx, int nsend,
                               float4 *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (B.st->hold) return;  // a held step of a group batch
  if (e < nsend) out[e] = B.pos[B.st->cur_pv][send_idx[e]];
}

__global__ void k_refresh_unpack(Bufs B, const int *__restrict__ ghost_slot, int nghost,
                                 const float4 *__restrict__ in) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (B.st->hold) return;  // a held step of a group batch
  if (e < nghost) {
    PM_CHECK(ghost_slot[e] >= 0);
    B.pos[B.st->cur_pv][ghost_slot[e]] = in[e];
  }
}

// SPH runs (NEXT-3): positions and velocities, with P and rho in their w
// lanes -- everything the stepping sweep reads of a partner (32 B per ghost);
// DEM runs (W = 3): also the angular velocity (48 B)
template <int W>
__global__ void k_refresh_pack_pv(Bufs B, const int *__restrict__ send_idx, int nsend,
                                  float4 *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nsend) {
    const int cp = B.st->cur_pv, i = send_idx[e];
    out[W * e] = B.pos[cp][i];
    out[W * e + 1] = B.vel[cp][i];
    if (W == 3) out[W * e + 2] = B.omega[cp][i];
  }
}

template <int W>
__global__ void k_refresh_unpack_pv(Bufs B, const int *__restrict__ ghost_slot, int nghost,
                                    const float4 *__restrict__ in) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nghost) {
    const int cp = B.st->cur_pv, k = ghost_slot[e];
    B.pos[cp][k] = in[W * e];
    B.vel[cp][k] = in[W * e + 1];
    if (W == 3) B.omega[cp][k] = in[W * e + 2];
  }
}

// fused refresh tables: per send entry e (send order), its particle
// send_idx[e] and its destination (peer, ghost slot) -> CSR by particle
__global__ void k_peer_count(const int *__restrict__ send_idx, int nsend, int32_t *cnt) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nsend) atomicAdd(&cnt[send_idx[e]], 1);
}

__global__ void k_peer_fill(const int *__restrict__ send_idx, const int *__restrict__ dst_peer,
                            const int *__restrict__ dst_slot, int nsend,
                            const int32_t *__restrict__ off, int32_t *fill, int2 *__restrict__ dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nsend) return;
  const int i = send_idx[e];
  dst[off[i] + atomicAdd(&fill[i], 1)] = make_int2(dst_peer[e], dst_slot[e]);
}

// ghost_put (half lists across sub-domains, SURVEY NEXT-1 / PAPER.md:116):
// the force shares a sub-domain accumulated on its ghost copies go back to
// the owners (arrival order -> the owners' send order) and are added there
__global__ void k_ghost_put_pack(Bufs B, const int *__restrict__ ghost_slot, int nghost,
                                 float4 *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nghost) out[e] = B.force[ghost_slot[e]];
}

__global__ void k_ghost_put_add(Bufs B, const int *__restrict__ send_idx, int nsend,
                                const float4 *__restrict__ in) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nsend) return;
  const float4 f = in[e];
  float4 *p = B.force + send_idx[e];
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(f.x), "f"(f.y),
               "f"(f.z), "f"(0.f)
               : "memory");
}

inline unsigned nb(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int dist_record_bytes(int what) {
  switch (what) {
    case 0: return (int)sizeof(MigRec);
    case 1: return (int)sizeof(GhostRec);
    case 2: return 16;
    case 3: return 32;
    case 4: return 48;
    case 5: return dem_hist_record_bytes();
    default: return -1;
  }
}

void launch_dist_plan(const Params &P, const Bufs &B, const Dist &D, int n_owned, int what,
                      uint32_t *mask, int *blk_counts, const int *order, int *dir_base,
                      long long *totals, int *list, cudaStream_t s) {
  const unsigned g = nb(n_owned > 0 ? n_owned : 1, kDirBlock * kDirItems);
  k_dist_mark<<<g, kDirBlock, 0, s>>>(P, B, D, n_owned, what, mask, blk_counts);
  k_dist_scan<<<27, 1024, 0, s>>>(blk_counts, (int)g, totals);
  k_dist_fill<<<g, kDirBlock, 0, s>>>(mask, n_owned, blk_counts, totals, order, dir_base, list);
}

void launch_dist_pack(const Bufs &B, int what, const int *list, int nsend, void *out,
                      cudaStream_t s) {
  if (nsend > 0) k_dist_pack<<<nb(nsend), 256, 0, s>>>(B, what, list, nsend, out);
}

void launch_dist_compact(const Bufs &B, const int *stay, int n_stay, cudaStream_t s) {
  if (n_stay > 0) k_dist_compact<<<nb(n_stay), 256, 0, s>>>(B, stay, n_stay);
}

void launch_dist_unpack(const Bufs &B, int what, const void *in, int nrecv, int base,
                        cudaStream_t s) {
  if (nrecv > 0) k_dist_unpack<<<nb(nrecv), 256, 0, s>>>(B, what, in, nrecv, base);
}

// Slice classes of a decomposed context after a build (§3.6
// "interior and ghost iterators ... overlapping communication with
// computation"): a 32-row slice is interior (0) when none of its particles
// is a ghost or lies within the ghost width r_g of a decomposed face of the
// sub-domain -- its rows (built with r_v <= r_g) then hold owned partners
// only, so its forces can run while the ghost refresh is in flight;
// otherwise boundary (1).
__global__ void k_warp_class(Dist D, Bufs B, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if ((i >> 5) >= ((n + 31) >> 5)) return;  // whole warp
  State *st = B.st;
  bool near = false;
  if (i < n) {
    if (B.kind[st->cur_id][i] & kGhostBit) {
      near = true;
    } else {
      const float4 x = B.pos[st->cur_pv][i];
      const float c[3] = {x.x, x.y, x.z};
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (D.p[d] > 1)
          near |= (c[d] - D.slo[d] < D.rg) || (D.shi[d] - c[d] <= D.rg);
    }
  }
  const bool b = __any_sync(0xffffffffu, near);
  if ((threadIdx.x & 31) == 0) B.wclass[i >> 5] = b ? 1 : 0;
}

void launch_warp_class(const Dist &D, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n > 0) k_warp_class<<<nb(n), 256, 0, s>>>(D, B, (int)n);
}

void launch_dist_remap(const int *invperm, int *send_idx, int nsend, int *ghost_slot, int nghost,
                       int n_owned, cudaStream_t s) {
  const int m = nsend > nghost ? nsend : nghost;
  if (m > 0)
    k_dist_remap<<<nb(m), 256, 0, s>>>(invperm, send_idx, nsend, ghost_slot, nghost, n_owned);
}

void launch_refresh_pack(const Bufs &B, const int *send_idx, int nsend, void *out,
                         cudaStream_t s) {
  if (nsend > 0)
    k_refresh_pack<<<nb(nsend), 256, 0, s>>>(B, send_idx, nsend, reinterpret_cast<float4 *>(out));
}

void launch_refresh_pv(const Bufs &B, int pack, const int *idx, int m, void *buf, int with_w,
                       cudaStream_t s) {
  if (m <= 0) return;
  float4 *f = reinterpret_cast<float4 *>(buf);
  if (pack && with_w) k_refresh_pack_pv<3><<<nb(m), 256, 0, s>>>(B, idx, m, f);
  else if (pack) k_refresh_pack_pv<2><<<nb(m), 256, 0, s>>>(B, idx, m, f);
  else if (with_w) k_refresh_unpack_pv<3><<<nb(m), 256, 0, s>>>(B, idx, m, f);
  else k_refresh_unpack_pv<2><<<nb(m), 256, 0, s>>>(B, idx, m, f);
}

// cnt: n + 1 zeroed ints; tmp: scan_tiles(n + 1) ints; B.ps_off: n + 1 ints;
// B.ps_dst: nsend int2
void launch_peer_csr(const Bufs &B, const int *send_idx, const int *dst_peer, const int *dst_slot,
                     int nsend, int32_t *cnt, int n, int32_t *tmp, cudaStream_t s) {
  if (nsend > 0) k_peer_count<<<nb(nsend), 256, 0, s>>>(send_idx, nsend, cnt);
  launch_exclusive_scan(cnt, B.ps_off, tmp, n + 1, s);  // zeroes cnt again
  if (nsend > 0)
    k_peer_fill<<<nb(nsend), 256, 0, s>>>(send_idx, dst_peer, dst_slot, nsend, B.ps_off, cnt,
                                          B.ps_dst);
}

void launch_ghost_put(const Bufs &B, int pack, const int *idx, int m, void *buf, cudaStream_t s) {
  if (m <= 0) return;
  if (pack) k_ghost_put_pack<<<nb(m), 256, 0, s>>>(B, idx, m, reinterpret_cast<float4 *>(buf));
  else k_ghost_put_add<<<nb(m), 256, 0, s>>>(B, idx, m, reinterpret_cast<const float4 *>(buf));
}

void launch_refresh_unpack(const Bufs &B, const int *ghost_slot, int nghost, const void *in,
                           cudaStream_t s) {
  if (nghost > 0)
    k_refresh_unpack<<<nb(nghost), 256, 0, s>>>(B, ghost_slot, nghost,
                                                reinterpret_cast<const float4 *>(in));
}

}  // namespace pm
