// k_dem.cu -- discrete element method.
//
// PAPER.md:520-540 (§4.5): Hertzian contacts with elastic deformation of the
// grains.  Eq. 9 overlap delta = 2R - r_pq; Eq. 10 tangential deformation
// u_t += v_t dt over the duration of a contact; Eqs. 11-12 normal and
// tangential forces sqrt(delta/2R)(k delta n - gamma m_eff v); Coulomb cap
// ("rescaled to enforce Coulomb's law"); Eq. 13 leapfrog for v, r and the
// angular velocity.  Readings R29-R33 fix what the paper leaves
// open: relative velocity at the contact point with the rotation term,
// u_t kept tangential, gamma_t, mu, torque arm -R n, plane walls.  The same
// definitions are written out in oracle/pm_oracle.c orc_dem_run.
//
// Contacts are found in the Verlet list (r_v = 2R + skin, the int32 rows of
// k_verlet.cu); the tangential history of an ordered pair (p, q) lives in the
// list slot of q in p's row (float4, same SELL layout) and is carried to the
// new list at a rebuild by matching partner gids (k_dem_remap).  Both ordered
// pairs evolve with opposite v_t, so F_qp = -F_pq: linear momentum is kept up
// to rounding.  fp32, thread per particle, no atomics.
#include "pm_internal.cuh"

namespace pm {

namespace {

__device__ __forceinline__ float3 cross3(const float3 &a, const float3 &b) {
  return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// One DEM step for particle i (thread per particle): the contact sum of
// Eqs. 9-12 over the Verlet row, the plane walls, then the Eq. 13 leapfrog
// fused in (as the LJ sweep fuses velocity Verlet): pos/vel/omega are read
// from buffer cur_pv and written to cur_pv ^ 1, so the sweep reads only the
// old state.  Contacts are processed two at a time with all their loads
// (partner x, v, omega and the slot's history) issued before the arithmetic.
// PM: periodic axes as a compile-time bit mask (the contact loop's pair
// difference takes the R4 branches only on those axes)
template <int PM>
__global__ void __launch_bounds__(256, 4) k_dem_step(Params P, Bufs B, int n, float dt) {
  State *st = B.st;
  if (st->abort) return;  // a failed in-graph rebuild: the host resumes here
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int cp = st->cur_pv, ci = st->cur_id;
  bool far = false;
  if (i < n && P.dist && (B.kind[ci][i] & kGhostBit)) {
    // ghost copy of a decomposed context: carried through the buffer flip,
    // refreshed (x, v, omega) by its owner before the next step
    B.pos[cp ^ 1][i] = B.pos[cp][i];
    B.vel[cp ^ 1][i] = B.vel[cp][i];
    B.omega[cp ^ 1][i] = B.omega[cp][i];
  } else if (i < n) {
    const float4 *__restrict__ pos = B.pos[cp];
    const float4 *__restrict__ vel = B.vel[cp];
    const float4 *__restrict__ om = B.omega[cp];
    const DEM &D = P.dem;
    const float4 xi = pos[i], vi = vel[i], wi = om[i];
    float3 f = make_float3(D.m * D.g[0], D.m * D.g[1], D.m * D.g[2]);
    float3 tq = make_float3(0.f, 0.f, 0.f);
    const int cnt = B.cnt[i];
    const int64_t base = nbr_row_base(B, i);
    const float twoR = 2.0f * D.R, inv2R = 1.0f / (2.0f * D.R);
    auto contact = [&](const float4 &xj, const float4 &vj, const float4 &wj, const float4 &h,
                       int64_t slot) {
      // r_pq = x_i - x_j (R4 minimum image on periodic axes)
      const float rx = -pair_delta1(xi.x, xj.x, P.box.L[0], P.box.halfL[0], PM & 1);
      const float ry = -pair_delta1(xi.y, xj.y, P.box.L[1], P.box.halfL[1], (PM >> 1) & 1);
      const float rz = -pair_delta1(xi.z, xj.z, P.box.L[2], P.box.halfL[2], (PM >> 2) & 1);
      const float r2 = rx * rx + ry * ry + rz * rz;
      const float rr = sqrtf(r2);
      const float delta = twoR - rr;
      if (!(delta > 0.0f) || rr == 0.0f) {  // no contact: the history ends
        if (h.x != 0.f || h.y != 0.f || h.z != 0.f) B.hist[slot] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
      }
      const float inv_r = 1.0f / rr;
      const float3 nv = make_float3(rx * inv_r, ry * inv_r, rz * inv_r);
      const float3 wxn = cross3(make_float3(wi.x + wj.x, wi.y + wj.y, wi.z + wj.z), nv);
      const float3 vpq = make_float3(vi.x - vj.x - D.R * wxn.x, vi.y - vj.y - D.R * wxn.y,
                                     vi.z - vj.z - D.R * wxn.z);
      const float vn = vpq.x * nv.x + vpq.y * nv.y + vpq.z * nv.z;
      const float3 vnv = make_float3(vn * nv.x, vn * nv.y, vn * nv.z);
      const float3 vt = make_float3(vpq.x - vnv.x, vpq.y - vnv.y, vpq.z - vnv.z);
      const float un = h.x * nv.x + h.y * nv.y + h.z * nv.z;
      float3 u = make_float3(h.x - un * nv.x + vt.x * dt, h.y - un * nv.y + vt.y * dt,
                             h.z - un * nv.z + vt.z * dt);
      const float sq = sqrtf(delta * inv2R);
      const float3 fn = make_float3(sq * (D.kn * delta * nv.x - D.gn * D.meff * vnv.x),
                                    sq * (D.kn * delta * nv.y - D.gn * D.meff * vnv.y),
                                    sq * (D.kn * delta * nv.z - D.gn * D.meff * vnv.z));
      float3 ft = make_float3(sq * (-D.kt * u.x - D.gt * D.meff * vt.x),
                              sq * (-D.kt * u.y - D.gt * D.meff * vt.y),
                              sq * (-D.kt * u.z - D.gt * D.meff * vt.z));
      const float fnm = sqrtf(fn.x * fn.x + fn.y * fn.y + fn.z * fn.z);
      const float ftm = sqrtf(ft.x * ft.x + ft.y * ft.y + ft.z * ft.z);
      if (ftm > D.mu * fnm && ftm > 0.0f) {  // Coulomb: slide, rescale the spring
        const float sc = D.mu * fnm / ftm;
        ft = make_float3(ft.x * sc, ft.y * sc, ft.z * sc);
        u = make_float3(-(ft.x / sq + D.gt * D.meff * vt.x) / D.kt,
                        -(ft.y / sq + D.gt * D.meff * vt.y) / D.kt,
                        -(ft.z / sq + D.gt * D.meff * vt.z) / D.kt);
      }
      B.hist[slot] = make_float4(u.x, u.y, u.z, 0.f);
      const float3 tc = cross3(make_float3(-D.R * nv.x, -D.R * nv.y, -D.R * nv.z), ft);
      f = make_float3(f.x + fn.x + ft.x, f.y + fn.y + ft.y, f.z + fn.z + ft.z);
      tq = make_float3(tq.x + tc.x, tq.y + tc.y, tq.z + tc.z);
    };
    // the next pair's indices are loaded one iteration ahead
    int64_t s0 = base;
    int ja = cnt > 0 ? B.nbr[s0] : 0;
    int jb = cnt > 1 ? B.nbr[s0 + 32] : ja;
    for (int k = 0; k < cnt; k += 2) {
      const bool two = k + 1 < cnt;
      const int64_t sn = s0 + 64;
      const int na = (k + 2 < cnt) ? B.nbr[sn] : ja;
      const int nb_ = (k + 3 < cnt) ? B.nbr[sn + 32] : na;
      const float4 x0 = __ldg(pos + ja), x1 = __ldg(pos + jb);
      const float4 v0 = __ldg(vel + ja), v1 = __ldg(vel + jb);
      const float4 w0 = __ldg(om + ja), w1 = __ldg(om + jb);
      const float4 h0 = B.hist[s0];
      const float4 h1 = two ? B.hist[s0 + 32] : h0;
      contact(x0, v0, w0, h0, s0);
      if (two) contact(x1, v1, w1, h1, s0 + 32);
      ja = na;
      jb = nb_;
      s0 = sn;
    }
    // plane walls at the box faces: normal Hertz force with damping (R33)
    const float xv[3] = {xi.x, xi.y, xi.z}, vv[3] = {vi.x, vi.y, vi.z};
    float fw[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (!D.walls[2 * d + side]) continue;
        const float dist = side == 0 ? xv[d] - P.box.lo[d] : P.box.hi[d] - xv[d];
        const float delta = D.R - dist;
        if (!(delta > 0.0f)) continue;
        const float nd = side == 0 ? 1.0f : -1.0f;
        const float sq = sqrtf(delta * inv2R);
        fw[d] += sq * (D.kn * delta - D.gn * D.meff * vv[d] * nd) * nd;
      }
    }
    f = make_float3(f.x + fw[0], f.y + fw[1], f.z + fw[2]);
    B.force[i] = make_float4(f.x, f.y, f.z, 0.f);
    B.torque[i] = make_float4(tq.x, tq.y, tq.z, 0.f);
    if (!isfinite(f.x + f.y + f.z + tq.x + tq.y + tq.z))
      raise_error(st, -8 /*PM_E_NONFINITE*/, (long long)B.gid[ci][i]);
    // Eq. 13 leapfrog: v += dt F/m; x += dt v; w += dt T/I; rebuild test
    float4 v = vi;
    v.x = fmaf(dt * D.inv_m, f.x, v.x);
    v.y = fmaf(dt * D.inv_m, f.y, v.y);
    v.z = fmaf(dt * D.inv_m, f.z, v.z);
    float r3[3] = {fmaf(dt, v.x, xi.x), fmaf(dt, v.y, xi.y), fmaf(dt, v.z, xi.z)};
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (P.box.per[d]) r3[d] = wrap1(r3[d], P.box.lo[d], P.box.hi[d], P.box.L[d]);
    const float4 xn = make_float4(r3[0], r3[1], r3[2], xi.w);
    float4 w = wi;
    w.x = fmaf(dt * D.inv_I, tq.x, w.x);
    w.y = fmaf(dt * D.inv_I, tq.y, w.y);
    w.z = fmaf(dt * D.inv_I, tq.z, w.z);
    B.omega[cp ^ 1][i] = w;
    B.pos[cp ^ 1][i] = xn;
    B.vel[cp ^ 1][i] = v;
    const float4 xr = B.xref[i];
    const float dx = pair_delta1(xr.x, xn.x, P.box.L[0], P.box.halfL[0], P.box.per[0]);
    const float dy = pair_delta1(xr.y, xn.y, P.box.L[1], P.box.halfL[1], P.box.per[1]);
    const float dz = pair_delta1(xr.z, xn.z, P.box.L[2], P.box.halfL[2], P.box.per[2]);
    far = dist2(dx, dy, dz) > P.half_skin2;
    for (int d = 0; d < 3; ++d)
      if (!P.box.per[d] && (r3[d] < P.box.lo[d] || r3[d] >= P.box.hi[d])) far = true;
  }
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) st->need_rebuild = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->pending_flip = 1;
    st->steps_done += 1;
  }
}

// Before a rebuild: keep the list rows, their histories, counts and slice
// offsets for k_dem_remap (row entries only, coalesced along the slices).
__global__ void __launch_bounds__(256) k_dem_save(Bufs B, int n) {
  State *st = B.st;
  if (st->abort) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= (n + 31) / 32) B.slice_off_old[i] = B.slice_off[i];
  if (i >= n) return;
  if (B.gid_old) B.gid_old[i] = B.gid[st->cur_id][i];  // decomposed: partners by gid
  const int cnt = B.cnt[i];
  B.cnt_old[i] = cnt;
  const int64_t base = nbr_row_base(B, i);
  for (int k = 0; k < cnt; ++k) {
    const int64_t slot = base + ((int64_t)k << 5);
    B.nbr_old[slot] = B.nbr[slot];
    B.hist_old[slot] = B.hist[slot];
  }
}

// Step head of the DEM graph: apply the pending buffer flip and open the
// rebuild branch when a particle moved more than skin/2 (no abort pending).
__global__ void k_dem_step_begin(Bufs B, cudaGraphConditionalHandle h) {
  State *st = B.st;
  if (st->pending_flip) {
    st->cur_pv ^= 1;
    st->pending_flip = 0;
  }
  const unsigned c = (st->abort == 0 && st->need_rebuild) ? 1u : 0u;
  st->do_rebuild = (int)c;
  cudaGraphSetConditional(h, c);
}

// After a rebuild: the history of each new list slot (i, j) is the old
// slot with the same partner gid in the old row of the same particle
// (old index perm[i]); 0 for new contacts.
__global__ void __launch_bounds__(256) k_dem_remap(Bufs B, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || B.st->abort) return;
  const int ci = B.st->cur_id, ci_old = ci ^ 1;  // the rebuild flipped once
  const int o = B.perm[i];
  const int64_t *gnew = B.gid[ci], *gold = B.gid[ci_old];
  const int64_t obase = B.slice_off_old[o >> 5] * 32 + (o & 31);
  const int ocnt = B.cnt_old[o];
  const int64_t base = nbr_row_base(B, i);
  const int cnt = B.cnt[i];
  for (int k = 0; k < cnt; ++k) {
    const int64_t slot = base + ((int64_t)k << 5);
    const int64_t gj = gnew[B.nbr[slot]];
    float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < ocnt; ++q) {
      const int64_t os = obase + ((int64_t)q << 5);
      if (gold[B.nbr_old[os]] == gj) {
        h = B.hist_old[os];
        break;
      }
    }
    B.hist[slot] = h;
  }
}

// Decomposed DEM ("collisions involving ghost particles need to
// be properly accounted for in the lists of the respective source
// particles"): a grain that migrates takes its contact histories along, as
// (partner gid, u_t) pairs next to its migration record (PM_MSG_MIGRATE_HIST,
// same list and order as PM_MSG_MIGRATE).  Contacts with ghosts are kept by
// each owner for its own ordered pair, so nothing else travels.
struct DemHistEntry {
  long long gid;
  float ux, uy, uz, pad;
};
struct DemHistRec {
  long long gid;
  int n, pad;
  DemHistEntry e[kDemHist];
};

__global__ void __launch_bounds__(256) k_dem_hist_pack(Bufs B, const int *__restrict__ list,
                                                        int nsend, DemHistRec *__restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nsend) return;
  State *st = B.st;
  const int ci = st->cur_id;
  const int i = list[e];
  const int64_t *g = B.gid[ci];
  DemHistRec &r = out[e];
  r.gid = g[i];
  r.pad = 0;
  int m = 0;
  const int64_t base = nbr_row_base(B, i);
  for (int k = 0; k < B.cnt[i]; ++k) {
    const int64_t slot = base + ((int64_t)k << 5);
    const float4 h = B.hist[slot];
    if (h.x == 0.f && h.y == 0.f && h.z == 0.f) continue;
    if (m == kDemHist) {
      raise_error(st, -9 /*PM_E_CAPACITY*/, (long long)g[i]);
      break;
    }
    r.e[m].gid = g[B.nbr[slot]];
    r.e[m].ux = h.x;
    r.e[m].uy = h.y;
    r.e[m].uz = h.z;
    r.e[m].pad = 0.f;
    ++m;
  }
  r.n = m;
}

// After a decomposed rebuild: new particle i came from pre-sort index
// q = perm[i] = a stayer (pre-migration index stay_old[q], rows saved by
// k_dem_save) or arrival q - n_stay (its DemHistRec); ghosts have no row.
__global__ void __launch_bounds__(256) k_dem_remap_dist(Bufs B, int n,
                                                         const int *__restrict__ stay_old,
                                                         int n_stay,
                                                         const DemHistRec *__restrict__ hin,
                                                         int n_arr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  State *st = B.st;
  if (i >= n || st->abort) return;
  const int ci = st->cur_id;
  if (B.kind[ci][i] & kGhostBit) return;
  const int q = B.perm[i];
  const int64_t *gnew = B.gid[ci];
  const int64_t base = nbr_row_base(B, i);
  const int cnt = B.cnt[i];
  if (q < n_stay) {
    const int o = stay_old[q];
    const int64_t obase = B.slice_off_old[o >> 5] * 32 + (o & 31);
    const int ocnt = B.cnt_old[o];
    for (int k = 0; k < cnt; ++k) {
      const int64_t slot = base + ((int64_t)k << 5);
      const int64_t gj = gnew[B.nbr[slot]];
      float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = 0; t < ocnt; ++t) {
        const int64_t os = obase + ((int64_t)t << 5);
        if (B.gid_old[B.nbr_old[os]] == gj) {
          h = B.hist_old[os];
          break;
        }
      }
      B.hist[slot] = h;
    }
  } else {
    const int a = q - n_stay;
    const DemHistRec *r = (a < n_arr) ? hin + a : nullptr;
    const int m = r ? r->n : 0;
    for (int k = 0; k < cnt; ++k) {
      const int64_t slot = base + ((int64_t)k << 5);
      const int64_t gj = gnew[B.nbr[slot]];
      float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = 0; t < m; ++t)
        if (r->e[t].gid == gj) {
          h = make_float4(r->e[t].ux, r->e[t].uy, r->e[t].uz, 0.f);
          break;
        }
      B.hist[slot] = h;
    }
  }
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void launch_dem_step(const Params &P, const Bufs &B, int64_t n, float dt, cudaStream_t s) {
  if (n <= 0) return;
  const int pm = (P.box.per[0] ? 1 : 0) | (P.box.per[1] ? 2 : 0) | (P.box.per[2] ? 4 : 0);
  switch (pm) {
    case 0: k_dem_step<0><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    case 1: k_dem_step<1><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    case 2: k_dem_step<2><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    case 3: k_dem_step<3><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    case 4: k_dem_step<4><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    case 5: k_dem_step<5><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    case 6: k_dem_step<6><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
    default: k_dem_step<7><<<nb(n), 256, 0, s>>>(P, B, (int)n, dt); break;
  }
}

void launch_dem_remap(const Bufs &B, int64_t n, cudaStream_t s) {
  if (n > 0) k_dem_remap<<<nb(n), 256, 0, s>>>(B, (int)n);
}

void launch_dem_save(const Bufs &B, int64_t n, cudaStream_t s) {
  if (n > 0) k_dem_save<<<nb(n + 64), 256, 0, s>>>(B, (int)n);
}

int dem_hist_record_bytes() { return (int)sizeof(DemHistRec); }

void launch_dem_hist_pack(const Bufs &B, const int *list, int nsend, void *out, cudaStream_t s) {
  if (nsend > 0)
    k_dem_hist_pack<<<nb(nsend), 256, 0, s>>>(B, list, nsend, reinterpret_cast<DemHistRec *>(out));
}

void launch_dem_remap_dist(const Bufs &B, int64_t n, const int *stay_old, int n_stay,
                           const void *hist_in, int n_arr, cudaStream_t s) {
  if (n > 0)
    k_dem_remap_dist<<<nb(n), 256, 0, s>>>(B, (int)n, stay_old, n_stay,
                                           reinterpret_cast<const DemHistRec *>(hist_in), n_arr);
}

void launch_dem_step_begin(const Bufs &B, cudaGraphConditionalHandle h, cudaStream_t s) {
  k_dem_step_begin<<<1, 1, 0, s>>>(B, h);
}

}  // namespace pm
