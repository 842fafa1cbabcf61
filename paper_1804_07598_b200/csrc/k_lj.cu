// k_lj.cu -- Lennard-Jones sweep and velocity-Verlet integrator
// (SURVEY §8(a) rows a6, a7).
//
// PAPER.md:162 (§4.1) V_LJ(r) = 4 eps [(sigma/r)^12 - (sigma/r)^6]; the
// force is -dV/dr along (x_i - x_j) (reading R7, PAPER.md:212 typo):
//   F_i = sum_j 24 eps (2 sigma^12 / r^14 - sigma^6 / r^8) (x_i - x_j)
// over the full Verlet list, pairs with d2_32 < r_cut^2 (R6).
// Velocity Verlet: v += dt/2 F/m; x += dt v; ...
//
// B200 design: one thread per particle (cell order, so
// a warp's 32 rows share neighbour cells and the position gathers hit L1),
// per-thread fp32 accumulation, no atomics.  The neighbour stream is read
// with streaming loads (ld.global.cs) so the 0.3 GB list does not evict the
// L2-resident positions.  The periodic minimum-image correction (R4) is only
// evaluated on the axes along which the warp has a particle within r_v +
// skin of a periodic face (warp-uniform 3-bit mask, one loop variant per
// case).  In pm_step_vv the sweep is fused with the
// integrator: the second half-kick of step n, the first half-kick and drift
// of step n+1, the wrap and the skin/2 displacement test run in the epilogue
// and write the alternate position/velocity buffers.
#include "pm_internal.cuh"

namespace pm {

namespace {

struct Acc {
  float fx, fy, fz, u, w;
  int np;
};

// R4 along one axis, branch-free (same arithmetic as pair_delta1): all three
// candidates are computed and selected, so boundary warps do not diverge.
__device__ __forceinline__ float r4_delta(float a, float b, float L, float halfL) {
  const float e = __fsub_rn(b, a);
  const float up = __fsub_rn(__fsub_rn(b, L), a);  // e > L/2: shift x_j by -L
  const float dn = __fsub_rn(b, __fsub_rn(a, L));  // e < -L/2: shift x_i by -L
  return e > halfL ? up : (e < -halfL ? dn : e);
}

// One pair, branch-free: the contribution is selected to zero when the pair
// is outside r_cut (R6) or the slot is padding (valid == false).
// MIM: bit d set = R4 on axis d (the warp has a row near a periodic face
// of axis d); the other axes take the plain difference, which R4 reduces to
// there (|e| <= L/2 for every listed pair of such rows).
template <int MIM, bool CAPPED, bool ENERGY, bool MASK>
__device__ __forceinline__ void lj_pair(const Params &P, const float4 &xi, const float4 &xj,
                                        bool valid, Acc &a) {
  const float dx = (MIM & 1) ? r4_delta(xi.x, xj.x, P.box.L[0], P.box.halfL[0])
                             : __fsub_rn(xj.x, xi.x);
  const float dy = (MIM & 2) ? r4_delta(xi.y, xj.y, P.box.L[1], P.box.halfL[1])
                             : __fsub_rn(xj.y, xi.y);
  const float dz = (MIM & 4) ? r4_delta(xi.z, xj.z, P.box.L[2], P.box.halfL[2])
                             : __fsub_rn(xj.z, xi.z);
  const float d2 = dist2(dx, dy, dz);
  const bool in = (MASK ? valid : true) && (d2 < P.lj.rc2);
  float f, r6i;
  if (CAPPED) {
    const float r2e = fmaxf(d2, P.lj.r_min * P.lj.r_min);
    const float r2ie = fast_rcp(r2e);
    r6i = r2ie * r2ie * r2ie;
    const float g = r6i * (P.lj.c12 * r6i - P.lj.c6);
    f = g * fast_rsqrt(r2e) * fast_rsqrt(d2);
  } else {
    const float r2i = fast_rcp(d2);
    r6i = r2i * r2i * r2i;
    f = r2i * (r6i * (P.lj.c12 * r6i - P.lj.c6));
  }
  f = in ? f : 0.0f;
  // F_i += f (x_i - x_j) = -f * delta
  a.fx = fmaf(-f, dx, a.fx);
  a.fy = fmaf(-f, dy, a.fy);
  a.fz = fmaf(-f, dz, a.fz);
  if (ENERGY) {
    a.u += in ? 0.5f * r6i * (P.lj.e12 * r6i - P.lj.e6) : 0.0f;
    a.w += in ? 0.5f * f * d2 : 0.0f;
    a.np += in ? 1 : 0;
  }
}

// Row sweep, software-pipelined: the index stream (the only HBM-resident
// operand) is prefetched two groups of 4 ahead with streaming loads (each a
// coalesced 128-byte line across the warp); the 4 position gathers of a group
// are issued together.  Full groups run unmasked; the last partial group is
// padded by the builder with the row's own index (always a valid gather) and
// masked.
struct Idx4 {
  int a, b, c, d;
};

__device__ __forceinline__ Idx4 ld_idx4(const int *__restrict__ p) {
  Idx4 r;
  r.a = __ldcs(p);
  r.b = __ldcs(p + 32);
  r.c = __ldcs(p + 64);
  r.d = __ldcs(p + 96);
  return r;
}

// a group of 4 entries: SELL-32 (4 coalesced lines across the warp) or a
// row-major row (one 16-byte load of the lane's own row)
template <bool RM>
__device__ __forceinline__ Idx4 ld_group(const int *__restrict__ p) {
  if (!RM) return ld_idx4(p);
  // (L1-cached: the lane's next group is the other half of the same sector)
  const int4 v = __ldg(reinterpret_cast<const int4 *>(p));
  return Idx4{v.x, v.y, v.z, v.w};
}

template <int MIM, bool CAPPED, bool ENERGY, bool MASK>
__device__ __forceinline__ void lj_group(const Params &P, const float4 *__restrict__ pos,
                                         const Idx4 &j, int rem, const float4 &xi, Acc &a) {
  const float4 x0 = __ldg(pos + j.a);
  const float4 x1 = __ldg(pos + j.b);
  const float4 x2 = __ldg(pos + j.c);
  const float4 x3 = __ldg(pos + j.d);
  lj_pair<MIM, CAPPED, ENERGY, false>(P, xi, x0, true, a);
  lj_pair<MIM, CAPPED, ENERGY, MASK>(P, xi, x1, rem > 1, a);
  lj_pair<MIM, CAPPED, ENERGY, MASK>(P, xi, x2, rem > 2, a);
  lj_pair<MIM, CAPPED, ENERGY, MASK>(P, xi, x3, rem > 3, a);
}

template <int MIM, bool CAPPED, bool ENERGY, bool RM = false>
__device__ __forceinline__ void lj_row(const Params &P, const float4 *__restrict__ pos,
                                       const int *__restrict__ nb, int cnt, const float4 &xi,
                                       Acc &a) {
  const int ng = (cnt + 3) >> 2;  // groups incl. a partial last one
  const int nfull = cnt >> 2;
  if (ng == 0) return;
  constexpr int GS = RM ? 4 : 128;  // ints between consecutive groups of a row
  Idx4 j0 = ld_group<RM>(nb);
  Idx4 j1 = (ng > 1) ? ld_group<RM>(nb + GS) : j0;
  int g = 0;
  // two groups per iteration: the prefetch registers rotate statically
  for (; g + 2 <= nfull; g += 2) {
    const Idx4 j2 = (g + 2 < ng) ? ld_group<RM>(nb + (g + 2) * GS) : j1;
    const Idx4 j3 = (g + 3 < ng) ? ld_group<RM>(nb + (g + 3) * GS) : j1;
    lj_group<MIM, CAPPED, ENERGY, false>(P, pos, j0, 4, xi, a);
    lj_group<MIM, CAPPED, ENERGY, false>(P, pos, j1, 4, xi, a);
    j0 = j2;
    j1 = j3;
  }
  if (g < nfull) {
    lj_group<MIM, CAPPED, ENERGY, false>(P, pos, j0, 4, xi, a);
    j0 = j1;
    ++g;
  }
  if (g < ng) lj_group<MIM, CAPPED, ENERGY, true>(P, pos, j0, cnt - 4 * g, xi, a);
}

__device__ __forceinline__ bool near_periodic_face(const Params &P, const float4 &x) {
  bool near = false;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float v = (d == 0) ? x.x : (d == 1) ? x.y : x.z;
    near |= P.box.per[d] &&
            (v < P.box.lo[d] + P.mi_margin || v >= P.box.hi[d] - P.mi_margin);
  }
  return near;
}

// The periodic axes along which the warp has a row within r_v + skin of a
// face (bit d for axis d; warp-uniform): only those axes need R4's
// minimum-image selection, the others reduce to the plain difference.
__device__ __forceinline__ int warp_mi_axes(const Params &P, bool active, const float4 &x) {
  int m = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float v = (d == 0) ? x.x : (d == 1) ? x.y : x.z;
    if (active && P.box.per[d] &&
        (v < P.box.lo[d] + P.mi_margin || v >= P.box.hi[d] - P.mi_margin))
      m |= 1 << d;
  }
  return __reduce_or_sync(0xffffffffu, (unsigned)m);
}

template <bool CAPPED, bool ENERGY, bool RM>
__device__ __forceinline__ Acc lj_force_of(const Params &P, const Bufs &B,
                                           const float4 *__restrict__ pos, int i, bool active,
                                           const float4 &xi) {
  Acc a = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
  const int mim = warp_mi_axes(P, active, xi);
  if (active) {
    const int cnt = B.cnt[i];
    const int *nb = B.nbr + nbr_row_base(B, i);
    if (RM) {  // row-major slices (long rows): the general minimum-image variant
      if (mim) lj_row<7, CAPPED, ENERGY, true>(P, pos, nb, cnt, xi, a);
      else lj_row<0, CAPPED, ENERGY, true>(P, pos, nb, cnt, xi, a);
      return a;
    }
    switch (mim) {  // warp-uniform
      case 0: lj_row<0, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a); break;
      case 1: lj_row<1, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a); break;
      case 2: lj_row<2, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a); break;
      case 4: lj_row<4, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a); break;
      default: lj_row<7, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a); break;  // edges, corners
    }
  }
  return a;
}

__device__ __forceinline__ void block_add_energy(State *st, double u, double w, double np) {
  __shared__ double sh[3][32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    w += __shfl_xor_sync(0xffffffffu, w, o);
    np += __shfl_xor_sync(0xffffffffu, np, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    sh[0][wid] = u;
    sh[1][wid] = w;
    sh[2][wid] = np;
  }
  __syncthreads();
  if (wid == 0) {
    u = lane < nw ? sh[0][lane] : 0.0;
    w = lane < nw ? sh[1][lane] : 0.0;
    np = lane < nw ? sh[2][lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, o);
      w += __shfl_xor_sync(0xffffffffu, w, o);
      np += __shfl_xor_sync(0xffffffffu, np, o);
    }
    if (lane == 0) {
      atomicAdd(&st->acc[0], u);
      atomicAdd(&st->acc[1], w);
      atomicAdd(&st->acc[2], np);
    }
  }
}

// A non-finite force (rare path): PM_E_COINCIDENT when the row holds a
// partner at distance 0 (identical wrapped coordinates; such pairs pass the
// list test 0 <= d2 < r_v^2 in any cell, however crowded), else
// PM_E_NONFINITE.
__device__ __noinline__ void raise_bad_force(const int *nb, int stride, int cnt,
                                             const float4 *pos, int i, float xx, float xy,
                                             float xz, long long gid, State *st) {
  for (int k = 0; k < cnt; ++k) {
    const int j = nb[(int64_t)k * stride];
    const float4 xj = pos[j];
    if (j != i && xj.x == xx && xj.y == xy && xj.z == xz) {
      raise_error(st, -7 /*PM_E_COINCIDENT*/, gid);
      return;
    }
  }
  raise_error(st, -8 /*PM_E_NONFINITE*/, gid);
}

__device__ __forceinline__ void bad_force(const Bufs &B, State *st, const float4 *pos, int i,
                                          const float4 &xi) {
  raise_bad_force(B.nbr + nbr_row_base(B, i), nbr_stride(B), B.cnt[i], pos, i, xi.x, xi.y, xi.z,
                  (long long)B.gid[st->cur_id][i], st);
}

// pm_compute_lj: forces (+ energy) of the current positions.
template <bool CAPPED, bool ENERGY, bool RM = false>
__global__ void __launch_bounds__(256) k_lj(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const float4 xi = active ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  Acc a = lj_force_of<CAPPED, ENERGY, RM>(P, B, pos, i, active, xi);
  if (active) {
    B.force[i] = make_float4(a.fx, a.fy, a.fz, 0.f);
    if (!isfinite(a.fx + a.fy + a.fz)) bad_force(B, st, pos, i, xi);
  }
  if (ENERGY) block_add_energy(st, (double)a.u, (double)a.w, (double)a.np);
}

__device__ __forceinline__ float3 wrap3(const Params &P, float x, float y, float z) {
  float r[3] = {x, y, z};
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (P.box.per[d]) r[d] = wrap1(r[d], P.box.lo[d], P.box.hi[d], P.box.L[d]);
  return make_float3(r[0], r[1], r[2]);
}

__device__ __forceinline__ bool moved_too_far(const Params &P, const float3 &x, const float4 &r) {
  const float dx = pair_delta1(r.x, x.x, P.box.L[0], P.box.halfL[0], P.box.per[0]);
  const float dy = pair_delta1(r.y, x.y, P.box.L[1], P.box.halfL[1], P.box.per[1]);
  const float dz = pair_delta1(r.z, x.z, P.box.L[2], P.box.halfL[2], P.box.per[2]);
  return dist2(dx, dy, dz) > P.half_skin2;
}

// v += k F, then (vmax > 0, reading R22) v <- v min(1, vmax / |v|).
__device__ __forceinline__ void kick_limited(float4 &v, float k, const Acc &a, float vmax) {
  v.x = fmaf(k, a.fx, v.x);
  v.y = fmaf(k, a.fy, v.y);
  v.z = fmaf(k, a.fz, v.z);
  if (vmax > 0.f) {
    const float s2 = v.x * v.x + v.y * v.y + v.z * v.z;
    if (s2 > vmax * vmax) {
      const float sc = vmax * rsqrtf(s2);
      v.x *= sc;
      v.y *= sc;
      v.z *= sc;
    }
  }
}

// One fused velocity-Verlet step (pm_step_vv), mode read from the state:
//  inner: F(x); v += dt F/m (2nd half-kick of this step + 1st of the next);
//         x' = wrap(x + dt v); displacement test vs xref; -> alternate buffers
//  final: F(x); v += dt/2 F/m; F stored; x copied  -> alternate buffers
// The velocity-Verlet epilogue of one particle after its force a (see
// k_lj_step); writes the alternate buffers and sets `far`.
template <bool PEER = false>
__device__ __forceinline__ void vv_epilogue(const Params &P, const Bufs &B, State *st, int i,
                                            bool active, const float4 &xi, const Acc &a,
                                            float dt, int mode, int cp, bool &far) {
  // ghost copies (multi-GPU) are not integrated: after an inner step the
  // refresh overwrites them; the final step (positions unchanged) carries
  // them over so the state stays consistent for getters / energy passes
  const bool ghost = active && P.dist && (B.kind[st->cur_id][i] & kGhostBit);
  if (ghost && mode != kModeInner) B.pos[cp ^ 1][i] = xi;
  if (active && !ghost) {
    float4 v = B.vel[cp][i];
    const float im = P.lj.inv_mass;
    if (mode == kModeInner) {
      if (P.vmax > 0.f) {  // reading R22: limit after each of the two half kicks
        kick_limited(v, 0.5f * dt * im, a, P.vmax);
        kick_limited(v, 0.5f * dt * im, a, P.vmax);
      } else {
        const float k = dt * im;
        v.x = fmaf(k, a.fx, v.x);
        v.y = fmaf(k, a.fy, v.y);
        v.z = fmaf(k, a.fz, v.z);
      }
      const float3 xn = wrap3(P, fmaf(dt, v.x, xi.x), fmaf(dt, v.y, xi.y), fmaf(dt, v.z, xi.z));
      far = moved_too_far(P, xn, B.xref[i]);
      const float4 x4 = make_float4(xn.x, xn.y, xn.z, xi.w);
      B.pos[cp ^ 1][i] = x4;
      if (PEER) {  // fused ghost refresh: straight into the peers' ghost slots
        const int e1 = B.ps_off[i + 1];
        for (int e = B.ps_off[i]; e < e1; ++e) {
          const int2 d = B.ps_dst[e];
          P.peer_pos[d.x][cp ^ 1][d.y] = x4;
        }
      }
    } else {
      kick_limited(v, 0.5f * dt * im, a, P.vmax);
      B.pos[cp ^ 1][i] = xi;
      B.force[i] = make_float4(a.fx, a.fy, a.fz, 0.f);
    }
    B.vel[cp ^ 1][i] = v;
    if (!isfinite(a.fx + a.fy + a.fz)) bad_force(B, st, B.pos[cp], i, xi);
  }
}

// One fused velocity-Verlet step (pm_step_vv), mode read from the state:
//  inner: F(x); v += dt F/m (2nd half-kick of this step + 1st of the next);
//         x' = wrap(x + dt v); displacement test vs xref; -> alternate buffers
//  final: F(x); v += dt/2 F/m; F stored; x copied  -> alternate buffers
template <bool CAPPED, bool PEER = false, bool RM = false>
__global__ void __launch_bounds__(256, 6) k_lj_step(Params P, Bufs B, int n, float dt, int mode_arg,
                                                 int wphase) {
  State *st = B.st;
  if (st->abort || st->hold) return;
  const int mode = mode_arg >= 0 ? mode_arg : st->mode;
  const int cp = st->cur_pv;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (wphase >= 0) {  // one half of an overlapped step: interior or boundary slices
    if (wphase == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
      st->pending_flip = 1;
      st->steps_done += 1;
    }
    if ((i >> 5) >= ((n + 31) >> 5) || B.wclass[i >> 5] != wphase) return;  // whole warp
  }
  const bool active = i < n;
  const float4 *__restrict__ pos = B.pos[cp];
  const float4 xi = active ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  Acc a = lj_force_of<CAPPED, false, RM>(P, B, pos, i, active, xi);
  bool far = false;
  vv_epilogue<PEER>(P, B, st, i, active, xi, a, dt, mode, cp, far);
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) st->need_rebuild = 1;
  if (wphase < 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    st->pending_flip = 1;
    st->steps_done += 1;
  }
}

// ---------------------------------------------------------------------------
// Half (Newton) list, SURVEY §8(f) NEXT-1 ("compute every
// interaction pair only once"): row i holds j > i only; the sweep adds
// f (x_i - x_j) to its own accumulator and f (x_j - x_i) to F_j with one
// vectorised fire-and-forget reduction (red.global.add.v4.f32, sm_90+); the
// integrator runs as a separate epilogue kernel once all reductions landed.
// Sums are not bit-reproducible (reduction order); single-GPU contexts only.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_add4(float4 *p, float x, float y, float z) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x), "f"(y),
               "f"(z), "f"(0.f)
               : "memory");
}

template <bool MI, bool CAPPED, bool ENERGY>
__device__ __forceinline__ void lj_pair_half(const Params &P, const float4 &xi, const float4 &xj,
                                             int j, bool valid, Acc &a, float4 *__restrict__ F) {
  float dx, dy, dz;
  if (MI) {
    dx = P.box.per[0] ? r4_delta(xi.x, xj.x, P.box.L[0], P.box.halfL[0]) : __fsub_rn(xj.x, xi.x);
    dy = P.box.per[1] ? r4_delta(xi.y, xj.y, P.box.L[1], P.box.halfL[1]) : __fsub_rn(xj.y, xi.y);
    dz = P.box.per[2] ? r4_delta(xi.z, xj.z, P.box.L[2], P.box.halfL[2]) : __fsub_rn(xj.z, xi.z);
  } else {
    dx = __fsub_rn(xj.x, xi.x);
    dy = __fsub_rn(xj.y, xi.y);
    dz = __fsub_rn(xj.z, xi.z);
  }
  const float d2 = dist2(dx, dy, dz);
  const bool in = valid && (d2 < P.lj.rc2);
  float f, r6i;
  if (CAPPED) {
    const float r2e = fmaxf(d2, P.lj.r_min * P.lj.r_min);
    const float r2ie = fast_rcp(r2e);
    r6i = r2ie * r2ie * r2ie;
    const float g = r6i * (P.lj.c12 * r6i - P.lj.c6);
    f = g * fast_rsqrt(r2e) * fast_rsqrt(d2);
  } else {
    const float r2i = fast_rcp(d2);
    r6i = r2i * r2i * r2i;
    f = r2i * (r6i * (P.lj.c12 * r6i - P.lj.c6));
  }
  if (in) {
    a.fx = fmaf(-f, dx, a.fx);
    a.fy = fmaf(-f, dy, a.fy);
    a.fz = fmaf(-f, dz, a.fz);
    red_add4(F + j, f * dx, f * dy, f * dz);
    if (ENERGY) {
      a.u += r6i * (P.lj.e12 * r6i - P.lj.e6);  // the whole pair: both halves
      a.w += f * d2;
      a.np += 2;
    }
  }
}

template <bool MI, bool CAPPED, bool ENERGY>
__device__ __forceinline__ void lj_row_half(const Params &P, const float4 *__restrict__ pos,
                                            const int *__restrict__ nb, int cnt,
                                            const float4 &xi, Acc &a, float4 *__restrict__ F) {
  const int ng = (cnt + 3) >> 2;
  if (ng == 0) return;
  Idx4 j0 = ld_idx4(nb);
  Idx4 j1 = (ng > 1) ? ld_idx4(nb + 128) : j0;
  for (int g = 0; g < ng; ++g) {
    const Idx4 j2 = (g + 2 < ng) ? ld_idx4(nb + (g + 2) * 128) : j1;
    const int rem = cnt - 4 * g;
    const float4 x0 = __ldg(pos + j0.a), x1 = __ldg(pos + j0.b);
    const float4 x2 = __ldg(pos + j0.c), x3 = __ldg(pos + j0.d);
    lj_pair_half<MI, CAPPED, ENERGY>(P, xi, x0, j0.a, true, a, F);
    lj_pair_half<MI, CAPPED, ENERGY>(P, xi, x1, j0.b, rem > 1, a, F);
    lj_pair_half<MI, CAPPED, ENERGY>(P, xi, x2, j0.c, rem > 2, a, F);
    lj_pair_half<MI, CAPPED, ENERGY>(P, xi, x3, j0.d, rem > 3, a, F);
    j0 = j1;
    j1 = j2;
  }
}

// F must be zero on entry (the launcher clears it).
template <bool CAPPED, bool ENERGY>
__global__ void __launch_bounds__(256) k_lj_half(Params P, Bufs B, int n) {
  State *st = B.st;
  if (st->abort) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const float4 xi = active ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  Acc a = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
  const bool mi = __any_sync(0xffffffffu, active && near_periodic_face(P, xi));
  if (active) {
    const int cnt = B.cnt[i];
    const int *nb = B.nbr + nbr_row_base(B, i);
    if (mi) lj_row_half<true, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a, B.force);
    else lj_row_half<false, CAPPED, ENERGY>(P, pos, nb, cnt, xi, a, B.force);
    red_add4(B.force + i, a.fx, a.fy, a.fz);
  }
  if (ENERGY) block_add_energy(st, (double)a.u, (double)a.w, (double)a.np);
}

// The integrator of the Newton path: the epilogue of k_lj_step on F = force.
__global__ void __launch_bounds__(256) k_lj_half_vv(Params P, Bufs B, int n, float dt,
                                                     int mode_arg) {
  State *st = B.st;
  if (st->abort) return;
  const int mode = mode_arg >= 0 ? mode_arg : st->mode;
  const int cp = st->cur_pv;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  bool far = false;
  if (active) {
    const float4 xi = B.pos[cp][i];
    const float4 f = B.force[i];
    const Acc a = {f.x, f.y, f.z, 0.f, 0.f, 0};
    vv_epilogue(P, B, st, i, true, xi, a, dt, mode, cp, far);
  }
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) st->need_rebuild = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->pending_flip = 1;
    st->steps_done += 1;
  }
}

// First half-kick + drift from stored forces (start of pm_step_vv).
__global__ void __launch_bounds__(256) k_kick_drift(Params P, Bufs B, int n, float dt) {
  State *st = B.st;
  if (st->abort) return;
  const int cp = st->cur_pv;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool far = false;
  if (i < n && !(P.dist && (B.kind[st->cur_id][i] & kGhostBit))) {
    const float4 f = B.force[i];
    float4 v = B.vel[cp][i];
    const float4 x = B.pos[cp][i];
    Acc fa = {f.x, f.y, f.z, 0.f, 0.f, 0};
    kick_limited(v, 0.5f * dt * P.lj.inv_mass, fa, P.vmax);
    const float3 xn = wrap3(P, fmaf(dt, v.x, x.x), fmaf(dt, v.y, x.y), fmaf(dt, v.z, x.z));
    far = moved_too_far(P, xn, B.xref[i]);
    B.pos[cp ^ 1][i] = make_float4(xn.x, xn.y, xn.z, x.w);
    B.vel[cp ^ 1][i] = v;
  }
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) st->need_rebuild = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->pending_flip = 1;
}

// Start of every step: apply a pending buffer flip, advance the step index,
// choose the step-kernel mode and set the graph's rebuild condition.
__global__ void k_step_begin(Bufs B, cudaGraphConditionalHandle h, int use_handle) {
  State *st = B.st;
  if (st->pending_flip) {
    st->cur_pv ^= 1;
    st->pending_flip = 0;
  }
  st->step_index += 1;
  st->mode = (st->step_index >= st->step_target) ? kModeFinal : kModeInner;
  const unsigned c = (st->abort == 0 && st->need_rebuild) ? 1u : 0u;
  st->do_rebuild = (int)c;
  if (use_handle) cudaGraphSetConditional(h, c);
}

__global__ void __launch_bounds__(256) k_ke(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double ke = 0.0;
  if (i < n && !(P.dist && (B.kind[st->cur_id][i] & kGhostBit))) {
    const float4 v = B.vel[st->cur_pv][i];
    ke = 0.5 * (double)(1.0f / P.lj.inv_mass) *
         ((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ke += __shfl_xor_sync(0xffffffffu, ke, o);
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = ke;
  __syncthreads();
  if (wid == 0) {
    ke = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ke += __shfl_xor_sync(0xffffffffu, ke, o);
    if (lane == 0) atomicAdd(&st->acc[3], ke);
  }
}

// An empty sub-domain still takes part in the buffer flips of a step (the
// fused ghost refresh picks the peer buffer from the sender's parity, so every
// rank must flip in lockstep even with no particles).
__global__ void k_empty_step(State *st, int count_step) {
  if (st->abort || st->hold) return;
  st->pending_flip = 1;
  if (count_step) st->steps_done += 1;
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

static void launch_lj_half(const Params &P, const Bufs &B, int64_t n, int want_energy,
                           cudaStream_t s) {
  cudaMemsetAsync(B.force, 0, sizeof(float4) * (size_t)n, s);
  const bool capped = P.lj.r_min > 0.f;
  if (capped) {
    if (want_energy) k_lj_half<true, true><<<nb(n), 256, 0, s>>>(P, B, (int)n);
    else k_lj_half<true, false><<<nb(n), 256, 0, s>>>(P, B, (int)n);
  } else {
    if (want_energy) k_lj_half<false, true><<<nb(n), 256, 0, s>>>(P, B, (int)n);
    else k_lj_half<false, false><<<nb(n), 256, 0, s>>>(P, B, (int)n);
  }
}

template <bool RM>
void launch_lj_rm(const Params &P, const Bufs &B, int64_t n, int want_energy, cudaStream_t s) {
  const bool capped = P.lj.r_min > 0.f;
  if (capped) {
    if (want_energy) k_lj<true, true, RM><<<nb(n), 256, 0, s>>>(P, B, (int)n);
    else k_lj<true, false, RM><<<nb(n), 256, 0, s>>>(P, B, (int)n);
  } else {
    if (want_energy) k_lj<false, true, RM><<<nb(n), 256, 0, s>>>(P, B, (int)n);
    else k_lj<false, false, RM><<<nb(n), 256, 0, s>>>(P, B, (int)n);
  }
}

void launch_lj(const Params &P, const Bufs &B, int64_t n, int want_energy, cudaStream_t s) {
  if (n <= 0) return;
  if (P.newton) {
    launch_lj_half(P, B, n, want_energy, s);
    return;
  }
  if (B.rm) launch_lj_rm<true>(P, B, n, want_energy, s);
  else launch_lj_rm<false>(P, B, n, want_energy, s);
}

// Decomposed half lists: the sweep alone (ghost shares accumulate in the
// ghost slots until pm_dist_ghost_put), then the integrator alone.
void launch_lj_half_forces(const Params &P, const Bufs &B, int64_t n, int want_energy,
                           cudaStream_t s) {
  if (n > 0) launch_lj_half(P, B, n, want_energy, s);
}

void launch_lj_half_integrate(const Params &P, const Bufs &B, int64_t n, float dt, int mode,
                              cudaStream_t s) {
  if (n > 0) k_lj_half_vv<<<nb(n), 256, 0, s>>>(P, B, (int)n, dt, mode);
  else k_empty_step<<<1, 1, 0, s>>>(B.st, 1);
}

void launch_lj_step_mode(const Params &P, const Bufs &B, int64_t n, float dt, int mode,
                         cudaStream_t s, int wphase) {
  if (n <= 0) {
    k_empty_step<<<1, 1, 0, s>>>(B.st, 1);
    return;
  }
  if (P.newton) {  // clear F -> half sweep -> integrator
    launch_lj_half(P, B, n, 0, s);
    k_lj_half_vv<<<nb(n), 256, 0, s>>>(P, B, (int)n, dt, mode);
    return;
  }
  const bool capped = P.lj.r_min > 0.f, peer = P.peer_n > 0;  // peer: fused ghost refresh
  const unsigned g = nb(n);
  if (B.rm) {  // row-major slices (long rows)
    if (peer) {
      if (capped) k_lj_step<true, true, true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
      else k_lj_step<false, true, true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
    } else {
      if (capped) k_lj_step<true, false, true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
      else k_lj_step<false, false, true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
    }
    return;
  }
  if (peer) {
    if (capped) k_lj_step<true, true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
    else k_lj_step<false, true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
    return;
  }
  if (capped) k_lj_step<true><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
  else k_lj_step<false><<<g, 256, 0, s>>>(P, B, (int)n, dt, mode, wphase);
}

void launch_lj_step(const Params &P, const Bufs &B, int64_t n, float dt, cudaStream_t s) {
  launch_lj_step_mode(P, B, n, dt, -1, s);
}

void launch_kick_drift(const Params &P, const Bufs &B, int64_t n, float dt, cudaStream_t s) {
  if (n > 0) k_kick_drift<<<nb(n), 256, 0, s>>>(P, B, (int)n, dt);
  else k_empty_step<<<1, 1, 0, s>>>(B.st, 0);
}

void launch_step_begin(const Bufs &B, cudaGraphConditionalHandle h, int use_handle,
                       cudaStream_t s) {
  k_step_begin<<<1, 1, 0, s>>>(B, h, use_handle);
}

void launch_ke(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n > 0) k_ke<<<nb(n), 256, 0, s>>>(P, B, (int)n);
}

}  // namespace pm
