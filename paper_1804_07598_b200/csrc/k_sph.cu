// k_sph.cu -- WCSPH density/pressure pass.
//
// PAPER.md:330-350 (§4.2): Eq. 1 momentum, Eq. 3 Tait EOS, Eq. 4 constant b,
// Eq. 5 artificial viscosity; "classic cubic SPH kernel [34]".
// Readings: R16 density summation with the self term, R17
// a_p = -sum m (...) grad_p W(x_p - x_q), R18 (P_p+P_q)/(rho_p rho_q) as
// printed, R20 Monaghan viscosity branch (v_pq . r_pq < 0) with cbar = c0.
// Both passes sweep the full Verlet list built with r_v = 2h (skin 0), one
// thread per particle, fp32, no atomics.
#include "pm_internal.cuh"

namespace pm {

namespace {

// dW/dr / dw_norm (branch-free: both pieces evaluated and selected)
__device__ __forceinline__ float dw_shape(float q) {
  const float inner = q * fmaf(2.25f, q, -3.0f);
  const float t = 2.0f - q;
  const float outer = -0.75f * t * t;
  return q < 1.0f ? inner : (q < 2.0f ? outer : 0.0f);
}

template <bool PER>
__device__ __forceinline__ float3 delta3t(const Params &P, const float4 &xi, const float4 &xj) {
  if (!PER) return make_float3(__fsub_rn(xj.x, xi.x), __fsub_rn(xj.y, xi.y), __fsub_rn(xj.z, xi.z));
  return make_float3(pair_delta1(xi.x, xj.x, P.box.L[0], P.box.halfL[0], P.box.per[0]),
                     pair_delta1(xi.y, xj.y, P.box.L[1], P.box.halfL[1], P.box.per[1]),
                     pair_delta1(xi.z, xj.z, P.box.L[2], P.box.halfL[2], P.box.per[2]));
}

// Density summation in fp64: the Tait EOS
// amplifies density errors by gamma / ((rho/rho0)^gamma - 1) ~ 370 near rho0,
// so fp32 sums (~2e-7 relative) would give ~1e-3 errors in the pressure
// force.  Pair differences of the fp32 positions are exact in fp64 on
// non-periodic axes; B200 runs fp64 at half the fp32 rate.
__device__ __forceinline__ double w_shape64(double q) {
  if (q < 1.0) return fma(q * q, fma(0.75, q, -1.5), 1.0);
  if (q < 2.0) {
    const double t = 2.0 - q;
    return 0.25 * t * t * t;
  }
  return 0.0;
}

// Both passes read the row in groups of 4 with the index stream prefetched
// two groups ahead (as the LJ sweep); rows are padded to a multiple of 4 with
// the row's own index, masked here.
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

template <class F>
__device__ __forceinline__ void for_row(const int *__restrict__ nb, int cnt, F &&pair) {
  const int ng = (cnt + 3) >> 2;
  if (ng == 0) return;
  Idx4 j0 = ld_idx4(nb);
  Idx4 j1 = (ng > 1) ? ld_idx4(nb + 128) : j0;
  for (int g = 0; g < ng; ++g) {
    const Idx4 j2 = (g + 2 < ng) ? ld_idx4(nb + (g + 2) * 128) : j1;
    const int rem = cnt - 4 * g;
    pair(j0.a, j0.b, j0.c, j0.d, rem);
    j0 = j1;
    j1 = j2;
  }
}

template <bool PER>
__device__ __forceinline__ double w_of(const Params &P, const float4 &xi, const float4 &xj,
                                       double inv_h) {
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float xa = a == 0 ? xi.x : a == 1 ? xi.y : xi.z;
    const float xb = a == 0 ? xj.x : a == 1 ? xj.y : xj.z;
    d[a] = (PER && P.box.per[a]) ? (double)pair_delta1(xa, xb, P.box.L[a], P.box.halfL[a], 1)
                                 : (double)xb - (double)xa;
  }
  const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  return w_shape64(r * inv_h);
}

template <bool PER>
__global__ void __launch_bounds__(256) k_sph_density(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const float4 xi = pos[i];
  const int cnt = B.cnt[i];
  const int *nb = B.nbr + nbr_row_base(B, i);
  const double inv_h = 1.0 / (double)P.sph.h;
  double s = 0.0;
  for_row(nb, cnt, [&](int ja, int jb, int jc, int jd, int rem) {
    const float4 xa = __ldg(pos + ja), xb = __ldg(pos + jb);
    const float4 xc = __ldg(pos + jc), xd = __ldg(pos + jd);
    s += w_of<PER>(P, xi, xa, inv_h);
    if (rem > 1) s += w_of<PER>(P, xi, xb, inv_h);
    if (rem > 2) s += w_of<PER>(P, xi, xc, inv_h);
    if (rem > 3) s += w_of<PER>(P, xi, xd, inv_h);
  });
  const double h = P.sph.h;
  const double rho = (double)P.sph.mass / (3.14159265358979323846 * h * h * h) * (1.0 + s);
  const double x = rho / (double)P.sph.rho0;
  double xg;
  if (P.sph.gamma == 7.0f) {
    const double x2 = x * x;
    xg = x2 * x2 * x2 * x;
  } else {
    xg = pow(x, (double)P.sph.gamma);
  }
  const double pr = (double)P.sph.b * (xg - 1.0);
  B.rhoP[st->cur_id][i] = make_float2((float)rho, (float)pr);
  if (!isfinite(rho + pr)) raise_error(st, -8 /*PM_E_NONFINITE*/, (long long)B.gid[st->cur_id][i]);
}

// Forces of the pass: rho and P were packed into vel.w and pos.w by
// k_sph_pack_w (as during a run), so a pair costs two 16-byte gathers.
template <bool PER>
__global__ void __launch_bounds__(256, 3) k_sph_forces(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (B.kind[st->cur_id][i] & 1) {
    B.force[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const float4 *__restrict__ vel = B.vel[st->cur_pv];
  const float4 xi = pos[i];
  const float4 vi = vel[i];
  const int cnt = B.cnt[i];
  const int *nb = B.nbr + nbr_row_base(B, i);
  float ax = 0.f, ay = 0.f, az = 0.f;
  const float acb = P.sph.alpha * P.sph.cbar;
  // gathers of the four pairs first, one approximate reciprocal per pair (as k_sph_rates)
  auto pair = [&](const float4 &xj, const float4 &vj, bool valid) {
    const float3 d = delta3t<PER>(P, xi, xj);  // x_j - x_i
    const float d2 = dist2(d.x, d.y, d.z);
    const float rinv = fast_rsqrt(d2);
    const float q = d2 * rinv * P.sph.inv_h;
    const float dwdr = P.sph.dw_norm * dw_shape(q);
    // v_ij . r_ij with r_ij = x_i - x_j = -d
    const float vr = -((vi.x - vj.x) * d.x + (vi.y - vj.y) * d.y + (vi.z - vj.z) * d.z);
    const float den_mu = d2 + P.sph.eta2, rr = vi.w * vj.w, rs = vi.w + vj.w;
    const float rcp = fast_rcp(den_mu * rr * rs);  // the three quotients from one reciprocal
    const float mu = P.sph.h * vr * (rr * rs) * rcp;
    const float pi_ij = vr < 0.0f ? -2.0f * acb * mu * (den_mu * rr * rcp) : 0.0f;
    const float coef = P.sph.mass * ((xi.w + xj.w) * (den_mu * rs * rcp) + pi_ij);
    // a_i -= coef * grad_i W,  grad_i W = (x_i - x_j)/r dW/dr = -d rinv dwdr
    const float sc = (valid && q < 2.0f) ? coef * rinv * dwdr : 0.0f;
    ax = fmaf(sc, d.x, ax);
    ay = fmaf(sc, d.y, ay);
    az = fmaf(sc, d.z, az);
  };
  for_row(nb, cnt, [&](int ja, int jb, int jc, int jd, int rem) {
    const float4 xa = __ldg(pos + ja), xb = __ldg(pos + jb);
    const float4 xc = __ldg(pos + jc), xd = __ldg(pos + jd);
    const float4 va = __ldg(vel + ja), vb = __ldg(vel + jb);
    const float4 vc = __ldg(vel + jc), vd = __ldg(vel + jd);
    pair(xa, va, true);
    pair(xb, vb, rem > 1);
    pair(xc, vc, rem > 2);
    pair(xd, vd, rem > 3);
  });
  ax += P.sph.g[0];
  ay += P.sph.g[1];
  az += P.sph.g[2];
  B.force[i] = make_float4(ax, ay, az, 0.f);
  if (!isfinite(ax + ay + az)) raise_error(st, -8 /*PM_E_NONFINITE*/, (long long)B.gid[st->cur_id][i]);
}

// rho, P of the pass into the w lanes the force sweep gathers
__global__ void __launch_bounds__(256) k_sph_pack_w(Bufs B, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 rp = B.rhoP[B.st->cur_id][i];
  B.pos[B.st->cur_pv][i].w = rp.y;
  B.vel[B.st->cur_pv][i].w = rp.x;
}

// ---------------------------------------------------------------------------
// WCSPH time stepping (SURVEY §8(f) NEXT-3; PAPER.md:335 Eq. 2, :358
// "Verlet time-stepping [46] with dynamic step size"; readings R26-R28 in
// DESIGN.md, the same definitions as oracle/pm_oracle.c orc_sph_run):
//   k_sph_rates : D_p = sum_q m v_pq . grad_p W (all particles), a_p = Eq. 1
//                 + g (fluid), and the step-size bounds sqrt(h/|a_p|) (fluid)
//                 and h/(c0 + max_q |mu_pq|), reduced with atomicMin;
//   k_sph_dt    : dt = cfl * min(bounds); Euler step on the first and every
//                 `every`-th step, else leapfrog Verlet;
//   k_sph_verlet: rho' (all), v', x' (fluid), P' = EOS(rho'), rebuild test.
// fp32 like the sweeps.  During a run the density and pressure ride in
// vel.w and pos.w (what the sweep gathers) and the previous-step velocity and
// density in vold (w = density); vold and rhoP (the getters' copy) travel with
// the particles through the cell-sort reorder (Params::sph_state) and the
// multi-GPU migration records; ghosts receive pos and vel each step.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_min_atomic(unsigned *dst, float v) {
  unsigned u = __float_as_uint(v);  // v >= 0: uint order = float order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u = min(u, __shfl_xor_sync(0xffffffffu, u, o));
  if ((threadIdx.x & 31) == 0) atomicMin(dst, u);
}

template <bool PER>
__global__ void __launch_bounds__(256, 3) k_sph_rates(Params P, Bufs B, int n) {
  State *st = B.st;
  if (st->abort) return;  // a failed in-graph rebuild: the host resumes
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int cp = st->cur_pv, ci = st->cur_id;
  // ghost copies of a decomposed context: no row, no rate, no step bound
  const bool active = i < n && !(P.dist && (B.kind[ci][i] & kGhostBit));
  // pos.w = P and vel.w = rho during a run (k_sph_init_run, k_sph_verlet):
  // two 16-byte gathers per pair instead of three.
  const float4 *__restrict__ pos = B.pos[cp];
  const float4 *__restrict__ vel = B.vel[cp];
  float ax = 0.f, ay = 0.f, az = 0.f, D = 0.f, mumax = 0.f;
  bool fluid = false;
  if (active) {
    fluid = !(B.kind[ci][i] & 1);
    const float4 xi = pos[i];
    const float4 vi = vel[i];
    const float acb = P.sph.alpha * P.sph.cbar;
    // The four pairs' gathers are issued before any of their arithmetic
    // (memory-level parallelism per thread); the three quotients of a pair
    // come from one approximate reciprocal (no IEEE slow path branching the
    // loop) and the kernel derivative is branch-free.
    auto pair = [&](const float4 &xj, const float4 &vj, bool valid) {
      const float3 d = delta3t<PER>(P, xi, xj);  // x_j - x_i
      const float d2 = dist2(d.x, d.y, d.z);
      const float rinv = fast_rsqrt(d2);
      const float q = d2 * rinv * P.sph.inv_h;
      const bool in = valid && q < 2.0f && d2 > 0.0f;
      const float dwdr = P.sph.dw_norm * dw_shape(q);
      // r_ij = x_i - x_j = -d;  grad_i W = r_ij / r dW/dr = -d rinv dwdr
      const float vx = vi.x - vj.x, vy = vi.y - vj.y, vz = vi.z - vj.z;
      const float vd = vx * d.x + vy * d.y + vz * d.z;  // = -(v_ij . r_ij)
      const float gsc = rinv * dwdr;
      const float vr = -vd;
      // the three quotients from one reciprocal: 1 / [(d2 + eta2) rho_i rho_j
      // (rho_i + rho_j)]
      const float den_mu = d2 + P.sph.eta2, rr = vi.w * vj.w, rs = vi.w + vj.w;
      const float rcp = fast_rcp(den_mu * rr * rs);
      const float mu = P.sph.h * vr * (rr * rs) * rcp;       // h vr / (d2 + eta2)
      const float inv_rr = den_mu * rs * rcp;                // 1 / (rho_i rho_j)
      const float inv_rs = den_mu * rr * rcp;                // 1 / (rho_i + rho_j)
      const float pi_ij = vr < 0.0f ? -2.0f * acb * mu * inv_rs : 0.0f;
      const float coef = P.sph.mass * ((xi.w + xj.w) * inv_rr + pi_ij);
      const float sc = in ? coef * gsc : 0.0f;
      ax = fmaf(sc, d.x, ax);  // a_i -= coef grad_i W
      ay = fmaf(sc, d.y, ay);
      az = fmaf(sc, d.z, az);
      D += in ? -P.sph.mass * vd * gsc : 0.0f;  // m v_ij . grad_i W
      mumax = in ? fmaxf(mumax, fabsf(mu)) : mumax;
    };
    const int cnt = B.cnt[i];
    const int *nb = B.nbr + nbr_row_base(B, i);
    for_row(nb, cnt, [&](int ja, int jb, int jc, int jd, int rem) {
      const float4 xa = __ldg(pos + ja), xb = __ldg(pos + jb);
      const float4 xc = __ldg(pos + jc), xd = __ldg(pos + jd);
      const float4 va = __ldg(vel + ja), vb = __ldg(vel + jb);
      const float4 vc = __ldg(vel + jc), vd = __ldg(vel + jd);
      pair(xa, va, true);
      pair(xb, vb, rem > 1);
      pair(xc, vc, rem > 2);
      pair(xd, vd, rem > 3);
    });
    if (fluid) {
      ax += P.sph.g[0];
      ay += P.sph.g[1];
      az += P.sph.g[2];
    } else {
      ax = ay = az = 0.f;
    }
    B.force[i] = make_float4(ax, ay, az, 0.f);
    B.drho[i] = D;
    if (!isfinite(ax + ay + az + D))
      raise_error(st, -8 /*PM_E_NONFINITE*/, (long long)B.gid[ci][i]);
  }
  const float INF = __int_as_float(0x7f800000);
  const float am = sqrtf(ax * ax + ay * ay + az * az);
  const float dtf = (active && fluid && am > 0.f) ? sqrtf(P.sph.h / am) : INF;
  const float dtcv = active ? P.sph.h / (P.sph.cbar + mumax) : INF;
  warp_min_atomic(&st->dtf_bits, dtf);
  warp_min_atomic(&st->dtcv_bits, dtcv);
}

__global__ void k_sph_dt(State *st, float cfl, int every) {
  if (st->abort) return;
  const float dt = cfl * fminf(__uint_as_float(st->dtf_bits), __uint_as_float(st->dtcv_bits));
  st->sph_dt = dt;
  st->sph_dt_min = fminf(st->sph_dt_min, dt);
  st->sph_dt_max = fmaxf(st->sph_dt_max, dt);
  st->sph_time += (double)dt;
  const long long s = st->sph_step;
  st->mode = (s == 0 || (every > 0 && (s + 1) % every == 0)) ? 1 : 0;  // 1: Euler step
  st->sph_step = s + 1;
  st->dtf_bits = 0x7f800000u;
  st->dtcv_bits = 0x7f800000u;
  if (!(dt > 0.f) || !isfinite(dt)) {
    if (atomicCAS(&st->abort, 0, -8 /*PM_E_NONFINITE*/) == 0) st->err_gid = -1;
  }
}

// decomposed runs: the global minimum of the ranks' step bounds replaces the
// local one before k_sph_dt
__global__ void k_sph_set_bound(State *st, float bound) {
  st->dtf_bits = __float_as_uint(bound);
  st->dtcv_bits = 0x7f800000u;
}

__device__ __forceinline__ float tait(const Params &P, float rho) {
  const float x = rho * P.sph.inv_rho0;
  float xg;
  if (P.sph.gamma == 7.0f) {
    const float x2 = x * x;
    xg = x2 * x2 * x2 * x;
  } else {
    xg = powf(x, P.sph.gamma);
  }
  return P.sph.b * (xg - 1.0f);
}

__global__ void __launch_bounds__(256) k_sph_verlet(Params P, Bufs B, int n) {
  State *st = B.st;
  if (st->abort) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int cp = st->cur_pv, ci = st->cur_id;
  bool far = false;
  if (i < n) {
    const float4 x = B.pos[cp][i];
    const float4 v = B.vel[cp][i];
    if (P.dist && (B.kind[ci][i] & kGhostBit)) {  // ghost copy: refreshed by its owner
      B.pos[cp ^ 1][i] = x;
      B.vel[cp ^ 1][i] = v;
    } else {
      const float dt = st->sph_dt;
      const bool euler = st->mode == 1;
      const float D = B.drho[i];
      const float4 vo = B.vold[ci][i];
      const float rho = v.w, rold = vo.w;
      const float rn = euler ? fmaf(dt, D, rho) : fmaf(2.0f * dt, D, rold);
      const float pn = tait(P, rn);
      B.rhoP[ci][i] = make_float2(rn, pn);
      float4 xn = x, vn = v;
      if (!(B.kind[ci][i] & 1)) {
        const float4 a = B.force[i];
        const float h2 = 0.5f * dt * dt;
        vn.x = euler ? fmaf(dt, a.x, v.x) : fmaf(2.0f * dt, a.x, vo.x);
        vn.y = euler ? fmaf(dt, a.y, v.y) : fmaf(2.0f * dt, a.y, vo.y);
        vn.z = euler ? fmaf(dt, a.z, v.z) : fmaf(2.0f * dt, a.z, vo.z);
        float r3[3] = {fmaf(h2, a.x, fmaf(dt, v.x, x.x)), fmaf(h2, a.y, fmaf(dt, v.y, x.y)),
                       fmaf(h2, a.z, fmaf(dt, v.z, x.z))};
#pragma unroll
        for (int d = 0; d < 3; ++d)
          if (P.box.per[d]) r3[d] = wrap1(r3[d], P.box.lo[d], P.box.hi[d], P.box.L[d]);
        xn = make_float4(r3[0], r3[1], r3[2], 0.f);
        const float4 xr = B.xref[i];
        const float dx = pair_delta1(xr.x, xn.x, P.box.L[0], P.box.halfL[0], P.box.per[0]);
        const float dy = pair_delta1(xr.y, xn.y, P.box.L[1], P.box.halfL[1], P.box.per[1]);
        const float dz = pair_delta1(xr.z, xn.z, P.box.L[2], P.box.halfL[2], P.box.per[2]);
        far = dist2(dx, dy, dz) > P.half_skin2;
        if (!P.box.per[0] && (xn.x < P.box.lo[0] || xn.x >= P.box.hi[0])) far = true;
        if (!P.box.per[1] && (xn.y < P.box.lo[1] || xn.y >= P.box.hi[1])) far = true;
        if (!P.box.per[2] && (xn.z < P.box.lo[2] || xn.z >= P.box.hi[2])) far = true;
      }
      B.vold[ci][i] = v;  // w = rho: the previous-step density of the next step
      xn.w = pn;          // the packed P and rho k_sph_rates gathers
      vn.w = rn;
      B.pos[cp ^ 1][i] = xn;
      B.vel[cp ^ 1][i] = vn;
    }
  }
  if (__any_sync(0xffffffffu, far) && (threadIdx.x & 31) == 0) st->need_rebuild = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->pending_flip = 1;
    st->steps_done += 1;
  }
}

__global__ void __launch_bounds__(256) k_sph_set_rho(Params P, Bufs B, int n, const float *rho) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) B.rhoP[B.st->cur_id][i] = make_float2(rho[i], tait(P, rho[i]));
}

__global__ void __launch_bounds__(256) k_sph_init_run(Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int ci = st->cur_id;
  if (i < n) {
    const float2 rp = B.rhoP[ci][i];
    B.pos[st->cur_pv][i].w = rp.y;  // packed for k_sph_rates
    B.vel[st->cur_pv][i].w = rp.x;
    B.vold[ci][i] = B.vel[st->cur_pv][i];  // w = rho: the previous-step density
  }
  if (i == 0) {
    st->sph_step = 0;
    st->sph_time = 0.0;
    st->sph_dt = 0.f;
    st->sph_dt_min = __int_as_float(0x7f800000);
    st->sph_dt_max = 0.f;
    st->dtf_bits = 0x7f800000u;
    st->dtcv_bits = 0x7f800000u;
  }
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

static bool any_periodic(const Params &P) { return P.box.per[0] || P.box.per[1] || P.box.per[2]; }

// non-periodic boxes (the dam break) take the plain pair difference
void launch_sph_density(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  if (any_periodic(P)) k_sph_density<true><<<nb(n), 256, 0, s>>>(P, B, (int)n);
  else k_sph_density<false><<<nb(n), 256, 0, s>>>(P, B, (int)n);
}

void launch_sph_forces(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_sph_pack_w<<<nb(n), 256, 0, s>>>(B, (int)n);
  if (any_periodic(P)) k_sph_forces<true><<<nb(n), 256, 0, s>>>(P, B, (int)n);
  else k_sph_forces<false><<<nb(n), 256, 0, s>>>(P, B, (int)n);
}

void launch_sph_set_rho(const Params &P, const Bufs &B, int64_t n, const float *rho,
                        cudaStream_t s) {
  if (n > 0) k_sph_set_rho<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, B, (int)n, rho);
}

void launch_sph_init_run(const Bufs &B, int64_t n, cudaStream_t s) {
  k_sph_init_run<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(B, (int)n);
}

void launch_sph_rates(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  if (P.box.per[0] || P.box.per[1] || P.box.per[2])
    k_sph_rates<true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, B, (int)n);
  else
    k_sph_rates<false><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, B, (int)n);
}

// dt from `bound` (the global minimum) -> integrate (the caller applies the flip)
void launch_sph_update(const Params &P, const Bufs &B, int64_t n, float bound, float cfl,
                       int every, cudaStream_t s) {
  if (n <= 0) return;
  k_sph_set_bound<<<1, 1, 0, s>>>(B.st, bound);
  k_sph_dt<<<1, 1, 0, s>>>(B.st, cfl, every);
  k_sph_verlet<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, B, (int)n);
}

// rates -> dt -> integrate (the caller applies the buffer flip)
void launch_sph_step(const Params &P, const Bufs &B, int64_t n, float cfl, int every,
                     cudaStream_t s) {
  if (n <= 0) return;
  const unsigned nb = (unsigned)((n + 255) / 256);
  if (P.box.per[0] || P.box.per[1] || P.box.per[2])
    k_sph_rates<true><<<nb, 256, 0, s>>>(P, B, (int)n);
  else
    k_sph_rates<false><<<nb, 256, 0, s>>>(P, B, (int)n);
  k_sph_dt<<<1, 1, 0, s>>>(B.st, cfl, every);
  k_sph_verlet<<<nb, 256, 0, s>>>(P, B, (int)n);
}

}  // namespace pm
