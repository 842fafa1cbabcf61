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

// dW/dr / dw_norm
__device__ __forceinline__ float dw_shape(float q) {
  if (q < 1.0f) return q * fmaf(2.25f, q, -3.0f);
  if (q < 2.0f) {
    const float t = 2.0f - q;
    return -0.75f * t * t;
  }
  return 0.0f;
}

__device__ __forceinline__ float3 delta3(const Params &P, const float4 &xi, const float4 &xj) {
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

__device__ __forceinline__ double w_of(const Params &P, const float4 &xi, const float4 &xj,
                                       double inv_h) {
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float xa = a == 0 ? xi.x : a == 1 ? xi.y : xi.z;
    const float xb = a == 0 ? xj.x : a == 1 ? xj.y : xj.z;
    d[a] = P.box.per[a] ? (double)pair_delta1(xa, xb, P.box.L[a], P.box.halfL[a], 1)
                        : (double)xb - (double)xa;
  }
  const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  return w_shape64(r * inv_h);
}

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
    s += w_of(P, xi, xa, inv_h);
    if (rem > 1) s += w_of(P, xi, xb, inv_h);
    if (rem > 2) s += w_of(P, xi, xc, inv_h);
    if (rem > 3) s += w_of(P, xi, xd, inv_h);
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
  B.rhoP[i] = make_float2((float)rho, (float)pr);
  if (!isfinite(rho + pr)) raise_error(st, -8 /*PM_E_NONFINITE*/, (long long)B.gid[st->cur_id][i]);
}

__global__ void __launch_bounds__(256) k_sph_forces(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (B.kind[st->cur_id][i] & 1) {
    B.force[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const float4 *__restrict__ vel = B.vel[st->cur_pv];
  const float2 *__restrict__ rhoP = B.rhoP;
  const float4 xi = pos[i];
  const float4 vi = vel[i];
  const float2 rpi = rhoP[i];
  const int cnt = B.cnt[i];
  const int *nb = B.nbr + nbr_row_base(B, i);
  float ax = 0.f, ay = 0.f, az = 0.f;
  const float acb = P.sph.alpha * P.sph.cbar;
  auto pair = [&](int j, bool valid) {
    const float3 d = delta3(P, xi, __ldg(pos + j));  // x_j - x_i
    const float d2 = dist2(d.x, d.y, d.z);
    const float rinv = fast_rsqrt(d2);
    const float q = d2 * rinv * P.sph.inv_h;
    const float dwdr = P.sph.dw_norm * dw_shape(q);
    const float4 vj = __ldg(vel + j);
    const float2 rpj = __ldg(rhoP + j);
    // v_ij . r_ij with r_ij = x_i - x_j = -d
    const float vr = -((vi.x - vj.x) * d.x + (vi.y - vj.y) * d.y + (vi.z - vj.z) * d.z);
    const float mu = P.sph.h * vr / (d2 + P.sph.eta2);
    const float pi_ij = vr < 0.0f ? -acb * mu / (0.5f * (rpi.x + rpj.x)) : 0.0f;
    const float coef = P.sph.mass * ((rpi.y + rpj.y) / (rpi.x * rpj.x) + pi_ij);
    // a_i -= coef * grad_i W,  grad_i W = (x_i - x_j)/r dW/dr = -d rinv dwdr
    const float sc = (valid && q < 2.0f) ? coef * rinv * dwdr : 0.0f;
    ax = fmaf(sc, d.x, ax);
    ay = fmaf(sc, d.y, ay);
    az = fmaf(sc, d.z, az);
  };
  for_row(nb, cnt, [&](int ja, int jb, int jc, int jd, int rem) {
    pair(ja, true);
    pair(jb, rem > 1);
    pair(jc, rem > 2);
    pair(jd, rem > 3);
  });
  ax += P.sph.g[0];
  ay += P.sph.g[1];
  az += P.sph.g[2];
  B.force[i] = make_float4(ax, ay, az, 0.f);
  if (!isfinite(ax + ay + az)) raise_error(st, -8 /*PM_E_NONFINITE*/, (long long)B.gid[st->cur_id][i]);
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

void launch_sph_density(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n > 0) k_sph_density<<<nb(n), 256, 0, s>>>(P, B, (int)n);
}

void launch_sph_forces(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n > 0) k_sph_forces<<<nb(n), 256, 0, s>>>(P, B, (int)n);
}

}  // namespace pm
