// k_verlet.cu -- Verlet neighbour list with skin.
//
// PAPER.md:164 (§4.1) "OpenFPM's implementation of Verlet lists [46]";
// PAPER.md:48 (§2) cell lists reduce the cut-off sum to O(N).  The list is
// the FULL list (both directions, no atomics in the force sweep): row i holds
// every j != i with d2_32(i, j) < r_v^2 (R4/R5), found over the 27-cell
// stencil of the cell list.  Layout: SELL-32 (one slice = one warp of 32
// consecutive cell-ordered particles) with a fixed per-row capacity; entry k
// of the 32 rows of a slice is one contiguous 128-byte line.
#include "pm_internal.cuh"

#include <algorithm>

namespace pm {

namespace {

// Scan one contiguous candidate range [b, e) (one x-run of cells in cell
// order).  Periodic images are handled per run (R4 "per-run
// shift"): if the run's cells were reached across the low face the whole run
// lies at the high end of the box and every candidate is shifted by -L
// (fl(x_j - L), exact by Sterbenz); if reached across the high face, the
// lane's own coordinate is shifted instead (xi_eff = fl(x_i - L), exact).
// For n >= 3 cells per periodic axis this reproduces R4's choice for every
// pair that can be a neighbour, so membership is bit-identical.  PAIRMI:
// apply the per-pair R4 rule along the axes in `pmi` -- a run that covers a
// whole periodic x-row, and the decomposed axes of a multi-GPU sub-domain
// (ghosts carry global wrapped coordinates).
//
// The membership test is d2 < rv2 (one compare); the particle itself is
// dropped by index, so a coincident distinct pair (d2 = 0) is listed and
// raised as PM_E_COINCIDENT by the cell sort (cells of <= 32 members) or the
// force sweep's non-finite path.  Lanes outside the current segment carry
// xi = +inf and never hit.
template <bool SHIFTJ, bool PAIRMI>
__device__ __forceinline__ float d2_of(const Params &P, const float4 &xi_eff, const float3 &csh,
                                       int pmi, const float4 &xj) {
  float dx = SHIFTJ ? __fsub_rn(__fsub_rn(xj.x, csh.x), xi_eff.x) : __fsub_rn(xj.x, xi_eff.x);
  float dy = SHIFTJ ? __fsub_rn(__fsub_rn(xj.y, csh.y), xi_eff.y) : __fsub_rn(xj.y, xi_eff.y);
  float dz = SHIFTJ ? __fsub_rn(__fsub_rn(xj.z, csh.z), xi_eff.z) : __fsub_rn(xj.z, xi_eff.z);
  if (PAIRMI) {
    if (pmi & 1) dx = pair_delta1(xi_eff.x, xj.x, P.box.L[0], P.box.halfL[0], 1);
    if (pmi & 2) dy = pair_delta1(xi_eff.y, xj.y, P.box.L[1], P.box.halfL[1], 1);
    if (pmi & 4) dz = pair_delta1(xi_eff.z, xj.z, P.box.L[2], P.box.halfL[2], 1);
  }
  return dist2(dx, dy, dz);
}

// Eight candidates j0 + u0 + u (u < 8) into bits u0 + u of the lane's hit
// mask: one compare d2 < rv2 and one predicated OR with an immediate each.
// The particle itself (d2 = 0) passes and is dropped at expansion; CLAMP:
// loads past the range end e are clamped to e - 1 (their bits are masked).
template <bool SHIFTJ, bool PAIRMI, int U0, bool CLAMP>
__device__ __forceinline__ void test8(const Params &P, const float4 *__restrict__ pos, int j0,
                                      int e, const float4 &xi_eff, const float3 &csh, int pmi,
                                      unsigned &msk) {
  float4 x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u)  // same address in all lanes
    x[u] = pos[CLAMP ? min(j0 + U0 + u, e - 1) : j0 + U0 + u];
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (d2_of<SHIFTJ, PAIRMI>(P, xi_eff, csh, pmi, x[u]) < P.rv2) msk |= 1u << (U0 + u);
}

// Candidates are tested 32 at a time into a per-lane hit mask; only the set
// bits (about 11% of them) are expanded into row entries, in candidate order.
// Membership is 0 < d2 < rv2 (R5): d2 == 0 is the particle itself (dropped
// by index; a coincident distinct pair is raised as PM_E_COINCIDENT by the
// cell sort).  Lanes outside the current segment carry xi = +inf and never
// hit.  An overflowing row keeps rewriting its last slot (min(k, cap-1)) and
// the build is retried.
// NMODE: 0 full rows; 1 half rows (j > i); 2 half rows of a decomposed
// context: owned partners j > i, ghost partners by the globally consistent
// rule gid_j > gid_i (each cross-boundary pair on exactly one rank, which
// returns the partner's share by pm_dist_ghost_put)
struct GhostRule {
  const int32_t *kind;
  const int64_t *gid;
  long long gid_self;
};

template <bool SHIFTJ, bool PAIRMI, int NMODE>
__device__ __forceinline__ void scan_run(const Params &P, const float4 *__restrict__ pos, int b,
                                         int e, const float4 &xi_eff, float3 csh, int pmi,
                                         int self, int cap, int *__restrict__ row, int &k,
                                         const GhostRule &gr) {
  for (int j0 = b; j0 < e; j0 += 32) {
    unsigned msk = 0u;
    if (j0 + 32 <= e) {
      test8<SHIFTJ, PAIRMI, 0, false>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      test8<SHIFTJ, PAIRMI, 8, false>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      test8<SHIFTJ, PAIRMI, 16, false>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      test8<SHIFTJ, PAIRMI, 24, false>(P, pos, j0, e, xi_eff, csh, pmi, msk);
    } else {
      const int rem = e - j0;  // 1..31, warp-uniform
      test8<SHIFTJ, PAIRMI, 0, true>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      if (rem > 8) test8<SHIFTJ, PAIRMI, 8, true>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      if (rem > 16) test8<SHIFTJ, PAIRMI, 16, true>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      if (rem > 24) test8<SHIFTJ, PAIRMI, 24, true>(P, pos, j0, e, xi_eff, csh, pmi, msk);
      msk &= (1u << rem) - 1u;
    }
    if (NMODE == 1) {  // half list (NEXT-1): only j > i, each pair once
      const int t = self - j0;
      msk &= t < 0 ? 0xffffffffu : (t >= 31 ? 0u : (0xffffffffu << (t + 1)));
    } else if (self >= j0 && self < j0 + 32) {  // drop the particle itself
      msk &= ~(1u << (self - j0));
    }
    while (msk) {
      const int u = __ffs(msk) - 1;
      msk &= msk - 1u;
      if (NMODE == 2) {
        const int j = j0 + u;
        if ((gr.kind[j] & kGhostBit) ? (gr.gid[j] < gr.gid_self) : (j < self)) continue;
      }
      row[(int64_t)min(k, cap - 1) << 5] = j0 + u;
      ++k;
    }
  }
}

template <int NMODE>
__device__ __forceinline__ void scan_any(const Params &P, const float4 *__restrict__ pos, int b,
                                         int e, const float4 &xi_eff, float3 csh, int pmi,
                                         int self, int cap, int *__restrict__ row, int &k,
                                         const GhostRule &gr) {
  const bool sj = csh.x != 0.f || csh.y != 0.f || csh.z != 0.f;
  if (pmi) scan_run<true, true, NMODE>(P, pos, b, e, xi_eff, csh, pmi, self, cap, row, k, gr);
  else if (sj) scan_run<true, false, NMODE>(P, pos, b, e, xi_eff, csh, 0, self, cap, row, k, gr);
  else scan_run<false, false, NMODE>(P, pos, b, e, xi_eff, csh, 0, self, cap, row, k, gr);
}

// Thread per particle (row), warp-uniform candidate stream.  The warp's 32
// consecutive cell-ordered particles occupy a few consecutive cells; for each
// x-row segment [c_first, c_last] of those cells, every lane scans the union
// of the segment's 27-cell stencils: 9 (dy, dz) rows, each one contiguous x
// range [c_first - 1, c_last + 1] of cells = one contiguous index range in
// cell order.  A lane only tests candidates of its own segment, and the
// union has no repeats, so row i gets every j with d2 < r_v^2 exactly once
// (the extra candidates of the union are farther than r_v and rejected by
// the same pinned test).  All lanes read the same position each iteration
// (broadcast), there is no divergence, and rows come out in a fixed order.
// RCH: stencil half-width in cells (P.reach), 1 (27 cells) or 2 (125 cells);
// NMODE: row kind (scan_run)
template <int RCH, int NMODE>
__global__ void __launch_bounds__(256, 4) k_verlet(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int wbase = i - lane;
  if (wbase >= n) return;  // whole warp out of range
  // rows: every particle on one GPU; owned particles only in a sub-domain
  const bool active = i < n && !(P.dist && (B.kind[st->cur_id][i] & kGhostBit));
  // capacity of this warp's slice (warp == slice: 256-thread blocks)
  const int cap = (i - lane < n) ? nbr_row_cap(B, i - lane) : 0;
  const int nx = P.grid.n[0], ny = P.grid.n[1], nz = P.grid.n[2];
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const float4 xi = active ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  GhostRule gr{nullptr, nullptr, 0};
  if (NMODE == 2) {
    gr.kind = B.kind[st->cur_id];
    gr.gid = B.gid[st->cur_id];
    gr.gid_self = active ? B.gid[st->cur_id][i] : 0;
  }
  int cell = -1;
  if (active) {
    const int c0 = local_coord(P.box, P.grid, 0, xi.x);
    const int c1 = local_coord(P.box, P.grid, 1, xi.y);
    const int c2 = local_coord(P.box, P.grid, 2, xi.z);
    cell = c0 + nx * (c1 + ny * c2);
  }
  // axes with the per-pair R4 rule: decomposed (globally periodic, locally open)
  const int pmi_dec = (P.box.per[0] && !P.grid.wrap[0] ? 1 : 0) |
                      (P.box.per[1] && !P.grid.wrap[1] ? 2 : 0) |
                      (P.box.per[2] && !P.grid.wrap[2] ? 4 : 0);
  const int row_id = active ? cell / nx : 0x7fffffff;  // (cy, cz) row of my cell
  int *__restrict__ row = B.nbr + nbr_row_base(B, i - lane) + lane;
  int k = 0;
  const float INF = __int_as_float(0x7f800000);
  const float Lx = P.box.L[0], Ly = P.box.L[1], Lz = P.box.L[2];
  unsigned todo = __ballot_sync(0xffffffffu, active);
  while (todo) {
    // segment = lanes whose cell lies in the row of the lowest pending lane
    const int lead = __ffs(todo) - 1;
    const int seg_row = __shfl_sync(0xffffffffu, row_id, lead);
    const bool mine = active && row_id == seg_row;
    const unsigned seg = __ballot_sync(0xffffffffu, mine);
    todo &= ~seg;
    int cmin = mine ? cell % nx : 0x7fffffff, cmax = mine ? cell % nx : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
      cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    const int cy = seg_row % ny, cz = seg_row / ny;
    constexpr int R = RCH;
    int xa = cmin - R, xb = cmax + R;
    // per-pair R4 along x: a run covering a whole periodic x-row, or (a
    // decomposed x) a run touching cells that may hold wrapped particles
    int pmi_x = 0;
    if (!P.grid.wrap[0]) {
      xa = max(xa, 0);
      xb = min(xb, nx - 1);
      if ((pmi_dec & 1) && !(xa >= P.grid.safe_lo[0] && xb <= P.grid.safe_hi[0])) pmi_x = 1;
    } else if (xb - xa + 1 >= nx) {
      xa = 0;
      xb = nx - 1;
      pmi_x = 1;
    }
    for (int dz = -R; dz <= R; ++dz) {
      int qz = cz + dz;
      float shz = 0.f, lz = 0.f;  // candidate shift / own shift along z
      if (qz < 0 || qz >= nz) {
        if (!P.grid.wrap[2]) continue;
        if (qz < 0) { qz += nz; shz = Lz; } else { qz -= nz; lz = Lz; }
      }
      for (int dy = -R; dy <= R; ++dy) {
        int qy = cy + dy;
        float shy = 0.f, ly = 0.f;
        if (qy < 0 || qy >= ny) {
          if (!P.grid.wrap[1]) continue;
          if (qy < 0) { qy += ny; shy = Ly; } else { qy -= ny; ly = Ly; }
        }
        const int rowc = nx * (qy + ny * qz);
        const int pmi = pmi_x |
                        ((pmi_dec & 2) && !(min(cy, qy) >= P.grid.safe_lo[1] &&
                                            max(cy, qy) <= P.grid.safe_hi[1]) ? 2 : 0) |
                        ((pmi_dec & 4) && !(min(cz, qz) >= P.grid.safe_lo[2] &&
                                            max(cz, qz) <= P.grid.safe_hi[2]) ? 4 : 0);
        // x range [xa, xb] of cells, split at the periodic seam
        int a0 = xa, b0 = xb, a1 = 0, b1 = -1;
        float sx0 = 0.f, lx0 = 0.f, sx1 = 0.f, lx1 = 0.f;
        if (xa < 0) {  // part [xa, -1] wrapped to the high end
          a0 = xa + nx; b0 = nx - 1; sx0 = Lx;
          a1 = 0; b1 = xb;
        } else if (xb > nx - 1) {  // part [nx, xb] wrapped to the low end
          a0 = xa; b0 = nx - 1;
          a1 = 0; b1 = xb - nx; lx1 = Lx;
        }
        // lanes outside this segment test against +inf: they never hit
        const float4 xe0 = mine ? make_float4(__fsub_rn(xi.x, lx0), __fsub_rn(xi.y, ly),
                                              __fsub_rn(xi.z, lz), 0.f)
                                : make_float4(INF, INF, INF, 0.f);
        scan_any<NMODE>(P, pos, B.start[rowc + a0], B.start[rowc + b0 + 1], xe0,
                 make_float3((pmi & 1) ? 0.f : sx0, shy, shz), pmi, i, cap, row, k, gr);
        if (b1 >= a1) {
          const float4 xe1 = mine ? make_float4(__fsub_rn(xi.x, lx1), __fsub_rn(xi.y, ly),
                                                __fsub_rn(xi.z, lz), 0.f)
                                  : make_float4(INF, INF, INF, 0.f);
          scan_any<NMODE>(P, pos, B.start[rowc + a1], B.start[rowc + b1 + 1], xe1,
                   make_float3(sx1, shy, shz), pmi & ~1, i, cap, row, k, gr);
        }
      }
    }
  }
  if (active) {
    // pad the row to a multiple of 4 with this particle's own index (a valid
    // index; the force sweep reads groups of 4 and masks padding slots)
    for (int q = k; q < cap && (q & 3) != 0; ++q) row[q << 5] = i;
  }
  if (i < n) B.cnt[i] = active ? k : 0;  // ghost rows are empty
  int kmax = k;
  long long ksum = k;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
  }
  if (lane == 0 && ksum > 0) {
    atomicMax(&st->max_row, kmax);
    atomicAdd(reinterpret_cast<unsigned long long *>(&st->nnz), (unsigned long long)ksum);
    if (kmax > cap) {  // the host re-lays the slices out from the exact counts
      atomicMax(&st->overflow_need, kmax);
      raise_error(st, -9 /*PM_E_CAPACITY*/, -1);
    }
  }
}

__global__ void k_reset_build_stats(State *st) {
  st->max_row = 0;
  st->nnz = 0;
  if (st->coinc_gid >= 0) raise_error(st, -7 /*PM_E_COINCIDENT*/, st->coinc_gid);
}

// CSR export of the list for the getters: col_gid[row_ptr[i] + k] = gid(nbr).
__global__ void __launch_bounds__(256) k_verlet_export(Bufs B, int n,
                                                      const int64_t *__restrict__ row_ptr,
                                                      int64_t *__restrict__ col_gid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t *gid = B.gid[B.st->cur_id];
  const int *nb = B.nbr + nbr_row_base(B, i);
  const int c = B.cnt[i];
  for (int k = 0; k < c; ++k) col_gid[row_ptr[i] + k] = gid[nb[k << 5]];
}

// Image shift of every list entry (R4/R5 sets of (gid_i, gid_j, shift)): per
// periodic axis -1 / +1 when the pinned rule moved x_j by -L / x_i by -L at
// the build (positions of the last build, xref), 0 otherwise.
__global__ void __launch_bounds__(256) k_verlet_shifts(Params P, Bufs B, int n,
                                                      const int64_t *__restrict__ row_ptr,
                                                      int8_t *__restrict__ col_shift) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int *nb = B.nbr + nbr_row_base(B, i);
  const int c = B.cnt[i];
  const float4 xi = B.xref[i];
  for (int k = 0; k < c; ++k) {
    const float4 xj = B.xref[nb[k << 5]];
    const float a[3] = {xi.x, xi.y, xi.z}, b[3] = {xj.x, xj.y, xj.z};
    int8_t *o = col_shift + 3 * (row_ptr[i] + k);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float e = __fsub_rn(b[d], a[d]);
      o[d] = (int8_t)(P.box.per[d] ? (e > P.box.halfL[d] ? -1 : (e < -P.box.halfL[d] ? 1 : 0)) : 0);
    }
  }
}

}  // namespace

void launch_verlet(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  k_reset_build_stats<<<1, 1, 0, s>>>(B.st);
  if (n <= 0) return;
  const unsigned g = (unsigned)((n + 255) / 256);
  const int nm = P.newton ? (P.dist ? 2 : 1) : 0;
  if (P.reach == 2) {
    if (nm == 1) k_verlet<2, 1><<<g, 256, 0, s>>>(P, B, (int)n);
    else k_verlet<2, 0><<<g, 256, 0, s>>>(P, B, (int)n);
  } else {
    if (nm == 2) k_verlet<1, 2><<<g, 256, 0, s>>>(P, B, (int)n);
    else if (nm == 1) k_verlet<1, 1><<<g, 256, 0, s>>>(P, B, (int)n);
    else k_verlet<1, 0><<<g, 256, 0, s>>>(P, B, (int)n);
  }
}

void launch_verlet_shifts(const Params &P, const Bufs &B, int64_t n, const int64_t *row_ptr,
                          int8_t *col_shift, cudaStream_t s) {
  if (n > 0)
    k_verlet_shifts<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, B, (int)n, row_ptr, col_shift);
}

void launch_verlet_export(const Bufs &B, int64_t n, const int64_t *row_ptr, int64_t *col_gid,
                          cudaStream_t s) {
  if (n > 0)
    k_verlet_export<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(B, (int)n, row_ptr, col_gid);
}

}  // namespace pm
