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
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Staged build (the default whenever the widest slice fits in shared memory).
// Same segments, runs and pinned test as k_verlet, mapped differently:
//  * per (dy, dz) stencil row, lane t computes the row's candidate runs (up to
//    two pieces split at the periodic seam) into a per-warp piece table;
//  * the warp walks the pieces in stages of 128 candidates: each lane loads 4
//    candidates with coalesced 16-byte loads one stage AHEAD (registers), the
//    stage is written to shared memory with the run's candidate shift applied
//    (x, y of candidate pairs interleaved for paired fp32 arithmetic);
//  * every lane tests its own particle against the staged candidates two at a
//    time with sub/mul/fma.rn.f32x2 (FADD2/FMUL2/FFMA2: each half is the
//    single-rounded operation of R4/R4', so d2 is bit-identical to the scalar
//    test); hits are appended to the warp's rows kept in shared memory in the
//    SELL-32 layout of the slice (entry k of lane l at [k][l], conflict-free);
//  * at the end the slice's rows leave as full 128-byte lines (16-byte stores
//    over a contiguous range): no partial-line writes, no write amplification.
// ---------------------------------------------------------------------------
namespace stg {
constexpr int kWarps = 4;       // warps per block (independent of each other)
constexpr int kStage = 128;     // candidates per stage
constexpr int kOffBits = 10;    // row entry in shared memory: piece << 10 | offset
constexpr int kMaxPieceLen = 1 << kOffBits;
// stage: A = (x0, x1, y0, y1) and Z = (z0, z1, code0, code1) per candidate
// pair, then the stage slot of every own lane's self candidate (int[32])
constexpr int kStageBytes = kStage / 2 * 16 + kStage / 2 * 16 + 32 * 4;
template <int RCH>
struct Geo {
  static constexpr int NR = (2 * RCH + 1) * (2 * RCH + 1);  // stencil rows
  static constexpr int NP = 2 * NR;                        // pieces (seam split)
  static constexpr int kTable = NP * 40;                   // be + csh + osh
  __host__ __device__ static size_t warp_bytes(int wcap) {
    return (size_t)((kStageBytes + kTable + wcap * 64 + 15) & ~15);
  }
};
}  // namespace stg

typedef unsigned long long u64;
__device__ __forceinline__ u64 f2_pack(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(u64 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 f2_sub(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 f2_mul(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 f2_fma(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// The staged build's rows while a segment is scanned: per lane either 16-bit
// codes in shared memory (piece << 10 | offset in the piece, decoded when the
// segment ends) or, for segments with pieces longer than 1024 candidates
// (crowded cells), int32 indices stored straight into the global row.
struct StRows {
  unsigned short *sm;  // [k][lane] codes (64 bytes per line)
  int *gl;             // global row of this lane: entry k at gl[k * gs]
  bool direct;
  int gs;              // row stride: 32 (SELL-32 slices) or 1 (row-major slices)
};

// Append the hits of one group of 32 staged candidates (stage slots g + u,
// their codes in SZ) through the bit mask (overflow, half lists, direct rows).
template <int NMODE>
__device__ __forceinline__ void st_expand(unsigned msk, const float4 *__restrict__ SZ, int g,
                                          const int2 *__restrict__ PBE, int selfslot, int self,
                                          int cap, int lane, const StRows &R, int &k,
                                          const GhostRule &gr) {
  if (selfslot >= g && selfslot < g + 32) msk &= ~(1u << (selfslot - g));
  while (msk) {
    const int u = __ffs(msk) - 1;
    msk &= msk - 1u;
    const int v = g + u;
    const float4 zc = SZ[v >> 1];
    const unsigned code = __float_as_uint((v & 1) ? zc.w : zc.z);
    const int j = R.direct ? (int)code
                           : PBE[code >> stg::kOffBits].x + (int)(code & (stg::kMaxPieceLen - 1));
    if (NMODE == 1 && j <= self) continue;  // half rows: j > i only
    if (NMODE == 2) {
      if ((gr.kind[j] & kGhostBit) ? (gr.gid[j] < gr.gid_self) : (j < self)) continue;
    }
    const int kk = min(k, cap - 1);
    PM_CHECK(j >= 0 && kk >= 0);
    if (R.direct) R.gl[(int64_t)kk * R.gs] = j;
    else R.sm[(kk << 5) + lane] = (unsigned short)code;
    ++k;
  }
}

// R4 along one axis for two candidates at once (b = pair, a = the lane's
// coordinate): e = b - a; e > L/2: (b - L) - a; e < -L/2: b - (a - L); else e
// -- the single-rounded operations of pair_delta1, so bit-identical.  An axis
// without the per-pair rule passes hL = +inf (always e).
__device__ __forceinline__ u64 f2_r4(u64 B, float a, float L, float hL) {
  const u64 A = f2_pack(a, a);
  const u64 E = f2_sub(B, A);
  const u64 U = f2_sub(f2_sub(B, f2_pack(L, L)), A);
  const float am = __fsub_rn(a, L);
  const u64 D = f2_sub(B, f2_pack(am, am));
  float e0, e1, u0, u1, d0, d1;
  f2_unpack(E, e0, e1);
  f2_unpack(U, u0, u1);
  f2_unpack(D, d0, d1);
  const float r0 = e0 > hL ? u0 : (e0 < -hL ? d0 : e0);
  const float r1 = e1 > hL ? u1 : (e1 < -hL ? d1 : e1);
  return f2_pack(r0, r1);
}

// One group of up to 32 staged candidates (g .. g + gn, padded with +inf to
// a multiple of 8), appended to the lane's 16-bit row by predicated stores.
// PMI: the per-pair R4 rule on the axes in pmi (decomposed axes near the
// global faces, runs covering a whole periodic row).
template <bool PMI>
__device__ __forceinline__ void st_fast_group(const float4 *__restrict__ SA,
                                              const float4 *__restrict__ SZ, int g, int gn,
                                              const float4 &xe, const Box &box, int pmi,
                                              float rv2, unsigned short *rows, int lane,
                                              int &k) {
  const float INF = __int_as_float(0x7f800000);
  const u64 XI = f2_pack(xe.x, xe.x), YI = f2_pack(xe.y, xe.y), ZI = f2_pack(xe.z, xe.z);
  const float hx = (pmi & 1) ? box.halfL[0] : INF, hy = (pmi & 2) ? box.halfL[1] : INF,
              hz = (pmi & 4) ? box.halfL[2] : INF;
  const unsigned rows_sa = smem_u32(rows);
  unsigned bo = rows_sa + (unsigned)(((k << 5) + lane) << 1);
#pragma unroll
  for (int u8 = 0; u8 < 4; ++u8) {
    if (u8 >= ((gn + 7) >> 3)) break;
    // 8 candidates: loads first, then the arithmetic, then the appends
    float4 a[4], z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = SA[(g >> 1) + 4 * u8 + q];
#pragma unroll
    for (int q = 0; q < 4; ++q) z[q] = SZ[(g >> 1) + 4 * u8 + q];
    float sd[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      u64 dx, dy, dz;
      if (PMI) {
        dx = f2_r4(f2_pack(a[q].x, a[q].y), xe.x, box.L[0], hx);
        dy = f2_r4(f2_pack(a[q].z, a[q].w), xe.y, box.L[1], hy);
        dz = f2_r4(f2_pack(z[q].x, z[q].y), xe.z, box.L[2], hz);
      } else {
        dx = f2_sub(f2_pack(a[q].x, a[q].y), XI);
        dy = f2_sub(f2_pack(a[q].z, a[q].w), YI);
        dz = f2_sub(f2_pack(z[q].x, z[q].y), ZI);
      }
      u64 s2 = f2_mul(dx, dx);
      s2 = f2_fma(dy, dy, s2);
      s2 = f2_fma(dz, dz, s2);
      f2_unpack(s2, sd[2 * q], sd[2 * q + 1]);
    }
    // the hits only: a store with few active lanes costs one shared-memory
    // wavefront and (almost) never a bank conflict; the codes ride in Z.zw
#define PM_APPEND(S, C)                                                                \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, %3;\n\t"                      \
               "@p st.shared.u16 [%0], %2;\n\t@p add.u32 %0, %0, 64;\n\t}"             \
               : "+r"(bo)                                                              \
               : "f"(S), "r"(__float_as_uint(C)), "f"(rv2))
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      PM_APPEND(sd[2 * q], z[q].z);
      PM_APPEND(sd[2 * q + 1], z[q].w);
    }
#undef PM_APPEND
  }
  asm volatile("" ::: "memory");  // the C++ reads after this see the appends
  k = (int)((bo - rows_sa) >> 6);
  PM_CHECK(((bo - rows_sa) & 63u) == (unsigned)(lane << 1));
}

template <int RCH, int NMODE, bool RM = false>
__global__ void __launch_bounds__(stg::kWarps * 32, 5)
    k_verlet_st(Params P, Bufs B, int n, int wcap) {
  using namespace stg;
  constexpr int NR = Geo<RCH>::NR, NP = Geo<RCH>::NP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *wbase_s = smem_raw + (size_t)wid * Geo<RCH>::warp_bytes(wcap);
  float4 *SA = reinterpret_cast<float4 *>(wbase_s);
  float4 *SZ = reinterpret_cast<float4 *>(wbase_s + kStage / 2 * 16);
  int *SELF = reinterpret_cast<int *>(wbase_s + kStage / 2 * 32);  // stage slot of lane's self
  int2 *PBE = reinterpret_cast<int2 *>(wbase_s + kStageBytes);
  float4 *PCS = reinterpret_cast<float4 *>(wbase_s + kStageBytes + NP * 8);
  float4 *POS = PCS + NP;
  unsigned short *rows = reinterpret_cast<unsigned short *>(wbase_s + kStageBytes + NP * 40);
  State *st = B.st;
  const int i = (blockIdx.x * kWarps + wid) * 32 + lane;
  const int wbase = i - lane;
  if (wbase >= n) return;  // whole warp out of range
  const bool active = i < n && !(P.dist && (B.kind[st->cur_id][i] & kGhostBit));
  const int cap = nbr_row_cap(B, wbase);
  // the lane's row (a row of the slice also for i >= n); RM: row-major slices
  int *grow = B.nbr + B.slice_off[wbase >> 5] * 32 + (RM ? (int64_t)lane * cap : lane);
  constexpr int gs = RM ? 1 : 32;
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
  const int pmi_dec = (P.box.per[0] && !P.grid.wrap[0] ? 1 : 0) |
                      (P.box.per[1] && !P.grid.wrap[1] ? 2 : 0) |
                      (P.box.per[2] && !P.grid.wrap[2] ? 4 : 0);
  const int row_id = active ? cell / nx : 0x7fffffff;
  int k = 0;
  const float INF = __int_as_float(0x7f800000);
  const float rv2 = P.rv2;
  unsigned todo = __ballot_sync(0xffffffffu, active);
  while (todo) {
    const int lead = __ffs(todo) - 1;
    const int seg_row = __shfl_sync(0xffffffffu, row_id, lead);
    const bool mine = active && row_id == seg_row;
    const unsigned seg = __ballot_sync(0xffffffffu, mine);
    todo &= ~seg;
    int cmin = mine ? cell % nx : 0x7fffffff, cmax = mine ? cell % nx : -1;
    cmin = __reduce_min_sync(0xffffffffu, cmin);
    cmax = __reduce_max_sync(0xffffffffu, cmax);
    const int cy = seg_row % ny, cz = seg_row / ny;
    int xa = cmin - RCH, xb = cmax + RCH;
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
    __syncwarp();  // the previous segment's readers are done with the table
    bool long_piece = false;
    for (int t = lane; t < NR; t += 32) {  // stencil row t = (dz, dy), dz outer
      const int dz = t / (2 * RCH + 1) - RCH, dy = t % (2 * RCH + 1) - RCH;
      int2 be0 = make_int2(0, 0), be1 = make_int2(0, 0);
      float4 c0 = make_float4(0.f, 0.f, 0.f, 0.f), o0 = c0, c1 = c0, o1 = c0;
      bool ok = true;
      int qz = cz + dz;
      float shz = 0.f, lz = 0.f;
      if (qz < 0 || qz >= nz) {
        if (!P.grid.wrap[2]) ok = false;
        else if (qz < 0) { qz += nz; shz = P.box.L[2]; }
        else { qz -= nz; lz = P.box.L[2]; }
      }
      int qy = cy + dy;
      float shy = 0.f, ly = 0.f;
      if (qy < 0 || qy >= ny) {
        if (!P.grid.wrap[1]) ok = false;
        else if (qy < 0) { qy += ny; shy = P.box.L[1]; }
        else { qy -= ny; ly = P.box.L[1]; }
      }
      if (ok) {
        const int rowc = nx * (qy + ny * qz);
        const int pmi = pmi_x |
                        ((pmi_dec & 2) && !(min(cy, qy) >= P.grid.safe_lo[1] &&
                                            max(cy, qy) <= P.grid.safe_hi[1]) ? 2 : 0) |
                        ((pmi_dec & 4) && !(min(cz, qz) >= P.grid.safe_lo[2] &&
                                            max(cz, qz) <= P.grid.safe_hi[2]) ? 4 : 0);
        int a0 = xa, b0 = xb, a1 = 0, b1 = -1;
        float sx0 = 0.f, lx0 = 0.f, sx1 = 0.f, lx1 = 0.f;
        if (xa < 0) {
          a0 = xa + nx; b0 = nx - 1; sx0 = P.box.L[0];
          a1 = 0; b1 = xb;
        } else if (xb > nx - 1) {
          a0 = xa; b0 = nx - 1;
          a1 = 0; b1 = xb - nx; lx1 = P.box.L[0];
        }
        be0 = make_int2(B.start[rowc + a0], B.start[rowc + b0 + 1]);
        c0 = make_float4((pmi & 1) ? 0.f : sx0, shy, shz, __int_as_float(pmi));
        o0 = make_float4(lx0, ly, lz, 0.f);
        if (b1 >= a1) {
          be1 = make_int2(B.start[rowc + a1], B.start[rowc + b1 + 1]);
          c1 = make_float4(sx1, shy, shz, __int_as_float(pmi & ~1));
          o1 = make_float4(lx1, ly, lz, 0.f);
        }
      }
      long_piece |= (be0.y - be0.x > kMaxPieceLen) || (be1.y - be1.x > kMaxPieceLen);
      PBE[2 * t] = be0;
      PCS[2 * t] = c0;
      POS[2 * t] = o0;
      PBE[2 * t + 1] = be1;
      PCS[2 * t + 1] = c1;
      POS[2 * t + 1] = o1;
    }
    // wcap == 0: no shared-memory rows at all (rows too long for shared memory,
    // clustered inputs): every segment appends straight to its global rows
    const StRows R{rows, grow, wcap == 0 || __any_sync(0xffffffffu, long_piece) != 0, gs};
    __syncwarp();
    // bounding box of the segment's particles: candidates farther than r_v
    // (+1e-3) from it cannot be a neighbour of any lane and are not staged
    // (the pinned test decides for the rest; the margin only keeps extras)
    float bx0 = mine ? xi.x : INF, by0 = mine ? xi.y : INF, bz0 = mine ? xi.z : INF;
    float bx1 = mine ? xi.x : -INF, by1 = mine ? xi.y : -INF, bz1 = mine ? xi.z : -INF;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, o2));
      by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, o2));
      bz0 = fminf(bz0, __shfl_xor_sync(0xffffffffu, bz0, o2));
      bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, o2));
      by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, o2));
      bz1 = fmaxf(bz1, __shfl_xor_sync(0xffffffffu, bz1, o2));
    }
    const float rcull = sqrtf(rv2) + 1e-3f;
    const float rcull2 = rcull * rcull;
    // stage iterator over the pieces: (p, o) = piece, offset inside it
    int p = 0;
    while (p < NP && PBE[p].x >= PBE[p].y) ++p;
    int o = 0;
    float4 pre[4];
    if (p < NP) {
      const int2 be = PBE[p];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = be.x + lane + 32 * q;
        pre[q] = (j < be.y) ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    while (p < NP) {
      const int2 be = PBE[p];
      const int jb = be.x + o;
      const int craw = min(kStage, be.y - jb);
      const float4 csh = PCS[p], osh = POS[p];
      const int pmi = __float_as_int(csh.w);
      __syncwarp();  // the previous stage's readers are done
      SELF[lane] = -1;
      // the box in this piece's frame (own shift), the candidates in it
      // (candidate shift); no culling along per-pair-R4 axes
      const float lx0 = __fsub_rn(bx0, osh.x), lx1 = __fsub_rn(bx1, osh.x);
      const float ly0 = __fsub_rn(by0, osh.y), ly1 = __fsub_rn(by1, osh.y);
      const float lz0 = __fsub_rn(bz0, osh.z), lz1 = __fsub_rn(bz1, osh.z);
      int cntc = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = lane + 32 * q;
        const float cx = __fsub_rn(pre[q].x, csh.x), cy2 = __fsub_rn(pre[q].y, csh.y),
                    cz2 = __fsub_rn(pre[q].z, csh.z);
        const float ddx = (pmi & 1) ? 0.f : fmaxf(fmaxf(lx0 - cx, cx - lx1), 0.f);
        const float ddy = (pmi & 2) ? 0.f : fmaxf(fmaxf(ly0 - cy2, cy2 - ly1), 0.f);
        const float ddz = (pmi & 4) ? 0.f : fmaxf(fmaxf(lz0 - cz2, cz2 - lz1), 0.f);
        const bool keep = u < craw && ddx * ddx + ddy * ddy + ddz * ddz < rcull2;
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          const int v = cntc + __popc(km & ((1u << lane) - 1u));
          float *a = reinterpret_cast<float *>(&SA[v >> 1]);
          float *z = reinterpret_cast<float *>(&SZ[v >> 1]);
          a[v & 1] = cx;
          a[2 + (v & 1)] = cy2;
          z[v & 1] = cz2;
          // the entry's code (piece, offset); rows appended straight to global
          // memory carry the index itself (pieces may exceed the offset field)
          z[2 + (v & 1)] = __uint_as_float(R.direct ? (unsigned)(jb + u)
                                                    : (unsigned)((p << kOffBits) + o + u));
          const int jj = jb + u - wbase;  // a warp's own particle: its self slot
          if (jj >= 0 && jj < 32) SELF[jj] = v;
        }
        cntc += __popc(km);
      }
      const int cnt8 = (cntc + 7) & ~7;  // the tail up to a multiple of 8 holds +inf
      if (lane < cnt8 - cntc) {
        const int v = cntc + lane;
        float *a = reinterpret_cast<float *>(&SA[v >> 1]);
        float *z = reinterpret_cast<float *>(&SZ[v >> 1]);
        a[v & 1] = INF;
        a[2 + (v & 1)] = INF;
        z[v & 1] = INF;
        z[2 + (v & 1)] = 0.f;
      }
      // advance and prefetch the next stage (overlaps this stage's tests)
      int pn = p, on = o + kStage;
      if (on >= be.y - be.x) {
        on = 0;
        ++pn;
        while (pn < NP && PBE[pn].x >= PBE[pn].y) ++pn;
      }
      if (pn < NP) {
        const int2 bn = PBE[pn];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = bn.x + on + lane + 32 * q;
          pre[q] = (j < bn.y) ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      __syncwarp();
      const float4 xe = mine ? make_float4(__fsub_rn(xi.x, osh.x), __fsub_rn(xi.y, osh.y),
                                           __fsub_rn(xi.z, osh.z), 0.f)
                             : make_float4(INF, INF, INF, 0.f);
      const u64 XI = f2_pack(xe.x, xe.x), YI = f2_pack(xe.y, xe.y), ZI = f2_pack(xe.z, xe.z);
      const int sslot = SELF[lane];  // this lane's own candidate in this stage (-1: none)
      for (int g = 0; g < cntc; g += 32) {
        const int gn = min(32, cntc - g);
        // (every store of the group, the +inf padding included, stays below cap)
        if (NMODE == 0 && !R.direct && !__any_sync(0xffffffffu, k + ((gn + 7) & ~7) > cap)) {
          // fast path: every candidate's code is stored at the row's next
          // slot and the slot advances on a hit (no mask, no divergent
          // expansion); the +inf tail of the stage never hits
          const int k0 = k;
          if (pmi) st_fast_group<true>(SA, SZ, g, gn, xe, P.box, pmi, rv2, rows, lane, k);
          else st_fast_group<false>(SA, SZ, g, gn, xe, P.box, 0, rv2, rows, lane, k);
          // the particle itself (d2 = 0) was appended once: swap-remove it
          if (mine && sslot >= g && sslot < g + gn) {
            const unsigned short sc = (unsigned short)((p << kOffBits) + (i - PBE[p].x));
            for (int t = k0; t < k; ++t) {
              if (rows[(t << 5) + lane] == sc) {
                rows[(t << 5) + lane] = rows[((k - 1) << 5) + lane];
                --k;
                break;
              }
            }
          }
          continue;
        }
        unsigned msk = 0u;
        if (pmi) {  // per-pair R4 on the axes in pmi (scalar, rare)
          for (int u = 0; u < gn; ++u) {
            const int v = g + u;
            const float *a = reinterpret_cast<const float *>(&SA[v >> 1]);
            const float *z = reinterpret_cast<const float *>(&SZ[v >> 1]);
            const float4 xj = make_float4(a[v & 1], a[2 + (v & 1)], z[v & 1], 0.f);  // z.xy
            if (d2_of<false, true>(P, xe, make_float3(0.f, 0.f, 0.f), pmi, xj) < rv2)
              msk |= 1u << u;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (2 * q >= gn) break;
            const float4 a = SA[(g >> 1) + q];
            const float4 z = SZ[(g >> 1) + q];
            const u64 dx = f2_sub(f2_pack(a.x, a.y), XI);
            const u64 dy = f2_sub(f2_pack(a.z, a.w), YI);
            const u64 dz = f2_sub(f2_pack(z.x, z.y), ZI);
            u64 s2 = f2_mul(dx, dx);
            s2 = f2_fma(dy, dy, s2);
            s2 = f2_fma(dz, dz, s2);
            float s0, s1;
            f2_unpack(s2, s0, s1);
            if (s0 < rv2) msk |= 1u << (2 * q);
            if (s1 < rv2) msk |= 2u << (2 * q);
          }
          if (gn < 32) msk &= (1u << gn) - 1u;
        }
        st_expand<NMODE>(msk, SZ, g, PBE, mine ? sslot : -1, i, cap, lane, R, k, gr);
      }
      p = pn;
      o = on;
    }
    // segment end: the segment's rows go to global memory (decoded), padded
    // to a multiple of 4 with the particle's own index (the sweeps read groups
    // of 4 and mask padding slots)
    __syncwarp();
    const int kseg = __reduce_max_sync(0xffffffffu, mine ? min(k, cap) : 0);
    if (!R.direct) {
      for (int kk = 0; kk < kseg; ++kk) {
        if (mine && kk < k) {
          const unsigned c = rows[(kk << 5) + lane];
          PM_CHECK((int)(c >> kOffBits) < NP);
          const int j = PBE[c >> kOffBits].x + (int)(c & (kMaxPieceLen - 1));
          PM_CHECK(j >= 0 && j < n && j != i && j < PBE[c >> kOffBits].y);
          grow[(int64_t)kk * gs] = j;
        }
      }
    }
    if (mine)
      for (int q = min(k, cap); q < cap && (q & 3) != 0; ++q) grow[(int64_t)q * gs] = i;
  }
  if (i < n) B.cnt[i] = active ? k : 0;
  const int kmax = __reduce_max_sync(0xffffffffu, k);
  const unsigned ksum = __reduce_add_sync(0xffffffffu, (unsigned)k);
  if (lane == 0 && ksum > 0) {
    atomicMax(&st->max_row, kmax);
    atomicAdd(reinterpret_cast<unsigned long long *>(&st->nnz), (unsigned long long)ksum);
    if (kmax > cap) {
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
  const int gs = nbr_stride(B);
  for (int k = 0; k < c; ++k) col_gid[row_ptr[i] + k] = gid[nb[(int64_t)k * gs]];
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
    const float4 xj = B.xref[nb[(int64_t)k * nbr_stride(B)]];
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

// Shared memory of the staged build per block; 0 when the widest slice does
// not fit (clustered inputs with rows of thousands of entries: k_verlet).
template <int RCH>
static size_t staged_smem(int wcap) {
  const size_t tot = stg::kWarps * stg::Geo<RCH>::warp_bytes(wcap);
  return (wcap > 0 && tot <= 200 * 1024) ? tot : 0;
}

template <int RCH, int NMODE, bool RM = false>
static void launch_st(const Params &P, const Bufs &B, int64_t n, size_t sm, int wcap,
                      cudaStream_t s) {
  static size_t set = 0;
  if (sm > set) {
    cudaFuncSetAttribute(k_verlet_st<RCH, NMODE, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    set = sm;
  }
  const unsigned g = (unsigned)((n + stg::kWarps * 32 - 1) / (stg::kWarps * 32));
  k_verlet_st<RCH, NMODE, RM><<<g, stg::kWarps * 32, sm, s>>>(P, B, (int)n, wcap);
}

void launch_verlet(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  k_reset_build_stats<<<1, 1, 0, s>>>(B.st);
  if (n <= 0) return;
  const unsigned g = (unsigned)((n + 255) / 256);
  const int nm = P.newton ? (P.dist ? 2 : 1) : 0;
  // rows in shared memory when the widest slice fits, else the same kernel
  // appending straight to global rows (wcap = 0)
  size_t sm = P.reach == 2 ? staged_smem<2>(P.nbr_cap) : staged_smem<1>(P.nbr_cap);
  int wcap = P.nbr_cap;
  if (!sm) {
    wcap = 0;
    sm = stg::kWarps * (P.reach == 2 ? stg::Geo<2>::warp_bytes(0) : stg::Geo<1>::warp_bytes(0));
  }
  static const int staged_env = [] {
    const char *e = std::getenv("PM_VERLET_STAGED");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  if (staged_env || B.rm) {  // (the round-1 builder writes SELL-32 only)
    if (P.reach == 2) {
      if (nm == 1) launch_st<2, 1>(P, B, n, sm, wcap, s);
      else if (B.rm) launch_st<2, 0, true>(P, B, n, sm, wcap, s);
      else launch_st<2, 0>(P, B, n, sm, wcap, s);
    } else {
      if (nm == 2) launch_st<1, 2>(P, B, n, sm, wcap, s);
      else if (nm == 1) launch_st<1, 1>(P, B, n, sm, wcap, s);
      else if (B.rm) launch_st<1, 0, true>(P, B, n, sm, wcap, s);
      else launch_st<1, 0>(P, B, n, sm, wcap, s);
    }
    return;
  }
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
