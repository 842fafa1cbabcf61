// k_verlet.cu -- Verlet neighbour list with skin.
//
// PAPER.md:164 (§4.1) "OpenFPM's implementation of Verlet lists [46]";
// PAPER.md:48 (§2) cell lists reduce the cut-off sum to O(N).  The list is
// the FULL list (both directions, no atomics in the force sweep): row i holds
// every j != i with d2_32(i, j) < r_v^2 (R4/R5), found over the 27-cell
// stencil of the cell list.  Layout: SELL-32 (one slice = one warp of 32
// consecutive cell-ordered particles) with a fixed per-row capacity, entries
// interleaved by 4 so that the force sweep reads one coalesced int4 per lane
// per 4 neighbours.
#include "pm_internal.cuh"

namespace pm {

namespace {

__device__ __forceinline__ void put4(int4 &acc, int k, int j) {
  switch (k & 3) {
    case 0: acc.x = j; break;
    case 1: acc.y = j; break;
    case 2: acc.z = j; break;
    default: acc.w = j; break;
  }
}

__global__ void __launch_bounds__(256) k_verlet(Params P, Bufs B, int n) {
  State *st = B.st;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int cap = P.nbr_cap;
  int k = 0;
  if (i < n) {
    const float4 *__restrict__ pos = B.pos[st->cur_pv];
    const float4 xi = pos[i];
    const int c0 = cell_coord(xi.x, P.box.lo[0], P.grid.inv_w[0], P.grid.n[0]);
    const int c1 = cell_coord(xi.y, P.box.lo[1], P.grid.inv_w[1], P.grid.n[1]);
    const int c2 = cell_coord(xi.z, P.box.lo[2], P.grid.inv_w[2], P.grid.n[2]);
    int4 *__restrict__ out = reinterpret_cast<int4 *>(B.nbr) + nbr_base4(i, cap);
    int4 acc = make_int4(i, i, i, i);
    bool coincident = false;
    for (int dz = -1; dz <= 1; ++dz) {
      int cz = c2 + dz;
      if (cz < 0 || cz >= P.grid.n[2]) {
        if (!P.box.per[2]) continue;
        cz += (cz < 0) ? P.grid.n[2] : -P.grid.n[2];
      }
      for (int dy = -1; dy <= 1; ++dy) {
        int cy = c1 + dy;
        if (cy < 0 || cy >= P.grid.n[1]) {
          if (!P.box.per[1]) continue;
          cy += (cy < 0) ? P.grid.n[1] : -P.grid.n[1];
        }
        const int row = P.grid.n[0] * (cy + P.grid.n[1] * cz);
        for (int dx = -1; dx <= 1; ++dx) {
          int cx = c0 + dx;
          if (cx < 0 || cx >= P.grid.n[0]) {
            if (!P.box.per[0]) continue;
            cx += (cx < 0) ? P.grid.n[0] : -P.grid.n[0];
          }
          const int c = cx + row;
          const int s = B.start[c], e = B.start[c + 1];
          for (int j = s; j < e; ++j) {
            if (j == i) continue;
            const float4 xj = pos[j];
            const float dx_ = pair_delta1(xi.x, xj.x, P.box.L[0], P.box.halfL[0], P.box.per[0]);
            const float dy_ = pair_delta1(xi.y, xj.y, P.box.L[1], P.box.halfL[1], P.box.per[1]);
            const float dz_ = pair_delta1(xi.z, xj.z, P.box.L[2], P.box.halfL[2], P.box.per[2]);
            const float d2 = dist2(dx_, dy_, dz_);
            if (d2 < P.rv2) {
              coincident |= (d2 == 0.0f);
              if (k < cap) {
                put4(acc, k, j);
                if ((k & 3) == 3) out[(k >> 2) * 32] = acc;
              }
              ++k;
            }
          }
        }
      }
    }
    if ((k & 3) != 0 && k < cap) out[(k >> 2) * 32] = acc;
    B.cnt[i] = k < cap ? k : cap;
    if (coincident) raise_error(st, -7 /*PM_E_COINCIDENT*/, (long long)B.gid[st->cur_id][i]);
  }
  // warp reductions of the row statistics
  int kmax = k;
  long long ksum = k;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
  }
  if ((threadIdx.x & 31) == 0 && ksum > 0) {
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
}

// CSR export of the list for the getters: col_gid[row_ptr[i] + k] = gid(nbr).
__global__ void __launch_bounds__(256) k_verlet_export(Bufs B, int n, int cap,
                                                      const int64_t *__restrict__ row_ptr,
                                                      int64_t *__restrict__ col_gid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t *gid = B.gid[B.st->cur_id];
  const int *nb = B.nbr + nbr_base4(i, cap) * 4;
  const int c = B.cnt[i];
  for (int k = 0; k < c; ++k) col_gid[row_ptr[i] + k] = gid[nb[(k >> 2) * 128 + (k & 3)]];
}

}  // namespace

void launch_verlet(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  k_reset_build_stats<<<1, 1, 0, s>>>(B.st);
  if (n > 0) k_verlet<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, B, (int)n);
}

void launch_verlet_export(const Bufs &B, int64_t n, int cap, const int64_t *row_ptr,
                          int64_t *col_gid, cudaStream_t s) {
  if (n > 0)
    k_verlet_export<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(B, (int)n, cap, row_ptr, col_gid);
}

}  // namespace pm
