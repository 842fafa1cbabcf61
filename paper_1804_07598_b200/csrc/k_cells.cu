// k_cells.cu -- cell-list construction.
//
// PAPER.md:48 (§2) "Cell Lists [45]"; PAPER.md:276/308 getCellListSym /
// updateCellListSym; PAPER.md:128 (§3.6) cache-friendly re-ordering of the
// particles.  B200 design: one fused pass computes the
// wrap, the cell id and an atomic slot claim (warp-aggregated with
// __match_any_sync), a 3-phase scan produces the cell starts, the slots are
// scattered and each cell's segment is sorted by storage index (warp bitonic
// for <= 32 entries), which makes the counting sort stable and the result
// bit-exact; a gather then reorders every particle array into cell order.
#include "pm_internal.cuh"

namespace pm {

namespace {

__global__ void k_zero_i32(int32_t *__restrict__ p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) p[i] = 0;
}

// a1 + a2: wrap (R1), cell id (R3), slot claim.
__global__ void __launch_bounds__(256) k_cell_ids(Params P, Bufs B, int64_t n) {
  State *st = B.st;
  const int cur = st->cur_pv;
  float4 *__restrict__ pos = B.pos[cur];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {  // k_segsort (later on the stream) records coincidences / big cells
    st->coinc_gid = -1;
    st->n_big = 0;
  }
  int c = -1;
  if (i < n) {
    float4 p = pos[i];
    float x[3] = {p.x, p.y, p.z};
    bool moved = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (P.box.per[d]) {
        float w = wrap1(x[d], P.box.lo[d], P.box.hi[d], P.box.L[d]);
        moved |= (w != x[d]);
        x[d] = w;
      } else if (!(x[d] >= P.box.lo[d] && x[d] < P.box.hi[d])) {
        raise_error(st, -6 /*PM_E_DOMAIN*/, (long long)B.gid[st->cur_id][i]);
      }
    }
    if (moved) pos[i] = make_float4(x[0], x[1], x[2], p.w);
    int cx = local_coord(P.box, P.grid, 0, x[0]);
    int cy = local_coord(P.box, P.grid, 1, x[1]);
    int cz = local_coord(P.box, P.grid, 2, x[2]);
    c = cx + P.grid.n[0] * (cy + P.grid.n[1] * cz);
    B.cell_of[i] = c;
  }
  // warp-aggregated slot claim: lanes with the same cell share one atomic
  const unsigned full = 0xffffffffu;
  const unsigned grp = __match_any_sync(full, c);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(grp) - 1;
  int base = 0;
  if (c >= 0 && lane == leader) base = atomicAdd(&B.count[c], __popc(grp));
  base = __shfl_sync(full, base, leader);
  if (c >= 0) B.slot[i] = base + __popc(grp & ((1u << lane) - 1u));
}

constexpr int kScanThreads = 512;
constexpr int kScanPer = 4;
constexpr int kScanTile = kScanThreads * kScanPer;

template <int NT>
__device__ int block_exclusive_scan(int v, int *total) {
  __shared__ int warp_sums[NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = (lane < NT / 32) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) warp_sums[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  int warp_excl = (wid == 0) ? 0 : warp_sums[wid - 1];
  *total = warp_sums[NT / 32 - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// a3 phase 1: per-tile exclusive scan of the counts, tile totals.
// The counts are consumed here and reset to zero for the next build (so no
// separate zeroing pass runs before k_cell_ids).
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(int32_t *__restrict__ count,
                                                             int32_t *__restrict__ start,
                                                             int32_t *__restrict__ tile_sum,
                                                             int ncell) {
  const int base = blockIdx.x * kScanTile + threadIdx.x * kScanPer;
  int v[kScanPer];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    v[k] = (base + k < ncell) ? count[base + k] : 0;
    s += v[k];
  }
#pragma unroll
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < ncell) count[base + k] = 0;
  int total;
  int ex = block_exclusive_scan<kScanThreads>(s, &total);
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    if (base + k < ncell) start[base + k] = ex;
    ex += v[k];
  }
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// a3 phase 2: exclusive scan of the tile totals (one block, chunked).
__global__ void __launch_bounds__(1024) k_scan_sums(int32_t *__restrict__ tile_sum, int ntiles,
                                                    int32_t *__restrict__ start, int ncell) {
  int carry = 0;
  for (int b = 0; b < ntiles; b += 1024) {
    int i = b + threadIdx.x;
    int v = (i < ntiles) ? tile_sum[i] : 0;
    int total;
    int ex = block_exclusive_scan<1024>(v, &total);
    if (i < ntiles) tile_sum[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) start[ncell] = carry;
}

// a3 phase 3: add tile offsets.
__global__ void __launch_bounds__(kScanThreads) k_scan_add(int32_t *__restrict__ start,
                                                           const int32_t *__restrict__ tile_sum,
                                                           int ncell) {
  const int base = blockIdx.x * kScanTile + threadIdx.x * kScanPer;
  const int off = tile_sum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < ncell) start[base + k] += off;
}

// a4: scatter storage indices to their claimed slots (unordered within a cell).
__global__ void __launch_bounds__(256) k_scatter(Bufs B, int32_t *__restrict__ tmp, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  tmp[B.start[B.cell_of[i]] + B.slot[i]] = (int32_t)i;
}

// a4: stable order inside each cell = ascending storage index.  One warp per
// cell: bitonic sort in registers for <= 32 entries, rank-by-count otherwise.
// Coincident particles (identical positions, PM_E_COINCIDENT: LJ undefined)
// always share a cell, so they are detected here, by comparing the members
// of each cell pairwise (the Verlet builder's strict 0 < d2 test would
// otherwise drop such a pair silently).
__device__ __forceinline__ bool same_pos(const float4 &a, const float4 &b) {
  return a.x == b.x && a.y == b.y && a.z == b.z;
}

// One cell of m >= 2 members, s = its first slot, by the whole warp.
__device__ __forceinline__ void warp_cell(const Bufs &B, const int32_t *__restrict__ tmp,
                                          int cell, int s, int m, int lane) {
  State *st = B.st;
  const float4 *__restrict__ pos = B.pos[st->cur_pv];
  const unsigned full = 0xffffffffu;
  if (m <= 32) {
    int v = (lane < m) ? tmp[s + lane] : 0x7fffffff;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        int o = __shfl_xor_sync(full, v, j);
        bool up = (lane & k) == 0;
        bool lower = (lane & j) == 0;
        v = (lower == up) ? min(v, o) : max(v, o);
      }
    }
    if (lane < m) B.perm[s + lane] = v;
    // coincidence: lanes with equal position bits have equal hashes; one
    // match_any finds candidate groups, an exact compare confirms (rare)
    const float nan = __int_as_float(0x7fc00000);  // idle lanes never compare equal
    const float4 p = (lane < m) ? pos[v] : make_float4(nan, nan, nan, 0.f);
    const unsigned hx = __float_as_uint(p.x), hy = __float_as_uint(p.y), hz = __float_as_uint(p.z);
    const unsigned h = (lane < m) ? (hx * 0x9E3779B1u) ^ (hy * 0x85EBCA77u) ^ (hz * 0xC2B2AE3Du)
                                  : 0xFFFFFFFFu - (unsigned)lane;  // distinct for idle lanes
    const unsigned grp = __match_any_sync(full, h) & ~(1u << lane);
    bool dup = false;
    if (__any_sync(full, grp != 0u)) {
      for (int o = 1; o < 32; ++o) {  // exact check, only when hashes collide
        const int src = (lane + o) & 31;
        const float4 q = make_float4(__shfl_sync(full, p.x, src), __shfl_sync(full, p.y, src),
                                     __shfl_sync(full, p.z, src), 0.f);
        dup |= ((grp >> src) & 1u) && same_pos(p, q);
      }
    }
    if (dup) st->coinc_gid = (long long)B.gid[st->cur_id][v];
    return;
  }
  // more than 32 members: defer to the block-level sort (k_segsort_big)
  if (lane == 0) B.big_cells[atomicAdd(&st->n_big, 1)] = cell;
}


__global__ void __launch_bounds__(256) k_segsort(Bufs B, const int32_t *__restrict__ tmp,
                                                 int ncell) {
  const int cell = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (cell >= ncell) return;  // whole warp exits together
  const int s = B.start[cell], e = B.start[cell + 1], m = e - s;
  if (m == 0) return;
  if (m == 1) {
    if (lane == 0) B.perm[s] = tmp[s];
    return;
  }
  warp_cell(B, tmp, cell, s, m, lane);
}

// Sparse grids (fewer than ~4 particles per cell, e.g. a granular bed in a
// large domain): one lane per cell.  Cells of <= 8 members are sorted in
// registers by an optimal 19-comparator network and checked pairwise for
// coincident positions by their own lane; wider cells are taken by the whole
// warp, one after another (warp_cell).  Same result as k_segsort.
constexpr int kThinMax = 8;

__device__ __forceinline__ void cswap(int &a, int &b) {
  const int lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

__global__ void __launch_bounds__(256) k_segsort_thin(Bufs B, const int32_t *__restrict__ tmp,
                                                      int ncell) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int s = 0, m = 0;
  if (cell < ncell) {
    s = B.start[cell];
    m = B.start[cell + 1] - s;
  }
  if (m == 1) B.perm[s] = tmp[s];
  if (m >= 2 && m <= kThinMax) {
    int v[kThinMax];
#pragma unroll
    for (int k = 0; k < kThinMax; ++k) v[k] = (k < m) ? tmp[s + k] : 0x7fffffff;
    cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[4], v[6]); cswap(v[5], v[7]);
    cswap(v[0], v[4]); cswap(v[1], v[5]); cswap(v[2], v[6]); cswap(v[3], v[7]);
    cswap(v[0], v[1]); cswap(v[2], v[3]); cswap(v[4], v[5]); cswap(v[6], v[7]);
    cswap(v[2], v[4]); cswap(v[3], v[5]);
    cswap(v[1], v[4]); cswap(v[3], v[6]);
    cswap(v[1], v[2]); cswap(v[3], v[4]); cswap(v[5], v[6]);
    State *st = B.st;
    const float4 *__restrict__ pos = B.pos[st->cur_pv];
    float4 p[kThinMax];
#pragma unroll
    for (int k = 0; k < kThinMax; ++k) {
      if (k < m) {
        B.perm[s + k] = v[k];
        p[k] = pos[v[k]];
      }
    }
    int dup = -1;
#pragma unroll
    for (int k = 1; k < kThinMax; ++k)
#pragma unroll
      for (int l = 0; l < k; ++l)
        if (k < m && same_pos(p[k], p[l])) dup = v[k];
    if (dup >= 0) st->coinc_gid = (long long)B.gid[st->cur_id][dup];
  }
  unsigned wide = __ballot_sync(0xffffffffu, m > kThinMax);
  while (wide) {
    const int l = __ffs(wide) - 1;
    wide &= wide - 1;
    const int ws = __shfl_sync(0xffffffffu, s, l), wm = __shfl_sync(0xffffffffu, m, l);
    warp_cell(B, tmp, cell - lane + l, ws, wm, lane);
  }
}

// Cells with more than 32 members (clustered inputs, up to ~3000): one block
// per cell, bitonic sort of the storage indices in shared memory (<= 8192
// members; beyond, rank by counting).  Coincident particles in such cells are
// found by the force sweep's non-finite path, which scans the row for a
// partner at distance 0 and raises PM_E_COINCIDENT (k_lj.cu raise_bad_force).
constexpr int kBigSort = 8192;

__global__ void __launch_bounds__(512) k_segsort_big(Bufs B, const int32_t *__restrict__ tmp) {
  __shared__ int key[kBigSort];
  State *st = B.st;
  const int nbig = st->n_big;
  for (int b = blockIdx.x; b < nbig; b += gridDim.x) {
    const int cell = B.big_cells[b];
    const int s = B.start[cell], m = B.start[cell + 1] - s;
    if (m <= kBigSort) {
      int n2 = 64;
      while (n2 < m) n2 <<= 1;
      for (int t = threadIdx.x; t < n2; t += blockDim.x) key[t] = (t < m) ? tmp[s + t] : 0x7fffffff;
      __syncthreads();
      for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int t = threadIdx.x; t < n2; t += blockDim.x) {
            const int u = t ^ j;
            if (u > t) {
              const int a = key[t], c = key[u];
              const bool up = (t & k) == 0;
              if ((a > c) == up) {
                key[t] = c;
                key[u] = a;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int t = threadIdx.x; t < m; t += blockDim.x) B.perm[s + t] = key[t];
      __syncthreads();
    } else {
      for (int p = threadIdx.x; p < m; p += blockDim.x) {
        const int v = tmp[s + p];
        int r = 0;
        for (int q = 0; q < m; ++q) r += (tmp[s + q] < v);
        B.perm[s + r] = v;
      }
    }
  }
}

// a4: gather every particle array into cell order (alternate buffers).
__global__ void __launch_bounds__(256) k_reorder(Bufs B, int64_t n, int sph_state,
                                                 int dem_state) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  State *st = B.st;
  const int cp = st->cur_pv, ci = st->cur_id;
  const int j = B.perm[k];
  B.invperm[j] = (int32_t)k;
  const float4 p = B.pos[cp][j];
  B.pos[cp ^ 1][k] = p;
  B.xref[k] = p;
  B.vel[cp ^ 1][k] = B.vel[cp][j];
  B.gid[ci ^ 1][k] = B.gid[ci][j];
  B.kind[ci ^ 1][k] = B.kind[ci][j];
  if (sph_state) {  // SPH time stepping state travels with the particles
    B.rhoP[ci ^ 1][k] = B.rhoP[ci][j];
    B.vold[ci ^ 1][k] = B.vold[ci][j];
  }
  if (dem_state) B.omega[cp ^ 1][k] = B.omega[cp][j];  // double-buffered per step
}

__global__ void k_flip(Bufs B, int flip_pv, int flip_id, int count_rebuild) {
  State *st = B.st;
  if (flip_pv) st->cur_pv ^= 1;
  if (flip_id) st->cur_id ^= 1;
  if (count_rebuild) {
    st->n_rebuilds += 1;
    st->need_rebuild = 0;
  }
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_zero_i32(int32_t *p, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  unsigned g = blocks_for(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  k_zero_i32<<<g, 256, 0, s>>>(p, n);
}

void launch_cell_ids(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  // B.count is all zero here: allocated zeroed, and every scan resets it
  if (n > 0) k_cell_ids<<<blocks_for(n, 256), 256, 0, s>>>(P, B, n);
}

void launch_scan(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  (void)n;
  const int ncell = P.grid.ncell;
  const int ntiles = (ncell + kScanTile - 1) / kScanTile;
  k_scan_tiles<<<ntiles, kScanThreads, 0, s>>>(B.count, B.start, B.scan_tmp, ncell);
  k_scan_sums<<<1, 1024, 0, s>>>(B.scan_tmp, ntiles, B.start, ncell);
  k_scan_add<<<ntiles, kScanThreads, 0, s>>>(B.start, B.scan_tmp, ncell);
}

// Generic exclusive scan of n ints (count is zeroed, start[n] = total);
// tmp needs scan_tiles(n) ints.
int scan_tiles(int n) { return (n + kScanTile - 1) / kScanTile; }

void launch_exclusive_scan(int32_t *count, int32_t *start, int32_t *tmp, int n, cudaStream_t s) {
  const int ntiles = scan_tiles(n);
  if (ntiles == 0) return;
  k_scan_tiles<<<ntiles, kScanThreads, 0, s>>>(count, start, tmp, n);
  k_scan_sums<<<1, 1024, 0, s>>>(tmp, ntiles, start, n);
  k_scan_add<<<ntiles, kScanThreads, 0, s>>>(start, tmp, n);
}

void launch_sort_reorder(const Params &P, const Bufs &B, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  int32_t *tmp = B.sorttmp;
  k_scatter<<<blocks_for(n, 256), 256, 0, s>>>(B, tmp, n);
  if (n < 4 * (int64_t)P.grid.ncell)  // sparse grid: lane per cell
    k_segsort_thin<<<blocks_for(P.grid.ncell, 256), 256, 0, s>>>(B, tmp, P.grid.ncell);
  else
    k_segsort<<<blocks_for((int64_t)P.grid.ncell * 32, 256), 256, 0, s>>>(B, tmp, P.grid.ncell);
  k_segsort_big<<<148, 512, 0, s>>>(B, tmp);
  k_reorder<<<blocks_for(n, 256), 256, 0, s>>>(B, n, P.sph_state, P.dem_state);
}

void launch_flip(const Bufs &B, int flip_pv, int flip_id, int count_rebuild, cudaStream_t s) {
  k_flip<<<1, 1, 0, s>>>(B, flip_pv, flip_id, count_rebuild);
}

}  // namespace pm
