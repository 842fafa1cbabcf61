// Microbenchmark: does the order of the entries inside each Verlet row change
// the force sweep's time?  (the sweep is bound by L1 data-pipe
// wavefronts of its scattered float4 gathers, ~13 per gather.)
//
// Host: a cfg2-like system (1,048,576 particles at rho = 0.8, periodic box
// 128 x 128 x 64 lattice constants), cells of side >= r_v, particles in cell
// order, full Verlet rows (r_v = 2.8) in the library's SELL-32x4 layout
// (4 entries of a lane contiguous, 32 lanes of a warp side by side).  Layouts:
//   plain   each row in candidate (cell, storage) order -- the shipped build
//   greedy  per warp and slot, the line (8 consecutive particles) needed by
//           most not-yet-served lanes is served first (set cover per slot),
//           so the 32 gathers of one instruction touch few 128-byte lines
// Device: the sweep's gather loop (4 gathers per index group) with the LJ
// pair, forces written out; CUDA events over 50 launches per layout.
// Kernel variants (the `launch` switch; DESIGN §11 lists the results):
//   k_sweep<G>      G index groups per iteration (memory-level parallelism)
//   k_sweep_pf<M>   indices one group ahead; M = 1: every gather an L1 hit,
//                   M = 2: no index stream either (the compute floor)
//   k_sweep16       16-bit codes (piece table per warp), 8 per 16-byte load
//   k_sweep_cpa/cpw index stream staged through shared memory by cp.async
//   k_sweep_bal     a warp's rows dealt out evenly (no padding), owner lanes
//   k_sweep1k       1024-thread CTAs (with brick-ordered cells: argv 2-4)
//
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//          -o gather_order tools/micro/gather_order.cu
// Run:   ./gather_order [lattice|poisson] [bx by bz] [nz]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                           \
    }                                                                         \
  } while (0)

struct Sell {
  std::vector<int> idx;      // SELL-32x4 entries
  std::vector<int64_t> base; // per warp: offset of its first group
  std::vector<int> cnt;      // per particle
};

// G index groups (4 entries each) per iteration: all 4*G gathers issued
// before any pair is evaluated (memory-level parallelism per warp)
template <int G>
__global__ void __launch_bounds__(256) k_sweep(const float4 *__restrict__ pos,
                                               const int *__restrict__ nbr,
                                               const long long *__restrict__ wbase,
                                               const int *__restrict__ cnt, float4 *out,
                                               int n, float rc2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 xi = pos[i];
  const int c = cnt[i];
  const int *nb = nbr + wbase[i >> 5] + (threadIdx.x & 31) * 4;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  for (int g = 0; 4 * g < c; g += G) {
    int jj[4 * G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      int4 j = make_int4(i, i, i, i);
      if (4 * (g + q) < c) j = __ldcs(reinterpret_cast<const int4 *>(nb + (int64_t)(g + q) * 128));
      jj[4 * q] = j.x, jj[4 * q + 1] = j.y, jj[4 * q + 2] = j.z, jj[4 * q + 3] = j.w;
    }
    float4 xj[4 * G];
#pragma unroll
    for (int s = 0; s < 4 * G; ++s) xj[s] = __ldg(pos + (4 * g + s < c ? jj[s] : i));
#pragma unroll
    for (int s = 0; s < 4 * G; ++s) {
      const float dx = xj[s].x - xi.x, dy = xj[s].y - xi.y, dz = xj[s].z - xi.z;
      const float r2 = dx * dx + dy * dy + dz * dz;
      if (4 * g + s < c && r2 < rc2 && r2 > 0.f) {
        const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
        const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
        fx -= f * dx;
        fy -= f * dy;
        fz -= f * dz;
      }
    }
  }
  out[i] = make_float4(fx, fy, fz, 0.f);
}

// k_sweep<1> with the next group's indices loaded one iteration ahead
// MODE 0: as the sweep; 1: the index stream is read but every gather is of
// the row's own line (i ^ 1, an L1 hit); 2: no index loads (j = i ^ 1)
template <int MODE>
__global__ void __launch_bounds__(256) k_sweep_pf(const float4 *__restrict__ pos,
                                                  const int *__restrict__ nbr,
                                                  const long long *__restrict__ wbase,
                                                  const int *__restrict__ cnt, float4 *out,
                                                  int n, float rc2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 xi = pos[i];
  const int c = cnt[i];
  const int *nb = nbr + wbase[i >> 5] + (threadIdx.x & 31) * 4;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  int4 jn = (MODE < 2 && c > 0) ? __ldcs(reinterpret_cast<const int4 *>(nb)) : make_int4(i, i, i, i);
  int acc = 0;
  for (int g = 0; 4 * g < c; ++g) {
    const int4 j = jn;
    if (MODE < 2 && 4 * (g + 1) < c) jn = __ldcs(reinterpret_cast<const int4 *>(nb + (int64_t)(g + 1) * 128));
    int jj[4] = {j.x, j.y, j.z, j.w};
    if (MODE >= 1) {
      acc += jj[0] ^ jj[1] ^ jj[2] ^ jj[3];
#pragma unroll
      for (int s = 0; s < 4; ++s) jj[s] = i ^ 1;
    }
    float4 xj[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) xj[s] = __ldg(pos + (4 * g + s < c ? jj[s] : i));
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const float dx = xj[s].x - xi.x, dy = xj[s].y - xi.y, dz = xj[s].z - xi.z;
      const float r2 = dx * dx + dy * dy + dz * dz;
      if (4 * g + s < c && r2 < rc2 && r2 > 0.f) {
        const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
        const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
        fx -= f * dx;
        fy -= f * dy;
        fz -= f * dz;
      }
    }
  }
  out[i] = make_float4(fx, fy, fz, (float)acc);
}

// k_sweep<1> with the index stream staged through shared memory by cp.async
// (4-byte copies of the lane's own entries, RING groups ahead): the index
// loads' DRAM latency leaves the dependency chain of the gathers
template <int RING>
__global__ void __launch_bounds__(256) k_sweep_cpa(const float4 *__restrict__ pos,
                                                   const int *__restrict__ nbr,
                                                   const long long *__restrict__ wbase,
                                                   const int *__restrict__ cnt, float4 *out,
                                                   int n, float rc2) {
  __shared__ int ring[8][RING * 4][32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4 xi = pos[i];
  const int c = cnt[i];
  const int ng = (c + 3) >> 2;
  const int *nb = nbr + wbase[i >> 5] + lane * 4;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  auto issue = [&](int g) {
    if (g < ng) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&ring[w][(g % RING) * 4 + s][lane]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(nb + (int64_t)g * 128 + s));
      }
    }
    asm volatile("cp.async.commit_group;");
  };
#pragma unroll
  for (int g = 0; g < RING - 1; ++g) issue(g);
  for (int g = 0; g < ng; ++g) {
    issue(g + RING - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(RING - 1));
    int jj[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) jj[s] = ring[w][(g % RING) * 4 + s][lane];
    float4 xj[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) xj[s] = __ldg(pos + (4 * g + s < c ? jj[s] : i));
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const float dx = xj[s].x - xi.x, dy = xj[s].y - xi.y, dz = xj[s].z - xi.z;
      const float r2 = dx * dx + dy * dy + dz * dz;
      if (4 * g + s < c && r2 < rc2 && r2 > 0.f) {
        const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
        const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
        fx -= f * dx;
        fy -= f * dy;
        fz -= f * dz;
      }
    }
  }
  asm volatile("cp.async.wait_all;");
  out[i] = make_float4(fx, fy, fz, 0.f);
}

// the same with the warp's 512-byte group chunks copied cooperatively
// (16 bytes per lane, cp.async.cg: L2 only), a warp-uniform loop over the
// slice's longest row, lanes past their row masked
template <int RING>
__global__ void __launch_bounds__(256) k_sweep_cpw(const float4 *__restrict__ pos,
                                                   const int *__restrict__ nbr,
                                                   const long long *__restrict__ wbase,
                                                   const int *__restrict__ cnt, float4 *out,
                                                   int n, float rc2) {
  __shared__ __align__(16) int ring[8][RING][128];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4 xi = pos[i];
  const int c = cnt[i];
  const int ngm = (__reduce_max_sync(0xffffffffu, c) + 3) >> 2;
  const int *chunk = nbr + wbase[i >> 5];
  float fx = 0.f, fy = 0.f, fz = 0.f;
  auto issue = [&](int g) {
    if (g < ngm) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&ring[w][g % RING][lane * 4]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(chunk + (int64_t)g * 128 + lane * 4));
    }
    asm volatile("cp.async.commit_group;");
  };
#pragma unroll
  for (int g = 0; g < RING - 1; ++g) issue(g);
  for (int g = 0; g < ngm; ++g) {
    issue(g + RING - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(RING - 1));
    __syncwarp();
    int jj[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) jj[s] = ring[w][g % RING][s * 32 + lane];
    __syncwarp();
    float4 xj[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) xj[s] = __ldg(pos + (4 * g + s < c ? jj[s] : i));
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const float dx = xj[s].x - xi.x, dy = xj[s].y - xi.y, dz = xj[s].z - xi.z;
      const float r2 = dx * dx + dy * dy + dz * dz;
      if (4 * g + s < c && r2 < rc2 && r2 > 0.f) {
        const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
        const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
        fx -= f * dx;
        fy -= f * dy;
        fz -= f * dz;
      }
    }
  }
  asm volatile("cp.async.wait_all;");
  out[i] = make_float4(fx, fy, fz, 0.f);
}

// Balanced rows: a warp's rows concatenated and dealt out evenly (every lane
// ceil(T/32) or fewer entries, no SELL padding to the longest row); each entry
// carries its owner lane (bits 27-31); the owner's position comes from shared
// memory and the partial forces return to the owners by shared atomics.
// SELL-32 column layout of the dealt entries, 4 per group, one group ahead.
__global__ void __launch_bounds__(256) k_sweep_bal(const float4 *__restrict__ pos,
                                                   const int *__restrict__ nbr,
                                                   const long long *__restrict__ wbase,
                                                   const int *__restrict__ qn, float4 *out,
                                                   int n, float rc2) {
  __shared__ float4 xs[8][32];
  __shared__ float fs[8][32][4];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  xs[w][lane] = pos[i];
  fs[w][lane][0] = fs[w][lane][1] = fs[w][lane][2] = 0.f;
  __syncwarp();
  const int c = qn[i];  // entries dealt to this lane
  const int *nb = nbr + wbase[i >> 5] + lane;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  int cur = -1;
  float4 xo = make_float4(0.f, 0.f, 0.f, 0.f);
  int jn = c > 0 ? __ldcs(nb) : 0;
  for (int t = 0; t < c; ++t) {
    const int e = jn;
    if (t + 1 < c) jn = __ldcs(nb + (int64_t)(t + 1) * 32);
    const int o = (unsigned)e >> 27, j = e & ((1 << 27) - 1);
    if (o != cur) {
      if (cur >= 0) {
        atomicAdd(&fs[w][cur][0], fx);
        atomicAdd(&fs[w][cur][1], fy);
        atomicAdd(&fs[w][cur][2], fz);
      }
      fx = fy = fz = 0.f;
      cur = o;
      xo = xs[w][o];
    }
    const float4 xj = __ldg(pos + j);
    const float dx = xj.x - xo.x, dy = xj.y - xo.y, dz = xj.z - xo.z;
    const float r2 = dx * dx + dy * dy + dz * dz;
    if (r2 < rc2 && r2 > 0.f) {
      const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
      const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
      fx -= f * dx;
      fy -= f * dy;
      fz -= f * dz;
    }
  }
  if (cur >= 0) {
    atomicAdd(&fs[w][cur][0], fx);
    atomicAdd(&fs[w][cur][1], fy);
    atomicAdd(&fs[w][cur][2], fz);
  }
  __syncwarp();
  out[i] = make_float4(fs[w][lane][0], fs[w][lane][1], fs[w][lane][2], 0.f);
}

// k_sweep<1> in CTAs of 1024 threads (4 x 256 consecutive rows share an SM)
__global__ void __launch_bounds__(1024) k_sweep1k(const float4 *__restrict__ pos,
                                                  const int *__restrict__ nbr,
                                                  const long long *__restrict__ wbase,
                                                  const int *__restrict__ cnt, float4 *out,
                                                  int n, float rc2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 xi = pos[i];
  const int c = cnt[i];
  const int *nb = nbr + wbase[i >> 5] + (threadIdx.x & 31) * 4;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  for (int g = 0; 4 * g < c; ++g) {
    const int4 j = __ldcs(reinterpret_cast<const int4 *>(nb + (int64_t)g * 128));
    const int jj[4] = {j.x, j.y, j.z, j.w};
    float4 xj[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) xj[s] = __ldg(pos + (4 * g + s < c ? jj[s] : i));
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const float dx = xj[s].x - xi.x, dy = xj[s].y - xi.y, dz = xj[s].z - xi.z;
      const float r2 = dx * dx + dy * dy + dz * dz;
      if (4 * g + s < c && r2 < rc2 && r2 > 0.f) {
        const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
        const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
        fx -= f * dx;
        fy -= f * dy;
        fz -= f * dz;
      }
    }
  }
  out[i] = make_float4(fx, fy, fz, 0.f);
}

// 16-bit codes: (piece << 10) | (j & 1023), piece = index into the warp's
// table of distinct j >> 10 (<= 32, one per lane); 8 codes per lane per
// 16-byte load (SELL-32x8)
__global__ void __launch_bounds__(256) k_sweep16(const float4 *__restrict__ pos,
                                                 const uint16_t *__restrict__ nbr,
                                                 const long long *__restrict__ wbase,
                                                 const int *__restrict__ ptab,
                                                 const int *__restrict__ cnt, float4 *out,
                                                 int n, float rc2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const float4 xi = pos[i];
  const int c = cnt[i];
  const int cmax = __reduce_max_sync(0xffffffffu, c);
  const int mypiece = ptab[(i >> 5) * 32 + lane] << 10;
  const uint16_t *nb = nbr + wbase[i >> 5] + lane * 8;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  for (int g = 0; 8 * g < cmax; ++g) {
    uint4 q = make_uint4(0, 0, 0, 0);
    if (8 * g < c) q = __ldcs(reinterpret_cast<const uint4 *>(nb + (int64_t)g * 256));
    const unsigned w4[4] = {q.x, q.y, q.z, q.w};
    int jj[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const unsigned code = (w4[s >> 1] >> (16 * (s & 1))) & 0xffffu;
      jj[s] = __shfl_sync(0xffffffffu, mypiece, code >> 10) | (code & 1023);
    }
    float4 xj[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) xj[s] = __ldg(pos + (8 * g + s < c ? jj[s] : i));
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const float dx = xj[s].x - xi.x, dy = xj[s].y - xi.y, dz = xj[s].z - xi.z;
      const float r2 = dx * dx + dy * dy + dz * dz;
      if (8 * g + s < c && r2 < rc2 && r2 > 0.f) {
        const float ir2 = 1.f / r2, ir6 = ir2 * ir2 * ir2;
        const float f = 24.f * ir2 * ir6 * (2.f * ir6 - 1.f);
        fx -= f * dx;
        fy -= f * dy;
        fz -= f * dz;
      }
    }
  }
  out[i] = make_float4(fx, fy, fz, 0.f);
}

struct Sell16 {
  std::vector<uint16_t> idx;
  std::vector<int64_t> base;
  std::vector<int> ptab;
};

static int g_nz = 64;
static void make_system(bool lattice, std::vector<float4> &pos, float L[3]) {
  const double a = std::pow(0.8, -1.0 / 3.0);
  const int nx = 128, ny = 128, nz = g_nz;
  L[0] = nx * a, L[1] = ny * a, L[2] = nz * a;
  std::mt19937_64 g(11);
  std::normal_distribution<double> nd(0.0, 0.15);
  std::uniform_real_distribution<double> ud(0.0, 1.0);
  pos.resize((size_t)nx * ny * nz);
  size_t k = 0;
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x, ++k) {
        double p[3];
        if (lattice) {
          p[0] = (x + 0.5 + nd(g)) * a, p[1] = (y + 0.5 + nd(g)) * a, p[2] = (z + 0.5 + nd(g)) * a;
        } else {
          p[0] = ud(g) * L[0], p[1] = ud(g) * L[1], p[2] = ud(g) * L[2];
        }
        for (int d = 0; d < 3; ++d) p[d] = std::fmod(p[d] + L[d], (double)L[d]);
        pos[k] = make_float4((float)p[0], (float)p[1], (float)p[2], 0.f);
      }
}

int main(int argc, char **argv) {
  const bool lattice = argc > 1 && std::strcmp(argv[1], "lattice") == 0;
  if (argc > 5) g_nz = std::atoi(argv[5]);
  const float rv = 2.8f, rc = 2.5f;
  std::vector<float4> p0;
  float L[3];
  make_system(lattice, p0, L);
  const int n = (int)p0.size();
  int nc[3];
  float cs[3];
  for (int d = 0; d < 3; ++d) nc[d] = (int)std::floor(L[d] / rv), cs[d] = L[d] / nc[d];
  const int ncell = nc[0] * nc[1] * nc[2];
  std::vector<int> cid(n);
  for (int i = 0; i < n; ++i) {
    const float v[3] = {p0[i].x, p0[i].y, p0[i].z};
    int c3[3];
    for (int d = 0; d < 3; ++d) c3[d] = std::min((int)(v[d] / cs[d]), nc[d] - 1);
    cid[i] = c3[0] + nc[0] * (c3[1] + nc[1] * c3[2]);
  }
  // storage key: cells in bricks of bx x by x bz (x fastest inside a brick,
  // bricks in linear order); 1 1 1 = the library's linear cell order
  const int bx = argc > 2 ? std::atoi(argv[2]) : 1, by = argc > 3 ? std::atoi(argv[3]) : 1,
            bz = argc > 4 ? std::atoi(argv[4]) : 1;
  const int nbx = (nc[0] + bx - 1) / bx, nby = (nc[1] + by - 1) / by;
  std::vector<int64_t> skey(n);
  for (int i = 0; i < n; ++i) {
    const int c = cid[i];
    const int x = c % nc[0], y = (c / nc[0]) % nc[1], z = c / (nc[0] * nc[1]);
    const int64_t brick = x / bx + nbx * ((int64_t)(y / by) + nby * (z / bz));
    skey[i] = brick * (bx * by * bz) + (x % bx) + bx * ((y % by) + by * (z % bz));
  }
  std::printf("bricks %d x %d x %d\n", bx, by, bz);
  // cell order; inside a cell a seeded shuffle (a liquid's order after rebuilds)
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::mt19937 gs(5);
  std::shuffle(ord.begin(), ord.end(), gs);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return skey[a] < skey[b]; });
  std::vector<float4> pos(n);
  std::vector<int> c1(n);
  for (int i = 0; i < n; ++i) pos[i] = p0[ord[i]], c1[i] = cid[ord[i]];
  std::vector<int> cbeg(ncell, 0), cend(ncell, 0);
  for (int i = n - 1; i >= 0; --i) cbeg[c1[i]] = i;
  for (int i = 0; i < n; ++i) cend[c1[i]] = i + 1;
  // rows in candidate order: stencil cells (z, y, x ascending), storage order
  std::vector<std::vector<int>> rows(n);
  const float rv2 = rv * rv;
  for (int i = 0; i < n; ++i) {
    const int c = c1[i];
    const int cx = c % nc[0], cy = (c / nc[0]) % nc[1], cz = c / (nc[0] * nc[1]);
    std::vector<int> cells;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int x = (cx + dx + nc[0]) % nc[0], y = (cy + dy + nc[1]) % nc[1],
                    z = (cz + dz + nc[2]) % nc[2];
          cells.push_back(x + nc[0] * (y + nc[1] * z));
        }
    std::sort(cells.begin(), cells.end(), [&](int a, int b) { return cbeg[a] < cbeg[b]; });
    for (int cc : cells)
      for (int j = cbeg[cc]; j < cend[cc]; ++j) {
        if (j == i) continue;
        float d[3] = {pos[j].x - pos[i].x, pos[j].y - pos[i].y, pos[j].z - pos[i].z};
        for (int q = 0; q < 3; ++q) d[q] -= L[q] * std::rint(d[q] / L[q]);
        if (d[0] * d[0] + d[1] * d[1] + d[2] * d[2] < rv2) rows[i].push_back(j);
      }
  }
  const int nw = (n + 31) / 32;
  auto to_sell = [&](const std::vector<std::vector<int>> &r, Sell &S) {
    S.base.assign(nw + 1, 0);
    S.cnt.assign(n, 0);
    for (int w = 0; w < nw; ++w) {
      size_t m = 0;
      for (int k = 0; k < 32 && w * 32 + k < n; ++k) m = std::max(m, r[w * 32 + k].size());
      S.base[w + 1] = S.base[w] + (int64_t)((m + 3) / 4) * 128;
    }
    S.idx.assign(S.base[nw], 0);
    for (int i = 0; i < n; ++i) {
      const int w = i >> 5, k = i & 31;
      S.cnt[i] = (int)r[i].size();
      for (size_t t = 0; t < r[i].size(); ++t)
        S.idx[S.base[w] + (t / 4) * 128 + k * 4 + (t % 4)] = r[i][t];
    }
  };
  bool u16_ok = true;
  auto to_sell16 = [&](const std::vector<std::vector<int>> &r, Sell16 &S) {
    S.base.assign(nw + 1, 0);
    S.ptab.assign((size_t)nw * 32, 0);
    int maxp = 0;
    for (int w = 0; w < nw; ++w) {
      size_t m = 0;
      std::vector<int> pc;
      for (int k = 0; k < 32; ++k) {
        m = std::max(m, r[w * 32 + k].size());
        for (int j : r[w * 32 + k]) pc.push_back(j >> 10);
      }
      std::sort(pc.begin(), pc.end());
      pc.erase(std::unique(pc.begin(), pc.end()), pc.end());
      maxp = std::max(maxp, (int)pc.size());
      if (pc.size() > 32) { std::printf("u16: too many pieces, skipped\n"); u16_ok = false; return; }
      for (size_t p = 0; p < pc.size(); ++p) S.ptab[(size_t)w * 32 + p] = pc[p];
      S.base[w + 1] = S.base[w] + (int64_t)((m + 7) / 8) * 256;
    }
    S.idx.assign(S.base[nw], 0);
    for (int i = 0; i < n; ++i) {
      const int w = i >> 5, k = i & 31;
      const int *pt = &S.ptab[(size_t)w * 32];
      for (size_t t = 0; t < r[i].size(); ++t) {
        const int j = r[i][t];
        int p = 0;
        while (pt[p] != (j >> 10)) ++p;
        S.idx[S.base[w] + (t / 8) * 256 + k * 8 + (t % 8)] = (uint16_t)((p << 10) | (j & 1023));
      }
    }
    std::printf("u16 list: %.1f MB, max pieces per warp %d\n", S.idx.size() * 2 / 1e6, maxp);
  };
  // greedy reorder per warp
  std::vector<std::vector<int>> rg(n);
  double lines_plain = 0, lines_greedy = 0, slots = 0;
  for (int w = 0; w < nw; ++w) {
    const int i0 = w * 32, nk = std::min(32, n - i0);
    std::vector<int> lines;
    for (int k = 0; k < nk; ++k)
      for (int j : rows[i0 + k]) lines.push_back(j >> 3);
    std::sort(lines.begin(), lines.end());
    lines.erase(std::unique(lines.begin(), lines.end()), lines.end());
    const int nl = (int)lines.size();
    // per (line, lane): pending entries
    std::vector<std::vector<int>> pend((size_t)nl * 32);
    std::vector<uint32_t> mask(nl, 0);
    std::vector<int> rem(32, 0);
    size_t m = 0;
    for (int k = 0; k < nk; ++k) {
      for (int j : rows[i0 + k]) {
        const int l = (int)(std::lower_bound(lines.begin(), lines.end(), j >> 3) - lines.begin());
        pend[(size_t)l * 32 + k].push_back(j);
        mask[l] |= 1u << k;
      }
      rem[k] = (int)rows[i0 + k].size();
      m = std::max(m, rows[i0 + k].size());
    }
    for (size_t t = 0; t < m; ++t) {
      std::vector<int> lp;
      for (int k = 0; k < nk; ++k)
        if (t < rows[i0 + k].size()) lp.push_back(rows[i0 + k][t] >> 3);
      std::sort(lp.begin(), lp.end());
      lines_plain += std::unique(lp.begin(), lp.end()) - lp.begin();
      uint32_t un = 0;
      for (int k = 0; k < nk; ++k)
        if (rem[k]) un |= 1u << k;
      while (un) {
        int best = -1, bc = 0;
        for (int l = 0; l < nl; ++l) {
          const int c = __builtin_popcount(mask[l] & un);
          if (c > bc) bc = c, best = l;
        }
        uint32_t sv = mask[best] & un;
        lines_greedy += 1;
        while (sv) {
          const int k = __builtin_ctz(sv);
          sv &= sv - 1;
          auto &v = pend[(size_t)best * 32 + k];
          rg[i0 + k].push_back(v.back());
          v.pop_back();
          if (v.empty()) mask[best] &= ~(1u << k);
          rem[k]--;
          un &= ~(1u << k);
        }
      }
      slots += 1;
    }
  }
  std::printf("%s: n %d, mean row %.2f, lines per slot: plain %.2f greedy %.2f\n",
              lattice ? "lattice" : "poisson", n,
              [&] { double s = 0; for (auto &r : rows) s += r.size(); return s / n; }(),
              lines_plain / slots, lines_greedy / slots);
  Sell A, B;
  to_sell(rows, A);
  // balanced layout: per warp, entries dealt evenly (SELL-32 columns, 1 per slot)
  std::vector<int> balq(n, 0);
  std::vector<int64_t> balbase(nw + 1, 0);
  for (int w = 0; w < nw; ++w) {
    int64_t T = 0;
    for (int k = 0; k < 32; ++k) T += rows[w * 32 + k].size();
    const int64_t q = (T + 31) / 32;
    balbase[w + 1] = balbase[w] + q * 32;
  }
  std::vector<int> balidx(balbase[nw], 0);
  double padded_sell = 0, padded_bal = 0;
  for (int w = 0; w < nw; ++w) {
    int64_t T = 0;
    size_t m = 0;
    for (int k = 0; k < 32; ++k) T += rows[w * 32 + k].size(), m = std::max(m, rows[w * 32 + k].size());
    const int64_t q = (T + 31) / 32;
    padded_sell += 32.0 * m;
    padded_bal += 32.0 * q;
    int64_t e = 0;
    for (int k = 0; k < 32; ++k)
      for (int j : rows[w * 32 + k]) {
        const int L = (int)(e / q), t = (int)(e % q);
        balidx[balbase[w] + (int64_t)t * 32 + L] = (k << 27) | j;
        balq[w * 32 + L] = t + 1;
        ++e;
      }
  }
  std::printf("slots per entry: SELL %.3f balanced %.3f\n", padded_sell / (double)A.idx.size() * A.idx.size() / padded_sell * padded_sell / std::max(1.0, [&]{double t=0; for (auto &r : rows) t += r.size(); return t;}()), padded_bal / [&]{double t=0; for (auto &r : rows) t += r.size(); return t;}());
  int *dbal, *dbalq;
  long long *dbalbase;
  CK(cudaMalloc(&dbal, balidx.size() * sizeof(int)));
  CK(cudaMalloc(&dbalq, n * sizeof(int)));
  CK(cudaMalloc(&dbalbase, (nw + 1) * sizeof(long long)));
  CK(cudaMemcpy(dbal, balidx.data(), balidx.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dbalq, balq.data(), n * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dbalbase, balbase.data(), (nw + 1) * sizeof(long long), cudaMemcpyHostToDevice));
  to_sell(rg, B);
  float4 *dpos, *dout[2];
  int *didx[2], *dcnt;
  long long *dbase[2];
  CK(cudaMalloc(&dpos, n * sizeof(float4)));
  CK(cudaMalloc(&dcnt, n * sizeof(int)));
  CK(cudaMemcpy(dpos, pos.data(), n * sizeof(float4), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dcnt, A.cnt.data(), n * sizeof(int), cudaMemcpyHostToDevice));
  Sell *S[2] = {&A, &B};
  for (int v = 0; v < 2; ++v) {
    CK(cudaMalloc(&dout[v], n * sizeof(float4)));
    CK(cudaMalloc(&didx[v], S[v]->idx.size() * sizeof(int)));
    CK(cudaMalloc(&dbase[v], (nw + 1) * sizeof(long long)));
    CK(cudaMemcpy(didx[v], S[v]->idx.data(), S[v]->idx.size() * sizeof(int),
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dbase[v], S[v]->base.data(), (nw + 1) * sizeof(long long),
                  cudaMemcpyHostToDevice));
  }
  Sell16 A16, B16;
  to_sell16(rows, A16);
  to_sell16(rg, B16);
  Sell16 *S16[2] = {&A16, &B16};
  uint16_t *d16[2];
  long long *db16[2];
  int *dpt[2];
  for (int v = 0; v < 2; ++v) {
    if (!u16_ok) { S16[v]->idx.assign(1, 0); S16[v]->base.assign(nw + 1, 0); S16[v]->ptab.assign((size_t)nw * 32, 0); }
    CK(cudaMalloc(&d16[v], S16[v]->idx.size() * 2));
    CK(cudaMalloc(&db16[v], (nw + 1) * sizeof(long long)));
    CK(cudaMalloc(&dpt[v], (size_t)nw * 32 * sizeof(int)));
    CK(cudaMemcpy(d16[v], S16[v]->idx.data(), S16[v]->idx.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db16[v], S16[v]->base.data(), (nw + 1) * sizeof(long long),
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dpt[v], S16[v]->ptab.data(), (size_t)nw * 32 * sizeof(int),
                  cudaMemcpyHostToDevice));
  }
  std::printf("i32 list: %.1f MB\n", A.idx.size() * 4 / 1e6);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char *name[2] = {"plain", "greedy"};
  auto launch = [&](int G, int v) {
    const int nbk = (n + 255) / 256;
    if (G == 7) { k_sweep_pf<1><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 8) { k_sweep_pf<2><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 11) { k_sweep_cpw<3><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 12) { k_sweep_cpw<6><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 9) { k_sweep_cpa<3><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 10) { k_sweep_cpa<5><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 13) { k_sweep_bal<<<nbk, 256>>>(dpos, dbal, dbalbase, dbalq, dout[v], n, rc * rc); return; }
    if (G == 6) { k_sweep_pf<0><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 5) { k_sweep1k<<<(n + 1023) / 1024, 1024>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc); return; }
    if (G == 1) k_sweep<1><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc);
    if (G == 2) k_sweep<2><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc);
    if (G == 3) k_sweep<3><<<nbk, 256>>>(dpos, didx[v], dbase[v], dcnt, dout[v], n, rc * rc);
    if (G == 4 && u16_ok) k_sweep16<<<nbk, 256>>>(dpos, d16[v], db16[v], dpt[v], dcnt, dout[v], n, rc * rc);
  };
  for (int rep = 0; rep < 2; ++rep)
    for (int G : {1, 6, 13})
      for (int v = 0; v < 2; ++v) {
        for (int w = 0; w < 5; ++w) launch(G, v);
        cudaEventRecord(e0);
        for (int w = 0; w < 50; ++w) launch(G, v);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("%s %s: %.4f ms per sweep, %.3f ns per particle\n", G == 13 ? "balanced rows (dealt evenly, owner lanes)" : G == 11 ? "cp.async warp chunks ring 3" : G == 12 ? "cp.async warp chunks ring 6" : G == 9 ? "cp.async index ring 3" : G == 10 ? "cp.async index ring 5" : G == 8 ? "no index loads, L1-hit gathers" : G == 7 ? "index stream, L1-hit gathers" : G == 6 ? "i32 G=1 index prefetch" : G == 5 ? "i32 1024-thread CTAs" : G == 4 ? "u16x8" : G == 1 ? "i32 G=1" : G == 2 ? "i32 G=2" : "i32 G=3", name[v], ms / 50, ms / 50 * 1e6 / n);
      }
  std::vector<float4> f0(n), f1(n);
  launch(13, 0);
  CK(cudaMemcpy(f0.data(), dout[0], n * sizeof(float4), cudaMemcpyDeviceToHost));
  launch(1, 0);
  CK(cudaMemcpy(f1.data(), dout[0], n * sizeof(float4), cudaMemcpyDeviceToHost));
  double md = 0, mf = 0;
  for (int i = 0; i < n; ++i) {
    md = std::max(md, (double)std::fabs(f0[i].x - f1[i].x));
    mf = std::max(mf, (double)std::fabs(f0[i].x));
  }
  std::printf("max |Fx| %.3g, max |dFx| balanced vs i32 (plain) %.3g\n", mf, md);
  return 0;
}
