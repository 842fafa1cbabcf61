// pm_internal.cuh -- shared device-side definitions of the CUDA path.
//
// Nothing here is shared with oracle/ (the oracle and the CUDA
// path share no code).  The decision functions below implement readings
// R1 (wrap), R3 (cell id) and R4 (pair distance) of DESIGN.md with explicit
// round-to-nearest intrinsics so that nvcc cannot contract or reorder them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef PM_DEV
#define PM_DEV __device__ __forceinline__
#endif

namespace pm {

constexpr int kWarp = 32;

// ----------------------------------------------------------------------------
// Per-context constant parameters, passed to kernels by value.
// ----------------------------------------------------------------------------
struct Box {
  float lo[3], hi[3];
  float L[3];      // fl32(hi - lo)
  float halfL[3];  // L / 2 (exact)
  int per[3];      // periodic axis flags
};

struct Grid {
  int n[3];        // cells per axis (R2)
  float inv_w[3];  // fp32(n / (hi - lo)) (R2)
  int ncell;
};

struct LJ {
  float rc2;       // fl32(r_cut * r_cut)
  float c12;       // 48 eps sigma^12
  float c6;        // 24 eps sigma^6
  float e12;       // 4 eps sigma^12
  float e6;        // 4 eps sigma^6
  float r_min;     // capped mode (R22) when > 0
  float inv_mass;
  float eps, sigma;
};

struct SPH {
  float h, inv_h, mass, rho0, inv_rho0, gamma, b, alpha, cbar, eta2;
  float w_norm;     // 1 / (pi h^3)
  float dw_norm;    // 1 / (pi h^4)
  float g[3];
};

struct Params {
  Box box;
  Grid grid;
  LJ lj;
  SPH sph;
  float rv2;        // fl32(r_v * r_v)
  float half_skin2; // (skin/2)^2
  float mi_margin;  // r_v + skin: particles farther than this from every
                    // periodic face cannot have a list partner across it
  int nbr_cap;      // slots per row (multiple of 4)
};

// Device buffers (pointers fixed between reallocations; captured in graphs).
// Double-buffered arrays are selected by State::cur_pv / cur_id at run time.
struct Bufs {
  float4 *pos[2];
  float4 *vel[2];
  int64_t *gid[2];
  int32_t *kind[2];
  float4 *xref;        // positions at the last build (cell order)
  float4 *force;       // forces / SPH accelerations (current order)
  float2 *rhoP;        // SPH density, pressure (current order)
  int32_t *cell_of;    // cell id in the storage order the build started from
  int32_t *slot;       // unordered slot within the cell (atomic claim)
  int32_t *count;      // [ncell]
  int32_t *start;      // [ncell + 1]
  int32_t *perm;       // [n] sorted k -> storage index
  int32_t *sorttmp;    // [n] scatter target before the per-cell sort
  int32_t *scan_tmp;   // block sums for the scan
  int32_t *nbr;        // SELL-32 neighbour slots, int4-interleaved
  int32_t *cnt;        // [n] neighbour row lengths
  struct State *st;    // device-resident state
};

// Device-resident mutable state (one per context).
struct State {
  int cur_pv;           // which pos/vel buffer is current
  int cur_id;           // which gid/kind buffer is current
  int pending_flip;     // a kernel wrote the alternate pos/vel buffers
  int need_rebuild;     // displacement > skin/2 seen
  int abort;            // sticky device error (pm_status code), stops a step loop
  int mode;             // step kernel mode (kModeInner / kModeFinal)
  int max_row;          // longest row of the last build
  int overflow_need;    // required capacity after an overflow
  long long err_gid;    // particle that raised a device error
  long long step_index; // steps begun in the current pm_step_vv call
  long long step_target;
  long long n_rebuilds;
  long long nnz;        // entries of the last build
  long long steps_done; // force-step kernels completed (not aborted)
  int do_rebuild;       // rebuild decision of the current step (non-graph path)
  double acc[4];        // energy: U_raw, virial, npairs, KE
};

enum { kModeInner = 0, kModeFinal = 1 };

// ----------------------------------------------------------------------------
// R1: fp32 periodic wrap into [lo, hi).
// ----------------------------------------------------------------------------
PM_DEV float wrap1(float x, float lo, float hi, float L) {
  if (x >= hi) {
    x = __fsub_rn(x, L);
  } else if (x < lo) {
    x = __fadd_rn(x, L);
  }
  if (x >= hi) x = lo;
  return x;
}

// R3: c = min(max(floor(fl(fl(x - lo) * inv_w)), 0), n - 1).
PM_DEV int cell_coord(float x, float lo, float inv_w, int n) {
  float u = __fmul_rn(__fsub_rn(x, lo), inv_w);
  float f = floorf(u);
  int c = (int)f;
  if (f < 0.0f) c = 0;
  if (c > n - 1) c = n - 1;
  return c;
}

// R4: delta = x_j - x_i with the Sterbenz-ordered periodic correction.
PM_DEV float pair_delta1(float a, float b, float L, float halfL, int per) {
  float e = __fsub_rn(b, a);
  if (per) {
    if (e > halfL) return __fsub_rn(__fsub_rn(b, L), a);
    if (e < -halfL) return __fsub_rn(b, __fsub_rn(a, L));
  }
  return e;
}

// R4': d2 = fma(dz, dz, fma(dy, dy, dx * dx)), each single-rounded.
PM_DEV float dist2(float dx, float dy, float dz) {
  float s = __fmul_rn(dx, dx);
  s = __fmaf_rn(dy, dy, s);
  s = __fmaf_rn(dz, dz, s);
  return s;
}

PM_DEV float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

PM_DEV float fast_rsqrt(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// SELL-32 neighbour slot layout: row i = 32 * slice + lane; entry k of the
// row lives at nbr[(slice * cap + k) * 32 + lane] -- a warp reading entry k
// of its 32 rows touches one contiguous 128-byte line.
PM_DEV int64_t nbr_row_base(int i, int cap) {
  return (int64_t)(i >> 5) * cap * 32 + (i & 31);
}

PM_DEV void raise_error(State *st, int code, long long gid) {
  if (atomicCAS(&st->abort, 0, code) == 0) st->err_gid = gid;
}

}  // namespace pm

// ----------------------------------------------------------------------------
// Host-side launchers (defined in the k_*.cu files).
// ----------------------------------------------------------------------------
namespace pm {
void launch_zero_i32(int32_t *p, int64_t n, cudaStream_t s);
void launch_cell_ids(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_scan(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_sort_reorder(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_flip(const Bufs &B, int flip_pv, int flip_id, int count_rebuild, cudaStream_t s);
void launch_verlet(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_lj(const Params &P, const Bufs &B, int64_t n, int want_energy, cudaStream_t s);
void launch_lj_step(const Params &P, const Bufs &B, int64_t n, float dt, cudaStream_t s);
void launch_kick_drift(const Params &P, const Bufs &B, int64_t n, float dt, cudaStream_t s);
void launch_step_begin(const Bufs &B, cudaGraphConditionalHandle h, int use_handle,
                       cudaStream_t s);
void launch_ke(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_sph_density(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_sph_forces(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_verlet_export(const Bufs &B, int64_t n, int cap, const int64_t *row_ptr,
                          int64_t *col_gid, cudaStream_t s);
}  // namespace pm
