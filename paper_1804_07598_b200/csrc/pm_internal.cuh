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

// Device-side bounds checks of the debug build (build.build(checks=True) ->
// libpm_checks.so, -DPM_CHECKS): a failed check prints its location and traps
// the kernel (the call then reports PM_E_CUDA).  compute-sanitizer is not
// available on the GPU pool (profiles/r02_compute_sanitizer_refused.txt).
#ifdef PM_CHECKS
#include <cstdio>
#define PM_CHECK(cond)                                                          \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("PM_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define PM_CHECK(cond) \
  do {                 \
  } while (0)
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

// Cell grid in the context's local frame.  Single GPU: o = box.lo,
// wrap = box.per, unwrap = 0 (exactly R2/R3).  Decomposed axis of a
// multi-GPU sub-domain: o = slo - r_v, the extent covers the ghost layers,
// wrap = 0 (no local periodic stencil) and unwrap = 1 (a global coordinate is
// mapped to the image nearest the sub-domain before binning).
struct Grid {
  int n[3];        // cells per axis (R2)
  float inv_w[3];  // fp32(n / extent) (R2)
  float o[3];      // frame origin
  float ext[3];    // frame extent
  int wrap[3];     // periodic stencil along this axis
  int unwrap[3];   // bin the nearest image (decomposed axes)
  int safe_lo[3], safe_hi[3];  // decomposed axes: cells whose extent lies strictly
                               // inside the global box (no wrapped particle)
  int ncell;
};

// Decomposition of the global periodic box into p[0] x p[1] x p[2] cuboids;
// this context owns cuboid c.  Ownership along axis d: the pinned fp32 rule
// min(max(floor(fl(fl(x - glo) * inv_s)), 0), p - 1).
constexpr int kMaxCuts = 15;  // non-uniform cuts: at most 16 slabs per axis

struct Dist {
  int p[3], c[3];
  float glo[3], inv_s[3];
  float slo[3], shi[3];  // this sub-domain (fp32)
  float rg;              // ghost selection width (r_v with a 1e-5 margin)
  int cuts;              // 1: ownership by the cut positions below (load balancing)
  float cut[3][kMaxCuts];  // interior cut positions per axis, increasing: slab c =
                           // #{k : x >= cut[d][k]}
};

constexpr int kGhostBit = 1 << 30;  // kind flag of a ghost copy
constexpr int kGroupHoldMax = 64;   // in-process group members per hold update

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

// DEM (Eqs. 9-13; readings R29-R33)
struct DEM {
  float R, m, inv_m, inv_I, kn, kt, gn, gt, mu, meff;
  float g[3];
  int walls[6];  // plane walls at the box faces x-lo, x-hi, y-lo, y-hi, z-lo, z-hi
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
  int dist;         // 1: sub-domain context (ghosts present, skip them as rows)
  float vmax;       // velocity limit (reading R22), 0 = off
  int sph_state;    // 1: the cell-sort reorder also permutes the SPH stepping state
  int dem_state;    // 1: ... and the DEM angular velocities
  int newton;       // 1: half (Newton) list, j > i in cell order (NEXT-1)
  int reach;        // stencil half-width in cells: 1 (side >= r_v) or 2 (side >= r_v/2);
                    // kept out of Grid: the sweeps' hot constants stay where they were
  DEM dem;
  // fused ghost refresh (decomposed LJ): the sweep's epilogue stores each new
  // position straight into the peers' ghost slots (peer_pos[peer][buffer]);
  // appended last so the hot constants above keep their offsets
  int peer_n;
  float4 *peer_pos[26][2];
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
  float2 *rhoP[2];     // SPH density, pressure (by State::cur_id: the stepping
                       // reorder permutes them with the particles)
  float4 *vold[2];     // SPH stepping: velocities of the previous step (Verlet);
                       // w = the density of the previous step
  float *drho;         // SPH stepping: density rate (Eq. 2), current order
  float4 *omega[2];    // DEM angular velocities (by State::cur_id)
  float4 *torque;      // DEM torques, current order
  float4 *hist;        // DEM tangential displacement per list slot (SELL layout of nbr)
  float4 *hist_old;    // ... of the previous list, kept across a rebuild
  int32_t *nbr_old;    // previous list (rows, layout, lengths) for the history remap
  int64_t *slice_off_old;
  int32_t *cnt_old;
  int64_t *gid_old;    // decomposed DEM: gid of every local index before a rebuild
  int32_t *cell_of;    // cell id in the storage order the build started from
  int32_t *slot;       // unordered slot within the cell (atomic claim)
  int32_t *count;      // [ncell]
  int32_t *start;      // [ncell + 1]
  int32_t *perm;       // [n] sorted k -> storage index
  int32_t *invperm;    // [n] storage index -> sorted k (multi-GPU remap)
  int32_t *sorttmp;    // [n] scatter target before the per-cell sort
  int32_t *scan_tmp;   // block sums for the scan
  int32_t *nbr;        // SELL-32 neighbour slots (see nbr_row_base)
  int64_t *slice_off;  // [nslices + 1] slice offsets in 128-byte lines
  int32_t *big_cells;  // cells with > 32 particles (block-level sort)
  int32_t *cnt;        // [n] neighbour row lengths
  struct State *st;    // device-resident state
  int32_t *ps_off;     // fused refresh: per local particle, its destinations
  int2 *ps_dst;        //   ps_dst[ps_off[i] .. ps_off[i+1]) = (peer, ghost slot)
  uint8_t *wclass;     // decomposed contexts, per 32-row slice: 1 if a row of it may
                       // have ghost partners (boundary), 0 interior (k_warp_class)
  int rm;              // 1: row-major slices (each row contiguous; long rows, LJ
                       // full lists only -- see nbr_row_base)
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
  int n_big;            // number of entries in Bufs::big_cells
  long long coinc_gid;  // a particle with a coincident partner (-1: none), set
                        // by the cell sort, raised as PM_E_COINCIDENT by the
                        // Verlet build (the cell list itself is well defined)
  // SPH time stepping (pm_sph_run)
  unsigned dtf_bits;    // min over fluid of sqrt(h/|a|) (fp32 bits; >= 0 so uint order)
  unsigned dtcv_bits;   // min over particles of h/(c0 + max |mu|)
  float sph_dt;         // step size of the current step
  float sph_dt_min, sph_dt_max;
  long long sph_step;   // steps taken (Euler step every `every`)
  double sph_time;      // simulated time
  double acc[4];        // energy: U_raw, virial, npairs, KE
  int hold;             // group step batches (pm_dist_run): the global rebuild flag
                        // of the previous step; while set the step kernels of the
                        // batch's remaining steps (sweep, refresh pack / unpack)
                        // do nothing, so the host need not synchronise per step
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
PM_DEV int cell_coord_u(float u, float inv_w, int n) {
  float f = floorf(__fmul_rn(u, inv_w));
  int c = (int)f;
  if (f < 0.0f) c = 0;
  if (c > n - 1) c = n - 1;
  return c;
}

PM_DEV int cell_coord(float x, float lo, float inv_w, int n) {
  return cell_coord_u(__fsub_rn(x, lo), inv_w, n);
}

// Cell coordinate along axis d in the local frame (identical to R3 when the
// axis is not decomposed).
PM_DEV int local_coord(const Box &box, const Grid &g, int d, float x) {
  float u = __fsub_rn(x, g.o[d]);
  if (g.unwrap[d]) {
    if (u < 0.0f) u = __fadd_rn(u, box.L[d]);
    else if (u >= g.ext[d]) u = __fsub_rn(u, box.L[d]);
  }
  return cell_coord_u(u, g.inv_w[d], g.n[d]);
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

// SELL-32 neighbour slot layout with per-slice widths: row i = 32 * slice +
// lane; entry k of the row lives at nbr[(slice_off[slice] + k) * 32 + lane]
// (a warp reading entry k of its 32 rows touches one contiguous 128-byte
// line); the slice's capacity is slice_off[slice + 1] - slice_off[slice].
// Uniform liquids get equal widths; clustered inputs (rows from 0 to ~12k
// entries) get widths from the exact counts of the previous build.
// Row-major slices (Bufs::rm, LJ contexts whose widest slice is >= kRowMajorMin
// entries): the same slice storage, row i contiguous at slice_off * 32 +
// lane * width, entry k at + k -- a lane's appends in the build then fill
// whole sectors in order instead of one slot of a line shared by lanes whose
// rows drift apart by thousands of entries.
constexpr int kRowMajorMin = 512;
PM_DEV int64_t nbr_row_base(const Bufs &B, int i) {
  const int64_t s = B.slice_off[i >> 5];
  if (B.rm) return s * 32 + (int64_t)(i & 31) * (B.slice_off[(i >> 5) + 1] - s);
  return s * 32 + (i & 31);
}
// distance between consecutive entries of a row
PM_DEV int nbr_stride(const Bufs &B) { return B.rm ? 1 : 32; }

PM_DEV int nbr_row_cap(const Bufs &B, int i) {
  return (int)(B.slice_off[(i >> 5) + 1] - B.slice_off[i >> 5]);
}

PM_DEV void raise_error(State *st, int code, long long gid) {
  if (atomicCAS(&st->abort, 0, code) == 0) st->err_gid = gid;
}

// ----------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, sm_90+) completing on a shared-memory
// mbarrier: one elected thread sets the expected byte count, any thread may
// issue copies (16-byte aligned, sizes multiple of 16), every thread waits.
// ----------------------------------------------------------------------------
PM_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

PM_DEV void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

PM_DEV void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

PM_DEV void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bounded wait: returns false if the phase did not complete within ~2^24
// polls (a byte-count mismatch would otherwise hang the GPU; the caller
// raises a device error instead).
PM_DEV bool mbar_wait(uint64_t *bar, unsigned parity) {
  for (int it = 0; it < (1 << 24); ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return true;
  }
  return false;
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
void launch_sph_init_run(const Bufs &B, int64_t n, cudaStream_t s);
constexpr int kDemHist = 24;  // contacts a migrating grain carries (PM_MSG_MIGRATE_HIST)
int dem_hist_record_bytes();
void launch_dem_hist_pack(const Bufs &B, const int *list, int nsend, void *out, cudaStream_t s);
void launch_dem_remap_dist(const Bufs &B, int64_t n, const int *stay_old, int n_stay,
                           const void *hist_in, int n_arr, cudaStream_t s);
void launch_dem_step(const Params &P, const Bufs &B, int64_t n, float dt, cudaStream_t s);
void launch_dem_remap(const Bufs &B, int64_t n, cudaStream_t s);
void launch_dem_save(const Bufs &B, int64_t n, cudaStream_t s);
void launch_dem_step_begin(const Bufs &B, cudaGraphConditionalHandle h, cudaStream_t s);
void launch_sph_set_rho(const Params &P, const Bufs &B, int64_t n, const float *rho,
                        cudaStream_t s);
void launch_sph_rates(const Params &P, const Bufs &B, int64_t n, cudaStream_t s);
void launch_sph_update(const Params &P, const Bufs &B, int64_t n, float bound, float cfl,
                       int every, cudaStream_t s);
void launch_sph_step(const Params &P, const Bufs &B, int64_t n, float cfl, int every,
                     cudaStream_t s);
void launch_verlet_shifts(const Params &P, const Bufs &B, int64_t n, const int64_t *row_ptr,
                          int8_t *col_shift, cudaStream_t s);
void launch_verlet_export(const Bufs &B, int64_t n, const int64_t *row_ptr, int64_t *col_gid,
                          cudaStream_t s);
void launch_exclusive_scan(int32_t *count, int32_t *start, int32_t *tmp, int n, cudaStream_t s);
int scan_tiles(int n);
void launch_peer_csr(const Bufs &B, const int *send_idx, const int *dst_peer, const int *dst_slot,
                     int nsend, int32_t *cnt, int n, int32_t *tmp, cudaStream_t s);
void launch_lj_half_forces(const Params &P, const Bufs &B, int64_t n, int want_energy,
                           cudaStream_t s);
void launch_lj_half_integrate(const Params &P, const Bufs &B, int64_t n, float dt, int mode,
                              cudaStream_t s);
void launch_ghost_put(const Bufs &B, int pack, const int *idx, int m, void *buf, cudaStream_t s);
void launch_warp_class(const Dist &D, const Bufs &B, int64_t n, cudaStream_t s);
// wphase: -1 every row; 0 / 1 only the slices whose wclass is 0 (interior) /
// 1 (boundary) -- the two halves of an overlapped step (the second one does
// the step's bookkeeping)
void launch_lj_step_mode(const Params &P, const Bufs &B, int64_t n, float dt, int mode,
                         cudaStream_t s, int wphase = -1);
int dist_record_bytes(int what);
void launch_dist_plan(const Params &P, const Bufs &B, const Dist &D, int n_owned, int what,
                      uint32_t *mask, int *blk_counts, const int *order, int *dir_base,
                      long long *totals, int *list, cudaStream_t s);
void launch_dist_pack(const Bufs &B, int what, const int *list, int nsend, void *out,
                      cudaStream_t s);
void launch_dist_compact(const Bufs &B, const int *stay, int n_stay, cudaStream_t s);
void launch_dist_unpack(const Bufs &B, int what, const void *in, int nrecv, int base,
                        cudaStream_t s);
void launch_dist_remap(const int *invperm, int *send_idx, int nsend, int *ghost_slot, int nghost,
                       int n_owned, cudaStream_t s);
void launch_refresh_pack(const Bufs &B, const int *send_idx, int nsend, void *out,
                         cudaStream_t s);
void launch_refresh_pv(const Bufs &B, int pack, const int *idx, int m, void *buf, int with_w,
                       cudaStream_t s);
void launch_refresh_unpack(const Bufs &B, const int *ghost_slot, int nghost, const void *in,
                           cudaStream_t s);
}  // namespace pm
