/*
 * pm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the particle hot path of
 * arXiv 1804.07598 (OpenFPM).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (-ffp-contract=off: every float expression below is evaluated exactly as
 * written, one IEEE round-to-nearest per operation; x86-64 uses SSE, not x87).
 *
 * What it computes:
 *  - Integer structures (wrap, cell ids, counts, start, perm, Verlet sets) are
 *    defined by fp32 decision functions (readings R1-R6 in DESIGN.md), written
 *    here as plain C float expressions.
 *  - Real-valued results (forces, energies, densities, accelerations) are
 *    evaluated in fp64 from the same fp32 inputs, by the plain O(N) per row
 *    sum over ALL other particles -- the definition the cell/Verlet lists
 *    reorganise (§2: "Cell Lists [45] or Verlet Lists [46] ...
 *    reduces the computational cost to O(N)").
 *
 * Pins: tests/test_oracle_pins.py -- every function below has at least one
 * pin that does not re-type it.  The Eq. 5 viscosity VALUE is pinned by a
 * hand-computed pair (tests/golden/sph_viscosity_pair.txt; the constants
 * alpha, eta are inputs -- their values are reading R20, the paper gives
 * none), the virial by a closed form and the dilation identity
 * W = -dU_s/dlambda, the image shifts by reconstruction of the minimum image,
 * the CPU method (orc_md_cells_run) by the brute-force trajectory.  Partly
 * pinned (the pins cover some terms only, noted at the function): the SPH
 * time stepping (R26-R28: exact free fall fixes the x and v updates of both
 * the Verlet and the Euler step, the continuity sign and momentum; the
 * coefficient of the density update is not separately fixed) and the DEM
 * wall model (R33: the normal wall force by the Hertz resting depth; the
 * walls have no tangential friction by reading).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------ */
/* R1: fp32 periodic wrap into the half-open box [lo, hi).             */
/* PAPER.md:166 (§4.1) "Periodic boundary conditions are imposed in all */
/* three coordinate directions"; the face convention is reading R1.    */
/* ------------------------------------------------------------------ */
static float wrap1(float x, float lo, float hi) {
  float L = hi - lo;
  if (x >= hi) {
    x = x - L;
  } else if (x < lo) {
    x = x + L;
  }
  if (x >= hi) x = lo; /* fl(-tiny + L) == L */
  return x;
}

/* Returns the number of particles outside [lo,hi) on a non-periodic axis. */
int64_t orc_wrap(int64_t n, float *pos4, const float lo[3], const float hi[3],
                 const int32_t per[3]) {
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 3; ++d) {
      float x = pos4[4 * i + d];
      if (per[d]) {
        pos4[4 * i + d] = wrap1(x, lo[d], hi[d]);
      } else if (!(x >= lo[d] && x < hi[d])) {
        bad++;
      }
    }
  }
  return bad;
}

/* ------------------------------------------------------------------ */
/* R2: cell grid.  n_d = floor((hi-lo) / (r_v / cell_div)) in fp64 on the */
/* fp32 inputs; inv_w_d = fp32(n_d / (hi-lo)).  PAPER.md:48 (§2) Cell   */
/* Lists; cell side >= interaction radius so a 27-cell stencil suffices. */
/* ------------------------------------------------------------------ */
int orc_cell_grid(const float lo[3], const float hi[3], float rv, int32_t cell_div,
                  int32_t ncell[3], float inv_w[3]) {
  for (int d = 0; d < 3; ++d) {
    double ext = (double)hi[d] - (double)lo[d];
    double side = (double)rv / (double)cell_div;
    double nd = floor(ext / side);
    if (nd < 1) nd = 1;
    ncell[d] = (int32_t)nd;
    inv_w[d] = (float)(nd / ext);
  }
  return 0;
}

/* R3: c_d = min(max(floor(fl(fl(x - lo) * inv_w)), 0), n_d - 1);
 *     id = c_x + n_x (c_y + n_y c_z). */
void orc_cell_ids(int64_t n, const float *pos4, const float lo[3], const float inv_w[3],
                  const int32_t ncell[3], int32_t *cell_of) {
  for (int64_t i = 0; i < n; ++i) {
    int32_t c[3];
    for (int d = 0; d < 3; ++d) {
      float t = pos4[4 * i + d] - lo[d];
      float u = t * inv_w[d];
      float f = floorf(u);
      int32_t cd = (int32_t)f;
      if (f < 0.0f) cd = 0;
      if (cd > ncell[d] - 1) cd = ncell[d] - 1;
      c[d] = cd;
    }
    cell_of[i] = c[0] + ncell[0] * (c[1] + ncell[1] * c[2]);
  }
}

/* Step 5 of the oracle definition: counts, exclusive start (start[ncell] = n)
 * and the stable permutation: perm[k] = storage index of the k-th particle in
 * (cell, storage index) order.  Plain stable counting sort. */
void orc_counting_sort(int64_t n, const int32_t *cell_of, int64_t ncell_total,
                       int32_t *count, int32_t *start, int32_t *perm) {
  memset(count, 0, sizeof(int32_t) * (size_t)ncell_total);
  for (int64_t i = 0; i < n; ++i) count[cell_of[i]]++;
  int64_t acc = 0;
  for (int64_t c = 0; c < ncell_total; ++c) {
    start[c] = (int32_t)acc;
    acc += count[c];
  }
  start[ncell_total] = (int32_t)acc;
  int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ncell_total > 0 ? ncell_total : 1));
  memcpy(next, start, sizeof(int32_t) * (size_t)ncell_total);
  for (int64_t i = 0; i < n; ++i) perm[next[cell_of[i]]++] = (int32_t)i;
  free(next);
}

/* ------------------------------------------------------------------ */
/* R4: fp32 pair difference delta = x_j - x_i with the Sterbenz-ordered  */
/* periodic correction, and d2 = fma(dz,dz, fma(dy,dy, dx*dx)) (reading  */
/* R4': single-rounded fused multiply-adds, fmaf is exact).   */
/* ------------------------------------------------------------------ */
static float pair_delta1(float a, float b, float L, float halfL, int per) {
  float e = b - a;
  if (per) {
    if (e > halfL) {
      float bb = b - L;
      return bb - a;
    } else if (e < -halfL) {
      float aa = a - L;
      return b - aa;
    }
  }
  return e;
}

static float pair_d2_f32(const float *xi, const float *xj, const float L[3],
                         const float halfL[3], const int32_t per[3], int8_t shift[3]) {
  float dl[3];
  for (int d = 0; d < 3; ++d) {
    dl[d] = pair_delta1(xi[d], xj[d], L[d], halfL[d], per[d]);
    if (shift) {
      float e = xj[d] - xi[d];
      shift[d] = (int8_t)(per[d] ? (e > halfL[d] ? -1 : (e < -halfL[d] ? 1 : 0)) : 0);
    }
  }
  float s = dl[0] * dl[0];
  s = fmaf(dl[1], dl[1], s);
  s = fmaf(dl[2], dl[2], s);
  return s;
}

static void box_consts(const float lo[3], const float hi[3], float L[3], float halfL[3]) {
  for (int d = 0; d < 3; ++d) {
    L[d] = hi[d] - lo[d];
    halfL[d] = L[d] * 0.5f;
  }
}

float orc_pair_d2(const float xi[3], const float xj[3], const float lo[3], const float hi[3],
                  const int32_t per[3]) {
  float L[3], hL[3];
  box_consts(lo, hi, L, hL);
  return pair_d2_f32(xi, xj, L, hL, per, NULL);
}

/* fp64 minimum-image delta x_i - x_j of the fp64 values of fp32 positions,
 * with L the fp64 value of the fp32 box length (oracle step 8). */
static void delta64(const float *xi, const float *xj, const double L[3], const int32_t per[3],
                    double out[3]) {
  for (int d = 0; d < 3; ++d) {
    double e = (double)xi[d] - (double)xj[d];
    if (per[d]) {
      if (e > 0.5 * L[d]) e -= L[d];
      else if (e < -0.5 * L[d]) e += L[d];
    }
    out[d] = e;
  }
}

/* ------------------------------------------------------------------ */
/* R5: Verlet set N_i = { j != i : d2_32(i,j) < fl(rv*rv) }, brute force  */
/* over all j (§4.1 Verlet lists [46]).        */
/* rows: which particles (storage index) to build; output CSR over rows   */
/* with cols = storage index of j (ascending) and shift codes.            */
/* Returns total entries, or -(needed) if cap is too small.               */
/* ------------------------------------------------------------------ */
int64_t orc_verlet_rows(int64_t n, const float *pos4, const float lo[3], const float hi[3],
                        const int32_t per[3], float rv, const int64_t *rows, int64_t nrows,
                        int64_t *row_ptr, int32_t *cols, int8_t *shifts, int64_t cap) {
  float L[3], hL[3];
  box_consts(lo, hi, L, hL);
  float rv2 = rv * rv;
  int64_t *cnt = (int64_t *)calloc((size_t)(nrows > 0 ? nrows : 1), sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows[r];
    int64_t c = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      if (pair_d2_f32(pos4 + 4 * i, pos4 + 4 * j, L, hL, per, NULL) < rv2) c++;
    }
    cnt[r] = c;
  }
  int64_t tot = 0;
  for (int64_t r = 0; r < nrows; ++r) {
    row_ptr[r] = tot;
    tot += cnt[r];
  }
  row_ptr[nrows] = tot;
  if (tot > cap) {
    free(cnt);
    return -tot;
  }
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows[r];
    int64_t k = row_ptr[r];
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      int8_t sh[3];
      if (pair_d2_f32(pos4 + 4 * i, pos4 + 4 * j, L, hL, per, sh) < rv2) {
        cols[k] = (int32_t)j;
        if (shifts) {
          shifts[3 * k + 0] = sh[0];
          shifts[3 * k + 1] = sh[1];
          shifts[3 * k + 2] = sh[2];
        }
        k++;
      }
    }
  }
  free(cnt);
  return tot;
}

/* ------------------------------------------------------------------ */
/* Lennard-Jones (§4.1):                                  */
/*   V(r) = 4 eps [ (sigma/r)^12 - (sigma/r)^6 ]                        */
/*   F_i = sum_j -dV/dr * (x_i - x_j)/r                                  */
/*       = sum_j 24 eps (2 sigma^12 / r^14 - sigma^6 / r^8) (x_i - x_j)  */
/* (reading R7: the Listing 4.1 exponent at PAPER.md:212 is a typo).     */
/* Inclusion: d2_32 < fl(rc*rc) (R6, strict).  Capped mode (R22):        */
/* r_eff = max(r, r_min), f = -V'(r_eff) along (x_i - x_j)/r.            */
/* Outputs per row (fp64): F[3], U_i = 1/2 sum_j V, W_i = 1/2 sum_j d.f, */
/* npair_i = #included j.  Returns #pairs with r == 0 (coincident).      */
/* ------------------------------------------------------------------ */
static double lj_V(double r, double eps, double sig) {
  double sr6 = pow(sig / r, 6.0);
  return 4.0 * eps * (sr6 * sr6 - sr6);
}

/* -dV/dr */
static double lj_mdVdr(double r, double eps, double sig) {
  double sr6 = pow(sig / r, 6.0);
  return 24.0 * eps * (2.0 * sr6 * sr6 - sr6) / r;
}

int64_t orc_lj_rows(int64_t n, const float *pos4, const float lo[3], const float hi[3],
                    const int32_t per[3], float rc, double eps, double sigma, double r_min,
                    const int64_t *rows, int64_t nrows, double *F3, double *U, double *W,
                    int64_t *npair) {
  float L[3], hL[3];
  box_consts(lo, hi, L, hL);
  double L64[3] = {L[0], L[1], L[2]};
  float rc2 = rc * rc;
  int64_t ncoinc = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : ncoinc)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows[r];
    double f[3] = {0, 0, 0}, u = 0, w = 0;
    int64_t np = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      if (!(pair_d2_f32(pos4 + 4 * i, pos4 + 4 * j, L, hL, per, NULL) < rc2)) continue;
      double dl[3];
      delta64(pos4 + 4 * i, pos4 + 4 * j, L64, per, dl);
      double rr = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
      if (rr == 0.0) {
        ncoinc++;
        continue;
      }
      double re = (r_min > 0 && rr < r_min) ? r_min : rr;
      double fm = lj_mdVdr(re, eps, sigma); /* magnitude along +(x_i - x_j) */
      for (int d = 0; d < 3; ++d) f[d] += fm * dl[d] / rr;
      u += 0.5 * lj_V(re, eps, sigma);
      w += 0.5 * fm * rr;
      np++;
    }
    F3[3 * r + 0] = f[0];
    F3[3 * r + 1] = f[1];
    F3[3 * r + 2] = f[2];
    if (U) U[r] = u;
    if (W) W[r] = w;
    if (npair) npair[r] = np;
  }
  return ncoinc;
}

double orc_lj_V(double r, double eps, double sigma) { return lj_V(r, eps, sigma); }
double orc_lj_mdVdr(double r, double eps, double sigma) { return lj_mdVdr(r, eps, sigma); }

/* ------------------------------------------------------------------ */
/* Velocity Verlet in fp64 ("symplectic Velocity-verlet",  */
/* Listing 4.1 lines 58-59, 72 at PAPER.md:291-293, 320), m = mass:     */
/*   v += dt/2 F/m ; x += dt v ; wrap ; F = F(x) ; v += dt/2 F/m          */
/* Forces by the plain O(N^2) fp64 sum with fp64 cutoff r < rc (this is   */
/* an fp64 trajectory: no fp32 decisions).  trace[(s)*4 + {0,1,2,3}] =  */
/* {KE, U_raw, U_shift, npairs} at s = 0..nsteps.                         */
/* ------------------------------------------------------------------ */
static void forces64(int64_t n, const double *x, const double L[3], const int32_t per[3],
                     double rc, double eps, double sig, double r_min, double *F, double *Uraw,
                     double *Ushift, double *npairs) {
  double vrc = lj_V(rc, eps, sig);
  double u = 0, us = 0, np = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : u, us, np)
  for (int64_t i = 0; i < n; ++i) {
    double f[3] = {0, 0, 0};
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double dl[3];
      for (int d = 0; d < 3; ++d) {
        double e = x[3 * i + d] - x[3 * j + d];
        if (per[d]) {
          if (e > 0.5 * L[d]) e -= L[d];
          else if (e < -0.5 * L[d]) e += L[d];
        }
        dl[d] = e;
      }
      double rr = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
      if (!(rr < rc) || rr == 0.0) continue;
      double re = (r_min > 0 && rr < r_min) ? r_min : rr;
      double fm = lj_mdVdr(re, eps, sig);
      for (int d = 0; d < 3; ++d) f[d] += fm * dl[d] / rr;
      double v = lj_V(re, eps, sig);
      u += 0.5 * v;
      us += 0.5 * (v - vrc);
      np += 1.0;
    }
    F[3 * i + 0] = f[0];
    F[3 * i + 1] = f[1];
    F[3 * i + 2] = f[2];
  }
  *Uraw = u;
  *Ushift = us;
  *npairs = np;
}

void orc_vv_run(int64_t n, double *x, double *v, const double lo[3], const double hi[3],
                const int32_t per[3], double rc, double eps, double sigma, double r_min,
                double mass, double dt, int64_t nsteps, double *trace) {
  double L[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  double *F = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  double u, us, np;
  forces64(n, x, L, per, rc, eps, sigma, r_min, F, &u, &us, &np);
  for (int64_t s = 0;; ++s) {
    if (trace) {
      double ke = 0;
      for (int64_t i = 0; i < 3 * n; ++i) ke += 0.5 * mass * v[i] * v[i];
      trace[4 * s + 0] = ke;
      trace[4 * s + 1] = u;
      trace[4 * s + 2] = us;
      trace[4 * s + 3] = np;
    }
    if (s == nsteps) break;
    for (int64_t i = 0; i < 3 * n; ++i) v[i] += 0.5 * dt * F[i] / mass;
    for (int64_t i = 0; i < n; ++i) {
      for (int d = 0; d < 3; ++d) {
        double xx = x[3 * i + d] + dt * v[3 * i + d];
        if (per[d]) {
          if (xx >= hi[d]) xx -= L[d];
          else if (xx < lo[d]) xx += L[d];
        }
        x[3 * i + d] = xx;
      }
    }
    forces64(n, x, L, per, rc, eps, sigma, r_min, F, &u, &us, &np);
    for (int64_t i = 0; i < 3 * n; ++i) v[i] += 0.5 * dt * F[i] / mass;
  }
  free(F);
}

/* ------------------------------------------------------------------ */
/* SPH (§4.2, Eqs. 1, 3, 4, 5; readings R15-R21).     */
/* Cubic spline W (the "classic cubic SPH kernel [34]"):  */
/*   W(r,h) = 1/(pi h^3) { 1 - 1.5 q^2 + 0.75 q^3   (0 <= q < 1)         */
/*                         0.25 (2 - q)^3          (1 <= q < 2)         */
/*                         0                        (q >= 2) },  q = r/h */
/* ------------------------------------------------------------------ */
static const double ORC_PI = 3.14159265358979323846;

double orc_sph_W(double r, double h) {
  double q = r / h;
  double c = 1.0 / (ORC_PI * h * h * h);
  if (q < 1.0) return c * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
  if (q < 2.0) {
    double t = 2.0 - q;
    return c * 0.25 * t * t * t;
  }
  return 0.0;
}

double orc_sph_dWdr(double r, double h) {
  double q = r / h;
  double c = 1.0 / (ORC_PI * h * h * h * h);
  if (q < 1.0) return c * (-3.0 * q + 2.25 * q * q);
  if (q < 2.0) {
    double t = 2.0 - q;
    return c * (-0.75 * t * t);
  }
  return 0.0;
}

/* Density by summation (reading R16) including the self term, and the Tait
 * EOS Eq. 3: P = b [ (rho/rho0)^gamma - 1 ].  All particles (fluid and
 * boundary) get rho and P.  Neighbours: every q != p with fp64 r < 2h. */
void orc_sph_density_rows(int64_t n, const float *pos4, const float lo[3], const float hi[3],
                          const int32_t per[3], double h, double mass, double rho0, double b,
                          double gamma, const int64_t *rows, int64_t nrows, double *rho_out,
                          double *P_out) {
  float L[3], hL[3];
  box_consts(lo, hi, L, hL);
  double L64[3] = {L[0], L[1], L[2]};
  double w0 = orc_sph_W(0.0, h);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t p = rows[r];
    double rho = mass * w0;
    for (int64_t q = 0; q < n; ++q) {
      if (q == p) continue;
      double dl[3];
      delta64(pos4 + 4 * p, pos4 + 4 * q, L64, per, dl);
      double r2 = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
      if (!(r2 < 4.0 * h * h)) continue; /* W = 0 for r >= 2h */
      double rr = sqrt(r2);
      if (rr < 2.0 * h) rho += mass * orc_sph_W(rr, h);
    }
    rho_out[r] = rho;
    P_out[r] = b * (pow(rho / rho0, gamma) - 1.0);
  }
}

/* Eq. 1 with readings R17 (sign: a_p = -sum m (...) grad_p W(x_p - x_q)),
 * R18 ((P_p + P_q)/(rho_p rho_q) as printed), R20 (Pi_pq: Monaghan, nonzero
 * only for v_pq . r_pq < 0; cbar = c0, alpha, eta2 given; pinned by the
 * branch pins and by one hand-computed approaching pair,
 * tests/golden/sph_viscosity_pair.txt), g added to fluid particles only; boundary
 * particles (kind 1) get a = 0.  rho/P are per-particle inputs (storage
 * order, fp64) so the force pass can be pinned independently of the
 * density pass. */
void orc_sph_accel_rows(int64_t n, const float *pos4, const float *vel4, const double *rho,
                        const double *P, const int32_t *kind, const float lo[3],
                        const float hi[3], const int32_t per[3], double h, double mass,
                        double alpha, double cbar, double eta2, const double g[3],
                        const int64_t *rows, int64_t nrows, double *a_out) {
  float L[3], hL[3];
  box_consts(lo, hi, L, hL);
  double L64[3] = {L[0], L[1], L[2]};
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t p = rows[r];
    double a[3] = {0, 0, 0};
    if (kind && kind[p] != 0) {
      a_out[3 * r + 0] = a_out[3 * r + 1] = a_out[3 * r + 2] = 0.0;
      continue;
    }
    for (int64_t q = 0; q < n; ++q) {
      if (q == p) continue;
      double dl[3]; /* r_pq = x_p - x_q */
      delta64(pos4 + 4 * p, pos4 + 4 * q, L64, per, dl);
      double r2 = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
      if (!(r2 < 4.0 * h * h)) continue; /* grad W = 0 for r >= 2h */
      double rr = sqrt(r2);
      if (!(rr < 2.0 * h) || rr == 0.0) continue;
      double dw = orc_sph_dWdr(rr, h);
      double gradW[3] = {dl[0] / rr * dw, dl[1] / rr * dw, dl[2] / rr * dw};
      double vpq[3] = {(double)vel4[4 * p + 0] - vel4[4 * q + 0],
                       (double)vel4[4 * p + 1] - vel4[4 * q + 1],
                       (double)vel4[4 * p + 2] - vel4[4 * q + 2]};
      double vr = vpq[0] * dl[0] + vpq[1] * dl[1] + vpq[2] * dl[2];
      double Pi = 0.0;
      if (vr < 0.0) {
        double mu = h * vr / (rr * rr + eta2);
        double rbar = 0.5 * (rho[p] + rho[q]);
        Pi = -alpha * cbar * mu / rbar;
      }
      double coef = mass * ((P[p] + P[q]) / (rho[p] * rho[q]) + Pi);
      for (int d = 0; d < 3; ++d) a[d] -= coef * gradW[d];
    }
    for (int d = 0; d < 3; ++d) a_out[3 * r + d] = a[d] + g[d];
  }
}

/* ------------------------------------------------------------------ */
/* WCSPH time stepping (§4.2):   */
/* continuity density Eq. 2, Tait EOS Eq. 3, momentum Eq. 1 with Eq. 5,  */
/* "Verlet time-stepping [46] with dynamic step size" as in DualSPHysics */
/* (the scheme itself is not in the paper -- readings      */
/* R26-R28 in DESIGN.md; parity unpinned beyond the self-consistency     */
/* pins of tests/test_oracle_pins.py).  fp64 state, O(N^2) pair loop.    */
/*   D_p  = sum_q m v_pq . grad_p W(r_pq)          (R26, all particles)   */
/*   a_p  = Eq. 1 (fluid; boundary a = 0)                                 */
/*   dt   = cfl * min( min_fluid sqrt(h/|a_p|),                          */
/*                     min_p h / (c0 + max_q |h v_pq.r_pq/(r^2+eta2)|) )  */
/*   Verlet (R27): v' = v_prev + 2 dt a, rho' = rho_prev + 2 dt D;       */
/*   every Ns-th step and the first: v' = v + dt a, rho' = rho + dt D;   */
/*   x' = x + dt v + dt^2/2 a (fluid); boundary x, v fixed, rho evolves. */
/* ------------------------------------------------------------------ */
static void sph_rates64(int64_t n, const double *x, const double *v, const double *rho,
                        const double *P, const int32_t *kind, const double L[3],
                        const int32_t per[3], double h, double mass, double alpha, double cbar,
                        double eta2, const double g[3], double *a, double *D, double *dtf,
                        double *dtcv) {
  double fmin = 1e300, cvmin = 1e300;
#pragma omp parallel for schedule(dynamic, 16) reduction(min : fmin, cvmin)
  for (int64_t p = 0; p < n; ++p) {
    double ap[3] = {0, 0, 0}, dp = 0.0, mumax = 0.0;
    for (int64_t q = 0; q < n; ++q) {
      if (q == p) continue;
      double dl[3]; /* r_pq = x_p - x_q (minimum image on periodic axes) */
      for (int d = 0; d < 3; ++d) {
        double e = x[3 * p + d] - x[3 * q + d];
        if (per[d]) {
          if (e > 0.5 * L[d]) e -= L[d];
          else if (e < -0.5 * L[d]) e += L[d];
        }
        dl[d] = e;
      }
      double r2 = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
      if (!(r2 < 4.0 * h * h) || r2 == 0.0) continue;
      double rr = sqrt(r2);
      double dw = orc_sph_dWdr(rr, h);
      double gw[3] = {dl[0] / rr * dw, dl[1] / rr * dw, dl[2] / rr * dw};
      double vpq[3] = {v[3 * p] - v[3 * q], v[3 * p + 1] - v[3 * q + 1],
                       v[3 * p + 2] - v[3 * q + 2]};
      double vr = vpq[0] * dl[0] + vpq[1] * dl[1] + vpq[2] * dl[2];
      dp += mass * (vpq[0] * gw[0] + vpq[1] * gw[1] + vpq[2] * gw[2]);
      double mu = h * vr / (r2 + eta2);
      if (fabs(mu) > mumax) mumax = fabs(mu);
      double Pi = 0.0;
      if (vr < 0.0) Pi = -alpha * cbar * mu / (0.5 * (rho[p] + rho[q]));
      double coef = mass * ((P[p] + P[q]) / (rho[p] * rho[q]) + Pi);
      for (int d = 0; d < 3; ++d) ap[d] -= coef * gw[d];
    }
    D[p] = dp;
    double cv = h / (cbar + mumax);
    if (cv < cvmin) cvmin = cv;
    if (kind && kind[p] != 0) {
      a[3 * p] = a[3 * p + 1] = a[3 * p + 2] = 0.0;
    } else {
      for (int d = 0; d < 3; ++d) a[3 * p + d] = ap[d] + g[d];
      double am = sqrt(a[3 * p] * a[3 * p] + a[3 * p + 1] * a[3 * p + 1] +
                       a[3 * p + 2] * a[3 * p + 2]);
      double f = am > 0 ? sqrt(h / am) : 1e300;
      if (f < fmin) fmin = f;
    }
  }
  *dtf = fmin;
  *dtcv = cvmin;
}

/* x, v: fp64 (n x 3) in/out; rho: fp64 in/out.  trace[s] = dt of step s.
 * Positions on periodic axes are wrapped into [lo, hi). */
void orc_sph_run(int64_t n, double *x, double *v, double *rho, const int32_t *kind,
                 const double lo[3], const double hi[3], const int32_t per[3], double h,
                 double mass, double rho0, double b, double gamma, double alpha, double cbar,
                 double eta2, const double g[3], double cfl, int64_t every, int64_t nsteps,
                 double *trace) {
  double L[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  size_t n3 = sizeof(double) * 3 * (size_t)(n > 0 ? n : 1), n1 = n3 / 3;
  double *a = (double *)malloc(n3), *D = (double *)malloc(n1), *P = (double *)malloc(n1);
  double *vprev = (double *)malloc(n3), *rprev = (double *)malloc(n1);
  memcpy(vprev, v, n3);
  memcpy(rprev, rho, n1);
  for (int64_t s = 0; s < nsteps; ++s) {
    for (int64_t p = 0; p < n; ++p) P[p] = b * (pow(rho[p] / rho0, gamma) - 1.0);
    double dtf, dtcv;
    sph_rates64(n, x, v, rho, P, kind, L, per, h, mass, alpha, cbar, eta2, g, a, D, &dtf, &dtcv);
    double dt = cfl * (dtf < dtcv ? dtf : dtcv);
    if (trace) trace[s] = dt;
    int euler = (s == 0) || (every > 0 && (s + 1) % every == 0);
    for (int64_t p = 0; p < n; ++p) {
      double rn = euler ? rho[p] + dt * D[p] : rprev[p] + 2.0 * dt * D[p];
      rprev[p] = rho[p];
      rho[p] = rn;
      if (kind && kind[p] != 0) continue;
      for (int d = 0; d < 3; ++d) {
        double vo = v[3 * p + d], an = a[3 * p + d];
        double vn = euler ? vo + dt * an : vprev[3 * p + d] + 2.0 * dt * an;
        double xx = x[3 * p + d] + dt * vo + 0.5 * dt * dt * an;
        if (per[d]) {
          if (xx >= hi[d]) xx -= L[d];
          else if (xx < lo[d]) xx += L[d];
        }
        x[3 * p + d] = xx;
        vprev[3 * p + d] = vo;
        v[3 * p + d] = vn;
      }
    }
  }
  free(a);
  free(D);
  free(P);
  free(vprev);
  free(rprev);
}

/* ------------------------------------------------------------------ */
/* DEM (§4.5, Eqs. 9-13), fp64,   */
/* O(N^2) contact search, contact history keyed by the (gid_p, gid_q)    */
/* pair.  Readings (R29-R33):                                   */
/*   n = r_pq / |r_pq| (r_pq = r_p - r_q, minimum image on periodic axes), */
/*   delta = 2R - |r_pq| (Eq. 9), contact iff delta > 0;                  */
/*   v_pq = v_p - v_q - R (w_p + w_q) x n (relative velocity at the       */
/*   contact point); v_n = (v_pq.n) n, v_t = v_pq - v_n;                  */
/*   u_t <- u_t - (u_t.n) n + v_t dt (Eq. 10, kept tangential);           */
/*   s = sqrt(delta / 2R); F_n = s (kn delta n - gn meff v_n) (Eq. 11);    */
/*   F_t = s (-kt u_t - gt meff v_t) (Eq. 12), meff = m/2; Coulomb: if    */
/*   |F_t| > mu |F_n|, F_t <- F_t mu|F_n|/|F_t| and u_t is rescaled to    */
/*   match (u_t = -(F_t/s + gt meff v_t)/kt);                              */
/*   F_p += F_n + F_t; T_p += (-R n) x F_t;  walls (flags per box face,   */
/*   planes at the faces) act like a fixed sphere touching the plane:     */
/*   normal Hertz force with damping only;  gravity g.                    */
/*   Leapfrog (Eq. 13): v += dt F/m; x += dt v; w += dt T/I.              */
/* A contact that ends loses its history.  Pinned by closed forms (free   */
/* fall, resting depth on a wall, elastic head-on collision, momentum);   */
/* the wall model itself (R33) is "parity unpinned" beyond those.         */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t a, b;
  double u[3];
} dem_hist_t;

static int64_t dem_find(dem_hist_t *h, int64_t nh, int64_t a, int64_t b) {
  for (int64_t k = 0; k < nh; ++k)
    if (h[k].a == a && h[k].b == b) return k;
  return -1;
}

static void cross3(const double a[3], const double b[3], double c[3]) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

/* x, v, w: fp64 (n x 3) in/out; gid: unique ids; walls[6]: x-lo, x-hi,
 * y-lo, y-hi, z-lo, z-hi plane flags.  hist_cap: max stored contacts. */
int64_t orc_dem_run(int64_t n, double *x, double *v, double *w, const int64_t *gid,
                    const double lo[3], const double hi[3], const int32_t per[3],
                    const int32_t walls[6], double R, double m, double I, double kn, double kt,
                    double gn, double gt, double mu, const double g[3], double dt,
                    int64_t nsteps, int64_t hist_cap) {
  double L[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  dem_hist_t *hist = (dem_hist_t *)calloc((size_t)(hist_cap > 0 ? hist_cap : 1), sizeof(dem_hist_t));
  dem_hist_t *nhist = (dem_hist_t *)calloc((size_t)(hist_cap > 0 ? hist_cap : 1), sizeof(dem_hist_t));
  int64_t nh = 0;
  double *F = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  double *T = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  const double meff = 0.5 * m;
  for (int64_t s = 0; s < nsteps; ++s) {
    int64_t nn = 0;
    for (int64_t p = 0; p < n; ++p) {
      double f[3] = {m * g[0], m * g[1], m * g[2]}, t[3] = {0, 0, 0};
      for (int64_t q = 0; q < n; ++q) {
        if (q == p) continue;
        double r[3];
        for (int d = 0; d < 3; ++d) {
          double e = x[3 * p + d] - x[3 * q + d];
          if (per[d]) {
            if (e > 0.5 * L[d]) e -= L[d];
            else if (e < -0.5 * L[d]) e += L[d];
          }
          r[d] = e;
        }
        double rr = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        double delta = 2.0 * R - rr;
        if (!(delta > 0.0) || rr == 0.0) continue;
        double nv[3] = {r[0] / rr, r[1] / rr, r[2] / rr};
        double ws[3] = {w[3 * p] + w[3 * q], w[3 * p + 1] + w[3 * q + 1], w[3 * p + 2] + w[3 * q + 2]};
        double wxn[3];
        cross3(ws, nv, wxn);
        double vpq[3];
        for (int d = 0; d < 3; ++d) vpq[d] = v[3 * p + d] - v[3 * q + d] - R * wxn[d];
        double vn = vpq[0] * nv[0] + vpq[1] * nv[1] + vpq[2] * nv[2];
        double vnv[3] = {vn * nv[0], vn * nv[1], vn * nv[2]};
        double vt[3] = {vpq[0] - vnv[0], vpq[1] - vnv[1], vpq[2] - vnv[2]};
        double u[3] = {0, 0, 0};
        int64_t k = dem_find(hist, nh, gid[p], gid[q]);
        if (k >= 0) memcpy(u, hist[k].u, sizeof u);
        double un = u[0] * nv[0] + u[1] * nv[1] + u[2] * nv[2];
        for (int d = 0; d < 3; ++d) u[d] = u[d] - un * nv[d] + vt[d] * dt;
        double sq = sqrt(delta / (2.0 * R));
        double fn[3], ft[3];
        for (int d = 0; d < 3; ++d) {
          fn[d] = sq * (kn * delta * nv[d] - gn * meff * vnv[d]);
          ft[d] = sq * (-kt * u[d] - gt * meff * vt[d]);
        }
        double fnm = sqrt(fn[0] * fn[0] + fn[1] * fn[1] + fn[2] * fn[2]);
        double ftm = sqrt(ft[0] * ft[0] + ft[1] * ft[1] + ft[2] * ft[2]);
        if (ftm > mu * fnm && ftm > 0.0) {
          double sc = mu * fnm / ftm;
          for (int d = 0; d < 3; ++d) {
            ft[d] *= sc;
            u[d] = -(ft[d] / sq + gt * meff * vt[d]) / kt;
          }
        }
        if (nn < hist_cap) {
          nhist[nn].a = gid[p];
          nhist[nn].b = gid[q];
          memcpy(nhist[nn].u, u, sizeof u);
          ++nn;
        }
        double arm[3] = {-R * nv[0], -R * nv[1], -R * nv[2]}, tq[3];
        cross3(arm, ft, tq);
        for (int d = 0; d < 3; ++d) {
          f[d] += fn[d] + ft[d];
          t[d] += tq[d];
        }
      }
      /* walls: plane at the face, normal Hertz + damping */
      for (int d = 0; d < 3; ++d) {
        for (int side = 0; side < 2; ++side) {
          if (!walls[2 * d + side]) continue;
          double dist = side == 0 ? x[3 * p + d] - lo[d] : hi[d] - x[3 * p + d];
          double delta = R - dist;
          if (!(delta > 0.0)) continue;
          double nd = side == 0 ? 1.0 : -1.0; /* normal into the domain */
          double vn = v[3 * p + d] * nd;
          double sq = sqrt(delta / (2.0 * R));
          f[d] += sq * (kn * delta - gn * meff * vn) * nd;
        }
      }
      memcpy(F + 3 * p, f, sizeof f);
      memcpy(T + 3 * p, t, sizeof t);
    }
    dem_hist_t *tmp = hist;
    hist = nhist;
    nhist = tmp;
    nh = nn;
    for (int64_t p = 0; p < n; ++p) {
      for (int d = 0; d < 3; ++d) {
        v[3 * p + d] += dt / m * F[3 * p + d];
        double xx = x[3 * p + d] + dt * v[3 * p + d];
        if (per[d]) {
          if (xx >= hi[d]) xx -= L[d];
          else if (xx < lo[d]) xx += L[d];
        }
        x[3 * p + d] = xx;
        w[3 * p + d] += dt / I * T[3 * p + d];
      }
    }
  }
  free(F);
  free(T);
  free(hist);
  free(nhist);
  return nh;
}

/* ------------------------------------------------------------------ */
/* CPU baseline of the method itself (SURVEY §8(d) "Oracle timing"):     */
/* fp64 cell list + Verlet list with skin + velocity Verlet, the O(N)    */
/* reorganisation of orc_vv_run's O(N^2) sum (§2 "Cell Lists */
/* [45] or Verlet Lists [46] ... reduces the computational cost to O(N)"; */
/* PAPER.md:164 Verlet lists; PAPER.md:166 velocity Verlet; Listing 4.1   */
/* order at PAPER.md:291-320).  Plain code, no blocking: cells of side    */
/* >= r_v = rc + skin (n_d = floor(L_d / r_v) >= 3 per periodic axis),    */
/* row i = every j != i with fp64 minimum-image r^2 < r_v^2 over the 27   */
/* neighbour cells, rebuilt when a particle moved more than skin/2 since  */
/* the last build; forces over the row with r^2 < rc^2 (OpenMP over rows, */
/* full rows, no atomics).  Pinned against orc_vv_run (same trajectory up */
/* to summation order) in tests/test_oracle_pins.py.                      */
/* Returns the number of list builds, or -1 if a periodic axis has fewer  */
/* than 3 cells.  trace as orc_vv_run (may be NULL).                      */
/* ------------------------------------------------------------------ */
typedef struct {
  int nc[3];
  double inv_w[3];
  int64_t *start, *idx; /* cell starts (ncell + 1), particles by cell */
  int64_t *row_ptr;     /* n + 1 */
  int32_t *cols;
  int64_t cols_cap;
} md_lists_t;

static int md_cell_coord(double x, double lo, double inv_w, int nc) {
  int c = (int)floor((x - lo) * inv_w);
  if (c < 0) c = 0;
  if (c > nc - 1) c = nc - 1;
  return c;
}

static double md_min_image(double e, double L, int per) {
  if (per) {
    if (e > 0.5 * L) e -= L;
    else if (e < -0.5 * L) e += L;
  }
  return e;
}

static void md_build(int64_t n, const double *x, const double lo[3], const double L[3],
                     const int32_t per[3], double rv, md_lists_t *M) {
  int64_t ncell = (int64_t)M->nc[0] * M->nc[1] * M->nc[2];
  int64_t *cell = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  memset(M->start, 0, sizeof(int64_t) * (size_t)(ncell + 1));
  for (int64_t i = 0; i < n; ++i) {
    int c0 = md_cell_coord(x[3 * i + 0], lo[0], M->inv_w[0], M->nc[0]);
    int c1 = md_cell_coord(x[3 * i + 1], lo[1], M->inv_w[1], M->nc[1]);
    int c2 = md_cell_coord(x[3 * i + 2], lo[2], M->inv_w[2], M->nc[2]);
    cell[i] = c0 + (int64_t)M->nc[0] * (c1 + (int64_t)M->nc[1] * c2);
    M->start[cell[i] + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) M->start[c + 1] += M->start[c];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncell > 0 ? ncell : 1));
  memcpy(fill, M->start, sizeof(int64_t) * (size_t)ncell);
  for (int64_t i = 0; i < n; ++i) M->idx[fill[cell[i]]++] = i;
  free(fill);
  double rv2 = rv * rv;
  /* two passes over the rows: count, then fill */
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
      int64_t cc = cell[i];
      int c[3] = {(int)(cc % M->nc[0]), (int)((cc / M->nc[0]) % M->nc[1]),
                  (int)(cc / ((int64_t)M->nc[0] * M->nc[1]))};
      int64_t k = pass ? M->row_ptr[i] : 0;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            int q[3] = {c[0] + dx, c[1] + dy, c[2] + dz}, ok = 1;
            for (int d = 0; d < 3; ++d) {
              if (q[d] < 0 || q[d] >= M->nc[d]) {
                if (!per[d]) ok = 0;
                else q[d] = (q[d] + M->nc[d]) % M->nc[d];
              }
            }
            if (!ok) continue;
            int64_t qc = q[0] + (int64_t)M->nc[0] * (q[1] + (int64_t)M->nc[1] * q[2]);
            for (int64_t t = M->start[qc]; t < M->start[qc + 1]; ++t) {
              int64_t j = M->idx[t];
              if (j == i) continue;
              double r2 = 0.0;
              for (int d = 0; d < 3; ++d) {
                double e = md_min_image(x[3 * i + d] - x[3 * j + d], L[d], per[d]);
                r2 += e * e;
              }
              if (r2 < rv2) {
                if (pass) M->cols[k] = (int32_t)j;
                k++;
              }
            }
          }
      if (!pass) M->row_ptr[i + 1] = k;
    }
    if (!pass) {
      M->row_ptr[0] = 0;
      for (int64_t i = 0; i < n; ++i) M->row_ptr[i + 1] += M->row_ptr[i];
      if (M->row_ptr[n] > M->cols_cap) {
        free(M->cols);
        M->cols_cap = M->row_ptr[n] + M->row_ptr[n] / 4 + 1;
        M->cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)M->cols_cap);
      }
    }
  }
  free(cell);
}

static void md_forces(int64_t n, const double *x, const double L[3], const int32_t per[3],
                      const md_lists_t *M, double rc, double eps, double sig, double r_min,
                      double *F, double *Uraw, double *Ushift, double *npairs) {
  double vrc = lj_V(rc, eps, sig), rc2 = rc * rc;
  double u = 0, us = 0, np = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : u, us, np)
  for (int64_t i = 0; i < n; ++i) {
    double f[3] = {0, 0, 0};
    for (int64_t t = M->row_ptr[i]; t < M->row_ptr[i + 1]; ++t) {
      int64_t j = M->cols[t];
      double dl[3], r2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        dl[d] = md_min_image(x[3 * i + d] - x[3 * j + d], L[d], per[d]);
        r2 += dl[d] * dl[d];
      }
      if (!(r2 < rc2) || r2 == 0.0) continue;
      double rr = sqrt(r2);
      double re = (r_min > 0 && rr < r_min) ? r_min : rr;
      double fm = lj_mdVdr(re, eps, sig);
      for (int d = 0; d < 3; ++d) f[d] += fm * dl[d] / rr;
      double v = lj_V(re, eps, sig);
      u += 0.5 * v;
      us += 0.5 * (v - vrc);
      np += 1.0;
    }
    F[3 * i + 0] = f[0];
    F[3 * i + 1] = f[1];
    F[3 * i + 2] = f[2];
  }
  *Uraw = u;
  *Ushift = us;
  *npairs = np;
}

int64_t orc_md_cells_run(int64_t n, double *x, double *v, const double lo[3], const double hi[3],
                         const int32_t per[3], double rc, double skin, double eps, double sigma,
                         double r_min, double mass, double dt, int64_t nsteps, double *trace) {
  double L[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
  double rv = rc + skin;
  md_lists_t M;
  memset(&M, 0, sizeof M);
  for (int d = 0; d < 3; ++d) {
    M.nc[d] = (int)floor(L[d] / rv);
    if (M.nc[d] < 1) M.nc[d] = 1;
    if (per[d] && M.nc[d] < 3) return -1;
    M.inv_w[d] = M.nc[d] / L[d];
  }
  int64_t ncell = (int64_t)M.nc[0] * M.nc[1] * M.nc[2];
  size_t nn = (size_t)(n > 0 ? n : 1);
  M.start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncell + 1));
  M.idx = (int64_t *)malloc(sizeof(int64_t) * nn);
  M.row_ptr = (int64_t *)malloc(sizeof(int64_t) * (nn + 1));
  double *F = (double *)malloc(sizeof(double) * 3 * nn);
  double *xref = (double *)malloc(sizeof(double) * 3 * nn);
  int64_t builds = 0;
  md_build(n, x, lo, L, per, rv, &M);
  memcpy(xref, x, sizeof(double) * 3 * (size_t)n);
  builds++;
  double u, us, np;
  md_forces(n, x, L, per, &M, rc, eps, sigma, r_min, F, &u, &us, &np);
  double half2 = 0.25 * skin * skin;
  for (int64_t s = 0;; ++s) {
    if (trace) {
      double ke = 0;
      for (int64_t i = 0; i < 3 * n; ++i) ke += 0.5 * mass * v[i] * v[i];
      trace[4 * s + 0] = ke;
      trace[4 * s + 1] = u;
      trace[4 * s + 2] = us;
      trace[4 * s + 3] = np;
    }
    if (s == nsteps) break;
    int far = 0;
#pragma omp parallel for schedule(static) reduction(| : far)
    for (int64_t i = 0; i < n; ++i) {
      double d2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        v[3 * i + d] += 0.5 * dt * F[3 * i + d] / mass;
        double xx = x[3 * i + d] + dt * v[3 * i + d];
        if (per[d]) {
          if (xx >= hi[d]) xx -= L[d];
          else if (xx < lo[d]) xx += L[d];
        }
        x[3 * i + d] = xx;
        double e = md_min_image(xx - xref[3 * i + d], L[d], per[d]);
        d2 += e * e;
      }
      if (d2 > half2) far = 1;
    }
    if (far) {
      md_build(n, x, lo, L, per, rv, &M);
      memcpy(xref, x, sizeof(double) * 3 * (size_t)n);
      builds++;
    }
    md_forces(n, x, L, per, &M, rc, eps, sigma, r_min, F, &u, &us, &np);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < 3 * n; ++i) v[i] += 0.5 * dt * F[i] / mass;
  }
  free(M.start);
  free(M.idx);
  free(M.row_ptr);
  free(M.cols);
  free(F);
  free(xref);
  return builds;
}
