/*
 * pm.h -- C-ABI of the B200-native particle hot path (arXiv 1804.07598, OpenFPM).
 *
 * The calls follow the paper's problem statement for a particle client
 * (Listing 4.1, §4.1): set the domain, box and boundary
 * conditions, place particles (the vector_dist constructor
 * and Init_grid), build the cell list (getCellListSym,
 * PAPER.md:276) and the Verlet list with skin ("Verlet lists
 * [46]"), compute pairwise interactions (applyKernel_in_sym, PAPER.md:278,
 * 319), take velocity-Verlet steps, and map /
 * ghost-exchange (map(), ghost_get<>(); §3.4).
 *
 * Conventions (all entry points):
 *  - Every call returns pm_status: PM_OK (0) or a negative error.  No C++
 *    exception crosses the ABI.  The message of the last error is
 *    pm_last_error(ctx).  Errors are sticky per context until pm_place.
 *  - A pm_ctx is bound to one CUDA device and one CUDA stream, and must be
 *    used from one host thread at a time.
 *  - Particle arrays: pos4/vel4/force4 are n x 4 float32 (x, y, z, pad),
 *    16-byte aligned; gid int64[n]; kind int32[n] (0 = fluid / LJ particle,
 *    1 = fixed boundary particle); rho/pres float32[n].
 *  - Memory: `mem` = PM_HOST (pageable or pinned host pointers) or PM_DEVICE
 *    (device pointers on the context's device).  Inputs are copied (stream
 *    ordered on the context stream) before the call returns for PM_HOST, and
 *    before any later work on the stream for PM_DEVICE; the caller may reuse
 *    them after that.  The library owns all its device memory.
 *  - Getters synchronise the context stream and write caller-owned buffers.
 *    Particle arrays are returned in the library's current internal order
 *    (cell order after a build); gid tells the identity of each row.
 *  - Radii use strict inequality: a pair is in a list iff d2 < r^2 where d2 is
 *    the pinned fp32 squared distance of DESIGN.md reading R4 (periodic
 *    minimum image by the Sterbenz-ordered rule).
 */
#ifndef PM_H
#define PM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pm_ctx_s *pm_ctx;
typedef int32_t pm_status;

enum {
  PM_OK = 0,
  PM_E_INVAL = -1,      /* bad argument / usage error (message says which) */
  PM_E_STATE = -2,      /* call out of order (e.g. forces before a list exists) */
  PM_E_NOMEM = -3,      /* device allocation failed */
  PM_E_CUDA = -4,       /* CUDA runtime error */
  PM_E_NCCL = -5,       /* communicator error */
  PM_E_DOMAIN = -6,     /* particle outside [lo,hi) on a NON-periodic axis */
  PM_E_COINCIDENT = -7, /* pair at distance 0 (LJ undefined) */
  PM_E_NONFINITE = -8,  /* non-finite force / density */
  PM_E_CAPACITY = -9    /* neighbour capacity overflow survived realloc + retry */
};

enum { PM_HOST = 0, PM_DEVICE = 1 };

typedef struct {
  int32_t device;      /* CUDA device ordinal */
  int32_t cell_div;    /* cells per r_v along each axis (reading R2): 1 (side >= r_v,
                          27-cell stencil) or 2 (side >= r_v/2, 125-cell stencil;
                          single-GPU contexts); PM_E_INVAL otherwise */
  int32_t nbr_cap;     /* initial neighbour slots per particle (0 = auto from density) */
  int32_t use_graphs;  /* 1: pm_step_vv, pm_sph_run and pm_dem_run run each step as
                          one CUDA graph launch (rebuild as a conditional node, no
                          host round trip per step); 0: plain launches, one host
                          read of the rebuild flag per step (PM_USE_GRAPHS=0 in the
                          environment sets the default to 0: profiling) */
  void *cuda_stream;   /* cudaStream_t to run on; NULL = library-owned stream */
} pm_opts;

/* Fills defaults: device 0, cell_div 1, nbr_cap 0, use_graphs 1, NULL stream. */
pm_status pm_opts_default(pm_opts *opts);
/* Library identification string (static storage). */
const char *pm_version(void);

pm_status pm_create(const pm_opts *opts, pm_ctx *out);
void pm_destroy(pm_ctx ctx);
const char *pm_last_error(pm_ctx ctx);

/* Simulation box [lo, hi) per axis; periodic[d] != 0 for a periodic axis
 * ("Box<3,float> box(...)", "size_t bc[3] = {PERIODIC,...}").
 * Errors: PM_E_INVAL if hi <= lo. */
pm_status pm_set_domain(pm_ctx ctx, const float lo[3], const float hi[3],
                        const int32_t periodic[3]);

/* Interaction radius r_cut and Verlet skin; the list radius is
 * r_v = fl32(r_cut + skin) (reading R5).  PAPER.md:240 "Ghost<3,float>
 * ghost(r_cut)"; the skin is BASELINE.json configs[0..2] (0.3 sigma).
 * Errors: PM_E_INVAL if r_cut <= 0, skin < 0, or a periodic extent is shorter
 * than 3 r_v (the 27-cell stencil needs >= 3 distinct cells per axis). */
pm_status pm_set_cutoff(pm_ctx ctx, float r_cut, float skin);

/* Lennard-Jones parameters: V = 4 eps [(s/r)^12 - (s/r)^6];
 * mass of every particle.  flags: PM_LJ_CAPPED selects the capped force of
 * reading R22 (r_eff = max(r, r_min), BASELINE.json configs[4]); without it
 * r_min must be 0 (the plain potential).  Errors: PM_E_INVAL for eps, sigma or
 * mass <= 0, unknown flags, PM_LJ_CAPPED with r_min <= 0, or r_min != 0
 * without PM_LJ_CAPPED. */
enum { PM_LJ_CAPPED = 1 };
pm_status pm_set_lj(pm_ctx ctx, float epsilon, float sigma, float mass, int32_t flags,
                    float r_min);

/* Half (Newton) neighbour lists, SURVEY §8(f) NEXT-1 ("compute
 * every interaction pair only once"; the symmetric cell/Verlet lists of
 * getCellListSym).  on = 1: each row keeps only j > i in the
 * current (cell) order, the force sweep adds f (x_i - x_j) to F_i and
 * f (x_j - x_i) to F_j with vectorised global reductions, and the
 * velocity-Verlet update runs as a separate kernel; forces, energies and the
 * virial agree with the full list up to summation order (not bit-
 * reproducible run to run).  The lists are rebuilt at the next call that
 * needs them.  LJ only: SPH and DEM return PM_E_STATE with half lists;
 * decomposed contexts step them with the NEWTON_* phases and
 * pm_dist_ghost_put_*.  Default 0 (full lists: atomic-free, deterministic). */
pm_status pm_set_newton(pm_ctx ctx, int32_t on);

/* Velocity limit of reading R22 (clustered BASELINE.json configs[4]): after
 * every kick, v <- v * min(1, vmax / |v|), so no particle drifts more than
 * vmax * dt per step.  vmax = 0 (default) disables the limit. */
pm_status pm_set_vlimit(pm_ctx ctx, float vmax);

/* WCSPH parameters (Eqs. 1, 3-5; readings R15-R21):
 * smoothing length h (kernel support 2h), particle mass, rest density rho0,
 * EOS exponent gamma and constant b (Eq. 3), viscosity alpha, cbar and
 * eta2 (Eq. 5), gravity g. */
typedef struct {
  float h, mass, rho0, gamma, b, alpha, cbar, eta2;
  float g[3];
} pm_sph_params;
pm_status pm_set_sph(pm_ctx ctx, const pm_sph_params *p);

/* DEM parameters (§4.5 Eqs. 9-13;
 * readings R29-R33): particle radius R, mass m, moment of inertia I,
 * normal/tangential elastic constants kn, kt (Eqs. 11-12), damping gamma_n,
 * gamma_t, Coulomb coefficient mu, gravity g, and plane walls at the box
 * faces (flags x-lo, x-hi, y-lo, y-hi, z-lo, z-hi; only on non-periodic
 * axes).  Contacts come from the Verlet list: set r_cut = 2R and a skin. */
typedef struct {
  float R, m, I, kn, kt, gamma_n, gamma_t, mu;
  float g[3];
  int32_t walls[6];
} pm_dem_params;
pm_status pm_set_dem(pm_ctx ctx, const pm_dem_params *p);

/* nsteps DEM steps of size dt: Hertzian normal force with damping (Eq. 11),
 * tangential spring with per-contact history (Eq. 10) and damping (Eq. 12),
 * Coulomb cap, torques, walls, gravity; leapfrog (Eq. 13) for velocity,
 * position and angular velocity.  Angular velocities start at 0 at
 * pm_place.  The contact histories follow the particles through Verlet
 * rebuilds (matched by gid).  Errors: PM_E_DOMAIN (a particle left an open
 * axis), PM_E_NONFINITE.  rebuilds may be NULL. */
pm_status pm_dem_run(pm_ctx ctx, float dt, int64_t nsteps, int64_t *rebuilds);

/* Angular velocities and torques (n x 4 floats each, current internal order
 * as pm_get_state); either may be NULL. */
pm_status pm_get_dem(pm_ctx ctx, float *omega4, float *torque4);

/* Place n particles (replaces any previous set).  pos4 required; vel4, gid,
 * kind may be NULL (zero velocity, gid = 0..n-1, kind = 0).  Positions on
 * periodic axes are wrapped (reading R1) at the next build.  Grows device
 * buffers as needed (PM_E_NOMEM).  Clears a sticky error. */
pm_status pm_place(pm_ctx ctx, int64_t n, const float *pos4, const float *vel4,
                   const int64_t *gid, const int32_t *kind, int32_t mem);

/* Cell list ("Cell Lists [45]"): wrap, cell
 * id, count, exclusive scan, stable reorder of all particle arrays into cell
 * order (PAPER.md:128 cache-friendly re-ordering).  PM_E_STATE without
 * domain / cutoff / particles; PM_E_DOMAIN for a particle outside a
 * non-periodic axis. */
pm_status pm_build_cells(pm_ctx ctx);

/* Verlet list with skin ("Verlet lists [46]"): for every
 * particle, all j != i with d2 < r_v^2 over the 27-cell stencil.  Builds the
 * cell list first.  Grows the neighbour capacity and retries once on
 * overflow (else PM_E_CAPACITY); PM_E_COINCIDENT for a pair at distance 0. */
pm_status pm_build_verlet(pm_ctx ctx);

/* LJ forces over the Verlet list (pairs with d2 < r_cut^2; PAPER.md:162,
 * 203-214; reading R7 for the force expression), written to the force array.
 * want_energy != 0 also accumulates fp64 potential energy, virial and pair
 * count (pm_get_thermo).  PM_E_STATE without a list. */
pm_status pm_compute_lj(pm_ctx ctx, int32_t want_energy);

/* SPH density summation + Tait EOS (Eqs. 3-4, reading R16) for every
 * particle; then pressure + viscous acceleration (Eqs. 1, 5) for fluid
 * particles (kind 0; kind 1 gets 0), written to the force array.  Need a
 * Verlet list built with r_cut = 2h. */
pm_status pm_sph_density(pm_ctx ctx);
pm_status pm_sph_forces(pm_ctx ctx);

/* WCSPH time stepping (Eq. 2 continuity
 * density, :358 "Verlet time-stepping [46] with dynamic step size" as in
 * DualSPHysics; readings R26-R28 in DESIGN.md).  nsteps steps of:
 *   D_p = sum_q m v_pq . grad_p W (all particles), a_p = Eq. 1 + g (fluid),
 *   dt  = cfl * min( min_fluid sqrt(h/|a_p|), min_p h/(c0 + max_q |mu_pq|) ),
 *   Verlet: v' = v_prev + 2 dt a, rho' = rho_prev + 2 dt D (an Euler step
 *   v' = v + dt a, rho' = rho + dt D on the first and every `every`-th
 *   step), x' = x + dt v + dt^2/2 a for fluid; boundary particles (kind 1)
 *   keep x and v, their density evolves; P' = Tait EOS (Eq. 3).
 * The densities at the start are the current ones (pm_sph_density is run
 * first if they are not valid); the Verlet list (r_cut = 2h, skin > 0) is
 * rebuilt whenever a particle moved more than skin/2 or left an open axis.
 * Single context only (PM_E_STATE on a decomposed context).  Errors:
 * PM_E_NONFINITE (rates or dt), PM_E_DOMAIN (a fluid particle left an open
 * axis).  out may be NULL. */
/* Set the SPH densities (n floats, in the CURRENT internal order -- the order
 * pm_get_state returns) and their pressures by the Tait EOS (Eq. 3); e.g. a
 * hydrostatic initial profile for pm_sph_run.  mem: PM_HOST / PM_DEVICE. */
pm_status pm_set_rho(pm_ctx ctx, const float *rho, int32_t mem);

typedef struct {
  int64_t steps;     /* steps completed */
  int64_t rebuilds;  /* Verlet rebuilds during the call */
  double time;       /* simulated time of the call */
  float dt_min, dt_max, dt_last;
} pm_sph_run_stats;
pm_status pm_sph_run(pm_ctx ctx, int64_t nsteps, float cfl, int32_t every,
                     pm_sph_run_stats *out);

typedef struct {
  int64_t steps;     /* steps completed by this call */
  int64_t rebuilds;  /* Verlet rebuilds during this call */
  int32_t max_row;   /* longest neighbour row at the last build */
  int32_t nbr_cap;   /* current neighbour capacity per row */
  double mean_row;   /* mean neighbour row length at the last build */
} pm_run_stats;

/* nsteps velocity-Verlet steps, with
 * the Verlet list rebuilt on the device whenever the largest displacement
 * since the last build exceeds skin/2 (BASELINE.json configs[1]).  Forces are
 * computed first if they are not valid.  out may be NULL. */
pm_status pm_step_vv(pm_ctx ctx, float dt, int64_t nsteps, pm_run_stats *out);

/* Counts: owned and ghost particles, cells, neighbour entries of the last
 * build.  Any pointer may be NULL. */
pm_status pm_count(pm_ctx ctx, int64_t *n_owned, int64_t *n_ghost, int64_t *n_cells,
                   int64_t *nnz);

/* Cell list of the last build: cell_of[n] in the storage order the build
 * started from, cell_start[ncell+1], perm[n] (k-th particle in cell order =
 * storage index perm[k]; ties in storage order).  Any pointer may be NULL. */
pm_status pm_get_cells(pm_ctx ctx, int32_t *cell_of, int32_t *cell_start, int32_t *perm);

/* Verlet list of the last build in CSR over the current internal order:
 * row_ptr[n_owned+n_ghost+1] (ghost rows are empty), col_gid[nnz] (gid of each
 * neighbour).  Caller-allocated. */
pm_status pm_get_verlet(pm_ctx ctx, int64_t *row_ptr, int64_t *col_gid);

/* Image shift of every entry of pm_get_verlet's CSR (same order): col_shift
 * [3 * nnz] int8, per axis -1 when the R4 rule moved the partner by -L,
 * +1 when it moved this particle by -L (partner seen at +L), 0 otherwise
 * (positions of the last build).  With periodic extents >= 3 r_v a pair has
 * at most one image, so (gid_i, gid_j, shift) is the list's complete set
 * description.  Caller-allocated. */
pm_status pm_get_verlet_shifts(pm_ctx ctx, int8_t *col_shift);

/* Particle state in the current internal order.  Any pointer may be NULL.
 * force4 holds LJ forces or SPH accelerations (last computed); rho/pres the
 * SPH density and pressure.  The fourth components of pos4/vel4 are carried,
 * not computed: after pm_sph_forces and pm_sph_run they hold the pressure and
 * the density the SPH sweeps gather with the positions and velocities. */
pm_status pm_get_state(pm_ctx ctx, float *pos4, float *vel4, float *force4, int64_t *gid,
                       float *rho, float *pres, int32_t mem);

/* kind[n_owned + n_ghost] in the current internal order (bit 30 marks a ghost
 * copy on a decomposed context; bit 0: fixed SPH boundary particle). */
pm_status pm_get_kind(pm_ctx ctx, int32_t *kind);

/* Thermodynamics (fp64 reductions on the device): kinetic energy of the
 * current velocities; potential energy raw and shifted by V(r_cut) per pair
 * (reading R9), virial and pair count of the last energy pass
 * (pm_compute_lj with want_energy, or pm_thermo_compute). */
pm_status pm_get_thermo(pm_ctx ctx, double *ke, double *pe_raw, double *pe_shift,
                        double *virial, int64_t *npairs);
/* Recompute the LJ energy of the current positions (list must be valid). */
pm_status pm_thermo_compute(pm_ctx ctx);

/* Profiling: when on, pm_step_vv records CUDA events around every force
 * kernel and every rebuild; pm_get_profile returns summed device times (ms)
 * and launch counts since the last reset. */
pm_status pm_set_profiling(pm_ctx ctx, int32_t on);
pm_status pm_get_profile(pm_ctx ctx, double *force_ms, int64_t *force_launches,
                         double *step_ms, int64_t *steps);

/* ------------------------------------------------------------------------
 * Multi-GPU: spatial decomposition.  PAPER.md:62 (§3.1):
 * "sub-domains are extended by a ghost layer ... given by the particle
 * interaction radius"; PAPER.md:112-118 (§3.4): map() migrates particles that
 * crossed sub-domain boundaries to the neighbour owning them, ghost_get()
 * populates the ghost layers, optionally with a subset of properties (the
 * per-step refresh moves positions only, Listing 4.1 ghost_get<>()).
 *
 * One context per GPU owns one cuboid of the global periodic box set with
 * pm_set_domain.  The library builds, packs and unpacks the messages; the
 * caller moves the bytes (NCCL through torch.distributed, or an in-process
 * copy) and exchanges the counts.  Direction index of a neighbour cuboid:
 * d = (ax+1) + 3 (ay+1) + 9 (az+1) with a in {-1, 0, 1}; d = 13 is "self".
 * Ghost copies keep the owner's wrapped global coordinates (never shifted
 * copies): pair distances use the global-box rule R4, so a pair's d2 is the
 * same whether the partner is a ghost or a local periodic image.
 * ---------------------------------------------------------------------- */
enum {
  PM_MSG_MIGRATE = 0,
  PM_MSG_GHOST = 1,
  PM_MSG_REFRESH = 2,
  PM_MSG_REFRESH_PV = 3,   /* SPH runs: position + velocity */
  PM_MSG_REFRESH_PVW = 4,  /* DEM runs: position + velocity + angular velocity */
  PM_MSG_MIGRATE_HIST = 5  /* DEM runs: contact histories of the migrating grains */
};
enum {
  PM_PHASE_PROLOGUE = 0,
  PM_PHASE_STEP = 1,
  PM_PHASE_FINAL = 2,
  PM_PHASE_FORCES = 3,
  PM_PHASE_NEWTON_FORCES = 4,  /* half lists: F = 0, sweep (ghost shares stay on the ghosts) */
  PM_PHASE_NEWTON_STEP = 5,    /* half lists, after pm_dist_ghost_put: kick / drift */
  PM_PHASE_NEWTON_FINAL = 6    /* ... last half kick, forces kept */
};

/* Bytes per message record: migrate 64 (pos, vel, SPH previous-step velocity
 * or DEM angular velocity, gid, kind), ghost 32 (pos, gid, kind), refresh 16
 * (pos), refresh with velocities 32 (pos, vel; SPH runs), refresh with
 * angular velocities 48 (DEM runs), migrating contact histories 592 (gid,
 * count, up to 24 (partner gid, u_t) pairs).  Returns -1 for an unknown kind. */
int32_t pm_record_bytes(int32_t what);

/* This context owns cuboid pcoord of a pgrid[0] x pgrid[1] x pgrid[2]
 * decomposition of the (periodic) domain.  Call after pm_set_domain and
 * pm_set_cutoff, before pm_place.  The ghost width is r_v = r_cut + skin.
 * Errors: PM_E_INVAL if a decomposed axis is not periodic or a sub-domain is
 * thinner than 2 r_v. */
pm_status pm_set_decomposition(pm_ctx ctx, const int32_t pgrid[3], const int32_t pcoord[3]);

/* The same with load-balanced (non-uniform) cuboids (
 * PAPER.md:122, §3.5 dynamic load balancing): cuts holds the interior cut
 * positions of axis x (pgrid[0]-1 floats, increasing), then y, then z; a
 * particle belongs to slab c = #{k : x >= cut_k} along each axis (exact fp32
 * compares).  The cuts are a tensor product, so neighbours stay the 26 grid
 * directions.  Errors: PM_E_INVAL for more than 15 cuts per axis, cuts not
 * increasing inside the box, or a slab thinner than 2 r_v. */
pm_status pm_set_decomposition_cuts(pm_ctx ctx, const int32_t pgrid[3], const int32_t pcoord[3],
                                    const float *cuts);

/* Build the outgoing message lists of kind `what` (MIGRATE: owned particles
 * whose owner changed -- counts[13] = particles that stay; GHOST: owned
 * particles within r_v of each neighbour face/edge/corner, up to 7 copies).
 * Lists are stable (ascending local index) and laid out in the direction
 * order order[0..25] (all d != 13).  counts[27] receives records per
 * direction.  Synchronises. */
pm_status pm_dist_plan(pm_ctx ctx, int32_t what, const int32_t order[26], int64_t counts[27]);

/* Write the planned records, in list order, to the device buffer send_dev
 * (>= sum of counts * pm_record_bytes(what) bytes).  For MIGRATE this also
 * removes the leavers (stable compaction of the stayers) and drops all ghosts;
 * for GHOST it keeps the list for the per-step refresh. */
pm_status pm_dist_pack(pm_ctx ctx, int32_t what, void *send_dev);

/* Append nrecv records from the device buffer recv_dev: MIGRATE arrivals
 * become owned particles, GHOST records become ghosts (kind bit 30 set).
 * Grows buffers as needed (PM_E_NOMEM). */
pm_status pm_dist_unpack(pm_ctx ctx, int32_t what, const void *recv_dev, int64_t nrecv);

/* After migration and the ghost exchange: cell list over owned + ghosts, the
 * refresh lists remapped to cell order, Verlet rows for owned particles. */
pm_status pm_dist_finish(pm_ctx ctx);

/* Per-step positions-only ghost refresh: pack the current positions of the
 * last GHOST plan's list (16 B each, same order), unpack the received ones
 * into this context's ghost copies. */
pm_status pm_dist_refresh_pack(pm_ctx ctx, void *send_dev);
pm_status pm_dist_refresh_unpack(pm_ctx ctx, const void *recv_dev);

/* One phase of a decomposed velocity-Verlet run (owned particles only):
 * PROLOGUE = v += dt/2 F/m, x += dt v, wrap (from stored forces); STEP =
 * forces, then the fused kick / drift (as in pm_step_vv); FINAL = forces and
 * the last half kick, forces stored; FORCES = forces only.  need_rebuild
 * (nullable): synchronise and return (and clear) the local flag "some owned
 * particle moved more than skin/2 since the last build". */
pm_status pm_dist_step(pm_ctx ctx, float dt, int32_t phase, int32_t *need_rebuild);

/* Fused ghost refresh (SURVEY §8(e) "the K6 epilogue ... stores straight into
 * peer windows"): after a rebuild, each sub-domain registers, for every entry
 * of its ghost send list (pm_dist_plan(GHOST) order), the receiving peer
 * (index into the peer tables) and the receiver's ghost slot (the receiver's
 * pm_dist_ghost_slots, in its arrival order), plus each peer's two position
 * buffers (pm_dist_pos_buffers; across processes opened through CUDA IPC:
 * pm_dist_ipc_handles / pm_dist_ipc_open).  PM_PHASE_STEP of pm_dist_step
 * then writes every new position of a sent particle into the peers' next
 * position buffer from the sweep's epilogue (no pack, no message, no
 * unpack); the caller only orders the step before the peers' next step (the
 * per-step flag all-reduce).  pm_dist_finish disables it until the next
 * setup; npeers = 0 disables it.  dst_peer / dst_slot: device int32[n_send]. */
pm_status pm_dist_pos_buffers(pm_ctx ctx, void **pos0, void **pos1);
pm_status pm_dist_ghost_slots(pm_ctx ctx, int32_t *dev_out);
pm_status pm_dist_peer_setup(pm_ctx ctx, int32_t npeers, void *const *peer_pos0,
                             void *const *peer_pos1, const int32_t *dst_peer,
                             const int32_t *dst_slot);
/* 128 bytes: CUDA IPC handles of this context's two position buffers. */
pm_status pm_dist_ipc_handles(pm_ctx ctx, void *out);
pm_status pm_dist_ipc_open(pm_ctx ctx, const void *in, void **pos0, void **pos1);
pm_status pm_dist_ipc_close_all(pm_ctx ctx);

/* Synchronise and return (and clear) the local rebuild flag -- the
 * need_rebuild of pm_dist_step as a separate call, so a caller can time the
 * step kernels with events before the host round trip. */
pm_status pm_dist_read_flag(pm_ctx ctx, int32_t *need_rebuild);

/* Half (Newton) lists on a decomposed context (SURVEY §8(f) NEXT-1 with its
 * reverse exchange; PAPER.md:116 ghost_put, :164 "compute every interaction
 * pair only once"): rows keep owned partners later in the local order and
 * ghost partners with a larger gid, so every pair -- also across a
 * sub-domain face -- is computed on exactly one rank.  A step:
 * pm_dist_step(NEWTON_FORCES) -> ghost_put (pack the shares accumulated on
 * the ghost copies, 16 B each in arrival order, send them back to the owners
 * with the ghost round's counts reversed, add them there) ->
 * pm_dist_step(NEWTON_STEP or NEWTON_FINAL). */
pm_status pm_dist_ghost_put_pack(pm_ctx ctx, void *send_dev);
pm_status pm_dist_ghost_put_unpack(pm_ctx ctx, const void *recv_dev);

/* Decomposed DEM (SURVEY §8(f) NEXT-4 on the §8(e) decomposition; PAPER.md:
 * 479 "collisions involving ghost particles need to be properly accounted for
 * in the lists of the respective source particles", §4.5).  Each owner keeps
 * the tangential history of its own ordered pairs, ghost partners included,
 * so between rebuilds nothing but the ghosts' x, v, omega travels
 * (pm_dist_refresh_pvw_*, 48 B per ghost).  At a rebuild:
 *   pm_dist_plan(MIGRATE) also saves every local row with its histories and
 *   partner gids; pm_dist_pack(PM_MSG_MIGRATE_HIST) BEFORE pm_dist_pack
 *   (MIGRATE) writes each leaver's nonzero histories as (partner gid, u_t)
 *   pairs (same list and order as MIGRATE: the caller ships both with the
 *   same counts); pm_dist_unpack(MIGRATE_HIST) after pm_dist_unpack(MIGRATE);
 *   pm_dist_finish carries every history onto the new rows by partner gid.
 * A grain with more than 24 live contacts at a migration raises
 * PM_E_CAPACITY.  Walls apply on non-decomposed axes only (decomposed axes
 * are periodic).  pm_dist_dem_init after pm_set_dem, before the first
 * rebuild; pm_dist_dem_step = contacts + leapfrog of the owned grains
 * (ghosts carried), need_rebuild as pm_dist_step. */
pm_status pm_dist_dem_init(pm_ctx ctx);
pm_status pm_dist_dem_step(pm_ctx ctx, float dt, int32_t *need_rebuild);
pm_status pm_dist_refresh_pvw_pack(pm_ctx ctx, void *send_dev);
pm_status pm_dist_refresh_pvw_unpack(pm_ctx ctx, const void *recv_dev);

/* Decomposed WCSPH time stepping (SURVEY §8(f) NEXT-3 "multi-GPU SPH ghosts
 * (vel/rho/P)"; PAPER.md:335 Eq. 2, :358 Verlet scheme with dynamic step
 * size; the per-step operations of pm_sph_run, readings R26-R28).  Per step
 * every rank calls
 *   pm_dist_sph_rates  -> its local step bound (synchronises);
 *   the caller reduces the bounds to their global minimum over all ranks;
 *   pm_dist_sph_update(bound) -> dt = cfl * bound, Verlet / Euler update of
 *                        the owned particles; need_rebuild as pm_dist_step;
 *   a rebuild (MIGRATE, GHOST rounds + pm_dist_finish) when any rank asks;
 *   the ghost refresh with velocities (pm_dist_refresh_pv_*: 32 B per ghost,
 *   position and velocity whose w lanes carry P and rho).
 * pm_dist_sph_init (after pm_set_sph and the initial densities, pm_set_rho,
 * before the first rebuild) packs rho and P into the velocity and position w
 * lanes and starts the Verlet state; migration records carry it.  Ghost
 * copies have no row, no rate and no step bound.  Decomposed axes must be
 * periodic (pm_set_decomposition). */
pm_status pm_dist_sph_init(pm_ctx ctx);
pm_status pm_dist_sph_rates(pm_ctx ctx, float *bound);
pm_status pm_dist_sph_update(pm_ctx ctx, float bound, float cfl, int32_t every,
                             int32_t *need_rebuild);
pm_status pm_dist_refresh_pv_pack(pm_ctx ctx, void *send_dev);
pm_status pm_dist_refresh_pv_unpack(pm_ctx ctx, const void *recv_dev);

/* ---------------------------------------------------------------------------
 * Multi-GPU groups: map() and ghost_get<>() behind the ABI (SURVEY §8(b),
 * §8(e); §3.1 sub-domains with a ghost layer of interaction
 * width; §3.4 map / ghost_get "only communicate"; Listing
 * 4.1 map() and ghost_get<>() at PAPER.md:299-303).
 *
 * A group is one px x py x pz cuboid decomposition of the periodic box (as
 * pm_set_decomposition); each member context owns one sub-domain, index
 * cx + px (cy + py cz).  Members are created by pm_create_dist (one per
 * process and GPU, a library-owned NCCL communicator; nranks = px py pz) or
 * pm_create_dist_local (all sub-domains in this process on one GPU: the
 * in-process loopback group, messages as device copies -- or through NCCL
 * self-communication with via_nccl = 1, to exercise the NCCL path on one
 * GPU).  Every member is then set up as a plain context: pm_set_domain,
 * pm_set_cutoff, pm_set_lj, pm_place (any particles: map sends them to their
 * owners; the decomposition is applied at the first pm_map).  Decomposed axes
 * must be periodic and sub-domains at least 2 r_v thick (PM_E_INVAL).
 *
 * Collective calls: every member calls them, in the same order; the call of
 * the LAST local member does the work for all local members (so one host
 * thread drives a loopback group member by member) and writes the outputs;
 * earlier members' calls return PM_OK without touching their outputs.
 * Members of one process share one CUDA stream (opts.cuda_stream, or a
 * group-owned stream) on which NCCL is called.  Errors: PM_E_NCCL when NCCL
 * cannot be loaded or a communicator call fails; PM_E_STATE when members call
 * different collectives.  pm_destroy of the last member frees the group and
 * its communicator. */

/* 128 bytes of an NCCL unique id (rank 0 creates it and broadcasts it, e.g.
 * with torch.distributed.broadcast_object_list). */
pm_status pm_nccl_unique_id(uint8_t id[128]);

/* The member of rank `rank` (its sub-domain index) of an nranks-process group
 * with decomposition grid[3] (grid[0] grid[1] grid[2] == nranks); initialises
 * the group's NCCL communicator (ncclCommInitRank, collective over ranks). */
pm_status pm_create_dist(const pm_opts *opts, int32_t rank, int32_t nranks, const uint8_t id[128],
                         const int32_t grid[3], pm_ctx *out);

/* All grid[0] grid[1] grid[2] members in this process: out[sub-domain]. */
pm_status pm_create_dist_local(const pm_opts *opts, const int32_t grid[3], int32_t via_nccl,
                               pm_ctx *out);

/* This member's sub-domain, the number of sub-domains, its rank and the
 * number of ranks.  PM_E_STATE for a context that is not a group member. */
pm_status pm_dist_info(pm_ctx ctx, int32_t *sub_domain, int32_t *nsub, int32_t *rank,
                       int32_t *nranks);

/* map() (collective): every owned particle outside its sub-domain moves to
 * the owner (64-byte records, ghosts dropped).  Synchronises (counts). */
pm_status pm_map(pm_ctx ctx);

/* ghost_get<>() (collective): ghost copies of every owned particle within r_v
 * of a neighbour's face, edge or corner (32-byte records), then each member's
 * cell list over owned + ghosts and Verlet rows of its owned particles. */
pm_status pm_ghost_get(pm_ctx ctx);

/* nsteps velocity-Verlet steps of the whole group (collective): per step the
 * positions-only ghost refresh (16 B per ghost), the fused force sweep and
 * kick/drift of every member, and the global rebuild flag (MAX all-reduce on
 * the device); when any particle moved more than skin/2, pm_map +
 * pm_ghost_get.  Steps are enqueued in batches (env PM_GROUP_BATCH, default
 * 4) with one host synchronisation per batch: kernels of steps after a set
 * flag do nothing.  Forces are computed first when not valid.  out: steps and
 * rebuilds (performer).  Errors: PM_E_STATE when members call different
 * collectives; device errors of any member (PM_E_NONFINITE, ...). */
pm_status pm_dist_run(pm_ctx ctx, float dt, int64_t nsteps, pm_run_stats *out);

/* Global (all sub-domains) kinetic energy, raw and shifted LJ energy, virial
 * and ordered pair count (collective; recomputes the energy pass). */
pm_status pm_dist_thermo(pm_ctx ctx, double *ke, double *pe_raw, double *pe_shift,
                         double *virial, int64_t *npairs);

#ifdef __cplusplus
}
#endif

#endif /* PM_H */
