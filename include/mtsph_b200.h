/*
 * mtsph_b200.h -- C ABI of the B200-native multi-rate SPH hot path.
 *
 * Shared library: paper_2309_04010_b200/libmtsph_b200.so (sm_100a).
 * Plain pointers and sizes only; no torch types.  All functions return an
 * mtsph_status (0 = ok); on failure mtsph_last_error() holds a message and
 * mtsph_last_error_ids() the offending particle ids (original numbering),
 * mirroring the reference's error classes (errors.py).
 *
 * Two layers:
 *
 *  1. Drop-in replacements for the reference's compiled particle loops
 *     (/root/reference/pkg/src/mtsph/_accel.py).  Same argument meaning and
 *     array layout as the numba kernels (numpy C order, int64 CSR), HOST
 *     pointers; each call stages to HBM, runs the sm_100a kernel and copies
 *     the result back.  These are what a ctypes shim for `mtsph._accel`
 *     binds.
 *
 *  2. Device-resident problems (neighbourhood, necking solid, porous
 *     membrane) whose state stays in HBM for the whole run; one call runs
 *     a complete inner relaxation loop (scenarios.py relax_step repeated
 *     under stepping.py:158's kinetic-energy criterion) without host
 *     round trips.  These back the drop-in Problem objects of the Python
 *     package (paper_2309_04010_b200.scenarios).
 */
#ifndef MTSPH_B200_H
#define MTSPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTSPH_ABI_VERSION 1

typedef int mtsph_status;
enum {
    MTSPH_OK = 0,
    MTSPH_ERR_ARG = 1,          /* bad argument / unsupported dimension      */
    MTSPH_ERR_CUDA = 2,         /* CUDA runtime failure or no device         */
    MTSPH_ERR_GEOMETRY = 3,     /* errors.py:12  GeometryError               */
    MTSPH_ERR_SINGULAR = 4,     /* errors.py:16  SingularMomentMatrixError   */
    MTSPH_ERR_INVERSION = 5,    /* errors.py:29  ElementInversionError       */
    MTSPH_ERR_RETURN_MAP = 6,   /* errors.py:41  ReturnMapError              */
    MTSPH_ERR_NONFINITE = 7,    /* errors.py:54  SimulationError             */
};

int mtsph_abi_version(void);
const char *mtsph_last_error(void);
/* copies up to cap ids of the last failure; returns how many there were */
int64_t mtsph_last_error_ids(int64_t *ids, int64_t cap);
/* number of CUDA devices visible (0 on a CPU-only host) */
int mtsph_device_count(void);
/* select the GPU new problems (and their streams) are created on; one
 * process per GPU calls it with its local rank before creating any      */
mtsph_status mtsph_set_device(int ordinal);

/* ------------------------------------------------------------------ */
/* Layer 1: _accel.py drop-ins (host pointers, reference layout)       */
/* ------------------------------------------------------------------ */

/* _accel.py:16  out[a] = sum_b vol[b] (src[b]-src[a]) (x) grad_ab        */
mtsph_status mtsph_velocity_gradient_gather(
    int64_t n, int d, const double *src, const int64_t *indptr,
    const int64_t *idx, const double *grad, const double *vol, double *out);

/* _accel.py:34  out[a] = sum_b vol[b] (tens[a]+tens[b]) . grad_ab        */
mtsph_status mtsph_pair_tensor_divergence(
    int64_t n, int d, const double *tens, const int64_t *indptr,
    const int64_t *idx, const double *grad, const double *vol, double *out);

/* _accel.py:52  out[a] += sum_b vol[b] (tens[a]+tens[b]) . (amap[a] grad) */
mtsph_status mtsph_pair_tensor_divergence_mapped(
    int64_t n, int d, const double *tens, const double *amap,
    const int64_t *indptr, const int64_t *idx, const double *grad,
    const double *vol, double *out);

/* _accel.py:76  out[a] = coeff[a] sum_b vol[b] (sat[a]-sat[b]) (amap[a] grad) */
mtsph_status mtsph_scalar_difference_flux(
    int64_t n, int d, const double *sat, const double *coeff,
    const double *amap, const int64_t *indptr, const int64_t *idx,
    const double *vol, const double *grad, double *out);

/* _accel.py:171 sequential pairwise implicit damping sweep, in place.
 * Reproduces the reference's serial group order exactly (level-scheduled
 * on the GPU: groups in one level touch disjoint particles).  The group
 * size limit is the reference's (64 pairs).                             */
mtsph_status mtsph_damping_sweep(
    int64_t n, int d, double *vel, int64_t npairs, const int64_t *pair_i,
    const int64_t *pair_j, const double *pair_damp, const double *inv_mass_i,
    const double *inv_mass_j, int64_t ngroups, const int64_t *group_ptr,
    double eta, double dt);

/* _accel.py:210 antisymmetric flux-divergence mass rate                  */
mtsph_status mtsph_conservative_mass_rate(
    int64_t n, int d, const double *flux, const double *amap, int64_t npairs,
    const int64_t *pair_i, const int64_t *pair_j, const double *pair_grad,
    const double *vol, double *out);

/* _accel.py:240 fused mixture-stress momentum RHS                        */
mtsph_status mtsph_porous_stress_rhs(
    int64_t n, int d, const double *def_grad, const double *pressure,
    const double *corr, const int64_t *indptr, const int64_t *idx,
    const double *grad0, const double *vol0, double mu, double lam,
    double *tbuf, double *out_j, double *out_rate);

/* ------------------------------------------------------------------ */
/* Layer 2: device-resident neighbourhoods and problems                */
/* ------------------------------------------------------------------ */

/* damping-sweep ordering */
enum {
    MTSPH_SWEEP_NONE = 0,      /* no pair schedule (no damping)             */
    MTSPH_SWEEP_SERIAL = 1,    /* the reference's exact serial group order  */
    MTSPH_SWEEP_COLOURED = 2,  /* 3^d-coloured midpoint-cell tasks; keeps the
                                  reference's groups and mirror symmetry   */
    MTSPH_SWEEP_TILED = 3,     /* B200 throughput: 2^d-coloured cell blocks
                                  staged in shared memory, greedy
                                  edge-coloured pairs inside a block       */
};

typedef struct mtsph_nbh mtsph_nbh;

/* neighbors.py:59 + :232.  Builds the fixed reference-configuration
 * neighbourhood on the GPU (cell lists, Morton particle order, SELL-32
 * neighbour table, correction matrices, damping pair schedule).          */
mtsph_status mtsph_nbh_create(int64_t n, int d, const double *pos,
                              const double *vol, const double *h_axes,
                              int sweep, mtsph_nbh **out);
mtsph_status mtsph_nbh_destroy(mtsph_nbh *nb);
/* sizes in the reference's layout (directed CSR entries, unique pairs,
 * damping groups, colours or levels of the sweep schedule)              */
mtsph_status mtsph_nbh_sizes(const mtsph_nbh *nb, int64_t *nnz, int64_t *npairs,
                             int64_t *ngroups, int64_t *nphases);
/* export in the reference layout and numbering (NULL outputs skipped).
 * pair arrays follow the schedule order of the chosen sweep.           */
mtsph_status mtsph_nbh_export(const mtsph_nbh *nb, int64_t *indptr, int64_t *idx,
                              double *grad0, int64_t *pair_i, int64_t *pair_j,
                              double *pair_damp, double *pair_grad,
                              int64_t *pair_group, double *corr);
/* internal (Morton) order: perm[k] = original id of internal particle k  */
mtsph_status mtsph_nbh_permutation(const mtsph_nbh *nb, int64_t *perm);

/* --- necking solid (scenarios.py:41 NeckingProblem) --- */

typedef struct {
    int64_t n;
    int d;
    const double *pos;          /* (n,d) reference positions               */
    const double *vol;          /* (n,)                                     */
    const double *rho0;         /* (n,)                                     */
    const uint8_t *constrained; /* (n,) 1 = velocity prescribed             */
    const int8_t *side;         /* (n,) -1 left clamp, +1 right clamp, 0    */
    const uint8_t *mid_mask;    /* (n,) mid-span section (neck radius)      */
    double h_axes[3];
    double shear_modulus, bulk_modulus;
    int plastic;                /* 0: Neo-Hookean only (solids.py:148)      */
    int hardening_law;          /* 0: reference saturation+linear (plasticity.py:64)
                                   1: power law s0 (1 + a/e0)^m             */
    double hard[4];             /* law 0: s0, sinf, delta, H; law 1: s0, e0, m, - */
    double rm_tol;              /* return-map tolerance (<=0: 1e-8 s0)     */
    int rm_max_iter;            /* 50 in the reference                      */
    int sweep;                  /* MTSPH_SWEEP_*                            */
    /* multi-rank (NULL for a single domain): */
    const uint8_t *ghost;       /* (n,) 1 = halo copy of another rank's particle */
    const double *grid;         /* 6 doubles: global scaled-space bounds lo[3], hi[3]
                                   of the cell grid (X/h), shared by all ranks */
    int tile;                   /* tiled sweep block edge in cells (power of 2);
                                   0: automatic (4, halved until the halo fits
                                   shared memory).  Ranks of one decomposition
                                   must use their partition plan's edge. */
} mtsph_solid_desc;

typedef struct mtsph_solid mtsph_solid;

typedef struct {
    double eta;            /* damping viscosity                           */
    double cfl;            /* 0.6                                          */
    double criterion;      /* absolute kinetic-energy threshold           */
    double dt_outer;       /* for the default cap 10*ceil(dt_outer/dt)   */
    int64_t max_inner;     /* 0 = default cap                              */
    int64_t min_inner;     /* >= 1                                         */
} mtsph_inner_params;

typedef struct {
    int64_t n_inner;       /* relaxation steps taken                      */
    int cap_hit;           /* loop ended on the safety cap                */
    double ek;             /* last pre-damping kinetic energy             */
    double min_dt;         /* smallest inner step used                    */
    double last_dt;
} mtsph_inner_result;

mtsph_status mtsph_solid_create(const mtsph_solid_desc *desc, mtsph_solid **out);
mtsph_status mtsph_solid_destroy(mtsph_solid *s);
/* NeckingProblem.advance_slow: arm the boundary ramp of one outer step  */
mtsph_status mtsph_solid_set_ramp(mtsph_solid *s, double end_disp, int64_t ramp_steps,
                                  int64_t ramp_left);
mtsph_status mtsph_solid_ramp_left(const mtsph_solid *s, int64_t *ramp_left);
/* solids.py:187 stable step                                              */
mtsph_status mtsph_solid_stable_dt(mtsph_solid *s, double cfl, double *dt);
/* one relax_step at a host-chosen dt; returns the pre-damping E_k        */
mtsph_status mtsph_solid_relax_step(mtsph_solid *s, double dt, double eta, double *ek);
/* the whole inner loop on the device (graph-captured chunks)            */
mtsph_status mtsph_solid_relax(mtsph_solid *s, const mtsph_inner_params *p,
                               mtsph_inner_result *r);
/* exactly nsteps inner steps as one CUDA graph with CUDA events captured
 * around every kernel class (benchmark path; the stopping rule is
 * disabled).  timing[0] = device ms of the whole region, timing[1..5] =
 * summed ms of kick/drift, stress, divergence, damping sweep, reductions
 * + control; timing[6] = kernel launches in the region.                 */
mtsph_status mtsph_solid_run_steps(mtsph_solid *s, const mtsph_inner_params *p,
                                   int64_t nsteps, double timing[7]);
/* fp32 variant (the north star's "fp32 variant reported separately"):
 * bits = 32 moves the state to single-precision arrays (displacement,
 * F - I, C_p^-1 - I, velocities, divergence records, sweep coefficients)
 * and runs relax_step / relax / run_steps with the fp32 kernels
 * (csrc/solid32.cuh; the return map stays fp64).  get / set / measure
 * read and write through the fp64 copy.  bits = 64 converts back.  Tiled
 * sweep, single domain only.  No reference counterpart: the reference is
 * fp64 throughout.                                                       */
mtsph_status mtsph_solid_set_precision(mtsph_solid *s, int bits);
mtsph_status mtsph_solid_precision(const mtsph_solid *s, int *bits);
/* --- multi-rank phases (slab decomposition, tiled sweep; the host driver
 * paper_2309_04010_b200/distributed.py exchanges halos between them) --- */
enum {
    MTSPH_PHASE_KICK_DRIFT = 1,  /* v += dt/2 a, boundary, x += dt v (owned)        */
    MTSPH_PHASE_STRESS = 2,      /* dF/dt gather, F update, return map, T (owned)    */
    MTSPH_PHASE_ACCEL = 3,       /* divergence + kick; out[0] = sum m v^2, out[1] = max |a|^2 */
    MTSPH_PHASE_SWEEP = 4,       /* damping, tasks of colour `arg` (forward, or
                                    reverse when arg >= 64: colour arg - 64)       */
    MTSPH_PHASE_VMAX = 5,        /* out[0] = max |v|^2 (owned)                       */
    MTSPH_PHASE_AMAX = 6,        /* out[0] = max |v|^2, out[1] = max |a|^2 (free)    */
    MTSPH_PHASE_SWEEP_ALL = 7,   /* damping, the whole sweep (both passes, every
                                    colour) in one persistent dataflow launch --
                                    only for a rank with no ghosts (world size 1) */
};
/* Device-controlled multi-rank loop (no host synchronisation per phase):
 * phase_async only enqueues a phase on the solid's stream (the reductions
 * stay on the device); rank_partials writes this rank's {sum m v^2,
 * max |a|^2, max |v|^2, error flag} (owned particles) to 4 doubles of
 * device memory; the caller all-gathers them over the ranks (NCCL) into
 * [nranks][4] and control_ranks applies the stopping rule and next step
 * (stepping.py:177-195, solids.py:187) on the device, identically on every
 * rank.  mode 0: initial step size (after the AMAX phase), 1: end of an
 * inner step (after ACCEL ... VMAX).  begin_loop sets the loop parameters
 * as mtsph_solid_relax does; loop_state reads the control block back.    */
mtsph_status mtsph_solid_phase_async(mtsph_solid *s, int phase, int arg);
mtsph_status mtsph_solid_begin_loop(mtsph_solid *s, const mtsph_inner_params *p);
mtsph_status mtsph_solid_rank_partials(mtsph_solid *s, int mode, double *dev_out4);
mtsph_status mtsph_solid_control_ranks(mtsph_solid *s, const double *dev_gathered, int nranks,
                                       int mode);
mtsph_status mtsph_solid_loop_state(mtsph_solid *s, mtsph_inner_result *r, int *done);
/* set the step size and viscosity used by the next phases                */
mtsph_status mtsph_solid_set_step(mtsph_solid *s, double dt, double eta);
mtsph_status mtsph_solid_phase(mtsph_solid *s, int phase, int arg, double out[2]);
/* number of damping colours of the tiled schedule                        */
mtsph_status mtsph_solid_colours(const mtsph_solid *s, int *ncolours);
/* copy a field of the listed particles (ORIGINAL local ids) to / from a
 * packed host buffer: "vel" (d doubles each) or "T" (d*d doubles each)   */
mtsph_status mtsph_solid_pack(mtsph_solid *s, const char *field, int64_t m,
                              const int64_t *ids, double *host);
mtsph_status mtsph_solid_unpack(mtsph_solid *s, const char *field, int64_t m,
                                const int64_t *ids, const double *host);
/* device-resident exchange (NCCL send/recv of device buffers, no host
 * staging).  Map ORIGINAL local ids to the solid's internal ids once, keep
 * them on the device, and pack / unpack between device buffers; both are
 * enqueued on the solid's stream (returned by mtsph_solid_stream, a
 * cudaStream_t) without synchronising the host.                          */
mtsph_status mtsph_solid_internal_ids(mtsph_solid *s, int64_t m, const int64_t *ids,
                                      int64_t *internal);
mtsph_status mtsph_solid_stream(const mtsph_solid *s, void **stream);
mtsph_status mtsph_solid_pack_device(mtsph_solid *s, const char *field, int64_t m,
                                     const int64_t *dev_internal_ids, double *dev_out);
mtsph_status mtsph_solid_unpack_device(mtsph_solid *s, const char *field, int64_t m,
                                       const int64_t *dev_internal_ids, const double *dev_in);

/* observables: reaction_force, neck radius, max alpha, min mid alpha,
 * all-finite flag (1/0)                                                 */
mtsph_status mtsph_solid_measure(mtsph_solid *s, double out[5]);
/* field access in original numbering.  field names: "pos","vel","F",
 * "accel","cp_inv","alpha","ref_pos"                                    */
mtsph_status mtsph_solid_get(mtsph_solid *s, const char *field, double *host);
mtsph_status mtsph_solid_set(mtsph_solid *s, const char *field, const double *host);
/* neighbour entries, pairs, groups, sweep phases of the problem         */
mtsph_status mtsph_solid_sizes(const mtsph_solid *s, int64_t out[4]);
/* launches of this library's kernels since creation (bench evidence)    */
mtsph_status mtsph_solid_launches(const mtsph_solid *s, int64_t *count);

/* --- porous membrane (scenarios.py:171 PorousProblem) --- */

typedef struct {
    int64_t n;
    int d;
    const double *pos, *vol;
    const uint8_t *constrained;
    const uint8_t *contact;     /* droplet contact region                   */
    double h_axes[3];
    double density0, diffusivity, pressure_coeff, shear_modulus, lame_lambda,
           bulk_modulus, porosity, fluid_density0, initial_saturation;
    double contact_time, evaporation_rate;
    int sweep;
    /* multi-rank (NULL for a single domain), as in mtsph_solid_desc:   */
    const uint8_t *ghost;       /* (n,) 1 = halo copy of another rank's particle */
    const double *grid;         /* 6 doubles: global scaled-space grid bounds    */
    int tile;                   /* tiled sweep block edge in cells (0: auto)     */
} mtsph_porous_desc;

typedef struct mtsph_porous mtsph_porous;

mtsph_status mtsph_porous_create(const mtsph_porous_desc *desc, mtsph_porous **out);
mtsph_status mtsph_porous_destroy(mtsph_porous *p);
/* PorousProblem.advance_slow: one explicit diffusion update; returns the
 * number of clamped particles                                           */
mtsph_status mtsph_porous_advance_slow(mtsph_porous *p, double dt_outer, double t,
                                       int64_t *clamped);
/* device time (CUDA events on the problem's stream) of the kernels of the
 * last advance_slow, in ms (benchmark instrumentation)                   */
mtsph_status mtsph_porous_outer_ms(const mtsph_porous *p, double *ms);
/* neighbour entries, damping pairs, groups, sweep colours (tiled) or
   dependency levels (serial), as mtsph_solid_sizes                      */
mtsph_status mtsph_porous_sizes(const mtsph_porous *p, int64_t out[4]);
mtsph_status mtsph_porous_stable_dt(mtsph_porous *p, double cfl, double *dt);
mtsph_status mtsph_porous_relax_step(mtsph_porous *p, double dt, double eta, double *ek);
mtsph_status mtsph_porous_relax(mtsph_porous *p, const mtsph_inner_params *ip,
                                mtsph_inner_result *r);
/* PorousProblem.measure's velocity refresh (split_velocities)           */
mtsph_status mtsph_porous_refresh_velocities(mtsph_porous *p);
/* fields: "pos","ref_pos","F","momentum","vel_solid","vel_fluid",
 * "fluid_mass","flux","saturation","pressure"                           */
mtsph_status mtsph_porous_get(mtsph_porous *p, const char *field, double *host);
mtsph_status mtsph_porous_set(mtsph_porous *p, const char *field, const double *host);
mtsph_status mtsph_porous_launches(const mtsph_porous *p, int64_t *count);
/* --- multi-rank porous phases (slab decomposition, tiled sweep; driver
 * paper_2309_04010_b200/distributed.py DecomposedPorous).  Ghost particles
 * are never updated and never reduced; their fields come from exchanges. */
enum {
    MTSPH_POR_KICK = 1,       /* M += dt/2 rate, v_s, x += dt v_s (owned)            */
    MTSPH_POR_STRESS = 2,     /* dF/dt gather + F update, constitutive, T~ (owned)   */
    MTSPH_POR_ACCEL = 3,      /* divergence + flux rate + kick; out = sum m v^2, max |a|^2 */
    MTSPH_POR_SWEEP = 4,      /* damping, colour arg (reverse when arg >= 64)        */
    MTSPH_POR_POSTSTEP = 5,   /* momentum rebuild; out[0] = max |v|^2                */
    MTSPH_POR_AMAX = 6,       /* before the loop: out = max |v|^2, max |a|^2         */
    MTSPH_POR_PREP_MAP = 7,   /* outer: J, V, s, D rho_l and the map A (owned)       */
    MTSPH_POR_FLUX_MASS = 8,  /* outer: flux q, packed for the mass update           */
    MTSPH_POR_MASS = 9,       /* outer: mass update; out[0] = clamped particles      */
    MTSPH_POR_PREP = 10,      /* outer: J, V, s, D rho_l                             */
    MTSPH_POR_FLUX = 11,      /* outer: flux q, packed for the flux rate             */
    MTSPH_POR_POST = 12,      /* outer: pressure, masses, momentum, velocity split   */
    MTSPH_POR_FLUXRATE = 13,  /* outer: advected-momentum rate                       */
};
/* step size / viscosity of the inner phases; dt and time of the outer ones */
mtsph_status mtsph_porous_set_step(mtsph_porous *p, double dt, double eta);
mtsph_status mtsph_porous_set_outer(mtsph_porous *p, double dt_outer, double t);
mtsph_status mtsph_porous_phase(mtsph_porous *p, int phase, int arg, double out[2]);
/* host-staged field exchange for the listed particles (ORIGINAL local
 * ids): "vel" (d), "T" (d*d), "satvol" (2), "rm" (16 in 3D, 8 in 2D),
 * "rf" (8), "inv_mix" (1) doubles per particle                          */
mtsph_status mtsph_porous_pack(mtsph_porous *p, const char *field, int64_t m,
                               const int64_t *ids, double *host);
mtsph_status mtsph_porous_unpack(mtsph_porous *p, const char *field, int64_t m,
                                 const int64_t *ids, const double *host);
mtsph_status mtsph_porous_colours(const mtsph_porous *p, int *ncolours);
/* device-resident exchange and device-controlled inner loop, as the
 * mtsph_solid_* functions of the same names; begin_loop also takes the
 * whole problem's free volume (the E_k normaliser) when > 0             */
mtsph_status mtsph_porous_phase_async(mtsph_porous *p, int phase, int arg);
mtsph_status mtsph_porous_begin_loop(mtsph_porous *p, const mtsph_inner_params *ip,
                                     double vol_movable);
mtsph_status mtsph_porous_rank_partials(mtsph_porous *p, int mode, double *dev_out4);
mtsph_status mtsph_porous_control_ranks(mtsph_porous *p, const double *dev_gathered,
                                        int nranks, int mode);
mtsph_status mtsph_porous_loop_state(mtsph_porous *p, mtsph_inner_result *r, int *done);
mtsph_status mtsph_porous_internal_ids(mtsph_porous *p, int64_t m, const int64_t *ids,
                                       int64_t *internal);
mtsph_status mtsph_porous_stream(const mtsph_porous *p, void **stream);
mtsph_status mtsph_porous_pack_device(mtsph_porous *p, const char *field, int64_t m,
                                      const int64_t *ids_dev, double *out_dev);
mtsph_status mtsph_porous_unpack_device(mtsph_porous *p, const char *field, int64_t m,
                                        const int64_t *ids_dev, const double *in_dev);

#ifdef __cplusplus
}
#endif
#endif /* MTSPH_B200_H */
