/*
 * les_b200.h -- C ABI of the B200-native DPRI-LES time step.
 *
 * Drop-in boundary for the reference hot path (gmcf_mini, pure Python):
 *   gmcf_mini.les.step / velnw / bondv1 / velfg_merged / feedbf /
 *   les_viscosity / adam / divergence / strain_magnitude / press
 *   gmcf_mini.sor.solve_pressure / redblack_iteration / twinned_sweep
 * Each entry point below cites the reference function (file:line under
 * /root/reference/pkg/src/gmcf_mini/) whose behaviour it reproduces.  The
 * reference has no FFI; its "operator API" is those module-level Python
 * functions, which the Python shim in paper_1504_02264_b200/ rebinds onto
 * this library through ctypes.
 *
 * Conventions
 *  - Fields are float32, C order (im+2, jm+2, km+2), k contiguous, halo 1
 *    (les.py:56-63).  fgh / fgh_old carry a trailing axis of 3.
 *  - A domain handle owns device-resident state for one x-slab of the grid
 *    (the whole grid on one GPU).  Host pointers passed to upload/download and
 *    to the solver entry points are plain host memory (pinned or pageable).
 *  - Every function returns 0 on success and a negative LESB_E* code on
 *    error (message in lesb_last_error()); lesb_step returns 1 when a stage
 *    produced non-finite values (NumericsError in the reference,
 *    les.py:384-390) and writes the stage index (LESB_STAGE_*) to *fail_stage.
 *  - Results are bitwise identical to the reference for all fields; float64
 *    residual sums agree to summation-order tolerance (rtol 1e-12).
 */
#ifndef LES_B200_H
#define LES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LESB_ABI_VERSION 1

typedef struct lesb_domain* lesb_handle;

/* field ids (FlowState attributes, les.py:41-47; rhs is press' work array) */
enum {
    LESB_U = 0, LESB_V = 1, LESB_W = 2, LESB_P = 3, LESB_MASK = 4,
    LESB_FGH = 5, LESB_FGH_OLD = 6, LESB_RHS = 7
};

/* gmcf_mini.sor.Scheme (sor.py:29-31) */
enum { LESB_REDBLACK = 0, LESB_TWINNED = 1 };

/* halo_fn policies of solve_pressure (sor.py:255): None keeps the stored
 * halo of p0; PRESS is les._pressure_halo (les.py:341-355). */
enum { LESB_HALO_STORED = 0, LESB_HALO_PRESS = 1 };

/* stage names in step order (les.py:401-409) */
enum {
    LESB_STAGE_VELNW = 0, LESB_STAGE_BONDV1 = 1, LESB_STAGE_VELFG = 2,
    LESB_STAGE_FEEDBF = 3, LESB_STAGE_LES = 4, LESB_STAGE_ADAM = 5,
    LESB_STAGE_PRESS = 6
};

enum {
    LESB_OK = 0, LESB_NONFINITE = 1,
    LESB_E_ARG = -1, LESB_E_CUDA = -2, LESB_E_STATE = -3, LESB_E_NOMEM = -4
};

/* Geometry and physics of one domain (FlowState.create, les.py:54-63, and
 * Grid, sor.py:64-105).  For an x-slab of a decomposed grid, i_offset is the
 * global index of local interior plane 1 minus 1, and west/east_boundary say
 * whether the local low/high x face is a physical boundary of the global
 * grid (single GPU: both 1, i_offset 0). */
typedef struct lesb_desc {
    int im, jm, km;          /* local interior extents */
    int i_offset;
    int west_boundary, east_boundary;
    const float* dx1;        /* im+3 entries: global dx1[i_offset .. i_offset+im+2] */
    const float* dy1;        /* jm+2 */
    const float* dzn;        /* km+2 */
    float dt, vn, cs;
    const float* csd2;       /* (cs*cbrt(dx dy dz))^2 per interior cell, im*jm*km, or NULL */
    float csd2_scalar;       /* used when csd2 == NULL (uniform grids) */
    int device;              /* CUDA ordinal */
} lesb_desc;

/* SorCoeffs (sor.py:108-118).  cn1 == NULL means cn1 is the constant
 * cn1_scalar everywhere (build_uniform_coeffs, sor.py:121-137). */
typedef struct lesb_coeffs {
    const float* cn1;        /* im*jm*km or NULL */
    float cn1_scalar;
    const float *cn2l, *cn2s; /* im each */
    const float *cn3l, *cn3s; /* jm each */
    const float *cn4l, *cn4s; /* km each */
} lesb_coeffs;

const char* lesb_last_error(void);
int lesb_abi_version(void);

/* ---- domain lifetime and data movement (FlowState, les.py:37-71) ---- */
int lesb_create(const lesb_desc* desc, lesb_handle* out);
int lesb_destroy(lesb_handle h);
int lesb_set_coeffs(lesb_handle h, const lesb_coeffs* c);          /* FlowState.coeffs(), les.py:65-68 */
int lesb_set_physics(lesb_handle h, float dt, float vn, float cs, const float* csd2, float csd2_scalar);
int lesb_upload(lesb_handle h, int field, const float* host);       /* host -> device, full halo array */
int lesb_download(lesb_handle h, int field, float* host);           /* device -> host */
/* Asynchronous state copies, overlapping the steps (no reference counterpart:
 * the reference's FlowState arrays are host numpy, les.py:37-71; these serve
 * its dump / restart pattern, dump.py:42-56 and cli.py:202-219, without
 * stalling the device).  lesb_stage_upload starts the host -> device copy of
 * `host` (pinned for overlap) into the field's staging buffer and returns;
 * `host` must stay unchanged until the next synchronising call after
 * lesb_stage_commit, which enqueues the staged fields becoming the state at
 * that point of the domain's stream.  lesb_download_async enqueues a snapshot
 * of the field as of that point and its copy to `host`; lesb_copies_wait
 * blocks until every staged and asynchronous copy has finished. */
int lesb_stage_upload(lesb_handle h, int field, const float* host);
int lesb_stage_commit(lesb_handle h);
int lesb_download_async(lesb_handle h, int field, float* host);
int lesb_copies_wait(lesb_handle h);
void* lesb_device_ptr(lesb_handle h, int field);                    /* plumbing for NCCL halo exchange */
void* lesb_stream(lesb_handle h);                                   /* the domain's cudaStream_t */
int lesb_synchronize(lesb_handle h);
int lesb_check_finite(lesb_handle h, int* all_finite);              /* les.py:387-390 over the 6 fields */

/* ---- stages, each alone, in place (les.py:178-338) ---- */
int lesb_velnw(lesb_handle h);                                      /* les.py:218-241 */
int lesb_bondv1(lesb_handle h, const float* in_u, const float* in_v, const float* in_w); /* les.py:244-266 */
int lesb_velfg(lesb_handle h);                                      /* velfg_merged / velfg_twopass, les.py:178-215 */
int lesb_feedbf(lesb_handle h);                                     /* les.py:269-282 */
int lesb_les_viscosity(lesb_handle h);                              /* les.py:299-320 */
int lesb_adam(lesb_handle h);                                       /* les.py:323-327 */
int lesb_divergence(lesb_handle h, float* out_host);                /* les.py:330-338, (im,jm,km) */
int lesb_strain_magnitude(lesb_handle h, float* out_host);          /* les.py:285-296, (im,jm,km) */
int lesb_press(lesb_handle h, int n_iter, int scheme, float omega,
               double* residuals_out);                              /* les.py:358-381 */
/* solve_pressure on the domain's device-resident p (in place) and rhs (set
 * with lesb_upload(LESB_RHS)): the sor-bench path (cli.py:222-283,
 * sor.py:255-309) without host copies.  halo_policy LESB_HALO_STORED or
 * LESB_HALO_PRESS; residuals_out (host, n_iter doubles) may be NULL. */
int lesb_sor_solve(lesb_handle h, int n_iter, int scheme, float omega, int halo_policy,
                   double* residuals_out);

/* ---- the time step (les.py:393-416) ---- */
/* One step, synchronous: inflow (3 x km floats, host) in, residuals
 * (n_iter doubles, host, may be NULL) and the failing stage out.  Returns
 * LESB_OK, LESB_NONFINITE (fail_stage set) or an error. */
int lesb_step(lesb_handle h, const float* in_u, const float* in_v, const float* in_w,
              int n_iter, int scheme, float omega, double* residuals_out, int* fail_stage);
/* n_steps steps with one host synchronisation at the end.  inflow holds
 * n_profiles blocks of 3*km floats (u, v, w); step s uses block
 * min(s, n_profiles-1).  On a non-finite stage the first failing step
 * (0-based) and stage are reported and *steps_done counts completed steps.
 * The steps are enqueued before the failure is known, so after
 * LESB_NONFINITE the fields hold the end of the last enqueued step, not the
 * reference's state after the failing stage; callers that need that state
 * (the reference's per-step loop) use lesb_step. */
int lesb_run_steps(lesb_handle h, int n_steps, const float* inflow, int n_profiles,
                   int n_iter, int scheme, float omega,
                   int* steps_done, int* fail_stage);
/* Enqueue one step on the domain stream without synchronising (inflow must
 * already be resident via lesb_set_inflow).  Failure flags accumulate on
 * the device; read them with lesb_poll_failure. */
int lesb_set_inflow(lesb_handle h, const float* in_u, const float* in_v, const float* in_w);
int lesb_step_async(lesb_handle h, int n_iter, int scheme, float omega);
int lesb_poll_failure(lesb_handle h, int* steps_done, int* fail_step, int* fail_stage);
/* Number of kernel launches one asynchronous step (lesb_step_async)
 * enqueues, its bookkeeping included (evidence for gpu_launches). */
int lesb_kernels_per_step(lesb_handle h, int n_iter, int scheme);
/* Device-to-device copy of the seven state fields between two domains of
 * the same shape on the same device (benchmark re-initialisation). */
int lesb_copy_state(lesb_handle dst, lesb_handle src);
/* Capture CUDA events between the step phases; lesb_last_step_times then
 * returns, for the last replayed step, ms of [velnw+bondv1, fused
 * velfg..rhs, SOR passes, halo + residual reduction]. */
int lesb_set_timing(lesb_handle h, int on);
/* Red-black solver implementation: 0 auto (shared-memory-resident persistent
 * kernel when the grid fits the SMs' shared memory and the coefficients are
 * uniform, else colour passes), 1 colour passes only, 2 resident when
 * possible, 3 colour-fused streaming iterations when possible.  Results are
 * bitwise identical whichever runs. */
int lesb_set_sor_path(lesb_handle h, int path);
int lesb_sor_path_in_use(lesb_handle h, int scheme);  /* 1 passes, 2 resident, 3 fused */
/* Default for domains created afterwards and for the host-buffer solver
 * entry points (initially $LESB_SOR_PATH or 0). */
int lesb_set_default_sor_path(int path);
int lesb_last_step_times(lesb_handle h, float* ms4);

/* ---- SOR solver on host buffers (sor.py:181-309) ---- */
/* solve_pressure(p0, rhs, c, omega, n_iter, scheme, workers, halo_fn):
 * p0, rhs: (im+2)(jm+2)(km+2) host arrays; p_out same shape; residuals n_iter. */
int lesb_solve_pressure(int im, int jm, int km, const float* p0, const float* rhs,
                        const lesb_coeffs* c, float omega, int n_iter, int scheme,
                        int halo_policy, float* p_out, double* residuals, int device);
/* redblack_iteration(p, rhs, c, omega, halo_fn): p updated in place. */
int lesb_redblack_iteration(int im, int jm, int km, float* p, const float* rhs,
                            const lesb_coeffs* c, float omega, int halo_policy,
                            double* residual, int device);
/* twinned_sweep(tp, rhs, c, omega, nrd) on de-interleaved components:
 * reads src, replaces the interior of dst (its halo is kept). */
int lesb_twinned_sweep(int im, int jm, int km, const float* src, float* dst, const float* rhs,
                       const lesb_coeffs* c, float omega, double* residual, int device);

/* ---- x-slab decomposition over several GPUs ----
 * A slab is a domain created with i_offset / west_boundary / east_boundary
 * describing its planes of the global grid.  After linking, lesb_step and
 * lesb_press exchange the halo planes: velocities after velnw+bondv1 (depth 1
 * low, 2 high), pressure after every colour pass / sweep and after the final
 * halo.  Results equal the single-domain step bitwise. */
/* ncclGetUniqueId into out (>= 128 bytes); returns the id size. */
/* ---- boundary-range launch geometry (sor.py:312-349; the paper's gid -> face map) ----
 * lesb_boundary_decode: device decode of gids [gid0, gid0 + n) exactly as
 *   map_boundary_gid (sor.py:319-338): face 0 YZ (j, k), 1 ZX (k, i), 2 XY (j, i),
 *   -1 PADDING (c0 = c1 = -1); host output arrays of n ints.
 * lesb_boundary_audit: cli.py:286-320 on the device -- one launch of blocks of
 *   nthreads threads x nunits gids over padded_range (sor.py:341-349);
 *   stats[8] = {boundary_range, padded_range, in-range gids decoded to padding,
 *   padding gids escaping the guard, points covered once, points covered more
 *   than once, points never covered, smallest violating gid or -1}.
 * lesb_boundp_faces: the pressure halo refresh (les.py:341-355) of the
 *   face-interior halo cells (the cells the SOR stencil reads), one launch over
 *   the boundary range; edges and corners are left as they are. */
int lesb_boundary_decode(int ip, int jp, int kp, long long gid0, long long n, int* face, int* c0, int* c1);
int lesb_boundary_audit(int ip, int jp, int kp, int nthreads, int nunits, long long* stats);
int lesb_boundp_faces(lesb_handle h);

int lesb_nccl_unique_id(void* out, int nbytes);
/* One process per GPU: rank r's neighbours are r-1 (west) and r+1 (east). */
int lesb_link_nccl(lesb_handle h, const void* unique_id, int nranks, int rank);
/* In-process slabs (west to east) on one device, stepped with lesb_group_step. */
int lesb_link_local(lesb_handle* hs, int n);
int lesb_group_step(lesb_handle* hs, int n, const float* in_u, const float* in_v, const float* in_w, int n_iter,
                    int scheme, float omega, double* residuals_out, int* fail_stage);
/* solve_pressure (sor.py:255-309) on in-process slabs: each slab's p / rhs
 * (LESB_P, LESB_RHS uploads) solved together; residuals = the sum of the
 * slabs' histories.  sor-bench's x-slab table (cli.py:222-283). */
int lesb_group_sor_solve(lesb_handle* hs, int n, int n_iter, int scheme, float omega, int halo_policy,
                         double* residuals_out);

#ifdef __cplusplus
}
#endif
#endif /* LES_B200_H */
