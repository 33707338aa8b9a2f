/*
 * swof.h -- C ABI of the B200-native FullSWOF_2D explicit time step (arXiv 1307.4839).
 *
 * One context = one structured nx x ny grid advanced by Heun steps of the well-balanced,
 * positivity-preserving finite-volume scheme of PAPER.md §3 on one CUDA device:
 *   per stage (Algorithm 1): boundary conditions -> MUSCL reconstruction of
 *   h, h+z, u, v with the discharge-conserving velocity modification -> hydrostatic
 *   reconstruction -> HLL flux with interface sources ->
 *   scheme: flux divergence + centred slope source, rain, Green-Ampt
 *   infiltration -> semi-implicit friction;
 *   per step: Heun average and the CFL time step of the new state.
 * The readings of points the paper leaves open are listed in DESIGN.md §3:
 * 2D sum-form CFL dt = n_CFL / (a_x/dx + a_y/dy) on cell-centred speeds, exact 2-layer wall
 * mirror, critical-depth inflow ghost, Green-Ampt as printed with V = 0 -> unlimited capacity.
 *
 * Conventions
 *   - Host arrays are row-major ny x nx (x fastest), fp64, SI units, no ghost cells.  Any pointer
 *     argument documented as "host or device" may be a host pointer (pageable or pinned) or a CUDA
 *     device pointer (unified addressing); the library copies, the caller keeps ownership.
 *   - All device work is enqueued on the context's stream; every call returns only after that work
 *     has completed (host-synchronous).  A context is not thread-safe: one context per stream.
 *   - Return codes: SWOF_OK (0) or a positive SWOF_E* code; swof_last_error() gives the message.
 *     SWOF_ENUMERIC is sticky until the next swof_set_state.
 */
#ifndef SWOF_H
#define SWOF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWOF_OK 0
#define SWOF_EINVAL 1    /* bad parameter / argument / initial state (h < 0 or non-finite)      */
#define SWOF_ENUMERIC 2  /* NaN/Inf reached the CFL maximum, or one clamp of h exceeded clamp_fail */
#define SWOF_ECUDA 3     /* CUDA runtime failure                                                */
#define SWOF_ENOMEM 4    /* device or pinned-host allocation failed / workspace too small       */
#define SWOF_ESTATE 5    /* call order: swof_step/run/get_state before swof_set_state            */

/* friction laws, P:80-90 (C_f = n^2, 1/K^2, f/(8g), 1/C^2) */
#define SWOF_FRIC_NONE 0
#define SWOF_FRIC_MANNING 1
#define SWOF_FRIC_STRICKLER 2
#define SWOF_FRIC_DARCY_WEISBACH 3
#define SWOF_FRIC_CHEZY 4

/* boundary types per side: ghost cells, 2 layers */
#define SWOF_BC_WALL 0      /* exact mirror of interior layers 0,1; normal discharge negated     */
#define SWOF_BC_FREE 1      /* zero-gradient copy of interior layer 0 (h, q, z)                  */
#define SWOF_BC_PERIODIC 2  /* wrap (both opposite sides must be PERIODIC)                      */
#define SWOF_BC_INFLOW 3    /* imposed (h_c(q), q = Q(t)/W, 0) on [k0, k1), WALL elsewhere        */
#define SWOF_BC_HALO 4      /* S/N only: the side borders another row strip of a decomposed grid
                               (the paper's MPI strips): its 2 ghost rows
                               are filled by the caller's halo exchange, see swof_halo_rows        */

/* scheme variants; zero-initialised params give the paper's recommended
 * scheme: HLL, second order (MUSCL + Heun), CFL on cell-centred speeds, Green-Ampt as printed */
#define SWOF_FLUX_HLL 0
#define SWOF_FLUX_RUSANOV 1  /* F = (F_L + F_R)/2 - c/2 (U_R - U_L), c = max(|u| + sqrt(g h)) */
#define SWOF_CFL_CELL 0      /* a = max over cells of |u| + sqrt(g h) (Q10)               */
#define SWOF_CFL_FACE 1      /* over every cell's reconstructed face values (Q22)        */
#define SWOF_GA_PRINTED 0    /* I_C = K_s (A + (h_f - h_over)/Z_f)                           */
#define SWOF_GA_DARCY 1      /* I_C = K_s (A + (h_f + h_over)/Z_f) (Q15)                            */

#define SWOF_SIDE_W 0
#define SWOF_SIDE_E 1
#define SWOF_SIDE_S 2
#define SWOF_SIDE_N 3
#define SWOF_MAX_TABLE 16

/* diagnostic flags */
#define SWOF_FLAG_NONFINITE 1u  /* NaN/Inf in the CFL maximum -> stepping halted                 */
#define SWOF_FLAG_BIGCLAMP 2u   /* a single negative-height clamp larger than params.clamp_fail
                                   -> stepping halted: the step that raised it is not completed, so
                                   the state stays that of the last completed step (SPEC's
                                   NegativeHeight abort)                                   */
#define SWOF_FLAG_BADINPUT 4u   /* set_state saw h < 0 or a non-finite value                     */

typedef struct swof_params {
    int32_t nx, ny;          /* cells, >= 1                                                     */
    double dx, dy;           /* cell sizes [m], > 0                                              */
    double g;                /* gravity [m/s^2] (9.81)                                     */
    double cfl;              /* n_CFL in (0, 1]                                          */
    double dt_max;           /* [s] > 0; also the step of an all-dry domain                      */
    double h_eps;            /* dry threshold [m] >= 1e-300: wet <=> h > h_eps                    */
    int32_t fric_law;        /* SWOF_FRIC_*                                                      */
    double fric_coef;        /* n, K, f or C (> 0 unless NONE); ignored when a per-cell field is given */
    int32_t ga_enabled;      /* Green-Ampt                                           */
    double ga_Ks;            /* saturated conductivity [m/s] >= 0                                 */
    double ga_hf;            /* wetting-front capillary head [m]                                  */
    double ga_A;             /* modified Green-Ampt offset (dimensionless)                        */
    double ga_dtheta;        /* theta_s - theta_i > 0                                             */
    double ga_vinf0;         /* initial infiltrated volume per area [m] when set_state gets NULL  */
    int32_t n_rain;          /* rain table entries, 0..16                                         */
    double rain_t[SWOF_MAX_TABLE];     /* ascending start times [s]; R(t) = rate[k] on [t_k, t_k+1) */
    double rain_rate[SWOF_MAX_TABLE];  /* [m/s] >= 0; R = 0 before rain_t[0]                     */
    int32_t bc[4];           /* SWOF_BC_* for W, E, S, N                                          */
    int32_t inflow_k0[4];    /* inflow segment [k0, k1) along the side (cells)                    */
    int32_t inflow_k1[4];
    int32_t n_hydro[4];      /* hydrograph points per side, 1..16 for INFLOW                      */
    double hydro_t[4][SWOF_MAX_TABLE];  /* ascending times [s]                                    */
    double hydro_q[4][SWOF_MAX_TABLE];  /* Q [m^3/s] over the segment; piecewise linear, clamped  */
    int64_t dt_hist_cap;     /* dt history capacity (0 -> 1<<20 steps)                             */
    int32_t graph_steps;     /* Heun steps per captured CUDA graph (0 -> 16; rounded up to even)  */
    double clamp_fail;       /* a single negative-height clamp above this [m] raises SWOF_FLAG_BIGCLAMP,
                                halts stepping and returns SWOF_ENUMERIC.  0 -> 1e-6 m, not SURVEY
                                §8b's 1e-10 m: full-size cfg4 clamps 2.28e-10 m in step 0, a
                                film the cell-centred CFL of U^n does not bound, reproduced bit for
                                bit by the oracle (DESIGN.md §3 Q17); 1e-6 m is still a positivity
                                failure, not round-off                                             */
    int32_t flux;            /* SWOF_FLUX_*                                                       */
    int32_t order;           /* 2 (or 0): MUSCL + Heun; 1: first order in
                                space (no reconstruction) and explicit Euler in time      */
    int32_t cfl_mode;        /* SWOF_CFL_*                                                        */
    int32_t ga_form;         /* SWOF_GA_*                                                         */
    double inflow_width[4];  /* width W [m] that Q(t) is spread over per side (0: the segment's own
                                (k1 - k0) * dy or dx); a strip of a decomposed grid passes the global
                                segment's width and its share of Q so that q = Q/W is unchanged   */
    int32_t dry_skip;        /* 1: rows of a warp's strip whose cells all hold h = 0 exactly skip the
                                face and slope work (results unchanged); pays on mostly dry domains
                                (cfg3: +14 %), costs 6-10 % on wet ones, so off by default        */
} swof_params;

typedef struct swof_diag {
    double t;                /* simulated time [s]                                                */
    int64_t step;            /* Heun steps taken                                                  */
    double dt_next;          /* CFL time step of the current state (before t_end clipping)        */
    double volume;           /* sum h dx dy [m^3], fixed-order sum                                */
    double vinf_volume;      /* sum V dx dy [m^3] (0 without Green-Ampt)                          */
    double h_min, h_max;     /* [m]                                                               */
    int64_t wet_cells;       /* h > h_eps                                                         */
    int64_t clamps;          /* negative heights set to 0 since set_state                         */
    double clamped_mass;     /* sum of the clamped -h' [m] (per cell, not times the area)         */
    double clamp_max;        /* largest single clamp [m]                                          */
    uint32_t flags;          /* SWOF_FLAG_* (sticky until set_state)                              */
    int64_t big_clamp_cell;  /* row-major index j*nx+i of the largest clamp so far, -1 if none     */
    int64_t big_clamp_step;  /* step in which that clamp happened, -1 if none                     */
} swof_diag;

typedef struct swof_ctx swof_ctx;

/* Bytes of device workspace a context needs for these parameters (padded SoA fields, device
 * scalar state, dt history, reduction scratch).  Returns SWOF_EINVAL on bad parameters. */
int swof_workspace_size(const swof_params* p, size_t* bytes);

/* Create a context.  z: topography, ny x nx (host or device), copied, fixed for the context's life
 * (P:71-72).  fric_field: per-cell friction coefficient of p->fric_law, or NULL to use
 * p->fric_coef everywhere.  d_workspace: device memory of >= swof_workspace_size bytes that must
 * outlive the context (e.g. a torch allocation), or NULL to let the library cudaMalloc it.
 * cuda_stream: a cudaStream_t, or NULL for the legacy default stream.  The CUDA device current on
 * the calling thread is used. */
int swof_create(const swof_params* p, const double* z, const double* fric_field, void* d_workspace,
                size_t ws_bytes, void* cuda_stream, swof_ctx** out);

/* Load the state U = (h, hu, hv) and the infiltrated volume V (NULL ->
 * p->ga_vinf0 everywhere) at time t0; resets step, dt history, clamp counters and flags, and
 * computes the first CFL step.  Host or device pointers.  h must be >= 0 and finite everywhere
 * (SWOF_EINVAL otherwise); cells with h <= h_eps may carry nonzero discharge (treated as still). */
int swof_set_state(swof_ctx* c, const double* h, const double* hu, const double* hv, const double* v_inf,
                   double t0);

/* Advance nsteps time steps (Heun, or explicit Euler at order 1) with dt = min(CFL dt, dt_max) each
 * (no t_end clipping).  A halt flag stops stepping at the last completed step (the remaining steps are
 * device-side no-ops).  Returns SWOF_ENUMERIC if a flag is set afterwards. */
int swof_step(swof_ctx* c, int64_t nsteps);

/* Advance until t >= t_end or max_steps steps were taken; the last dt is clipped so that t lands on
 * t_end exactly.  steps_done (nullable) receives the number of steps taken by this call.  max_steps is
 * counted from the current step and saturates (INT64_MAX = no cap).  A halt flag (non-finite CFL
 * maximum, a clamp above clamp_fail) stops the run at the last completed step: SWOF_ENUMERIC. */
int swof_run(swof_ctx* c, double t_end, int64_t max_steps, int64_t* steps_done);

/* The three getters take a const context: the state is not changed (they use the context's stream,
 * its diagnostics scratch and its last-error text).
 * Copy the state out (host or device pointers; any of the arrays may be NULL; v_inf is left
 * untouched when Green-Ampt is off).  t and step (nullable) receive the simulated time and count. */
int swof_get_state(const swof_ctx* c, double* h, double* hu, double* hv, double* v_inf, double* t, int64_t* step);

/* Copy min(cap, steps taken) entries of the dt history (host pointer); n receives that count. */
int swof_get_dt_history(const swof_ctx* c, double* dt, int64_t cap, int64_t* n);

/* Fixed-order diagnostics of the current state (not part of the time loop). */
int swof_get_diag(const swof_ctx* c, swof_diag* d);

/* Testing/profiling entry points (same kernels as swof_step):
 * swof_predictor: run only the predictor stage U* = S(U^n; t^n) of the next step and copy U*, V*
 *   out (host or device; nullable); the state is not advanced (at order 1, U* is the next state).
 * swof_step_profiled: like swof_step but launched eagerly with CUDA events around every kernel;
 *   ms[0], ms[1] receive the summed device time of the predictor and of the rest of the step
 *   (corrector, or the order-1 commit; plus the face-CFL pass if any). */
int swof_predictor(swof_ctx* c, double* h, double* hu, double* hv, double* v_inf);
int swof_step_profiled(swof_ctx* c, int64_t nsteps, double* ms);

/* Bounds-checked builds (-DSWOF_CHECK=1): the source line of the first failed index check in
 * csrc/swof_kernels.cuh since the library was loaded, 0 if none (always 0 in normal builds), -1 on error. */
int swof_check_line(void);

/* Number of kernel launches one time step issues with the default scheme (2: predictor and
 * corrector).  swof_ctx_launches_per_step: the same for a context's scheme (2, or 3 with SWOF_CFL_FACE:
 * the reconstructed-value CFL maxima are a separate stencil pass). */
int swof_launches_per_step(void);
int swof_ctx_launches_per_step(const swof_ctx* c);

/* Self-test of the kernels' slow-path-free IEEE reciprocal, division and square root against CUDA's
 * library operators on n random operands (exponents in [-60, 60], sqrt in [-80, 40]) on the current
 * device; mismatches[0..2] receive the bitwise mismatch counts (rcp, div, sqrt), all 0 when exact. */
int swof_selftest_math(int64_t n, uint64_t seed, int64_t* mismatches);

/* ---- row-strip decomposition (PAPER.md P:731-760 on NVLink) ----
 * A strip is an ordinary context whose S and/or N side is SWOF_BC_HALO.  The caller (one rank per GPU,
 * or several strips driven from one process) runs each time step as
 *   phase 0 (predictor) -> exchange set 1 -> phase 1 (corrector / order-1 commit) -> exchange set 0
 *   -> phase 2 (face CFL, if any) -> all-reduce (max) of the 2 words at swof_cfl_maxima
 * and, once after swof_create, exchanges set 2 (z); after swof_set_state it exchanges set 0, calls
 * swof_refresh_cfl and all-reduces.  Every strip then computes exactly what the undivided grid
 * computes on its rows (bit for bit: the ghost rows carry the neighbours' values).
 *
 * swof_halo_rows: device pointers of the 2 boundary rows this strip sends to its neighbour on `side`
 *   (SWOF_SIDE_S or SWOF_SIDE_N) and of the 2 ghost rows it receives from it, for field set `set`:
 *   0 = the state U^n (h, hu, hv), read by the predictor; 1 = the predictor's output U* (h, hu, hv),
 *   read by the corrector; 2 = the topography z (send[0]/recv[0] only, the others NULL).  Each block is
 *   2 rows x pitch doubles, contiguous (*bytes).  The S block of a strip goes to the N ghost rows of
 *   the strip below and vice versa.
 * swof_enqueue_phase: enqueue phase 0, 1 or 2 of the next time step on the context's stream and return
 *   without synchronising (phase 2 is a no-op unless SWOF_CFL_FACE; it ends the step).
 * swof_cfl_maxima: device pointer to the 2 uint64 words (a_x, a_y as IEEE bit patterns; max-reduce them
 *   as unsigned or as int64) that the next step's kernels derive dt from.
 * swof_refresh_cfl: recompute those maxima from the current state (cell or face form, local rows).
 * swof_set_limits: t_end and the absolute step limit of the following phases (steps past them are
 *   exact no-ops); swof_step / swof_run set their own.
 * swof_sync: wait for the context's stream; returns SWOF_ENUMERIC if a flag is set. */
int swof_halo_rows(swof_ctx* c, int32_t set, int32_t side, double** send, double** recv, size_t* bytes);
/* Fused halo exchange: the kernels that produce U* (set 1) and U^{n+1} (set 0) also store this strip's 2
 * boundary rows on `side` straight into the neighbour's ghost rows -- set0[k], set1[k] (k = h, hu, hv) are
 * the neighbour's receive blocks for this side (its swof_halo_rows(set, opposite side) recv pointers, in
 * this process's address space: same device, or NVLink peer memory mapped with CUDA IPC).  The caller
 * then replaces the per-phase exchanges of sets 0 and 1 by a barrier between strips (the state loaded by
 * swof_set_state still needs one ordinary exchange).  NULL arrays disable it. */
int swof_set_halo_push(swof_ctx* c, int32_t side, double* const* set0, double* const* set1);
/* CUDA IPC for strips in different processes: swof_ipc_handle writes the 64-byte cudaIpcMemHandle_t of
 * the context's workspace (library-allocated only: d_workspace == NULL at create) and its base address
 * in the owner's address space (subtract it from swof_halo_rows pointers to get offsets); swof_ipc_open
 * maps a neighbour's workspace into this process (peer access enabled lazily), swof_ipc_close unmaps. */
int swof_ipc_handle(swof_ctx* c, void* handle, uint64_t* ws_base);
int swof_ipc_open(const void* handle, void** base);
int swof_ipc_close(void* base);
/* Enqueue a copy of `bytes` between any two addresses (host, device, mapped peer) on cuda_stream; used
 * by the strip driver to pull a neighbour's rows out of its mapped workspace. */
int swof_copy(void* dst, const void* src, size_t bytes, void* cuda_stream);
int swof_enqueue_phase(swof_ctx* c, int32_t phase);
int swof_cfl_maxima(swof_ctx* c, uint64_t** dev_ptr);
int swof_refresh_cfl(swof_ctx* c);
int swof_set_limits(swof_ctx* c, double t_end, int64_t step_limit);
int swof_sync(swof_ctx* c);

/* D8 flow direction of a DEM (the paper's user function): for every point
 * of the ny x nx row-major raster z (x fastest, rows growing northwards), dir receives the code 1..8 of
 * the lowest of its 8 neighbours that is > 0 and strictly below the point -- neighbours enumerated E,
 * SE, S, SW, W, NW, N, NE (SPEC.md flow_direction), the first one on ties -- or 0 if there is none.
 * Neighbours outside the raster are absent; values <= 0 (no-data) are never chosen.  z (fp64, or fp32
 * for the _f32 entry point, the paper's DMatrix<float>) and dir (1 byte per point) may be host or device
 * pointers; host buffers are staged through temporary device memory.  Work is enqueued on cuda_stream
 * (NULL: legacy default stream); the call returns after it completed.  Returns SWOF_EINVAL for a NULL
 * pointer or nx, ny < 1, SWOF_ENOMEM / SWOF_ECUDA on runtime failures.  Needs no context. */
int swof_flow_direction(const double* z, int32_t nx, int32_t ny, uint8_t* dir, void* cuda_stream);
int swof_flow_direction_f32(const float* z, int32_t nx, int32_t ny, uint8_t* dir, void* cuda_stream);

void swof_destroy(swof_ctx* c);
const char* swof_last_error(const swof_ctx* c);
const char* swof_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* SWOF_H */
