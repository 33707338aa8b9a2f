/*
 * swof_oracle.h -- CPU ORACLE for the FullSWOF_2D explicit time step (arXiv 1307.4839).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_1307_4839_b200/csrc, include/swof.h), and neither includes the other.
 *
 * Plain, slow, single-threaded fp64, whole-array passes in the order of the paper's Algorithm 1
 * (PAPER.md:773-788): boundary conditions -> second-order (MUSCL) reconstruction -> hydrostatic
 * reconstruction -> numerical flux -> scheme computation -> frictions, twice, then Heun.
 * Build with -O2 -ffp-contract=off (no FMA contraction), IEEE division and sqrt.
 *
 * Citations: "P:n" = line n of /root/reference/PAPER.md (read at development time only).
 * Readings of points the paper leaves open are SURVEY.md §8c Q1..Q21, restated in DESIGN.md §3.
 * Pins (tests/): the transverse HLL component (Q2) by the hand-derived face pin with a
 * transverse velocity (golden face_pins.json), both CFL forms (Q10, Q22) by closed forms (3x3 stage,
 * face-CFL worked example), Green-Ampt as printed and in the Darcy form (Q15) by SPEC examples and
 * hand-derived capacities, the inflow ghost (Q18) by the inflow mass rate (q) and the closed-form momentum
 * flux of the critical state (h_c), icbrt (Q20) by libm cbrt to 2 ulp.  No function is left "parity
 * unpinned"; V0 = 3 mm (Q15) is problem data.
 */
#ifndef SWOF_ORACLE_H
#define SWOF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_FRIC_NONE = 0, OR_FRIC_MANNING = 1, OR_FRIC_STRICKLER = 2, OR_FRIC_DARCY = 3, OR_FRIC_CHEZY = 4 };
enum { OR_BC_WALL = 0, OR_BC_FREE = 1, OR_BC_PERIODIC = 2, OR_BC_INFLOW = 3 };
enum { OR_W = 0, OR_E = 1, OR_S = 2, OR_N = 3 };
/* scheme variants; the zero values are the default scheme */
enum { OR_FLUX_HLL = 0, OR_FLUX_RUSANOV = 1 };       /* numerical flux */
enum { OR_CFL_CELL = 0, OR_CFL_FACE = 1 };           /* CFL on cell values or reconstructed values */
enum { OR_GA_PRINTED = 0, OR_GA_DARCY = 1 };         /* Green-Ampt h_over sign (Q15) */
#define OR_MAX_TABLE 16

typedef struct {
    int32_t nx, ny;
    double dx, dy;
    double g, cfl, dt_max, h_eps;
    int32_t fric_law;
    double fric_coef;            /* used when no per-cell field is given */
    int32_t ga_enabled;
    double ga_Ks, ga_hf, ga_A, ga_dtheta, ga_vinf0;
    int32_t n_rain;
    double rain_t[OR_MAX_TABLE], rain_rate[OR_MAX_TABLE];
    int32_t bc[4];               /* W, E, S, N */
    int32_t in_k0[4], in_k1[4];  /* inflow segment [k0, k1) per side */
    int32_t n_hydro[4];
    double hydro_t[4][OR_MAX_TABLE], hydro_q[4][OR_MAX_TABLE];
    int32_t flux;                /* OR_FLUX_*                                                      */
    int32_t order;               /* 2 (or 0): MUSCL + Heun; 1: first order in space, explicit Euler */
    int32_t cfl_mode;            /* OR_CFL_*                                                       */
    int32_t ga_form;             /* OR_GA_*                                                        */
} or_params;

/* per-run counters (used for the algorithmic op count F_alg and the clamp audit) */
typedef struct {
    int64_t face_dry, face_left, face_right, face_mid;   /* HLL branch taken, over all stages */
    int64_t cell_stage;                                   /* cells x stages */
    int64_t cell_wet_fric;                                /* friction applied on a wet cell */
    int64_t ga_capped;                                    /* GA with finite capacity (V > 0) */
    int64_t clamps;                                       /* h' < 0 set to 0 */
    double clamped_mass;                                  /* sum of -h' over clamps [m] */
    double clamp_max;                                     /* largest single clamp [m] */
} or_counters;

/* ---- pointwise operations (exported for the formula pins) ---- */
double or_minmod(double a, double b);
double or_icbrt(double x);                                         /* x^(-1/3), Q20 */
double or_rain_rate(const or_params* P, double t);                 /* P:75, Q14 */
double or_hydrograph(const or_params* P, int side, double t);      /* piecewise linear Q(t) */
double or_friction_gcf(int law, double coef, double g);            /* g*C_f */
/* MUSCL + velocity modification for one cell along one axis.
   in: s_m, s_c, s_p for h, eta=h+z, u(normal), v(transverse); rh_c = 1/h_c or 0.
   out[10] = hm, hp, etam, etap, zm, zp, um, up, vm, vp  ("m" = cell's low face, "p" = high face) */
void or_muscl_cell(const double h3[3], const double eta3[3], const double u3[3], const double v3[3],
                   double rh_c, double out[10]);
/* hydrostatic reconstruction + HLL + interface sources at one face.
   l = left cell's high-face values, r = right cell's low-face values (h, eta, z, normal vel, transverse vel).
   out[9] = Fm, Fn, Ft, S_L, S_R, H_L, H_R, c1, c2 ; returns branch 0 dry, 1 left, 2 right, 3 middle */
double or_centered_source(double g, double hm, double hp, double zm, double zp);
int or_face(double g, double h_eps, const double l[5], const double r[5], double out[9]);
/* the same with the Rusanov flux (textbook local Lax-Friedrichs): F = (F_L + F_R)/2 - c/2 (U_R - U_L),
   c = max(|un_L| + sqrt(g H_L), |un_R| + sqrt(g H_R)); out[7] = c, out[8] = 0; returns 0 dry, 3 otherwise */
int or_face_rusanov(double g, double h_eps, const double l[5], const double r[5], double out[9]);
/* Green-Ampt for one cell: in h_r (post-rain height), V, dt; out h*, V' */
void or_green_ampt(const or_params* P, double h_r, double V, double dt, double* h_out, double* V_out);
/* semi-implicit friction on one cell; state s = stage input, (hs,hus,hvs); (hst,hup,hvp) post-source */
void or_friction(double gcf, int law, double h_eps, double dt, double hs, double hus, double hvs,
                 double hst, double hup, double hvp, double* hu_out, double* hv_out);

/* ---- whole-array operations; arrays are row-major ny x nx without ghosts ---- */
/* CFL (Q10/Q17): dt = min(cfl/(ax/dx + ay/dy), dt_max, t_end - t). Writes ax, ay if non-NULL. */
double or_cfl_dt(const or_params* P, const double* h, const double* hu, const double* hv,
                 double t, double t_end, double* ax, double* ay);
/* CFL on reconstructed values (reading Q22): a_x = max over cells of the speeds
   |u| + sqrt(g h) of the cell's two x-face reconstructions (h_{i-1/2+}, u_{i-1/2+}), (h_{i+1/2-}, u_{i+1/2-})
   (ghosts filled at t_ghost), a_y likewise; dt as or_cfl_dt. */
double or_cfl_dt_face(const or_params* P, const double* z, const double* h, const double* hu, const double* hv,
                      double t_ghost, double t, double t_end, double* ax, double* ay);
/* one stage S(U, V; t_s, dt) of SURVEY.md §8c c1. v_in/v_out may be NULL if GA disabled.
   fric may be NULL (scalar coefficient). */
int or_stage(const or_params* P, const double* z, const double* fric,
             const double* h, const double* hu, const double* hv, const double* v_in,
             double t_s, double dt,
             double* h_out, double* hu_out, double* hv_out, double* v_out, or_counters* C);
/* one Heun step in place, with the given dt (t = t^n). */
int or_heun_step(const or_params* P, const double* z, const double* fric,
                 double* h, double* hu, double* hv, double* v, double t, double dt, or_counters* C);
/* time loop: nsteps steps (Heun; explicit Euler when order == 1) (or until t >= t_end), dt from the CFL of the current state unless
   dt_forced > 0.  dt_hist (capacity cap) receives every dt.  Returns 0 or a negative error. */
int or_run(const or_params* P, const double* z, const double* fric,
           double* h, double* hu, double* hv, double* v,
           double* t, int64_t nsteps, double t_end, double dt_forced,
           double* dt_hist, int64_t cap, int64_t* steps_done, or_counters* C);
/* D8 flow direction of a DEM (the user function listed at P:683-708): per cell,
   min = own value, index = 0; for the 8 neighbours i = 0..7 in the order E, SE, S, SW, W, NW, N, NE
   (SPEC.md flow_direction; j grows northwards), if (n_i > 0 && n_i < min) { index = i + 1; min = n_i; }.
   Neighbours outside the grid are absent.  dir receives 0..8. */
void or_flow_direction(const double* z, int32_t nx, int32_t ny, uint8_t* dir);
void or_flow_direction_f32(const float* z, int32_t nx, int32_t ny, uint8_t* dir);
/* fixed-order pairwise sum (volume audits) */
double or_pairwise_sum(const double* x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
