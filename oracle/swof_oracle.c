/*
 * swof_oracle.c -- CPU ORACLE (test infrastructure only; see swof_oracle.h).
 *
 * A plain, slow, single-threaded fp64 transcription of the scheme of PAPER.md §3,
 * organised as whole-array passes in the order of Algorithm 1.  No blocking, no
 * fusion: each pass reads the previous pass's arrays.  Evaluation order of every expression is
 * the canonical sheet of SURVEY.md §8c c1 (restated in DESIGN.md §3); compile with
 * -ffp-contract=off so that no multiply-add is contracted.
 */
#include "swof_oracle.h"

#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define GH 2 /* ghost width = scheme order */

/* Optional OpenMP-over-rows build (liboracle_omp.so, gcc -fopenmp; development aid for the full-size
 * digests of tools/oracle_digests.py): the outer row loops of the whole-array passes run in parallel.
 * Every element is still computed by the same expression from the same inputs, so the state is bitwise
 * identical to the serial build (tests/test_oracle_omp.py); only the order of the diagnostic counter
 * sums differs.  The default liboracle.so is built without -fopenmp: these pragmas are then inert. */
#ifdef _OPENMP
#define OR_PAR_FOR _Pragma("omp parallel for schedule(static)")
#define OR_PAR_FOR_RED(...) _Pragma(OR_STR(omp parallel for schedule(static) reduction(__VA_ARGS__)))
#define OR_PAR_FOR_SCHEME \
    _Pragma("omp parallel for schedule(static) reduction(+ : n_clamps, n_capped, n_cells, cl_mass) reduction(max : cl_max)")
#else
#define OR_PAR_FOR_SCHEME
#define OR_PAR_FOR
#define OR_PAR_FOR_RED(...)
#endif
#define OR_STR2(x) #x
#define OR_STR(x) OR_STR2(x)

static double dmin(double a, double b) { return (a < b) ? a : b; }
static double dmax(double a, double b) { return (a > b) ? a : b; }

/* ------------------------------------------------------------------------------------------ */
/* pointwise operations                                                                       */
/* ------------------------------------------------------------------------------------------ */

/* minmod limiter, exactly as printed */
double or_minmod(double a, double b) {
    if (a >= 0.0 && b >= 0.0) return dmin(a, b);
    if (a <= 0.0 && b <= 0.0) return dmax(a, b);
    return 0.0;
}

/* Canonical inverse cube root x^(-1/3) for finite x > 0: exponent split
 * x = m' 2^(3q) with m' in [0.5, 4), chord initial guess on the octave of m' (<= 2.7 % error), then
 * 4 Newton steps (error 2.7e-2 -> 1.5e-3 -> 4.3e-6 -> 3.7e-11 -> 2.7e-21)
 * y <- y + y (1 - m' y^3) / 3.  Used for h^(4/3) in Manning/Strickler friction and the
 * critical depth of the inflow ghost (Q18).  Pinned against libm cbrt in tests/test_oracle_unit.py. */
double or_icbrt(double x) {
    int e;
    double m = frexp(x, &e); /* x = m 2^e, m in [0.5, 1) */
    int q = (e >= 0) ? e / 3 : -((-e + 2) / 3);
    int r = e - 3 * q; /* 0, 1, 2 */
    double mp = ldexp(m, r);
    double lo, yl, yh;
    if (r == 0) { lo = 0.5; yl = 1.2599210498948732; yh = 1.0; }
    else if (r == 1) { lo = 1.0; yl = 1.0; yh = 0.7937005259840998; }
    else { lo = 2.0; yl = 0.7937005259840998; yh = 0.6299605249474366; }
    double y = yl + (yh - yl) * ((mp - lo) / lo);
    const double third = 1.0 / 3.0;
    for (int it = 0; it < 4; ++it) {
        double y3 = (y * y) * y;
        double t = 1.0 - mp * y3;
        y = y + (y * t) * third;
    }
    return ldexp(y, -q);
}

/* rain intensity R(t) >= 0, piecewise constant with half-open windows [t_k, t_k+1) (Q14) */
double or_rain_rate(const or_params* P, double t) {
    double R = 0.0;
    for (int k = 0; k < P->n_rain; ++k)
        if (t >= P->rain_t[k]) R = P->rain_rate[k];
    return R;
}

/* inflow hydrograph Q(t), piecewise linear between table points, constant beyond the ends */
double or_hydrograph(const or_params* P, int side, double t) {
    int n = P->n_hydro[side];
    const double* T = P->hydro_t[side];
    const double* Q = P->hydro_q[side];
    if (n <= 0) return 0.0;
    if (t <= T[0]) return Q[0];
    if (t >= T[n - 1]) return Q[n - 1];
    int k = 0;
    while (k + 1 < n - 1 && t >= T[k + 1]) ++k;
    return Q[k] + (Q[k + 1] - Q[k]) * ((t - T[k]) / (T[k + 1] - T[k]));
}

/* g*C_f for the two friction families: Manning C_f = n^2, Strickler 1/K^2,
 * Darcy-Weisbach f/(8g) (so g*C_f = f/8 exactly), Chezy 1/C^2. */
double or_friction_gcf(int law, double coef, double g) {
    switch (law) {
        case OR_FRIC_MANNING: return g * (coef * coef);
        case OR_FRIC_STRICKLER: return g / (coef * coef);
        case OR_FRIC_DARCY: return coef / 8.0;
        case OR_FRIC_CHEZY: return g / (coef * coef);
        default: return 0.0;
    }
}

/* MUSCL reconstruction of one cell along one axis.
 * Slopes: Ds = minmod((s_c - s_m)/dx, (s_p - s_c)/dx) and face = s_c -+ dx/2 Ds, read as
 * delta = 0.5 * minmod(s_c - s_m, s_p - s_c) (Q4; bitwise identical for power-of-two dx).
 * Reconstructed variables h, h+z, u, v; z deduced as eta - h (Q3).
 * Velocity modification: u_{i-1/2+} = u_i - (h_{i+1/2-}/h_i) delta_u and
 * u_{i+1/2-} = u_i + (h_{i-1/2+}/h_i) delta_u; on dry cells both faces take u_i (Q5). */
/* order 1 (first-order scheme): no reconstruction, every slope is 0, so each face carries the
 * cell value (z_face = eta - h as at second order) */
static void muscl_cell_ord(const double h3[3], const double eta3[3], const double u3[3], const double v3[3],
                           double rh_c, int order, double out[10]);

void or_muscl_cell(const double h3[3], const double eta3[3], const double u3[3], const double v3[3],
                   double rh_c, double out[10]) {
    muscl_cell_ord(h3, eta3, u3, v3, rh_c, 2, out);
}

static void muscl_cell_ord(const double h3[3], const double eta3[3], const double u3[3], const double v3[3],
                           double rh_c, int order, double out[10]) {
    double dh = 0.0, de = 0.0, du = 0.0, dv = 0.0;
    if (order != 1) {
        dh = 0.5 * or_minmod(h3[1] - h3[0], h3[2] - h3[1]);
        de = 0.5 * or_minmod(eta3[1] - eta3[0], eta3[2] - eta3[1]);
        du = 0.5 * or_minmod(u3[1] - u3[0], u3[2] - u3[1]);
        dv = 0.5 * or_minmod(v3[1] - v3[0], v3[2] - v3[1]);
    }
    double hm = h3[1] - dh, hp = h3[1] + dh;
    double em = eta3[1] - de, ep = eta3[1] + de;
    double zm = em - hm, zp = ep - hp; /* z deduced as eta - h on each face */
    double um, up, vm, vp;
    if (rh_c > 0.0) {
        double am = hp * rh_c; /* h_{i+1/2-}/h_i, used on the low face */
        double ap = hm * rh_c; /* h_{i-1/2+}/h_i, used on the high face */
        um = u3[1] - am * du;
        up = u3[1] + ap * du;
        vm = v3[1] - am * dv;
        vp = v3[1] + ap * dv;
    } else {
        um = up = u3[1];
        vm = vp = v3[1];
    }
    out[0] = hm; out[1] = hp; out[2] = em; out[3] = ep; out[4] = zm; out[5] = zp;
    out[6] = um; out[7] = up; out[8] = vm; out[9] = vp;
}

/* hydrostatic reconstruction at one face, read with eta_face - max(z) (Q7) */
static void hydrostatic(const double l[5], const double r[5], double* zs, double* HL, double* HR) {
    *zs = dmax(l[2], r[2]);
    *HL = dmax(l[1] - *zs, 0.0);
    *HR = dmax(r[1] - *zs, 0.0);
}

/* HLL numerical flux on U = (H, H*un, H*ut) with normal wave speeds
 * c1 = min(un_L - c_L, un_R - c_R), c2 = max(un_L + c_L, un_R + c_R); the transverse
 * momentum is the third HLL component (Q2).  Dry-dry face -> zero flux (Q8).
 * Returns the branch (0 dry, 1 F(U_L), 2 F(U_R), 3 middle). */
static int hll(double g, double h_eps, double HL, double nl, double tl, double HR, double nr, double tr,
               double F[3], double* c1o, double* c2o) {
    *c1o = 0.0; *c2o = 0.0;
    if (HL <= h_eps && HR <= h_eps) { F[0] = F[1] = F[2] = 0.0; return 0; }
    double g2 = 0.5 * g;
    double qL = HL * nl, pL = HL * tl;
    double qR = HR * nr, pR = HR * tr;
    double cL = sqrt(g * HL), cR = sqrt(g * HR);
    double c1 = dmin(nl - cL, nr - cR);
    double c2 = dmax(nl + cL, nr + cR);
    *c1o = c1; *c2o = c2;
    double FL[3] = {qL, qL * nl + g2 * (HL * HL), qL * tl};
    double FR[3] = {qR, qR * nr + g2 * (HR * HR), qR * tr};
    if (c1 >= 0.0) { F[0] = FL[0]; F[1] = FL[1]; F[2] = FL[2]; return 1; }
    if (c2 <= 0.0) { F[0] = FR[0]; F[1] = FR[1]; F[2] = FR[2]; return 2; }
    double UL[3] = {HL, qL, pL}, UR[3] = {HR, qR, pR};
    double rr = 1.0 / (c2 - c1);
    double m = c1 * c2;
    for (int k = 0; k < 3; ++k) F[k] = ((c2 * FL[k] - c1 * FR[k]) + m * (UR[k] - UL[k])) * rr;
    return 3;
}

/* Rusanov numerical flux (P:302 names it; textbook local Lax-Friedrichs form) on the same
 * U = (H, H*un, H*ut): F = (F(U_L) + F(U_R))/2 - (c/2)(U_R - U_L) with the single wave-speed bound
 * c = max(|un_L| + sqrt(g H_L), |un_R| + sqrt(g H_R)).  Dry-dry face -> zero flux (as Q8). */
static int rusanov(double g, double h_eps, double HL, double nl, double tl, double HR, double nr, double tr,
                   double F[3], double* co) {
    *co = 0.0;
    if (HL <= h_eps && HR <= h_eps) { F[0] = F[1] = F[2] = 0.0; return 0; }
    double g2 = 0.5 * g;
    double qL = HL * nl, pL = HL * tl;
    double qR = HR * nr, pR = HR * tr;
    double cL = sqrt(g * HL), cR = sqrt(g * HR);
    double c = dmax(fabs(nl) + cL, fabs(nr) + cR);
    *co = c;
    double FL[3] = {qL, qL * nl + g2 * (HL * HL), qL * tl};
    double FR[3] = {qR, qR * nr + g2 * (HR * HR), qR * tr};
    double UL[3] = {HL, qL, pL}, UR[3] = {HR, qR, pR};
    double hc = 0.5 * c;
    for (int k = 0; k < 3; ++k) F[k] = 0.5 * (FL[k] + FR[k]) - hc * (UR[k] - UL[k]);
    return 3;
}

/* interface source corrections S_{i+1/2L}, S_{i-1/2R} */
static void iface_sources(double g, double hl, double HL, double hr, double HR, double* SL, double* SR) {
    double g2 = 0.5 * g;
    *SL = g2 * (hl * hl - HL * HL);
    *SR = g2 * (hr * hr - HR * HR);
}

/* centred slope source Fc_i = -g (h_{i-1/2+} + h_{i+1/2-})/2 (z_{i+1/2-} - z_{i-1/2+}),
 * evaluated as (g/2 (h_m + h_p)) (z_m - z_p) */
double or_centered_source(double g, double hm, double hp, double zm, double zp) {
    return (0.5 * g * (hm + hp)) * (zm - zp);
}

int or_face(double g, double h_eps, const double l[5], const double r[5], double out[9]) {
    double zs, HL, HR, F[3], c1, c2, SL, SR;
    hydrostatic(l, r, &zs, &HL, &HR);
    int br = hll(g, h_eps, HL, l[3], l[4], HR, r[3], r[4], F, &c1, &c2);
    iface_sources(g, l[0], HL, r[0], HR, &SL, &SR);
    out[0] = F[0]; out[1] = F[1]; out[2] = F[2]; out[3] = SL; out[4] = SR;
    out[5] = HL; out[6] = HR; out[7] = c1; out[8] = c2;
    return br;
}

int or_face_rusanov(double g, double h_eps, const double l[5], const double r[5], double out[9]) {
    double zs, HL, HR, F[3], c, SL, SR;
    hydrostatic(l, r, &zs, &HL, &HR);
    int br = rusanov(g, h_eps, HL, l[3], l[4], HR, r[3], r[4], F, &c);
    iface_sources(g, l[0], HL, r[0], HR, &SL, &SR);
    out[0] = F[0]; out[1] = F[1]; out[2] = F[2]; out[3] = SL; out[4] = SR;
    out[5] = HL; out[6] = HR; out[7] = c; out[8] = 0.0;
    return br;
}

/* modified Green-Ampt: I_C = K_s (A + (h_f - h_over)/Z_f), Z_f = V/dtheta, read as
 * K_s (A + ((h_f - h_over) dtheta)/V), clamped >= 0; infiltrated depth min(h_over, dt I_C);
 * V = 0 -> unlimited capacity (limit of the printed formula, Q15). */
void or_green_ampt(const or_params* P, double h_r, double V, double dt, double* h_out, double* V_out) {
    double cap;
    if (V == 0.0) cap = INFINITY;
    else {
        /* as printed: h_f - h_over; the Darcy-consistent switch (Q15) takes h_f + h_over */
        double dh = (P->ga_form == OR_GA_DARCY) ? P->ga_hf + h_r : P->ga_hf - h_r;
        cap = dmax(P->ga_Ks * (P->ga_A + (dh * P->ga_dtheta) / V), 0.0) * dt;
    }
    double inf = dmin(h_r, cap);
    *h_out = h_r - inf;
    *V_out = V + inf;
}

/* semi-implicit friction generalised to both families (Q11):
 * q^{n+1} = q* / (1 + dt gC_f |u^n| / h*^a), a = 4/3 (Manning/Strickler) or 1 (Darcy/Chezy);
 * |u^n| from the stage-input state; dry cells (h* <= h_eps) carry no momentum. */
void or_friction(double gcf, int law, double h_eps, double dt, double hs, double hus, double hvs,
                 double hst, double hup, double hvp, double* hu_out, double* hv_out) {
    if (hst <= h_eps) { *hu_out = 0.0; *hv_out = 0.0; return; }
    if (law == OR_FRIC_NONE) { *hu_out = hup; *hv_out = hvp; return; }
    double rhs = (hs > h_eps) ? 1.0 / hs : 0.0;
    double umag = sqrt(hus * hus + hvs * hvs) * rhs;
    double k = (dt * gcf) * umag;
    double w;
    if (law == OR_FRIC_MANNING || law == OR_FRIC_STRICKLER) {
        double s = or_icbrt(hst); /* h*^(-1/3) */
        w = k * ((s * s) * (s * s));
    } else {
        w = k / hst;
    }
    double rd = 1.0 / (1.0 + w); /* q* / (1 + ...) evaluated as q* (1 / (1 + ...)) */
    *hu_out = hup * rd;
    *hv_out = hvp * rd;
}

/* ------------------------------------------------------------------------------------------ */
/* whole-array passes                                                                          */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
    int nx, ny, pw; /* padded width = nx + 4 */
    /* padded state for the stage being evaluated */
    double *h, *hu, *hv, *z;
    /* primitives (padded) */
    double *rh, *u, *v, *eta;
    /* reconstruction, per axis, padded layout: [axis][10] */
    double* rec[2][10];
    /* per-face arrays: x faces (ny rows, nx+1), y faces (ny+1 rows, nx) */
    double *fx_zs, *fx_HL, *fx_HR, *fx_Fm, *fx_Fn, *fx_Ft, *fx_SL, *fx_SR;
    double *fy_zs, *fy_HL, *fy_HR, *fy_Fm, *fy_Fn, *fy_Ft, *fy_SL, *fy_SR;
    /* post-source fields before friction (interior) */
    double *hs, *hup, *hvp;
    /* stage outputs (interior) */
    double *U1h, *U1hu, *U1hv, *U1v, *U2h, *U2hu, *U2hv, *U2v;
} ws_t;

#define PIX(W, i, j) ((size_t)((j) + GH) * (size_t)(W)->pw + (size_t)((i) + GH))

static void* xcalloc(size_t n) { return calloc(n ? n : 1, sizeof(double)); }

static int ws_alloc(ws_t* W, int nx, int ny) {
    memset(W, 0, sizeof(*W));
    W->nx = nx; W->ny = ny; W->pw = nx + 2 * GH;
    size_t np = (size_t)(nx + 2 * GH) * (size_t)(ny + 2 * GH);
    size_t nfx = (size_t)ny * (size_t)(nx + 1), nfy = (size_t)(ny + 1) * (size_t)nx;
    size_t nc = (size_t)nx * (size_t)ny;
    double** padded[] = {&W->h, &W->hu, &W->hv, &W->z, &W->rh, &W->u, &W->v, &W->eta};
    for (unsigned k = 0; k < sizeof(padded) / sizeof(padded[0]); ++k)
        if (!(*padded[k] = xcalloc(np))) return -1;
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 10; ++k)
            if (!(W->rec[a][k] = xcalloc(np))) return -1;
    double** fx[] = {&W->fx_zs, &W->fx_HL, &W->fx_HR, &W->fx_Fm, &W->fx_Fn, &W->fx_Ft, &W->fx_SL, &W->fx_SR};
    double** fy[] = {&W->fy_zs, &W->fy_HL, &W->fy_HR, &W->fy_Fm, &W->fy_Fn, &W->fy_Ft, &W->fy_SL, &W->fy_SR};
    for (int k = 0; k < 8; ++k) {
        if (!(*fx[k] = xcalloc(nfx))) return -1;
        if (!(*fy[k] = xcalloc(nfy))) return -1;
    }
    double** cells[] = {&W->hs, &W->hup, &W->hvp, &W->U1h, &W->U1hu, &W->U1hv, &W->U1v,
                        &W->U2h, &W->U2hu, &W->U2hv, &W->U2v};
    for (unsigned k = 0; k < sizeof(cells) / sizeof(cells[0]); ++k)
        if (!(*cells[k] = xcalloc(nc))) return -1;
    return 0;
}

static void ws_free(ws_t* W) {
    double* all[] = {W->h, W->hu, W->hv, W->z, W->rh, W->u, W->v, W->eta,
                     W->fx_zs, W->fx_HL, W->fx_HR, W->fx_Fm, W->fx_Fn, W->fx_Ft, W->fx_SL, W->fx_SR,
                     W->fy_zs, W->fy_HL, W->fy_HR, W->fy_Fm, W->fy_Fn, W->fy_Ft, W->fy_SL, W->fy_SR,
                     W->hs, W->hup, W->hvp, W->U1h, W->U1hu, W->U1hv, W->U1v, W->U2h, W->U2hu, W->U2hv, W->U2v};
    for (unsigned k = 0; k < sizeof(all) / sizeof(all[0]); ++k) free(all[k]);
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 10; ++k) free(W->rec[a][k]);
}

/* ---- Algorithm 1 step "Boundary Conditions" ----
 * Ghost cells, 2 layers.  WALL: exact mirror of interior layers 0 and 1 with the normal discharge
 * negated (Q16); FREE: zero-gradient copy of layer 0 (h, q, z); PERIODIC: wrap; INFLOW: on the
 * segment [k0, k1) both variables imposed, (h_c, q_in, 0) with h_c = (q^2/g)^(1/3) the critical
 * depth (Q18), z copied from layer 0; outside the segment the side is a WALL. */
static int wrap(int i, int n) { int r = i % n; return r < 0 ? r + n : r; }

static double inflow_q(const or_params* P, int side, double t) {
    double width = (double)(P->in_k1[side] - P->in_k0[side]) * ((side == OR_W || side == OR_E) ? P->dy : P->dx);
    return or_hydrograph(P, side, t) / width;
}

static double critical_depth(double q, double g) {
    if (q == 0.0) return 0.0;
    double x = (q * q) / g;
    double s = or_icbrt(x);
    return x * (s * s);
}

static void fill_ghosts(const or_params* P, ws_t* W, double t_s) {
    int nx = W->nx, ny = W->ny;
    /* x sides: rows j in [0, ny) */
    for (int side = OR_W; side <= OR_E; ++side) {
        int type = P->bc[side];
        double q = 0.0, hc = 0.0;
        if (type == OR_BC_INFLOW) { q = inflow_q(P, side, t_s); hc = critical_depth(q, P->g); }
        for (int j = 0; j < ny; ++j) {
            for (int k = 0; k < GH; ++k) {
                int gi = (side == OR_W) ? -1 - k : nx + k;
                size_t d = PIX(W, gi, j);
                int inseg = (type == OR_BC_INFLOW) && j >= P->in_k0[side] && j < P->in_k1[side];
                int src; double sgn = 1.0;
                if (type == OR_BC_PERIODIC) src = wrap(gi, nx);
                else if (type == OR_BC_FREE || inseg) src = (side == OR_W) ? 0 : nx - 1;
                else { int kk = k < nx - 1 ? k : nx - 1; src = (side == OR_W) ? kk : nx - 1 - kk; sgn = -1.0; }
                size_t s = PIX(W, src, j);
                W->z[d] = W->z[s];
                if (inseg) {
                    W->h[d] = hc; W->hu[d] = (side == OR_W) ? q : -q; W->hv[d] = 0.0;
                } else {
                    W->h[d] = W->h[s]; W->hu[d] = sgn * W->hu[s]; W->hv[d] = W->hv[s];
                }
            }
        }
    }
    /* y sides: columns i in [0, nx) */
    for (int side = OR_S; side <= OR_N; ++side) {
        int type = P->bc[side];
        double q = 0.0, hc = 0.0;
        if (type == OR_BC_INFLOW) { q = inflow_q(P, side, t_s); hc = critical_depth(q, P->g); }
        for (int i = 0; i < nx; ++i) {
            for (int k = 0; k < GH; ++k) {
                int gj = (side == OR_S) ? -1 - k : ny + k;
                size_t d = PIX(W, i, gj);
                int inseg = (type == OR_BC_INFLOW) && i >= P->in_k0[side] && i < P->in_k1[side];
                int src; double sgn = 1.0;
                if (type == OR_BC_PERIODIC) src = wrap(gj, ny);
                else if (type == OR_BC_FREE || inseg) src = (side == OR_S) ? 0 : ny - 1;
                else { int kk = k < ny - 1 ? k : ny - 1; src = (side == OR_S) ? kk : ny - 1 - kk; sgn = -1.0; }
                size_t s = PIX(W, i, src);
                W->z[d] = W->z[s];
                if (inseg) {
                    W->h[d] = hc; W->hu[d] = 0.0; W->hv[d] = (side == OR_S) ? q : -q;
                } else {
                    W->h[d] = W->h[s]; W->hu[d] = W->hu[s]; W->hv[d] = sgn * W->hv[s];
                }
            }
        }
    }
}

/* ---- Algorithm 1 step "Second order reconstruction" ----
 * primitives on every cell incl. ghosts: rh = 1/h on wet cells (h > h_eps, Q6) else 0, u = hu rh,
 * v = hv rh, eta = h + z; then MUSCL per axis on cells -1 .. n (ghost layer 0 included). */
static void primitives(const or_params* P, ws_t* W) {
    OR_PAR_FOR
    for (int j = -GH; j < W->ny + GH; ++j)
        for (int i = -GH; i < W->nx + GH; ++i) {
            size_t c = PIX(W, i, j);
            double h = W->h[c];
            double rh = (h > P->h_eps) ? 1.0 / h : 0.0;
            W->rh[c] = rh;
            W->u[c] = W->hu[c] * rh;
            W->v[c] = W->hv[c] * rh;
            W->eta[c] = h + W->z[c];
        }
}

static void muscl_axis(ws_t* W, int axis, int order) {
    /* axis 0: x (neighbours i-1, i+1; normal velocity u); axis 1: y (j-1, j+1; normal velocity v) */
    int nx = W->nx, ny = W->ny;
    int i0 = axis == 0 ? -1 : 0, i1 = axis == 0 ? nx + 1 : nx;
    int j0 = axis == 0 ? 0 : -1, j1 = axis == 0 ? ny : ny + 1;
    ptrdiff_t st = axis == 0 ? 1 : W->pw;
    const double* un = axis == 0 ? W->u : W->v;
    const double* ut = axis == 0 ? W->v : W->u;
    OR_PAR_FOR
    for (int j = j0; j < j1; ++j)
        for (int i = i0; i < i1; ++i) {
            size_t c = PIX(W, i, j);
            double h3[3] = {W->h[c - st], W->h[c], W->h[c + st]};
            double e3[3] = {W->eta[c - st], W->eta[c], W->eta[c + st]};
            double n3[3] = {un[c - st], un[c], un[c + st]};
            double t3[3] = {ut[c - st], ut[c], ut[c + st]};
            double out[10];
            muscl_cell_ord(h3, e3, n3, t3, W->rh[c], order, out);
            for (int k = 0; k < 10; ++k) W->rec[axis][k][c] = out[k];
        }
}

enum { R_HM = 0, R_HP, R_EM, R_EP, R_ZM, R_ZP, R_NM, R_NP, R_TM, R_TP };

/* face f along an axis lies between cell L (index f-1) and R (index f) */
static void face_lr(const ws_t* W, int axis, int f, int row, double l[5], double r[5]) {
    size_t cl = axis == 0 ? PIX(W, f - 1, row) : PIX(W, row, f - 1);
    size_t cr = axis == 0 ? PIX(W, f, row) : PIX(W, row, f);
    double* const* R = W->rec[axis];
    l[0] = R[R_HP][cl]; l[1] = R[R_EP][cl]; l[2] = R[R_ZP][cl]; l[3] = R[R_NP][cl]; l[4] = R[R_TP][cl];
    r[0] = R[R_HM][cr]; r[1] = R[R_EM][cr]; r[2] = R[R_ZM][cr]; r[3] = R[R_NM][cr]; r[4] = R[R_TM][cr];
}

/* ---- Algorithm 1 step "Hydrostatic reconstruction" ---- */
static void hydrostatic_axis(ws_t* W, int axis) {
    int nf = axis == 0 ? W->nx + 1 : W->ny + 1;
    int nr = axis == 0 ? W->ny : W->nx;
    double* ZS = axis == 0 ? W->fx_zs : W->fy_zs;
    double* HL = axis == 0 ? W->fx_HL : W->fy_HL;
    double* HR = axis == 0 ? W->fx_HR : W->fy_HR;
    OR_PAR_FOR
    for (int row = 0; row < nr; ++row)
        for (int f = 0; f < nf; ++f) {
            double l[5], r[5];
            face_lr(W, axis, f, row, l, r);
            size_t k = axis == 0 ? (size_t)row * nf + f : (size_t)f * nr + row;
            hydrostatic(l, r, &ZS[k], &HL[k], &HR[k]);
        }
}

/* ---- Algorithm 1 step "Numerical flux computation" ---- */
static void flux_axis(const or_params* P, ws_t* W, int axis, or_counters* C) {
    int nf = axis == 0 ? W->nx + 1 : W->ny + 1;
    int nr = axis == 0 ? W->ny : W->nx;
    double* HL = axis == 0 ? W->fx_HL : W->fy_HL;
    double* HR = axis == 0 ? W->fx_HR : W->fy_HR;
    double* Fm = axis == 0 ? W->fx_Fm : W->fy_Fm;
    double* Fn = axis == 0 ? W->fx_Fn : W->fy_Fn;
    double* Ft = axis == 0 ? W->fx_Ft : W->fy_Ft;
    double* SL = axis == 0 ? W->fx_SL : W->fy_SL;
    double* SR = axis == 0 ? W->fx_SR : W->fy_SR;
    long long n_dry = 0, n_left = 0, n_right = 0, n_mid = 0;
    OR_PAR_FOR_RED(+ : n_dry, n_left, n_right, n_mid)
    for (int row = 0; row < nr; ++row)
        for (int f = 0; f < nf; ++f) {
            double l[5], r[5], F[3], c1, c2;
            face_lr(W, axis, f, row, l, r);
            size_t k = axis == 0 ? (size_t)row * nf + f : (size_t)f * nr + row;
            int br = (P->flux == OR_FLUX_RUSANOV)
                         ? rusanov(P->g, P->h_eps, HL[k], l[3], l[4], HR[k], r[3], r[4], F, &c1)
                         : hll(P->g, P->h_eps, HL[k], l[3], l[4], HR[k], r[3], r[4], F, &c1, &c2);
            iface_sources(P->g, l[0], HL[k], r[0], HR[k], &SL[k], &SR[k]);
            Fm[k] = F[0]; Fn[k] = F[1]; Ft[k] = F[2];
            if (br == 0) n_dry++;
            else if (br == 1) n_left++;
            else if (br == 2) n_right++;
            else n_mid++;
        }
    if (C) {
        C->face_dry += n_dry;
        C->face_left += n_left;
        C->face_right += n_right;
        C->face_mid += n_mid;
    }
}

/* ---- Algorithm 1 step "Scheme computation" ----
 * U' = U - dt/dx [F_{i+1/2L} - F_{i-1/2R} - Fc_i] per axis, summed over the two axes (Q1);
 * Fc_i = -g (h_{i-1/2+} + h_{i+1/2-})/2 (z_{i+1/2-} - z_{i-1/2+}); then clamp h' >= 0
 * (Q17), explicit rain h + R(t_s) dt, Green-Ampt. */
static void scheme(const or_params* P, ws_t* W, const double* v_in, double t_s, double dt,
                   double* v_out, or_counters* C) {
    int nx = W->nx, ny = W->ny;
    double lx = dt / P->dx, ly = dt / P->dy;
    double Rdt = or_rain_rate(P, t_s) * dt;
    long long n_clamps = 0, n_capped = 0, n_cells = 0;
    double cl_mass = 0.0, cl_max = C ? C->clamp_max : 0.0;
    OR_PAR_FOR_SCHEME
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t c = PIX(W, i, j);
            size_t ic = (size_t)j * nx + i;
            size_t xw = (size_t)j * (nx + 1) + i, xe = xw + 1;             /* x faces i, i+1 */
            size_t ys = (size_t)j * nx + i, yn = (size_t)(j + 1) * nx + i; /* y faces j, j+1 */
            double* const* X = W->rec[0];
            double* const* Y = W->rec[1];
            double Fcx = or_centered_source(P->g, X[R_HM][c], X[R_HP][c], X[R_ZM][c], X[R_ZP][c]);
            double Fcy = or_centered_source(P->g, Y[R_HM][c], Y[R_HP][c], Y[R_ZM][c], Y[R_ZP][c]);
            double Dmx = W->fx_Fm[xe] - W->fx_Fm[xw];
            double Dnx = ((W->fx_Fn[xe] + W->fx_SL[xe]) - (W->fx_Fn[xw] + W->fx_SR[xw])) - Fcx;
            double Dtx = W->fx_Ft[xe] - W->fx_Ft[xw];
            double Dmy = W->fy_Fm[yn] - W->fy_Fm[ys];
            double Dny = ((W->fy_Fn[yn] + W->fy_SL[yn]) - (W->fy_Fn[ys] + W->fy_SR[ys])) - Fcy;
            double Dty = W->fy_Ft[yn] - W->fy_Ft[ys];
            double h1 = W->h[c] - (lx * Dmx + ly * Dmy);
            double hu1 = W->hu[c] - (lx * Dnx + ly * Dty);
            double hv1 = W->hv[c] - (lx * Dtx + ly * Dny);
            if (h1 < 0.0) {
                n_clamps++;
                cl_mass += -h1;
                if (-h1 > cl_max) cl_max = -h1;
                h1 = 0.0;
            }
            double hr = h1 + Rdt;
            double hst = hr, V = 0.0;
            if (P->ga_enabled) {
                or_green_ampt(P, hr, v_in[ic], dt, &hst, &V);
                v_out[ic] = V;
                if (v_in[ic] != 0.0) n_capped++;
            }
            W->hs[ic] = hst;
            W->hup[ic] = hu1;
            W->hvp[ic] = hv1;
            n_cells++;
        }
    if (C) {
        C->clamps += n_clamps;
        C->clamped_mass += cl_mass;
        C->clamp_max = cl_max;
        C->ga_capped += n_capped;
        C->cell_stage += n_cells;
    }
}

/* ---- Algorithm 1 step "Frictions" ---- */
static void frictions(const or_params* P, ws_t* W, const double* fric, const double* h_in,
                      const double* hu_in, const double* hv_in, double dt,
                      double* h_out, double* hu_out, double* hv_out, or_counters* C) {
    size_t n = (size_t)W->nx * W->ny;
    double gcf0 = or_friction_gcf(P->fric_law, P->fric_coef, P->g);
    long long n_wet = 0;
    OR_PAR_FOR_RED(+ : n_wet)
    for (size_t c = 0; c < n; ++c) {
        double gcf = fric ? or_friction_gcf(P->fric_law, fric[c], P->g) : gcf0;
        double hu, hv;
        or_friction(gcf, P->fric_law, P->h_eps, dt, h_in[c], hu_in[c], hv_in[c],
                    W->hs[c], W->hup[c], W->hvp[c], &hu, &hv);
        if (W->hs[c] > P->h_eps && P->fric_law != OR_FRIC_NONE) n_wet++;
        h_out[c] = W->hs[c];
        hu_out[c] = hu;
        hv_out[c] = hv;
    }
    if (C) C->cell_wet_fric += n_wet;
}

static void load_padded(ws_t* W, const double* z, const double* h, const double* hu, const double* hv) {
    OR_PAR_FOR
    for (int j = 0; j < W->ny; ++j)
        for (int i = 0; i < W->nx; ++i) {
            size_t c = PIX(W, i, j), s = (size_t)j * W->nx + i;
            W->z[c] = z[s]; W->h[c] = h[s]; W->hu[c] = hu[s]; W->hv[c] = hv[s];
        }
}

/* one stage S of SURVEY.md §8c c1, Algorithm 1 body */
static void stage_ws(const or_params* P, ws_t* W, const double* z, const double* fric,
                     const double* h, const double* hu, const double* hv, const double* v_in,
                     double t_s, double dt, double* h_out, double* hu_out, double* hv_out, double* v_out,
                     or_counters* C) {
    load_padded(W, z, h, hu, hv);
    fill_ghosts(P, W, t_s);               /* Boundary Conditions */
    primitives(P, W);                     /* Second order reconstruction */
    muscl_axis(W, 0, P->order);
    muscl_axis(W, 1, P->order);
    hydrostatic_axis(W, 0);               /* Hydrostatic reconstruction */
    hydrostatic_axis(W, 1);
    flux_axis(P, W, 0, C);                /* Numerical flux computation */
    flux_axis(P, W, 1, C);
    scheme(P, W, v_in, t_s, dt, v_out, C);/* Scheme computation */
    frictions(P, W, fric, h, hu, hv, dt, h_out, hu_out, hv_out, C); /* Frictions */
}

int or_stage(const or_params* P, const double* z, const double* fric,
             const double* h, const double* hu, const double* hv, const double* v_in,
             double t_s, double dt, double* h_out, double* hu_out, double* hv_out, double* v_out,
             or_counters* C) {
    ws_t W;
    if (ws_alloc(&W, P->nx, P->ny)) { ws_free(&W); return -1; }
    stage_ws(P, &W, z, fric, h, hu, hv, v_in, t_s, dt, h_out, hu_out, hv_out, v_out, C);
    ws_free(&W);
    return 0;
}

/* Heun's predictor-corrector: U* = S(U^n; t^n), U** = S(U*; t^n + dt),
 * U^{n+1} = (U^n + U**)/2; V is averaged the same way (Q12). */
static void heun_ws(const or_params* P, ws_t* W, const double* z, const double* fric,
                    double* h, double* hu, double* hv, double* v, double t, double dt, or_counters* C) {
    size_t n = (size_t)P->nx * P->ny;
    stage_ws(P, W, z, fric, h, hu, hv, v, t, dt, W->U1h, W->U1hu, W->U1hv, W->U1v, C);
    stage_ws(P, W, z, fric, W->U1h, W->U1hu, W->U1hv, W->U1v, t + dt, dt,
             W->U2h, W->U2hu, W->U2hv, W->U2v, C);
    OR_PAR_FOR
    for (size_t c = 0; c < n; ++c) {
        h[c] = 0.5 * (h[c] + W->U2h[c]);
        hu[c] = 0.5 * (hu[c] + W->U2hu[c]);
        hv[c] = 0.5 * (hv[c] + W->U2hv[c]);
        if (P->ga_enabled) v[c] = 0.5 * (v[c] + W->U2v[c]);
    }
}

/* explicit Euler for the first-order scheme (order 1): U^{n+1} = S(U^n; t^n) */
static void euler_ws(const or_params* P, ws_t* W, const double* z, const double* fric,
                     double* h, double* hu, double* hv, double* v, double t, double dt, or_counters* C) {
    size_t n = (size_t)P->nx * P->ny;
    stage_ws(P, W, z, fric, h, hu, hv, v, t, dt, W->U1h, W->U1hu, W->U1hv, W->U1v, C);
    OR_PAR_FOR
    for (size_t c = 0; c < n; ++c) {
        h[c] = W->U1h[c];
        hu[c] = W->U1hu[c];
        hv[c] = W->U1hv[c];
        if (P->ga_enabled) v[c] = W->U1v[c];
    }
}

int or_heun_step(const or_params* P, const double* z, const double* fric,
                 double* h, double* hu, double* hv, double* v, double t, double dt, or_counters* C) {
    ws_t W;
    if (ws_alloc(&W, P->nx, P->ny)) { ws_free(&W); return -1; }
    heun_ws(P, &W, z, fric, h, hu, hv, v, t, dt, C);
    ws_free(&W);
    return 0;
}

/* CFL condition on cell-centred values (Q10): a_x = max(|u| + sqrt(g h)),
 * a_y = max(|v| + sqrt(g h)); dt = min(n_CFL / (a_x/dx + a_y/dy), dt_max, t_end - t).
 * The 2D sum form is the positivity condition of the additive two-axis update (Q17): the min form
 * n_CFL min(dx/a_x, dy/a_y) let real clamps (2 cm) appear on cfg4-like puddles. */
double or_cfl_dt(const or_params* P, const double* h, const double* hu, const double* hv,
                 double t, double t_end, double* axo, double* ayo) {
    size_t n = (size_t)P->nx * P->ny;
    double ax = 0.0, ay = 0.0;
    for (size_t c = 0; c < n; ++c) {
        double rh = (h[c] > P->h_eps) ? 1.0 / h[c] : 0.0;
        double cc = sqrt(P->g * h[c]);
        double su = fabs(hu[c] * rh) + cc;
        double sv = fabs(hv[c] * rh) + cc;
        if (su > ax || su != su) ax = su; /* a NaN, once seen, stays */
        if (sv > ay || sv != sv) ay = sv;
    }
    if (axo) *axo = ax;
    if (ayo) *ayo = ay;
    double dt = P->cfl / (ax / P->dx + ay / P->dy); /* 2D sum form (Q17 reading) */
    dt = dmin(dt, P->dt_max);
    dt = dmin(dt, t_end - t);
    return dt;
}

/* CFL on the reconstructed values: "at second order, variables (h_i, u_i) in (cfl) are
 * replaced by the reconstructed values".  Read (Q22) as: every cell contributes the speeds of
 * its own two face reconstructions per axis, |u_{i-1/2+}| + sqrt(g h_{i-1/2+}) and
 * |u_{i+1/2-}| + sqrt(g h_{i+1/2-}) (MUSCL values with the velocity modification, before the
 * hydrostatic reconstruction; ghosts at t_ghost feed the slopes of the edge cells).  At order 1 the
 * faces carry the cell values, so this equals or_cfl_dt. */
double or_cfl_dt_face(const or_params* P, const double* z, const double* h, const double* hu, const double* hv,
                      double t_ghost, double t, double t_end, double* axo, double* ayo) {
    ws_t W;
    if (ws_alloc(&W, P->nx, P->ny)) { ws_free(&W); return NAN; }
    load_padded(&W, z, h, hu, hv);
    fill_ghosts(P, &W, t_ghost);
    primitives(P, &W);
    muscl_axis(&W, 0, P->order);
    muscl_axis(&W, 1, P->order);
    double a[2] = {0.0, 0.0};
    for (int axis = 0; axis < 2; ++axis)
        for (int j = 0; j < P->ny; ++j)
            for (int i = 0; i < P->nx; ++i) {
                size_t c = PIX(&W, i, j);
                double* const* R = W.rec[axis];
                double sm = fabs(R[R_NM][c]) + sqrt(P->g * R[R_HM][c]);
                double sp = fabs(R[R_NP][c]) + sqrt(P->g * R[R_HP][c]);
                if (sm > a[axis] || sm != sm) a[axis] = sm;
                if (sp > a[axis] || sp != sp) a[axis] = sp;
            }
    ws_free(&W);
    if (axo) *axo = a[0];
    if (ayo) *ayo = a[1];
    double dt = P->cfl / (a[0] / P->dx + a[1] / P->dy);
    dt = dmin(dt, P->dt_max);
    dt = dmin(dt, t_end - t);
    return dt;
}

int or_run(const or_params* P, const double* z, const double* fric,
           double* h, double* hu, double* hv, double* v,
           double* t, int64_t nsteps, double t_end, double dt_forced,
           double* dt_hist, int64_t cap, int64_t* steps_done, or_counters* C) {
    ws_t W;
    if (ws_alloc(&W, P->nx, P->ny)) { ws_free(&W); return -1; }
    int64_t n = 0;
    int rc = 0;
    for (; n < nsteps; ++n) {
        if (*t >= t_end) break;
        double dt = dt_forced > 0.0 ? dt_forced
                  : (P->cfl_mode == OR_CFL_FACE) ? or_cfl_dt_face(P, z, h, hu, hv, *t, *t, t_end, NULL, NULL)
                  : or_cfl_dt(P, h, hu, hv, *t, t_end, NULL, NULL);
        if (!isfinite(dt) || !(dt > 0.0)) { rc = -2; break; }
        if (P->order == 1) euler_ws(P, &W, z, fric, h, hu, hv, v, *t, dt, C);
        else heun_ws(P, &W, z, fric, h, hu, hv, v, *t, dt, C);
        *t = *t + dt;
        if (dt_hist && n < cap) dt_hist[n] = dt;
    }
    if (steps_done) *steps_done = n;
    ws_free(&W);
    return rc;
}

double or_pairwise_sum(const double* x, int64_t n) {
    if (n <= 8) {
        double s = 0.0;
        for (int64_t k = 0; k < n; ++k) s += x[k];
        return s;
    }
    int64_t m = n / 2;
    return or_pairwise_sum(x, m) + or_pairwise_sum(x + m, n - m);
}

/* ------------------------------------------------------------------------------------------ */
/* D8 flow direction: "getting the minimum value for the eight neighbors around the */
/* current point and saving the corresponding direction", transcribed from the listing P:683-708 */
/* ------------------------------------------------------------------------------------------ */
static const int D8_DI[8] = {1, 1, 0, -1, -1, -1, 0, 1};   /* E, SE, S, SW, W, NW, N, NE */
static const int D8_DJ[8] = {0, -1, -1, -1, 0, 1, 1, 1};

void or_flow_direction(const double* z, int32_t nx, int32_t ny, uint8_t* dir) {
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            int index = 0;
            double min = z[(size_t)j * nx + i];
            for (int k = 0; k < 8; ++k) {
                int ii = i + D8_DI[k], jj = j + D8_DJ[k];
                if (ii < 0 || ii >= nx || jj < 0 || jj >= ny) continue;   /* absent neighbour */
                double n = z[(size_t)jj * nx + ii];
                if (n > 0 && n < min) {
                    index = k + 1;
                    min = n;
                }
            }
            dir[(size_t)j * nx + i] = (uint8_t)index;
        }
}

void or_flow_direction_f32(const float* z, int32_t nx, int32_t ny, uint8_t* dir) {
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            int index = 0;
            float min = z[(size_t)j * nx + i];
            for (int k = 0; k < 8; ++k) {
                int ii = i + D8_DI[k], jj = j + D8_DJ[k];
                if (ii < 0 || ii >= nx || jj < 0 || jj >= ny) continue;
                float n = z[(size_t)jj * nx + ii];
                if (n > 0 && n < min) {
                    index = k + 1;
                    min = n;
                }
            }
            dir[(size_t)j * nx + i] = (uint8_t)index;
        }
}
