/* examples/lake_and_dam.c -- the C ABI (include/swof.h) from plain C, no Python and no CUDA calls: host
 * arrays in, host arrays out.
 *
 *   gcc -O2 -I include examples/lake_and_dam.c -L paper_1307_4839_b200 -lswof \
 *       -Wl,-rpath,$PWD/paper_1307_4839_b200 -o examples/lake_and_dam && examples/lake_and_dam
 *
 * Two runs on one B200:
 *  1. lake at rest over a Gaussian bump, closed walls, Manning friction: the scheme is well balanced
 *     (hydrostatic reconstruction), so the discharges stay zero to round-off and the free surface
 *     flat;
 *  2. a dam break onto a dry, sloping bed with walls: h >= 0 everywhere (positivity) and the
 *     water volume conserved to round-off (no rain, no infiltration, no outflow).
 * Prints one line per run and exits non-zero if a property fails. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "swof.h"

#define CHECK(x)                                                                        \
    do {                                                                                \
        int rc_ = (x);                                                                  \
        if (rc_ != SWOF_OK) {                                                           \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, swof_strerror(rc_));       \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

static void defaults(swof_params* p, int nx, int ny, double dx) {
    memset(p, 0, sizeof(*p));
    p->nx = nx;
    p->ny = ny;
    p->dx = p->dy = dx;
    p->g = 9.81;
    p->cfl = 0.4;
    p->dt_max = 1.0;
    p->h_eps = 1e-12;
    p->fric_law = SWOF_FRIC_MANNING;
    p->fric_coef = 0.03;
    for (int s = 0; s < 4; ++s) p->bc[s] = SWOF_BC_WALL;
}

static int lake_at_rest(void) {
    const int nx = 200, ny = 120;
    swof_params p;
    defaults(&p, nx, ny, 1.0);
    size_t n = (size_t)nx * ny;
    double *z = malloc(n * 8), *h = malloc(n * 8), *hu = calloc(n, 8), *hv = calloc(n, 8);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const double x = i + 0.5 - 100.0, y = j + 0.5 - 60.0;
            z[(size_t)j * nx + i] = 0.8 * exp(-(x * x + y * y) / 300.0);
            h[(size_t)j * nx + i] = 1.0 - z[(size_t)j * nx + i];
        }
    swof_ctx* c;
    CHECK(swof_create(&p, z, NULL, NULL, 0, NULL, &c));
    CHECK(swof_set_state(c, h, hu, hv, NULL, 0.0));
    CHECK(swof_step(c, 200));
    double t;
    int64_t steps;
    CHECK(swof_get_state(c, h, hu, hv, NULL, &t, &steps));
    double qmax = 0.0, emax = 0.0;
    for (size_t k = 0; k < n; ++k) {
        qmax = fmax(qmax, fmax(fabs(hu[k]), fabs(hv[k])));
        emax = fmax(emax, fabs(h[k] + z[k] - 1.0));
    }
    swof_destroy(c);
    printf("lake at rest: %lld steps, t = %.4f s, max |q| = %.3e m^2/s, max |eta - 1| = %.3e m\n",
           (long long)steps, t, qmax, emax);
    free(z); free(h); free(hu); free(hv);
    return (steps == 200 && qmax <= 1e-13 && emax <= 1e-13) ? 0 : 1;
}

static int dam_break(void) {
    const int nx = 400, ny = 60;
    swof_params p;
    defaults(&p, nx, ny, 0.5);
    size_t n = (size_t)nx * ny;
    double *z = malloc(n * 8), *h = malloc(n * 8), *hu = calloc(n, 8), *hv = calloc(n, 8);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            z[(size_t)j * nx + i] = 0.01 * (nx - i) * p.dx;
            h[(size_t)j * nx + i] = (i < nx / 4) ? 2.0 : 0.0;
        }
    swof_ctx* c;
    CHECK(swof_create(&p, z, NULL, NULL, 0, NULL, &c));
    CHECK(swof_set_state(c, h, hu, hv, NULL, 0.0));
    swof_diag d0, d1;
    CHECK(swof_get_diag(c, &d0));
    int64_t done;
    CHECK(swof_run(c, 20.0, INT64_MAX, &done));
    CHECK(swof_get_diag(c, &d1));
    CHECK(swof_get_state(c, h, hu, hv, NULL, NULL, NULL));
    double hmin = 1e300;
    for (size_t k = 0; k < n; ++k) hmin = fmin(hmin, h[k]);
    swof_destroy(c);
    const double rel = fabs(d1.volume - d0.volume) / d0.volume;
    printf("dam break: %lld steps to t = %.3f s, min h = %.3e m, volume change %.3e (relative), wet %lld cells, clamps %lld\n",
           (long long)done, d1.t, hmin, rel, (long long)d1.wet_cells, (long long)d1.clamps);
    free(z); free(h); free(hu); free(hv);
    return (d1.t == 20.0 && hmin >= 0.0 && rel <= 1e-12 && d1.flags == 0) ? 0 : 1;
}

int main(void) {
    int bad = lake_at_rest();
    bad |= dam_break();
    printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
