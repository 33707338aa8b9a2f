// swof_pair.cuh -- experiment (SWOF_PAIR=1): the marching stage kernel split over a warp pair per column
// strip.  The producer warp (Y) marches the register window: primitives, y slopes and reconstruction, the
// y face, the x slopes / reconstruction of the finalised row and its centred sources; it hands each row's
// x-face inputs, y faces and sources to the consumer warp (X) through a double-buffered shared-memory slot
// (named barriers FULL/EMPTY per slot).  X computes the x face, the update, sources, Heun and the CFL
// maxima, and stores.  Each warp holds about half the state, so more warps fit per SM.  Same arithmetic
// as march_kernel, hence the same bits.
#pragma once

namespace swof {

#ifndef SWOF_PAIR_NP
#define SWOF_PAIR_NP 2
#endif
#ifndef SWOF_PAIR_NS
#define SWOF_PAIR_NS 2
#endif
constexpr int PR_NP = SWOF_PAIR_NP;      // pairs per CTA
constexpr int PR_NS = SWOF_PAIR_NS;      // hand-over slots per pair (named barriers: 2 PR_NS + 1 per pair <= 15)
constexpr int PR_NW = 2 * PR_NP;         // warps per CTA
constexpr int PR_NV = 18;                // doubles per lane and row handed from Y to X
#ifndef SWOF_PAIR_MINB
#define SWOF_PAIR_MINB 4
#endif

__device__ __forceinline__ void nb_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

template <bool CORRECTOR, class PH>
__global__ void __launch_bounds__(PR_NW * 32, SWOF_PAIR_MINB) pair_kernel(const KParams P, const KBufs B, const int par) {
    __shared__ double s_sc[6];
    __shared__ Ghost s_g;
    __shared__ int s_done;
    __shared__ double s_slot[PR_NP][PR_NS][PR_NV][32];
    __shared__ double s_south[PR_NP][4][32];
    DevState* st = B.st;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool leader = blockIdx.x == 0 && tid == 0;
    if (tid == 0) {
        const double t = st->t[par];
        const long long step = st->step[par];
        const double ax = u2d(st->amax[par][0]), ay = u2d(st->amax[par][1]);
        const double t_end = st->t_end;
        const bool finite = isfinite(ax) && isfinite(ay);
        const bool done = !(t < t_end) || step >= st->step_limit || !finite;
        if (leader) {
            if (done) {
                if (!CORRECTOR) {
                    st->amax[par ^ 1][0] = st->amax[par][0];
                    st->amax[par ^ 1][1] = st->amax[par][1];
                    if (!finite) atomicOr(&st->flags, FLAG_NONFINITE);
                } else {
                    st->t[par ^ 1] = t;
                    st->step[par ^ 1] = step;
                }
            } else if (!CORRECTOR) {
                st->amax[par ^ 1][0] = 0ull;
                st->amax[par ^ 1][1] = 0ull;
            }
        }
        const double dt0 = cfl_dt(P, ax, ay, t, t_end);
        const double ts0 = CORRECTOR ? t + dt0 : t;
        s_done = done;
        s_sc[0] = dt0;
        s_sc[1] = ts0;
        s_sc[2] = dt0 / P.dx;
        s_sc[3] = dt0 / P.dy;
        s_sc[4] = rain_rate(P, ts0) * dt0;
        s_sc[5] = (ph_ff<PH>(P) || ph_fk<PH>(P) == 0) ? 0.0 : dt0 * friction_gcf(P.fric_law, P.fric_coef, P.g);
        for (int k = 0; k < 4; ++k) {
            s_g.q[k] = 0.0;
            s_g.hc[k] = 0.0;
            if (P.bc[k] == BC_INFLOW) {
                s_g.q[k] = hydrograph(P, k, ts0) / P.width[k];
                s_g.hc[k] = critical_depth(s_g.q[k], P.g);
            }
        }
    }
    __syncthreads();
    if (s_done) return;
    const int nx = P.nx, ny = P.ny, pitch = P.pitch;
    const int nstrip = (nx + M_OWN - 1) / M_OWN;
    const int pair = warp >> 1, role = warp & 1;                   // role 0: Y (producer), 1: X (consumer)
    const int wid = blockIdx.x * PR_NP + pair;
    const int s = wid % nstrip, g = wid / nstrip;
    const int i0 = s * M_OWN, j0 = g * P.march_h;
    // named barriers (0 = __syncthreads): FULL/EMPTY per slot and pair, SOUTH once per pair
    const int FULL0 = 1 + (2 * PR_NS + 1) * pair, EMPTY0 = FULL0 + PR_NS, SOUTH = FULL0 + 2 * PR_NS;
    double amx = 0.0, amy = 0.0;
    if (j0 < ny) {
        const double* __restrict__ in_h = CORRECTOR ? B.Bh : B.Ah;
        const double* __restrict__ in_hu = CORRECTOR ? B.Bhu : B.Ahu;
        const double* __restrict__ in_hv = CORRECTOR ? B.Bhv : B.Ahv;
        const double h_eps = P.h_eps, g2 = 0.5 * P.g;
        const bool rus = ph_rusanov<PH>(P);
        const bool ord1 = ph_order1<PH>(P);
        const double2 z2 = make_double2(0.0, 0.0);
        const int gi = i0 - HALO + lane;
        const bool own_col = lane >= HALO && lane < HALO + M_OWN && gi < nx;
        const int jend = j0 + P.march_h < ny ? j0 + P.march_h : ny;
        if (role == 0) {
            // ---------------- producer: the register window ----------------
            const bool fastx = i0 - HALO >= 0 && i0 - HALO + 32 <= nx;
            auto prim = [&](double h, double hu, double hv, double z, MPrim& m) {
                const double rh = (h > h_eps) ? drcp(h) : 0.0;
                m.h = h;
                m.e = h + z;
                m.u = hu * rh;
                m.v = hv * rh;
                m.rh = rh;
            };
            MPrim A, Bw, C;
            double rh_, rhu, rhv, rz;
            march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, j0 - 2, rh_, rhu, rhv, rz);
            prim(rh_, rhu, rhv, rz, A);
            march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, j0 - 1, rh_, rhu, rhv, rz);
            prim(rh_, rhu, rhv, rz, Bw);
            march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, j0, rh_, rhu, rhv, rz);
            FaceIn plusA;
            double2 slA = z2;
            plusA.h = plusA.e = plusA.z = plusA.n = plusA.t = 0.0;
            for (int j = j0; j <= jend + 1; ++j) {
                prim(rh_, rhu, rhv, rz, C);
                if (j <= jend) {
                    const int jn = j + 1;
                    if (fastx && jn < ny) {
                        const size_t on = (size_t)jn * pitch + gi;
                        rh_ = in_h[on];
                        rhu = in_hu[on];
                        rhv = in_hv[on];
                        rz = B.z[on];
                    } else {
                        march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, jn, rh_, rhu, rhv, rz);
                    }
                }
                const double2 saB = ord1 ? z2 : half_slopes(A.h, Bw.h, C.h, A.e, Bw.e, C.e);
                const double2 sbB = ord1 ? z2 : half_slopes(A.v, Bw.v, C.v, A.u, Bw.u, C.u);
                const FaceIn minusB = recon_minus(make_double2(Bw.h, Bw.e), Bw.v, Bw.u, Bw.rh, saB, sbB);
                const FaceIn plusB = recon_plus(make_double2(Bw.h, Bw.e), Bw.v, Bw.u, Bw.rh, saB, sbB);
                if (j - 1 >= j0) {
                    double2 nfa, nfb;
                    if (M_SLOW(face_flux<false>(P.g, h_eps, plusA, minusB, nfa, nfb, rus)))
                        face_flux<true>(P.g, h_eps, plusA, minusB, nfa, nfb, rus);
                    if (j - 2 >= j0) {
                        const int r = j - 2 - j0, b = r % PR_NS;
                        const double2 heA = make_double2(A.h, A.e);
                        const double2 cL = shup2(heA), cR = shdn2(heA);
                        const double2 uvA = make_double2(A.u, A.v);
                        const double2 uL = shup2(uvA), uR = shdn2(uvA);
                        const double2 sa = ord1 ? z2 : half_slopes(cL.x, A.h, cR.x, cL.y, A.e, cR.y);
                        const double2 sb = ord1 ? z2 : half_slopes(uL.x, A.u, uR.x, uL.y, A.v, uR.y);
                        const FaceIn pl = recon_plus(heA, A.u, A.v, A.rh, sa, sb);
                        const FaceIn mi = recon_minus(heA, A.u, A.v, A.rh, sa, sb);
                        const double Fcx = centred_source(g2, A.h, A.e, sa.x, sa.y);
                        const double Fcy = centred_source(g2, A.h, A.e, slA.x, slA.y);
                        const double lph = shup(pl.h), lpe = shup(pl.e), lpz = shup(pl.z), lpn = shup(pl.n),
                                     lpt = shup(pl.t);
                        if (r >= PR_NS) nb_sync(EMPTY0 + b);              // X has read this slot's row r-NS
                        double* q = &s_slot[pair][b][0][lane];
                        q[0 * 32] = lph; q[1 * 32] = lpe; q[2 * 32] = lpz; q[3 * 32] = lpn; q[4 * 32] = lpt;
                        q[5 * 32] = mi.h; q[6 * 32] = mi.e; q[7 * 32] = mi.z; q[8 * 32] = mi.n; q[9 * 32] = mi.t;
                        q[10 * 32] = nfa.x; q[11 * 32] = nfa.y; q[12 * 32] = nfb.x; q[13 * 32] = nfb.y;
                        q[14 * 32] = Fcx; q[15 * 32] = Fcy; q[16 * 32] = A.h; q[17 * 32] = A.rh;
                        nb_arrive(FULL0 + b);
                    } else {
                        // the south face of row j0 (no row to finalise yet)
                        double* q = &s_south[pair][0][lane];
                        q[0] = nfa.x; q[32] = nfa.y; q[64] = nfb.x; q[96] = nfb.y;
                        nb_arrive(SOUTH);
                    }
                }
                plusA = plusB;
                slA = saB;
                A = Bw;
                Bw = C;
            }
            // drain: the last NS rows' EMPTY arrivals of X
            const int nrows = jend - j0;
            for (int r = nrows - PR_NS > 0 ? nrows - PR_NS : 0; r < nrows; ++r) nb_sync(EMPTY0 + r % PR_NS);
        } else {
            // ---------------- consumer: x face, update, sources, stores ----------------
            double2 sfa, sfb;
            nb_sync(SOUTH);                                            // the south face of row j0
            {
                const double* q = &s_south[pair][0][lane];
                sfa = make_double2(q[0], q[32]);
                sfb = make_double2(q[64], q[96]);
            }
            for (int f = j0; f < jend; ++f) {
                const int r = f - j0, b = r % PR_NS;
                const bool own = own_col;
                const size_t o = (size_t)(own ? f : 0) * pitch + (own ? gi : 0);
                double V = 0.0, cf = P.fric_coef, Ah0 = 0.0, Ahu0 = 0.0, Ahv0 = 0.0, VA0 = 0.0;
                const double hus = in_hu[o];
                const double hvs = in_hv[o];
                if (ph_ga<PH>(P)) V = CORRECTOR ? B.VB[o] : B.VA[o];
                if (ph_ff<PH>(P)) cf = B.fric[o];
                if (CORRECTOR) {
                    Ah0 = B.Ah[o];
                    Ahu0 = B.Ahu[o];
                    Ahv0 = B.Ahv[o];
                    if (ph_ga<PH>(P)) VA0 = B.VA[o];
                }
                nb_sync(FULL0 + b);
                FaceIn lp, mi;
                const double* q = &s_slot[pair][b][0][lane];
                lp.h = q[0 * 32]; lp.e = q[1 * 32]; lp.z = q[2 * 32]; lp.n = q[3 * 32]; lp.t = q[4 * 32];
                mi.h = q[5 * 32]; mi.e = q[6 * 32]; mi.z = q[7 * 32]; mi.n = q[8 * 32]; mi.t = q[9 * 32];
                const double2 nfa = make_double2(q[10 * 32], q[11 * 32]), nfb = make_double2(q[12 * 32], q[13 * 32]);
                const double Fcx = q[14 * 32], Fcy = q[15 * 32], Ah = q[16 * 32], Arh = q[17 * 32];
                nb_arrive(EMPTY0 + b);
                double2 wa, wb;
                if (M_SLOW(face_flux<false>(P.g, h_eps, lp, mi, wa, wb, rus))) face_flux<true>(P.g, h_eps, lp, mi, wa, wb, rus);
                const double2 ea = shdn2(wa), eb = shdn2(wb);
                const double lx = s_sc[2], ly = s_sc[3];
                const double pxm = lx * (ea.x - wa.x);
                const double qx = lx * ((ea.y - wb.x) - Fcx), qy = lx * (eb.y - wb.y);
                const double Dm = nfa.x - sfa.x;
                const double Dn = (nfa.y - sfb.x) - Fcy;
                const double Dt = nfb.y - sfb.y;
                const double hh = Ah - (pxm + ly * Dm);
                const double hu1 = hus - (qx + ly * Dt);
                const double hv1 = hvs - (qy + ly * Dn);
                const double cl = (own && hh < 0.0) ? -hh : 0.0;
                const double h1 = hh < 0.0 ? 0.0 : hh;
                double hst, hu2, hv2, Vn;
                const double dt = s_sc[0], Rdt = s_sc[4], dtgcf0 = s_sc[5];
                if (M_SLOW(cell_sources<PH, false>(P, dt, dtgcf0, Rdt, h1, hu1, hv1, V, cf, Arh, hus, hvs, hst, hu2, hv2, Vn)))
                    cell_sources<PH, true>(P, dt, dtgcf0, Rdt, h1, hu1, hv1, V, cf, Arh, hus, hvs, hst, hu2, hv2, Vn);
                if (cl > 0.0) {
                    atomicAdd(&st->clamps, 1ull);
                    atomicAdd(&st->clamped_mass, cl);
                    if (atomicMax(&st->clamp_max_bits, d2u(cl)) < d2u(cl)) {
                        atomicExch((unsigned long long*)&st->big_clamp_cell, (unsigned long long)((long long)f * nx + gi));
                        atomicExch((unsigned long long*)&st->big_clamp_step, (unsigned long long)st->step[par]);
                    }
                    if (cl > P.clamp_fail) atomicOr(&st->flags, FLAG_BIGCLAMP);
                }
                if (own) {
                    if (!CORRECTOR) {
                        B.Bh[o] = hst;
                        B.Bhu[o] = hu2;
                        B.Bhv[o] = hv2;
                        if (ph_ga<PH>(P)) B.VB[o] = Vn;
                    } else {
                        const double hN = 0.5 * (Ah0 + hst);
                        const double huN = 0.5 * (Ahu0 + hu2);
                        const double hvN = 0.5 * (Ahv0 + hv2);
                        B.Ah[o] = hN;
                        B.Ahu[o] = huN;
                        B.Ahv[o] = hvN;
                        if (ph_ga<PH>(P)) B.VA[o] = 0.5 * (VA0 + Vn);
                        if (P.cfl_mode == 0) {
                            double su, sv;
                            if (cfl_speeds<false>(P, hN, huN, hvN, su, sv)) cfl_speeds<true>(P, hN, huN, hvN, su, sv);
                            amx = (su > amx || su != su) ? su : amx;
                            amy = (sv > amy || sv != sv) ? sv : amy;
                        }
                    }
                }
                sfa = nfa;
                sfb = nfb;
            }
        }
    }
    if (CORRECTOR) {
        __shared__ unsigned long long red[2][PR_NW];
        unsigned long long bx = d2u(amx), by = d2u(amy);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, off);
            const unsigned long long oy = __shfl_xor_sync(0xffffffffu, by, off);
            bx = ox > bx ? ox : bx;
            by = oy > by ? oy : by;
        }
        if (lane == 0) { red[0][warp] = bx; red[1][warp] = by; }
        __syncthreads();
        if (tid == 0) {
            unsigned long long mx = 0, my = 0;
            for (int w = 0; w < PR_NW; ++w) {
                mx = red[0][w] > mx ? red[0][w] : mx;
                my = red[1][w] > my ? red[1][w] : my;
            }
            atomicMax(&st->amax[par ^ 1][0], mx);
            atomicMax(&st->amax[par ^ 1][1], my);
            if (leader) {
                const double tn = st->t[par];
                const long long n = st->step[par];
                st->t[par ^ 1] = tn + s_sc[0];
                st->step[par ^ 1] = n + 1;
                if (n < B.dt_cap) B.dt_hist[n] = s_sc[0];
            }
        }
    }
}

template <bool C, int FK, bool GA, bool FF>
constexpr StageFn pair_fn() { return pair_kernel<C, Phys<FK, GA, FF>>; }
template <bool C>
__host__ inline StageFn select_pair(int fk, bool ga, bool ff, bool generic) {
    if (generic) return pair_kernel<C, PhysRT>;
    static const StageFn tab[3][2][2] = {
        {{pair_fn<C, 0, false, false>(), pair_fn<C, 0, false, true>()}, {pair_fn<C, 0, true, false>(), pair_fn<C, 0, true, true>()}},
        {{pair_fn<C, 1, false, false>(), pair_fn<C, 1, false, true>()}, {pair_fn<C, 1, true, false>(), pair_fn<C, 1, true, true>()}},
        {{pair_fn<C, 2, false, false>(), pair_fn<C, 2, false, true>()}, {pair_fn<C, 2, true, false>(), pair_fn<C, 2, true, true>()}},
    };
    return tab[fk][ga][ff];
}

}  // namespace swof
