// swof_march2.cuh -- the stage kernel (predictor and corrector of Algorithm 1's Heun step),
// two columns per lane.  Each warp (one per CTA) owns a strip of 60 columns and marches down a segment of rows
// (KParams::march_h): lane l holds columns i0-2+2l and i0-1+2l, lanes 1..30 own their pair, lanes 0 and 31 are
// the radius-2 x halo (2 of 32 lanes, against 4 of 32 with one column per lane).  The y direction (slopes,
// reconstruction, faces) lives in a 3-row register window per column; in x, the face between a lane's two
// columns is local and only the pair's outer neighbours go through warp shuffles.  Rows move as 16-byte
// double2 loads and stores.  Every cell and face is computed by the same per-item operations as the one-column
// kernel (swof_march.cuh) and the oracle -- the canonical sheet of DESIGN.md §3 -- hence the same bits; the
// two columns of a lane are independent chains the scheduler interleaves (2x the instruction-level
// parallelism at 8 warps per SM).
#pragma once

namespace swof {

constexpr int M2_OWN = 60;             // own columns per warp: lanes 1..30, two adjacent columns each
#ifndef SWOF_M2_MINB
#define SWOF_M2_MINB 8                 // CTAs (warps) per SM the register allocation must allow
#endif

struct Row2 { double2 h, hu, hv, z; };            // raw state of a lane's two cells (.x left, .y right)

__device__ __forceinline__ double2 ldg2(const double* p, size_t o) {
    return *reinterpret_cast<const double2*>(p + o);
}
__device__ __forceinline__ void stg2(double* p, size_t o, double a, double b, bool w0, bool w1) {
    if (w0 && w1) {
        *reinterpret_cast<double2*>(p + o) = make_double2(a, b);
    } else {
        if (w0) p[o] = a;
        if (w1) p[o + 1] = b;
    }
}
__device__ __forceinline__ void m2_load(const double* in_h, const double* in_hu, const double* in_hv, const double* z,
                                        size_t o, Row2& r) {
    r.h = ldg2(in_h, o);
    r.hu = ldg2(in_hu, o);
    r.hv = ldg2(in_hv, o);
    r.z = ldg2(z, o);
}
// the two cells (gx, gy), (gx + 1, gy) with the boundary ghosts of march_fetch
__device__ __forceinline__ void m2_fetch(const KParams& P, const KBufs& B, const double* in_h, const double* in_hu,
                                         const double* in_hv, const Ghost* G, int gx, int gy, Row2& r) {
    march_fetch(P, B, in_h, in_hu, in_hv, G, gx, gy, r.h.x, r.hu.x, r.hv.x, r.z.x);
    march_fetch(P, B, in_h, in_hu, in_hv, G, gx + 1, gy, r.h.y, r.hu.y, r.hv.y, r.z.y);
}

// PUSH / DRY as in march_kernel (swof_march.cuh): fused strip halo push; opt-in dry-row skip (a warp row is
// dry when all 64 of its cells hold h = 0 exactly -- value-identical results)
template <bool CORRECTOR, class PH, bool PUSH = false, bool DRY = false>
__global__ void __launch_bounds__(32, SWOF_M2_MINB) march2_kernel(const KParams P, const KBufs B, const int par) {
    __shared__ double s_sc[6];
    __shared__ Ghost s_g;
    __shared__ int s_done;
    DevState* st = B.st;
    const int lane = threadIdx.x;
    const bool leader = blockIdx.x == 0 && lane == 0;
    const int nx = P.nx, ny = P.ny, pitch = P.pitch;
    const int nstrip = (nx + M2_OWN - 1) / M2_OWN;
    const int s = blockIdx.x % nstrip, g = blockIdx.x / nstrip;
    const int i0 = s * M2_OWN;
    const int gx = i0 - HALO + 2 * lane;                           // this lane's left column
    const bool fastx = i0 - HALO >= 0 && i0 - HALO + 64 <= nx;    // all 64 columns inside (warp-uniform)
    int j0, jend;
    march_seg(P, g, j0, jend);
    const double* __restrict__ in_h = CORRECTOR ? B.Bh : B.Ah;
    const double* __restrict__ in_hu = CORRECTOR ? B.Bhu : B.Ahu;
    const double* __restrict__ in_hv = CORRECTOR ? B.Bhv : B.Ahv;
    // interior warps issue the loads of their first three rows before the step scalars are known
    const bool early = fastx && j0 >= 2 && j0 < ny;
    Row2 ew0, ew1, ew2;
    if (early) {
        size_t o = (size_t)(j0 - 2) * pitch + gx;
        m2_load(in_h, in_hu, in_hv, B.z, o, ew0);
        m2_load(in_h, in_hu, in_hv, B.z, o + pitch, ew1);
        m2_load(in_h, in_hu, in_hv, B.z, o + 2 * (size_t)pitch, ew2);
    }
    if (lane == 0) {
        const double t = st->t[par];
        const long long step = st->step[par];
        const double ax = u2d(st->amax[par][0]), ay = u2d(st->amax[par][1]);
        const double t_end = st->t_end;
        const bool finite = isfinite(ax) && isfinite(ay);
        // halt: past t_end, at the step limit, a non-finite CFL maximum, or a clamp above clamp_fail
        const bool done = !(t < t_end) || step >= st->step_limit || !finite || (st->flags & FLAG_BIGCLAMP) != 0;
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
    __syncwarp();
    if (s_done) return;
    const double dt = s_sc[0], lx = s_sc[2], ly = s_sc[3], Rdt = s_sc[4], dtgcf0 = s_sc[5];
    double amx = 0.0, amy = 0.0;
    if (j0 < ny) {
        const double h_eps = P.h_eps, g2 = 0.5 * P.g;
        const bool rus = ph_rusanov<PH>(P);              // Rusanov flux (generic instance only)
        const bool ord1 = ph_order1<PH>(P);              // first order: every slope is 0
        const double2 z2 = make_double2(0.0, 0.0);
        const bool inner = lane >= 1 && lane <= 30;
        const bool own0 = inner && gx < nx, own1 = inner && gx + 1 < nx;
        auto prim = [&](double h, double hu, double hv, double z, MPrim& m) {
            const double rh = (h > h_eps) ? drcp(h) : 0.0;
            m.h = h;
            m.e = h + z;
            m.u = hu * rh;
            m.v = hv * rh;
            m.rh = rh;
        };
        auto prim2 = [&](const Row2& r, MPrim* m) {
            prim(r.h.x, r.hu.x, r.hv.x, r.z.x, m[0]);
            prim(r.h.y, r.hu.y, r.hv.y, r.z.y, m[1]);
        };
        // window per column: A = row j-2, Bw = row j-1, C = row j
        MPrim A[2], Bw[2], C[2];
        Row2 raw;                                        // row j, fetched one row ahead
        if (early) {
            prim2(ew0, A);
            prim2(ew1, Bw);
            raw = ew2;
        } else {
            m2_fetch(P, B, in_h, in_hu, in_hv, &s_g, gx, j0 - 2, raw);
            prim2(raw, A);
            m2_fetch(P, B, in_h, in_hu, in_hv, &s_g, gx, j0 - 1, raw);
            prim2(raw, Bw);
            m2_fetch(P, B, in_h, in_hu, in_hv, &s_g, gx, j0, raw);
        }
        // carried from the previous row, per column: the high y face of row j-2, the south face flux of row
        // j-2 (Fm, Fn + S_R, Ft) and its y slopes {dh, de} (Fc_y)
        FaceIn plusA[2];
        double2 sfa[2], sfb[2], slA[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            plusA[c].h = plusA[c].e = plusA[c].z = plusA[c].n = plusA[c].t = 0.0;
            sfa[c] = sfb[c] = slA[c] = z2;
        }
        long long onx = (long long)(j0 + 1) * pitch + gx;
        long long ofn = (long long)(j0 - 2) * pitch + gx;
        bool dA = DRY && __all_sync(0xffffffffu, A[0].h == 0.0 && A[1].h == 0.0);
        bool dB = DRY && __all_sync(0xffffffffu, Bw[0].h == 0.0 && Bw[1].h == 0.0);
        for (int j = j0; j <= jend + 1; ++j) {
            prim2(raw, C);
            if (j <= jend) {
                const int jn = j + 1;
                if (fastx && jn < ny) {
                    SWOF_ASSERT(jn >= 0 && jn < ny && gx >= 0 && gx + 1 < nx);
                    m2_load(in_h, in_hu, in_hv, B.z, (size_t)onx, raw);
                } else {
                    m2_fetch(P, B, in_h, in_hu, in_hv, &s_g, gx, jn, raw);
                }
            }
            // the finalised row's own state, issued early; unconditional 16-byte loads (a lane owning neither
            // cell reads cells (0, 0), (1, 0), always allocated: pitch >= 32)
            const int f = j - 2;
            const bool w0 = own0 && f >= j0, w1 = own1 && f >= j0;
            const size_t o = (w0 || w1) ? (size_t)ofn : 0;
            onx += pitch;
            ofn += pitch;
            SWOF_ASSERT(!(w0 || w1) || (f >= 0 && f < ny && gx >= 0 && gx < nx));
            double2 V = z2, cf = make_double2(P.fric_coef, P.fric_coef), Ah0 = z2, Ahu0 = z2, Ahv0 = z2, VA0 = z2;
            const double2 hus = ldg2(in_hu, o);
            const double2 hvs = ldg2(in_hv, o);
            if (ph_ga<PH>(P)) V = ldg2(CORRECTOR ? B.VB : B.VA, o);
            if (ph_ff<PH>(P)) cf = ldg2(B.fric, o);
            if (CORRECTOR) {
                Ah0 = ldg2(B.Ah, o);
                Ahu0 = ldg2(B.Ahu, o);
                Ahv0 = ldg2(B.Ahv, o);
                if (ph_ga<PH>(P)) VA0 = ldg2(B.VA, o);
            }
            const bool dC = DRY && __all_sync(0xffffffffu, C[0].h == 0.0 && C[1].h == 0.0);
            // y slopes and y reconstruction of row j-1 (normal v, transverse u), both columns
            double2 saB[2], sbB[2];
            FaceIn minusB[2], plusB[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                saB[c] = sbB[c] = z2;
                minusB[c] = {0.0, 0.0, 0.0, 0.0, 0.0};
                plusB[c] = {0.0, 0.0, 0.0, 0.0, 0.0};
            }
            if (!(DRY && dA && dB && dC)) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    saB[c] = ord1 ? z2 : half_slopes(A[c].h, Bw[c].h, C[c].h, A[c].e, Bw[c].e, C[c].e);
                    sbB[c] = ord1 ? z2 : half_slopes(A[c].v, Bw[c].v, C[c].v, A[c].u, Bw[c].u, C[c].u);
                    const double2 he = make_double2(Bw[c].h, Bw[c].e);
                    minusB[c] = recon_minus(he, Bw[c].v, Bw[c].u, Bw[c].rh, saB[c], sbB[c]);
                    plusB[c] = recon_plus(he, Bw[c].v, Bw[c].u, Bw[c].rh, saB[c], sbB[c]);
                }
            }
            if (j - 1 >= j0) {
                // y faces between rows j-2 and j-1: the north faces of row j-2, the south faces of row j-1
                double2 nfa[2] = {z2, z2}, nfb[2] = {z2, z2};
                if (!(DRY && dA && dB)) {
                    bool bad = face_flux<false>(P.g, h_eps, plusA[0], minusB[0], nfa[0], nfb[0], rus);
                    bad |= face_flux<false>(P.g, h_eps, plusA[1], minusB[1], nfa[1], nfb[1], rus);
                    if (M_SLOW(bad)) {
                        face_flux<true>(P.g, h_eps, plusA[0], minusB[0], nfa[0], nfb[0], rus);
                        face_flux<true>(P.g, h_eps, plusA[1], minusB[1], nfa[1], nfb[1], rus);
                    }
                }
                if (j - 2 >= j0) {
                    // ---- finalise row f = j-2 (window A): x direction, update, sources ----
                    // faces: W0 = west of column 0 (from the left lane's column 1), W1 = between the two
                    // columns, E1 = east of column 1 (the right lane's W0)
                    double2 w0a = z2, w0b = z2, w1a = z2, w1b = z2, e1a = z2, e1b = z2;
                    double Fcx[2] = {0.0, 0.0};
                    if (!(DRY && dA)) {
                        const double2 he0 = make_double2(A[0].h, A[0].e), he1 = make_double2(A[1].h, A[1].e);
                        const double2 heL = shup2(he1), heR = shdn2(he0);
                        const double2 uvL = shup2(make_double2(A[1].u, A[1].v)), uvR = shdn2(make_double2(A[0].u, A[0].v));
                        const double2 sa0 = ord1 ? z2 : half_slopes(heL.x, A[0].h, A[1].h, heL.y, A[0].e, A[1].e);
                        const double2 sb0 = ord1 ? z2 : half_slopes(uvL.x, A[0].u, A[1].u, uvL.y, A[0].v, A[1].v);
                        const double2 sa1 = ord1 ? z2 : half_slopes(A[0].h, A[1].h, heR.x, A[0].e, A[1].e, heR.y);
                        const double2 sb1 = ord1 ? z2 : half_slopes(A[0].u, A[1].u, uvR.x, A[0].v, A[1].v, uvR.y);
                        const FaceIn pl0 = recon_plus(he0, A[0].u, A[0].v, A[0].rh, sa0, sb0);
                        const FaceIn mi0 = recon_minus(he0, A[0].u, A[0].v, A[0].rh, sa0, sb0);
                        const FaceIn pl1 = recon_plus(he1, A[1].u, A[1].v, A[1].rh, sa1, sb1);
                        const FaceIn mi1 = recon_minus(he1, A[1].u, A[1].v, A[1].rh, sa1, sb1);
                        FaceIn lp;                            // the left lane's column-1 high face
                        lp.h = shup(pl1.h);
                        lp.e = shup(pl1.e);
                        lp.z = shup(pl1.z);
                        lp.n = shup(pl1.n);
                        lp.t = shup(pl1.t);
                        bool bad = face_flux<false>(P.g, h_eps, lp, mi0, w0a, w0b, rus);
                        bad |= face_flux<false>(P.g, h_eps, pl0, mi1, w1a, w1b, rus);
                        if (M_SLOW(bad)) {
                            face_flux<true>(P.g, h_eps, lp, mi0, w0a, w0b, rus);
                            face_flux<true>(P.g, h_eps, pl0, mi1, w1a, w1b, rus);
                        }
                        e1a = shdn2(w0a);
                        e1b = shdn2(w0b);
                        Fcx[0] = centred_source(g2, A[0].h, A[0].e, sa0.x, sa0.y);
                        Fcx[1] = centred_source(g2, A[1].h, A[1].e, sa1.x, sa1.y);
                    }
                    // update of both columns: x half from the faces above, y half from the south
                    // (carried) and north (just computed) faces
                    double h1[2], hu1[2], hv1[2], cl[2];
                    const double husv[2] = {hus.x, hus.y}, hvsv[2] = {hvs.x, hvs.y};
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const double2 wa = c == 0 ? w0a : w1a, wb = c == 0 ? w0b : w1b;
                        const double2 ea = c == 0 ? w1a : e1a, eb = c == 0 ? w1b : e1b;
                        const double pxm = lx * (ea.x - wa.x);
                        const double qx = lx * ((ea.y - wb.x) - Fcx[c]), qy = lx * (eb.y - wb.y);
                        const double Fcy = centred_source(g2, A[c].h, A[c].e, slA[c].x, slA[c].y);
                        const double Dm = nfa[c].x - sfa[c].x;
                        const double Dn = (nfa[c].y - sfb[c].x) - Fcy;
                        const double Dt = nfb[c].y - sfb[c].y;
                        const double hh = A[c].h - (pxm + ly * Dm);
                        hu1[c] = husv[c] - (qx + ly * Dt);
                        hv1[c] = hvsv[c] - (qy + ly * Dn);
                        cl[c] = ((c == 0 ? w0 : w1) && hh < 0.0) ? -hh : 0.0;
                        h1[c] = hh < 0.0 ? 0.0 : hh;
                    }
                    double hst[2], hu2[2], hv2[2], Vn[2];
                    const double Vv[2] = {V.x, V.y}, cfv[2] = {cf.x, cf.y};
                    {
                        bool bad = cell_sources<PH, false>(P, dt, dtgcf0, Rdt, h1[0], hu1[0], hv1[0], Vv[0], cfv[0], A[0].rh,
                                                           husv[0], hvsv[0], hst[0], hu2[0], hv2[0], Vn[0]);
                        bad |= cell_sources<PH, false>(P, dt, dtgcf0, Rdt, h1[1], hu1[1], hv1[1], Vv[1], cfv[1], A[1].rh,
                                                       husv[1], hvsv[1], hst[1], hu2[1], hv2[1], Vn[1]);
                        if (M_SLOW(bad)) {
#pragma unroll
                            for (int c = 0; c < 2; ++c)
                                cell_sources<PH, true>(P, dt, dtgcf0, Rdt, h1[c], hu1[c], hv1[c], Vv[c], cfv[c], A[c].rh,
                                                       husv[c], hvsv[c], hst[c], hu2[c], hv2[c], Vn[c]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (cl[c] > 0.0) {
                            atomicAdd(&st->clamps, 1ull);
                            atomicAdd(&st->clamped_mass, cl[c]);
                            if (atomicMax(&st->clamp_max_bits, d2u(cl[c])) < d2u(cl[c])) {
                                atomicExch((unsigned long long*)&st->big_clamp_cell,
                                           (unsigned long long)((long long)f * nx + gx + c));
                                atomicExch((unsigned long long*)&st->big_clamp_step, (unsigned long long)st->step[par]);
                            }
                            if (cl[c] > P.clamp_fail) atomicOr(&st->flags, FLAG_BIGCLAMP);
                        }
                    }
                    if (!CORRECTOR) {
                        stg2(B.Bh, o, hst[0], hst[1], w0, w1);
                        stg2(B.Bhu, o, hu2[0], hu2[1], w0, w1);
                        stg2(B.Bhv, o, hv2[0], hv2[1], w0, w1);
                        if (ph_ga<PH>(P)) stg2(B.VB, o, Vn[0], Vn[1], w0, w1);
                        if (PUSH && (f < GHOST_ROWS || f >= ny - GHOST_ROWS)) {
                            if (w0) push_halo(B, 1, ny, pitch, f, gx, hst[0], hu2[0], hv2[0]);
                            if (w1) push_halo(B, 1, ny, pitch, f, gx + 1, hst[1], hu2[1], hv2[1]);
                        }
                    } else {
                        const double2 Ahv[3] = {Ah0, Ahu0, Ahv0};
                        double hN[2], huN[2], hvN[2];
                        hN[0] = 0.5 * (Ahv[0].x + hst[0]);
                        hN[1] = 0.5 * (Ahv[0].y + hst[1]);
                        huN[0] = 0.5 * (Ahv[1].x + hu2[0]);
                        huN[1] = 0.5 * (Ahv[1].y + hu2[1]);
                        hvN[0] = 0.5 * (Ahv[2].x + hv2[0]);
                        hvN[1] = 0.5 * (Ahv[2].y + hv2[1]);
                        stg2(B.Ah, o, hN[0], hN[1], w0, w1);
                        stg2(B.Ahu, o, huN[0], huN[1], w0, w1);
                        stg2(B.Ahv, o, hvN[0], hvN[1], w0, w1);
                        if (ph_ga<PH>(P)) stg2(B.VA, o, 0.5 * (VA0.x + Vn[0]), 0.5 * (VA0.y + Vn[1]), w0, w1);
                        if (PUSH && (f < GHOST_ROWS || f >= ny - GHOST_ROWS)) {
                            if (w0) push_halo(B, 0, ny, pitch, f, gx, hN[0], huN[0], hvN[0]);
                            if (w1) push_halo(B, 0, ny, pitch, f, gx + 1, hN[1], huN[1], hvN[1]);
                        }
                        if (P.cfl_mode == 0) {
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                if (c == 0 ? w0 : w1) {  // own cells only (divergent: no warp vote here)
                                    double su, sv;
                                    if (cfl_speeds<false>(P, hN[c], huN[c], hvN[c], su, sv))
                                        cfl_speeds<true>(P, hN[c], huN[c], hvN[c], su, sv);
                                    amx = (su > amx || su != su) ? su : amx;
                                    amy = (sv > amy || sv != sv) ? sv : amy;
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {                  // become the south faces of row j-1
                    sfa[c] = nfa[c];
                    sfb[c] = nfb[c];
                }
            }
            // slide the window
            dA = dB;
            dB = dC;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                plusA[c] = plusB[c];
                slA[c] = saB[c];
                A[c] = Bw[c];
                Bw[c] = C[c];
            }
        }
    }
    if (CORRECTOR) {
        unsigned long long bx = d2u(amx), by = d2u(amy);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, off);
            const unsigned long long oy = __shfl_xor_sync(0xffffffffu, by, off);
            bx = ox > bx ? ox : bx;
            by = oy > by ? oy : by;
        }
        if (lane == 0) {
            atomicMax(&st->amax[par ^ 1][0], bx);
            atomicMax(&st->amax[par ^ 1][1], by);
            if (leader) {
                const double tn = st->t[par];
                const long long n = st->step[par];
                st->t[par ^ 1] = tn + dt;
                st->step[par ^ 1] = n + 1;
                if (n < B.dt_cap) B.dt_hist[n] = dt;
            }
        }
    }
}

template <bool C, int FK, bool GA, bool FF, bool DRY>
constexpr StageFn march2_fn() { return march2_kernel<C, Phys<FK, GA, FF>, false, DRY>; }
template <bool C, bool D>
__host__ inline StageFn march2_spec(int fk, bool ga, bool ff) {
    static const StageFn tab[3][2][2] = {
        {{march2_fn<C, 0, false, false, D>(), march2_fn<C, 0, false, true, D>()},
         {march2_fn<C, 0, true, false, D>(), march2_fn<C, 0, true, true, D>()}},
        {{march2_fn<C, 1, false, false, D>(), march2_fn<C, 1, false, true, D>()},
         {march2_fn<C, 1, true, false, D>(), march2_fn<C, 1, true, true, D>()}},
        {{march2_fn<C, 2, false, false, D>(), march2_fn<C, 2, false, true, D>()},
         {march2_fn<C, 2, true, false, D>(), march2_fn<C, 2, true, true, D>()}},
    };
    return tab[fk][ga][ff];
}
template <bool C>
__host__ inline StageFn select_march2(int fk, bool ga, bool ff, bool generic, bool push = false, bool dry = false) {
    if (push) return dry ? march2_kernel<C, PhysRT, true, true> : march2_kernel<C, PhysRT, true>;
    if (generic) return dry ? march2_kernel<C, PhysRT, false, true> : march2_kernel<C, PhysRT>;
    return dry ? march2_spec<C, true>(fk, ga, ff) : march2_spec<C, false>(fk, ga, ff);
}

}  // namespace swof
