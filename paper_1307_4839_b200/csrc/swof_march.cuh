// swof_march.cuh -- the stage kernel (predictor and corrector of Algorithm 1's Heun step) with
// the stencil in registers: each warp (one per CTA) owns a strip of 28 columns (lanes 2..29 of the 32
// columns i0-2 .. i0+29) and marches down a segment of rows (KParams::march_h, chosen at create time).  The
// y direction (slopes, reconstruction, faces) lives in a 3-row register window, the x direction goes
// through warp shuffles (neighbour primitives, the left cell's high face, the east face's flux), so there
// is no shared-memory tile and no barrier in the stencil.  Same arithmetic as the oracle (the canonical
// sheet of DESIGN.md §3), hence the same bits.  DESIGN.md §5 has the design and its measurements, §8 the
// rejected variants; SWOF_MARCH_TMA=1 builds the TMA-fed experiment (§5 "TMA").
#pragma once
#include <type_traits>

namespace swof {

constexpr int M_HL = 2;                       // x-halo lanes per side (= the reconstruction radius)
constexpr int M_OWN = 32 - 2 * M_HL;          // own columns per warp
// the rare exact recomputation (SLOW) of an out-of-range lane, by the whole warp when any lane needs it (a
// warp vote and a uniform branch; SLOW gives the same bits).  The vote also closes the scheduling region there.
#if !SWOF_EXACT
// the tolerance build has no slow path, but keeps the warp vote (on a predicate that is never true): one
// unbroken row body measured 11 % slower (ptxas interleaves the whole row and runs short of registers at 168)
#define M_SLOW(...) ((void)(__VA_ARGS__), __any_sync(0xffffffffu, m_never))
#else
#define M_SLOW(...) __any_sync(0xffffffffu, (__VA_ARGS__))
#endif
#ifndef SWOF_MARCH_EARLY
#define SWOF_MARCH_EARLY 1             // interior warps load their first rows before the preamble (+0.75 %)
#endif
#ifndef SWOF_MARCH_NW
#define SWOF_MARCH_NW 1                // warps per CTA: 1 -- a CTA retires with its warp (+6.7 % against 4)
#endif
constexpr int M_NW = SWOF_MARCH_NW;    // warps per CTA (independent); rows per warp: KParams::march_h
#ifndef SWOF_MARCH_MINB
#define SWOF_MARCH_MINB 12             // CTAs per SM: 12 warps at <= 168 registers
#endif

struct MPrim { double h, e, u, v, rh; };

// ---- SWOF_MARCH_TMA (experiment, DESIGN.md §5 "TMA"): the next row of an interior warp comes from a
// shared-memory ring fed by TMA tensor-map loads (cp.async.bulk.tensor, UTMALDG) instead of 4 LDG per lane
#ifndef SWOF_MARCH_TMA
#define SWOF_MARCH_TMA 0
#endif
constexpr int TMA_ROWS = 4;            // rows per TMA box (32 columns x 4 rows x 8 B = 1 KB per field)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, unsigned long long* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

// a global load issued at its program point (volatile asm is neither removed nor moved past other volatile
// asm; the value is still scheduled like any register)
__device__ __forceinline__ double ld_early(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
using StageFn = void (*)(KParams, KBufs, int);

// rows [j0, jend) of segment row g: march_h rows high, the last wave's segments march_h2 rows high
__device__ __forceinline__ void march_seg(const KParams& P, int g, int& j0, int& jend) {
    if (g < P.march_g1) {
        j0 = g * P.march_h;
        jend = j0 + P.march_h;
    } else {
        j0 = P.march_g1 * P.march_h + (g - P.march_g1) * P.march_h2;
        jend = j0 + P.march_h2;
    }
    jend = jend < P.ny ? jend : P.ny;
}

__device__ __forceinline__ double2 shup2(double2 v) {
    return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shdn2(double2 v) {
    return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double shup(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shdn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// (h, hu, hv, z) of cell (gi, gj) with the boundary ghosts of stage_kernel's edge path; any cell
// outside in both directions (a corner, never used) returns zeros
__device__ __forceinline__ void march_fetch(const KParams& P, const KBufs& B, const double* in_h, const double* in_hu,
                                            const double* in_hv, const Ghost* G, int gx, int gy, double& h,
                                            double& hu, double& hv, double& z) {
    const int nx = P.nx, ny = P.ny;
    const bool xin = gx >= 0 && gx < nx, yin = gy >= 0 && gy < ny;
    if (xin && yin) {
        const size_t o = (size_t)gy * P.pitch + gx;
        h = in_h[o];
        hu = in_hu[o];
        hv = in_hv[o];
        z = B.z[o];
        return;
    }
    h = hu = hv = z = 0.0;
    if (!xin && !yin) return;
    int si = gx, sj = gy, side;
    bool fx = false, fy = false, inflow = false;
    if (!xin) {
        side = gx < 0 ? 0 : 1;
        const bool inseg = P.bc[side] == BC_INFLOW && gy >= P.k0[side] && gy < P.k1[side];
        si = bc_src(gx, nx, P.bc[0], P.bc[1], inseg, inseg, fx);
        inflow = inseg;
    } else {
        side = gy < 0 ? 2 : 3;
        const bool inseg = P.bc[side] == BC_INFLOW && gx >= P.k0[side] && gx < P.k1[side];
        sj = P.bc[side] == BC_HALO ? (gy < -GHOST_ROWS ? -GHOST_ROWS : gy >= ny + GHOST_ROWS ? ny + GHOST_ROWS - 1 : gy)
                                   : bc_src(gy, ny, P.bc[2], P.bc[3], inseg, inseg, fy);
        inflow = inseg;
    }
    SWOF_ASSERT(si >= 0 && si < nx && sj >= -GHOST_ROWS && sj < ny + GHOST_ROWS);
    const size_t o = (size_t)sj * P.pitch + si;
    z = B.z[o];
    if (inflow) {  // G in shared memory (one copy per CTA)
        h = G->hc[side];
        hu = side == 0 ? G->q[0] : (side == 1 ? -G->q[1] : 0.0);
        hv = side == 2 ? G->q[2] : (side == 3 ? -G->q[3] : 0.0);
    } else {
        h = in_h[o];
        hu = in_hu[o];
        hv = in_hv[o];
        if (fx) hu = -hu;
        if (fy) hv = -hv;
    }
}

// PUSH: also store the boundary rows into the neighbour strips' ghost rows (push_halo);
// DRY (opt-in swof_params.dry_skip): warp votes on rows whose 32 cells hold h = 0 exactly skip the faces of
// a dry row pair, the y stencil of three dry rows and the x stencil of a dry row.  A dry cell reconstructs
// to depth 0 whatever its neighbours (minmod of (-h_m, h_p) is 0), so those fluxes and sources are zero and
// the update reads zeros -- value-identical.  Measured: cfg3 12.0 -> 13.7 G cell-updates/s, and on the wet
// cfg4 it costs 6-10 % (the tiled kernel's tile skip: 14.1 G and 26 %).
template <bool CORRECTOR, class PH, bool PUSH = false, bool DRY = false>
__global__ void __launch_bounds__(M_NW * 32, SWOF_MARCH_MINB) march_kernel(const KParams P, const KBufs B, const int par) {
    __shared__ double s_sc[6];
    __shared__ Ghost s_g;
    __shared__ int s_done;
    DevState* st = B.st;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool leader = blockIdx.x == 0 && tid == 0;
    const bool m_never = P.nx < 0;     // never true (swof_create validates nx >= 1); see M_SLOW
    (void)m_never;
#if SWOF_MARCH_EARLY
    // interior warps issue the loads of their first three rows before the step scalars are known
    const double* __restrict__ e_h = CORRECTOR ? B.Bh : B.Ah;
    const double* __restrict__ e_hu = CORRECTOR ? B.Bhu : B.Ahu;
    const double* __restrict__ e_hv = CORRECTOR ? B.Bhv : B.Ahv;
    double ew[12];
    bool early;
    {
        const int nstrip0 = (P.nx + M_OWN - 1) / M_OWN;
        const int wid0 = blockIdx.x * M_NW + warp;
        int j00, jend0;
        march_seg(P, wid0 / nstrip0, j00, jend0);
        const int i00 = (wid0 % nstrip0) * M_OWN;
        early = i00 - M_HL >= 0 && i00 - M_HL + 32 <= P.nx && j00 >= 2 && j00 < P.ny;
        if (early) {
            size_t o = (size_t)(j00 - 2) * P.pitch + (i00 - M_HL + lane);
#pragma unroll
            for (int r = 0; r < 3; ++r, o += P.pitch) {
                ew[4 * r] = e_h[o];
                ew[4 * r + 1] = e_hu[o];
                ew[4 * r + 2] = e_hv[o];
                ew[4 * r + 3] = B.z[o];
            }
        }
    }
#endif
    if (tid == 0) {
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
    __syncthreads();
    if (s_done) return;
    const double dt = s_sc[0], lx = s_sc[2], ly = s_sc[3], Rdt = s_sc[4], dtgcf0 = s_sc[5];
    const int nx = P.nx, ny = P.ny, pitch = P.pitch;
    const int nstrip = (nx + M_OWN - 1) / M_OWN;
    const int wid = blockIdx.x * M_NW + warp;
    const int s = wid % nstrip, g = wid / nstrip;
    const int i0 = s * M_OWN;
    int j0, jend;
    march_seg(P, g, j0, jend);
    double amx = 0.0, amy = 0.0;
    if (j0 < ny) {
        const double* __restrict__ in_h = CORRECTOR ? B.Bh : B.Ah;
        const double* __restrict__ in_hu = CORRECTOR ? B.Bhu : B.Ahu;
        const double* __restrict__ in_hv = CORRECTOR ? B.Bhv : B.Ahv;
        const double h_eps = P.h_eps, g2 = 0.5 * P.g;
        const bool rus = ph_rusanov<PH>(P);              // Rusanov flux (generic instance only)
        const bool ord1 = ph_order1<PH>(P);              // first order: every slope is 0
        const double2 z2 = make_double2(0.0, 0.0);
        const int gi = i0 - M_HL + lane;
        const bool own_col = lane >= M_HL && lane < M_HL + M_OWN && gi < nx;
        const bool fastx = i0 - M_HL >= 0 && i0 - M_HL + 32 <= nx;   // all 32 columns inside (warp-uniform)
#if SWOF_MARCH_TMA
        // TMA ring: rows j0+1 .. jend+2 (the fetched rows) in chunks of TMA_ROWS, two stages; only for warps whose
        // fetched rows are all stored rows (interior strips, not the last segment: its ghosts are synthesised)
        __shared__ alignas(128) double s_ring[2][4][TMA_ROWS][32];
        __shared__ alignas(8) unsigned long long s_bar[2];
        const bool tma = B.tmaps != nullptr && fastx && jend + 1 < ny && j0 >= 2;
        const int nchunk = (jend - j0 + 2 + TMA_ROWS - 1) / TMA_ROWS;
        const char* tm = (const char*)B.tmaps + (CORRECTOR ? 4 * 128 : 0);
        auto tma_issue = [&](int c) {          // lane 0: chunk c into stage c & 1
            if (lane == 0 && c < nchunk) {
                unsigned long long* bar = &s_bar[c & 1];
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar, 4u * TMA_ROWS * 32 * 8);
                const int y = j0 + 1 + c * TMA_ROWS + GHOST_ROWS;          // tensor rows start at field row -2
#pragma unroll
                for (int f = 0; f < 4; ++f) tma_load_2d(&s_ring[c & 1][f][0][0], tm + f * 128, i0 - M_HL, y, bar);
            }
        };
        if (tma) {
            if (lane == 0) {
                mbar_init(&s_bar[0], 1);
                mbar_init(&s_bar[1], 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncwarp();
            tma_issue(0);
            tma_issue(1);
        }
#endif
        auto prim = [&](double h, double hu, double hv, double z, MPrim& m) {
            const double rh = drcp_sel(h > h_eps, h);
            m.h = h;
            m.e = h + z;
            m.u = hu * rh;
            m.v = hv * rh;
            m.rh = rh;
        };
        // the point-wise tail of a finalised cell (f, gc) at offset o (ok: an own cell): rain, Green-Ampt and
        // friction (cell_sources), the corrector's Heun average and CFL speeds, the stores
        auto tail_cell = [&](const bool ok, const int f, const int gc, const size_t o, const double h1, const double hu1,
                             const double hv1, const double u2, const double rhs, const double V, const double cf,
                             const double Ah0, const double Ahu0, const double Ahv0, const double VA0) {
            double hst, hu2, hv2, Vn;
            if (M_SLOW(cell_sources<PH, false>(P, dt, dtgcf0, Rdt, h1, hu1, hv1, V, cf, rhs, u2, hst, hu2, hv2, Vn)))
                cell_sources<PH, true>(P, dt, dtgcf0, Rdt, h1, hu1, hv1, V, cf, rhs, u2, hst, hu2, hv2, Vn);
            // the values this lane stores: U* (predictor) or the Heun average U^{n+1} (corrector), and the
            // corrector's CFL speeds, all formed before the store branch (so the speeds' rcp / sqrt chains overlap
            // the rest of the cell)
            double oh = hst, ohu = hu2, ohv = hv2, oV = Vn;
            if (CORRECTOR) {
                oh = 0.5 * (Ah0 + hst);
                ohu = 0.5 * (Ahu0 + hu2);
                ohv = 0.5 * (Ahv0 + hv2);
                oV = 0.5 * (VA0 + Vn);
                if (P.cfl_mode == 0) {
                    double su, sv;
                    if (M_SLOW(cfl_speeds<false>(P, oh, ohu, ohv, su, sv))) cfl_speeds<true>(P, oh, ohu, ohv, su, sv);
                    // su, sv are +0, positive or NaN (never -0): their bit patterns order like their values and a
                    // NaN's lies above every number's, as in the u64 reduction below, so the running maxima compare
                    // on the integer pipe (no DSETP; +0.2 % against the fp64 compare with a NaN test)
                    amx = (ok && d2u(su) > d2u(amx)) ? su : amx;
                    amy = (ok && d2u(sv) > d2u(amy)) ? sv : amy;
                }
            }
            if (ok) {
                double* const oA = CORRECTOR ? B.Ah : B.Bh;
                double* const oAu = CORRECTOR ? B.Ahu : B.Bhu;
                double* const oAv = CORRECTOR ? B.Ahv : B.Bhv;
                oA[o] = oh;
                oAu[o] = ohu;
                oAv[o] = ohv;
                if (ph_ga<PH>(P)) (CORRECTOR ? B.VA : B.VB)[o] = oV;
                if (PUSH && (f < GHOST_ROWS || f >= ny - GHOST_ROWS)) push_halo(B, CORRECTOR ? 0 : 1, ny, pitch, f, gc, oh, ohu, ohv);
            }
        };
        // window: A = row j-2, Bw = row j-1, C = row j
        MPrim A, Bw, C;
        double rh_, rhu, rhv, rz;                     // raw (h, hu, hv, z) of row j, fetched one row ahead
#if SWOF_MARCH_EARLY
        if (early) {
            prim(ew[0], ew[1], ew[2], ew[3], A);
            prim(ew[4], ew[5], ew[6], ew[7], Bw);
            rh_ = ew[8]; rhu = ew[9]; rhv = ew[10]; rz = ew[11];
        } else
#endif
        {
            march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, j0 - 2, rh_, rhu, rhv, rz);
            prim(rh_, rhu, rhv, rz, A);
            march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, j0 - 1, rh_, rhu, rhv, rz);
            prim(rh_, rhu, rhv, rz, Bw);
            march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, j0, rh_, rhu, rhv, rz);
        }
        // carried from the previous row: the high y face of row j-2 (for the face between j-2 and j-1), the
        // south face flux of row j-2 (Fm, Fn + S_R, Ft) and its y slopes {dh, de} (Fc_y)
        FaceIn plusA;
        double2 sfa = make_double2(0.0, 0.0), sfb = make_double2(0.0, 0.0), slA = make_double2(0.0, 0.0);
        plusA.h = plusA.e = plusA.z = plusA.n = plusA.t = 0.0;
        // offsets of (row j+1, gi) and (row j-2, gi), advanced by the pitch each row (+1.3 % against
        // recomputing them)
        long long onx = (long long)(j0 + 1) * pitch + gi;
        long long ofn = (long long)(j0 - 2) * pitch + gi;
        bool dA = DRY && __all_sync(0xffffffffu, A.h == 0.0), dB = DRY && __all_sync(0xffffffffu, Bw.h == 0.0);
        // this lane's clamp bookkeeping, flushed once after the march: no atomics in the row body
        unsigned int ncl = 0;
        double clm = 0.0, clx = 0.0;
        int clf = 0;                                  // row of this lane's largest clamp
        // one row j of the march.  FACE: the y face (j-2 | j-1) is formed (j >= j0 + 1); FIN: row j-2 is
        // finalised (j >= j0 + 2).  The prologue rows j0, j0 + 1 run without them, the steady-state rows with
        // both, so the steady-state body has no branch but the fetch's warp-uniform ghost test.
        auto row = [&](const int j, auto face_t, auto fin_t) {
            constexpr bool FACE = decltype(face_t)::value, FIN = decltype(fin_t)::value;
            prim(rh_, rhu, rhv, rz, C);
            {   // row j + 1 (the last row's fetch, past jend + 1, is never used: a valid cell or ghost)
                const int jn = j + 1;
#if SWOF_MARCH_TMA
                if (tma) {
                    const int k = jn - (j0 + 1), c = k / TMA_ROWS, r = k - c * TMA_ROWS;
                    if (r == 0) {
                        // chunk c - 1 (stage (c + 1) & 1) was read by the previous rows and its values are used:
                        // refill that stage with chunk c + 1, then wait for chunk c
                        if (c >= 1) tma_issue(c + 1);
                        mbar_wait(&s_bar[c & 1], (c >> 1) & 1);
                    }
                    rh_ = s_ring[c & 1][0][r][lane];
                    rhu = s_ring[c & 1][1][r][lane];
                    rhv = s_ring[c & 1][2][r][lane];
                    rz = s_ring[c & 1][3][r][lane];
                } else
#endif
                if (fastx && jn < ny) {
                    const size_t on = (size_t)onx;
                    SWOF_ASSERT(jn >= 0 && jn < ny && gi >= 0 && gi < nx);
                    rh_ = in_h[on];
                    rhu = in_hu[on];
                    rhv = in_hv[on];
                    rz = B.z[on];
                } else {
                    march_fetch(P, B, in_h, in_hu, in_hv, &s_g, gi, jn, rh_, rhu, rhv, rz);
                }
            }
            // the finalised row's own state, issued early; unconditional loads (a non-own lane reads cell
            // (0, 0), always allocated) keep the loop free of divergent branches
            const int f = j - 2;
            const bool own = FIN && own_col;
            const size_t o = own ? (size_t)ofn : 0;
            onx += pitch;
            ofn += pitch;
            SWOF_ASSERT(!own || (f >= 0 && f < ny && gi >= 0 && gi < nx));
            double V = 0.0, cf = P.fric_coef, Ah0 = 0.0, Ahu0 = 0.0, Ahv0 = 0.0, VA0 = 0.0, hus = 0.0, hvs = 0.0;
            // issued here, unconditionally (volatile: the compiler may not sink them into the own-lane store
            // branch, where their DRAM latency would be exposed)
            if (FIN) hus = ld_early(in_hu + o);
            if (FIN) hvs = ld_early(in_hv + o);
            if (FIN && ph_ga<PH>(P)) V = ld_early((CORRECTOR ? B.VB : B.VA) + o);
            if (FIN && ph_ff<PH>(P)) cf = ld_early(B.fric + o);
            if (FIN && CORRECTOR) {
                Ah0 = ld_early(B.Ah + o);
                Ahu0 = ld_early(B.Ahu + o);
                Ahv0 = ld_early(B.Ahv + o);
                if (ph_ga<PH>(P)) VA0 = ld_early(B.VA + o);
            }
            // DRY: warp rows whose 32 cells all hold h = 0 (carried: dA, dB of rows j-2, j-1; dC of row j)
            const bool dC = DRY && __all_sync(0xffffffffu, C.h == 0.0);
            // x direction of row f = j-2 (window A) by shuffles: slopes, reconstruction, the west face of every
            // lane (the east face is the next lane's west face) and the centred source; it runs after the y face
            // (before it: -2.1 %, before the y slopes: -1.2 %)
            double2 wa = z2, wb = z2, ea = z2, eb = z2;       // west / east face of this lane's cell
            double Fcx = 0.0;
            auto xpart = [&]() {
                    if (!(DRY && dA)) {                       // a dry row: every x face is dry-dry
                        const double2 heA = make_double2(A.h, A.e);
                        const double2 uvA = make_double2(A.u, A.v);
                        const double2 cL = shup2(heA), cR = shdn2(heA);
                        const double2 uL = shup2(uvA), uR = shdn2(uvA);
                        const double2 sa = ord1 ? z2 : half_slopes(cL.x, A.h, cR.x, cL.y, A.e, cR.y);
                        const double2 sb = ord1 ? z2 : half_slopes(uL.x, A.u, uR.x, uL.y, A.v, uR.y);
                        const FaceIn pl = recon_plus(heA, A.u, A.v, A.rh, sa, sb);
                        const FaceIn mi = recon_minus(heA, A.u, A.v, A.rh, sa, sb);
                        FaceIn lp;                            // the west neighbour's high face
                        lp.h = shup(pl.h);
                        lp.e = shup(pl.e);
                        lp.z = shup(pl.z);
                        lp.n = shup(pl.n);
                        lp.t = shup(pl.t);
                        if (M_SLOW(face_flux<false>(P.g, h_eps, lp, mi, wa, wb, rus)))
                            face_flux<true>(P.g, h_eps, lp, mi, wa, wb, rus);
                        ea = shdn2(wa);
                        eb = shdn2(wb);
                        Fcx = centred_source(g2, A.h, A.e, sa.x, sa.y);
                    }
            };
            // y slopes and y reconstruction of row m = j-1 (normal v, transverse u); not needed when rows
            // j-2..j are dry (both of row j-1's faces are dry-dry, its Fc_y multiplies a zero depth)
            double2 saB = z2, sbB = z2;
            FaceIn minusB = {0.0, 0.0, 0.0, 0.0, 0.0}, plusB = {0.0, 0.0, 0.0, 0.0, 0.0};
            if (!(DRY && dA && dB && dC)) {
                saB = ord1 ? z2 : half_slopes(A.h, Bw.h, C.h, A.e, Bw.e, C.e);
                sbB = ord1 ? z2 : half_slopes(A.v, Bw.v, C.v, A.u, Bw.u, C.u);
                minusB = recon_minus(make_double2(Bw.h, Bw.e), Bw.v, Bw.u, Bw.rh, saB, sbB);
                plusB = recon_plus(make_double2(Bw.h, Bw.e), Bw.v, Bw.u, Bw.rh, saB, sbB);
            }
            if (FACE) {
                // y face between rows j-2 and j-1: the north face of row j-2, the south face of row j-1
                double2 nfa = z2, nfb = z2;
                if (!(DRY && dA && dB)) {
                    if (M_SLOW(face_flux<false>(P.g, h_eps, plusA, minusB, nfa, nfb, rus)))
                        face_flux<true>(P.g, h_eps, plusA, minusB, nfa, nfb, rus);
                }
                if (FIN) {
                    // ---- finalise row f = j-2 (window A): x direction by shuffles, update, sources ----
                    xpart();
                    const double pxm = lx * (ea.x - wa.x);
                    const double qx = lx * ((ea.y - wb.x) - Fcx), qy = lx * (eb.y - wb.y);
                    // y half with the south (carried) and north (just computed) faces
                    const double Fcy = centred_source(g2, A.h, A.e, slA.x, slA.y);
                    const double Dm = nfa.x - sfa.x;
                    const double Dn = (nfa.y - sfb.x) - Fcy;
                    const double Dt = nfb.y - sfb.y;
                    const double hh = A.h - (pxm + ly * Dm);
                    const double hu1 = hus - (qx + ly * Dt);
                    const double hv1 = hvs - (qy + ly * Dn);
                    const double cl = (own && hh < 0.0) ? -hh : 0.0;
                    const double h1 = hh < 0.0 ? 0.0 : hh;
                    const double u2 = ph_fk<PH>(P) != 0 ? hus * hus + hvs * hvs : 0.0;
                    ncl += cl > 0.0 ? 1u : 0u;
                    clm += cl;
                    clf = cl > clx ? f : clf;
                    clx = cl > clx ? cl : clx;
                    tail_cell(own, f, gi, o, h1, hu1, hv1, u2, A.rh, V, cf, Ah0, Ahu0, Ahv0, VA0);
                }
                sfa = make_double2(nfa.x, nfa.y);              // becomes the south face of row j-1
                sfb = nfb;
            }
            // slide the window
            dA = dB;
            dB = dC;
            plusA = plusB;
            slA = saB;
            A = Bw;
            Bw = C;
        };
        row(j0, std::false_type{}, std::false_type{});
        row(j0 + 1, std::true_type{}, std::false_type{});
#pragma unroll 1
        for (int j = j0 + 2; j <= jend + 1; ++j) row(j, std::true_type{}, std::true_type{});
        if (__any_sync(0xffffffffu, ncl != 0u) && ncl != 0u) {   // rare: a clamp in this warp's segment
            atomicAdd(&st->clamps, (unsigned long long)ncl);
            atomicAdd(&st->clamped_mass, clm);
            if (atomicMax(&st->clamp_max_bits, d2u(clx)) < d2u(clx)) {
                atomicExch((unsigned long long*)&st->big_clamp_cell, (unsigned long long)((long long)clf * nx + gi));
                atomicExch((unsigned long long*)&st->big_clamp_step, (unsigned long long)st->step[par]);
            }
            if (clx > P.clamp_fail) atomicOr(&st->flags, FLAG_BIGCLAMP);
        }
    }
    if (CORRECTOR) {
        __shared__ unsigned long long red[2][M_NW];
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
            for (int w = 0; w < M_NW; ++w) {
                mx = red[0][w] > mx ? red[0][w] : mx;
                my = red[1][w] > my ? red[1][w] : my;
            }
            atomicMax(&st->amax[par ^ 1][0], mx);
            atomicMax(&st->amax[par ^ 1][1], my);
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
constexpr StageFn march_fn() { return march_kernel<C, Phys<FK, GA, FF>, false, DRY>; }
template <bool C, bool D>
__host__ inline StageFn march_spec(int fk, bool ga, bool ff) {
    static const StageFn tab[3][2][2] = {
        {{march_fn<C, 0, false, false, D>(), march_fn<C, 0, false, true, D>()},
         {march_fn<C, 0, true, false, D>(), march_fn<C, 0, true, true, D>()}},
        {{march_fn<C, 1, false, false, D>(), march_fn<C, 1, false, true, D>()},
         {march_fn<C, 1, true, false, D>(), march_fn<C, 1, true, true, D>()}},
        {{march_fn<C, 2, false, false, D>(), march_fn<C, 2, false, true, D>()},
         {march_fn<C, 2, true, false, D>(), march_fn<C, 2, true, true, D>()}},
    };
    return tab[fk][ga][ff];
}
// the default scheme runs physics-specialised instances (with or without the dry skip); the generic
// PhysRT instance serves the scheme variants and the fused halo push
template <bool C>
__host__ inline StageFn select_march(int fk, bool ga, bool ff, bool generic, bool push = false, bool dry = false) {
    if (push) return dry ? march_kernel<C, PhysRT, true, true> : march_kernel<C, PhysRT, true>;
    if (generic) return dry ? march_kernel<C, PhysRT, false, true> : march_kernel<C, PhysRT>;
    return dry ? march_spec<C, true>(fk, ga, ff) : march_spec<C, false>(fk, ga, ff);
}

}  // namespace swof
