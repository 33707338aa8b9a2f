// swof.cu -- C ABI (include/swof.h) of the B200-native FullSWOF_2D time step.
//
// Host side: parameter validation, workspace layout (padded SoA fp64 fields, 256-B aligned rows),
// device scalar state double-buffered by step parity, the step loop captured as a CUDA graph of
// `graph_steps` Heun steps (2 launches each), and fixed-order diagnostics.  No host round trip per
// step: every CTA derives dt_n from the CFL maxima the previous corrector left in device memory.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/swof.h"
#include "swof_kernels.cuh"
#include "swof_d8.cuh"
#include "swof_march.cuh"
#if SWOF_MARCH_TMA
#include <cuda.h>
#include <cudaTypedefs.h>
#endif

using namespace swof;

struct swof_ctx {
    swof_params p;
    KParams kp;
    KBufs kb;
    void* ws = nullptr;
    bool own_ws = false;
    size_t ws_bytes = 0;
    cudaStream_t stream = nullptr;
    int par = 0;                       // parity of the next step to launch
    bool have_state = false;
    int graph_steps = 16;
    cudaGraphExec_t graph = nullptr;   // graph_steps steps starting at parity 0
    DevState* h_st = nullptr;          // pinned mirror of the device scalar state
    double* d_part = nullptr;          // diag partials
    int diag_blocks = 0;
    StageFn kpred = nullptr, kcorr = nullptr;   // stage kernel instances for this context's physics
    dim3 cf_grid;                               // face-CFL pass tiles
    dim3 sgrid, sblock;                         // stage kernel launch shape
    size_t ssmem = 0;
    void* d_tmaps = nullptr;                    // SWOF_MARCH_TMA builds: the 8 tensor maps (KBufs::tmaps)
    std::string err;
};

namespace {

constexpr int DIAG_BLOCKS = 1184;      // 8 x 148 SMs

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
    size_t pitch;                      // doubles per row
    size_t field;                      // bytes per field
    size_t off_A, off_B, off_z, off_VA, off_VB, off_fric, off_st, off_hist, off_part, total;
};

Layout make_layout(const swof_params* p, bool fric_field) {
    Layout L{};
    L.pitch = align_up((size_t)p->nx, 32);
    // every field carries GHOST_ROWS spare rows below and above (the halo rows of a strip's HALO sides);
    // the field pointers address row 0, which stays 256-B aligned
    L.field = align_up(L.pitch * sizeof(double) * ((size_t)p->ny + 2 * GHOST_ROWS), 256);
    size_t o = 0;
    L.off_A = o; o += 3 * L.field;
    L.off_B = o; o += 3 * L.field;
    L.off_z = o; o += L.field;
    L.off_VA = o; o += p->ga_enabled ? L.field : 0;
    L.off_VB = o; o += p->ga_enabled ? L.field : 0;
    L.off_fric = o; o += fric_field ? L.field : 0;
    L.off_st = o; o += align_up(sizeof(DevState), 256);
    int64_t cap = p->dt_hist_cap > 0 ? p->dt_hist_cap : (int64_t)1 << 20;
    L.off_hist = o; o += align_up((size_t)cap * sizeof(double), 256);
    L.off_part = o; o += align_up((size_t)DIAG_BLOCKS * 5 * sizeof(double), 256);
    L.total = o;
    return L;
}

const char* validate(const swof_params* p) {
    if (!p) return "params is NULL";
    if (p->nx < 1 || p->ny < 1) return "nx, ny must be >= 1";
    if (!(p->dx > 0) || !(p->dy > 0) || !std::isfinite(p->dx) || !std::isfinite(p->dy)) return "dx, dy must be finite and > 0";
    if (!(p->g > 0) || !std::isfinite(p->g)) return "g must be > 0";
    if (!(p->cfl > 0) || p->cfl > 1) return "cfl must be in (0, 1]";
    if (!(p->dt_max > 0) || !std::isfinite(p->dt_max)) return "dt_max must be finite and > 0";
    // the kernels' fast reciprocal of wet depths needs h > h_eps >= 2^-1000 (1e-300 is 0 for any physics)
    if (!(p->h_eps >= 1e-300) || !std::isfinite(p->h_eps)) return "h_eps must be finite and >= 1e-300";
    if (p->fric_law < SWOF_FRIC_NONE || p->fric_law > SWOF_FRIC_CHEZY) return "unknown fric_law";
    if (p->ga_enabled) {
        if (!(p->ga_Ks >= 0) || !(p->ga_dtheta > 0) || !std::isfinite(p->ga_hf) || !std::isfinite(p->ga_A) ||
            !(p->ga_vinf0 >= 0))
            return "Green-Ampt needs Ks >= 0, dtheta > 0, finite hf and A, vinf0 >= 0";
    }
    if (p->n_rain < 0 || p->n_rain > SWOF_MAX_TABLE) return "n_rain out of range";
    for (int k = 0; k < p->n_rain; ++k) {
        if (!(p->rain_rate[k] >= 0) || !std::isfinite(p->rain_rate[k])) return "rain rates must be finite and >= 0";
        if (k > 0 && !(p->rain_t[k] > p->rain_t[k - 1])) return "rain_t must be ascending";
    }
    for (int s = 0; s < 4; ++s) {
        if (p->bc[s] < SWOF_BC_WALL || p->bc[s] > SWOF_BC_HALO) return "unknown boundary type";
        if (p->bc[s] == SWOF_BC_HALO && s < 2) return "HALO (strip) sides are S and N only";
        if (p->bc[s] == SWOF_BC_HALO && p->ny < 2) return "a strip needs >= 2 rows";
        if (!(p->inflow_width[s] >= 0) || !std::isfinite(p->inflow_width[s])) return "inflow_width must be finite and >= 0";
        const int n = (s < 2) ? p->ny : p->nx;
        if (p->bc[s] == SWOF_BC_INFLOW) {
            if (p->inflow_k0[s] < 0 || p->inflow_k1[s] > n || p->inflow_k0[s] >= p->inflow_k1[s])
                return "inflow segment out of range";
            if (p->n_hydro[s] < 1 || p->n_hydro[s] > SWOF_MAX_TABLE) return "inflow needs 1..16 hydrograph points";
            for (int k = 1; k < p->n_hydro[s]; ++k)
                if (!(p->hydro_t[s][k] > p->hydro_t[s][k - 1])) return "hydro_t must be ascending";
        }
    }
    if ((p->bc[0] == SWOF_BC_PERIODIC) != (p->bc[1] == SWOF_BC_PERIODIC) ||
        (p->bc[2] == SWOF_BC_PERIODIC) != (p->bc[3] == SWOF_BC_PERIODIC))
        return "periodic boundaries must be paired (W/E, S/N)";
    if (p->dt_hist_cap < 0) return "dt_hist_cap must be >= 0";
    if (p->graph_steps < 0) return "graph_steps must be >= 0";
    if (!(p->clamp_fail >= 0)) return "clamp_fail must be >= 0";
    if (p->flux != SWOF_FLUX_HLL && p->flux != SWOF_FLUX_RUSANOV) return "unknown flux";
    if (p->order < 0 || p->order > 2) return "order must be 0 (= 2), 1 or 2";
    if (p->cfl_mode != SWOF_CFL_CELL && p->cfl_mode != SWOF_CFL_FACE) return "unknown cfl_mode";
    if (p->ga_form != SWOF_GA_PRINTED && p->ga_form != SWOF_GA_DARCY) return "unknown ga_form";
    return nullptr;
}

int fail(swof_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

int cuda_fail(swof_ctx* c, cudaError_t e, const char* where) {
    return fail(c, SWOF_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                             \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
    } while (0)

constexpr int PW_BLOCKS = 1184;        // point-wise / face-CFL passes: 8 CTAs x 148 SMs, grid-stride

// one time step: predictor stage, then the corrector (Heun) or the order-1 commit
// (explicit Euler), then the reconstructed-value CFL pass when SWOF_CFL_FACE
void launch_second(swof_ctx* c, int par, cudaStream_t s) {
    if (c->kp.order == 1) euler_commit_kernel<<<PW_BLOCKS, PW_NT, 0, s>>>(c->kp, c->kb, par);
    else c->kcorr<<<c->sgrid, c->sblock, c->ssmem, s>>>(c->kp, c->kb, par);
    if (c->kp.cfl_mode == SWOF_CFL_FACE) cfl_face_kernel<<<c->cf_grid, dim3(CF_TX, CF_NTY), 0, s>>>(c->kp, c->kb, par, 0);
}
void launch_step(swof_ctx* c, int par, cudaStream_t s) {
    c->kpred<<<c->sgrid, c->sblock, c->ssmem, s>>>(c->kp, c->kb, par);
    launch_second(c, par, s);
}
void launch_step(swof_ctx* c, int par) { launch_step(c, par, c->stream); }

int build_graph(swof_ctx* c) {
    if (c->graph) return SWOF_OK;
    // capture on a private stream (the legacy default stream cannot be captured); the graph is
    // then launched on the context's stream
    cudaGraph_t g = nullptr;
    cudaStream_t cs = nullptr;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        for (int k = 0; k < c->graph_steps; ++k) launch_step(c, k & 1, cs);
        e = cudaStreamEndCapture(cs, &g);
    }
    cudaStreamDestroy(cs);
    if (e != cudaSuccess) return cuda_fail(c, e, "graph capture");
    e = cudaGraphInstantiate(&c->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { c->graph = nullptr; return cuda_fail(c, e, "cudaGraphInstantiate"); }
    return SWOF_OK;
}

// enqueue exactly n step launches (graph replays + eager remainder); keeps c->par in sync
int enqueue_steps(swof_ctx* c, int64_t n) {
    while (n > 0 && c->par != 0) { launch_step(c, c->par); c->par ^= 1; --n; }
    if (n >= c->graph_steps) {
        int rc = build_graph(c);
        if (rc) return rc;
        while (n >= c->graph_steps) {
            CK(cudaGraphLaunch(c->graph, c->stream));
            n -= c->graph_steps;
        }
    }
    while (n > 0) { launch_step(c, c->par); c->par ^= 1; --n; }
    CK(cudaGetLastError());
    return SWOF_OK;
}

int read_state(swof_ctx* c) {
    CK(cudaMemcpyAsync(c->h_st, c->kb.st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SWOF_OK;
}

int flags_rc(swof_ctx* c) {
    if (c->h_st->flags & (FLAG_NONFINITE | FLAG_BIGCLAMP)) {
        return fail(c, SWOF_ENUMERIC, (c->h_st->flags & FLAG_NONFINITE) ? "non-finite value reached the CFL maximum"
                                                                         : "a negative-height clamp exceeded clamp_fail");
    }
    return SWOF_OK;
}

int copy_field_in(swof_ctx* c, double* dst, const double* src) {
    const size_t w = (size_t)c->p.nx * sizeof(double);
    CK(cudaMemcpy2DAsync(dst, c->kp.pitch * sizeof(double), src, w, w, (size_t)c->p.ny, cudaMemcpyDefault, c->stream));
    return SWOF_OK;
}

int copy_field_out(swof_ctx* c, double* dst, const double* src) {
    const size_t w = (size_t)c->p.nx * sizeof(double);
    CK(cudaMemcpy2DAsync(dst, w, src, c->kp.pitch * sizeof(double), w, (size_t)c->p.ny, cudaMemcpyDefault, c->stream));
    return SWOF_OK;
}

__global__ void fill_kernel(double* a, int nx, int ny, int pitch, double v) {
    const long long n = (long long)nx * ny;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(k / nx), i = (int)(k - (long long)j * nx);
        a[(size_t)j * pitch + i] = v;
    }
}

}  // namespace

extern "C" {

int swof_launches_per_step(void) { return 2; }

int swof_check_line(void) {
    int line = 0;
    if (cudaMemcpyFromSymbol(&line, g_swof_assert_line, sizeof(int)) != cudaSuccess) return -1;
    return line;
}
int swof_ctx_launches_per_step(const swof_ctx* c) { return c ? 2 + (c->kp.cfl_mode == SWOF_CFL_FACE ? 1 : 0) : -1; }

int swof_selftest_math(int64_t n, uint64_t seed, int64_t* mismatches) {
    if (n < 0 || !mismatches) return SWOF_EINVAL;
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, 3 * sizeof(unsigned long long)) != cudaSuccess) return SWOF_ENOMEM;
    cudaMemset(d, 0, 3 * sizeof(unsigned long long));
    selftest_math_kernel<<<1184, 256>>>((long long)n, (unsigned long long)seed, d);
    unsigned long long h[3] = {0, 0, 0};
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return SWOF_ECUDA;
    for (int i = 0; i < 3; ++i) mismatches[i] = (int64_t)h[i];
    return SWOF_OK;
}

const char* swof_strerror(int code) {
    switch (code) {
        case SWOF_OK: return "ok";
        case SWOF_EINVAL: return "invalid argument";
        case SWOF_ENUMERIC: return "numerical failure";
        case SWOF_ECUDA: return "CUDA error";
        case SWOF_ENOMEM: return "out of memory";
        case SWOF_ESTATE: return "invalid call order";
        default: return "unknown error";
    }
}

const char* swof_last_error(const swof_ctx* c) { return c ? c->err.c_str() : "null context"; }

int swof_workspace_size(const swof_params* p, size_t* bytes) {
    if (validate(p) || !bytes) return SWOF_EINVAL;
    *bytes = make_layout(p, true).total;   // with room for a per-cell friction field
    return SWOF_OK;
}

// Picks the stage kernels (swof_march.cuh) for the context's physics and options and their launch shape.
static int choose_kernels(swof_ctx* c) {
    const KParams& k = c->kp;
    const bool ff = c->kb.fric != nullptr;
    const bool generic = k.flux != SWOF_FLUX_HLL || k.order == 1 || k.ga_form != SWOF_GA_PRINTED;
    const bool push = c->kb.push_any != 0, dry = c->p.dry_skip != 0;
    {
        c->kpred = select_march<false>(k.fk, k.ga != 0, ff, generic, push, dry);
        c->kcorr = select_march<true>(k.fk, k.ga != 0, ff, generic, push, dry);
        const int own_cols = M_OWN, nw = M_NW;
        // rows per warp segment, 1..64: minimise (waves of segments over the resident warp slots) x (rows +
        // ~3 rows of halo work per segment) -- small grids get short segments to fill the 148 SMs
        int occ_p = 0, occ_c = 0, dev = 0, nsm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, c->kpred, nw * 32, 0);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, c->kcorr, nw * 32, 0);
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return cuda_fail(c, e, "march kernel occupancy");
        const long long slots = (long long)(occ_p < occ_c ? occ_p : occ_c) * nsm * nw;
        const long long nstrip = (k.nx + own_cols - 1) / own_cols;
        int mh = 64;
        double best = 1e300;
        for (int h = 1; h <= 64; ++h) {
            const long long items = nstrip * ((k.ny + h - 1) / h);
            const double cost = (double)((items + slots - 1) / (slots > 0 ? slots : 1)) * (h + 3);
            if (cost < best) { best = cost; mh = h; }
        }
        const char* fixed = getenv("SWOF_MARCH_H");       // experiments
        if (fixed && atoi(fixed) > 0) mh = atoi(fixed);
        c->kp.march_h = mh;
        // on grids of >= 4 waves the last wave of segments is cut shorter (mh/4 rows) so that the SMs run dry
        // together (cfg3 +3 %, cfg4 +0.2 %; on 1-2 waves it costs up to 4 %)
        int g1 = (k.ny + mh - 1) / mh, h2 = mh;
        const char* tail = getenv("SWOF_MARCH_TAIL");
        const long long waves = nstrip * (long long)g1 / (slots > 0 ? slots : 1);
        const int tail_mode = tail ? atoi(tail) : 1;         // 0 off, 1 auto, 2 always (tests)
        if (tail_mode != 0 && mh >= 8 && (waves >= 4 || tail_mode == 2)) {
            h2 = mh / 4;
            long long g2 = (slots + nstrip - 1) / nstrip;                  // one wave of short segments
            if (tail_mode == 2) g2 = (k.ny / 2) / h2 > 0 ? (k.ny / 2) / h2 : 1;   // tests: half the rows
            const long long rows_tail = g2 * h2;
            const long long g1m = (k.ny - rows_tail) / mh;
            if (g1m >= 1) g1 = (int)g1m; else h2 = mh;
        }
        c->kp.march_g1 = g1;
        c->kp.march_h2 = h2;
        const long long nseg = g1 + (k.ny - (long long)g1 * mh + h2 - 1) / h2;
        const long long nwarps = nstrip * (k.ny > (long long)g1 * mh ? nseg : g1);
        c->sgrid = dim3((unsigned)((nwarps + nw - 1) / nw));
        c->sblock = dim3(nw * 32);
        c->ssmem = 0;
        return SWOF_OK;
    }
}

#if SWOF_MARCH_TMA
// the TMA tensor maps of the marching kernel's row ring (swof_march.cuh): for the predictor's input A and the
// corrector's input B, {h, hu, hv, z} as 2-D f64 tensors of nx x (ny + 2 GHOST_ROWS) elements (the spare rows
// included), row stride = the pitch, box 32 x TMA_ROWS; built once per context
static int make_tmaps(swof_ctx* c, const Layout& L) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 1;
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap maps[8];
    const KBufs& b = c->kb;
    double* f[8] = {b.Ah, b.Ahu, b.Ahv, b.z, b.Bh, b.Bhu, b.Bhv, b.z};
    for (int k = 0; k < 8; ++k) {
        const cuuint64_t dims[2] = {(cuuint64_t)c->p.nx, (cuuint64_t)c->p.ny + 2 * GHOST_ROWS};
        const cuuint64_t strides[1] = {(cuuint64_t)L.pitch * sizeof(double)};
        const cuuint32_t box[2] = {32, (cuuint32_t)TMA_ROWS};
        const cuuint32_t es[2] = {1, 1};
        if (encode(&maps[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, f[k] - (size_t)GHOST_ROWS * L.pitch, dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) return 1;
    }
    if (cudaMalloc(&c->d_tmaps, sizeof(maps)) != cudaSuccess) return 1;
    if (cudaMemcpy(c->d_tmaps, maps, sizeof(maps), cudaMemcpyHostToDevice) != cudaSuccess) return 1;
    c->kb.tmaps = c->d_tmaps;
    return 0;
}
#endif

int swof_create(const swof_params* p, const double* z, const double* fric_field, void* d_workspace, size_t ws_bytes,
                void* cuda_stream, swof_ctx** out) {
    if (!out) return SWOF_EINVAL;
    *out = nullptr;
    if (validate(p) || !z) return SWOF_EINVAL;
    if (p->fric_law == SWOF_FRIC_NONE && fric_field) return SWOF_EINVAL;
    if (!fric_field && p->fric_law != SWOF_FRIC_NONE && !(p->fric_coef > 0)) return SWOF_EINVAL;
    swof_ctx* c = new (std::nothrow) swof_ctx();
    if (!c) return SWOF_ENOMEM;
    c->p = *p;
    c->stream = (cudaStream_t)cuda_stream;
    c->graph_steps = p->graph_steps > 0 ? (p->graph_steps + 1) / 2 * 2 : 16;
    const bool has_ff = fric_field != nullptr;
    const Layout L = make_layout(p, has_ff);
    if (d_workspace) {
        if (ws_bytes < L.total || ((uintptr_t)d_workspace & 255)) { delete c; return SWOF_ENOMEM; }
        c->ws = d_workspace;
    } else {
        if (cudaMalloc(&c->ws, L.total) != cudaSuccess) { delete c; return SWOF_ENOMEM; }
        c->own_ws = true;
    }
    c->ws_bytes = L.total;
    if (cudaMallocHost((void**)&c->h_st, sizeof(DevState)) != cudaSuccess) { swof_destroy(c); return SWOF_ENOMEM; }

    char* base = (char*)c->ws;
    KBufs& b = c->kb;
    const size_t F = L.field;
    const size_t g = (size_t)GHOST_ROWS * L.pitch * sizeof(double);      // row 0 of a field
    b.Ah = (double*)(base + L.off_A + g); b.Ahu = (double*)(base + L.off_A + F + g); b.Ahv = (double*)(base + L.off_A + 2 * F + g);
    b.Bh = (double*)(base + L.off_B + g); b.Bhu = (double*)(base + L.off_B + F + g); b.Bhv = (double*)(base + L.off_B + 2 * F + g);
    b.z = (double*)(base + L.off_z + g);
    b.VA = p->ga_enabled ? (double*)(base + L.off_VA + g) : nullptr;
    b.VB = p->ga_enabled ? (double*)(base + L.off_VB + g) : nullptr;
    b.fric = has_ff ? (double*)(base + L.off_fric + g) : nullptr;
    b.st = (DevState*)(base + L.off_st);
    std::memset(b.push, 0, sizeof(b.push));
    b.push_any = 0;
    b.tmaps = nullptr;
    b.dt_hist = (double*)(base + L.off_hist);
    b.dt_cap = p->dt_hist_cap > 0 ? p->dt_hist_cap : (int64_t)1 << 20;
    c->d_part = (double*)(base + L.off_part);

    KParams& k = c->kp;
    std::memset(&k, 0, sizeof(k));
    k.nx = p->nx; k.ny = p->ny; k.pitch = (int)L.pitch;
    k.fric_law = p->fric_law; k.has_fric_field = has_ff; k.ga = p->ga_enabled != 0;
    k.dx = p->dx; k.dy = p->dy; k.g = p->g; k.cfl = p->cfl; k.dt_max = p->dt_max; k.h_eps = p->h_eps;
    k.fric_coef = p->fric_coef;
    k.clamp_fail = p->clamp_fail > 0 ? p->clamp_fail : 1e-6;
    k.Ks = p->ga_Ks; k.hf = p->ga_hf; k.A = p->ga_A; k.dtheta = p->ga_dtheta;
    k.fk = p->fric_law == SWOF_FRIC_NONE ? 0
         : (p->fric_law == SWOF_FRIC_MANNING || p->fric_law == SWOF_FRIC_STRICKLER) ? 1 : 2;
    k.flux = p->flux;
    k.order = p->order == 1 ? 1 : 2;
    k.cfl_mode = p->cfl_mode;
    k.ga_form = p->ga_form;
    k.n_rain = p->n_rain;
    for (int i = 0; i < p->n_rain; ++i) { k.rain_t[i] = p->rain_t[i]; k.rain_rate[i] = p->rain_rate[i]; }
    for (int s = 0; s < 4; ++s) {
        k.bc[s] = p->bc[s];
        k.k0[s] = p->inflow_k0[s]; k.k1[s] = p->inflow_k1[s];
        k.n_hydro[s] = p->bc[s] == SWOF_BC_INFLOW ? p->n_hydro[s] : 0;
        k.width[s] = p->inflow_width[s] > 0 ? p->inflow_width[s]
                   : (double)(p->inflow_k1[s] - p->inflow_k0[s]) * ((s < 2) ? p->dy : p->dx);
        for (int i = 0; i < k.n_hydro[s]; ++i) { k.hydro_t[s][i] = p->hydro_t[s][i]; k.hydro_q[s][i] = p->hydro_q[s][i]; }
    }
    c->diag_blocks = DIAG_BLOCKS;
    c->cf_grid = dim3((unsigned)((p->nx + CF_TX - 1) / CF_TX), (unsigned)((p->ny + CF_TY - 1) / CF_TY));

    {
        const int rc = choose_kernels(c);
        if (rc != SWOF_OK) { swof_destroy(c); return rc; }
    }
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMemsetAsync(c->ws, 0, L.total, c->stream);
    if (e != cudaSuccess) { int rc = cuda_fail(c, e, "swof_create"); fprintf(stderr, "swof: %s\n", c->err.c_str()); swof_destroy(c); return rc; }
    int rc = copy_field_in(c, b.z, z);
    if (!rc && has_ff) rc = copy_field_in(c, b.fric, fric_field);
    if (!rc) { e = cudaStreamSynchronize(c->stream); if (e != cudaSuccess) rc = cuda_fail(c, e, "swof_create sync"); }
    if (rc) { swof_destroy(c); return rc; }
    if (has_ff) {
        // per-cell coefficients must be > 0 (NonPositiveCoefficient)
        std::vector<double> tmp((size_t)p->nx);
        for (int j = 0; j < p->ny; ++j) {
            if (cudaMemcpy(tmp.data(), b.fric + (size_t)j * L.pitch, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) { swof_destroy(c); return SWOF_ECUDA; }
            for (double v : tmp) if (!(v > 0) || !std::isfinite(v)) { swof_destroy(c); return SWOF_EINVAL; }
        }
    }
#if SWOF_MARCH_TMA
    if (make_tmaps(c, L)) { swof_destroy(c); return SWOF_ECUDA; }
#endif
    *out = c;
    return SWOF_OK;
}

int swof_set_state(swof_ctx* c, const double* h, const double* hu, const double* hv, const double* v_inf, double t0) {
    if (!c) return SWOF_EINVAL;
    if (!h || !hu || !hv || !std::isfinite(t0)) return fail(c, SWOF_EINVAL, "set_state: h, hu, hv required, t0 finite");
    int rc;
    if ((rc = copy_field_in(c, c->kb.Ah, h)) || (rc = copy_field_in(c, c->kb.Ahu, hu)) || (rc = copy_field_in(c, c->kb.Ahv, hv)))
        return rc;
    if (c->kp.ga) {
        if (v_inf) { if ((rc = copy_field_in(c, c->kb.VA, v_inf))) return rc; }
        else fill_kernel<<<1184, 256, 0, c->stream>>>(c->kb.VA, c->p.nx, c->p.ny, c->kp.pitch, c->p.ga_vinf0);
    }
    DevState s;
    std::memset(&s, 0, sizeof(s));
    s.t[0] = t0;
    s.t_end = INFINITY;
    s.step_limit = INT64_MAX;
    s.big_clamp_cell = -1;
    s.big_clamp_step = -1;
    *c->h_st = s;
    CK(cudaMemcpyAsync(c->kb.st, c->h_st, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
    init_cfl_kernel<<<1184, 256, 0, c->stream>>>(c->kp, c->kb);
    if (c->kp.cfl_mode == SWOF_CFL_FACE) {               // replace the cell maxima by the face ones
        CK(cudaMemsetAsync(&c->kb.st->amax[0][0], 0, 2 * sizeof(unsigned long long), c->stream));
        cfl_face_kernel<<<c->cf_grid, dim3(CF_TX, CF_NTY), 0, c->stream>>>(c->kp, c->kb, 0, 1);
    }
    CK(cudaGetLastError());
    c->par = 0;
    if ((rc = read_state(c))) return rc;
    if (c->h_st->flags & FLAG_BADINPUT) {
        c->have_state = false;
        return fail(c, SWOF_EINVAL, "set_state: h < 0 or a non-finite value in the state");
    }
    c->have_state = true;
    return SWOF_OK;
}

int swof_step(swof_ctx* c, int64_t nsteps) {
    if (!c) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_step before swof_set_state");
    if (nsteps < 0) return fail(c, SWOF_EINVAL, "nsteps < 0");
    // no t_end clipping, no step limit
    const double inf = INFINITY;
    const long long lim = INT64_MAX;
    CK(cudaMemcpyAsync(&c->kb.st->t_end, &inf, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(&c->kb.st->step_limit, &lim, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    int rc = enqueue_steps(c, nsteps);
    if (rc) return rc;
    if ((rc = read_state(c))) return rc;
    return flags_rc(c);
}

int swof_run(swof_ctx* c, double t_end, int64_t max_steps, int64_t* steps_done) {
    if (!c) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_run before swof_set_state");
    if (max_steps < 0 || std::isnan(t_end)) return fail(c, SWOF_EINVAL, "swof_run: bad t_end / max_steps");
    int rc;
    if ((rc = read_state(c))) return rc;
    const long long step0 = c->h_st->step[c->par];
    // saturating: max_steps = INT64_MAX means 'no cap' whatever the steps already taken
    const long long lim = (max_steps > INT64_MAX - step0) ? (long long)INT64_MAX : step0 + max_steps;
    CK(cudaMemcpyAsync(&c->kb.st->t_end, &t_end, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(&c->kb.st->step_limit, &lim, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    // replay until the device reports done (t >= t_end, step limit, or a halt); steps past the end
    // are exact no-ops, so overshooting by a partial batch is harmless
    int64_t batch = c->graph_steps;
    for (;;) {
        const long long cur = c->h_st->step[c->par];
        const double tc = c->h_st->t[c->par];
        if (!(tc < t_end) || cur >= lim || (c->h_st->flags & (FLAG_NONFINITE | FLAG_BIGCLAMP))) break;
        int64_t left = lim - cur;
        int64_t n = left < batch ? left : batch;
        if ((rc = enqueue_steps(c, n))) return rc;
        if ((rc = read_state(c))) return rc;
        if (batch < 64 * c->graph_steps) batch *= 2;
    }
    if (steps_done) *steps_done = c->h_st->step[c->par] - step0;
    return flags_rc(c);
}

int swof_get_state(const swof_ctx* cc, double* h, double* hu, double* hv, double* v_inf, double* t, int64_t* step) {
    swof_ctx* c = const_cast<swof_ctx*>(cc);  // logically const: only scratch, the state cache and err change
    if (!c) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_get_state before swof_set_state");
    int rc;
    if (h && (rc = copy_field_out(c, h, c->kb.Ah))) return rc;
    if (hu && (rc = copy_field_out(c, hu, c->kb.Ahu))) return rc;
    if (hv && (rc = copy_field_out(c, hv, c->kb.Ahv))) return rc;
    if (v_inf && c->kp.ga && (rc = copy_field_out(c, v_inf, c->kb.VA))) return rc;
    if ((rc = read_state(c))) return rc;
    if (t) *t = c->h_st->t[c->par];
    if (step) *step = c->h_st->step[c->par];
    return SWOF_OK;
}

int swof_get_dt_history(const swof_ctx* cc, double* dt, int64_t cap, int64_t* n) {
    swof_ctx* c = const_cast<swof_ctx*>(cc);  // logically const: only scratch, the state cache and err change
    if (!c || (!dt && cap > 0) || cap < 0) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_get_dt_history before swof_set_state");
    int rc;
    if ((rc = read_state(c))) return rc;
    long long steps = c->h_st->step[c->par];
    long long m = steps < c->kb.dt_cap ? steps : c->kb.dt_cap;
    if (m > cap) m = cap;
    if (m > 0) {
        CK(cudaMemcpyAsync(dt, c->kb.dt_hist, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    if (n) *n = m;
    return SWOF_OK;
}

int swof_get_diag(const swof_ctx* cc, swof_diag* d) {
    swof_ctx* c = const_cast<swof_ctx*>(cc);  // logically const: only scratch, the state cache and err change
    if (!c || !d) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_get_diag before swof_set_state");
    diag_kernel<<<c->diag_blocks, DIAG_NT, 0, c->stream>>>(c->kp, c->kb, c->d_part);
    CK(cudaGetLastError());
    std::vector<double> part((size_t)c->diag_blocks * 5);
    CK(cudaMemcpyAsync(part.data(), c->d_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    int rc;
    if ((rc = read_state(c))) return rc;
    double sh = 0, sv = 0, mn = INFINITY, mx = 0, wet = 0;
    for (int b = 0; b < c->diag_blocks; ++b) {
        sh += part[b * 5 + 0];
        sv += part[b * 5 + 1];
        mn = std::fmin(mn, part[b * 5 + 2]);
        mx = std::fmax(mx, part[b * 5 + 3]);
        wet += part[b * 5 + 4];
    }
    const DevState& s = *c->h_st;
    std::memset(d, 0, sizeof(*d));
    d->t = s.t[c->par];
    d->step = s.step[c->par];
    double ax, ay;
    std::memcpy(&ax, &s.amax[c->par][0], 8);
    std::memcpy(&ay, &s.amax[c->par][1], 8);
    double dt = c->p.cfl / (ax / c->p.dx + ay / c->p.dy);
    d->dt_next = std::fmin(dt, c->p.dt_max);
    d->volume = sh * c->p.dx * c->p.dy;
    d->vinf_volume = sv * c->p.dx * c->p.dy;
    d->h_min = mn;
    d->h_max = mx;
    d->wet_cells = (int64_t)wet;
    d->clamps = (int64_t)s.clamps;
    d->clamped_mass = s.clamped_mass;
    std::memcpy(&d->clamp_max, &s.clamp_max_bits, 8);
    d->flags = s.flags;
    d->big_clamp_cell = s.big_clamp_cell;
    d->big_clamp_step = s.big_clamp_step;
    return SWOF_OK;
}

int swof_predictor(swof_ctx* c, double* h, double* hu, double* hv, double* v_inf) {
    if (!c) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_predictor before swof_set_state");
    // the predictor zeroes the other parity's maxima; keep a copy so the state is left untouched
    DevState saved;
    int rc;
    if ((rc = read_state(c))) return rc;
    saved = *c->h_st;
    c->kpred<<<c->sgrid, c->sblock, c->ssmem, c->stream>>>(c->kp, c->kb, c->par);
    CK(cudaGetLastError());
    if (h && (rc = copy_field_out(c, h, c->kb.Bh))) return rc;
    if (hu && (rc = copy_field_out(c, hu, c->kb.Bhu))) return rc;
    if (hv && (rc = copy_field_out(c, hv, c->kb.Bhv))) return rc;
    if (v_inf && c->kp.ga && (rc = copy_field_out(c, v_inf, c->kb.VB))) return rc;
    *c->h_st = saved;
    CK(cudaMemcpyAsync(c->kb.st, c->h_st, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SWOF_OK;
}

int swof_step_profiled(swof_ctx* c, int64_t nsteps, double* ms) {
    if (!c || !ms || nsteps < 0) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_step_profiled before swof_set_state");
    const double inf = INFINITY;
    const long long lim = INT64_MAX;
    CK(cudaMemcpyAsync(&c->kb.st->t_end, &inf, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(&c->kb.st->step_limit, &lim, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    cudaEvent_t ev[3];
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double acc[2] = {0, 0};
    for (int64_t n = 0; n < nsteps; ++n) {
        CK(cudaEventRecord(ev[0], c->stream));
        c->kpred<<<c->sgrid, c->sblock, c->ssmem, c->stream>>>(c->kp, c->kb, c->par);
        CK(cudaEventRecord(ev[1], c->stream));
        launch_second(c, c->par, c->stream);
        CK(cudaEventRecord(ev[2], c->stream));
        c->par ^= 1;
        CK(cudaEventSynchronize(ev[2]));
        float a, b;
        CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
        CK(cudaEventElapsedTime(&b, ev[1], ev[2]));
        acc[0] += a;
        acc[1] += b;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    ms[0] = acc[0];
    ms[1] = acc[1];
    int rc;
    if ((rc = read_state(c))) return rc;
    return flags_rc(c);
}

int swof_halo_rows(swof_ctx* c, int32_t set, int32_t side, double** send, double** recv, size_t* bytes) {
    if (!c || !send || !recv || (side != SWOF_SIDE_S && side != SWOF_SIDE_N) || set < 0 || set > 2)
        return SWOF_EINVAL;
    const size_t pitch = (size_t)c->kp.pitch, ny = (size_t)c->p.ny;
    double* f[3] = {nullptr, nullptr, nullptr};
    if (set == 0) { f[0] = c->kb.Ah; f[1] = c->kb.Ahu; f[2] = c->kb.Ahv; }
    else if (set == 1) { f[0] = c->kb.Bh; f[1] = c->kb.Bhu; f[2] = c->kb.Bhv; }
    else f[0] = c->kb.z;
    for (int k = 0; k < 3; ++k) {
        send[k] = recv[k] = nullptr;
        if (!f[k]) continue;
        if (side == SWOF_SIDE_S) {            // rows 0, 1 go south; rows -2, -1 come from the south
            send[k] = f[k];
            recv[k] = f[k] - GHOST_ROWS * pitch;
        } else {                              // rows ny-2, ny-1 go north; rows ny, ny+1 come from it
            send[k] = f[k] + (ny - GHOST_ROWS) * pitch;
            recv[k] = f[k] + ny * pitch;
        }
    }
    if (bytes) *bytes = GHOST_ROWS * pitch * sizeof(double);
    return SWOF_OK;
}

int swof_set_halo_push(swof_ctx* c, int32_t side, double* const* set0, double* const* set1) {
    if (!c || (side != SWOF_SIDE_S && side != SWOF_SIDE_N)) return SWOF_EINVAL;
    if (c->p.bc[side] != SWOF_BC_HALO) return fail(c, SWOF_EINVAL, "halo push needs a SWOF_BC_HALO side");
    const int s = side == SWOF_SIDE_S ? 0 : 1;
    for (int k = 0; k < 3; ++k) {
        c->kb.push[s][0][k] = set0 ? set0[k] : nullptr;
        c->kb.push[s][1][k] = set1 ? set1[k] : nullptr;
    }
    c->kb.push_any = 0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) c->kb.push_any |= c->kb.push[a][b][0] != nullptr;
    // the pushing kernels are the generic tiled instance compiled with the fused exchange
    const int rc = choose_kernels(c);
    if (rc != SWOF_OK) return rc;
    if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }   // kernels changed
    return SWOF_OK;
}

int swof_ipc_handle(swof_ctx* c, void* handle, uint64_t* ws_base) {
    if (!c || !handle) return SWOF_EINVAL;
    if (!c->own_ws) return fail(c, SWOF_EINVAL, "IPC export needs the library-allocated workspace");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->ws));
    std::memcpy(handle, &h, sizeof(h));
    if (ws_base) *ws_base = (uint64_t)(uintptr_t)c->ws;
    return SWOF_OK;
}

int swof_ipc_open(const void* handle, void** base) {
    if (!handle || !base) return SWOF_EINVAL;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) { cudaGetLastError(); return SWOF_ECUDA; }
    return SWOF_OK;
}

int swof_ipc_close(void* base) {
    if (!base) return SWOF_EINVAL;
    return cudaIpcCloseMemHandle(base) == cudaSuccess ? SWOF_OK : SWOF_ECUDA;
}

int swof_copy(void* dst, const void* src, size_t bytes, void* cuda_stream) {
    if ((!dst || !src) && bytes) return SWOF_EINVAL;
    if (!bytes) return SWOF_OK;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)cuda_stream) == cudaSuccess ? SWOF_OK
                                                                                                      : SWOF_ECUDA;
}

int swof_enqueue_phase(swof_ctx* c, int32_t phase) {
    if (!c) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_enqueue_phase before swof_set_state");
    if (phase == 0) {
        c->kpred<<<c->sgrid, c->sblock, c->ssmem, c->stream>>>(c->kp, c->kb, c->par);
    } else if (phase == 1) {
        if (c->kp.order == 1) euler_commit_kernel<<<PW_BLOCKS, PW_NT, 0, c->stream>>>(c->kp, c->kb, c->par);
        else c->kcorr<<<c->sgrid, c->sblock, c->ssmem, c->stream>>>(c->kp, c->kb, c->par);
    } else if (phase == 2) {
        if (c->kp.cfl_mode == SWOF_CFL_FACE) cfl_face_kernel<<<c->cf_grid, dim3(CF_TX, CF_NTY), 0, c->stream>>>(c->kp, c->kb, c->par, 0);
        c->par ^= 1;                          // the step is complete
    } else {
        return fail(c, SWOF_EINVAL, "phase must be 0, 1 or 2");
    }
    CK(cudaGetLastError());
    return SWOF_OK;
}

int swof_cfl_maxima(swof_ctx* c, uint64_t** dev_ptr) {
    if (!c || !dev_ptr) return SWOF_EINVAL;
    *dev_ptr = (uint64_t*)&c->kb.st->amax[c->par][0];
    return SWOF_OK;
}

int swof_refresh_cfl(swof_ctx* c) {
    if (!c) return SWOF_EINVAL;
    if (!c->have_state) return fail(c, SWOF_ESTATE, "swof_refresh_cfl before swof_set_state");
    if (c->par != 0) return fail(c, SWOF_ESTATE, "swof_refresh_cfl only right after swof_set_state");
    CK(cudaMemsetAsync(&c->kb.st->amax[0][0], 0, 2 * sizeof(unsigned long long), c->stream));
    if (c->kp.cfl_mode == SWOF_CFL_FACE) cfl_face_kernel<<<c->cf_grid, dim3(CF_TX, CF_NTY), 0, c->stream>>>(c->kp, c->kb, 0, 1);
    else init_cfl_kernel<<<1184, 256, 0, c->stream>>>(c->kp, c->kb);
    CK(cudaGetLastError());
    return SWOF_OK;
}

int swof_set_limits(swof_ctx* c, double t_end, int64_t step_limit) {
    if (!c || std::isnan(t_end)) return SWOF_EINVAL;
    const long long lim = (long long)step_limit;
    CK(cudaMemcpyAsync(&c->kb.st->t_end, &t_end, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(&c->kb.st->step_limit, &lim, sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));      // the host values are stack temporaries
    return SWOF_OK;
}

int swof_sync(swof_ctx* c) {
    if (!c) return SWOF_EINVAL;
    int rc;
    if ((rc = read_state(c))) return rc;
    return flags_rc(c);
}

}  // extern "C"

namespace {
bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
int flow_direction_impl(const T* z, int32_t nx, int32_t ny, uint8_t* dir, void* stream) {
    if (!z || !dir || nx < 1 || ny < 1) return SWOF_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = (size_t)nx * (size_t)ny;
    const T* dz = z;
    uint8_t* dd = dir;
    T* tz = nullptr;
    uint8_t* td = nullptr;
    int rc = SWOF_OK;
    if (!is_device_ptr(z)) {                             // host raster: stage it on the device
        if (cudaMalloc(&tz, n * sizeof(T)) != cudaSuccess) return SWOF_ENOMEM;
        if (cudaMemcpyAsync(tz, z, n * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess) rc = SWOF_ECUDA;
        dz = tz;
    }
    if (!rc && !is_device_ptr(dir)) {
        if (cudaMalloc(&td, n) != cudaSuccess) rc = SWOF_ENOMEM;
        dd = td;
    }
    if (!rc) {
        const dim3 grid((unsigned)((nx + D8_TX - 1) / D8_TX), (unsigned)((ny + D8Tile<T>::TY - 1) / D8Tile<T>::TY));
        d8_kernel<T><<<grid, D8_NT, 0, s>>>(dz, nx, ny, dd);
        if (cudaGetLastError() != cudaSuccess) rc = SWOF_ECUDA;
    }
    if (!rc && td && cudaMemcpyAsync(dir, td, n, cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = SWOF_ECUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess && !rc) rc = SWOF_ECUDA;
    if (tz) cudaFree(tz);
    if (td) cudaFree(td);
    return rc;
}
}  // namespace

extern "C" {

int swof_flow_direction(const double* z, int32_t nx, int32_t ny, uint8_t* dir, void* cuda_stream) {
    return flow_direction_impl<double>(z, nx, ny, dir, cuda_stream);
}

int swof_flow_direction_f32(const float* z, int32_t nx, int32_t ny, uint8_t* dir, void* cuda_stream) {
    return flow_direction_impl<float>(z, nx, ny, dir, cuda_stream);
}

void swof_destroy(swof_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->own_ws && c->ws) cudaFree(c->ws);
    if (c->h_st) cudaFreeHost(c->h_st);
    if (c->d_tmaps) cudaFree(c->d_tmaps);
    delete c;
}

}  // extern "C"
