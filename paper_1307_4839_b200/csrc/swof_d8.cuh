// swof_d8.cuh -- sm_100a kernel of the D8 flow direction (the paper's user function
// is listed at P:683-708): for each DEM point, the direction (1..8: E, SE, S, SW, W, NW, N, NE; rows
// grow northwards; 0 = none) of the lowest of its 8 neighbours that is > 0 and strictly below the
// point, the first one in that order on ties -- exactly the listing's
//     min = own value; for i in 0..7: if (nghb[i] > 0 && nghb[i] < min) { index = i + 1; min = nghb[i]; }
// Neighbours outside the raster are absent.  HBM-bound: one read of the raster, one byte written per
// point.  A CTA stages a 256 x 32 tile plus its 1-point halo in shared memory with coalesced row loads
// (warp-per-row, all of a row's loads issued before its stores), then each thread walks the 32 rows of
// one column with a 3 x 3 register window (3 shared loads per point; lanes = consecutive columns:
// conflict-free shared reads, 32-byte coalesced code stores).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace swof {

constexpr int D8_NT = 256;
constexpr int D8_TX = D8_NT;                                         // one column per thread
constexpr int D8_LW = D8_TX + 2;
template <typename T> struct D8Tile {                                // rows walked by each thread (<= 48 KB smem)
    static constexpr int TY = sizeof(T) == 4 ? 32 : 16;
    static constexpr int LH = TY + 2;
};

template <typename T>
__global__ void __launch_bounds__(D8_NT) d8_kernel(const T* __restrict__ z, int nx, int ny, uint8_t* __restrict__ dir) {
    constexpr int D8_TY = D8Tile<T>::TY, D8_LH = D8Tile<T>::LH;
    __shared__ T s[D8_LH][D8_LW];
    const int i0 = blockIdx.x * D8_TX, j0 = blockIdx.y * D8_TY;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // shared memory holds t = (v > 0) ? v : NaN: the listing's test "n > 0 && n < min" becomes "t < min"
    // (a NaN compares false), and the centre's own start value min = t_centre behaves exactly like the
    // raw value (a centre <= 0 or NaN admits no neighbour either way); absent neighbours are NaN too
    const T nan = __int_as_float(0x7fc00000) * T(1);
    // stage the tile + 1-point halo: warp w loads rows w, w + 8, ...; lanes walk the row
    for (int r = warp; r < D8_LH; r += D8_NT / 32) {
        const int gj = j0 + r - 1;
        const bool rowok = gj >= 0 && gj < ny;
        const T* row = z + (size_t)(rowok ? gj : 0) * nx;
        T v[(D8_LW + 31) / 32];
#pragma unroll
        for (int k = 0; k < (D8_LW + 31) / 32; ++k) {
            const int c = lane + 32 * k, gi = i0 + c - 1;
            const T x = (rowok && c < D8_LW && gi >= 0 && gi < nx) ? row[gi] : nan;
            v[k] = x > T(0) ? x : nan;
        }
#pragma unroll
        for (int k = 0; k < (D8_LW + 31) / 32; ++k) {
            const int c = lane + 32 * k;
            if (c < D8_LW) s[r][c] = v[k];
        }
    }
    __syncthreads();
    const int c = threadIdx.x;
    const int gi = i0 + c;
    if (gi >= nx) return;
    const int sc = c + 1;
    // 3 x 3 window sliding north: rows r-1 (south), r, r+1 (north) of columns sc-1, sc, sc+1
    T sw = s[0][sc - 1], so = s[0][sc], se = s[0][sc + 1];
    T w = s[1][sc - 1], ce = s[1][sc], e = s[1][sc + 1];
    uint8_t* out = dir + (size_t)j0 * nx + gi;
    const int nr = ny - j0 < D8_TY ? ny - j0 : D8_TY;
#pragma unroll 4
    for (int r = 1; r <= nr; ++r) {
        const T nw = s[r + 1][sc - 1], no = s[r + 1][sc], ne = s[r + 1][sc + 1];
        // E, SE, S, SW, W, NW, N, NE
        const T nb[8] = {e, se, so, sw, w, nw, no, ne};
        T mn = ce;
        int index = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (nb[k] < mn) {
                index = k + 1;
                mn = nb[k];
            }
        }
        *out = (uint8_t)index;
        out += nx;
        sw = w; so = ce; se = e;
        w = nw; ce = no; e = ne;
    }
}

}  // namespace swof
