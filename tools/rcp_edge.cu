// Check the kernels' fast IEEE reciprocal / division / sqrt against CUDA's operators on edge-case
// mantissas (near powers of two), where Newton-refined sequences are most likely to round wrongly.
#include <cstdio>
#include "../paper_1307_4839_b200/csrc/swof_kernels.cuh"
using namespace swof;
__global__ void k(long long n, unsigned long long* bad, double* ex) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int kind = (int)(i & 7);
        const long long j = i >> 3;
        const int e = (int)(j % 61) - 30;
        const long long m = j / 61;                       // offset from the power of two in ulps
        double base = ldexp(1.0, e);
        double y = (kind & 1) ? __longlong_as_double(__double_as_longlong(base) - 1 - m)
                              : __longlong_as_double(__double_as_longlong(base) + m);
        if (kind & 2) y = -y;
        const double r1 = drcp(y), r2 = 1.0 / y;
        if (__double_as_longlong(r1) != __double_as_longlong(r2)) {
            if (atomicAdd(&bad[0], 1ull) == 0) { ex[0] = y; ex[1] = r1; ex[2] = r2; }
            if (rcp_ok(y)) atomicAdd(&bad[3], 1ull);          // a mismatch outside the all-ones operands
        }
        const double x = 1.0 + (double)(m % 1000) * 0x1p-52;
        const double q1 = ddiv_fast(x, y), q2 = x / y;
        if (__double_as_longlong(q1) != __double_as_longlong(q2)) {
            if (atomicAdd(&bad[1], 1ull) == 0) { ex[3] = x; ex[4] = y; }
            if (rcp_ok(y)) atomicAdd(&bad[3], 1ull);
        }
        const double s = fabs(y);
        const double s1 = dsqrt_fast(s), s2 = sqrt(s);
        if (__double_as_longlong(s1) != __double_as_longlong(s2)) { if (atomicAdd(&bad[2], 1ull) == 0) { ex[5] = s; } }
    }
}
int main() {
    unsigned long long* bad; double* ex;
    cudaMallocManaged(&bad, 4 * sizeof(unsigned long long)); cudaMallocManaged(&ex, 8 * sizeof(double));
    for (int i = 0; i < 4; ++i) bad[i] = 0;
    const long long n = 8LL * 61 * 2000000;
    k<<<1184, 256>>>(n, bad, ex);
    cudaDeviceSynchronize();
    printf("operands %lld  rcp mismatches %llu  div %llu  sqrt %llu  not caught by rcp_ok %llu\n", n, bad[0], bad[1],
           bad[2], bad[3]);
    if (bad[0]) printf("rcp example y=%.17g fast=%.17g ieee=%.17g\n", ex[0], ex[1], ex[2]);
    if (bad[1]) printf("div example x=%.17g y=%.17g\n", ex[3], ex[4]);
    if (bad[2]) printf("sqrt example s=%.17g\n", ex[5]);
    return 0;
}
