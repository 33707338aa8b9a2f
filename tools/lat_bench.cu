// Latency of dependent fp64 instructions on sm_100a (one warp, a chain of N dependent ops; clock64 around it)
// and throughput with W warps per SM of independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu && tools/lat_bench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b) {
    double x = a + threadIdx.x * 1e-9, y = b;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) {
        if (OP == 0) x = x + y;                          // DADD
        if (OP == 1) x = x * y;                          // DMUL
        if (OP == 2) x = __fma_rn(x, y, b);              // DFMA
        if (OP == 3) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }   // MUFU
        if (OP == 4) x = (x < y) ? x : y + 0.0 * i;      // DSETP + FSEL chain (min)
        if (OP == 5) x = __shfl_xor_sync(0xffffffffu, x, 1);   // SHFL (x2 for a double)
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 64 * 8);
    const char* names[] = {"DADD", "DMUL", "DFMA", "MUFU.RCP64H", "DSETP+FSEL(min)", "SHFL(double)"};
    void (*k[])(double*, long long*, double, double) = {chain<0>, chain<1>, chain<2>, chain<3>, chain<4>, chain<5>};
    for (int op = 0; op < 6; ++op) {
        k[op]<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        // throughput: 148 SMs x W warps of independent chains, device time
        for (int w : {4, 8, 16, 32}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            k[op]<<<148, 32 * w>>>(out, cyc, 1.0000001, 0.9999999);
            cudaEventRecord(e0);
            k[op]<<<148, 32 * w>>>(out, cyc, 1.0000001, 0.9999999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 148.0 * 32 * w * N;
            printf("%-16s latency %.2f cyc | %2d warps/SM: %.3f T lane-ops/s\n", names[op], (double)c / N, w,
                   ops / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
