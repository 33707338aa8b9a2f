// fp64_peak.cu -- measure the B200 fp64 pipe: DFMA / DADD / DMUL issue rates and IEEE div/sqrt
// throughput (the ALU roofline denominator of DESIGN.md §5).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, double a, double b, int iters) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) {  // DFMA
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            } else if (OP == 1) {  // DADD
                x0 = x0 + a; x1 = x1 + a; x2 = x2 + a; x3 = x3 + a; x4 = x4 + a; x5 = x5 + a; x6 = x6 + a; x7 = x7 + a;
            } else if (OP == 2) {  // IEEE division
                x0 = b / x0; x1 = b / x1; x2 = b / x2; x3 = b / x3; x4 = b / x4; x5 = b / x5; x6 = b / x6; x7 = b / x7;
            } else {  // IEEE sqrt
                x0 = sqrt(x0 + b); x1 = sqrt(x1 + b); x2 = sqrt(x2 + b); x3 = sqrt(x3 + b);
                x4 = sqrt(x4 + b); x5 = sqrt(x5 + b); x6 = sqrt(x6 + b); x7 = sqrt(x7 + b);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <int OP>
double run(const char* name, int iters) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    k<OP><<<blocks, threads>>>(out, 0.999999, 1e-7, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, threads>>>(out, 0.999999, 1e-7, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 16 * 8;
    const double rate = ops / (ms * 1e-3) / 1e9;
    printf("{\"op\": \"%s\", \"Gop_per_s\": %.1f, \"ms\": %.3f, \"sms\": %d}\n", name, rate, ms, sms);
    cudaFree(out);
    return rate;
}

int main() {
    run<0>("dfma", 4000);
    run<1>("dadd", 4000);
    run<2>("ddiv_ieee", 200);
    run<3>("dsqrt_ieee", 200);
    run<0>("dfma", 4000);
    return 0;
}
