// Cost of one same-address u64 atomicMax per CTA at the stage kernels' grid size (139,776 CTAs of 256
// threads) vs spreading the CTAs over 64 addresses, with and without some work per CTA.
#include <cstdio>
__global__ void k(unsigned long long* a, int spread, int work, double* sink) {
    double x = threadIdx.x * 1e-3;
    for (int i = 0; i < work; ++i) x = x * 0.999 + 1e-7;
    if (x == 12345.0) sink[0] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int s = spread ? (blockIdx.x % 64) * 16 : 0;     // 128-byte apart slots
        atomicMax(&a[s], (unsigned long long)(blockIdx.x * 7 % 1000003));
        atomicMax(&a[s + 1], (unsigned long long)(blockIdx.x * 13 % 1000003));
    }
}
int main() {
    unsigned long long* a; double* sink;
    cudaMalloc(&a, 64 * 16 * 8); cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int work : {0, 200, 2000})
        for (int spread : {0, 1}) {
            k<<<139776, 256>>>(a, spread, work, sink);
            cudaEventRecord(e0);
            for (int r = 0; r < 5; ++r) k<<<139776, 256>>>(a, spread, work, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("work %4d spread %d: %.3f ms per launch\n", work, spread, ms / 5);
        }
    return 0;
}
