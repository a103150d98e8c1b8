// Dev microbenchmarks: does FP64 FMA issue overlap with SHFL / LDS on B200?
#include <cstdio>
#include <cuda_runtime.h>
template <int NFMA, int NSHFL, int NLDS>
__global__ void k(double* out, int iters) {
    __shared__ double sm[1024];
    const int lane = threadIdx.x & 31;
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x[8];
    for (int q = 0; q < 8; ++q) x[q] = threadIdx.x * 1e-6 + q;
    double s[4] = {1, 2, 3, 4};
    const int src = (lane + 1) & 31;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < NFMA; ++r) x[r % 8] = fma(x[r % 8], 0.999999999, 1e-9);
#pragma unroll
        for (int r = 0; r < NSHFL; ++r) s[r % 4] = __shfl_sync(0xffffffffu, s[r % 4], src) + 0.0f * r; // 32-bit each half
#pragma unroll
        for (int r = 0; r < NLDS; ++r) s[r % 4] += sm[(threadIdx.x + r * 33 + (int)s[0]) & 1023];
    }
    double t = 0;
    for (int q = 0; q < 8; ++q) t += x[q];
    for (int q = 0; q < 4; ++q) t += s[q];
    if (t == 1.2345) out[blockIdx.x] = t;
}
template <int A, int B, int C>
void run(const char* name, int warps_per_sm) {
    double* o;
    cudaMalloc(&o, 1 << 20);
    int sms = 148, iters = 20000;
    dim3 grid(sms * warps_per_sm / 4), block(128);
    k<A, B, C><<<grid, block>>>(o, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<A, B, C><<<grid, block>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_iters = (double)grid.x * 4 * iters;
    double clk = ms * 1e-3 * 1.965e9;
    // per SM per clock
    double dfma = warp_iters * A / sms / clk, shfl = warp_iters * B * 2 / sms / clk, lds = warp_iters * C / sms / clk;
    printf("%-28s warps/SM=%2d  ms=%8.3f  DFMA warp-inst/clk/SM=%.3f (peak 2)  SHFL32 %.3f  LDS64 %.3f\n", name,
           warps_per_sm, ms, dfma, shfl, lds);
    cudaFree(o);
}
int main() {
    for (int w : {8, 12, 16}) {
        run<72, 0, 0>("dfma only", w);
        run<0, 16, 0>("shfl(double) only", w);
        run<72, 16, 0>("72 dfma + 16 dshfl", w);
        run<72, 8, 0>("72 dfma + 8 dshfl", w);
        run<0, 0, 16>("lds64 only", w);
        run<72, 0, 16>("72 dfma + 16 lds64", w);
    }
    return 0;
}
