// Dev microbenchmarks 3: DFMA latency, ILP needed, and register-operand pressure on B200.
#include <cstdio>
#include <cuda_runtime.h>
// CH independent accumulation chains per lane; NW distinct weight registers (runtime values);
// MODE 0: fma(x, c, c') (constant operands), MODE 1: fma(w[r], y[(r+1)%CH], x[r%CH]) (3 distinct regs)
template <int CH, int MODE>
__global__ void k(double* out, const double* win, int iters) {
    double x[CH], y[CH], w[48];
    for (int q = 0; q < CH; ++q) { x[q] = threadIdx.x * 1e-6 + q; y[q] = 1.0 + q * 1e-3; }
    for (int q = 0; q < 48; ++q) w[q] = win[q];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 48; ++r) {
            if (MODE == 0) x[r % CH] = fma(x[r % CH], 0.999999999, 1e-9);
            else if (MODE == 1) x[r % CH] = fma(w[r], y[(r + 1) % CH], x[r % CH]);
            else if (MODE == 2) x[r % CH] = fma(w[r], y[(r / CH) % CH], x[r % CH]); // B shared by CH consecutive
            else if (MODE == 3) x[r % CH] = fma(w[r], 0.999999999, x[r % CH]);       // 2 register operands
            else x[r % CH] = fma(x[(r + 1) % CH], y[(r + 1) % CH], x[r % CH]);       // 3 regs, A/B not weights
        }
        if (MODE != 0) {
#pragma unroll
            for (int q = 0; q < CH; ++q) y[q] = x[q] * 1e-3; // keep y live and loop-carried
        }
    }
    double t = 0;
    for (int q = 0; q < CH; ++q) t += x[q] + y[q];
    if (t == 1.2345) out[blockIdx.x] = t;
}
template <int CH, int MODE>
void run(int warps_per_sm) {
    double *o, *w;
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&w, 48 * 8);
    double hw[48];
    for (int q = 0; q < 48; ++q) hw[q] = 1e-3 * (q + 1);
    cudaMemcpy(w, hw, sizeof hw, cudaMemcpyHostToDevice);
    int sms = 148, iters = 4000;
    dim3 grid(sms * warps_per_sm), block(32);
    k<CH, MODE><<<grid, block>>>(o, w, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<CH, MODE><<<grid, block>>>(o, w, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n_dp = (double)grid.x * iters * (48 + (MODE != 0 ? CH : 0));
    double clk = ms * 1e-3 * 1.965e9 * sms;
    printf("mode=%d chains=%d w/SM=%2d  DP warp-inst/clk/SM=%.3f (peak 2)  clk/dep-DP(1 warp)=%.1f\n", MODE, CH,
           warps_per_sm, n_dp / clk, warps_per_sm == 1 ? clk / sms / (iters * 48.0 / CH) : 0.0);
    cudaFree(o); cudaFree(w);
}
int main() {
    for (int w : {8, 12}) { run<4, 1>(w); run<8, 1>(w); run<4, 2>(w); run<8, 2>(w); run<4, 3>(w); run<8, 3>(w); run<8, 4>(w); }
    return 0;
}
