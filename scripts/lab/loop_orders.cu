// Lab: the FAST 16x16 mixed micro-step loop (2x4 blocks per lane, one warp per
// patch) in alternative instruction orders, for SASS reuse / RF-read analysis.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int BI = 2, BJ = 4, LI = 8, NPL = 8;
enum { WC, WE, WW, WN, WS, WD };
template <int V>
__global__ void __launch_bounds__(32) k_loop(const double* __restrict__ Wt, double* out, int nt) {
    const int lane = threadIdx.x;
    double w[6 * NPL], u[BI][BJ], c[BI][BJ];
    const double* wp = Wt + (size_t)blockIdx.x * 6 * NPL * 32 + lane;
#pragma unroll
    for (int q = 0; q < 6 * NPL; ++q) w[q] = __ldg(wp + q * 32);
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int b = 0; b < BJ; ++b) { u[a][b] = wp[(a * BJ + b) * 32] * 0.5; c[a][b] = wp[(8 + a * BJ + b) * 32] * 1e-3; }
#define WT(k, a, b) w[(k) * NPL + (a) * BJ + (b)]
    for (int step = 0; step < nt; ++step) {
        double hN[BI], hS[BI], cE[BJ + 2], cW[BJ + 2];
#pragma unroll
        for (int a = 0; a < BI; ++a) {
            hN[a] = __shfl_down_sync(0xffffffffu, u[a][0], LI);
            hS[a] = __shfl_up_sync(0xffffffffu, u[a][BJ - 1], LI);
        }
#pragma unroll
        for (int b = 0; b < BJ; ++b) {
            cE[b + 1] = __shfl_down_sync(0xffffffffu, u[0][b], 1);
            cW[b + 1] = __shfl_up_sync(0xffffffffu, u[BI - 1][b], 1);
        }
        cE[0] = cE[BJ + 1] = cW[0] = cW[BJ + 1] = 0.0;
        auto at = [&](int a, int b) -> double {
            if (a == BI) return cE[b + 1];
            if (a == -1) return cW[b + 1];
            if (b == BJ) return hN[a];
            if (b == -1) return hS[a];
            return u[a][b];
        };
        double nu[BI][BJ], e[BI][BJ];
#pragma unroll
        for (int a = 0; a < BI; ++a)
#pragma unroll
            for (int b = 0; b < BJ; ++b) e[a][b] = at(a + 1, b) - at(a - 1, b);
        double eN[BI], eS[BI];
#pragma unroll
        for (int a = 0; a < BI; ++a) {
            eN[a] = __shfl_down_sync(0xffffffffu, e[a][0], LI);
            eS[a] = __shfl_up_sync(0xffffffffu, e[a][BJ - 1], LI);
        }
        if (V == 0) { // production: term-major gather
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = fma(WT(WC, a, b), u[a][b], c[a][b]);
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = fma(WT(WN, a, b), at(a, b + 1), nu[a][b]);
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = fma(WT(WS, a, b), at(a, b - 1), nu[a][b]);
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = fma(WT(WE, a, b), at(a + 1, b), nu[a][b]);
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = fma(WT(WW, a, b), at(a - 1, b), nu[a][b]);
        } else if (V == 1) { // source-major scatter: each source value feeds its targets consecutively
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = c[a][b];
#pragma unroll
            for (int a = -1; a <= BI; ++a)
#pragma unroll
                for (int b = -1; b <= BJ; ++b) {
                    if ((a == -1 || a == BI) && (b == -1 || b == BJ)) continue;
                    const double s = at(a, b);
                    if (a >= 0 && a < BI && b >= 0 && b < BJ) nu[a][b] = fma(WT(WC, a, b), s, nu[a][b]);
                    if (a >= 0 && a < BI && b - 1 >= 0 && b - 1 < BJ) nu[a][b - 1] = fma(WT(WN, a, b - 1), s, nu[a][b - 1]);
                    if (a >= 0 && a < BI && b + 1 >= 0 && b + 1 < BJ) nu[a][b + 1] = fma(WT(WS, a, b + 1), s, nu[a][b + 1]);
                    if (b >= 0 && b < BJ && a - 1 >= 0 && a - 1 < BI) nu[a - 1][b] = fma(WT(WE, a - 1, b), s, nu[a - 1][b]);
                    if (b >= 0 && b < BJ && a + 1 >= 0 && a + 1 < BI) nu[a + 1][b] = fma(WT(WW, a + 1, b), s, nu[a + 1][b]);
                }
        } else if (V == 2) { // node-major gather chains (one node's 5 FMAs in a row)
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) {
                    double t = fma(WT(WC, a, b), u[a][b], c[a][b]);
                    t = fma(WT(WN, a, b), at(a, b + 1), t);
                    t = fma(WT(WS, a, b), at(a, b - 1), t);
                    t = fma(WT(WE, a, b), at(a + 1, b), t);
                    nu[a][b] = fma(WT(WW, a, b), at(a - 1, b), t);
                }
        } else if (V == 3 || V == 4) { // scatter, fenced source groups
#pragma unroll
            for (int a = 0; a < BI; ++a)
#pragma unroll
                for (int b = 0; b < BJ; ++b) nu[a][b] = c[a][b];
#pragma unroll
            for (int a = -1; a <= BI; ++a)
#pragma unroll
                for (int b = -1; b <= BJ; ++b) {
                    if ((a == -1 || a == BI) && (b == -1 || b == BJ)) continue;
                    const double s = at(a, b);
                    if (a >= 0 && a < BI && b >= 0 && b < BJ) nu[a][b] = fma(WT(WC, a, b), s, nu[a][b]);
                    if (a >= 0 && a < BI && b - 1 >= 0 && b - 1 < BJ) nu[a][b - 1] = fma(WT(WN, a, b - 1), s, nu[a][b - 1]);
                    if (a >= 0 && a < BI && b + 1 >= 0 && b + 1 < BJ) nu[a][b + 1] = fma(WT(WS, a, b + 1), s, nu[a][b + 1]);
                    if (b >= 0 && b < BJ && a - 1 >= 0 && a - 1 < BI) nu[a - 1][b] = fma(WT(WE, a - 1, b), s, nu[a - 1][b]);
                    if (b >= 0 && b < BJ && a + 1 >= 0 && a + 1 < BI) nu[a + 1][b] = fma(WT(WW, a + 1, b), s, nu[a + 1][b]);
                    if (V == 3) __syncwarp();
                    else asm volatile("" ::: "memory");
                }
        }
#pragma unroll
        for (int a = 0; a < BI; ++a)
#pragma unroll
            for (int b = 0; b < BJ; ++b) {
                const double up = b + 1 < BJ ? e[a][b + 1] : eN[a];
                const double dn = b > 0 ? e[a][b - 1] : eS[a];
                nu[a][b] = fma(WT(WD, a, b), up - dn, nu[a][b]);
            }
#pragma unroll
        for (int a = 0; a < BI; ++a)
#pragma unroll
            for (int b = 0; b < BJ; ++b) u[a][b] = nu[a][b];
    }
    double s = 0;
#pragma unroll
    for (int a = 0; a < BI; ++a)
#pragma unroll
        for (int b = 0; b < BJ; ++b) s += u[a][b];
    out[blockIdx.x * 32 + lane] = s;
}
template __global__ void k_loop<0>(const double*, double*, int);
template __global__ void k_loop<1>(const double*, double*, int);
template __global__ void k_loop<2>(const double*, double*, int);
template __global__ void k_loop<3>(const double*, double*, int);
template __global__ void k_loop<4>(const double*, double*, int);
