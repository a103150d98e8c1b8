// Boundary refresh, projective extrapolation for k > 0, and the blow-up guard.
#pragma once

#include "pd_device.cuh"

namespace pdb200::dev {

// refresh_boundary (gaptooth.cpp:296-310) from a perimeter array, or, with
// bnd == nullptr, keep the input field's boundary (copied from F) and apply
// the periodic seam U(Nxi,j) = U(0,j).  Non-patch nodes are exactly the
// boundary rows/columns (+ the seam column when periodic).
__global__ void k_refresh(Params p, double* __restrict__ out, const double* __restrict__ F,
                          const double* __restrict__ bnd, const int* __restrict__ fail_flag) {
    if (fail_flag && *fail_flag) return;
    const int N1 = p.Nxi, N2 = p.Neta, n2 = p.NF2;
    const int rows = 2 * (N1 + 1), cols = 2 * (N2 + 1);
    const double* S = bnd;
    const double* Nn = bnd ? bnd + (N1 + 1) : nullptr;
    const double* W = bnd ? bnd + 2 * (N1 + 1) : nullptr;
    const double* E = bnd ? W + (N2 + 1) : nullptr;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < rows + cols; t += gridDim.x * blockDim.x) {
        if (t < rows) { // S/N rows; corners are owned by the column pass (W/E or seam)
            const int i = t % (N1 + 1), j = t < N1 + 1 ? 0 : N2;
            if (p.periodic ? i == N1 : (i == 0 || i == N1)) continue;
            const size_t node = (size_t)i * n2 + j;
            out[node] = bnd ? (j == 0 ? S[i] : Nn[i]) : F[node];
        } else {
            const int u = t - rows, j = u % (N2 + 1), east = u >= N2 + 1;
            if (p.periodic) {
                if (!east) continue; // column 0 holds patch results (or its boundary rows)
                double v;
                if (j == 0) v = bnd ? S[0] : F[0];
                else if (j == N2) v = bnd ? Nn[0] : F[N2];
                else v = out[j]; // patch (0,j) result, written by the previous kernel
                out[(size_t)N1 * n2 + j] = v;
            } else {
                const size_t node = (size_t)(east ? N1 : 0) * n2 + j;
                out[node] = bnd ? (east ? E[j] : W[j]) : F[node];
            }
        }
    }
}

// out(i,j) = Uk + horizon * (Uk1 - Uk)/tau on patch nodes (cpi.cpp:67-74), k > 0.
__global__ void k_extrapolate(Params p, double* __restrict__ out, const double* __restrict__ Uk,
                              const double* __restrict__ Uk1, const int* __restrict__ pij, double horizon,
                              const int* __restrict__ fail_flag) {
    if (fail_flag && *fail_flag) return;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < p.P; q += gridDim.x * blockDim.x) {
        const size_t node = (size_t)pij[2 * q] * p.NF2 + pij[2 * q + 1];
        const double F = XDIV(XSUB(Uk1[node], Uk[node]), p.tau);
        out[node] = XADD(Uk[node], XMUL(horizon, F));
    }
}

// Blow-up guard of cpi.cpp:187-202 on the device: max |U| as the bit pattern
// of a non-negative double (monotone; NaN/inf compare above every finite
// value), reduced into slot[step]; the last block decides and raises
// fail_flag = step+1 so every later kernel of the run becomes a no-op.
__global__ void k_guard(const double* __restrict__ U, size_t n, unsigned long long* slot, unsigned int* counter,
                        int* fail_flag, int* fail_nonfinite, int step, double blowup) {
    if (*fail_flag) return;
    unsigned long long m = 0;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned long long)__double_as_longlong(fabs(U[t])));
    for (int o = 16; o; o >>= 1) m = max(m, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)m, o));
    __shared__ unsigned long long wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, wm[w]);
        atomicMax(slot + step, m);
        __threadfence();
        const unsigned int prev = atomicAdd(counter + step, 1u);
        if (prev == gridDim.x - 1) {
            const unsigned long long v = atomicAdd(slot + step, 0ull);
            const bool nonfinite = v >= 0x7FF0000000000000ull;
            if (nonfinite || __longlong_as_double((long long)v) > blowup) {
                *fail_nonfinite = nonfinite ? 1 : 0;
                atomicExch(fail_flag, step + 1);
            }
        }
    }
}

} // namespace pdb200::dev
