// Boundary refresh, projective extrapolation for k > 0, and the blow-up guard.
#pragma once

#include "pd_device.cuh"

namespace pdb200::dev {

// refresh_boundary (gaptooth.cpp:296-310) from a perimeter array, or, with
// bnd == nullptr, keep the input field's boundary (copied from F) and apply
// the periodic seam U(Nxi,j) = U(0,j).  Non-patch nodes are exactly the
// boundary rows/columns (+ the seam column when periodic).  One perimeter
// entry t; returns |value written| (0 when the entry writes nothing).
// seam_by_patches: the fused run's column-0 patches write the seam interior.
// max of a 64-bit unsigned over the warp with two 32-bit redux.sync (REDUX):
// the high words first, then the low words among the lanes holding that maximum
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned)v : 0u);
    return ((unsigned long long)mhi << 32) | mlo;
}

// Generic form: get(k) returns entry k of the perimeter row (S row, N row, W
// column, E column, as refresh_one's bnd layout); has_bnd false keeps F's values.
template <class Get>
__device__ __forceinline__ double refresh_gen(const Params& p, double* __restrict__ out, const double* __restrict__ F,
                                              bool has_bnd, Get get, int t, bool seam_by_patches) {
    const int N1 = p.Nxi, N2 = p.Neta, n2 = p.NF2;
    const int rows = 2 * (N1 + 1);
    if (t < rows) { // S/N rows; corners are owned by the column pass (W/E or seam)
        const int i = t % (N1 + 1), j = t < N1 + 1 ? 0 : N2;
        if (p.periodic ? i == N1 : (i == 0 || i == N1)) return 0.0;
        const size_t node = (size_t)i * n2 + j;
        const double v = has_bnd ? (j == 0 ? get(i) : get(N1 + 1 + i)) : F[node];
        out[node] = v;
        return fabs(v);
    }
    const int u = t - rows, j = u % (N2 + 1), east = u >= N2 + 1;
    const int W0 = 2 * (N1 + 1), E0 = W0 + N2 + 1;
    if (p.periodic) {
        if (!east) return 0.0; // column 0 holds patch results (or its boundary rows)
        double v;
        if (j == 0) v = has_bnd ? get(0) : F[0];
        else if (j == N2) v = has_bnd ? get(N1 + 1) : F[N2];
        else if (seam_by_patches) return 0.0;
        else v = out[j]; // patch (0,j) result, written before the refresh
        out[(size_t)N1 * n2 + j] = v;
        return fabs(v);
    }
    const size_t node = (size_t)(east ? N1 : 0) * n2 + j;
    const double v = has_bnd ? get(east ? E0 + j : W0 + j) : F[node];
    out[node] = v;
    return fabs(v);
}
__device__ __forceinline__ double refresh_one(const Params& p, double* __restrict__ out, const double* __restrict__ F,
                                              const double* __restrict__ bnd, int t, bool seam_by_patches) {
    return refresh_gen(p, out, F, bnd != nullptr, [&](int k) { return bnd[k]; }, t, seam_by_patches);
}

__device__ __forceinline__ void refresh_range(const Params& p, double* __restrict__ out, const double* __restrict__ F,
                                              const double* __restrict__ bnd, int t0, int stride) {
    const int n = 2 * (p.Nxi + 1) + 2 * (p.Neta + 1);
    for (int t = t0; t < n; t += stride) refresh_one(p, out, F, bnd, t, false);
}

__global__ void k_refresh(Params p, double* __restrict__ out, const double* __restrict__ F,
                          const double* __restrict__ bnd, const int* __restrict__ fail_flag) {
    if (fail_flag && *fail_flag) return;
    refresh_range(p, out, F, bnd, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// out(i,j) = Uk + horizon * (Uk1 - Uk)/tau on patch nodes (cpi.cpp:67-74), k > 0.
__global__ void k_extrapolate(Params p, double* __restrict__ out, const double* __restrict__ Uk,
                              const double* __restrict__ Uk1, const int* __restrict__ pij, double horizon,
                              const int* __restrict__ fail_flag) {
    if (fail_flag && *fail_flag) return;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < p.P; q += gridDim.x * blockDim.x) {
        const size_t node = (size_t)pij[2 * q] * p.NF2 + pij[2 * q + 1];
        const double F = XDIV(XSUB(Uk1[node], Uk[node]), p.tau);
        const double v = XADD(Uk[node], XMUL(horizon, F));
        out[node] = v;
        halo_store(p, node, v); // decomposed run with k > 0 (pd_extrapolate_halo)
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
    m = warp_max_u64(m);
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

// refresh_boundary (gaptooth.cpp:296-310) and the blow-up guard (cpi.cpp:187-202) of one
// macro step in ONE launch (the multi-launch run loop, k = 0): every thread refreshes its share
// of the perimeter and keeps what it wrote, then scans the nodes the refresh does not own (the
// patch nodes, written by the step kernel before this launch); together that is max |U| over the
// refreshed field, the same slot value and decision as k_refresh followed by k_guard.
__global__ void k_refresh_guard(Params p, double* __restrict__ out, const double* __restrict__ F,
                                const double* __restrict__ bnd, unsigned long long* slot, unsigned int* counter,
                                int* fail_flag, int* fail_nonfinite, int step, double blowup) {
    if (*fail_flag) return;
    const int stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
    const int nperim = 2 * (p.Nxi + 1) + 2 * (p.Neta + 1);
    unsigned long long m = 0;
    for (int t = t0; t < nperim; t += stride)
        m = max(m, (unsigned long long)__double_as_longlong(refresh_one(p, out, F, bnd, t, false)));
    // nodes outside the refresh: columns i_lo .. Nxi-1, rows 1 .. Neta-1 (column 0 holds patch
    // results when xi is periodic)
    const int i_lo = p.periodic ? 0 : 1, ni = p.Nxi - i_lo, nj = p.Neta - 1;
    const size_t n = (size_t)ni * nj;
    for (size_t t = t0; t < n; t += stride) {
        const size_t node = (size_t)(i_lo + (int)(t / nj)) * p.NF2 + 1 + (int)(t % nj);
        m = max(m, (unsigned long long)__double_as_longlong(fabs(out[node])));
    }
    m = warp_max_u64(m);
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

// ---- cpi::run's per-step exact-error metric (max_percent_error, cpi.cpp:79-94) ----
// max over the patch nodes i in [i_lo, Nxi-1], j in [1, Neta-1] (i_lo = 0 when
// periodic) with |exact| >= 1e-12 of |U - exact| / |exact| * 100, in the
// reference's operation order (no contraction: subtract, abs, divide, scale),
// reduced as the bit pattern of a non-negative double into err[step] (zeroed
// by the caller; 0 when no node qualifies, like the reference's `worst`).
// A tripped guard (fail_flag) makes it a no-op: cpi::run throws before it.
__global__ void k_exact_err(Params p, const double* __restrict__ U, const double* __restrict__ ex,
                            unsigned long long* err, const int* __restrict__ fail_flag, int step) {
    if (*fail_flag) return;
    const int i_lo = p.periodic ? 0 : 1;
    const int ni = p.Nxi - i_lo, nj = p.Neta - 1;
    const size_t n = (size_t)ni * nj;
    unsigned long long m = 0;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
        const size_t node = (size_t)(i_lo + (int)(t / nj)) * p.NF2 + 1 + (int)(t % nj);
        const double e = ex[node];
        if (fabs(e) < 1e-12) continue;
        const double pct = __dmul_rn(__ddiv_rn(fabs(__dsub_rn(U[node], e)), fabs(e)), 100.0);
        m = max(m, (unsigned long long)__double_as_longlong(pct));
    }
    m = warp_max_u64(m);
    __shared__ unsigned long long wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, wm[w]);
        if (m) atomicMax(err + step, m);
    }
}

// ---- whole linear-response run in one CTA (fields resident in shared memory) ----
// pd_run_device with PD_STEP_LINEAR when the macro field fits in shared memory:
// every macro step (k+1 linear substeps, the projective extrapolation, the
// boundary refresh and the blow-up guard, cpi.cpp:58-77, 175-202) runs inside
// one kernel with block barriers instead of four launches per step.  Same
// arithmetic, in the same order, as k_linear_step / k_extrapolate / k_refresh /
// k_guard, so results and statistics are identical to the multi-launch loop.
// Shared layout: A (macro field), B0/B1 (substep ping-pong; B1 only for k > 0).
__global__ void __launch_bounds__(1024)
k_linear_run_block(Params p, double* __restrict__ U, const int* __restrict__ pij, const double* __restrict__ row_w,
                   const double* __restrict__ bnd, size_t perim, int nsteps, double blowup,
                   unsigned long long* __restrict__ slot, int* __restrict__ fail, int full_field) {
    extern __shared__ double sfld[];
    __shared__ unsigned long long wm[32];
    __shared__ int s_stop;
    const size_t NF = (size_t)(p.Nxi + 1) * p.NF2;
    double* A = sfld;
    auto B = [&](int b) { return sfld + NF * (size_t)(1 + b); };
    const int tid = threadIdx.x, nth = blockDim.x;
    for (size_t q = tid; q < NF; q += nth) A[q] = U[q];
    double* const s_roww = sfld + NF * (size_t)(p.k == 0 ? 2 : 3); // [Neta+1][9], read every step
    for (int q = tid; q < (p.Neta + 1) * 9; q += nth) s_roww[q] = row_w[q];
    if (tid == 0) s_stop = 0;
    __syncthreads();
    const int k = p.k;
    if (k == 0 && full_field) { // every BASELINE config: one block barrier per macro step
        // The substep, the extrapolation and the boundary refresh of step n only
        // read the field of step n-1 (cur) and write the other buffer (nxt): each
        // thread extrapolates its own patches right after their linear step (the
        // column-0 patches also write the periodic seam), boundary threads refresh
        // the perimeter of nxt from the table (or keep cur's values), and every
        // written node enters the thread's max |U| — all nodes of the field are
        // written, so it is the guard's max over the field.  One barrier, then
        // every warp reduces the per-warp maxima (double-buffered by step parity)
        // and takes the same guard decision.  Same operations on the same values
        // as the phased loop below: bit-identical results and statistics.
        __shared__ unsigned long long wm2[2][32];
        const int lane = tid & 31, nw = nth >> 5;
        const int nperim = 2 * (p.Nxi + 1) + 2 * (p.Neta + 1);
        double* cur = A;
        double* nxt = B(0);
        // perimeter entries go to the threads after the patches' (when there are
        // spare threads), so a step's critical path is one of the two, not both
        const int t_off = p.P % nth;
        // the first patch's indices stay in registers for the whole run
        const int i0 = tid < p.P ? pij[2 * tid] : 0, j0 = tid < p.P ? pij[2 * tid + 1] : 0;
        for (int n = 0; n < nsteps; ++n) {
            const double* bn = bnd ? bnd + perim * 2 * (size_t)n : nullptr;
            unsigned long long mx = 0;
            for (int q = tid; q < p.P; q += nth) {
                const int i = q == tid ? i0 : pij[2 * q], j = q == tid ? j0 : pij[2 * q + 1];
                const double* w = s_roww + 9 * j;
                double acc = 0.0;
#pragma unroll
                for (int dp = -1; dp <= 1; ++dp) {
                    int ip = i + dp;
                    if (p.periodic) ip = ((ip % p.Nxi) + p.Nxi) % p.Nxi;
#pragma unroll
                    for (int dq = -1; dq <= 1; ++dq)
                        acc = XADD(acc, XMUL(w[3 * (dp + 1) + dq + 1], cur[(size_t)ip * p.NF2 + j + dq]));
                }
                const size_t node = (size_t)i * p.NF2 + j;
                const double u = cur[node];
                const double v = XADD(u, XMUL(p.dt_macro, XDIV(XSUB(acc, u), p.tau))); // cpi.cpp:54, 74
                nxt[node] = v;
                if (p.periodic && i == 0) nxt[(size_t)p.Nxi * p.NF2 + j] = v; // seam U(Nxi,j) = U(0,j)
                mx = max(mx, (unsigned long long)__double_as_longlong(fabs(v)));
            }
            for (int t = (tid - t_off + nth) % nth; t < nperim; t += nth)
                mx = max(mx, (unsigned long long)__double_as_longlong(refresh_one(p, nxt, cur, bn ? bn + perim : nullptr, t, true)));
            mx = warp_max_u64(mx);
            if (lane == 0) wm2[n & 1][tid >> 5] = mx;
            __syncthreads();
            mx = warp_max_u64(lane < nw ? wm2[n & 1][lane] : 0ull);
            const bool nonfinite = mx >= 0x7FF0000000000000ull;
            const bool trip = nonfinite || __longlong_as_double((long long)mx) > blowup;
            if (tid == 0) {
                slot[n] = mx;
                if (trip) {
                    fail[0] = n + 1;
                    fail[1] = nonfinite ? 1 : 0;
                }
            }
            double* t = cur;
            cur = nxt;
            nxt = t;
            if (trip) break; // the field after the failing step, as the phased loop leaves it
        }
        for (size_t q = tid; q < NF; q += nth) U[q] = cur[q];
        return;
    }
    const double horizon = XSUB(p.dt_macro, XMUL((double)k, p.tau)); // as projective_dev computes it
    for (int n = 0; n < nsteps; ++n) {
        const double* bn = bnd ? bnd + perim * (size_t)(k + 2) * n : nullptr;
        const double* src = A;
        for (int m = 0; m <= k; ++m) {
            double* dst = B(m & 1);
            for (int q = tid; q < p.P; q += nth) {
                const int i = pij[2 * q], j = pij[2 * q + 1];
                const double* w = s_roww + 9 * j;
                double acc = 0.0;
#pragma unroll
                for (int dp = -1; dp <= 1; ++dp) {
                    int ip = i + dp;
                    if (p.periodic) ip = ((ip % p.Nxi) + p.Nxi) % p.Nxi;
#pragma unroll
                    for (int dq = -1; dq <= 1; ++dq)
                        acc = XADD(acc, XMUL(w[3 * (dp + 1) + dq + 1], src[(size_t)ip * p.NF2 + j + dq]));
                }
                dst[(size_t)i * p.NF2 + j] = acc;
            }
            __syncthreads();
            if (k > 0) { // the substep field is read by the next substep: refresh its boundary
                refresh_range(p, dst, src, bn ? bn + perim * m : nullptr, tid, nth);
                __syncthreads();
            }
            src = dst;
        }
        // projective extrapolation on patch nodes, in place in A (cpi.cpp:67-74)
        const double* Uk = k == 0 ? A : B((k - 1) & 1);
        const double* Uk1 = B(k & 1);
        for (int q = tid; q < p.P; q += nth) {
            const size_t node = (size_t)pij[2 * q] * p.NF2 + pij[2 * q + 1];
            if (k == 0)
                A[node] = XADD(A[node], XMUL(p.dt_macro, XDIV(XSUB(Uk1[node], A[node]), p.tau)));
            else
                A[node] = XADD(Uk[node], XMUL(horizon, XDIV(XSUB(Uk1[node], Uk[node]), p.tau)));
        }
        __syncthreads();
        refresh_range(p, A, A, bn ? bn + perim * (size_t)(k + 1) : nullptr, tid, nth);
        __syncthreads();
        // blow-up guard (cpi.cpp:187-202), max |U| as a non-negative bit pattern
        unsigned long long mx = 0;
        for (size_t q = tid; q < NF; q += nth) mx = max(mx, (unsigned long long)__double_as_longlong(fabs(A[q])));
        mx = warp_max_u64(mx);
        if ((tid & 31) == 0) wm[tid >> 5] = mx;
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < (nth >> 5); ++w) mx = max(mx, wm[w]);
            slot[n] = mx;
            const bool nonfinite = mx >= 0x7FF0000000000000ull;
            if (nonfinite || __longlong_as_double((long long)mx) > blowup) {
                fail[0] = n + 1;
                fail[1] = nonfinite ? 1 : 0;
                s_stop = 1;
            }
        }
        __syncthreads();
        if (s_stop) break;
    }
    for (size_t q = tid; q < NF; q += nth) U[q] = A[q];
}

} // namespace pdb200::dev
