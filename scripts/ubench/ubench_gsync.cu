// Dev microbenchmark: cost of one grid-wide barrier per iteration on B200, for
// the single-launch run (k_fast_run).  Co-resident grid of 3 CTAs x 128 threads
// per SM (k_fast_run's shape).  Variants:
//   0 cooperative_groups grid.sync()
//   1 hand-rolled: one red.release.gpu.add per CTA on a monotone counter, spin
//     with ld.acquire.gpu until it reaches (iteration+1) * nblocks
//   2 as 1 + a dependent pair of L2 loads (index -> value) after the barrier,
//     a store + atomicMax before it (the per-step traffic of the run)
//   3 as 0 with the same traffic
// usage: ubench_gsync   (prints us per iteration)
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int V>
__global__ void __launch_bounds__(128, 3) k(int iters, unsigned* ctr, const int* idx, double* F, unsigned long long* mx) {
    cg::grid_group grid = cg::this_grid();
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        if (V >= 2) {
            const int j = __ldcg(idx + gt);
            acc += __ldcg(F + j);
            F[gt] = acc * 0.5;
            if ((threadIdx.x & 31) == 0) atomicMax(mx + (gt >> 5) % 32, (unsigned long long)__double_as_longlong(acc));
        }
        if (V == 0 || V == 3) {
            grid.sync();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned target = (unsigned)(it + 1) * gridDim.x;
                red_add_release(ctr, 1u);
                while (ld_acquire(ctr) < target) {
                }
            }
            __syncthreads();
        }
    }
    if (acc == 1.2345) F[0] = acc;
}

template <int V>
void run(int per_sm) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nb = sms * per_sm, nt = nb * 128;
    unsigned* ctr;
    int* idx;
    double* F;
    unsigned long long* mx;
    cudaMalloc(&ctr, 4);
    cudaMalloc(&idx, nt * 4);
    cudaMalloc(&F, nt * 8);
    cudaMalloc(&mx, 32 * 8);
    int* h = new int[nt];
    for (int i = 0; i < nt; ++i) h[i] = (i * 7919) % nt;
    cudaMemcpy(idx, h, nt * 4, cudaMemcpyHostToDevice);
    cudaMemset(F, 0, nt * 8);
    for (int rep = 0; rep < 2; ++rep) {
        const int iters = rep ? 2000 : 10;
        cudaMemset(ctr, 0, 4);
        void* args[] = {(void*)&iters, &ctr, &idx, &F, &mx};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k<V>, dim3(nb), dim3(128), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
        if (rep) printf("variant %d  %d CTAs/SM (%d CTAs): %.3f us per iteration\n", V, per_sm, nb, 1e3 * ms / iters);
    }
    cudaFree(ctr);
    cudaFree(idx);
    cudaFree(F);
    cudaFree(mx);
    delete[] h;
}

int main() {
    for (int per_sm : {1, 2, 3}) {
        run<0>(per_sm);
        run<1>(per_sm);
        run<2>(per_sm);
        run<3>(per_sm);
    }
    return 0;
}
