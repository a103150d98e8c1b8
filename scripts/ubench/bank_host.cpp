// Loads each cubin given on the command line (driver API) and times kernel "kb":
// DP warp-instructions per clock per SM (peak 2 = 64 DFMA lanes/clk/SM) at 8 and 12 warps/SM.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, s); exit(1); } } while (0)
static std::vector<char> slurp(const char* f) {
    FILE* fp = fopen(f, "rb"); if (!fp) { perror(f); exit(1); }
    fseek(fp, 0, SEEK_END); long n = ftell(fp); fseek(fp, 0, SEEK_SET);
    std::vector<char> b(n); if (fread(b.data(), 1, n, fp) != (size_t)n) exit(1); fclose(fp); return b;
}
int main(int argc, char** argv) {
    CK(cuInit(0)); CUdevice dev; CK(cuDeviceGet(&dev, 0)); CUcontext ctx; CK(cuCtxCreate(&ctx, 0, dev));
    int sms = 0, mhz = 0; CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
    CUdeviceptr o, w; CK(cuMemAlloc(&o, 1 << 20)); CK(cuMemAlloc(&w, 64 * 8));
    double hw[64]; for (int q = 0; q < 64; ++q) hw[q] = 1e-3 * (q + 1);
    CK(cuMemcpyHtoD(w, hw, sizeof hw));
    CUevent e0, e1; CK(cuEventCreate(&e0, 0)); CK(cuEventCreate(&e1, 0));
    for (int a = 1; a < argc; ++a) {
        std::vector<char> img = slurp(argv[a]);
        CUmodule m; CK(cuModuleLoadData(&m, img.data())); CUfunction f; CK(cuModuleGetFunction(&f, m, "kb"));
        printf("%-28s", argv[a]);
        for (int wps : {8, 12}) {
            int iters = 20000; void* args[] = {&o, &w, &iters};
            int warm = 10; void* wargs[] = {&o, &w, &warm};
            CK(cuLaunchKernel(f, sms * wps, 1, 1, 32, 1, 1, 0, 0, wargs, 0));
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cuEventRecord(e0, 0));
                CK(cuLaunchKernel(f, sms * wps, 1, 1, 32, 1, 1, 0, 0, args, 0));
                CK(cuEventRecord(e1, 0)); CK(cuEventSynchronize(e1));
                float ms; CK(cuEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
            }
            const double clk = best * 1e-3 * 1.965e9 * sms, ndp = (double)sms * wps * iters * 48;
            printf("  w/SM=%2d %.3f", wps, ndp / clk);
        }
        printf("   DP warp-inst/clk/SM (peak 2)\n");
        CK(cuModuleUnload(m));
    }
    return 0;
}
