// Controlled register-number test of the DFMA operand-read bound (VERDICT r1 "test the bank-conflict
// versus operand-collector hypothesis with controlled register parities").  The kernel is a pure
// DFMA loop: 48 FMAs per iteration, 8 accumulation chains, three distinct register operands each
// (the stencil's weight x neighbour + accumulator shape).  scripts/lab/sass_patch.py rewrites the
// register fields of the loop's DFMAs in the compiled cubin to chosen register numbers (bank
// classes) and clears/sets the reuse flags; bank_host.cpp loads each variant with the driver API
// and times it.  Timing only: the rewritten loop computes garbage.
extern "C" __global__ void __launch_bounds__(32) kb(double* out, const double* win, int iters) {
    double w[48], x[8], y[8];
#pragma unroll
    for (int q = 0; q < 48; ++q) w[q] = win[q] + threadIdx.x * 1e-9; // per-lane (not uniform registers)
#pragma unroll
    for (int q = 0; q < 8; ++q) { x[q] = threadIdx.x * 1e-6 + q; y[q] = win[48 + q] + threadIdx.x * 1e-9; }
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 48; ++r) x[r % 8] = fma(w[r], y[(r + 1) % 8], x[r % 8]);
    }
    double t = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += x[q];
    if (t == 1.2345) out[blockIdx.x] = t;
}
