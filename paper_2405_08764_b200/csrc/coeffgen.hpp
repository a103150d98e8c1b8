// On-device coefficient-table generator (pd_coeffgen.cu), internal interface.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host/geometry.hpp"
#include "patchdyn_b200.h"

namespace pdb200 {

struct CoeffGenStats {
    double max_abs_ac = 0.0;   // max(|A|, |C|): the explicit stability guard (microsim.cpp:253-262)
    double max_a_plus_c = 0.0; // max(|A| + |C|): the PD_DT_METRIC pin
    double max_abs_b = 0.0;    // max |B| (> 0: mixed term present)
    double device_ms = 0.0;    // generator kernel time (CUDA events)
    size_t nodes = 0;
};

bool coeffgen_supported(int problem);
// (i, j) of the patch each coefficient set is sampled at: [ncoeff_sets][2]
std::vector<int32_t> coeffgen_set_centres(const pd_engine_desc& d, const int32_t* patch_ij, int P);
// Generate [ncoeff_sets][PD_NCOEF][n1][n2] into coeffs_dev (and the separable
// source's spatial table into src_dev), either may be NULL (reduction only).
// Synchronises `stream`.  Throws NonPositiveJacobian / Unsupported / DeviceError.
CoeffGenStats coeffgen_run(const pd_problem_desc& pd, const pd_engine_desc& d, const int32_t* set_ij,
                           double* coeffs_dev, double* src_dev, cudaStream_t stream);

} // namespace pdb200
