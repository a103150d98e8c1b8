// Patch and neighbour index tables (host, bit-exact integer work).
//
// Patch order: j = 1..Neta-1 outer, i = i_lo..Nxi-1 inner, i_lo = 0 when xi is
// periodic (GapToothEngine ctor, proj/src/gaptooth.cpp:251-280).
// Neighbours: the 3x3 gather of build_stencil (gaptooth.cpp:74-104) as flat
// macro indices ip*(Neta+1) + j+q, with ip = ((iw+p) % Nxi + Nxi) % Nxi on a
// periodic side, stencil order vals[p+1][q+1], p along xi.
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "patchdyn_b200.h"

namespace pdb200 {
void set_global_error(const std::string& m);
}

extern "C" {

int32_t pd_patch_count(const pd_engine_desc* d) {
    if (!d) return -1;
    if (d->patch_ij) return d->npatches;
    return (d->Nxi - (d->periodic_xi ? 0 : 1)) * (d->Neta - 1);
}

pd_status pd_build_index_tables(const pd_engine_desc* d, int32_t* patch_ij, int32_t* neighbours) {
    if (!d || d->Nxi < 2 || d->Neta < 2) {
        pdb200::set_global_error("coarse grid needs at least 2 intervals per direction");
        return PD_VALIDATION_ERROR;
    }
    const int P = pd_patch_count(d);
    std::vector<int32_t> pij;
    if (d->patch_ij) {
        if (P < 1) {
            pdb200::set_global_error("empty patch table");
            return PD_VALIDATION_ERROR;
        }
        pij.assign(d->patch_ij, d->patch_ij + 2 * static_cast<size_t>(P));
    } else {
        pij.reserve(2 * static_cast<size_t>(P));
        const int i_lo = d->periodic_xi ? 0 : 1;
        for (int j = 1; j <= d->Neta - 1; ++j)
            for (int i = i_lo; i <= d->Nxi - 1; ++i) {
                pij.push_back(i);
                pij.push_back(j);
            }
    }
    const int NF2 = d->Neta + 1;
    for (int q = 0; q < P; ++q) {
        const int i = pij[2 * q], j = pij[2 * q + 1];
        const char* axis = nullptr;
        int bad = 0, hi = 0;
        if (j < 1 || j > d->Neta - 1) axis = "j", bad = j, hi = d->Neta - 1;
        else if (!d->periodic_xi && (i < 1 || i > d->Nxi - 1)) axis = "i", bad = i, hi = d->Nxi - 1;
        if (axis) { // IndexOutOfRange wrapped as MacroPatchError (gaptooth.cpp:76-86, 367-371)
            std::ostringstream m;
            m << "patch (" << i << "," << j << "): stencil center " << axis << "=" << bad << " outside interior [1,"
              << hi << "]";
            pdb200::set_global_error(m.str());
            return PD_MACRO_PATCH_ERROR;
        }
        if (neighbours) {
            const int iw = d->periodic_xi ? ((i % d->Nxi) + d->Nxi) % d->Nxi : i;
            for (int dp = -1; dp <= 1; ++dp) {
                const int ip = d->periodic_xi ? ((iw + dp) % d->Nxi + d->Nxi) % d->Nxi : i + dp;
                for (int dq = -1; dq <= 1; ++dq)
                    neighbours[9 * static_cast<size_t>(q) + 3 * (dp + 1) + (dq + 1)] = ip * NF2 + j + dq;
            }
        }
    }
    if (patch_ij) std::memcpy(patch_ij, pij.data(), pij.size() * sizeof(int32_t));
    return PD_OK;
}

} // extern "C"
