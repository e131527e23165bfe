// inst_coeffs.cu -- the tensor-core coefficient kernels k_coeffs_mma<NT, RHO> (k_coeffs.cuh) for one
// NT (-DHDF_CNT=<nt>: K <= 8 NT), all RHO specialisations.  One translation unit per NT (parallel build).
#define HDF_COEFFS_MMA_ONLY
#include "k_coeffs.cuh"

#ifndef HDF_CNT
#error "compile with -DHDF_CNT=<nt>"
#endif
#define HDF_CAT2(a, b) a##b
#define HDF_CAT(a, b) HDF_CAT2(a, b)

namespace hdf {
CoefFn HDF_CAT(coeffs_mma_kernel_nt, HDF_CNT)(int rho) {
    if (rho == 3) return k_coeffs_mma<HDF_CNT, 3>;
    if (rho == 6) return k_coeffs_mma<HDF_CNT, 6>;
    return k_coeffs_mma<HDF_CNT, 0>;
}
}  // namespace hdf
