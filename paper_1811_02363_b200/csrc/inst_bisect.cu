// inst_bisect.cu -- the clustering kernel k_bisect<RHO> (k_bisect.cuh) for one compile-time guide
// dimension, -DHDF_BRHO=<rho> (0 = runtime rho).  One translation unit per RHO, so that the build
// compiles the instantiations in parallel; hdf_api.cu launches them through bisect_kernel_rho<N>().
#include "k_bisect.cuh"

#ifndef HDF_BRHO
#error "compile with -DHDF_BRHO=<rho>"
#endif
#define HDF_CAT2(a, b) a##b
#define HDF_CAT(a, b) HDF_CAT2(a, b)

namespace hdf {
BisectFn HDF_CAT(bisect_kernel_rho, HDF_BRHO)() { return k_bisect<HDF_BRHO>; }
}  // namespace hdf
