// hdf_dispatch.h -- launchers of the radius-templated filter kernels (instantiated in inst_r*.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "k_hpass.cuh"
#include "k_vpass.cuh"

namespace hdf {

// Radii with compiled kernels.  A Gaussian radius R is run with the smallest compiled R' >= R and
// zero taps beyond R (exact); the box needs an exact match.
constexpr int kRadii[] = {1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 20, 24, 32};
constexpr int kNumRadii = sizeof(kRadii) / sizeof(kRadii[0]);

// J (rows per F1 step) = largest divisor of 2R that is <= 8.
constexpr int vpass_j(int R) {
    int best = 1;
    for (int j = 1; j <= 8; j++)
        if ((2 * R) % j == 0) best = j;
    return best;
}
// F1 threads per CTA from the register window size S = 2R + J.
constexpr int vpass_nt(int R) { return (2 * R + vpass_j(R)) <= 40 ? 1024 : ((2 * R + vpass_j(R)) <= 64 ? 768 : 512); }

struct VLaunch {
    dim3 grid;
    int threads;
    size_t smem;
};
struct HLaunch {
    dim3 grid;
    int threads;
    size_t smem;
    int maxjp;
};

cudaError_t launch_vpass(int R, bool box, const VLaunch& L, cudaStream_t st, const VParams& P);
cudaError_t launch_hpass(int R, bool box, const HLaunch& L, cudaStream_t st, const CUtensorMap& tp,
                         const CUtensorMap& tc, const HParams& P);

}  // namespace hdf
