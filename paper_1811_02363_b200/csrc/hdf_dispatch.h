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

// F1 (k_range_vpass): packed column pairs (FFMA2 / FADD2 on f32x2) with 512-thread CTAs when the u64
// register window 2R + J stays <= 42 entries (128 registers per thread); for the large radii (24, 32)
// packed pairs with 256-thread CTAs (255 registers: window 2R + J <= 72 entries, J <= 16); any other
// radius one column per thread (float window <= 80).  J = rows per step, a divisor of 2R, <= 16
// (fewer, longer steps amortise the per-step synchronisation).
constexpr int vpass_nt(int R) { return (R == 24 || R == 32) ? 256 : 512; }
constexpr bool vpass_pack(int R) {
    if (vpass_nt(R) == 256) return true;
    for (int j = 16; j >= 1; j--)
        if ((2 * R) % j == 0 && 2 * R + j <= 42) return true;
    return false;
}
constexpr int vpass_j(int R) {
    const int lim = vpass_nt(R) == 256 ? 72 : (vpass_pack(R) ? 42 : 80);
    for (int j = 16; j >= 1; j--)
        if ((2 * R) % j == 0 && 2 * R + j <= lim) return j;
    return 1;
}

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
