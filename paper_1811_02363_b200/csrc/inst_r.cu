// inst_r.cu -- explicit instantiation of the radius-templated filter kernels for one radius.
// Compiled once per radius with -DHDF_R=<R> (the build runs these compilations in parallel).
#include "hdf_dispatch.h"

#ifndef HDF_R
#error "compile with -DHDF_R=<radius>"
#endif

namespace hdf {

template <int R, int RHO, int NPC>
static cudaError_t vp(bool box, const VLaunch& L, cudaStream_t st, const VParams& P) {
    constexpr int J = vpass_j(R);
    constexpr bool PK = vpass_pack(R);
    constexpr int NT = vpass_nt(R);
    void (*kern)(const VParams) =
        box ? k_range_vpass<R, J, true, PK, RHO, NPC, NT> : k_range_vpass<R, J, false, PK, RHO, NPC, NT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    if (e != cudaSuccess) return e;
    kern<<<L.grid, L.threads, L.smem, st>>>(P);
    return cudaGetLastError();
}

// (rho, n + 1) specialisations of the range-weight stage: colour guides (rho 3, n 3) and the PCA-6
// NLM guide (rho 6, n 3); anything else runs the generic loops.
template <int R>
cudaError_t launch_vpass_t(bool box, const VLaunch& L, cudaStream_t st, const VParams& P) {
    if (P.rho == 3 && P.NP == 4) return vp<R, 3, 4>(box, L, st, P);
    if (P.rho == 6 && P.NP == 4) return vp<R, 6, 4>(box, L, st, P);
    if (P.NP == 32) return vp<R, 0, 32>(box, L, st, P);   // 31-band images (config 3): planes per cluster fixed
    return vp<R, 0, 0>(box, L, st, P);
}

template <int R, int MAXJP>
static cudaError_t hp(bool box, const HLaunch& L, cudaStream_t st, const CUtensorMap& tp, const CUtensorMap& tc,
                      const HParams& P) {
    void (*kern)(const CUtensorMap, const CUtensorMap, const HParams) =
        box ? k_hpass_combine<R, MAXJP, true> : k_hpass_combine<R, MAXJP, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    if (e != cudaSuccess) return e;
    kern<<<L.grid, L.threads, L.smem, st>>>(tp, tc, P);
    return cudaGetLastError();
}

template <int R>
cudaError_t launch_hpass_t(bool box, const HLaunch& L, cudaStream_t st, const CUtensorMap& tp, const CUtensorMap& tc,
                           const HParams& P) {
    switch (L.maxjp) {
        case 1: return hp<R, 1>(box, L, st, tp, tc, P);
        case 2: return hp<R, 2>(box, L, st, tp, tc, P);
        default: return hp<R, 4>(box, L, st, tp, tc, P);
    }
}

template cudaError_t launch_vpass_t<HDF_R>(bool, const VLaunch&, cudaStream_t, const VParams&);
template cudaError_t launch_hpass_t<HDF_R>(bool, const HLaunch&, cudaStream_t, const CUtensorMap&, const CUtensorMap&,
                                           const HParams&);

}  // namespace hdf
