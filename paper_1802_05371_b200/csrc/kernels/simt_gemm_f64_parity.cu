// simt_gemm_f64_parity.cu -- ahead-of-time instantiations of the SIMT family:
// gemm, double, bit-exact parity mode.  See simt.cuh / simt_tiles.cuh.
#include "simt.cuh"
#include "simt_tiles.cuh"

namespace ktune_dev {

#define CASE(A, B, C) \
    if (ms == A && ns == B && ks == C) return reinterpret_cast<const void*>(&simt_kernel<GemmProblem<double>, double, A, B, C, true>);

const void* simt_gemm_f64_parity(int ms, int ns, int ks) {
    if (ms == 0 && ns == 0 && ks == 0)
        return reinterpret_cast<const void*>(&simt_kernel<GemmProblem<double>, double, 0, 0, 0, true>);
    KTUNE_GEMM_TILES(CASE)
    return nullptr;
}

}  // namespace ktune_dev
