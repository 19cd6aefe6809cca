// simt_conv_f64_fast.cu -- ahead-of-time instantiations of the SIMT family:
// conv, double, FFMA fast mode.  See simt.cuh / simt_tiles.cuh.
#include "simt.cuh"
#include "simt_tiles.cuh"

namespace ktune_dev {

#define CASE(A, B, C) \
    if (ms == A && ns == B && ks == C) return reinterpret_cast<const void*>(&simt_kernel<ConvProblem<double>, double, A, B, C, false>);

const void* simt_conv_f64_fast(int ms, int ns, int ks) {
    if (ms == 0 && ns == 0 && ks == 0)
        return reinterpret_cast<const void*>(&simt_kernel<ConvProblem<double>, double, 0, 0, 0, false>);
    KTUNE_CONV_TILES(CASE)
    return nullptr;
}

}  // namespace ktune_dev
