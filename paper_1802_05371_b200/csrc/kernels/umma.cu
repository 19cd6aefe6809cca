// umma.cu -- placeholder until the tcgen05 family lands.
#include "umma.hpp"

namespace ktune {
namespace umma {

std::size_t gemm_workspace_bytes(const GemmInput&, const GemmTuning&) { return 0; }

void gemm(const GemmInput& in, const GemmTuning&, const void*, const void*, void*, void*, std::size_t, cudaStream_t) {
    throw unsupported_error(std::string("tensor-core family not built for ") + to_string(in.dtype));
}

dev::LaunchInfo gemm_launch_info(const GemmInput& in, const GemmTuning&) {
    throw unsupported_error(std::string("tensor-core family not built for ") + to_string(in.dtype));
}

}  // namespace umma
}  // namespace ktune
