#pragma once
// umma.hpp -- K4: the tcgen05/TMEM/TMA tensor-core GEMM family (bf16, f16,
// tf32 inputs; fp32 accumulate; fp32 output).  See umma.cu for the tuple
// mapping.
#include <cstddef>

#include "ktune/kernels.hpp"

namespace ktune {
namespace umma {

std::size_t gemm_workspace_bytes(const GemmInput& in, const GemmTuning& t);
void gemm(const GemmInput& in, const GemmTuning& t, const void* a, const void* b, void* c, void* ws,
          std::size_t ws_bytes, cudaStream_t stream);
dev::LaunchInfo gemm_launch_info(const GemmInput& in, const GemmTuning& t);

// K4c: implicit-GEMM convolution (bf16 / f16), see umma_conv.cu.
std::size_t conv_workspace_bytes(const ConvInput& in, const ConvTuning& t);
void conv(const ConvInput& in, const ConvTuning& t, const void* images, const void* filters, void* outputs, void* ws,
          std::size_t ws_bytes, cudaStream_t stream);
dev::LaunchInfo conv_launch_info(const ConvInput& in, const ConvTuning& t);

}  // namespace umma
}  // namespace ktune
