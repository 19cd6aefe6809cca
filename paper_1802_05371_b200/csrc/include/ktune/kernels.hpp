#pragma once
// Device entry points of the B200 build: the kernel templates that replace
// the reference's CPU executors execute_gemm<T> / execute_conv<T>
// (/root/reference/proj/include/ktune/backends.hpp:77-100).
//
// All pointers are DEVICE pointers owned by the caller; launches are
// asynchronous on `stream`.  Errors are thrown as the exception classes
// below (the C-ABI maps them to ktune_status codes).

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "ktune/space.hpp"

typedef struct CUstream_st* cudaStream_t;

namespace ktune {

// Dtype or tuple this build cannot execute (reference analogue:
// "cpu backend does not execute f16", backends.cpp:504-506).
struct unsupported_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
// Caller-provided workspace smaller than *_workspace_bytes().
struct workspace_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
// A CUDA runtime/driver call failed.
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace dev {

enum class Mode : int {
    fast = 0,    // FFMA / tensor cores; <= 1e-5 (fp32) of the naive oracle
    parity = 1,  // bit-identical to the reference executors (fp32/fp64 SIMT)
};

// Bytes of workspace a launch needs (0 when k_g splits collapse to one
// slice).  Every split workspace starts with a kSplitCounterBytes region of
// 32-bit arrival counters (one per output tile, SIMT family: the slice that
// arrives last folds all partials in slice order and resets its counter), so
// that region must be ZERO before a workspace's first use; every launch
// leaves it zero.  Partial tiles and the tensor-core family's token flags
// live after it.  One launch at a time per workspace.
constexpr std::size_t kSplitCounterBytes = std::size_t(1) << 20;
std::size_t gemm_workspace_bytes(const GemmInput& in, const GemmTuning& t);
std::size_t conv_workspace_bytes(const ConvInput& in, const ConvTuning& t);

void gemm(const GemmInput& in, const GemmTuning& t, Mode mode, const void* a, const void* b, void* c, void* ws,
          std::size_t ws_bytes, cudaStream_t stream);
void conv(const ConvInput& in, const ConvTuning& t, Mode mode, const void* images, const void* filters,
          void* outputs, void* ws, std::size_t ws_bytes, cudaStream_t stream);

// Kernel-family bookkeeping for measurement / reports.
struct LaunchInfo {
    int threads{0};
    std::size_t smem_bytes{0};
    int grid_x{0}, grid_y{0}, grid_z{0};
    bool generic{false};  // runtime-tile fallback instantiation
    const char* family{""};
};
LaunchInfo gemm_launch_info(const GemmInput& in, const GemmTuning& t, Mode mode);
LaunchInfo conv_launch_info(const ConvInput& in, const ConvTuning& t, Mode mode);

// Write-sweep over a buffer larger than L2 (K8): evicts operands between
// timed repetitions.
void l2_flush(cudaStream_t stream);

// Deterministic device fill with values in [0,1) (seeded; measurement
// operands -- the reference fills on the host, backends.cpp:481-484).
void fill_uniform(void* dst, std::int64_t n, Dtype dtype, std::uint64_t seed, cudaStream_t stream);

void check(int cuda_status, const char* what);

// Launch with programmatic stream serialization (PDL: the kernel's prologue
// overlaps the previous kernel on the stream; its griddepcontrol.wait orders
// the global-memory work) and, if cluster_x > 1, a (cluster_x, 1, 1) cluster.
// KTUNE_PDL=0 disables the attribute.
void launch(const void* kernel, dim3 grid, dim3 block, void** args, std::size_t smem, cudaStream_t stream,
            int cluster_x, const char* what);

}  // namespace dev
}  // namespace ktune
