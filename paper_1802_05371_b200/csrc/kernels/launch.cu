// launch.cu -- host-side dispatch of the SIMT family (K1/K2/K3) and the
// measurement helper kernels (K8 L2 flush, seeded device fill).
//
// Replaces the loop-nest drivers of execute_gemm / execute_conv
// (backends.cpp:228-444): validates like the reference (divisibility +
// operand shapes are the executor's checks, backends.cpp:231-240; resource
// legality is the measurement backend's, backends.cpp:503), derives the launch
// geometry from the tuple and picks the ahead-of-time instantiation.

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <random>
#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

#include "ktune/kernels.hpp"
#include "simt.cuh"
#include "simt_tiles.cuh"
#include "umma.hpp"

namespace ktune {
namespace dev {

void check(int status, const char* what) {
    if (status != cudaSuccess)
        throw cuda_error(std::string(what) + ": " + cudaGetErrorString(static_cast<cudaError_t>(status)));
}

namespace {

std::int64_t ceil_div(std::int64_t a, std::int64_t b) { return (a + b - 1) / b; }

void require_divisible(int big, int small, const char* what) {
    if (big % small != 0) throw std::invalid_argument(std::string("execute: ") + what);
}

int device_smem_optin() {
    static int value = [] {
        int dev = 0, v = 0;
        check(cudaGetDevice(&dev), "cudaGetDevice");
        check(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem attribute");
        return v;
    }();
    return value;
}

// Geometry shared by GEMM and CONV once mapped onto rows x cols x red.
struct Plan {
    ktune_dev::SimtParams p{};
    int threads{0};
    std::size_t smem{0};
    dim3 grid;
    int col_tiles{0}, row_tiles{0};
    int ms{0}, ns{0}, ks{0};  // register tile used for the lookup (0 = generic)
    bool generic{false};
    std::size_t ws_bytes{0};
    std::size_t counter_bytes{0};
};

// rows/red/out: problem extents; ml,nl,ms,ns,ks,kl,kg,u: mapped tuple.
Plan plan_simt(std::int64_t rows, std::int64_t red, std::int64_t out_elems, std::int64_t col_tiles, int ml, int nl,
               int ms, int ns, int ks, int kl, int kg, int u, int esize, bool a_rc, bool b_rc) {
    Plan pl;
    auto& p = pl.p;
    p.rows = rows;
    p.red = red;
    p.out_elems = out_elems;
    p.ml = ml;
    p.nl = nl;
    p.ms = ms;
    p.ns = ns;
    p.ks = ks;
    p.kl = kl;
    p.tm = ml / ms;
    p.tn = nl / ns;
    p.w = std::max(u / kl, ks);
    p.pad_a = a_rc ? 1 : 0;
    p.pad_b = b_rc ? 1 : 0;
    p.kg_span = ceil_div(red, kg);
    p.nz = int(ceil_div(red, p.kg_span));
    pl.threads = p.tm * p.tn * kl;
    if (pl.threads > 1024)
        throw unsupported_error("tuning needs " + std::to_string(pl.threads) + " threads per block; the device allows 1024");
    if (col_tiles > 0x7fffffff) throw unsupported_error("too many column tiles for one launch");
    pl.col_tiles = int(col_tiles);
    pl.row_tiles = int(ceil_div(rows, ml));
    if (pl.row_tiles > 65535 || p.nz > 65535) throw unsupported_error("grid too large for one launch");
    pl.grid = dim3(unsigned(pl.col_tiles), unsigned(pl.row_tiles), unsigned(p.nz));
    const std::size_t stage =
        std::size_t(2) * kl * p.w * std::size_t((ml + p.pad_a) + (nl + p.pad_b)) * std::size_t(esize);
    const std::size_t red_tile = std::size_t(ml) * nl * std::size_t(esize);
    pl.smem = std::size_t(2) * nl * sizeof(std::int64_t) + std::max(stage, red_tile);
    if (pl.smem > std::size_t(device_smem_optin()))
        throw unsupported_error("tuning needs " + std::to_string(pl.smem) + " bytes of shared memory; the device allows " +
                                std::to_string(device_smem_optin()));
    const bool in_envelope = ktune_dev::simt_thread_cap(ms, ns, ks) >= pl.threads;
    pl.generic = !in_envelope;
    pl.ms = ms;
    pl.ns = ns;
    pl.ks = ks;
    if (p.nz > 1) {
        pl.counter_bytes =
            (std::size_t(pl.col_tiles) * pl.row_tiles * std::size_t(p.nz - 1) * sizeof(unsigned long long) + 255) /
            256 * 256;
        pl.ws_bytes = pl.counter_bytes + std::size_t(p.nz - 1) * std::size_t(out_elems) * std::size_t(esize);
    }
    return pl;
}

const void* pick(bool conv, Dtype dt, Mode mode, Plan& pl) {
    using namespace ktune_dev;
    const bool par = (mode == Mode::parity);
    const void* (*fn)(int, int, int) = nullptr;
    if (!conv) {
        if (dt == Dtype::f32) fn = par ? &simt_gemm_f32_parity : &simt_gemm_f32_fast;
        else fn = par ? &simt_gemm_f64_parity : &simt_gemm_f64_fast;
    } else {
        if (dt == Dtype::f32) fn = par ? &simt_conv_f32_parity : &simt_conv_f32_fast;
        else fn = par ? &simt_conv_f64_parity : &simt_conv_f64_fast;
    }
    const void* k = pl.generic ? nullptr : fn(pl.ms, pl.ns, pl.ks);
    if (k == nullptr) {
        if (pl.ms * pl.ns * pl.ks > kGenericMaxAcc)
            throw unsupported_error("register tile of " + std::to_string(pl.ms * pl.ns * pl.ks) +
                                    " accumulators exceeds the generic kernel's " + std::to_string(kGenericMaxAcc));
        pl.generic = true;
        k = fn(0, 0, 0);
    }
    return k;
}

void prepare(const void* kernel, std::size_t smem) {
    static std::mutex mu;
    static std::unordered_map<const void*, std::size_t> configured;
    std::lock_guard<std::mutex> lock(mu);
    auto it = configured.find(kernel);
    if (it != configured.end() && it->second >= smem) return;
    check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max<std::size_t>(smem, 48 * 1024))),
          "cudaFuncSetAttribute(smem)");
    configured[kernel] = std::max<std::size_t>(smem, 48 * 1024);
}

// Launch tokens: a process-random salt mixed with a counter (never 0).
unsigned long long next_token() {
    static std::atomic<unsigned long long> counter{0};
    static const unsigned long long salt = [] {
        std::random_device rd;
        return (static_cast<unsigned long long>(rd()) << 32) ^ rd() ^
               static_cast<unsigned long long>(std::chrono::steady_clock::now().time_since_epoch().count());
    }();
    unsigned long long x = salt + 0x9e3779b97f4a7c15ULL * (counter.fetch_add(1) + 1);
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x == 0 ? 1 : x;
}

void bind_workspace(Plan& pl, void* ws, std::size_t ws_bytes) {
    if (pl.p.nz <= 1) return;
    if (ws == nullptr || ws_bytes < pl.ws_bytes)
        throw workspace_error("workspace of " + std::to_string(ws_bytes) + " bytes is smaller than the " +
                              std::to_string(pl.ws_bytes) + " bytes this tuning needs");
    pl.p.flags = static_cast<unsigned long long*>(ws);
    pl.p.ws = static_cast<unsigned char*>(ws) + pl.counter_bytes;
    pl.p.token = next_token();
}

Plan gemm_plan(const GemmInput& in, const GemmTuning& t) {
    in.validate();
    t.validate();
    require_divisible(t.m_l, t.m_s, "m_l not divisible by m_s");
    require_divisible(t.n_l, t.n_s, "n_l not divisible by n_s");
    require_divisible(t.u, t.k_s, "u not divisible by k_s");
    if (in.dtype != Dtype::f32 && in.dtype != Dtype::f64)
        throw unsupported_error(std::string("simt family does not execute ") + to_string(in.dtype));
    return plan_simt(in.m, in.k, in.m * in.n, ceil_div(in.n, t.n_l), t.m_l, t.n_l, t.m_s, t.n_s, t.k_s, t.k_l, t.k_g,
                     t.u, dtype_size_bytes(in.dtype), !in.trans_a, in.trans_b);
}

Plan conv_plan(const ConvInput& in, const ConvTuning& t) {
    in.validate();
    t.validate();
    require_divisible(t.k_l, t.k_s, "k_l not divisible by k_s");
    require_divisible(t.p_l, t.p_s, "p_l not divisible by p_s");
    require_divisible(t.q_l, t.q_s, "q_l not divisible by q_s");
    require_divisible(t.n_l, t.n_s, "n_l not divisible by n_s");
    require_divisible(t.u, t.c_s, "u not divisible by c_s");
    if (in.dtype != Dtype::f32 && in.dtype != Dtype::f64)
        throw unsupported_error(std::string("simt family does not execute ") + to_string(in.dtype));
    const std::int64_t col_tiles = ceil_div(in.p, t.p_l) * ceil_div(in.q, t.q_l) * ceil_div(in.n_batch, t.n_l);
    return plan_simt(in.k_filters, in.c * in.r * in.s, in.k_filters * in.p * in.q * in.n_batch, col_tiles, t.k_l,
                     t.p_l * t.q_l * t.n_l, t.k_s, t.p_s * t.q_s * t.n_s, t.c_s, t.c_l, t.c_g, t.u,
                     dtype_size_bytes(in.dtype), false, false);
}

template <typename T>
void launch_gemm_t(const GemmInput& in, Plan& pl, Mode mode, const void* a, const void* b, void* c, cudaStream_t s) {
    ktune_dev::GemmProblem<T> prob{static_cast<const T*>(a), static_cast<const T*>(b), in.m, in.n, in.k,
                                   in.trans_a ? 1 : 0, in.trans_b ? 1 : 0, pl.p.nl};
    pl.p.out = c;
    const void* k = pick(false, in.dtype, mode, pl);
    prepare(k, pl.smem);
    void* args[] = {&prob, &pl.p};
    check(cudaLaunchKernel(k, pl.grid, dim3(unsigned(pl.threads)), args, pl.smem, s), "gemm launch");
}

template <typename T>
void launch_conv_t(const ConvInput& in, const ConvTuning& t, Plan& pl, Mode mode, const void* img, const void* flt,
                   void* out, cudaStream_t s) {
    ktune_dev::ConvProblem<T> prob{};
    prob.flt = static_cast<const T*>(flt);
    prob.img = static_cast<const T*>(img);
    prob.Nb = in.n_batch;
    prob.P = in.p;
    prob.Q = in.q;
    prob.K = in.k_filters;
    prob.C = in.c;
    prob.R = in.r;
    prob.S = in.s;
    prob.H = in.h();
    prob.W = in.w();
    prob.pl = t.p_l;
    prob.ql = t.q_l;
    prob.nlb = t.n_l;
    prob.tiles_q = int(ceil_div(in.q, t.q_l));
    prob.tiles_n = int(ceil_div(in.n_batch, t.n_l));
    pl.p.out = out;
    const void* k = pick(true, in.dtype, mode, pl);
    prepare(k, pl.smem);
    void* args[] = {&prob, &pl.p};
    check(cudaLaunchKernel(k, pl.grid, dim3(unsigned(pl.threads)), args, pl.smem, s), "conv launch");
}

}  // namespace

std::size_t gemm_workspace_bytes(const GemmInput& in, const GemmTuning& t) {
    if (is_tensor_core_dtype(in.dtype)) return umma::gemm_workspace_bytes(in, t);
    return gemm_plan(in, t).ws_bytes;
}

std::size_t conv_workspace_bytes(const ConvInput& in, const ConvTuning& t) { return conv_plan(in, t).ws_bytes; }

void gemm(const GemmInput& in, const GemmTuning& t, Mode mode, const void* a, const void* b, void* c, void* ws,
          std::size_t ws_bytes, cudaStream_t stream) {
    if (is_tensor_core_dtype(in.dtype)) {
        umma::gemm(in, t, a, b, c, ws, ws_bytes, stream);
        return;
    }
    Plan pl = gemm_plan(in, t);
    bind_workspace(pl, ws, ws_bytes);
    if (in.dtype == Dtype::f32) launch_gemm_t<float>(in, pl, mode, a, b, c, stream);
    else launch_gemm_t<double>(in, pl, mode, a, b, c, stream);
}

void conv(const ConvInput& in, const ConvTuning& t, Mode mode, const void* images, const void* filters, void* outputs,
          void* ws, std::size_t ws_bytes, cudaStream_t stream) {
    Plan pl = conv_plan(in, t);
    bind_workspace(pl, ws, ws_bytes);
    if (in.dtype == Dtype::f32) launch_conv_t<float>(in, t, pl, mode, images, filters, outputs, stream);
    else launch_conv_t<double>(in, t, pl, mode, images, filters, outputs, stream);
}

LaunchInfo gemm_launch_info(const GemmInput& in, const GemmTuning& t, Mode mode) {
    if (is_tensor_core_dtype(in.dtype)) return umma::gemm_launch_info(in, t);
    Plan pl = gemm_plan(in, t);
    pick(false, in.dtype, mode, pl);
    return LaunchInfo{pl.threads, pl.smem, int(pl.grid.x), int(pl.grid.y), int(pl.grid.z), pl.generic, "simt"};
}

LaunchInfo conv_launch_info(const ConvInput& in, const ConvTuning& t, Mode mode) {
    Plan pl = conv_plan(in, t);
    pick(true, in.dtype, mode, pl);
    return LaunchInfo{pl.threads, pl.smem, int(pl.grid.x), int(pl.grid.y), int(pl.grid.z), pl.generic, "simt"};
}

// ---------------------------------------------------------------------------
// K8: L2 flush -- stream a write over 2x the L2 capacity.
// ---------------------------------------------------------------------------

namespace {

__global__ void flush_kernel(uint4* buf, std::size_t n16, unsigned salt) {
    const std::size_t stride = std::size_t(gridDim.x) * blockDim.x;
    for (std::size_t i = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride)
        buf[i] = make_uint4(salt, unsigned(i), salt ^ 0x9e3779b9u, unsigned(i >> 32));
}

// splitmix64-derived uniform [0,1) with 53 (f64) / 24 (f32) random bits.
__device__ __forceinline__ std::uint64_t mix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

template <typename T>
__global__ void fill_kernel(T* dst, std::int64_t n, std::uint64_t seed) {
    const std::int64_t stride = std::int64_t(gridDim.x) * blockDim.x;
    for (std::int64_t i = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const std::uint64_t r = mix64(seed ^ mix64(std::uint64_t(i)));
        dst[i] = T(double(r >> 11) * 0x1.0p-53);
    }
}

__global__ void fill_16bit_kernel(unsigned short* dst, std::int64_t n, std::uint64_t seed, int bf16) {
    const std::int64_t stride = std::int64_t(gridDim.x) * blockDim.x;
    for (std::int64_t i = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const std::uint64_t r = mix64(seed ^ mix64(std::uint64_t(i)));
        const float v = float(double(r >> 11) * 0x1.0p-53);
        unsigned short bits;
        if (bf16) {
            unsigned u = __float_as_uint(v);
            u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
            bits = static_cast<unsigned short>(u >> 16);
        } else {
            bits = __half_as_ushort(__float2half_rn(v));
        }
        dst[i] = bits;
    }
}

struct FlushBuffer {
    void* ptr{nullptr};
    std::size_t bytes{0};
    unsigned salt{0};
};

}  // namespace

void l2_flush(cudaStream_t stream) {
    static std::mutex mu;
    static std::unordered_map<int, FlushBuffer> per_device;
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    FlushBuffer* fb;
    {
        std::lock_guard<std::mutex> lock(mu);
        fb = &per_device[dev];
        if (fb->ptr == nullptr) {
            int l2 = 0;
            check(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev), "L2 size");
            fb->bytes = std::max<std::size_t>(std::size_t(l2) * 2, 64u << 20);
            check(cudaMalloc(&fb->ptr, fb->bytes), "cudaMalloc(flush)");
        }
        ++fb->salt;
    }
    int sms = 0;
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
    flush_kernel<<<sms * 4, 512, 0, stream>>>(static_cast<uint4*>(fb->ptr), fb->bytes / 16, fb->salt);
    check(cudaGetLastError(), "flush launch");
}

void fill_uniform(void* dst, std::int64_t n, Dtype dtype, std::uint64_t seed, cudaStream_t stream) {
    if (n <= 0) return;
    const int blocks = int(std::min<std::int64_t>((n + 255) / 256, 148 * 8));
    switch (dtype) {
        case Dtype::f32:
        case Dtype::tf32: fill_kernel<float><<<blocks, 256, 0, stream>>>(static_cast<float*>(dst), n, seed); break;
        case Dtype::f64: fill_kernel<double><<<blocks, 256, 0, stream>>>(static_cast<double*>(dst), n, seed); break;
        case Dtype::bf16:
            fill_16bit_kernel<<<blocks, 256, 0, stream>>>(static_cast<unsigned short*>(dst), n, seed, 1);
            break;
        case Dtype::f16:
            fill_16bit_kernel<<<blocks, 256, 0, stream>>>(static_cast<unsigned short*>(dst), n, seed, 0);
            break;
    }
    check(cudaGetLastError(), "fill launch");
}

}  // namespace dev
}  // namespace ktune
