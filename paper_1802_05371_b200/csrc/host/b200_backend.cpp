// Device measurement and host-buffer execution (see b200_backend.hpp).

#include "ktune/b200_backend.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace ktune {

namespace {

using dev::check;

// Grow-only device allocation.
struct DevBuf {
    void* ptr{nullptr};
    std::size_t bytes{0};
    void reserve(std::size_t n, bool zero) {
        if (n <= bytes) return;
        if (ptr) check(cudaFree(ptr), "cudaFree");
        ptr = nullptr;
        bytes = 0;
        check(cudaMalloc(&ptr, std::max<std::size_t>(n, 256)), "cudaMalloc");
        bytes = std::max<std::size_t>(n, 256);
        if (zero) {
            check(cudaMemset(ptr, 0, bytes), "cudaMemset");
            check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");  // visible to non-blocking streams
        }
    }
};

// Seeded operand buffers: the fill is a pure function of (seed, role, index),
// so a grown buffer's prefix equals a fresh fill and buffers can be reused
// across samples of different shapes.
struct Operand {
    DevBuf buf;
    std::int64_t filled{0};
    Dtype dtype{Dtype::f32};
    std::uint64_t seed{0};
};

struct DeviceState {
    std::mutex mu;  // one measurement at a time per device
    cudaStream_t stream{nullptr};
    cudaEvent_t ev0{nullptr}, ev1{nullptr};
    Operand ops[2];
    DevBuf out, ws;
    std::vector<cudaEvent_t> pool;  // timing events of measure_*_many
    // host-buffer staging
    DevBuf ha, hb, hc, hws;
    void init() {
        if (stream) return;
        check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
        check(cudaEventCreate(&ev0), "cudaEventCreate");
        check(cudaEventCreate(&ev1), "cudaEventCreate");
    }
};

DeviceState& state() {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<DeviceState>> all;
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    auto& p = all[dev];
    if (!p) p = std::make_unique<DeviceState>();
    return *p;
}

const void* operand(DeviceState& st, int role, Dtype dt, std::int64_t n, std::uint64_t seed) {
    Operand& op = st.ops[role];
    const std::size_t bytes = std::size_t(n) * dtype_size_bytes(dt);
    const std::uint64_t s = seed * 0x100000001b3ULL + std::uint64_t(role + 1);
    if (op.dtype != dt || op.seed != s || op.filled < n) {
        op.buf.reserve(bytes, false);
        const std::int64_t cap = std::int64_t(op.buf.bytes / dtype_size_bytes(dt));
        dev::fill_uniform(op.buf.ptr, cap, dt, s, st.stream);
        op.filled = cap;
        op.dtype = dt;
        op.seed = s;
    }
    return op.buf.ptr;
}

void require_legal(const LegalityVerdict& v) {
    if (!v)
        throw std::invalid_argument(std::string("illegal tuning: ") + to_string(v.reason) + " (" + v.detail + ")");
}

template <typename Launch>
MeasureResult time_it(DeviceState& st, const MeasureOptions& opt, double flops, Launch&& launch) {
    if (opt.repetitions < 1) throw std::invalid_argument("measure: repetitions must be >= 1");
    for (int i = 0; i < std::max(0, opt.warmup); ++i) launch();
    double best = std::numeric_limits<double>::infinity(), total = 0;
    for (int r = 0; r < opt.repetitions; ++r) {
        if (opt.flush_l2) dev::l2_flush(st.stream);
        check(cudaEventRecord(st.ev0, st.stream), "cudaEventRecord");
        launch();
        check(cudaEventRecord(st.ev1, st.stream), "cudaEventRecord");
        check(cudaEventSynchronize(st.ev1), "cudaEventSynchronize");
        float ms = 0;
        check(cudaEventElapsedTime(&ms, st.ev0, st.ev1), "cudaEventElapsedTime");
        const double s = std::max(double(ms) * 1e-3, 1e-9);
        best = std::min(best, s);
        total += s;
    }
    MeasureResult res;
    res.best_seconds = best;
    res.mean_seconds = total / opt.repetitions;
    res.gflops = flops / best / 1e9;
    return res;
}

}  // namespace

int output_elem_size(Dtype d) { return is_tensor_core_dtype(d) ? 4 : dtype_size_bytes(d); }

MeasureResult measure_gemm_device(const HardwareDescriptor& hw, const GemmInput& in, const GemmTuning& t,
                                  const MeasureOptions& opt) {
    require_legal(is_legal(in, t, hw));
    DeviceState& st = state();
    std::lock_guard<std::mutex> lock(st.mu);
    st.init();
    const void* a = operand(st, 0, in.dtype, in.m * in.k, opt.seed);
    const void* b = operand(st, 1, in.dtype, in.k * in.n, opt.seed);
    st.out.reserve(std::size_t(in.m * in.n) * output_elem_size(in.dtype), false);
    const std::size_t wsb = dev::gemm_workspace_bytes(in, t);
    st.ws.reserve(wsb, true);  // split-K counter region must start zeroed
    const double flops = 2.0 * double(in.m) * double(in.n) * double(in.k);
    return time_it(st, opt, flops, [&] {
        dev::gemm(in, t, opt.mode, a, b, st.out.ptr, st.ws.ptr, st.ws.bytes, st.stream);
    });
}

MeasureResult measure_conv_device(const HardwareDescriptor& hw, const ConvInput& in, const ConvTuning& t,
                                  const MeasureOptions& opt) {
    require_legal(is_legal(in, t, hw));
    DeviceState& st = state();
    std::lock_guard<std::mutex> lock(st.mu);
    st.init();
    const void* img = operand(st, 0, in.dtype, in.c * in.h() * in.w() * in.n_batch, opt.seed);
    const void* flt = operand(st, 1, in.dtype, in.c * in.r * in.s * in.k_filters, opt.seed);
    st.out.reserve(std::size_t(in.k_filters * in.p * in.q * in.n_batch) * output_elem_size(in.dtype), false);
    const std::size_t wsb = dev::conv_workspace_bytes(in, t);
    st.ws.reserve(wsb, true);  // split-K counter region must start zeroed
    const double flops = 2.0 * double(in.n_batch) * double(in.p) * double(in.q) * double(in.k_filters) *
                         double(in.c) * double(in.r) * double(in.s);
    return time_it(st, opt, flops, [&] {
        dev::conv(in, t, opt.mode, img, flt, st.out.ptr, st.ws.ptr, st.ws.bytes, st.stream);
    });
}

namespace {

template <typename In, typename Tu, typename Setup>
std::vector<double> time_many(const std::vector<In>& ins, const std::vector<Tu>& tus, const MeasureOptions& opt,
                              Setup setup) {
    if (ins.size() != tus.size()) throw std::invalid_argument("measure_many: inputs / tunings size mismatch");
    if (opt.repetitions < 1) throw std::invalid_argument("measure: repetitions must be >= 1");
    DeviceState& st = state();
    std::lock_guard<std::mutex> lock(st.mu);
    st.init();
    const std::size_t n = ins.size();
    const std::size_t need = n * std::size_t(opt.repetitions) * 2;
    while (st.pool.size() < need) {
        cudaEvent_t e;
        check(cudaEventCreate(&e), "cudaEventCreate");
        st.pool.push_back(e);
    }
    std::vector<double> out(n, -1.0), flops(n, 0.0);
    std::vector<char> ok(n, 0);
    for (std::size_t i = 0; i < n; ++i) {
        std::function<void()> launch;
        try {
            launch = setup(st, ins[i], tus[i], flops[i]);  // legality, operands, workspace, plan
            for (int w = 0; w < std::max(0, opt.warmup); ++w) launch();
        } catch (const unsupported_error&) {
            continue;  // outside this build's envelope: reported as -1
        }
        for (int r = 0; r < opt.repetitions; ++r) {
            if (opt.flush_l2) dev::l2_flush(st.stream);
            check(cudaEventRecord(st.pool[(i * opt.repetitions + r) * 2], st.stream), "cudaEventRecord");
            launch();
            check(cudaEventRecord(st.pool[(i * opt.repetitions + r) * 2 + 1], st.stream), "cudaEventRecord");
        }
        ok[i] = 1;
    }
    check(cudaStreamSynchronize(st.stream), "cudaStreamSynchronize");
    for (std::size_t i = 0; i < n; ++i) {
        if (!ok[i]) continue;
        double best = std::numeric_limits<double>::infinity();
        for (int r = 0; r < opt.repetitions; ++r) {
            float ms = 0;
            check(cudaEventElapsedTime(&ms, st.pool[(i * opt.repetitions + r) * 2],
                                       st.pool[(i * opt.repetitions + r) * 2 + 1]),
                  "cudaEventElapsedTime");
            best = std::min(best, std::max(double(ms) * 1e-3, 1e-9));
        }
        out[i] = flops[i] / best / 1e9;
    }
    return out;
}

}  // namespace

std::vector<double> measure_gemm_many(const HardwareDescriptor& hw, const std::vector<GemmInput>& in,
                                      const std::vector<GemmTuning>& t, const MeasureOptions& opt) {
    return time_many(in, t, opt, [&](DeviceState& st, const GemmInput& x, const GemmTuning& tu, double& flops) {
        require_legal(is_legal(x, tu, hw));
        (void)dev::gemm_launch_info(x, tu, opt.mode);  // throws unsupported_error before any launch
        const void* a = operand(st, 0, x.dtype, x.m * x.k, opt.seed);
        const void* b = operand(st, 1, x.dtype, x.k * x.n, opt.seed);
        st.out.reserve(std::size_t(x.m * x.n) * output_elem_size(x.dtype), false);
        st.ws.reserve(dev::gemm_workspace_bytes(x, tu), true);
        flops = 2.0 * double(x.m) * double(x.n) * double(x.k);
        return std::function<void()>([&st, x, tu, a, b, mode = opt.mode] {
            dev::gemm(x, tu, mode, a, b, st.out.ptr, st.ws.ptr, st.ws.bytes, st.stream);
        });
    });
}

std::vector<double> measure_conv_many(const HardwareDescriptor& hw, const std::vector<ConvInput>& in,
                                      const std::vector<ConvTuning>& t, const MeasureOptions& opt) {
    return time_many(in, t, opt, [&](DeviceState& st, const ConvInput& x, const ConvTuning& tu, double& flops) {
        require_legal(is_legal(x, tu, hw));
        (void)dev::conv_launch_info(x, tu, opt.mode);
        const void* img = operand(st, 0, x.dtype, x.c * x.h() * x.w() * x.n_batch, opt.seed);
        const void* flt = operand(st, 1, x.dtype, x.c * x.r * x.s * x.k_filters, opt.seed);
        st.out.reserve(std::size_t(x.k_filters * x.p * x.q * x.n_batch) * output_elem_size(x.dtype), false);
        st.ws.reserve(dev::conv_workspace_bytes(x, tu), true);
        flops = 2.0 * double(x.n_batch) * double(x.p) * double(x.q) * double(x.k_filters) * double(x.c) *
                double(x.r) * double(x.s);
        return std::function<void()>([&st, x, tu, img, flt, mode = opt.mode] {
            dev::conv(x, tu, mode, img, flt, st.out.ptr, st.ws.ptr, st.ws.bytes, st.stream);
        });
    });
}

bool B200Backend::accepts(const GemmInput& in, const GemmTuning& t) const {
    try {
        (void)dev::gemm_launch_info(in, t, opt_.mode);
        return true;
    } catch (const unsupported_error&) {
        return false;
    }
}

bool B200Backend::accepts(const ConvInput& in, const ConvTuning& t) const {
    try {
        (void)dev::conv_launch_info(in, t, opt_.mode);
        return true;
    } catch (const unsupported_error&) {
        return false;
    }
}

B200Backend::B200Backend(HardwareDescriptor hw, MeasureOptions opt) : hw_(std::move(hw)), opt_(opt) {
    hw_.validate();
    if (opt_.repetitions < 1) throw std::invalid_argument("B200Backend: repetitions must be >= 1");
}

double B200Backend::measure(const GemmInput& in, const GemmTuning& t) {
    return measure_gemm_device(hw_, in, t, opt_).gflops;
}

double B200Backend::measure(const ConvInput& in, const ConvTuning& t) {
    return measure_conv_device(hw_, in, t, opt_).gflops;
}

void execute_gemm_host(const GemmInput& in, const GemmTuning& t, dev::Mode mode, const void* a, std::int64_t a_len,
                       const void* b, std::int64_t b_len, void* c, std::int64_t c_len) {
    in.validate();
    t.validate();
    if (a_len != in.m * in.k || b_len != in.k * in.n || c_len != in.m * in.n)
        throw std::invalid_argument("execute_gemm: operand size mismatch");
    DeviceState& st = state();
    std::lock_guard<std::mutex> lock(st.mu);
    st.init();
    const std::size_t es = dtype_size_bytes(in.dtype), os = output_elem_size(in.dtype);
    const std::size_t wsb = dev::gemm_workspace_bytes(in, t);  // validates the tuple first
    st.ha.reserve(std::size_t(a_len) * es, false);
    st.hb.reserve(std::size_t(b_len) * es, false);
    st.hc.reserve(std::size_t(c_len) * os, false);
    st.hws.reserve(wsb, true);
    check(cudaMemcpyAsync(st.ha.ptr, a, std::size_t(a_len) * es, cudaMemcpyHostToDevice, st.stream), "H2D A");
    check(cudaMemcpyAsync(st.hb.ptr, b, std::size_t(b_len) * es, cudaMemcpyHostToDevice, st.stream), "H2D B");
    dev::gemm(in, t, mode, st.ha.ptr, st.hb.ptr, st.hc.ptr, st.hws.ptr, st.hws.bytes, st.stream);
    check(cudaMemcpyAsync(c, st.hc.ptr, std::size_t(c_len) * os, cudaMemcpyDeviceToHost, st.stream), "D2H C");
    check(cudaStreamSynchronize(st.stream), "cudaStreamSynchronize");
}

void execute_conv_host(const ConvInput& in, const ConvTuning& t, dev::Mode mode, const void* img, std::int64_t img_len,
                       const void* flt, std::int64_t flt_len, void* out, std::int64_t out_len) {
    in.validate();
    t.validate();
    if (img_len != in.c * in.h() * in.w() * in.n_batch || flt_len != in.c * in.r * in.s * in.k_filters ||
        out_len != in.k_filters * in.p * in.q * in.n_batch)
        throw std::invalid_argument("execute_conv: operand size mismatch");
    DeviceState& st = state();
    std::lock_guard<std::mutex> lock(st.mu);
    st.init();
    const std::size_t es = dtype_size_bytes(in.dtype), os = output_elem_size(in.dtype);
    const std::size_t wsb = dev::conv_workspace_bytes(in, t);
    st.ha.reserve(std::size_t(img_len) * es, false);
    st.hb.reserve(std::size_t(flt_len) * es, false);
    st.hc.reserve(std::size_t(out_len) * os, false);
    st.hws.reserve(wsb, true);
    check(cudaMemcpyAsync(st.ha.ptr, img, std::size_t(img_len) * es, cudaMemcpyHostToDevice, st.stream), "H2D images");
    check(cudaMemcpyAsync(st.hb.ptr, flt, std::size_t(flt_len) * es, cudaMemcpyHostToDevice, st.stream), "H2D filters");
    dev::conv(in, t, mode, st.ha.ptr, st.hb.ptr, st.hc.ptr, st.hws.ptr, st.hws.bytes, st.stream);
    check(cudaMemcpyAsync(out, st.hc.ptr, std::size_t(out_len) * os, cudaMemcpyDeviceToHost, st.stream), "D2H outputs");
    check(cudaStreamSynchronize(st.stream), "cudaStreamSynchronize");
}

}  // namespace ktune
