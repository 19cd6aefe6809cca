// Analytical cost model (host oracle, /root/reference/proj/src/backends.cpp
// :14-195).  Every floating-point expression keeps the reference's
// evaluation order so prices agree to the last bit.

#include "ktune/analytical.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace ktune {

namespace {

double cdiv(double a, double b) { return std::ceil(a / b); }

// Per-instruction cost for one warp when n warps share a pipe.
double pipe(double latency, double throughput, double n) { return std::max(latency / n, throughput); }

struct Occ {
    double wpb{0};       // warps per block
    double resident{0};  // co-resident blocks (wave accounting)
    double warps{0};     // occupancy before grid starvation
};

Occ occupy(const ResourceUsage& r, const HardwareDescriptor& hw) {
    Occ o;
    o.wpb = cdiv(double(r.threads_per_block), double(hw.warp_size));
    double blocks = std::floor(double(hw.max_threads_per_block) / double(r.threads_per_block));
    if (r.shared_bytes > 0)
        blocks = std::min(blocks, std::floor(double(hw.max_shared_bytes_per_block) / double(r.shared_bytes)));
    o.warps = std::min(double(hw.max_warps_per_multiprocessor), blocks * o.wpb);
    o.resident = std::max(1.0, std::min(blocks, std::floor(double(hw.max_warps_per_multiprocessor) / o.wpb)));
    return o;
}

struct Work {
    double macs, merge, loads, blocks, useful;
    std::int64_t merge_outputs;
    int splits;
};

AnalyticalCosts price(const Work& w, const ResourceUsage& res, const HardwareDescriptor& hw) {
    AnalyticalCosts c;
    const Occ o = occupy(res, hw);
    const double sm = double(hw.num_multiprocessors);
    c.thread_macs = w.macs;
    c.merge_flops = w.merge;
    c.thread_loads = w.loads;
    c.blocks = w.blocks;
    c.warps_per_block = o.wpb;
    c.resident_blocks = o.resident;
    c.mean_warps = std::min(o.warps, w.blocks * o.wpb / sm);
    c.waves = cdiv(w.blocks, o.resident * sm);
    const double ta = pipe(hw.alu_latency, hw.alu_throughput, c.mean_warps);
    const double tm = pipe(hw.mem_latency, hw.mem_throughput, c.mean_warps);
    const double per_wave = std::max(ta * w.macs, tm * w.loads) + ta * w.merge;
    c.main_cycles = per_wave * c.mean_warps * c.waves;
    c.merge_pass_cycles = 0.0;
    if (w.splits > 1) {
        // The k_g fold as a separate elementwise kernel: splits loads + adds per output.
        ResourceUsage mres;
        mres.shared_bytes = 0;
        mres.registers_per_thread = 16;
        mres.threads_per_block = std::min<std::int64_t>(hw.max_threads_per_block, 8 * hw.warp_size);
        const Occ mo = occupy(mres, hw);
        const double mblocks = cdiv(double(w.merge_outputs), double(mres.threads_per_block));
        const double mn = std::min(std::min(double(hw.max_warps_per_multiprocessor), mo.resident * mo.wpb),
                                   mblocks * mo.wpb / sm);
        const double g = double(w.splits);
        const double mwave =
            std::max(pipe(hw.alu_latency, hw.alu_throughput, mn) * g, pipe(hw.mem_latency, hw.mem_throughput, mn) * g);
        c.merge_pass_cycles = mwave * mn * cdiv(mblocks, mo.resident * sm);
    }
    c.total_cycles = c.main_cycles + c.merge_pass_cycles;
    c.seconds = c.total_cycles / hw.clock_hz;
    c.gflops = w.useful / c.seconds / 1.0e9;
    return c;
}

void need_legal(const LegalityVerdict& v) {
    if (!v) throw std::invalid_argument(std::string("illegal tuning: ") + to_string(v.reason) + " (" + v.detail + ")");
}

}  // namespace

double occupancy(const ResourceUsage& res, const HardwareDescriptor& hw) {
    hw.validate();
    if (res.threads_per_block < 1) throw std::invalid_argument("occupancy: threads_per_block must be >= 1");
    if (res.threads_per_block > hw.max_threads_per_block || res.shared_bytes > hw.max_shared_bytes_per_block) return 0.0;
    return occupy(res, hw).warps;
}

double peak_gflops(const HardwareDescriptor& hw) {
    return 2.0 * double(hw.num_multiprocessors) * double(hw.warp_size) * hw.clock_hz / hw.alu_throughput / 1.0e9;
}

AnalyticalCosts analytical_costs(const GemmInput& in, const GemmTuning& t, const HardwareDescriptor& hw) {
    need_legal(is_legal(in, t, hw));
    Work w;
    const double span = double(t.u) * t.k_l * t.k_g;
    const double steps = cdiv(double(in.k), span);
    const double tile = double(t.m_s) * t.n_s;
    w.macs = tile * steps * t.u;
    w.merge = tile * double((t.k_s - 1) + (t.k_l - 1));
    w.loads = steps * t.u * tile * (1.0 / t.m_l + 1.0 / t.n_l);
    w.blocks = cdiv(double(in.m), t.m_l) * cdiv(double(in.n), t.n_l) * double(t.k_g);
    w.useful = 2.0 * double(in.m) * double(in.n) * double(in.k);
    w.merge_outputs = in.m * in.n;
    w.splits = t.k_g;
    return price(w, estimate_resources(in, t), hw);
}

AnalyticalCosts analytical_costs(const ConvInput& in, const ConvTuning& t, const HardwareDescriptor& hw) {
    need_legal(is_legal(in, t, hw));
    Work w;
    const double crs = double(in.c) * in.r * in.s;
    const double span = double(t.u) * t.c_l * t.c_g;
    const double steps = cdiv(crs, span);
    const double tile = double(t.k_s) * t.p_s * t.q_s * t.n_s;
    w.macs = tile * steps * t.u;
    w.merge = tile * double((t.c_s - 1) + (t.c_l - 1));
    w.loads = steps * t.u * tile * (1.0 / t.k_l + 1.0 / (double(t.p_l) * t.q_l * t.n_l));
    w.blocks = cdiv(double(in.k_filters), t.k_l) * cdiv(double(in.p), t.p_l) * cdiv(double(in.q), t.q_l) *
               cdiv(double(in.n_batch), t.n_l) * double(t.c_g);
    w.useful = 2.0 * double(in.n_batch) * in.p * in.q * double(in.k_filters) * crs;
    w.merge_outputs = in.k_filters * in.p * in.q * in.n_batch;
    w.splits = t.c_g;
    return price(w, estimate_resources(in, t), hw);
}

double analytical_gflops(const GemmInput& in, const GemmTuning& t, const HardwareDescriptor& hw) {
    return analytical_costs(in, t, hw).gflops;
}

double analytical_gflops(const ConvInput& in, const ConvTuning& t, const HardwareDescriptor& hw) {
    return analytical_costs(in, t, hw).gflops;
}

}  // namespace ktune
