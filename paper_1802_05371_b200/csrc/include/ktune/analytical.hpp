#pragma once
// The analytical latency/throughput cost model (paper Eqs. (1)-(3)), kept as
// the deterministic host-side pricing model behind `--backend analytical` and
// the AnalyticalPredictor.  Surface and results mirror
// /root/reference/proj/include/ktune/backends.hpp:20-59 and
// src/backends.cpp:14-195 (tests/golden pins every number).  It prices the
// fictional device a HardwareDescriptor describes; it never runs on the GPU.

#include "ktune/space.hpp"

namespace ktune {

double occupancy(const ResourceUsage& res, const HardwareDescriptor& hw);

struct AnalyticalCosts {
    double thread_macs{0}, merge_flops{0}, thread_loads{0}, blocks{0}, warps_per_block{0}, resident_blocks{0},
        mean_warps{0}, waves{0}, main_cycles{0}, merge_pass_cycles{0}, total_cycles{0}, seconds{0}, gflops{0};
};

AnalyticalCosts analytical_costs(const GemmInput& in, const GemmTuning& t, const HardwareDescriptor& hw);
AnalyticalCosts analytical_costs(const ConvInput& in, const ConvTuning& t, const HardwareDescriptor& hw);
double analytical_gflops(const GemmInput& in, const GemmTuning& t, const HardwareDescriptor& hw);
double analytical_gflops(const ConvInput& in, const ConvTuning& t, const HardwareDescriptor& hw);
double peak_gflops(const HardwareDescriptor& hw);

}  // namespace ktune
