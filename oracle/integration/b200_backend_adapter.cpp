// oracle/integration/b200_backend_adapter.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The backend adapter of INTEGRATION.md route 1, compiled as written there:
// a reference `MeasurementBackend` (proj/include/ktune/backends.hpp:102-109)
// whose measure() calls this repository's C-ABI (include/ktune_b200.h).  It
// is built by `make -C oracle adapter` against the reference headers where
// they lie under /root/reference (never copied) and linked with the
// reference library (oracle/_ref/libktune_ref.so) and libktune_b200.so, so
// the reference's own generate_gemm_dataset drives the B200 path
// (tests/test_integration_adapter_gpu.py).
#include <stdexcept>
#include <string>

#include "ktune/backends.hpp"
#include "ktune_b200.h"

namespace ktune {

namespace {
ktune_hw to_c(const HardwareDescriptor& h) {
    return {h.max_shared_bytes_per_block, h.max_registers_per_thread, h.max_threads_per_block,
            h.max_warps_per_multiprocessor, h.warp_size, h.alu_latency, h.alu_throughput,
            h.mem_latency, h.mem_throughput, h.clock_hz, h.num_multiprocessors};
}
ktune_gemm_input to_c(const GemmInput& in) {
    return {in.m, in.n, in.k, int32_t(in.dtype), in.trans_a, in.trans_b, 0};
}
ktune_conv_input to_c(const ConvInput& in) {
    return {in.n_batch, in.p, in.q, in.k_filters, in.c, in.r, in.s, int32_t(in.dtype), 0};
}
void rethrow(int status) {  // reference error classes (backends.cpp:120-125, 504-506)
    if (status == KTUNE_OK) return;
    if (status == KTUNE_ERR_INVALID_ARGUMENT || status == KTUNE_ERR_UNSUPPORTED || status == KTUNE_ERR_WORKSPACE)
        throw std::invalid_argument(ktune_last_error());
    throw std::runtime_error(ktune_last_error());
}
}  // namespace

class B200Backend final : public MeasurementBackend {
  public:
    explicit B200Backend(HardwareDescriptor hw) : hw_(to_c(hw)) {}
    std::string name() const override { return "b200"; }
    double measure(const GemmInput& in, const GemmTuning& t) override {
        ktune_gemm_input ci = to_c(in);
        ktune_gemm_tuning ct{t.m_s, t.n_s, t.m_l, t.n_l, t.u, t.k_s, t.k_l, t.k_g};
        double g = 0;
        rethrow(ktune_measure_gemm(&hw_, &ci, &ct, nullptr, &g));
        return g;
    }
    double measure(const ConvInput& in, const ConvTuning& t) override {
        ktune_conv_input ci = to_c(in);
        ktune_conv_tuning ct{t.k_s, t.p_s, t.q_s, t.n_s, t.k_l, t.p_l, t.q_l, t.n_l, t.u, t.c_s, t.c_l, t.c_g};
        double g = 0;
        rethrow(ktune_measure_conv(&hw_, &ci, &ct, nullptr, &g));
        return g;
    }

  private:
    ktune_hw hw_;
};

}  // namespace ktune
