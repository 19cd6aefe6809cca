#pragma once
// The B200 measurement backend: the device-timed replacement of
// CpuBackend (/root/reference/proj/include/ktune/backends.hpp:102-137,
// src/backends.cpp:471-556) behind the reference's MeasurementBackend
// interface, so generate_*_dataset / infer_* call sites are unchanged.

#include <cstdint>
#include <string>
#include <vector>

#include "ktune/kernels.hpp"
#include "ktune/space.hpp"

namespace ktune {

// Mirror of backends.hpp:102-109.
class MeasurementBackend {
  public:
    virtual ~MeasurementBackend() = default;
    virtual std::string name() const = 0;
    virtual double measure(const GemmInput& in, const GemmTuning& t) = 0;
    virtual double measure(const ConvInput& in, const ConvTuning& t) = 0;
    // Whether measure() can run this legal pair (the reference's executors
    // run every legal tuple: default true).  generate_*_dataset redraws the
    // pairs a backend does not accept instead of aborting on them.
    virtual bool accepts(const GemmInput&, const GemmTuning&) const { return true; }
    virtual bool accepts(const ConvInput&, const ConvTuning&) const { return true; }
};

struct MeasureOptions {
    dev::Mode mode{dev::Mode::fast};
    int repetitions{3};  // best-of, like CpuBackend (backends.cpp:486-498)
    int warmup{1};
    bool flush_l2{true};
    std::uint64_t seed{0x5eedULL};
};

struct MeasureResult {
    double gflops{0};
    double best_seconds{0};
    double mean_seconds{0};
};

// One device measurement on the current CUDA device (thread-safe; calls are
// serialised per device, "one measurement at a time").
MeasureResult measure_gemm_device(const HardwareDescriptor& hw, const GemmInput& in, const GemmTuning& t,
                                  const MeasureOptions& opt);
MeasureResult measure_conv_device(const HardwareDescriptor& hw, const ConvInput& in, const ConvTuning& t,
                                  const MeasureOptions& opt);

// Many measurements with one host synchronisation per call: every pair's
// warm-up and timed repetitions (each after an L2 flush) are enqueued back to
// back with their CUDA events, then all events are read once.  Same protocol
// and result as measure_*_device per pair; a pair that fails to launch
// (unsupported by this build) yields -1 instead of aborting the batch.
std::vector<double> measure_gemm_many(const HardwareDescriptor& hw, const std::vector<GemmInput>& in,
                                      const std::vector<GemmTuning>& t, const MeasureOptions& opt);
std::vector<double> measure_conv_many(const HardwareDescriptor& hw, const std::vector<ConvInput>& in,
                                      const std::vector<ConvTuning>& t, const MeasureOptions& opt);

class B200Backend final : public MeasurementBackend {
  public:
    explicit B200Backend(HardwareDescriptor hw, MeasureOptions opt = {});
    // CSV backend tag (pipeline.cpp:70-75: no ',' or newline).
    std::string name() const override { return opt_.mode == dev::Mode::parity ? "b200-parity" : "b200"; }
    double measure(const GemmInput& in, const GemmTuning& t) override;
    double measure(const ConvInput& in, const ConvTuning& t) override;
    // inside this build's launch envelope (host-side planning, no launch)
    bool accepts(const GemmInput& in, const GemmTuning& t) const override;
    bool accepts(const ConvInput& in, const ConvTuning& t) const override;
    const HardwareDescriptor& hw() const { return hw_; }

  private:
    HardwareDescriptor hw_;
    MeasureOptions opt_;
};

// Host-buffer execution with the executor contract of backends.cpp:228-240
// (sizes checked, result copied back).  Uses a per-device staging pool.
void execute_gemm_host(const GemmInput& in, const GemmTuning& t, dev::Mode mode, const void* a, std::int64_t a_len,
                       const void* b, std::int64_t b_len, void* c, std::int64_t c_len);
void execute_conv_host(const ConvInput& in, const ConvTuning& t, dev::Mode mode, const void* img, std::int64_t img_len,
                       const void* flt, std::int64_t flt_len, void* out, std::int64_t out_len);

// Element size of the OUTPUT buffer (tensor-core families write fp32).
int output_elem_size(Dtype d);

}  // namespace ktune
