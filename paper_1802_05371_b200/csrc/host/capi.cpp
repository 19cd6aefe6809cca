// capi.cpp -- the extern "C" boundary declared in include/ktune_b200.h.
// Each entry converts POD structs to the C++ types of ktune/space.hpp,
// calls the library, and maps exceptions to ktune_status codes.

#include "ktune_b200.h"

#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "ktune/b200_backend.hpp"
#include "ktune/kernels.hpp"
#include "ktune/space.hpp"

using namespace ktune;

namespace {

thread_local std::string g_error;
thread_local std::string g_text;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return KTUNE_OK;
    } catch (const workspace_error& e) {
        g_error = e.what();
        return KTUNE_ERR_WORKSPACE;
    } catch (const unsupported_error& e) {
        g_error = e.what();
        return KTUNE_ERR_UNSUPPORTED;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return KTUNE_ERR_INVALID_ARGUMENT;
    } catch (const cuda_error& e) {
        g_error = e.what();
        return KTUNE_ERR_CUDA;
    } catch (const std::exception& e) {
        g_error = e.what();
        return KTUNE_ERR_RUNTIME;
    } catch (...) {
        g_error = "unknown error";
        return KTUNE_ERR_RUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (p == nullptr) throw std::invalid_argument(std::string(what) + " must not be NULL");
}

Dtype dtype_of(int32_t d) {
    if (d < 0 || d > 4) throw std::invalid_argument("unknown dtype code " + std::to_string(d));
    return static_cast<Dtype>(d);
}

GemmInput conv_in(const ktune_gemm_input* p) {
    need(p, "gemm input");
    GemmInput in;
    in.m = p->m;
    in.n = p->n;
    in.k = p->k;
    in.dtype = dtype_of(p->dtype);
    in.trans_a = p->trans_a != 0;
    in.trans_b = p->trans_b != 0;
    return in;
}

ConvInput conv_in(const ktune_conv_input* p) {
    need(p, "conv input");
    ConvInput in;
    in.n_batch = p->n_batch;
    in.p = p->p;
    in.q = p->q;
    in.k_filters = p->k_filters;
    in.c = p->c;
    in.r = p->r;
    in.s = p->s;
    in.dtype = dtype_of(p->dtype);
    return in;
}

GemmTuning conv_t(const ktune_gemm_tuning* p) {
    need(p, "gemm tuning");
    return GemmTuning{p->m_s, p->n_s, p->m_l, p->n_l, p->u, p->k_s, p->k_l, p->k_g};
}

ConvTuning conv_t(const ktune_conv_tuning* p) {
    need(p, "conv tuning");
    return ConvTuning{p->k_s, p->p_s, p->q_s, p->n_s, p->k_l, p->p_l, p->q_l, p->n_l, p->u, p->c_s, p->c_l, p->c_g};
}

HardwareDescriptor conv_hw(const ktune_hw* p) {
    need(p, "hardware descriptor");
    HardwareDescriptor hw;
    hw.max_shared_bytes_per_block = p->max_shared_bytes_per_block;
    hw.max_registers_per_thread = p->max_registers_per_thread;
    hw.max_threads_per_block = p->max_threads_per_block;
    hw.max_warps_per_multiprocessor = p->max_warps_per_multiprocessor;
    hw.warp_size = p->warp_size;
    hw.alu_latency = p->alu_latency;
    hw.alu_throughput = p->alu_throughput;
    hw.mem_latency = p->mem_latency;
    hw.mem_throughput = p->mem_throughput;
    hw.clock_hz = p->clock_hz;
    hw.num_multiprocessors = p->num_multiprocessors;
    return hw;
}

void put_hw(const HardwareDescriptor& hw, ktune_hw* out) {
    out->max_shared_bytes_per_block = hw.max_shared_bytes_per_block;
    out->max_registers_per_thread = hw.max_registers_per_thread;
    out->max_threads_per_block = hw.max_threads_per_block;
    out->max_warps_per_multiprocessor = hw.max_warps_per_multiprocessor;
    out->warp_size = hw.warp_size;
    out->alu_latency = hw.alu_latency;
    out->alu_throughput = hw.alu_throughput;
    out->mem_latency = hw.mem_latency;
    out->mem_throughput = hw.mem_throughput;
    out->clock_hz = hw.clock_hz;
    out->num_multiprocessors = hw.num_multiprocessors;
}

dev::Mode mode_of(int m) {
    if (m != KTUNE_MODE_FAST && m != KTUNE_MODE_PARITY) throw std::invalid_argument("unknown mode " + std::to_string(m));
    return static_cast<dev::Mode>(m);
}

MeasureOptions opts_of(const ktune_measure_options* o) {
    MeasureOptions m;
    if (o == nullptr) return m;
    m.mode = mode_of(o->mode);
    m.repetitions = o->repetitions;
    m.warmup = o->warmup;
    m.flush_l2 = o->flush_l2 != 0;
    m.seed = o->seed;
    return m;
}

}  // namespace

extern "C" {

int ktune_abi_version(void) { return KTUNE_B200_ABI_VERSION; }
const char* ktune_last_error(void) { return g_error.c_str(); }
const char* ktune_last_text(void) { return g_text.c_str(); }

int ktune_set_device(int device) {
    return guard([&] { dev::check(cudaSetDevice(device), "cudaSetDevice"); });
}

int ktune_hw_default(ktune_hw* out) {
    return guard([&] {
        need(out, "out");
        put_hw(HardwareDescriptor{}, out);
    });
}

int ktune_hw_from_json(const char* text, ktune_hw* out) {
    return guard([&] {
        need(text, "json text");
        need(out, "out");
        put_hw(HardwareDescriptor::from_json_text(text), out);
    });
}

int ktune_estimate_resources_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, ktune_resources* out) {
    return guard([&] {
        need(out, "out");
        auto r = estimate_resources(conv_in(in), conv_t(t));
        *out = ktune_resources{r.shared_bytes, r.registers_per_thread, r.threads_per_block};
    });
}

int ktune_estimate_resources_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, ktune_resources* out) {
    return guard([&] {
        need(out, "out");
        auto r = estimate_resources(conv_in(in), conv_t(t));
        *out = ktune_resources{r.shared_bytes, r.registers_per_thread, r.threads_per_block};
    });
}

int ktune_is_legal_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const ktune_gemm_tuning* t, int* accepted,
                        int* reason) {
    return guard([&] {
        need(accepted, "accepted");
        need(reason, "reason");
        auto v = is_legal(conv_in(in), conv_t(t), conv_hw(hw));
        *accepted = v.accepted ? 1 : 0;
        *reason = int(v.reason);
        g_text = v.detail;
    });
}

int ktune_is_legal_conv(const ktune_hw* hw, const ktune_conv_input* in, const ktune_conv_tuning* t, int* accepted,
                        int* reason) {
    return guard([&] {
        need(accepted, "accepted");
        need(reason, "reason");
        auto v = is_legal(conv_in(in), conv_t(t), conv_hw(hw));
        *accepted = v.accepted ? 1 : 0;
        *reason = int(v.reason);
        g_text = v.detail;
    });
}

int ktune_enumerate_legal_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const char* bounds_json,
                               ktune_gemm_tuning* out, int64_t cap, int64_t* count) {
    return guard([&] {
        need(count, "count");
        GemmBounds b = (bounds_json && bounds_json[0]) ? GemmBounds::from_json_text(bounds_json) : GemmBounds::defaults();
        auto list = enumerate_legal(conv_in(in), conv_hw(hw), b);
        *count = int64_t(list.size());
        for (int64_t i = 0; i < std::min<int64_t>(cap, *count); ++i) {
            const auto& x = list[std::size_t(i)];
            out[i] = ktune_gemm_tuning{x.m_s, x.n_s, x.m_l, x.n_l, x.u, x.k_s, x.k_l, x.k_g};
        }
    });
}

int ktune_enumerate_legal_conv(const ktune_hw* hw, const ktune_conv_input* in, const char* bounds_json,
                               ktune_conv_tuning* out, int64_t cap, int64_t* count) {
    return guard([&] {
        need(count, "count");
        ConvBounds b = (bounds_json && bounds_json[0]) ? ConvBounds::from_json_text(bounds_json) : ConvBounds::defaults();
        auto list = enumerate_legal(conv_in(in), conv_hw(hw), b);
        *count = int64_t(list.size());
        for (int64_t i = 0; i < std::min<int64_t>(cap, *count); ++i) {
            const auto& x = list[std::size_t(i)];
            out[i] = ktune_conv_tuning{x.k_s, x.p_s, x.q_s, x.n_s, x.k_l, x.p_l, x.q_l, x.n_l, x.u, x.c_s, x.c_l, x.c_g};
        }
    });
}

int ktune_encode_features_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, double* out14) {
    return guard([&] {
        need(out14, "out");
        auto f = encode_features(conv_in(in), conv_t(t));
        std::memcpy(out14, f.data(), f.size() * sizeof(double));
    });
}

int ktune_encode_features_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, double* out19) {
    return guard([&] {
        need(out19, "out");
        auto f = encode_features(conv_in(in), conv_t(t));
        std::memcpy(out19, f.data(), f.size() * sizeof(double));
    });
}

int ktune_build_indirection_table(const ktune_conv_input* in, int64_t* out4, int64_t cap, int64_t* count) {
    return guard([&] {
        need(count, "count");
        auto tab = build_indirection_table(conv_in(in));
        *count = int64_t(tab.size());
        for (int64_t i = 0; i < std::min<int64_t>(cap, *count); ++i) {
            const auto& e = tab[std::size_t(i)];
            out4[4 * i + 0] = e.c;
            out4[4 * i + 1] = e.r;
            out4[4 * i + 2] = e.s;
            out4[4 * i + 3] = e.image_offset;
        }
    });
}

int ktune_gemm_workspace_size(const ktune_gemm_input* in, const ktune_gemm_tuning* t, size_t* bytes) {
    return guard([&] {
        need(bytes, "bytes");
        *bytes = dev::gemm_workspace_bytes(conv_in(in), conv_t(t));
    });
}

int ktune_conv_workspace_size(const ktune_conv_input* in, const ktune_conv_tuning* t, size_t* bytes) {
    return guard([&] {
        need(bytes, "bytes");
        *bytes = dev::conv_workspace_bytes(conv_in(in), conv_t(t));
    });
}

int ktune_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, int mode, const void* a, const void* b, void* c,
               void* workspace, size_t workspace_bytes, void* stream) {
    return guard([&] {
        need(a, "a");
        need(b, "b");
        need(c, "c");
        dev::gemm(conv_in(in), conv_t(t), mode_of(mode), a, b, c, workspace, workspace_bytes,
                  static_cast<cudaStream_t>(stream));
    });
}

int ktune_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, int mode, const void* images,
               const void* filters, void* outputs, void* workspace, size_t workspace_bytes, void* stream) {
    return guard([&] {
        need(images, "images");
        need(filters, "filters");
        need(outputs, "outputs");
        dev::conv(conv_in(in), conv_t(t), mode_of(mode), images, filters, outputs, workspace, workspace_bytes,
                  static_cast<cudaStream_t>(stream));
    });
}

int ktune_execute_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, int mode, const void* a, int64_t a_len,
                       const void* b, int64_t b_len, void* c, int64_t c_len) {
    return guard([&] {
        need(a, "a");
        need(b, "b");
        need(c, "c");
        execute_gemm_host(conv_in(in), conv_t(t), mode_of(mode), a, a_len, b, b_len, c, c_len);
    });
}

int ktune_execute_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, int mode, const void* images,
                       int64_t images_len, const void* filters, int64_t filters_len, void* outputs,
                       int64_t outputs_len) {
    return guard([&] {
        need(images, "images");
        need(filters, "filters");
        need(outputs, "outputs");
        execute_conv_host(conv_in(in), conv_t(t), mode_of(mode), images, images_len, filters, filters_len, outputs,
                          outputs_len);
    });
}

int ktune_measure_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const ktune_gemm_tuning* t,
                       const ktune_measure_options* opts, double* gflops) {
    return guard([&] {
        need(gflops, "gflops");
        *gflops = measure_gemm_device(conv_hw(hw), conv_in(in), conv_t(t), opts_of(opts)).gflops;
    });
}

int ktune_measure_conv(const ktune_hw* hw, const ktune_conv_input* in, const ktune_conv_tuning* t,
                       const ktune_measure_options* opts, double* gflops) {
    return guard([&] {
        need(gflops, "gflops");
        *gflops = measure_conv_device(conv_hw(hw), conv_in(in), conv_t(t), opts_of(opts)).gflops;
    });
}

int ktune_l2_flush(void* stream) {
    return guard([&] { dev::l2_flush(static_cast<cudaStream_t>(stream)); });
}

}  // extern "C"
