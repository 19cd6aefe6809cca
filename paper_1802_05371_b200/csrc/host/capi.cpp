// capi.cpp -- the extern "C" boundary declared in include/ktune_b200.h.
// Each entry converts POD structs to the C++ types of ktune/space.hpp,
// calls the library, and maps exceptions to ktune_status codes.

#include "ktune_b200.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "capi_internal.hpp"
#include "ktune/tensor_file.hpp"

using namespace ktune;

namespace ktune::capi {

std::string& last_error() {
    thread_local std::string s;
    return s;
}

std::string& last_text() {
    thread_local std::string s;
    return s;
}

}  // namespace ktune::capi

using namespace ktune::capi;

extern "C" {

int ktune_abi_version(void) { return KTUNE_B200_ABI_VERSION; }
const char* ktune_last_error(void) { return last_error().c_str(); }
const char* ktune_last_text(void) { return last_text().c_str(); }

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
        last_text() = v.detail;
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
        last_text() = v.detail;
    });
}

int ktune_enumerate_legal_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const char* bounds_json,
                               ktune_gemm_tuning* out, int64_t cap, int64_t* count) {
    return guard([&] {
        need(count, "count");
        if (cap > 0) need(out, "out");
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
        if (cap > 0) need(out, "out");
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
        if (cap > 0) need(out4, "out4");
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

int ktune_gemm_launch_info(const ktune_gemm_input* in, const ktune_gemm_tuning* t, int mode, int* threads,
                           size_t* smem_bytes, int* grid3, char* family, size_t family_cap) {
    return guard([&] {
        need(threads, "threads");
        need(smem_bytes, "smem_bytes");
        need(grid3, "grid3");
        const dev::LaunchInfo li = dev::gemm_launch_info(conv_in(in), conv_t(t), mode_of(mode));
        *threads = li.threads;
        *smem_bytes = li.smem_bytes;
        grid3[0] = li.grid_x;
        grid3[1] = li.grid_y;
        grid3[2] = li.grid_z;
        if (family != nullptr && family_cap > 0) {
            std::snprintf(family, family_cap, "%s%s", li.family, li.generic ? "-generic" : "");
        }
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

int ktune_tensor_write(const char* path, int32_t dtype, const int64_t* dims, int32_t ndims, const void* data) {
    return guard([&] {
        need(path, "path");
        TensorFile t;
        t.dtype = dtype_of(dtype);
        if (ndims < 0 || (ndims > 0 && dims == nullptr)) throw std::invalid_argument("tensor_write: bad dims");
        for (int32_t i = 0; i < ndims; ++i)
            if (dims[i] < 1) throw std::invalid_argument("tensor_write: every dim must be >= 1");
        t.dims.assign(dims, dims + ndims);
        const std::int64_t n = ndims > 0 ? t.element_count() : 0;
        if (n > 0) need(data, "data");
        if (t.dtype == Dtype::f32) t.f32.assign(static_cast<const float*>(data), static_cast<const float*>(data) + n);
        else if (t.dtype == Dtype::f64) t.f64.assign(static_cast<const double*>(data), static_cast<const double*>(data) + n);
        write_tensor(path, t);
    });
}

int ktune_tensor_read(const char* path, int32_t* dtype, int64_t* dims8, int32_t* ndims, void* data, int64_t cap) {
    return guard([&] {
        need(path, "path");
        need(dtype, "dtype");
        need(dims8, "dims");
        need(ndims, "ndims");
        const TensorFile t = read_tensor(path);
        *dtype = int32_t(t.dtype);
        *ndims = int32_t(t.dims.size());
        for (std::size_t i = 0; i < t.dims.size(); ++i) dims8[i] = t.dims[i];
        const std::int64_t n = t.element_count();
        if (data != nullptr && cap >= n) {
            if (t.dtype == Dtype::f32) std::memcpy(data, t.f32.data(), std::size_t(n) * 4);
            else std::memcpy(data, t.f64.data(), std::size_t(n) * 8);
        }
    });
}

}  // extern "C"
