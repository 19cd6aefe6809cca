#pragma once
// Shared plumbing of the C-ABI translation units: exception -> status
// mapping and POD <-> C++ conversions (include/ktune_b200.h).

#include <string>

#include "ktune/b200_backend.hpp"
#include "ktune/kernels.hpp"
#include "ktune/space.hpp"
#include "ktune_b200.h"

namespace ktune::capi {

using namespace ktune;

std::string& last_error();
std::string& last_text();


template <typename F>
inline int guard(F&& f) {
    try {
        f();
        return KTUNE_OK;
    } catch (const workspace_error& e) {
        last_error() = e.what();
        return KTUNE_ERR_WORKSPACE;
    } catch (const unsupported_error& e) {
        last_error() = e.what();
        return KTUNE_ERR_UNSUPPORTED;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return KTUNE_ERR_INVALID_ARGUMENT;
    } catch (const cuda_error& e) {
        last_error() = e.what();
        return KTUNE_ERR_CUDA;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return KTUNE_ERR_RUNTIME;
    } catch (...) {
        last_error() = "unknown error";
        return KTUNE_ERR_RUNTIME;
    }
}

inline void need(const void* p, const char* what) {
    if (p == nullptr) throw std::invalid_argument(std::string(what) + " must not be NULL");
}

inline Dtype dtype_of(int32_t d) {
    if (d < 0 || d > 4) throw std::invalid_argument("unknown dtype code " + std::to_string(d));
    return static_cast<Dtype>(d);
}

inline GemmInput conv_in(const ktune_gemm_input* p) {
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

inline ConvInput conv_in(const ktune_conv_input* p) {
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

inline GemmTuning conv_t(const ktune_gemm_tuning* p) {
    need(p, "gemm tuning");
    return GemmTuning{p->m_s, p->n_s, p->m_l, p->n_l, p->u, p->k_s, p->k_l, p->k_g};
}

inline ConvTuning conv_t(const ktune_conv_tuning* p) {
    need(p, "conv tuning");
    return ConvTuning{p->k_s, p->p_s, p->q_s, p->n_s, p->k_l, p->p_l, p->q_l, p->n_l, p->u, p->c_s, p->c_l, p->c_g};
}

inline HardwareDescriptor conv_hw(const ktune_hw* p) {
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

inline void put_hw(const HardwareDescriptor& hw, ktune_hw* out) {
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

inline dev::Mode mode_of(int m) {
    if (m != KTUNE_MODE_FAST && m != KTUNE_MODE_PARITY) throw std::invalid_argument("unknown mode " + std::to_string(m));
    return static_cast<dev::Mode>(m);
}

inline MeasureOptions opts_of(const ktune_measure_options* o) {
    MeasureOptions m;
    if (o == nullptr) return m;
    m.mode = mode_of(o->mode);
    m.repetitions = o->repetitions;
    m.warmup = o->warmup;
    m.flush_l2 = o->flush_l2 != 0;
    m.seed = o->seed;
    return m;
}


}  // namespace ktune::capi
