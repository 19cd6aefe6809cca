// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library (ktune, built by
// oracle/Makefile from /root/reference/proj/src into oracle/_ref/).  Loaded by
// tests/ (to pin the oracle and generate golden fixtures) and by bench.py's
// --impl reference / cpu_baseline legs.  Never loaded by the product path.
//
// Every wrapper forwards to the reference symbol it names; nothing here
// re-implements reference behaviour.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "ktune/backends.hpp"
#include "ktune/param_space.hpp"
#include "ktune/perf_model.hpp"
#include "ktune/pipeline.hpp"
#include "ktune/tensor_file.hpp"
#include "ktune/sampler.hpp"

using namespace ktune;

namespace {

thread_local std::string g_text;
thread_local std::string g_err;

GemmInput gemm_in(std::int64_t m, std::int64_t n, std::int64_t k, int dtype, int ta, int tb) {
    GemmInput in;
    in.m = m;
    in.n = n;
    in.k = k;
    in.dtype = static_cast<Dtype>(dtype);
    in.trans_a = ta != 0;
    in.trans_b = tb != 0;
    return in;
}

ConvInput conv_in(const std::int64_t* d, int dtype) {
    ConvInput in;
    in.n_batch = d[0];
    in.p = d[1];
    in.q = d[2];
    in.k_filters = d[3];
    in.c = d[4];
    in.r = d[5];
    in.s = d[6];
    in.dtype = static_cast<Dtype>(dtype);
    return in;
}

GemmTuning gemm_t(const std::int32_t* v) {
    return gemm_tuning_from_values(std::vector<int>(v, v + 8));
}

ConvTuning conv_t(const std::int32_t* v) {
    return conv_tuning_from_values(std::vector<int>(v, v + 12));
}

HardwareDescriptor hw_of(const char* json) {
    if (json == nullptr || json[0] == '\0') return HardwareDescriptor{};
    return HardwareDescriptor::from_json_text(json);
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err.c_str(); }

// --- executors (backends.cpp:228-457) -------------------------------------
__attribute__((visibility("default"))) int ref_execute_gemm_f32(std::int64_t m, std::int64_t n, std::int64_t k,
                                                                int ta, int tb, const std::int32_t* tv,
                                                                const float* a, const float* b, float* c) {
    return guarded([&] {
        GemmInput in = gemm_in(m, n, k, 1, ta, tb);
        execute_gemm<float>(in, gemm_t(tv), std::span<const float>(a, std::size_t(m * k)),
                            std::span<const float>(b, std::size_t(k * n)),
                            std::span<float>(c, std::size_t(m * n)));
    });
}

__attribute__((visibility("default"))) int ref_execute_gemm_f64(std::int64_t m, std::int64_t n, std::int64_t k,
                                                                int ta, int tb, const std::int32_t* tv,
                                                                const double* a, const double* b, double* c) {
    return guarded([&] {
        GemmInput in = gemm_in(m, n, k, 2, ta, tb);
        execute_gemm<double>(in, gemm_t(tv), std::span<const double>(a, std::size_t(m * k)),
                             std::span<const double>(b, std::size_t(k * n)),
                             std::span<double>(c, std::size_t(m * n)));
    });
}

__attribute__((visibility("default"))) int ref_execute_conv_f32(const std::int64_t* d, const std::int32_t* tv,
                                                                const float* img, const float* flt, float* out) {
    return guarded([&] {
        ConvInput in = conv_in(d, 1);
        execute_conv<float>(in, conv_t(tv),
                            std::span<const float>(img, std::size_t(in.c * in.h() * in.w() * in.n_batch)),
                            std::span<const float>(flt, std::size_t(in.c * in.r * in.s * in.k_filters)),
                            std::span<float>(out, std::size_t(in.k_filters * in.p * in.q * in.n_batch)));
    });
}

__attribute__((visibility("default"))) int ref_execute_conv_f64(const std::int64_t* d, const std::int32_t* tv,
                                                                const double* img, const double* flt, double* out) {
    return guarded([&] {
        ConvInput in = conv_in(d, 2);
        execute_conv<double>(in, conv_t(tv),
                             std::span<const double>(img, std::size_t(in.c * in.h() * in.w() * in.n_batch)),
                             std::span<const double>(flt, std::size_t(in.c * in.r * in.s * in.k_filters)),
                             std::span<double>(out, std::size_t(in.k_filters * in.p * in.q * in.n_batch)));
    });
}

__attribute__((visibility("default"))) int ref_indirection(const std::int64_t* d, std::int64_t* out4) {
    return guarded([&] {
        auto tab = build_indirection_table(conv_in(d, 1));
        for (std::size_t i = 0; i < tab.size(); ++i) {
            out4[4 * i + 0] = tab[i].c;
            out4[4 * i + 1] = tab[i].r;
            out4[4 * i + 2] = tab[i].s;
            out4[4 * i + 3] = tab[i].image_offset;
        }
    });
}

// --- measurement (backends.cpp:471-556) ------------------------------------
__attribute__((visibility("default"))) int ref_cpu_measure_gemm(const char* hw, std::int64_t m, std::int64_t n,
                                                                std::int64_t k, int dtype, int ta, int tb,
                                                                const std::int32_t* tv, int reps, double* gflops) {
    return guarded([&] {
        CpuBackend be(hw_of(hw), reps);
        *gflops = be.measure(gemm_in(m, n, k, dtype, ta, tb), gemm_t(tv));
    });
}

__attribute__((visibility("default"))) int ref_cpu_measure_conv(const char* hw, const std::int64_t* d, int dtype,
                                                                const std::int32_t* tv, int reps, double* gflops) {
    return guarded([&] {
        CpuBackend be(hw_of(hw), reps);
        *gflops = be.measure(conv_in(d, dtype), conv_t(tv));
    });
}

// Whole-host throughput of the reference executor: `threads` concurrent
// copies of execute_gemm<float> on independent seeded operands (the
// reference itself is single-threaded; this is the "all host cores" figure).
// Each thread runs one warm-up then `reps` timed runs; returns aggregate
// GFLOPS = threads*reps*2MNK / wall seconds of the timed region.
__attribute__((visibility("default"))) int ref_host_gemm_gflops(std::int64_t m, std::int64_t n, std::int64_t k,
                                                                int ta, int tb, const std::int32_t* tv, int reps,
                                                                int threads, double* gflops, double* seconds) {
    return guarded([&] {
        GemmInput in = gemm_in(m, n, k, 1, ta, tb);
        GemmTuning t = gemm_t(tv);
        std::atomic<int> ready{0};
        std::atomic<bool> go{false};
        std::vector<std::thread> pool;
        std::chrono::steady_clock::time_point t0, t1;
        std::vector<double> done_at(std::size_t(threads), 0.0);
        for (int w = 0; w < threads; ++w) {
            pool.emplace_back([&, w] {
                std::mt19937_64 rng(0x5eedULL + std::uint64_t(w));
                std::vector<float> a(std::size_t(m * k)), b(std::size_t(k * n)), c(std::size_t(m * n));
                for (auto& x : a) x = float(unit_real(rng));
                for (auto& x : b) x = float(unit_real(rng));
                execute_gemm<float>(in, t, a, b, c);  // warm-up
                ready.fetch_add(1);
                while (!go.load()) std::this_thread::yield();
                for (int r = 0; r < reps; ++r) execute_gemm<float>(in, t, a, b, c);
                done_at[std::size_t(w)] = std::chrono::duration<double>(
                    std::chrono::steady_clock::now().time_since_epoch()).count();
            });
        }
        while (ready.load() < threads) std::this_thread::yield();
        t0 = std::chrono::steady_clock::now();
        go.store(true);
        for (auto& th : pool) th.join();
        double start = std::chrono::duration<double>(t0.time_since_epoch()).count();
        double end = 0;
        for (double d : done_at) end = std::max(end, d);
        *seconds = end - start;
        *gflops = double(threads) * reps * 2.0 * double(m) * double(n) * double(k) / *seconds / 1e9;
    });
}

// Operand fill of CpuBackend::measure: mt19937_64 + the reference unit_real
// (sampler.cpp:14-17, backends.cpp:481-484) -- pins the oracle's own engine.
__attribute__((visibility("default"))) int ref_fill_f64(std::uint64_t seed, std::int64_t n, double* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        for (std::int64_t i = 0; i < n; ++i) out[i] = unit_real(rng);
    });
}

// --- parameter space (param_space.cpp) ---------------------------------------
__attribute__((visibility("default"))) int ref_is_legal_gemm(const char* hw, std::int64_t m, std::int64_t n,
                                                             std::int64_t k, int dtype, int ta, int tb,
                                                             const std::int32_t* tv, int* accepted, int* reason) {
    return guarded([&] {
        auto v = is_legal(gemm_in(m, n, k, dtype, ta, tb), gemm_t(tv), hw_of(hw));
        *accepted = v.accepted ? 1 : 0;
        *reason = int(v.reason);
        g_text = v.detail;
    });
}

__attribute__((visibility("default"))) int ref_is_legal_conv(const char* hw, const std::int64_t* d, int dtype,
                                                             const std::int32_t* tv, int* accepted, int* reason) {
    return guarded([&] {
        auto v = is_legal(conv_in(d, dtype), conv_t(tv), hw_of(hw));
        *accepted = v.accepted ? 1 : 0;
        *reason = int(v.reason);
        g_text = v.detail;
    });
}

__attribute__((visibility("default"))) const char* ref_last_text() { return g_text.c_str(); }

__attribute__((visibility("default"))) int ref_resources_gemm(std::int64_t m, std::int64_t n, std::int64_t k,
                                                              int dtype, const std::int32_t* tv, std::int64_t* out3) {
    return guarded([&] {
        auto r = estimate_resources(gemm_in(m, n, k, dtype, 0, 0), gemm_t(tv));
        out3[0] = r.shared_bytes;
        out3[1] = r.registers_per_thread;
        out3[2] = r.threads_per_block;
    });
}

__attribute__((visibility("default"))) int ref_resources_conv(const std::int64_t* d, int dtype,
                                                              const std::int32_t* tv, std::int64_t* out3) {
    return guarded([&] {
        auto r = estimate_resources(conv_in(d, dtype), conv_t(tv));
        out3[0] = r.shared_bytes;
        out3[1] = r.registers_per_thread;
        out3[2] = r.threads_per_block;
    });
}

// Writes up to `cap` tunings (8 ints each); returns the total count in *count.
__attribute__((visibility("default"))) int ref_enumerate_gemm(const char* hw, const char* bounds, std::int64_t m,
                                                              std::int64_t n, std::int64_t k, int dtype, int ta,
                                                              int tb, std::int32_t* out, std::int64_t cap,
                                                              std::int64_t* count) {
    return guarded([&] {
        GemmBounds b = (bounds && bounds[0]) ? GemmBounds::from_json_text(bounds) : GemmBounds::defaults();
        auto list = enumerate_legal(gemm_in(m, n, k, dtype, ta, tb), hw_of(hw), b);
        *count = std::int64_t(list.size());
        for (std::int64_t i = 0; i < std::min<std::int64_t>(cap, *count); ++i) {
            auto v = to_values(list[std::size_t(i)]);
            for (int j = 0; j < 8; ++j) out[8 * i + j] = v[std::size_t(j)];
        }
    });
}

__attribute__((visibility("default"))) int ref_enumerate_conv(const char* hw, const char* bounds,
                                                              const std::int64_t* d, int dtype, std::int32_t* out,
                                                              std::int64_t cap, std::int64_t* count) {
    return guarded([&] {
        ConvBounds b = (bounds && bounds[0]) ? ConvBounds::from_json_text(bounds) : ConvBounds::defaults();
        auto list = enumerate_legal(conv_in(d, dtype), hw_of(hw), b);
        *count = std::int64_t(list.size());
        for (std::int64_t i = 0; i < std::min<std::int64_t>(cap, *count); ++i) {
            auto v = to_values(list[std::size_t(i)]);
            for (int j = 0; j < 12; ++j) out[12 * i + j] = v[std::size_t(j)];
        }
    });
}

__attribute__((visibility("default"))) int ref_features_gemm(std::int64_t m, std::int64_t n, std::int64_t k,
                                                             int dtype, int ta, int tb, const std::int32_t* tv,
                                                             double* out14) {
    return guarded([&] {
        auto f = encode_features(gemm_in(m, n, k, dtype, ta, tb), gemm_t(tv));
        std::memcpy(out14, f.data(), f.size() * sizeof(double));
    });
}

__attribute__((visibility("default"))) int ref_features_conv(const std::int64_t* d, int dtype,
                                                             const std::int32_t* tv, double* out19) {
    return guarded([&] {
        auto f = encode_features(conv_in(d, dtype), conv_t(tv));
        std::memcpy(out19, f.data(), f.size() * sizeof(double));
    });
}

__attribute__((visibility("default"))) int ref_analytical_gemm(const char* hw, std::int64_t m, std::int64_t n,
                                                               std::int64_t k, int dtype, int ta, int tb,
                                                               const std::int32_t* tv, double* gflops) {
    return guarded([&] { *gflops = analytical_gflops(gemm_in(m, n, k, dtype, ta, tb), gemm_t(tv), hw_of(hw)); });
}

__attribute__((visibility("default"))) int ref_analytical_conv(const char* hw, const std::int64_t* d, int dtype,
                                                               const std::int32_t* tv, double* gflops) {
    return guarded([&] { *gflops = analytical_gflops(conv_in(d, dtype), conv_t(tv), hw_of(hw)); });
}

__attribute__((visibility("default"))) int ref_peak_gflops(const char* hw, double* out) {
    return guarded([&] { *out = peak_gflops(hw_of(hw)); });
}

__attribute__((visibility("default"))) int ref_hw_json(const char* hw) {
    return guarded([&] { g_text = hw_of(hw).to_json_text(); });
}

__attribute__((visibility("default"))) int ref_bounds_json(const char* bounds, int conv) {
    return guarded([&] {
        if (conv)
            g_text = ((bounds && bounds[0]) ? ConvBounds::from_json_text(bounds) : ConvBounds::defaults()).to_json_text();
        else
            g_text = ((bounds && bounds[0]) ? GemmBounds::from_json_text(bounds) : GemmBounds::defaults()).to_json_text();
    });
}

// --- sampler (sampler.cpp) -----------------------------------------------
__attribute__((visibility("default"))) int ref_calibrate_gemm(const char* hw, const char* bounds, std::int64_t m,
                                                              std::int64_t n, std::int64_t k, int dtype,
                                                              std::int64_t draws, std::uint64_t seed, double alpha) {
    return guarded([&] {
        GemmBounds b = (bounds && bounds[0]) ? GemmBounds::from_json_text(bounds) : GemmBounds::defaults();
        auto model = calibrate(make_legality(gemm_in(m, n, k, dtype, 0, 0), hw_of(hw)), b.as_lists(), draws, seed,
                               alpha);
        g_text = model.to_json_text();
    });
}

__attribute__((visibility("default"))) int ref_calibrate_conv(const char* hw, const char* bounds,
                                                              const std::int64_t* d, int dtype, std::int64_t draws,
                                                              std::uint64_t seed, double alpha) {
    return guarded([&] {
        ConvBounds b = (bounds && bounds[0]) ? ConvBounds::from_json_text(bounds) : ConvBounds::defaults();
        auto model = calibrate(make_legality(conv_in(d, dtype), hw_of(hw)), b.as_lists(), draws, seed, alpha);
        g_text = model.to_json_text();
    });
}

__attribute__((visibility("default"))) int ref_acceptance_gemm(const char* hw, const char* sampler, std::int64_t m,
                                                               std::int64_t n, std::int64_t k, int dtype,
                                                               std::int64_t trials, std::uint64_t seed,
                                                               double* rate) {
    return guarded([&] {
        auto model = CategoricalModel::from_json_text(sampler);
        *rate = acceptance_rate(model, make_legality(gemm_in(m, n, k, dtype, 0, 0), hw_of(hw)), trials, seed);
    });
}

// --- dataset generation with the analytical backend (pipeline.cpp:463-556) --
// shapes_json: the fixture shape-table text (or empty); returns CSV in text.
__attribute__((visibility("default"))) int ref_generate_gemm(const char* hw, const char* bounds,
                                                             const char* sampler, const std::int64_t* shape_rows,
                                                             int n_shapes, double fixed_fraction, int dtype,
                                                             int n_samples, std::uint64_t seed, std::int64_t* attempts,
                                                             std::int64_t* dups) {
    return guarded([&] {
        HardwareDescriptor h = hw_of(hw);
        GemmBounds b = (bounds && bounds[0]) ? GemmBounds::from_json_text(bounds) : GemmBounds::defaults();
        auto model = CategoricalModel::from_json_text(sampler);
        GemmInputDistribution dist;
        for (int i = 0; i < n_shapes; ++i) {
            const std::int64_t* r = shape_rows + 6 * i;
            dist.shapes.push_back(gemm_in(r[0], r[1], r[2], int(r[3]), int(r[4]), int(r[5])));
        }
        dist.fixed_fraction = fixed_fraction;
        dist.dtype = static_cast<Dtype>(dtype);
        AnalyticalBackend be(h);
        GenerateReport rep;
        auto ds = generate_gemm_dataset(be, model, dist, b, h, n_samples, seed, &rep);
        *attempts = rep.attempts;
        *dups = rep.duplicates_rejected;
        g_text = to_csv_text(ds);
    });
}

__attribute__((visibility("default"))) int ref_generate_conv(const char* hw, const char* bounds,
                                                             const char* sampler, const std::int64_t* shape_rows,
                                                             int n_shapes, double fixed_fraction, int dtype,
                                                             int n_samples, std::uint64_t seed, std::int64_t* attempts,
                                                             std::int64_t* dups) {
    return guarded([&] {
        HardwareDescriptor h = hw_of(hw);
        ConvBounds b = (bounds && bounds[0]) ? ConvBounds::from_json_text(bounds) : ConvBounds::defaults();
        auto model = CategoricalModel::from_json_text(sampler);
        ConvInputDistribution dist;
        for (int i = 0; i < n_shapes; ++i) dist.shapes.push_back(conv_in(shape_rows + 8 * i, int(shape_rows[8 * i + 7])));
        dist.fixed_fraction = fixed_fraction;
        dist.dtype = static_cast<Dtype>(dtype);
        AnalyticalBackend be(h);
        GenerateReport rep;
        auto ds = generate_conv_dataset(be, model, dist, b, h, n_samples, seed, &rep);
        *attempts = rep.attempts;
        *dups = rep.duplicates_rejected;
        g_text = to_csv_text(ds);
    });
}

__attribute__((visibility("default"))) int ref_csv_roundtrip_gemm(const char* csv) {
    return guarded([&] { g_text = to_csv_text(gemm_dataset_from_csv_text(csv)); });
}

// --- MLP (perf_model.cpp) --------------------------------------------------
// Trains on a CSV dataset (to_training_set) and returns the model JSON.
__attribute__((visibility("default"))) int ref_train_gemm(const char* csv, const int* hidden, int n_hidden,
                                                          int epochs, double lr, int batch, std::uint64_t seed,
                                                          double val_fraction, int log_inputs,
                                                          double* best_val_mse, int* best_epoch) {
    return guarded([&] {
        auto ds = gemm_dataset_from_csv_text(csv);
        auto set = to_training_set(ds);
        MlpArchitecture arch;
        arch.input_dim = set.dim;
        arch.hidden_sizes.assign(hidden, hidden + n_hidden);
        arch.log_inputs = log_inputs != 0;
        TrainConfig cfg;
        cfg.epochs = epochs;
        cfg.learning_rate = lr;
        cfg.batch_size = batch;
        cfg.rng_seed = seed;
        cfg.validation_fraction = val_fraction;
        auto res = mlp_train(set, arch, cfg);
        *best_val_mse = res.best_val_mse;
        *best_epoch = res.best_epoch;
        MlpModel model;
        model.feature_version = kGemmFeatureVersion;
        model.weights = res.weights;
        g_text = model.to_json_text();
    });
}

__attribute__((visibility("default"))) int ref_init_weights(int input_dim, const int* hidden, int n_hidden,
                                                            std::uint64_t seed) {
    return guarded([&] {
        MlpArchitecture arch;
        arch.input_dim = input_dim;
        arch.hidden_sizes.assign(hidden, hidden + n_hidden);
        MlpModel model;
        model.feature_version = kGemmFeatureVersion;
        model.weights = init_weights(arch, seed);
        g_text = model.to_json_text();
    });
}

__attribute__((visibility("default"))) int ref_mlp_predict(const char* model_json, const double* rows,
                                                           std::int64_t n, int dim, double* out) {
    return guarded([&] {
        auto model = MlpModel::from_json_text(model_json);
        std::vector<std::vector<double>> r{static_cast<std::size_t>(n)};
        for (std::int64_t i = 0; i < n; ++i) r[std::size_t(i)].assign(rows + i * dim, rows + (i + 1) * dim);
        std::vector<double> o;
        model.predict_batch(r, o);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

__attribute__((visibility("default"))) int ref_mlp_backward(const char* model_json, const double* rows,
                                                            const double* y, std::int64_t n, int dim) {
    return guarded([&] {
        auto model = MlpModel::from_json_text(model_json);
        TrainingSet set;
        for (std::int64_t i = 0; i < n; ++i) set.add(std::span<const double>(rows + i * dim, std::size_t(dim)), y[i]);
        MlpModel g;
        g.feature_version = model.feature_version;
        g.weights = mlp_backward(model.weights, set);
        g_text = g.to_json_text();
    });
}

// --- inference + cache (pipeline.cpp:649-997) --------------------------------
__attribute__((visibility("default"))) int ref_infer_gemm_analytical(const char* hw, const char* bounds,
                                                                     const char* model_json, std::int64_t m,
                                                                     std::int64_t n, std::int64_t k, int dtype,
                                                                     int ta, int tb, int top_k) {
    return guarded([&] {
        HardwareDescriptor h = hw_of(hw);
        GemmBounds b = (bounds && bounds[0]) ? GemmBounds::from_json_text(bounds) : GemmBounds::defaults();
        AnalyticalBackend be(h);
        GemmInput in = gemm_in(m, n, k, dtype, ta, tb);
        if (model_json && model_json[0]) {
            MlpPredictor pred(MlpModel::from_json_text(model_json));
            g_text = to_json_text(infer_gemm(pred, in, h, b, top_k, be));
        } else {
            AnalyticalPredictor pred(h);
            g_text = to_json_text(infer_gemm(pred, in, h, b, top_k, be));
        }
    });
}

// --- KTN1 tensor files (tensor_file.cpp) ------------------------------------
__attribute__((visibility("default"))) int ref_write_tensor(const char* path, int f64, const std::int64_t* dims,
                                                            int ndims, const void* data) {
    return guarded([&] {
        TensorFile t;
        t.dtype = f64 ? Dtype::f64 : Dtype::f32;
        t.dims.assign(dims, dims + ndims);
        const std::int64_t n = t.element_count();
        if (f64) t.f64.assign(static_cast<const double*>(data), static_cast<const double*>(data) + n);
        else t.f32.assign(static_cast<const float*>(data), static_cast<const float*>(data) + n);
        write_tensor(path, t);
    });
}

__attribute__((visibility("default"))) int ref_cache_key_gemm(std::int64_t m, std::int64_t n, std::int64_t k,
                                                              int dtype, int ta, int tb) {
    return guarded([&] { g_text = cache_key(gemm_in(m, n, k, dtype, ta, tb)); });
}

__attribute__((visibility("default"))) int ref_cache_key_conv(const std::int64_t* d, int dtype) {
    return guarded([&] { g_text = cache_key(conv_in(d, dtype)); });
}

}  // extern "C"
