// capi_pipeline.cpp -- extern "C" entry points of the tuning pipeline
// (sampler, predraw/generation, datasets, MLP, runtime selection, cache);
// declarations and reference citations in include/ktune_b200.h.

#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "capi_internal.hpp"
#include "ktune/analytical.hpp"
#include "ktune/mlp.hpp"
#include "ktune/sampling.hpp"
#include "ktune/tuner.hpp"

using namespace ktune;
using namespace ktune::capi;

namespace {

GemmBounds gemm_bounds(const char* json) {
    return (json && json[0]) ? GemmBounds::from_json_text(json) : GemmBounds::defaults();
}

ConvBounds conv_bounds(const char* json) {
    return (json && json[0]) ? ConvBounds::from_json_text(json) : ConvBounds::defaults();
}

GemmInputDistribution gemm_dist(const ktune_gemm_distribution* d) {
    need(d, "distribution");
    GemmInputDistribution g;
    for (int i = 0; i < d->n_shapes; ++i) g.shapes.push_back(conv_in(d->shapes + i));
    if (d->weights) g.weights.assign(d->weights, d->weights + d->n_shapes);
    g.fixed_fraction = d->fixed_fraction;
    g.use_ranges = d->use_ranges != 0;
    g.m_lo = d->m_lo;
    g.m_hi = d->m_hi;
    g.n_lo = d->n_lo;
    g.n_hi = d->n_hi;
    g.k_lo = d->k_lo;
    g.k_hi = d->k_hi;
    g.dtype = dtype_of(d->dtype);
    g.randomize_transpose = d->randomize_transpose != 0;
    return g;
}

ConvInputDistribution conv_dist(const ktune_conv_distribution* d) {
    need(d, "distribution");
    ConvInputDistribution c;
    for (int i = 0; i < d->n_shapes; ++i) c.shapes.push_back(conv_in(d->shapes + i));
    if (d->weights) c.weights.assign(d->weights, d->weights + d->n_shapes);
    c.fixed_fraction = d->fixed_fraction;
    c.use_ranges = d->use_ranges != 0;
    c.n_lo = d->n_lo;
    c.n_hi = d->n_hi;
    c.p_lo = d->p_lo;
    c.p_hi = d->p_hi;
    c.q_lo = d->q_lo;
    c.q_hi = d->q_hi;
    c.k_lo = d->k_lo;
    c.k_hi = d->k_hi;
    c.c_lo = d->c_lo;
    c.c_hi = d->c_hi;
    if (d->rs_choices) {
        c.rs_choices.clear();
        for (int i = 0; i < d->n_rs; ++i) c.rs_choices.push_back({d->rs_choices[2 * i], d->rs_choices[2 * i + 1]});
    }
    c.dtype = dtype_of(d->dtype);
    return c;
}

ktune_gemm_input out_in(const GemmInput& in) {
    return ktune_gemm_input{in.m, in.n, in.k, int32_t(in.dtype), in.trans_a ? 1 : 0, in.trans_b ? 1 : 0, 0};
}

ktune_conv_input out_in(const ConvInput& in) {
    return ktune_conv_input{in.n_batch, in.p, in.q, in.k_filters, in.c, in.r, in.s, int32_t(in.dtype), 0};
}

ktune_gemm_tuning out_t(const GemmTuning& t) { return ktune_gemm_tuning{t.m_s, t.n_s, t.m_l, t.n_l, t.u, t.k_s, t.k_l, t.k_g}; }

ktune_conv_tuning out_t(const ConvTuning& t) {
    return ktune_conv_tuning{t.k_s, t.p_s, t.q_s, t.n_s, t.k_l, t.p_l, t.q_l, t.n_l, t.u, t.c_s, t.c_l, t.c_g};
}

std::unique_ptr<MeasurementBackend> make_backend(int32_t kind, const HardwareDescriptor& hw,
                                                 const ktune_measure_options* opts) {
    switch (kind) {
        case 0: return std::make_unique<AnalyticalBackend>(hw);
        case 1: {
            MeasureOptions o = opts_of(opts);
            if (!opts) o.mode = dev::Mode::fast;
            return std::make_unique<B200Backend>(hw, o);
        }
        case 2: {
            MeasureOptions o = opts_of(opts);
            o.mode = dev::Mode::parity;
            return std::make_unique<B200Backend>(hw, o);
        }
    }
    throw std::invalid_argument("unknown backend " + std::to_string(kind) + " (0 analytical, 1 b200, 2 b200-parity)");
}

std::unique_ptr<PerfPredictor> make_predictor(const char* model_json, const HardwareDescriptor& hw) {
    if (model_json && model_json[0]) return std::make_unique<MlpPredictor>(MlpModel::from_json_text(model_json));
    return std::make_unique<AnalyticalPredictor>(hw);
}

// Runtime-selection memo: cache key -> chosen tuning (per process).
std::mutex g_select_mu;
std::map<std::string, GemmTuning> g_select_memo;
std::map<std::string, ConvTuning> g_select_memo_conv;

template <typename In, typename Tu, typename Draw, typename OutIn, typename OutTu>
void shard_out(const std::vector<Draw>& draws, const std::vector<ShardRecord>& recs, const GenerateReport& rep,
               In* inputs_out, Tu* tunings_out, int64_t* index_out, double* gflops_out, int64_t cap, int64_t* count,
               int64_t* attempts, int64_t* duplicates, int64_t* unlaunchable, OutIn out_in_, OutTu out_t_) {
    if (inputs_out)
        for (std::size_t i = 0; i < draws.size(); ++i) inputs_out[i] = out_in_(draws[i].input);
    if (tunings_out)
        for (std::size_t i = 0; i < draws.size(); ++i) tunings_out[i] = out_t_(draws[i].tuning);
    if (int64_t(recs.size()) > cap)
        throw std::invalid_argument("shard: " + std::to_string(recs.size()) + " records exceed cap " +
                                    std::to_string(cap));
    for (std::size_t i = 0; i < recs.size(); ++i) {
        index_out[i] = recs[i].index;
        gflops_out[i] = recs[i].gflops;
    }
    *count = int64_t(recs.size());
    if (attempts) *attempts = rep.attempts;
    if (duplicates) *duplicates = rep.duplicates_rejected;
    if (unlaunchable) *unlaunchable = rep.unlaunchable_rejected;
}

// Sharded top-k re-measure (reference loop
// pipeline.cpp:674-680): infer_* calls backend.measure once per ranked
// candidate, in rank order.  ShardBackend measures the calls i with
// i % world == rank and records them (others -> -1, never measured);
// ReplayBackend feeds the gathered values back in the same order, so the
// sharded result equals the sequential one.
class ShardBackend final : public MeasurementBackend {
  public:
    ShardBackend(MeasurementBackend& real, int rank, int world) : real_(real), rank_(rank), world_(world) {
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard: rank must lie in [0, world)");
    }
    std::string name() const override { return real_.name(); }
    double measure(const GemmInput& in, const GemmTuning& t) override { return record(mine() ? real_.measure(in, t) : -1.0); }
    double measure(const ConvInput& in, const ConvTuning& t) override { return record(mine() ? real_.measure(in, t) : -1.0); }
    bool accepts(const GemmInput& in, const GemmTuning& t) const override { return real_.accepts(in, t); }
    bool accepts(const ConvInput& in, const ConvTuning& t) const override { return real_.accepts(in, t); }
    std::vector<double> values;

  private:
    bool mine() const { return int(values.size() % std::size_t(world_)) == rank_; }
    double record(double v) {
        values.push_back(v);
        return v;
    }
    MeasurementBackend& real_;
    int rank_, world_;
};

class ReplayBackend final : public MeasurementBackend {
  public:
    // `launch` (may be null): the backend whose launchability filter the
    // shards ranked with, so the replay ranks the same candidates.
    ReplayBackend(std::string name, const double* v, std::int64_t n, std::unique_ptr<MeasurementBackend> launch)
        : name_(std::move(name)), v_(v), n_(n), launch_(std::move(launch)) {}
    std::string name() const override { return name_; }
    double measure(const GemmInput&, const GemmTuning&) override { return take(); }
    double measure(const ConvInput&, const ConvTuning&) override { return take(); }
    bool accepts(const GemmInput& in, const GemmTuning& t) const override { return !launch_ || launch_->accepts(in, t); }
    bool accepts(const ConvInput& in, const ConvTuning& t) const override { return !launch_ || launch_->accepts(in, t); }

  private:
    double take() {
        if (i_ >= n_) throw std::invalid_argument("infer replay: fewer measurements than candidates");
        return v_[i_++];
    }
    std::string name_;
    const double* v_;
    std::int64_t n_, i_{0};
    std::unique_ptr<MeasurementBackend> launch_;
};

// The launchability filter behind a replayed backend name ("b200" /
// "b200-parity"; anything else accepts every legal tuple).
std::unique_ptr<MeasurementBackend> replay_filter(const char* name, const HardwareDescriptor& hw) {
    const std::string n = name ? name : "b200";
    if (n == "b200") return make_backend(1, hw, nullptr);
    if (n == "b200-parity") return make_backend(2, hw, nullptr);
    return nullptr;
}

}  // namespace

extern "C" {

int ktune_peak_gflops(const ktune_hw* hw, double* out) {
    return guard([&] {
        need(out, "out");
        *out = peak_gflops(conv_hw(hw));
    });
}

int ktune_analytical_gflops_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const ktune_gemm_tuning* t,
                                 double* out) {
    return guard([&] {
        need(out, "out");
        *out = analytical_gflops(conv_in(in), conv_t(t), conv_hw(hw));
    });
}

int ktune_analytical_gflops_conv(const ktune_hw* hw, const ktune_conv_input* in, const ktune_conv_tuning* t,
                                 double* out) {
    return guard([&] {
        need(out, "out");
        *out = analytical_gflops(conv_in(in), conv_t(t), conv_hw(hw));
    });
}

int ktune_calibrate_gemm(const ktune_hw* hw, const ktune_gemm_input* probe, const char* bounds_json, int64_t n_uniform,
                         uint64_t seed, double alpha) {
    return guard([&] {
        auto m = calibrate(make_legality(conv_in(probe), conv_hw(hw)), gemm_bounds(bounds_json).as_lists(), n_uniform,
                           seed, alpha);
        last_text() = m.to_json_text();
    });
}

int ktune_calibrate_conv(const ktune_hw* hw, const ktune_conv_input* probe, const char* bounds_json, int64_t n_uniform,
                         uint64_t seed, double alpha) {
    return guard([&] {
        auto m = calibrate(make_legality(conv_in(probe), conv_hw(hw)), conv_bounds(bounds_json).as_lists(), n_uniform,
                           seed, alpha);
        last_text() = m.to_json_text();
    });
}

int ktune_acceptance_rate_gemm(const ktune_hw* hw, const ktune_gemm_input* probe, const char* sampler_json,
                               int64_t n_trials, uint64_t seed, double* rate) {
    return guard([&] {
        need(sampler_json, "sampler_json");
        need(rate, "rate");
        *rate = acceptance_rate(CategoricalModel::from_json_text(sampler_json), make_legality(conv_in(probe), conv_hw(hw)),
                                n_trials, seed);
    });
}

int ktune_uniform_acceptance_rate_gemm(const ktune_hw* hw, const ktune_gemm_input* probe, const char* bounds_json,
                                       int64_t n_trials, uint64_t seed, double* rate) {
    return guard([&] {
        need(rate, "rate");
        *rate = uniform_acceptance_rate(gemm_bounds(bounds_json).as_lists(), make_legality(conv_in(probe), conv_hw(hw)),
                                        n_trials, seed);
    });
}

int ktune_predraw_gemm(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                       const ktune_gemm_distribution* dist, int32_t n_samples, uint64_t seed,
                       ktune_gemm_input* inputs_out, ktune_gemm_tuning* tunings_out, int64_t* attempts,
                       int64_t* duplicates) {
    return guard([&] {
        need(sampler_json, "sampler_json");
        need(inputs_out, "inputs_out");
        need(tunings_out, "tunings_out");
        GenerateReport rep;
        auto draws = predraw_gemm(CategoricalModel::from_json_text(sampler_json), gemm_dist(dist),
                                  gemm_bounds(bounds_json), conv_hw(hw), n_samples, seed, &rep);
        for (std::size_t i = 0; i < draws.size(); ++i) {
            inputs_out[i] = out_in(draws[i].input);
            tunings_out[i] = out_t(draws[i].tuning);
        }
        if (attempts) *attempts = rep.attempts;
        if (duplicates) *duplicates = rep.duplicates_rejected;
    });
}

int ktune_generate_gemm_shard(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                              const ktune_gemm_distribution* dist, int32_t n_samples, uint64_t seed, int32_t rank,
                              int32_t world, const ktune_measure_options* opts, const char* checkpoint_path,
                              ktune_gemm_input* inputs_out, ktune_gemm_tuning* tunings_out, int64_t* index_out,
                              double* gflops_out, int64_t cap, int64_t* count, int64_t* attempts,
                              int64_t* duplicates, int64_t* unlaunchable) {
    return guard([&] {
        need(sampler_json, "sampler_json");
        need(index_out, "index_out");
        need(gflops_out, "gflops_out");
        need(count, "count");
        GenerateReport rep;
        std::vector<GemmDraw> draws;
        auto recs = generate_gemm_shard(CategoricalModel::from_json_text(sampler_json), gemm_dist(dist),
                                        gemm_bounds(bounds_json), conv_hw(hw), n_samples, seed, rank, world,
                                        opts_of(opts), checkpoint_path ? checkpoint_path : "", &draws, &rep);
        shard_out(draws, recs, rep, inputs_out, tunings_out, index_out, gflops_out, cap, count, attempts, duplicates,
                  unlaunchable, [](const GemmInput& x) { return out_in(x); },
                  [](const GemmTuning& x) { return out_t(x); });
    });
}

int ktune_generate_conv_shard(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                              const ktune_conv_distribution* dist, int32_t n_samples, uint64_t seed, int32_t rank,
                              int32_t world, const ktune_measure_options* opts, const char* checkpoint_path,
                              ktune_conv_input* inputs_out, ktune_conv_tuning* tunings_out, int64_t* index_out,
                              double* gflops_out, int64_t cap, int64_t* count, int64_t* attempts,
                              int64_t* duplicates, int64_t* unlaunchable) {
    return guard([&] {
        need(sampler_json, "sampler_json");
        need(index_out, "index_out");
        need(gflops_out, "gflops_out");
        need(count, "count");
        GenerateReport rep;
        std::vector<ConvDraw> draws;
        auto recs = generate_conv_shard(CategoricalModel::from_json_text(sampler_json), conv_dist(dist),
                                        conv_bounds(bounds_json), conv_hw(hw), n_samples, seed, rank, world,
                                        opts_of(opts), checkpoint_path ? checkpoint_path : "", &draws, &rep);
        shard_out(draws, recs, rep, inputs_out, tunings_out, index_out, gflops_out, cap, count, attempts, duplicates,
                  unlaunchable, [](const ConvInput& x) { return out_in(x); },
                  [](const ConvTuning& x) { return out_t(x); });
    });
}

int ktune_shard_lpt(const double* costs, int64_t n, int32_t world, int32_t* rank_out) {
    return guard([&] {
        need(costs, "costs");
        need(rank_out, "rank_out");
        const auto shards = shard_lpt(std::vector<double>(costs, costs + n), world);
        for (std::size_t r = 0; r < shards.size(); ++r)
            for (std::int64_t i : shards[r]) rank_out[i] = int32_t(r);
    });
}

int ktune_predraw_conv(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                       const ktune_conv_distribution* dist, int32_t n_samples, uint64_t seed,
                       ktune_conv_input* inputs_out, ktune_conv_tuning* tunings_out, int64_t* attempts,
                       int64_t* duplicates) {
    return guard([&] {
        need(sampler_json, "sampler_json");
        need(inputs_out, "inputs_out");
        need(tunings_out, "tunings_out");
        GenerateReport rep;
        auto draws = predraw_conv(CategoricalModel::from_json_text(sampler_json), conv_dist(dist),
                                  conv_bounds(bounds_json), conv_hw(hw), n_samples, seed, &rep);
        for (std::size_t i = 0; i < draws.size(); ++i) {
            inputs_out[i] = out_in(draws[i].input);
            tunings_out[i] = out_t(draws[i].tuning);
        }
        if (attempts) *attempts = rep.attempts;
        if (duplicates) *duplicates = rep.duplicates_rejected;
    });
}

int ktune_generate_gemm(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                        const ktune_gemm_distribution* dist, int32_t n_samples, uint64_t seed, int32_t backend,
                        const ktune_measure_options* opts, int64_t* attempts, int64_t* duplicates) {
    return guard([&] {
        need(sampler_json, "sampler_json");
        const HardwareDescriptor h = conv_hw(hw);
        auto be = make_backend(backend, h, opts);
        GenerateReport rep;
        auto ds = generate_gemm_dataset(*be, CategoricalModel::from_json_text(sampler_json), gemm_dist(dist),
                                        gemm_bounds(bounds_json), h, n_samples, seed, &rep);
        if (attempts) *attempts = rep.attempts;
        if (duplicates) *duplicates = rep.duplicates_rejected;
        last_text() = to_csv_text(ds);
    });
}

int ktune_gemm_dataset_csv(const ktune_gemm_input* inputs, const ktune_gemm_tuning* tunings, const double* gflops,
                           int64_t n, const char* backend) {
    return guard([&] {
        need(backend, "backend");
        GemmDataset ds;
        for (int64_t i = 0; i < n; ++i)
            ds.samples.push_back({conv_in(inputs + i), conv_t(tunings + i), gflops[i], backend, 0});
        last_text() = to_csv_text(ds);
    });
}

int ktune_conv_dataset_csv(const ktune_conv_input* inputs, const ktune_conv_tuning* tunings, const double* gflops,
                           int64_t n, const char* backend) {
    return guard([&] {
        need(backend, "backend");
        ConvDataset ds;
        for (int64_t i = 0; i < n; ++i)
            ds.samples.push_back({conv_in(inputs + i), conv_t(tunings + i), gflops[i], backend, 0});
        last_text() = to_csv_text(ds);
    });
}

int ktune_dataset_canonical(const char* csv_text, int32_t kind) {
    return guard([&] {
        need(csv_text, "csv_text");
        last_text() = kind == 0 ? to_csv_text(gemm_dataset_from_csv_text(csv_text))
                                : to_csv_text(conv_dataset_from_csv_text(csv_text));
    });
}

namespace {
int mlp_train_impl(const char* csv_text, int32_t kind, const int32_t* hidden, int32_t n_hidden, int32_t log_inputs,
                   int32_t epochs, double learning_rate, int32_t batch_size, uint64_t seed, double validation_fraction,
                   double* best_val_mse, int32_t* best_epoch, double* history, bool fast);
}

int ktune_mlp_train(const char* csv_text, int32_t kind, const int32_t* hidden, int32_t n_hidden, int32_t log_inputs,
                    int32_t epochs, double learning_rate, int32_t batch_size, uint64_t seed, double validation_fraction,
                    double* best_val_mse, int32_t* best_epoch, double* history) {
    return mlp_train_impl(csv_text, kind, hidden, n_hidden, log_inputs, epochs, learning_rate, batch_size, seed,
                          validation_fraction, best_val_mse, best_epoch, history, false);
}

int ktune_mlp_train_fast(const char* csv_text, int32_t kind, const int32_t* hidden, int32_t n_hidden,
                         int32_t log_inputs, int32_t epochs, double learning_rate, int32_t batch_size, uint64_t seed,
                         double validation_fraction, double* best_val_mse, int32_t* best_epoch, double* history) {
    return mlp_train_impl(csv_text, kind, hidden, n_hidden, log_inputs, epochs, learning_rate, batch_size, seed,
                          validation_fraction, best_val_mse, best_epoch, history, true);
}

int ktune_mlp_sweep_gemm(const char* model_json, const ktune_hw* hw, const char* bounds_json,
                         const ktune_gemm_input* in, int32_t fast, int64_t* n_candidates, double* device_seconds,
                         double* total_seconds) {
    return guard([&] {
        need(model_json, "model_json");
        const HardwareDescriptor h = conv_hw(hw);
        const std::vector<GemmTuning> legal = enumerate_legal(conv_in(in), h, gemm_bounds(bounds_json));
        MlpPredictor p(MlpModel::from_json_text(model_json), fast != 0);
        std::vector<double> out;
        const auto t0 = std::chrono::steady_clock::now();
        p.predict_gemm(conv_in(in), legal, out);
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (n_candidates) *n_candidates = int64_t(legal.size());
        if (device_seconds) *device_seconds = fast ? p.last_device_seconds() : secs;
        if (total_seconds) *total_seconds = secs;
    });
}

}  // extern "C"

namespace {
int mlp_train_impl(const char* csv_text, int32_t kind, const int32_t* hidden, int32_t n_hidden, int32_t log_inputs,
                   int32_t epochs, double learning_rate, int32_t batch_size, uint64_t seed, double validation_fraction,
                   double* best_val_mse, int32_t* best_epoch, double* history, bool fast) {
    return guard([&] {
        need(csv_text, "csv_text");
        const TrainingSet set = kind == 0 ? to_training_set(gemm_dataset_from_csv_text(csv_text))
                                          : to_training_set(conv_dataset_from_csv_text(csv_text));
        MlpArchitecture arch;
        arch.input_dim = set.dim;
        if (hidden && n_hidden > 0) arch.hidden_sizes.assign(hidden, hidden + n_hidden);
        arch.log_inputs = log_inputs != 0;
        TrainConfig cfg;
        cfg.epochs = epochs;
        cfg.learning_rate = learning_rate;
        cfg.batch_size = batch_size;
        cfg.rng_seed = seed;
        cfg.validation_fraction = validation_fraction;
        cfg.fast = fast;
        TrainResult r = mlp_train(set, arch, cfg);
        if (best_val_mse) *best_val_mse = r.best_val_mse;
        if (best_epoch) *best_epoch = r.best_epoch;
        if (history)
            for (std::size_t e = 0; e < r.history.size(); ++e) {
                history[2 * e] = r.history[e].train_mse;
                history[2 * e + 1] = r.history[e].val_mse;
            }
        MlpModel m;
        m.feature_version = kind == 0 ? kGemmFeatureVersion : kConvFeatureVersion;
        m.weights = r.weights;
        last_text() = m.to_json_text();
    });
}
}  // namespace

extern "C" {

int ktune_mlp_init(int32_t input_dim, const int32_t* hidden, int32_t n_hidden, int32_t log_inputs, uint64_t seed,
                   const char* feature_version) {
    return guard([&] {
        MlpArchitecture arch;
        arch.input_dim = input_dim;
        if (hidden && n_hidden > 0) arch.hidden_sizes.assign(hidden, hidden + n_hidden);
        arch.log_inputs = log_inputs != 0;
        MlpModel m;
        m.feature_version = feature_version ? feature_version : kGemmFeatureVersion;
        m.weights = init_weights(arch, seed);
        last_text() = m.to_json_text();
    });
}

int ktune_mlp_predict_rows(const char* model_json, const double* rows, int64_t n, int32_t dim, double* out) {
    return guard([&] {
        need(model_json, "model_json");
        const MlpModel m = MlpModel::from_json_text(model_json);
        std::vector<std::vector<double>> r(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) r[std::size_t(i)].assign(rows + i * dim, rows + (i + 1) * dim);
        std::vector<double> o;
        m.predict_batch(r, o);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

int ktune_mlp_predict_gemm_fast(const char* model_json, const ktune_gemm_input* in,
                                const ktune_gemm_tuning* tunings, int64_t n, double* out) {
    return guard([&] {
        need(model_json, "model_json");
        MlpPredictor p(MlpModel::from_json_text(model_json), true);
        std::vector<GemmTuning> ts;
        for (int64_t i = 0; i < n; ++i) ts.push_back(conv_t(tunings + i));
        std::vector<double> o;
        p.predict_gemm(conv_in(in), ts, o);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

int ktune_mlp_predict_gemm(const char* model_json, const ktune_gemm_input* in, const ktune_gemm_tuning* tunings,
                           int64_t n, double* out) {
    return guard([&] {
        need(model_json, "model_json");
        MlpPredictor p(MlpModel::from_json_text(model_json));
        std::vector<GemmTuning> ts;
        for (int64_t i = 0; i < n; ++i) ts.push_back(conv_t(tunings + i));
        std::vector<double> o;
        p.predict_gemm(conv_in(in), ts, o);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

int ktune_mlp_predict_conv(const char* model_json, const ktune_conv_input* in, const ktune_conv_tuning* tunings,
                           int64_t n, double* out) {
    return guard([&] {
        need(model_json, "model_json");
        MlpPredictor p(MlpModel::from_json_text(model_json));
        std::vector<ConvTuning> ts;
        for (int64_t i = 0; i < n; ++i) ts.push_back(conv_t(tunings + i));
        std::vector<double> o;
        p.predict_conv(conv_in(in), ts, o);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

int ktune_mlp_evaluate(const char* model_json, const char* csv_text, int32_t kind, double* mse) {
    return guard([&] {
        need(model_json, "model_json");
        need(csv_text, "csv_text");
        need(mse, "mse");
        const MlpModel m = MlpModel::from_json_text(model_json);
        const TrainingSet set = kind == 0 ? to_training_set(gemm_dataset_from_csv_text(csv_text))
                                          : to_training_set(conv_dataset_from_csv_text(csv_text));
        *mse = mlp_evaluate(m.weights, set);
    });
}

int ktune_infer_gemm(const ktune_hw* hw, const char* bounds_json, const char* model_json, const ktune_gemm_input* in,
                     int32_t top_k, int32_t backend, const ktune_measure_options* opts) {
    return guard([&] {
        const HardwareDescriptor h = conv_hw(hw);
        auto be = make_backend(backend, h, opts);
        auto pred = make_predictor(model_json, h);
        last_text() = to_json_text(infer_gemm(*pred, conv_in(in), h, gemm_bounds(bounds_json), top_k, *be));
    });
}

int ktune_infer_conv(const ktune_hw* hw, const char* bounds_json, const char* model_json, const ktune_conv_input* in,
                     int32_t top_k, int32_t backend, const ktune_measure_options* opts) {
    return guard([&] {
        const HardwareDescriptor h = conv_hw(hw);
        auto be = make_backend(backend, h, opts);
        auto pred = make_predictor(model_json, h);
        last_text() = to_json_text(infer_conv(*pred, conv_in(in), h, conv_bounds(bounds_json), top_k, *be));
    });
}

int ktune_infer_gemm_shard(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                           const ktune_gemm_input* in, int32_t top_k, int32_t backend, const ktune_measure_options* opts,
                           int32_t rank, int32_t world, double* gflops_out, int64_t cap, int64_t* count) {
    return guard([&] {
        need(gflops_out, "gflops_out");
        need(count, "count");
        const HardwareDescriptor h = conv_hw(hw);
        auto be = make_backend(backend, h, opts);
        ShardBackend sb(*be, rank, world);
        auto pred = make_predictor(model_json, h);
        (void)infer_gemm(*pred, conv_in(in), h, gemm_bounds(bounds_json), top_k, sb);
        if (int64_t(sb.values.size()) > cap) throw std::invalid_argument("infer shard: cap smaller than top_k");
        std::copy(sb.values.begin(), sb.values.end(), gflops_out);
        *count = int64_t(sb.values.size());
    });
}

int ktune_infer_conv_shard(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                           const ktune_conv_input* in, int32_t top_k, int32_t backend, const ktune_measure_options* opts,
                           int32_t rank, int32_t world, double* gflops_out, int64_t cap, int64_t* count) {
    return guard([&] {
        need(gflops_out, "gflops_out");
        need(count, "count");
        const HardwareDescriptor h = conv_hw(hw);
        auto be = make_backend(backend, h, opts);
        ShardBackend sb(*be, rank, world);
        auto pred = make_predictor(model_json, h);
        (void)infer_conv(*pred, conv_in(in), h, conv_bounds(bounds_json), top_k, sb);
        if (int64_t(sb.values.size()) > cap) throw std::invalid_argument("infer shard: cap smaller than top_k");
        std::copy(sb.values.begin(), sb.values.end(), gflops_out);
        *count = int64_t(sb.values.size());
    });
}

int ktune_infer_gemm_replay(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                            const ktune_gemm_input* in, int32_t top_k, const char* backend_name, const double* gflops,
                            int64_t n) {
    return guard([&] {
        need(gflops, "gflops");
        const HardwareDescriptor h = conv_hw(hw);
        ReplayBackend rb(backend_name ? backend_name : "b200", gflops, n, replay_filter(backend_name, h));
        auto pred = make_predictor(model_json, h);
        last_text() = to_json_text(infer_gemm(*pred, conv_in(in), h, gemm_bounds(bounds_json), top_k, rb));
    });
}

int ktune_infer_conv_replay(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                            const ktune_conv_input* in, int32_t top_k, const char* backend_name, const double* gflops,
                            int64_t n) {
    return guard([&] {
        need(gflops, "gflops");
        const HardwareDescriptor h = conv_hw(hw);
        ReplayBackend rb(backend_name ? backend_name : "b200", gflops, n, replay_filter(backend_name, h));
        auto pred = make_predictor(model_json, h);
        last_text() = to_json_text(infer_conv(*pred, conv_in(in), h, conv_bounds(bounds_json), top_k, rb));
    });
}

int ktune_cache_key_gemm(const ktune_gemm_input* in) {
    return guard([&] { last_text() = cache_key(conv_in(in)); });
}

int ktune_cache_key_conv(const ktune_conv_input* in) {
    return guard([&] { last_text() = cache_key(conv_in(in)); });
}

int ktune_cache_lookup_gemm(const char* dir, const ktune_gemm_input* in, int* found) {
    return guard([&] {
        need(dir, "dir");
        need(found, "found");
        auto r = ResultCache(dir).lookup(conv_in(in));
        *found = r ? 1 : 0;
        last_text() = r ? to_json_text(*r) : std::string();
    });
}

int ktune_cache_lookup_conv(const char* dir, const ktune_conv_input* in, int* found) {
    return guard([&] {
        need(dir, "dir");
        need(found, "found");
        auto r = ResultCache(dir).lookup(conv_in(in));
        *found = r ? 1 : 0;
        last_text() = r ? to_json_text(*r) : std::string();
    });
}

int ktune_cache_store(const char* dir, const char* result_json) {
    return guard([&] {
        need(dir, "dir");
        need(result_json, "result_json");
        const std::string text(result_json);
        if (text.find("\"kind\": \"conv\"") != std::string::npos)
            ResultCache(dir).store(conv_result_from_json_text(text));
        else
            ResultCache(dir).store(gemm_result_from_json_text(text));
    });
}

int ktune_select_gemm(const ktune_hw* hw, const char* bounds_json, const char* model_json, const char* cache_dir,
                      const ktune_gemm_input* in, int32_t top_k, ktune_gemm_tuning* chosen, int32_t* source) {
    return guard([&] {
        need(chosen, "chosen");
        const GemmInput input = conv_in(in);
        // the in-memory argmax is valid only for the configuration that
        // filled it: the key covers the input signature, the hardware
        // descriptor, the bounds, the predictor model and top_k
        const HardwareDescriptor hwd = conv_hw(hw);
        const std::string key = cache_key(input) + "|" + fnv1a64_hex(hwd.to_json_text()) + "|" +
                                fnv1a64_hex(bounds_json ? bounds_json : "") + "|" +
                                fnv1a64_hex(model_json ? model_json : "") + "|" + std::to_string(top_k);
        {
            std::lock_guard<std::mutex> lock(g_select_mu);
            auto it = g_select_memo.find(key);
            if (it != g_select_memo.end()) {
                *chosen = out_t(it->second);
                if (source) *source = 0;
                return;
            }
        }
        std::optional<GemmInferenceResult> r;
        int32_t src = 1;
        if (cache_dir && cache_dir[0]) r = ResultCache(cache_dir).lookup(input);
        if (!r) {
            const HardwareDescriptor h = conv_hw(hw);
            B200Backend be(h);
            auto pred = make_predictor(model_json, h);
            r = infer_gemm(*pred, input, h, gemm_bounds(bounds_json), top_k, be);
            if (cache_dir && cache_dir[0]) ResultCache(cache_dir).store(*r);
            src = 2;
        }
        {
            std::lock_guard<std::mutex> lock(g_select_mu);
            g_select_memo[key] = r->chosen;
        }
        *chosen = out_t(r->chosen);
        if (source) *source = src;
    });
}

int ktune_select_conv(const ktune_hw* hw, const char* bounds_json, const char* model_json, const char* cache_dir,
                      const ktune_conv_input* in, int32_t top_k, ktune_conv_tuning* chosen, int32_t* source) {
    return guard([&] {
        need(chosen, "chosen");
        const ConvInput input = conv_in(in);
        const HardwareDescriptor hwd = conv_hw(hw);
        const std::string key = cache_key(input) + "|" + fnv1a64_hex(hwd.to_json_text()) + "|" +
                                fnv1a64_hex(bounds_json ? bounds_json : "") + "|" +
                                fnv1a64_hex(model_json ? model_json : "") + "|" + std::to_string(top_k);
        {
            std::lock_guard<std::mutex> lock(g_select_mu);
            auto it = g_select_memo_conv.find(key);
            if (it != g_select_memo_conv.end()) {
                *chosen = out_t(it->second);
                if (source) *source = 0;
                return;
            }
        }
        std::optional<ConvInferenceResult> r;
        int32_t src = 1;
        if (cache_dir && cache_dir[0]) r = ResultCache(cache_dir).lookup(input);
        if (!r) {
            B200Backend be(hwd);
            auto pred = make_predictor(model_json, hwd);
            r = infer_conv(*pred, input, hwd, conv_bounds(bounds_json), top_k, be);
            if (cache_dir && cache_dir[0]) ResultCache(cache_dir).store(*r);
            src = 2;
        }
        {
            std::lock_guard<std::mutex> lock(g_select_mu);
            g_select_memo_conv[key] = r->chosen;
        }
        *chosen = out_t(r->chosen);
        if (source) *source = src;
    });
}

}  // extern "C"
