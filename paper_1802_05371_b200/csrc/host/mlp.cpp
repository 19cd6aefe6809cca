// MLP host side: architecture/weights validation, seeded Glorot init, the
// ktune-mlp-1 JSON format, one-row host forward, host evaluation.
// Behavioural contract: /root/reference/proj/src/perf_model.cpp (:17-113,
// :201-290, :399-423 split, :452-518 JSON).  Training and batched
// prediction run on the GPU (kernels/mlp.cu).

#include "ktune/mlp.hpp"

#include <cmath>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "json.hpp"
#include "ktune/sampling.hpp"
#include "ktune/space.hpp"

namespace ktune {

void MlpArchitecture::validate() const {
    if (input_dim < 1) throw std::invalid_argument("architecture input_dim must be >= 1");
    for (int h : hidden_sizes)
        if (h < 1) throw std::invalid_argument("hidden layer sizes must be >= 1");
}

int MlpWeights::input_dim() const {
    if (layers.empty()) throw std::invalid_argument("mlp has no layers");
    return layers.front().in;
}

void MlpWeights::validate() const {
    if (layers.empty()) throw std::invalid_argument("mlp has no layers");
    for (std::size_t l = 0; l < layers.size(); ++l) {
        const auto& L = layers[l];
        if (L.in < 1 || L.out < 1) throw std::invalid_argument("mlp layer with empty dimension");
        if (L.w.size() != std::size_t(L.in) * std::size_t(L.out) || L.b.size() != std::size_t(L.out))
            throw std::invalid_argument("mlp layer weight shape mismatch");
        if (l + 1 < layers.size() && layers[l + 1].in != L.out)
            throw std::invalid_argument("mlp layer widths do not chain");
    }
    if (layers.back().out != 1) throw std::invalid_argument("mlp output layer must have one unit");
}

MlpWeights init_weights(const MlpArchitecture& arch, std::uint64_t seed) {
    arch.validate();
    MlpWeights w;
    w.log_inputs = arch.log_inputs;
    std::mt19937_64 rng(seed);
    std::vector<int> widths{arch.input_dim};
    widths.insert(widths.end(), arch.hidden_sizes.begin(), arch.hidden_sizes.end());
    widths.push_back(1);
    for (std::size_t l = 0; l + 1 < widths.size(); ++l) {
        MlpLayer L;
        L.in = widths[l];
        L.out = widths[l + 1];
        const double bound = std::sqrt(6.0 / double(L.in + L.out));
        L.w.resize(std::size_t(L.in) * std::size_t(L.out));
        for (double& x : L.w) x = (2.0 * unit_real(rng) - 1.0) * bound;
        L.b.assign(std::size_t(L.out), 0.0);
        w.layers.push_back(std::move(L));
    }
    return w;
}

namespace {

void log_row(const MlpWeights& w, std::span<const double> x, std::vector<double>& out) {
    out.assign(x.begin(), x.end());
    if (!w.log_inputs) return;
    for (double& v : out) {
        if (!(v > 0.0)) throw std::invalid_argument("features must be strictly positive under the log transform");
        v = std::log(v);
    }
}

double host_forward(const MlpWeights& w, std::vector<double> a) {
    std::vector<double> z;
    for (std::size_t l = 0; l < w.layers.size(); ++l) {
        const auto& L = w.layers[l];
        z.assign(std::size_t(L.out), 0.0);
        for (int o = 0; o < L.out; ++o) {
            double acc = L.b[std::size_t(o)];
            const double* wr = L.w.data() + std::size_t(o) * L.in;
            for (int i = 0; i < L.in; ++i) {
                const double prod = a[std::size_t(i)] * wr[i];
                acc = acc + prod;
            }
            z[std::size_t(o)] = acc;
        }
        if (l + 1 < w.layers.size())
            for (auto& v : z) v = v > 0.0 ? v : 0.0;
        a.swap(z);
    }
    return a[0];
}

}  // namespace

double mlp_forward(const MlpWeights& w, std::span<const double> features) {
    w.validate();
    if (int(features.size()) != w.input_dim()) throw std::invalid_argument("feature vector has wrong dimension");
    std::vector<double> a;
    log_row(w, features, a);
    return host_forward(w, std::move(a));
}

void TrainingSet::add(std::span<const double> x, double y) {
    if (dim == 0) dim = int(x.size());
    if (int(x.size()) != dim) throw std::invalid_argument("training row has wrong dimension");
    features.insert(features.end(), x.begin(), x.end());
    targets.push_back(y);
}

void TrainingSet::validate() const {
    if (dim < 1 || targets.empty() || features.size() != targets.size() * std::size_t(dim))
        throw std::invalid_argument("training set is empty or inconsistent");
}

double mlp_evaluate(const MlpWeights& w, const TrainingSet& data) {
    w.validate();
    data.validate();
    if (data.dim != w.input_dim()) throw std::invalid_argument("dataset dimension does not match the model");
    long double acc = 0.0L;
    std::vector<double> a;
    for (std::size_t i = 0; i < data.size(); ++i) {
        log_row(w, data.row(i), a);
        const long double e = host_forward(w, a) - data.targets[i];
        acc += e * e;
    }
    return double(acc / (long double)(data.size()));
}

void TrainConfig::validate() const {
    if (learning_rate <= 0 || batch_size < 1 || epochs < 1 || validation_fraction <= 0.0 ||
        validation_fraction >= 1.0 || clip_grad_norm <= 0.0)
        throw std::invalid_argument("bad training configuration");
}

double MlpModel::predict(std::span<const double> features) const { return mlp_forward(weights, features); }

std::string MlpModel::to_json_text() const {
    weights.validate();
    nlohmann::json j;
    j["format"] = "ktune-mlp-1";
    j["feature_version"] = feature_version;
    j["log_inputs"] = weights.log_inputs;
    j["layers"] = nlohmann::json::array();
    for (const auto& L : weights.layers) j["layers"].push_back({{"in", L.in}, {"out", L.out}, {"w", L.w}, {"b", L.b}});
    return j.dump() + "\n";
}

MlpModel MlpModel::from_json_text(const std::string& text) {
    nlohmann::json j = nlohmann::json::parse(text, nullptr, false);
    if (j.is_discarded()) throw std::runtime_error("malformed JSON in model file");
    MlpModel m;
    try {
        if (j.at("format").get<std::string>() != "ktune-mlp-1") throw std::runtime_error("unsupported model format");
        m.feature_version = j.at("feature_version").get<std::string>();
        m.weights.log_inputs = j.at("log_inputs").get<bool>();
        for (const auto& jl : j.at("layers")) {
            MlpLayer L;
            L.in = jl.at("in").get<int>();
            L.out = jl.at("out").get<int>();
            L.w = jl.at("w").get<std::vector<double>>();
            L.b = jl.at("b").get<std::vector<double>>();
            m.weights.layers.push_back(std::move(L));
        }
    } catch (const nlohmann::json::exception& e) {
        throw std::runtime_error(std::string("bad model file: ") + e.what());
    }
    m.weights.validate();
    return m;
}

void MlpModel::save(const std::string& path) const {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot write model file: " + path);
    out << to_json_text();
    if (!out) throw std::runtime_error("write failed: " + path);
}

MlpModel MlpModel::load(const std::string& path) {
    std::string text;
    try {
        text = read_text_file(path);
    } catch (const std::exception&) {
        throw std::runtime_error("cannot open model file: " + path);
    }
    try {
        return from_json_text(text);
    } catch (const std::exception& e) {
        throw std::runtime_error("model file " + path + ": " + e.what());
    }
}

TrainResult mlp_train(const TrainingSet& all, const MlpArchitecture& arch, const TrainConfig& cfg) {
    cfg.validate();
    all.validate();
    const std::size_t n = all.size();
    std::size_t n_val = std::size_t(std::llround(double(n) * cfg.validation_fraction));
    n_val = std::max<std::size_t>(1, std::min(n - 1, n_val));
    if (n < 2) throw std::invalid_argument("need at least two rows to split off validation");
    std::vector<std::size_t> perm(n);
    for (std::size_t i = 0; i < n; ++i) perm[i] = i;
    std::mt19937_64 rng(cfg.rng_seed ^ 0x9e3779b97f4a7c15ULL);
    for (std::size_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[index_below(rng, i)]);
    TrainingSet train, val;
    for (std::size_t i = 0; i < n; ++i) (i + n_val < n ? train : val).add(all.row(perm[i]), all.targets[perm[i]]);
    return mlp_train(train, val, arch, cfg);
}

}  // namespace ktune
