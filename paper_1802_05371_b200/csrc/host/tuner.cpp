// The tuning pipeline.  Behavioural contract: /root/reference/proj/src/
// pipeline.cpp (CSV :20-327, distributions :332-457, generation :463-556,
// predictors :562-616, inference :626-723, result JSON + cache :729-997).
// Formats are byte-identical (std::to_chars shortest doubles; nlohmann
// dump(2)); seeded sequences are bit-identical.

#include "ktune/tuner.hpp"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <map>
#include <fstream>
#include <numeric>
#include <set>
#include <sstream>
#include <stdexcept>

#include "json.hpp"

namespace ktune {

namespace {

using nlohmann::json;

std::string fmt_double(double v) {
    char buf[64];
    auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), v);
    if (ec != std::errc()) throw std::runtime_error("cannot format floating-point value");
    return std::string(buf, end);
}

template <typename T>
T parse_number(const std::string& s, const char* kind) {
    T v{};
    auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc() || end != s.data() + s.size())
        throw std::runtime_error(std::string("bad ") + kind + " field: '" + s + "'");
    return v;
}

bool parse_flag(const std::string& s) {
    if (s == "0") return false;
    if (s == "1") return true;
    throw std::runtime_error("bad boolean field: '" + s + "'");
}

std::vector<std::string> split_commas(const std::string& line) {
    std::vector<std::string> out(1);
    for (char c : line) {
        if (c == ',') out.emplace_back();
        else out.back().push_back(c);
    }
    return out;
}

void check_tag(const std::string& tag) {
    if (tag.empty() || tag.find(',') != std::string::npos || tag.find('\n') != std::string::npos)
        throw std::invalid_argument("backend tag unfit for CSV: '" + tag + "'");
}

std::int64_t wall_ms() {
    return std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::system_clock::now().time_since_epoch())
        .count();
}

std::string key_of(const GemmInput& in, const GemmTuning& t) {
    std::ostringstream k;
    k << in.m << '|' << in.n << '|' << in.k << '|' << to_string(in.dtype) << '|' << in.trans_a << '|' << in.trans_b;
    for (int v : to_values(t)) k << '|' << v;
    return k.str();
}

std::string key_of(const ConvInput& in, const ConvTuning& t) {
    std::ostringstream k;
    k << in.n_batch << '|' << in.p << '|' << in.q << '|' << in.k_filters << '|' << in.c << '|' << in.r << '|' << in.s
      << '|' << to_string(in.dtype);
    for (int v : to_values(t)) k << '|' << v;
    return k.str();
}

constexpr int kDuplicateRedrawLimit = 10000;

std::vector<std::vector<std::string>> csv_rows(const std::string& text, const char* header, std::size_t cols) {
    std::istringstream in(text);
    std::string line;
    if (!std::getline(in, line)) throw std::runtime_error("dataset is empty: missing header row");
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line != header)
        throw std::runtime_error("dataset header mismatch (wrong problem kind or schema): got '" + line + "'");
    std::vector<std::vector<std::string>> rows;
    std::size_t line_no = 1;
    while (std::getline(in, line)) {
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        auto f = split_commas(line);
        if (f.size() != cols)
            throw std::runtime_error("dataset line " + std::to_string(line_no) + ": expected " + std::to_string(cols) +
                                     " columns, got " + std::to_string(f.size()));
        rows.push_back(std::move(f));
    }
    return rows;
}

template <typename Sample>
void check_measured(const Sample& s) {
    if (!(std::isfinite(s.gflops) && s.gflops > 0.0)) throw std::runtime_error("dataset row with non-positive gflops");
}

template <typename DS>
void validate_rows(const DS& ds, const HardwareDescriptor& hw) {
    std::set<std::string> seen;
    for (std::size_t i = 0; i < ds.samples.size(); ++i) {
        const auto& s = ds.samples[i];
        if (auto v = is_legal(s.input, s.tuning, hw); !v)
            throw std::runtime_error("dataset row " + std::to_string(i) + " is illegal: " + v.detail);
        if (!(std::isfinite(s.gflops) && s.gflops > 0.0))
            throw std::runtime_error("dataset row " + std::to_string(i) + " has non-positive gflops");
        if (!seen.insert(key_of(s.input, s.tuning)).second)
            throw std::runtime_error("dataset row " + std::to_string(i) + " duplicates an earlier (input, tuning)");
    }
}

void weights_ok(std::size_t n, const std::vector<double>& w) {
    if (w.empty()) return;
    if (w.size() != n) throw std::invalid_argument("weights must parallel the shape list");
    double total = 0.0;
    for (double x : w) {
        if (!(x >= 0.0) || !std::isfinite(x)) throw std::invalid_argument("shape weights must be finite and >= 0");
        total += x;
    }
    if (!(total > 0.0)) throw std::invalid_argument("shape weights must have positive mass");
}

std::size_t pick_shape(std::mt19937_64& rng, std::size_t n, const std::vector<double>& w) {
    if (w.empty()) return index_below(rng, n);
    double total = 0.0;
    for (double x : w) total += x;
    const double x = unit_real(rng) * total;
    double acc = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        acc += w[i];
        if (x < acc) return i;
    }
    return n - 1;
}

// The shared sample -> dedup loop of generate_*_dataset; `emit` receives
// each distinct pair in order.
// `accept` (may be empty) is the measuring backend's launchability filter:
// rejected draws are redrawn and counted, never measured.
constexpr int kUnlaunchableRedrawLimit = 1000000;

template <typename In, typename Tu, typename Dist, typename Bounds, typename FromValues, typename Emit,
          typename Accept>
void draw_distinct(const CategoricalModel& model, const Dist& dist, const Bounds& bounds, const HardwareDescriptor& hw,
                   int n_samples, std::uint64_t seed, GenerateReport* report, FromValues from_values, Emit emit,
                   const Accept& accept) {
    if (n_samples < 1) throw std::invalid_argument("n_samples must be >= 1");
    dist.validate();
    model.validate();
    bounds.validate();
    std::mt19937_64 rng(seed);
    std::set<std::string> seen;
    GenerateReport rep;
    int consecutive = 0;
    int unlaunchable_run = 0;
    int produced = 0;
    while (produced < n_samples) {
        const In input = dist.draw(rng);
        const auto legal = make_legality(input, hw);
        const std::vector<int> vals = sample(model, legal, rng);
        ++rep.attempts;
        const Tu tuning = from_values(vals);
        if (accept && !accept(input, tuning)) {
            ++rep.unlaunchable_rejected;
            if (++unlaunchable_run > kUnlaunchableRedrawLimit)
                throw std::runtime_error("dataset generation stalled: " + std::to_string(kUnlaunchableRedrawLimit) +
                                         " consecutive draws the backend cannot launch");
            continue;
        }
        unlaunchable_run = 0;
        if (!seen.insert(key_of(input, tuning)).second) {
            ++rep.duplicates_rejected;
            if (++consecutive > kDuplicateRedrawLimit)
                throw std::runtime_error("dataset generation stalled: " + std::to_string(kDuplicateRedrawLimit) +
                                         " consecutive duplicate draws — space too small for " +
                                         std::to_string(n_samples) + " distinct samples");
            continue;
        }
        consecutive = 0;
        emit(input, tuning);
        ++produced;
    }
    if (report) *report = rep;
}

}  // namespace

// ---------------------------------------------------------------------------
// CSV
// ---------------------------------------------------------------------------

std::string to_csv_text(const GemmDataset& ds) {
    std::ostringstream out;
    out << kGemmCsvHeader << '\n';
    for (const auto& s : ds.samples) {
        check_tag(s.backend);
        out << s.input.m << ',' << s.input.n << ',' << s.input.k << ',' << to_string(s.input.dtype) << ','
            << int(s.input.trans_a) << ',' << int(s.input.trans_b);
        for (int v : to_values(s.tuning)) out << ',' << v;
        out << ',' << fmt_double(s.gflops) << ',' << s.backend << '\n';
    }
    return out.str();
}

std::string to_csv_text(const ConvDataset& ds) {
    std::ostringstream out;
    out << kConvCsvHeader << '\n';
    for (const auto& s : ds.samples) {
        check_tag(s.backend);
        out << s.input.n_batch << ',' << s.input.p << ',' << s.input.q << ',' << s.input.k_filters << ',' << s.input.c
            << ',' << s.input.r << ',' << s.input.s << ',' << to_string(s.input.dtype);
        for (int v : to_values(s.tuning)) out << ',' << v;
        out << ',' << fmt_double(s.gflops) << ',' << s.backend << '\n';
    }
    return out.str();
}

GemmDataset gemm_dataset_from_csv_text(const std::string& text) {
    GemmDataset ds;
    for (const auto& f : csv_rows(text, kGemmCsvHeader, 16)) {
        GemmSample s;
        s.input.m = parse_number<int>(f[0], "integer");
        s.input.n = parse_number<int>(f[1], "integer");
        s.input.k = parse_number<int>(f[2], "integer");
        s.input.dtype = dtype_from_string(f[3]);
        s.input.trans_a = parse_flag(f[4]);
        s.input.trans_b = parse_flag(f[5]);
        std::vector<int> v(8);
        for (int i = 0; i < 8; ++i) v[std::size_t(i)] = parse_number<int>(f[std::size_t(6 + i)], "integer");
        s.tuning = gemm_tuning_from_values(v);
        s.gflops = parse_number<double>(f[14], "numeric");
        s.backend = f[15];
        s.input.validate();
        s.tuning.validate();
        check_measured(s);
        ds.samples.push_back(std::move(s));
    }
    return ds;
}

ConvDataset conv_dataset_from_csv_text(const std::string& text) {
    ConvDataset ds;
    for (const auto& f : csv_rows(text, kConvCsvHeader, 22)) {
        ConvSample s;
        std::int64_t* dims[] = {&s.input.n_batch, &s.input.p, &s.input.q, &s.input.k_filters,
                                &s.input.c,       &s.input.r, &s.input.s};
        for (int i = 0; i < 7; ++i) *dims[i] = parse_number<int>(f[std::size_t(i)], "integer");
        s.input.dtype = dtype_from_string(f[7]);
        std::vector<int> v(12);
        for (int i = 0; i < 12; ++i) v[std::size_t(i)] = parse_number<int>(f[std::size_t(8 + i)], "integer");
        s.tuning = conv_tuning_from_values(v);
        s.gflops = parse_number<double>(f[20], "numeric");
        s.backend = f[21];
        s.input.validate();
        s.tuning.validate();
        check_measured(s);
        ds.samples.push_back(std::move(s));
    }
    return ds;
}

void save_gemm_dataset(const GemmDataset& ds, const std::string& path) { write_text_file_atomic(path, to_csv_text(ds)); }
void save_conv_dataset(const ConvDataset& ds, const std::string& path) { write_text_file_atomic(path, to_csv_text(ds)); }

GemmDataset load_gemm_dataset(const std::string& path) {
    std::string text;
    try {
        text = read_text_file(path);
    } catch (const std::exception&) {
        throw std::runtime_error(path + ": cannot open dataset: " + path);
    }
    try {
        return gemm_dataset_from_csv_text(text);
    } catch (const std::runtime_error& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
}

ConvDataset load_conv_dataset(const std::string& path) {
    std::string text;
    try {
        text = read_text_file(path);
    } catch (const std::exception&) {
        throw std::runtime_error(path + ": cannot open dataset: " + path);
    }
    try {
        return conv_dataset_from_csv_text(text);
    } catch (const std::runtime_error& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
}

void validate_dataset(const GemmDataset& ds, const HardwareDescriptor& hw) { validate_rows(ds, hw); }
void validate_dataset(const ConvDataset& ds, const HardwareDescriptor& hw) { validate_rows(ds, hw); }

TrainingSet to_training_set(const GemmDataset& ds) {
    TrainingSet set;
    for (const auto& s : ds.samples) set.add(encode_features(s.input, s.tuning), std::log(s.gflops));
    return set;
}

TrainingSet to_training_set(const ConvDataset& ds) {
    TrainingSet set;
    for (const auto& s : ds.samples) set.add(encode_features(s.input, s.tuning), std::log(s.gflops));
    return set;
}

// ---------------------------------------------------------------------------
// input distributions
// ---------------------------------------------------------------------------

int log_uniform_int(std::mt19937_64& rng, int lo, int hi) {
    if (lo < 1 || hi < lo) throw std::invalid_argument("log-uniform range must satisfy 1 <= lo <= hi");
    const double a = std::log(double(lo));
    const double b = std::log(double(hi) + 1.0);
    const int v = int(std::floor(std::exp(a + unit_real(rng) * (b - a))));
    return std::clamp(v, lo, hi);
}

void GemmInputDistribution::validate() const {
    if (shapes.empty() && !use_ranges) throw std::invalid_argument("distribution has neither shapes nor ranges");
    for (const auto& s : shapes) s.validate();
    weights_ok(shapes.size(), weights);
    if (!(fixed_fraction >= 0.0 && fixed_fraction <= 1.0))
        throw std::invalid_argument("fixed_fraction must lie in [0, 1]");
    if (use_ranges && (m_lo < 1 || m_hi < m_lo || n_lo < 1 || n_hi < n_lo || k_lo < 1 || k_hi < k_lo))
        throw std::invalid_argument("bad shape ranges");
}

GemmInput GemmInputDistribution::draw(std::mt19937_64& rng) const {
    bool from_list = !shapes.empty();
    if (from_list && use_ranges) from_list = unit_real(rng) < fixed_fraction;
    if (from_list) return shapes[pick_shape(rng, shapes.size(), weights)];
    GemmInput in;
    in.m = log_uniform_int(rng, m_lo, m_hi);
    in.n = log_uniform_int(rng, n_lo, n_hi);
    in.k = log_uniform_int(rng, k_lo, k_hi);
    in.dtype = dtype;
    if (randomize_transpose) {
        in.trans_a = index_below(rng, 2) == 1;
        in.trans_b = index_below(rng, 2) == 1;
    }
    return in;
}

void ConvInputDistribution::validate() const {
    if (shapes.empty() && !use_ranges) throw std::invalid_argument("distribution has neither shapes nor ranges");
    for (const auto& s : shapes) s.validate();
    weights_ok(shapes.size(), weights);
    if (!(fixed_fraction >= 0.0 && fixed_fraction <= 1.0))
        throw std::invalid_argument("fixed_fraction must lie in [0, 1]");
    if (use_ranges) {
        if (n_lo < 1 || n_hi < n_lo || p_lo < 1 || p_hi < p_lo || q_lo < 1 || q_hi < q_lo || k_lo < 1 || k_hi < k_lo ||
            c_lo < 1 || c_hi < c_lo)
            throw std::invalid_argument("bad shape ranges");
        if (rs_choices.empty()) throw std::invalid_argument("rs_choices must not be empty");
        for (auto [r, s] : rs_choices)
            if (r < 1 || s < 1) throw std::invalid_argument("filter sizes must be >= 1");
    }
}

ConvInput ConvInputDistribution::draw(std::mt19937_64& rng) const {
    bool from_list = !shapes.empty();
    if (from_list && use_ranges) from_list = unit_real(rng) < fixed_fraction;
    if (from_list) return shapes[pick_shape(rng, shapes.size(), weights)];
    ConvInput in;
    in.n_batch = log_uniform_int(rng, n_lo, n_hi);
    in.p = log_uniform_int(rng, p_lo, p_hi);
    in.q = log_uniform_int(rng, q_lo, q_hi);
    in.k_filters = log_uniform_int(rng, k_lo, k_hi);
    in.c = log_uniform_int(rng, c_lo, c_hi);
    const auto [r, s] = rs_choices[index_below(rng, rs_choices.size())];
    in.r = r;
    in.s = s;
    in.dtype = dtype;
    return in;
}

// ---------------------------------------------------------------------------
// generation
// ---------------------------------------------------------------------------

std::vector<GemmDraw> predraw_gemm(const CategoricalModel& model, const GemmInputDistribution& dist,
                                   const GemmBounds& bounds, const HardwareDescriptor& hw, int n_samples,
                                   std::uint64_t seed, GenerateReport* report, const GemmAccept& accept) {
    std::vector<GemmDraw> out;
    out.reserve(std::size_t(std::max(n_samples, 0)));
    draw_distinct<GemmInput, GemmTuning>(model, dist, bounds, hw, n_samples, seed, report, gemm_tuning_from_values,
                                         [&](const GemmInput& in, const GemmTuning& t) { out.push_back({in, t}); },
                                         accept);
    return out;
}

std::vector<ConvDraw> predraw_conv(const CategoricalModel& model, const ConvInputDistribution& dist,
                                   const ConvBounds& bounds, const HardwareDescriptor& hw, int n_samples,
                                   std::uint64_t seed, GenerateReport* report, const ConvAccept& accept) {
    std::vector<ConvDraw> out;
    out.reserve(std::size_t(std::max(n_samples, 0)));
    draw_distinct<ConvInput, ConvTuning>(model, dist, bounds, hw, n_samples, seed, report, conv_tuning_from_values,
                                         [&](const ConvInput& in, const ConvTuning& t) { out.push_back({in, t}); },
                                         accept);
    return out;
}

std::vector<std::vector<std::int64_t>> shard_lpt(const std::vector<double>& costs, int world) {
    if (world < 1) throw std::invalid_argument("shard_lpt: world size must be >= 1");
    std::vector<std::int64_t> order(costs.size());
    std::iota(order.begin(), order.end(), std::int64_t(0));
    std::stable_sort(order.begin(), order.end(), [&](std::int64_t a, std::int64_t b) { return costs[a] > costs[b]; });
    std::vector<double> load(static_cast<std::size_t>(world), 0.0);
    std::vector<std::vector<std::int64_t>> shards(static_cast<std::size_t>(world));
    for (std::int64_t i : order) {
        const auto r = std::size_t(std::min_element(load.begin(), load.end()) - load.begin());
        shards[r].push_back(i);
        load[r] += costs[std::size_t(i)];
    }
    for (auto& sh : shards) std::sort(sh.begin(), sh.end());
    return shards;
}

namespace {

double flops_of(const GemmInput& in) { return 2.0 * double(in.m) * double(in.n) * double(in.k); }
double flops_of(const ConvInput& in) {
    return 2.0 * double(in.n_batch) * double(in.p) * double(in.q) * double(in.k_filters) * double(in.c) *
           double(in.r) * double(in.s);
}

// Checkpoint of one rank: a header line, then "index,gflops" per measured
// sample, appended batch by batch (a killed run resumes where it stopped).
std::string shard_header(const char* kind, int rank, int world, int n, std::uint64_t seed, const MeasureOptions& o) {
    std::ostringstream h;
    h << "ktune-shard-1 " << kind << " rank=" << rank << " world=" << world << " n=" << n << " seed=" << seed
      << " mode=" << int(o.mode) << " reps=" << o.repetitions;
    return h.str();
}

std::map<std::int64_t, double> read_checkpoint(const std::string& path, const std::string& header) {
    std::map<std::int64_t, double> done;
    if (path.empty() || !std::filesystem::exists(path)) return done;
    std::ifstream in(path);
    std::string line;
    if (!std::getline(in, line) || line != header)
        throw std::runtime_error("checkpoint " + path + " belongs to a different run (header mismatch)");
    while (std::getline(in, line)) {
        const auto comma = line.find(',');
        if (comma == std::string::npos) continue;  // a torn last line of a killed run
        try {
            done[std::stoll(line.substr(0, comma))] = std::stod(line.substr(comma + 1));
        } catch (const std::exception&) {
            continue;
        }
    }
    return done;
}

template <typename Draw, typename MeasureMany>
std::vector<ShardRecord> run_shard(const char* kind, const std::vector<Draw>& draws, int n_samples,
                                   std::uint64_t seed, int rank, int world, const MeasureOptions& opt,
                                   const std::string& checkpoint, MeasureMany measure_many) {
    if (rank < 0 || rank >= world) throw std::invalid_argument("shard: rank must lie in [0, world)");
    std::vector<double> cost(draws.size());
    for (std::size_t i = 0; i < draws.size(); ++i) cost[i] = flops_of(draws[i].input);
    const auto shards = shard_lpt(cost, world);
    const std::string header = shard_header(kind, rank, world, n_samples, seed, opt);
    std::map<std::int64_t, double> done = read_checkpoint(checkpoint, header);
    std::vector<std::int64_t> todo;
    for (std::int64_t i : shards[std::size_t(rank)])
        if (!done.count(i)) todo.push_back(i);
    std::ofstream ck;
    if (!checkpoint.empty()) {
        const bool fresh = !std::filesystem::exists(checkpoint) || done.empty();
        ck.open(checkpoint, fresh ? std::ios::trunc : std::ios::app);
        if (!ck) throw std::runtime_error("cannot write checkpoint " + checkpoint);
        if (fresh) ck << header << '\n' << std::flush;
    }
    constexpr std::size_t kBatch = 64;
    for (std::size_t b = 0; b < todo.size(); b += kBatch) {
        const std::size_t e = std::min(todo.size(), b + kBatch);
        std::vector<std::int64_t> idx(todo.begin() + std::ptrdiff_t(b), todo.begin() + std::ptrdiff_t(e));
        const std::vector<double> g = measure_many(idx);
        for (std::size_t j = 0; j < idx.size(); ++j) {
            done[idx[j]] = g[j];
            if (ck.is_open()) ck << idx[j] << ',' << fmt_double(g[j]) << '\n';
        }
        if (ck.is_open()) ck << std::flush;
    }
    std::vector<ShardRecord> out;
    for (std::int64_t i : shards[std::size_t(rank)]) out.push_back({i, done.at(i)});
    return out;
}

}  // namespace

std::vector<ShardRecord> generate_gemm_shard(const CategoricalModel& model, const GemmInputDistribution& dist,
                                             const GemmBounds& bounds, const HardwareDescriptor& hw, int n_samples,
                                             std::uint64_t seed, int rank, int world, const MeasureOptions& opt,
                                             const std::string& checkpoint, std::vector<GemmDraw>* draws,
                                             GenerateReport* report) {
    B200Backend backend(hw, opt);
    auto seq = predraw_gemm(model, dist, bounds, hw, n_samples, seed, report,
                            GemmAccept([&](const GemmInput& in, const GemmTuning& t) { return backend.accepts(in, t); }));
    auto recs = run_shard("gemm", seq, n_samples, seed, rank, world, opt, checkpoint,
                          [&](const std::vector<std::int64_t>& idx) {
                              std::vector<GemmInput> in;
                              std::vector<GemmTuning> tu;
                              for (std::int64_t i : idx) {
                                  in.push_back(seq[std::size_t(i)].input);
                                  tu.push_back(seq[std::size_t(i)].tuning);
                              }
                              return measure_gemm_many(hw, in, tu, opt);
                          });
    if (draws) *draws = std::move(seq);
    return recs;
}

std::vector<ShardRecord> generate_conv_shard(const CategoricalModel& model, const ConvInputDistribution& dist,
                                             const ConvBounds& bounds, const HardwareDescriptor& hw, int n_samples,
                                             std::uint64_t seed, int rank, int world, const MeasureOptions& opt,
                                             const std::string& checkpoint, std::vector<ConvDraw>* draws,
                                             GenerateReport* report) {
    B200Backend backend(hw, opt);
    auto seq = predraw_conv(model, dist, bounds, hw, n_samples, seed, report,
                            ConvAccept([&](const ConvInput& in, const ConvTuning& t) { return backend.accepts(in, t); }));
    auto recs = run_shard("conv", seq, n_samples, seed, rank, world, opt, checkpoint,
                          [&](const std::vector<std::int64_t>& idx) {
                              std::vector<ConvInput> in;
                              std::vector<ConvTuning> tu;
                              for (std::int64_t i : idx) {
                                  in.push_back(seq[std::size_t(i)].input);
                                  tu.push_back(seq[std::size_t(i)].tuning);
                              }
                              return measure_conv_many(hw, in, tu, opt);
                          });
    if (draws) *draws = std::move(seq);
    return recs;
}

GemmDataset generate_gemm_dataset(MeasurementBackend& backend, const CategoricalModel& sampler_model,
                                  const GemmInputDistribution& dist, const GemmBounds& bounds,
                                  const HardwareDescriptor& hw, int n_samples, std::uint64_t seed,
                                  GenerateReport* report) {
    GemmDataset ds;
    draw_distinct<GemmInput, GemmTuning>(
        sampler_model, dist, bounds, hw, n_samples, seed, report, gemm_tuning_from_values,
        [&](const GemmInput& in, const GemmTuning& t) {
            const double g = backend.measure(in, t);
            if (!(std::isfinite(g) && g > 0.0)) throw std::runtime_error("backend returned non-positive gflops");
            ds.samples.push_back({in, t, g, backend.name(), wall_ms()});
        },
        GemmAccept([&](const GemmInput& in, const GemmTuning& t) { return backend.accepts(in, t); }));
    return ds;
}

ConvDataset generate_conv_dataset(MeasurementBackend& backend, const CategoricalModel& sampler_model,
                                  const ConvInputDistribution& dist, const ConvBounds& bounds,
                                  const HardwareDescriptor& hw, int n_samples, std::uint64_t seed,
                                  GenerateReport* report) {
    ConvDataset ds;
    draw_distinct<ConvInput, ConvTuning>(
        sampler_model, dist, bounds, hw, n_samples, seed, report, conv_tuning_from_values,
        [&](const ConvInput& in, const ConvTuning& t) {
            const double g = backend.measure(in, t);
            if (!(std::isfinite(g) && g > 0.0)) throw std::runtime_error("backend returned non-positive gflops");
            ds.samples.push_back({in, t, g, backend.name(), wall_ms()});
        },
        ConvAccept([&](const ConvInput& in, const ConvTuning& t) { return backend.accepts(in, t); }));
    return ds;
}

AnalyticalBackend::AnalyticalBackend(HardwareDescriptor hw) : hw_(std::move(hw)) { hw_.validate(); }
double AnalyticalBackend::measure(const GemmInput& in, const GemmTuning& t) { return analytical_gflops(in, t, hw_); }
double AnalyticalBackend::measure(const ConvInput& in, const ConvTuning& t) { return analytical_gflops(in, t, hw_); }

// ---------------------------------------------------------------------------
// predictors
// ---------------------------------------------------------------------------

MlpPredictor::MlpPredictor(MlpModel model, bool fast) : model_(std::move(model)), fast_(fast) {
    model_.weights.validate();
}
std::string MlpPredictor::name() const { return "mlp"; }

void MlpPredictor::predict_gemm(const GemmInput& input, const std::vector<GemmTuning>& tunings,
                                std::vector<double>& out) const {
    if (model_.feature_version != kGemmFeatureVersion)
        throw std::invalid_argument("model encodes '" + model_.feature_version + "', expected '" +
                                    kGemmFeatureVersion + "'");
    input.validate();
    std::vector<std::int32_t> flat;
    flat.reserve(tunings.size() * 8);
    for (const auto& t : tunings) {
        t.validate();
        for (int v : to_values(t)) flat.push_back(v);
    }
    const std::vector<double> head{double(input.m), double(input.n), double(input.k),
                                   double(dtype_size_bytes(input.dtype)), input.trans_a ? 2.0 : 1.0,
                                   input.trans_b ? 2.0 : 1.0};
    out.resize(tunings.size());
    if (fast_) mlp_predict_tuples_fast(model_.weights, head, flat.data(), std::int64_t(tunings.size()), 8, out.data(),
                                       &last_device_s_);
    else mlp_predict_tuples(model_.weights, head, flat.data(), std::int64_t(tunings.size()), 8, out.data());
}

void MlpPredictor::predict_conv(const ConvInput& input, const std::vector<ConvTuning>& tunings,
                                std::vector<double>& out) const {
    if (model_.feature_version != kConvFeatureVersion)
        throw std::invalid_argument("model encodes '" + model_.feature_version + "', expected '" +
                                    kConvFeatureVersion + "'");
    input.validate();
    std::vector<std::int32_t> flat;
    flat.reserve(tunings.size() * 12);
    for (const auto& t : tunings) {
        t.validate();
        for (int v : to_values(t)) flat.push_back(v);
    }
    const std::vector<double> head{double(input.n_batch), double(input.p), double(input.q), double(input.k_filters),
                                   double(input.c),       double(input.r), double(input.s)};
    out.resize(tunings.size());
    if (fast_) mlp_predict_tuples_fast(model_.weights, head, flat.data(), std::int64_t(tunings.size()), 12, out.data(),
                                       &last_device_s_);
    else mlp_predict_tuples(model_.weights, head, flat.data(), std::int64_t(tunings.size()), 12, out.data());
}

AnalyticalPredictor::AnalyticalPredictor(HardwareDescriptor hw) : hw_(std::move(hw)) { hw_.validate(); }
std::string AnalyticalPredictor::name() const { return "analytical-oracle"; }

void AnalyticalPredictor::predict_gemm(const GemmInput& input, const std::vector<GemmTuning>& tunings,
                                       std::vector<double>& out) const {
    out.resize(tunings.size());
    for (std::size_t i = 0; i < tunings.size(); ++i) out[i] = std::log(analytical_gflops(input, tunings[i], hw_));
}

void AnalyticalPredictor::predict_conv(const ConvInput& input, const std::vector<ConvTuning>& tunings,
                                       std::vector<double>& out) const {
    out.resize(tunings.size());
    for (std::size_t i = 0; i < tunings.size(); ++i) out[i] = std::log(analytical_gflops(input, tunings[i], hw_));
}

// ---------------------------------------------------------------------------
// inference
// ---------------------------------------------------------------------------

namespace {

// k best predictions, ties broken by the lexicographic tuning vector.
template <typename Tuning>
std::vector<std::size_t> best_k(const std::vector<Tuning>& tunings, const std::vector<double>& pred, std::size_t k) {
    std::vector<std::vector<int>> vals;
    vals.reserve(tunings.size());
    for (const auto& t : tunings) vals.push_back(to_values(t));
    std::vector<std::size_t> order(tunings.size());
    std::iota(order.begin(), order.end(), std::size_t(0));
    k = std::min(k, order.size());
    std::partial_sort(order.begin(), order.begin() + std::ptrdiff_t(k), order.end(),
                      [&](std::size_t a, std::size_t b) { return pred[a] != pred[b] ? pred[a] > pred[b] : vals[a] < vals[b]; });
    order.resize(k);
    return order;
}

template <typename Result, typename Input, typename Tuning, typename Bounds, typename Predict>
Result infer_any(const Input& input, const HardwareDescriptor& hw, const Bounds& bounds, int top_k,
                 MeasurementBackend& backend, Predict predict) {
    input.validate();
    if (top_k < 1) throw std::invalid_argument("top_k must be >= 1");
    std::vector<Tuning> legal = enumerate_legal(input, hw, bounds);
    if (legal.empty()) throw std::runtime_error("no legal configuration for this input");
    const auto legal_size = std::int64_t(legal.size());
    // Rank only what the measuring backend can run (the reference's CPU
    // executors run every legal tuple; the B200 families reject tuples
    // outside their launch envelope with unsupported_error, which would
    // otherwise abort the top-k re-measure).  legal_space_size stays the
    // whole legal space.
    legal.erase(std::remove_if(legal.begin(), legal.end(),
                               [&](const Tuning& t) { return !backend.accepts(input, t); }),
                legal.end());
    if (legal.empty()) throw std::runtime_error("no legal configuration this backend can launch for this input");
    std::vector<double> pred;
    predict(legal, pred);
    Result r;
    r.input = input;
    r.legal_space_size = legal_size;
    for (std::size_t idx : best_k(legal, pred, std::size_t(top_k))) r.top_k.push_back({legal[idx], pred[idx], 0.0});
    std::size_t best = 0;
    for (std::size_t i = 0; i < r.top_k.size(); ++i) {
        r.top_k[i].measured_gflops = backend.measure(input, r.top_k[i].tuning);
        if (r.top_k[i].measured_gflops > r.top_k[best].measured_gflops) best = i;
    }
    r.chosen = r.top_k[best].tuning;
    r.predicted_log_gflops = r.top_k[best].predicted_log_gflops;
    r.measured_gflops = r.top_k[best].measured_gflops;
    return r;
}

}  // namespace

GemmInferenceResult infer_gemm(const PerfPredictor& predictor, const GemmInput& input, const HardwareDescriptor& hw,
                               const GemmBounds& bounds, int top_k, MeasurementBackend& backend) {
    return infer_any<GemmInferenceResult, GemmInput, GemmTuning>(
        input, hw, bounds, top_k, backend,
        [&](const std::vector<GemmTuning>& legal, std::vector<double>& pred) { predictor.predict_gemm(input, legal, pred); });
}

ConvInferenceResult infer_conv(const PerfPredictor& predictor, const ConvInput& input, const HardwareDescriptor& hw,
                               const ConvBounds& bounds, int top_k, MeasurementBackend& backend) {
    return infer_any<ConvInferenceResult, ConvInput, ConvTuning>(
        input, hw, bounds, top_k, backend,
        [&](const std::vector<ConvTuning>& legal, std::vector<double>& pred) { predictor.predict_conv(input, legal, pred); });
}

// ---------------------------------------------------------------------------
// result JSON (ktune-result-1) + cache
// ---------------------------------------------------------------------------

namespace {

constexpr const char* kResultFormat = "ktune-result-1";

json input_json(const GemmInput& in) {
    return {{"m", in.m}, {"n", in.n}, {"k", in.k}, {"dtype", to_string(in.dtype)}, {"trans_a", in.trans_a},
            {"trans_b", in.trans_b}};
}

json input_json(const ConvInput& in) {
    return {{"n", in.n_batch}, {"p", in.p}, {"q", in.q}, {"k", in.k_filters},
            {"c", in.c},       {"r", in.r}, {"s", in.s}, {"dtype", to_string(in.dtype)}};
}

GemmInput gemm_input_of(const json& j) {
    GemmInput in;
    in.m = j.at("m").get<int>();
    in.n = j.at("n").get<int>();
    in.k = j.at("k").get<int>();
    in.dtype = dtype_from_string(j.at("dtype").get<std::string>());
    in.trans_a = j.at("trans_a").get<bool>();
    in.trans_b = j.at("trans_b").get<bool>();
    in.validate();
    return in;
}

ConvInput conv_input_of(const json& j) {
    ConvInput in;
    in.n_batch = j.at("n").get<int>();
    in.p = j.at("p").get<int>();
    in.q = j.at("q").get<int>();
    in.k_filters = j.at("k").get<int>();
    in.c = j.at("c").get<int>();
    in.r = j.at("r").get<int>();
    in.s = j.at("s").get<int>();
    in.dtype = dtype_from_string(j.at("dtype").get<std::string>());
    in.validate();
    return in;
}

template <typename Tuning>
json tuning_json(const Tuning& t, const std::vector<std::string>& names) {
    json j;
    const auto v = to_values(t);
    for (std::size_t i = 0; i < names.size(); ++i) j[names[i]] = v[i];
    return j;
}

std::vector<int> tuning_values(const json& j, const std::vector<std::string>& names) {
    std::vector<int> v;
    for (const auto& n : names) v.push_back(j.at(n).get<int>());
    return v;
}

template <typename Result>
std::string result_json(const Result& r, const char* kind, const char* version, const std::vector<std::string>& names) {
    json j;
    j["format"] = kResultFormat;
    j["kind"] = kind;
    j["feature_version"] = version;
    j["input"] = input_json(r.input);
    j["chosen"] = tuning_json(r.chosen, names);
    j["predicted_log_gflops"] = r.predicted_log_gflops;
    j["measured_gflops"] = r.measured_gflops;
    j["legal_space_size"] = r.legal_space_size;
    j["top_k"] = json::array();
    for (const auto& c : r.top_k)
        j["top_k"].push_back({{"tuning", tuning_json(c.tuning, names)},
                              {"predicted_log_gflops", c.predicted_log_gflops},
                              {"measured_gflops", c.measured_gflops}});
    return j.dump(2) + "\n";
}

template <typename Result, typename Candidate, typename InputOf, typename FromValues>
Result result_of(const std::string& text, const char* kind, const std::vector<std::string>& names, InputOf input_of,
                 FromValues from_values) {
    json j = json::parse(text, nullptr, false);
    if (j.is_discarded()) throw std::runtime_error("malformed JSON result");
    try {
        if (j.at("format").get<std::string>() != kResultFormat || j.at("kind").get<std::string>() != kind)
            throw std::runtime_error(std::string("not a ") + kind + " inference result");
        Result r;
        r.input = input_of(j.at("input"));
        r.chosen = from_values(tuning_values(j.at("chosen"), names));
        r.predicted_log_gflops = j.at("predicted_log_gflops").get<double>();
        r.measured_gflops = j.at("measured_gflops").get<double>();
        r.legal_space_size = j.at("legal_space_size").get<std::int64_t>();
        for (const auto& jc : j.at("top_k")) {
            Candidate c;
            c.tuning = from_values(tuning_values(jc.at("tuning"), names));
            c.predicted_log_gflops = jc.at("predicted_log_gflops").get<double>();
            c.measured_gflops = jc.at("measured_gflops").get<double>();
            r.top_k.push_back(std::move(c));
        }
        return r;
    } catch (const json::exception& e) {
        throw std::runtime_error(std::string("bad result JSON: ") + e.what());
    }
}


std::string descriptor(const GemmInput& in) {
    std::ostringstream s;
    s << "gemm|m=" << in.m << "|n=" << in.n << "|k=" << in.k << "|dtype=" << to_string(in.dtype)
      << "|ta=" << in.trans_a << "|tb=" << in.trans_b;
    return s.str();
}

std::string descriptor(const ConvInput& in) {
    std::ostringstream s;
    s << "conv|n=" << in.n_batch << "|p=" << in.p << "|q=" << in.q << "|k=" << in.k_filters << "|c=" << in.c
      << "|r=" << in.r << "|s=" << in.s << "|dtype=" << to_string(in.dtype);
    return s.str();
}

template <typename Result, typename Input, typename Parse>
std::optional<Result> lookup_in(const std::string& dir, const Input& input, Parse parse) {
    const auto path = std::filesystem::path(dir) / cache_key(input);
    if (!std::filesystem::exists(path)) return std::nullopt;
    try {
        Result r = parse(read_text_file(path.string()));
        if (!(r.input == input)) throw std::runtime_error("entry stores a different input");
        return r;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "warning: skipping corrupt cache entry %s: %s\n", path.string().c_str(), e.what());
        return std::nullopt;
    }
}

}  // namespace

std::string to_json_text(const GemmInferenceResult& r) {
    return result_json(r, "gemm", kGemmFeatureVersion, gemm_param_names());
}

std::string to_json_text(const ConvInferenceResult& r) {
    return result_json(r, "conv", kConvFeatureVersion, conv_param_names());
}

GemmInferenceResult gemm_result_from_json_text(const std::string& text) {
    return result_of<GemmInferenceResult, GemmCandidate>(text, "gemm", gemm_param_names(), gemm_input_of,
                                                         gemm_tuning_from_values);
}

ConvInferenceResult conv_result_from_json_text(const std::string& text) {
    return result_of<ConvInferenceResult, ConvCandidate>(text, "conv", conv_param_names(), conv_input_of,
                                                         conv_tuning_from_values);
}

std::string fnv1a64_hex(const std::string& text) {
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : text) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    char buf[17];
    std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
    return buf;
}

std::string cache_key(const GemmInput& input) { return "gemm-" + fnv1a64_hex(descriptor(input)) + ".json"; }
std::string cache_key(const ConvInput& input) { return "conv-" + fnv1a64_hex(descriptor(input)) + ".json"; }

ResultCache::ResultCache(std::string dir) : dir_(std::move(dir)) {
    if (dir_.empty()) throw std::invalid_argument("cache directory must not be empty");
    std::filesystem::create_directories(dir_);
}

ResultCache ResultCache::from_env_or(const std::string& fallback_dir) {
    const char* env = std::getenv(kCacheDirEnvVar);
    return (env != nullptr && env[0] != '\0') ? ResultCache(env) : ResultCache(fallback_dir);
}

std::optional<GemmInferenceResult> ResultCache::lookup(const GemmInput& input) const {
    return lookup_in<GemmInferenceResult>(dir_, input, gemm_result_from_json_text);
}

std::optional<ConvInferenceResult> ResultCache::lookup(const ConvInput& input) const {
    return lookup_in<ConvInferenceResult>(dir_, input, conv_result_from_json_text);
}

void ResultCache::store(const GemmInferenceResult& result) const {
    std::filesystem::create_directories(dir_);
    write_text_file_atomic((std::filesystem::path(dir_) / cache_key(result.input)).string(), to_json_text(result));
}

void ResultCache::store(const ConvInferenceResult& result) const {
    std::filesystem::create_directories(dir_);
    write_text_file_atomic((std::filesystem::path(dir_) / cache_key(result.input)).string(), to_json_text(result));
}

}  // namespace ktune
