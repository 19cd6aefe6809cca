// ktune_b200 -- the `ktune` command-line front end over the B200 build.
//
// Drop-in for the reference CLI (/root/reference/proj/tools/ktune.cpp:700-806):
// the same six verbs (calibrate, generate, train, infer, bench, report), the
// same flags, ktune-report-1 JSON reports with every wall-clock value under
// "timing", atomic artifact writes and the same exit codes -- 0 success,
// 1 runtime failure, 2 usage error raised before anything is written
// (ktune.cpp:35-38, 783-805).  The measurement backend registry
// (make_backend, ktune.cpp:186-191) offers "analytical" (the reference's
// deterministic cost model) and "b200" / "b200-parity" (device measurement
// through B200Backend); there is no CPU executor in this build, so
// "--backend cpu" is a usage error that says so.  CLI11 is not available
// here, so the parser below is a small hand-written one with the same
// surface (--opt value, --opt=value, comma-delimited lists, flags).

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <cmath>
#include <string>
#include <vector>

#include <json.hpp>

#include "ktune/analytical.hpp"
#include "ktune/b200_backend.hpp"
#include "ktune/mlp.hpp"
#include "ktune/sampling.hpp"
#include "ktune/space.hpp"
#include "ktune/tuner.hpp"
#include "ktune_b200.h"

namespace {

using nlohmann::json;
using namespace ktune;

// Exit code 2: bad flags, missing or malformed prerequisites.
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

double wall_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------------------
// argument parsing
// ---------------------------------------------------------------------------

struct Spec {
    std::string name;  // without leading dashes
    bool flag;         // true: no value
    std::string help;
};

class Args {
  public:
    Args(std::string verb, std::vector<Spec> specs) : verb_(std::move(verb)), specs_(std::move(specs)) {}

    void parse(const std::vector<std::string>& argv) {
        for (std::size_t i = 0; i < argv.size(); ++i) {
            const std::string& a = argv[i];
            if (a == "-h" || a == "--help") {
                help_ = true;
                continue;
            }
            if (a.rfind("--", 0) != 0) throw UsageError(verb_ + ": unexpected argument '" + a + "'");
            std::string key = a.substr(2), val;
            bool has_val = false;
            if (auto eq = key.find('='); eq != std::string::npos) {
                val = key.substr(eq + 1);
                key = key.substr(0, eq);
                has_val = true;
            }
            const Spec* s = find(key);
            if (s == nullptr) throw UsageError(verb_ + ": unknown option --" + key);
            if (s->flag) {
                if (has_val) throw UsageError(verb_ + ": --" + key + " takes no value");
                flags_.insert(key);
                continue;
            }
            if (!has_val) {
                if (i + 1 >= argv.size()) throw UsageError(verb_ + ": --" + key + " needs a value");
                val = argv[++i];
            }
            values_[key] = val;
        }
    }

    bool help() const { return help_; }
    void print_help() const {
        std::printf("usage: ktune_b200 %s [options]\n", verb_.c_str());
        for (const auto& s : specs_)
            std::printf("  --%-16s %s\n", (s.name + (s.flag ? "" : " <v>")).c_str(), s.help.c_str());
    }
    bool has(const std::string& k) const { return values_.count(k) != 0; }
    bool flag(const std::string& k) const { return flags_.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") const {
        auto it = values_.find(k);
        return it == values_.end() ? def : it->second;
    }
    long long integer(const std::string& k, long long def) const {
        if (!has(k)) return def;
        return parse_int(k, str(k));
    }
    double real(const std::string& k, double def) const {
        if (!has(k)) return def;
        const std::string v = str(k);
        try {
            std::size_t pos = 0;
            const double d = std::stod(v, &pos);
            if (pos != v.size()) throw std::invalid_argument("trailing characters");
            return d;
        } catch (const std::exception&) {
            throw UsageError(verb_ + ": --" + k + " expects a number, got '" + v + "'");
        }
    }
    std::vector<int> int_list(const std::string& k, std::vector<int> def) const {
        if (!has(k)) return def;
        std::vector<int> out;
        std::stringstream ss(str(k));
        std::string item;
        while (std::getline(ss, item, ',')) out.push_back(int(parse_int(k, item)));
        return out;
    }

  private:
    const Spec* find(const std::string& k) const {
        for (const auto& s : specs_)
            if (s.name == k) return &s;
        return nullptr;
    }
    long long parse_int(const std::string& k, const std::string& v) const {
        try {
            std::size_t pos = 0;
            const long long x = std::stoll(v, &pos);
            if (pos != v.size()) throw std::invalid_argument("trailing characters");
            return x;
        } catch (const std::exception&) {
            throw UsageError(verb_ + ": --" + k + " expects an integer, got '" + v + "'");
        }
    }

    std::string verb_;
    std::vector<Spec> specs_;
    std::map<std::string, std::string> values_;
    std::set<std::string> flags_;
    bool help_{false};
};

// ---------------------------------------------------------------------------
// files
// ---------------------------------------------------------------------------

void need_file(const std::string& path, const std::string& what, const std::string& hint) {
    if (path.empty()) throw UsageError(what + " required: " + hint);
    if (!std::filesystem::exists(path)) throw UsageError(what + " not found: " + path + " -- " + hint);
}

void write_atomically(const std::string& path, const std::string& text) {
    const std::string tmp = path + ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw std::runtime_error("cannot write " + tmp);
        out << text;
        if (!out) throw std::runtime_error("write failed: " + tmp);
    }
    std::filesystem::rename(tmp, path);
}

void emit_report(const std::string& path, json j, json timing) {
    if (path.empty()) return;
    j["timing"] = std::move(timing);
    write_atomically(path, j.dump(2) + "\n");
}

template <typename F>
auto as_usage(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const UsageError&) {
        throw;
    } catch (const std::exception& e) {
        throw UsageError(e.what());
    }
}

HardwareDescriptor hw_from(const Args& a) {
    const std::string p = a.str("hw");
    need_file(p, "hardware descriptor", "pass --hw <file>");
    return as_usage([&] { return HardwareDescriptor::load(p); });
}

template <typename B>
B bounds_from(const Args& a) {
    const std::string p = a.str("bounds");
    need_file(p, "bounds file", "pass --bounds <file>");
    return as_usage([&] { return B::load(p); });
}

CategoricalModel sampler_from(const std::string& p) {
    need_file(p, "sampler model", "run `ktune_b200 calibrate` first");
    return as_usage([&] { return CategoricalModel::load(p); });
}

MlpModel model_from(const std::string& p) {
    need_file(p, "performance model", "run `ktune_b200 train` first");
    return as_usage([&] { return MlpModel::load(p); });
}

std::string dataset_kind(const std::string& p) {
    need_file(p, "dataset", "run `ktune_b200 generate` first");
    std::ifstream in(p);
    std::string header;
    std::getline(in, header);
    if (!header.empty() && header.back() == '\r') header.pop_back();
    if (header == kGemmCsvHeader) return "gemm";
    if (header == kConvCsvHeader) return "conv";
    throw UsageError("dataset " + p + " has an unrecognized header");
}

// Shape tables: the reference's {"kind", "shapes": [{name, m, n, ...}]}
// (proj/fixtures/shapes/*.json) or this repo's fixtures/shapes/benchmarks.json
// (column lists for both kinds; `want_kind` picks one).
struct Shapes {
    std::string kind;
    std::vector<std::pair<std::string, GemmInput>> gemm;
    std::vector<std::pair<std::string, ConvInput>> conv;
};

Shapes shapes_from(const std::string& p, const std::string& want_kind, Dtype dtype) {
    need_file(p, "shapes file", "pass --shapes <file>");
    std::ifstream in(p);
    json j = json::parse(in, nullptr, false);
    if (j.is_discarded()) throw UsageError("shapes file " + p + " is not valid JSON");
    Shapes out;
    try {
        if (j.contains("shapes")) {
            out.kind = j.at("kind").get<std::string>();
            for (const auto& s : j.at("shapes")) {
                const Dtype dt = s.contains("dtype") ? dtype_from_string(s.at("dtype").get<std::string>()) : dtype;
                if (out.kind == "gemm") {
                    GemmInput g{s.at("m").get<std::int64_t>(), s.at("n").get<std::int64_t>(),
                                s.at("k").get<std::int64_t>(), dt, s.at("trans_a").get<bool>(),
                                s.at("trans_b").get<bool>()};
                    g.validate();
                    out.gemm.emplace_back(s.at("name").get<std::string>(), g);
                } else if (out.kind == "conv") {
                    ConvInput c{s.at("n").get<std::int64_t>(), s.at("p").get<std::int64_t>(),
                                s.at("q").get<std::int64_t>(), s.at("k").get<std::int64_t>(),
                                s.at("c").get<std::int64_t>(), s.at("r").get<std::int64_t>(),
                                s.at("s").get<std::int64_t>(), dt};
                    c.validate();
                    out.conv.emplace_back(s.at("name").get<std::string>(), c);
                } else {
                    throw UsageError("shapes file kind must be gemm or conv");
                }
            }
        } else {
            out.kind = want_kind.empty() ? "gemm" : want_kind;
            for (const auto& r : j.at(out.kind)) {
                if (out.kind == "gemm") {
                    GemmInput g{r.at(1).get<std::int64_t>(), r.at(2).get<std::int64_t>(), r.at(3).get<std::int64_t>(),
                                dtype, r.at(4).get<int>() != 0, r.at(5).get<int>() != 0};
                    g.validate();
                    out.gemm.emplace_back(r.at(0).get<std::string>(), g);
                } else {
                    ConvInput c{r.at(1).get<std::int64_t>(), r.at(2).get<std::int64_t>(), r.at(3).get<std::int64_t>(),
                                r.at(4).get<std::int64_t>(), r.at(5).get<std::int64_t>(), r.at(6).get<std::int64_t>(),
                                r.at(7).get<std::int64_t>(), dtype};
                    c.validate();
                    out.conv.emplace_back(r.at(0).get<std::string>(), c);
                }
            }
        }
    } catch (const json::exception& e) {
        throw UsageError("bad shapes file " + p + ": " + e.what());
    } catch (const std::invalid_argument& e) {
        throw UsageError("bad shapes file " + p + ": " + e.what());
    }
    if (out.gemm.empty() && out.conv.empty()) throw UsageError("shapes file " + p + " lists no shapes");
    return out;
}

std::unique_ptr<MeasurementBackend> backend_from(const std::string& name, const HardwareDescriptor& hw) {
    if (name == "analytical") return std::make_unique<AnalyticalBackend>(hw);
    if (name == "b200" || name == "b200-parity") {
        MeasureOptions opt;
        opt.mode = name == "b200" ? dev::Mode::fast : dev::Mode::parity;
        return std::make_unique<B200Backend>(hw, opt);
    }
    if (name == "cpu")
        throw UsageError("backend 'cpu': this build has no CPU executor (every executor runs on the B200); "
                         "use --backend b200 (or analytical)");
    throw UsageError("unknown backend '" + name + "' (expected analytical|b200|b200-parity)");
}

Dtype dtype_arg(const Args& a) {
    return as_usage([&] { return dtype_from_string(a.str("dtype", "f32")); });
}

std::string joined(const std::vector<int>& v) {
    std::string s;
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? " " : "") + std::to_string(v[i]);
    return s;
}

template <typename T>
json named(const T& t, const std::vector<std::string>& names) {
    json j;
    const auto v = to_values(t);
    for (std::size_t i = 0; i < names.size(); ++i) j[names[i]] = v[i];
    return j;
}

template <typename Dataset>
void gflops_range(const Dataset& ds, double& lo, double& hi, double& sum) {
    lo = 1e300;
    hi = 0;
    sum = 0;
    for (const auto& s : ds.samples) {
        lo = std::min(lo, s.gflops);
        hi = std::max(hi, s.gflops);
        sum += s.gflops;
    }
}

// ---------------------------------------------------------------------------
// verbs
// ---------------------------------------------------------------------------

int do_calibrate(const Args& a) {
    const HardwareDescriptor hw = hw_from(a);
    const Dtype dtype = dtype_arg(a);
    const std::string out = a.str("out");
    if (out.empty()) throw UsageError("pass --out <file> for the sampler model");
    const std::string kind = a.str("kind", "gemm");
    LegalityFn legal;
    std::vector<std::vector<int>> lists;
    // probe inputs of the reference CLI (ktune.cpp:244, 248)
    if (kind == "gemm") {
        lists = bounds_from<GemmBounds>(a).as_lists();
        legal = make_legality(GemmInput{512, 512, 512, dtype, false, false}, hw);
    } else if (kind == "conv") {
        lists = bounds_from<ConvBounds>(a).as_lists();
        legal = make_legality(ConvInput{16, 24, 240, 32, 16, 3, 3, dtype}, hw);
    } else {
        throw UsageError("--kind must be gemm or conv");
    }
    const auto seed = std::uint64_t(a.integer("seed", 0));
    const auto draws = a.integer("draws", kDefaultCalibrationDraws);
    const auto trials = a.integer("trials", 10000);
    const double alpha = a.real("alpha", 100.0);
    const double t0 = wall_s();
    const CategoricalModel model = calibrate(legal, lists, draws, seed, alpha);
    const double cat = acceptance_rate(model, legal, trials, seed + 1);
    const double uni = uniform_acceptance_rate(lists, legal, trials, seed + 2);
    const double secs = wall_s() - t0;
    model.save(out);
    std::printf("sampler model written to %s\n", out.c_str());
    std::printf("%-12s %12s %12s\n", "", "categorical", "uniform");
    std::printf("%-12s %11.2f%% %11.2f%%\n", "acceptance", 100 * cat, 100 * uni);
    if (uni > 0) std::printf("%-12s %11.1fx\n", "improvement", cat / uni);
    json j{{"format", "ktune-report-1"}, {"command", "calibrate"}, {"kind", kind}, {"alpha", alpha},
           {"draws", draws}, {"trials", trials}, {"seed", seed}};
    j["acceptance"] = {{"categorical", cat}, {"uniform", uni}, {"ratio", uni > 0 ? cat / uni : 0.0}};
    j["outputs"] = {{"sampler_model", out}};
    emit_report(a.str("report"), j, {{"seconds", secs}});
    return 0;
}

// --merge: the dataset CSV from the shard files of `generate --shard R/N`
// (the file-based form of the all-gather: rows placed by sequence index).
int do_merge(const Args& a, const std::string& out) {
    std::vector<std::string> files;
    {
        std::stringstream ss(a.str("merge"));
        std::string f;
        while (std::getline(ss, f, ','))
            if (!f.empty()) files.push_back(f);
    }
    std::string header, csv_header, kind;
    std::map<long long, std::string> rows;
    long long n = -1;
    for (const auto& f : files) {
        std::ifstream in(f);
        if (!in) throw UsageError("cannot read shard file " + f);
        std::string h, ch, line;
        std::getline(in, h);
        std::getline(in, ch);
        if (h.rfind("ktune-shard-records-1 ", 0) != 0) throw UsageError(f + " is not a shard file");
        std::istringstream hs(h);
        std::string tag, k, nfield;
        hs >> tag >> k >> nfield;
        const long long nn = std::stoll(nfield.substr(nfield.find('=') + 1));
        if (n >= 0 && (nn != n || k != kind || ch != csv_header)) throw UsageError(f + " belongs to another run");
        n = nn;
        kind = k;
        csv_header = ch;
        while (std::getline(in, line)) {
            const auto c = line.find(',');
            if (c == std::string::npos) continue;
            rows[std::stoll(line.substr(0, c))] = line.substr(c + 1);
        }
    }
    if (n < 0 || (long long)rows.size() != n)
        throw UsageError("shards cover " + std::to_string(rows.size()) + " of " + std::to_string(n) + " samples");
    std::ofstream o(out);
    o << csv_header << '\n';
    for (const auto& r : rows) o << r.second << '\n';
    std::printf("merged %zu shard file(s): %lld %s samples to %s\n", files.size(), n, kind.c_str(), out.c_str());
    return 0;
}

// --shard R/N: this rank's share of the sequence (LPT by 2MNK), measured on
// the B200 with batched syncs and an optional resumable --checkpoint; writes
// a shard file of "index,<dataset row>" lines for --merge.
template <typename Draw, typename Dataset>
void write_shard(const std::string& out, const std::string& kind, std::int64_t n, const std::vector<Draw>& draws,
                 const std::vector<ShardRecord>& recs, const std::string& backend) {
    Dataset one;
    std::ofstream o(out);
    if (!o) throw std::runtime_error("cannot write " + out);
    std::string head;
    {
        Dataset empty;
        head = to_csv_text(empty);
        head = head.substr(0, head.find('\n'));
    }
    o << "ktune-shard-records-1 " << kind << " n=" << n << '\n' << head << '\n';
    for (const auto& r : recs) {
        if (!(std::isfinite(r.gflops) && r.gflops > 0.0))
            throw std::runtime_error("sample " + std::to_string(r.index) + " failed to launch");
        one.samples.clear();
        one.samples.push_back({draws[std::size_t(r.index)].input, draws[std::size_t(r.index)].tuning, r.gflops,
                               backend, 0});
        std::string text = to_csv_text(one);
        text = text.substr(text.find('\n') + 1);
        while (!text.empty() && text.back() == '\n') text.pop_back();
        o << r.index << ',' << text << '\n';
    }
}

int do_generate(const Args& a) {
    if (!a.str("merge").empty()) {
        if (a.str("out").empty()) throw UsageError("pass --out <file> for the merged dataset CSV");
        return do_merge(a, a.str("out"));
    }
    const HardwareDescriptor hw = hw_from(a);
    const CategoricalModel sampler = sampler_from(a.str("sampler"));
    const std::string out = a.str("out");
    if (out.empty()) throw UsageError("pass --out <file> for the dataset CSV");
    const auto samples = a.integer("samples", 1000);
    if (samples < 1) throw UsageError("--samples must be >= 1");
    std::string kind;
    if (sampler.params.size() == gemm_param_names().size()) kind = "gemm";
    else if (sampler.params.size() == conv_param_names().size()) kind = "conv";
    else throw UsageError("sampler model has an unrecognized dimensionality");
    const Dtype dtype = dtype_arg(a);
    Shapes shapes;
    if (!a.str("shapes").empty()) {
        shapes = shapes_from(a.str("shapes"), kind, dtype);
        if (shapes.kind != kind)
            throw UsageError("shapes file kind (" + shapes.kind + ") does not match the sampler model (" + kind + ")");
    }
    const double fraction = a.real("shape-fraction", 0.5);
    const auto seed = std::uint64_t(a.integer("seed", 0));
    auto backend = backend_from(a.str("backend", "analytical"), hw);
    const double t0 = wall_s();
    GenerateReport rep;
    json j{{"format", "ktune-report-1"}, {"command", "generate"}, {"kind", kind}, {"samples", samples},
           {"seed", seed}, {"backend", a.str("backend", "analytical")}};
    double lo = 0, hi = 0, sum = 0;
    std::size_t rows = 0;
    int shard_rank = -1, shard_world = 0;
    if (!a.str("shard").empty()) {
        const std::string sh = a.str("shard");
        const auto slash = sh.find('/');
        if (slash == std::string::npos) throw UsageError("--shard expects R/N");
        shard_rank = std::atoi(sh.substr(0, slash).c_str());
        shard_world = std::atoi(sh.substr(slash + 1).c_str());
        if (shard_world < 1 || shard_rank < 0 || shard_rank >= shard_world) throw UsageError("--shard R/N: 0 <= R < N");
        const std::string be = a.str("backend", "analytical");
        if (be != "b200" && be != "b200-parity") throw UsageError("--shard needs --backend b200 or b200-parity");
        MeasureOptions opt;
        opt.mode = be == "b200" ? dev::Mode::fast : dev::Mode::parity;
        std::vector<ShardRecord> recs;
        if (kind == "gemm") {
            GemmInputDistribution dist;
            dist.dtype = dtype;
            dist.fixed_fraction = fraction;
            for (const auto& s : shapes.gemm) dist.shapes.push_back(s.second);
            std::vector<GemmDraw> draws;
            recs = generate_gemm_shard(sampler, dist, bounds_from<GemmBounds>(a), hw, int(samples), seed, shard_rank,
                                       shard_world, opt, a.str("checkpoint"), &draws, &rep);
            write_shard<GemmDraw, GemmDataset>(out, kind, samples, draws, recs, be);
        } else {
            ConvInputDistribution dist;
            dist.dtype = dtype;
            dist.fixed_fraction = fraction;
            for (const auto& s : shapes.conv) dist.shapes.push_back(s.second);
            std::vector<ConvDraw> draws;
            recs = generate_conv_shard(sampler, dist, bounds_from<ConvBounds>(a), hw, int(samples), seed, shard_rank,
                                       shard_world, opt, a.str("checkpoint"), &draws, &rep);
            write_shard<ConvDraw, ConvDataset>(out, kind, samples, draws, recs, be);
        }
        std::printf("shard %d/%d: wrote %zu of %lld %s samples to %s\n", shard_rank, shard_world, recs.size(),
                    (long long)samples, kind.c_str(), out.c_str());
        j["shard"] = {{"rank", shard_rank}, {"world", shard_world}, {"records", recs.size()}};
        j["attempts"] = rep.attempts;
        j["duplicates_rejected"] = rep.duplicates_rejected;
        j["unlaunchable_rejected"] = rep.unlaunchable_rejected;
        j["outputs"] = {{"shard", out}};
        emit_report(a.str("report"), j, {{"seconds", wall_s() - t0}});
        return 0;
    }
    if (kind == "gemm") {
        const auto bounds = bounds_from<GemmBounds>(a);
        GemmInputDistribution dist;
        dist.dtype = dtype;
        dist.fixed_fraction = fraction;
        for (const auto& s : shapes.gemm) dist.shapes.push_back(s.second);
        const auto ds = generate_gemm_dataset(*backend, sampler, dist, bounds, hw, int(samples), seed, &rep);
        save_gemm_dataset(ds, out);
        gflops_range(ds, lo, hi, sum);
        rows = ds.samples.size();
    } else {
        const auto bounds = bounds_from<ConvBounds>(a);
        ConvInputDistribution dist;
        dist.dtype = dtype;
        dist.fixed_fraction = fraction;
        for (const auto& s : shapes.conv) dist.shapes.push_back(s.second);
        const auto ds = generate_conv_dataset(*backend, sampler, dist, bounds, hw, int(samples), seed, &rep);
        save_conv_dataset(ds, out);
        gflops_range(ds, lo, hi, sum);
        rows = ds.samples.size();
    }
    std::printf("wrote %zu %s samples to %s (gflops %.2f .. %.2f)\n", rows, kind.c_str(), out.c_str(), lo, hi);
    std::printf("sampler draws: %lld (%lld duplicate redraws)\n", (long long)rep.attempts,
                (long long)rep.duplicates_rejected);
    j["gflops_min"] = lo;
    j["gflops_max"] = hi;
    j["attempts"] = rep.attempts;
    j["duplicates_rejected"] = rep.duplicates_rejected;
    j["outputs"] = {{"dataset", out}};
    emit_report(a.str("report"), j, {{"seconds", wall_s() - t0}});
    return 0;
}

int do_train(const Args& a) {
    const std::string path = a.str("dataset");
    const std::string kind = dataset_kind(path);
    const std::string out = a.str("out");
    if (out.empty()) throw UsageError("pass --out <file> for the trained model");
    const TrainingSet data = kind == "gemm" ? to_training_set(load_gemm_dataset(path))
                                            : to_training_set(load_conv_dataset(path));
    MlpArchitecture arch;
    arch.input_dim = data.dim;
    arch.hidden_sizes = a.int_list("hidden", {32, 64, 32});
    arch.log_inputs = !a.flag("raw-features");
    TrainConfig cfg;
    cfg.learning_rate = a.real("lr", 1e-3);
    cfg.batch_size = int(a.integer("batch", 256));
    cfg.epochs = int(a.integer("epochs", 200));
    cfg.rng_seed = std::uint64_t(a.integer("seed", 0));
    cfg.validation_fraction = a.real("val-fraction", 0.1);
    const double t0 = wall_s();
    const TrainResult res = mlp_train(data, arch, cfg);
    const double secs = wall_s() - t0;
    MlpModel model;
    model.feature_version = kind == "gemm" ? kGemmFeatureVersion : kConvFeatureVersion;
    model.weights = res.weights;
    model.save(out);
    std::printf("trained on %zu rows (%s), %d epochs\n", data.size(), kind.c_str(), cfg.epochs);
    std::printf("best validation MSE %.6f at epoch %d\n", res.best_val_mse, res.best_epoch);
    std::printf("model written to %s\n", out.c_str());
    json j{{"format", "ktune-report-1"}, {"command", "train"}, {"kind", kind}, {"rows", data.size()},
           {"epochs", cfg.epochs}, {"seed", cfg.rng_seed}, {"hidden", arch.hidden_sizes},
           {"log_features", arch.log_inputs}, {"best_epoch", res.best_epoch}, {"best_val_mse", res.best_val_mse}};
    json hist = json::array();
    for (const auto& e : res.history) hist.push_back({{"train_mse", e.train_mse}, {"val_mse", e.val_mse}});
    j["history"] = std::move(hist);
    j["outputs"] = {{"model", out}};
    emit_report(a.str("report"), j, {{"seconds", secs}});
    return 0;
}

int do_infer(const Args& a) {
    if (!a.has("shape")) throw UsageError("infer: --shape is required (m,n,k or n,p,q,k,c,r,s)");
    const std::vector<int> shape = a.int_list("shape", {});
    MlpModel model = model_from(a.str("model"));
    const HardwareDescriptor hw = hw_from(a);
    auto backend = backend_from(a.str("backend", "analytical"), hw);
    const MlpPredictor predictor(std::move(model));
    std::optional<ResultCache> cache;
    if (!a.flag("no-cache")) cache.emplace(ResultCache::from_env_or(a.str("cache-dir", ".ktune-cache")));
    const int top_k = int(a.integer("top-k", kDefaultTopK));
    const Dtype dtype = dtype_arg(a);
    const std::string out = a.str("out");
    if (shape.size() == 3) {
        const GemmInput in{shape[0], shape[1], shape[2], dtype, a.flag("trans-a"), a.flag("trans-b")};
        as_usage([&] { in.validate(); return 0; });
        if (cache) {
            if (auto hit = cache->lookup(in)) {
                std::printf("cache hit (%s)\n", (std::filesystem::path(cache->dir()) / cache_key(in)).string().c_str());
                std::printf("chosen: %s\n", joined(to_values(hit->chosen)).c_str());
                std::printf("measured: %.3f gflops\n", hit->measured_gflops);
                if (!out.empty()) write_atomically(out, to_json_text(*hit));
                return 0;
            }
        }
        const auto res = infer_gemm(predictor, in, hw, bounds_from<GemmBounds>(a), top_k, *backend);
        if (cache) cache->store(res);
        std::printf("legal space: %lld, re-measured top %zu\n", (long long)res.legal_space_size, res.top_k.size());
        std::printf("chosen (m_s n_s m_l n_l u k_s k_l k_g): %s\n", joined(to_values(res.chosen)).c_str());
        std::printf("predicted: %.3f log-gflops, measured: %.3f gflops\n", res.predicted_log_gflops,
                    res.measured_gflops);
        if (!out.empty()) write_atomically(out, to_json_text(res));
        return 0;
    }
    if (shape.size() == 7) {
        const ConvInput in{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5], shape[6], dtype};
        as_usage([&] { in.validate(); return 0; });
        if (cache) {
            if (auto hit = cache->lookup(in)) {
                std::printf("cache hit\n");
                std::printf("chosen: %s\n", joined(to_values(hit->chosen)).c_str());
                std::printf("measured: %.3f gflops\n", hit->measured_gflops);
                if (!out.empty()) write_atomically(out, to_json_text(*hit));
                return 0;
            }
        }
        const auto res = infer_conv(predictor, in, hw, bounds_from<ConvBounds>(a), top_k, *backend);
        if (cache) cache->store(res);
        std::printf("legal space: %lld, re-measured top %zu\n", (long long)res.legal_space_size, res.top_k.size());
        std::printf("chosen: %s\n", joined(to_values(res.chosen)).c_str());
        std::printf("predicted: %.3f log-gflops, measured: %.3f gflops\n", res.predicted_log_gflops,
                    res.measured_gflops);
        if (!out.empty()) write_atomically(out, to_json_text(res));
        return 0;
    }
    throw UsageError("--shape takes m,n,k for gemm or n,p,q,k,c,r,s for conv (got " + std::to_string(shape.size()) +
                     " values)");
}

int do_bench(const Args& a) {
    const HardwareDescriptor hw = hw_from(a);
    const Shapes shapes = shapes_from(a.str("shapes"), a.str("kind"), dtype_arg(a));
    auto backend = backend_from(a.str("backend", "analytical"), hw);
    const bool exhaustive = a.flag("exhaustive") || a.str("model").empty();
    std::unique_ptr<PerfPredictor> predictor;
    if (exhaustive) predictor = std::make_unique<AnalyticalPredictor>(hw);
    else predictor = std::make_unique<MlpPredictor>(model_from(a.str("model")));
    // exhaustive: the analytical ranking only orders the whole legal space,
    // every candidate is measured (ktune.cpp:557-573)
    const int top_k = exhaustive ? std::numeric_limits<int>::max() / 2 : int(a.integer("top-k", kDefaultTopK));
    json rows = json::array();
    const double t0 = wall_s();
    if (shapes.kind == "gemm") {
        const auto bounds = bounds_from<GemmBounds>(a);
        std::printf("%-20s %6s %6s %6s  %-24s %10s\n", "shape", "m", "n", "k", "tuning (m_s n_s m_l n_l u k_s k_l k_g)",
                    "gflops");
        for (const auto& [name, in] : shapes.gemm) {
            const auto res = infer_gemm(*predictor, in, hw, bounds, top_k, *backend);
            std::printf("%-20s %6lld %6lld %6lld  %-24s %10.2f\n", name.c_str(), (long long)in.m, (long long)in.n,
                        (long long)in.k, joined(to_values(res.chosen)).c_str(), res.measured_gflops);
            rows.push_back({{"name", name}, {"m", in.m}, {"n", in.n}, {"k", in.k}, {"trans_a", in.trans_a},
                            {"trans_b", in.trans_b}, {"dtype", to_string(in.dtype)},
                            {"chosen", named(res.chosen, gemm_param_names())},
                            {"measured_gflops", res.measured_gflops}, {"legal_space_size", res.legal_space_size}});
        }
    } else {
        const auto bounds = bounds_from<ConvBounds>(a);
        std::printf("%-20s  %-36s %10s\n", "shape", "tuning (k_s p_s q_s n_s k_l p_l q_l n_l u c_s c_l c_g)",
                    "gflops");
        for (const auto& [name, in] : shapes.conv) {
            const auto res = infer_conv(*predictor, in, hw, bounds, top_k, *backend);
            std::printf("%-20s  %-36s %10.2f\n", name.c_str(), joined(to_values(res.chosen)).c_str(),
                        res.measured_gflops);
            rows.push_back({{"name", name}, {"n", in.n_batch}, {"p", in.p}, {"q", in.q}, {"k", in.k_filters},
                            {"c", in.c}, {"r", in.r}, {"s", in.s}, {"dtype", to_string(in.dtype)},
                            {"chosen", named(res.chosen, conv_param_names())},
                            {"measured_gflops", res.measured_gflops}, {"legal_space_size", res.legal_space_size}});
        }
    }
    json j{{"format", "ktune-report-1"}, {"command", "bench"}, {"kind", shapes.kind},
           {"backend", a.str("backend", "analytical")}, {"mode", exhaustive ? "exhaustive" : "model"}};
    j["results"] = std::move(rows);
    emit_report(a.str("out"), j, {{"seconds", wall_s() - t0}});
    return 0;
}

int do_report(const Args& a) {
    const std::string path = a.str("dataset");
    const std::string kind = dataset_kind(path);
    TrainingSet data;
    std::size_t rows = 0;
    double lo = 0, hi = 0, sum = 0;
    if (kind == "gemm") {
        const auto ds = load_gemm_dataset(path);
        rows = ds.samples.size();
        gflops_range(ds, lo, hi, sum);
        data = to_training_set(ds);
    } else {
        const auto ds = load_conv_dataset(path);
        rows = ds.samples.size();
        gflops_range(ds, lo, hi, sum);
        data = to_training_set(ds);
    }
    if (rows == 0) throw UsageError("dataset is empty");
    const double mean = sum / double(rows);
    std::printf("dataset: %s (%s)\n", path.c_str(), kind.c_str());
    std::printf("rows: %zu\n", rows);
    std::printf("gflops: min %.3f  mean %.3f  max %.3f\n", lo, mean, hi);
    json j{{"format", "ktune-report-1"}, {"command", "report"}, {"kind", kind}, {"dataset", path}, {"rows", rows}};
    j["gflops"] = {{"min", lo}, {"mean", mean}, {"max", hi}};
    if (!a.str("model").empty()) {
        const MlpModel model = model_from(a.str("model"));
        const std::string expect = kind == "gemm" ? kGemmFeatureVersion : kConvFeatureVersion;
        if (model.feature_version != expect)
            throw UsageError("model encodes '" + model.feature_version + "' but the dataset is " + kind);
        const double mse = mlp_evaluate(model.weights, data);
        std::printf("model %s: MSE %.6f (log-gflops)\n", a.str("model").c_str(), mse);
        j["model"] = a.str("model");
        j["mse_log_gflops"] = mse;
    }
    emit_report(a.str("out"), j, json::object());
    return 0;
}

struct Verb {
    const char* help;
    std::vector<Spec> specs;
    std::function<int(const Args&)> run;
};

const std::map<std::string, Verb>& verbs() {
    static const std::map<std::string, Verb> v = {
        {"calibrate",
         {"fit the categorical sampler from uniform draws",
          {{"kind", false, "gemm or conv"}, {"hw", false, "hardware descriptor JSON"},
           {"bounds", false, "parameter bounds JSON"}, {"dtype", false, "f32|f64|f16|bf16|tf32"},
           {"seed", false, "rng seed (default 0)"}, {"draws", false, "uniform calibration draws"},
           {"trials", false, "acceptance-rate trials"}, {"alpha", false, "Dirichlet pseudo-count"},
           {"out", false, "sampler model output path"}, {"report", false, "JSON report path"}},
          do_calibrate}},
        {"generate",
         {"sample, measure, and record a dataset",
          {{"hw", false, "hardware descriptor JSON"}, {"bounds", false, "parameter bounds JSON"},
           {"sampler", false, "calibrated sampler model"}, {"shapes", false, "fixture shapes JSON (optional)"},
           {"shape-fraction", false, "probability of drawing a fixture shape"},
           {"backend", false, "analytical|b200|b200-parity"}, {"dtype", false, "f32|f64|bf16|f16|tf32"},
           {"samples", false, "number of samples"}, {"seed", false, "rng seed (default 0)"},
           {"out", false, "dataset CSV output path"}, {"report", false, "JSON report path"},
           {"shard", false, "R/N: measure rank R's share of N (b200 backends); --out gets a shard file"},
           {"checkpoint", false, "resumable per-rank progress file for --shard"},
           {"merge", false, "comma list of shard files: write the merged dataset to --out"}},
          do_generate}},
        {"train",
         {"fit the MLP performance model",
          {{"dataset", false, "dataset CSV"}, {"hidden", false, "hidden layer sizes (comma list)"},
           {"epochs", false, "training epochs"}, {"lr", false, "learning rate"}, {"batch", false, "minibatch size"},
           {"val-fraction", false, "validation split"}, {"seed", false, "rng seed (default 0)"},
           {"raw-features", true, "skip the log transform of input features"},
           {"out", false, "model output path"}, {"report", false, "JSON report path"}},
          do_train}},
        {"infer",
         {"pick a tuning for one input shape",
          {{"model", false, "trained model JSON"}, {"hw", false, "hardware descriptor JSON"},
           {"bounds", false, "parameter bounds JSON"}, {"backend", false, "analytical|b200|b200-parity"},
           {"dtype", false, "f32|f64|bf16|f16|tf32"}, {"shape", false, "m,n,k or n,p,q,k,c,r,s"},
           {"trans-a", true, "transpose A (gemm)"}, {"trans-b", true, "transpose B (gemm)"},
           {"top-k", false, "candidates to re-measure"},
           {"cache-dir", false, "result cache directory (env KTUNE_CACHE_DIR overrides)"},
           {"no-cache", true, "bypass the result cache"}, {"out", false, "result JSON path"}},
          do_infer}},
        {"bench",
         {"replay a fixture shape table",
          {{"model", false, "trained model JSON (optional)"}, {"hw", false, "hardware descriptor JSON"},
           {"bounds", false, "parameter bounds JSON"}, {"shapes", false, "fixture shapes JSON"},
           {"kind", false, "gemm|conv (tables holding both kinds)"}, {"dtype", false, "dtype for untyped tables"},
           {"backend", false, "analytical|b200|b200-parity"}, {"top-k", false, "candidates to re-measure"},
           {"exhaustive", true, "measure the whole legal space instead of using the model"},
           {"out", false, "JSON report path"}},
          do_bench}},
        {"report",
         {"summarize a dataset (and model fit)",
          {{"dataset", false, "dataset CSV"}, {"model", false, "model JSON to evaluate (optional)"},
           {"out", false, "JSON report path"}},
          do_report}},
    };
    return v;
}

void usage() {
    std::printf("ktune_b200 -- input-aware kernel auto-tuning pipeline (B200 build)\n\nverbs:\n");
    for (const auto& [name, v] : verbs()) std::printf("  %-10s %s\n", name.c_str(), v.help);
    std::printf("\nrun `ktune_b200 <verb> --help` for the options of a verb\n");
}

}  // namespace

// The CLI lives inside libktune_b200.so behind one C entry point, so the
// executable (tools/ktune_main.c) is a few KB that links the library instead
// of a second copy of every kernel; the C++ API stays hidden in the .so.
extern "C" KTUNE_API int ktune_cli_main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        std::fprintf(stderr, "error: a subcommand is required\n");
        return 2;
    }
    const std::string verb = argv[1];
    if (verb == "-h" || verb == "--help") {
        usage();
        return 0;
    }
    const auto it = verbs().find(verb);
    if (it == verbs().end()) {
        usage();
        std::fprintf(stderr, "error: unknown subcommand '%s'\n", verb.c_str());
        return 2;
    }
    try {
        Args args(verb, it->second.specs);
        args.parse(std::vector<std::string>(argv + 2, argv + argc));
        if (args.help()) {
            args.print_help();
            return 0;
        }
        return it->second.run(args);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
