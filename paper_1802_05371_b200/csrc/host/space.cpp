// Tuning space: descriptors, resource model, legality, enumeration, features.
// Behavioural contract: /root/reference/proj/src/param_space.cpp (validation
// :57-114, JSON :140-202, resources :204-231, legality :253-314, bounds
// :318-475, enumeration :536-628, features :630-659) and the indirection
// table of backends.cpp:197-216.  Written table-driven: every tuple is a flat
// int vector in canonical order, and each kind contributes a small "shape"
// descriptor (names, divisibility pairs, resource formula).

#include "ktune/space.hpp"

#include <array>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "json.hpp"

namespace ktune {

using nlohmann::json;

namespace {

bool pow2(std::int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

void need_positive(std::int64_t v, const char* what) {
    if (v >= 1) return;
    throw std::invalid_argument(std::string(what) + " must be >= 1, got " + std::to_string(v));
}

void need_pow2_field(int v, const std::string& what) {
    if (v >= 1 && v <= 256 && pow2(v)) return;
    throw std::invalid_argument(what + " must be a power of two in [1, 256], got " + std::to_string(v));
}

json parse_or_throw(const std::string& text, const char* what) {
    json j = json::parse(text, nullptr, false);
    if (j.is_discarded()) throw std::runtime_error(std::string("malformed JSON in ") + what);
    return j;
}

// Divisibility constraints as (big, small) index pairs into the canonical
// value vector, in the order the reference checks them.
struct DivRule {
    int big, small;
    const char* detail;
};

constexpr std::array<DivRule, 3> kGemmDiv{{{2, 0, "m_l not divisible by m_s"},
                                           {3, 1, "n_l not divisible by n_s"},
                                           {4, 5, "u not divisible by k_s"}}};
constexpr std::array<DivRule, 5> kConvDiv{{{4, 0, "k_l not divisible by k_s"},
                                           {5, 1, "p_l not divisible by p_s"},
                                           {6, 2, "q_l not divisible by q_s"},
                                           {7, 3, "n_l not divisible by n_s"},
                                           {8, 9, "u not divisible by c_s"}}};

// Resources from a canonical value vector (no validation, no strings).
ResourceUsage gemm_res(int esize, const int* v) {
    const std::int64_t ms = v[0], ns = v[1], ml = v[2], nl = v[3], u = v[4], kl = v[6];
    ResourceUsage r;
    r.shared_bytes = 2 * esize * (ml * u + u * nl);          // A m_l x u + B u x n_l, double-buffered
    r.registers_per_thread = ms * ns + ms + ns + 8;          // tile + fragments + bookkeeping
    r.threads_per_block = (ml / ms) * (nl / ns) * kl;
    return r;
}

ResourceUsage conv_res(int esize, const int* v) {
    const std::int64_t ks = v[0], ps = v[1], qs = v[2], ns = v[3], kl = v[4], pl = v[5], ql = v[6], nl = v[7],
                       u = v[8], cl = v[10];
    ResourceUsage r;
    r.shared_bytes = 2 * esize * (nl * pl * ql * u + u * kl);  // image gather + filter slice
    r.registers_per_thread = ks * ps * qs * ns + ps * qs * ns + ks + 8;
    r.threads_per_block = (kl / ks) * (pl / ps) * (ql / qs) * (nl / ns) * cl;
    return r;
}

// 0 = accepted, else 1 + RejectReason.
template <std::size_t ND>
int quick_verdict(const std::array<DivRule, ND>& rules, const ResourceUsage& r, const int* v,
                  const HardwareDescriptor& hw, int* which_rule) {
    for (std::size_t i = 0; i < ND; ++i) {
        if (v[rules[i].big] % v[rules[i].small] != 0) {
            if (which_rule) *which_rule = int(i);
            return 1 + int(RejectReason::divisibility);
        }
    }
    if (r.shared_bytes > hw.max_shared_bytes_per_block) return 1 + int(RejectReason::shared_memory);
    if (r.registers_per_thread > hw.max_registers_per_thread) return 1 + int(RejectReason::registers);
    if (r.threads_per_block > hw.max_threads_per_block) return 1 + int(RejectReason::threads);
    return 0;
}

template <std::size_t ND>
LegalityVerdict verdict_of(const std::array<DivRule, ND>& rules, const ResourceUsage& r, const int* v,
                           const HardwareDescriptor& hw) {
    int rule = -1;
    int code = quick_verdict(rules, r, v, hw, &rule);
    LegalityVerdict out;
    if (code == 0) return out;
    out.accepted = false;
    out.reason = RejectReason(code - 1);
    switch (out.reason) {
        case RejectReason::divisibility: out.detail = rules[std::size_t(rule)].detail; break;
        case RejectReason::shared_memory:
            out.detail = std::to_string(r.shared_bytes) + " shared bytes > " +
                         std::to_string(hw.max_shared_bytes_per_block);
            break;
        case RejectReason::registers:
            out.detail = std::to_string(r.registers_per_thread) + " registers > " +
                         std::to_string(hw.max_registers_per_thread);
            break;
        case RejectReason::threads:
            out.detail = std::to_string(r.threads_per_block) + " threads > " +
                         std::to_string(hw.max_threads_per_block);
            break;
    }
    return out;
}

// Lexicographic walk of the Cartesian product of `lists`, pruning a prefix as
// soon as a divisibility rule whose operands are both fixed fails (pruned
// prefixes contain no legal tuple, so the surviving order equals the
// reference's nested loops).
template <std::size_t ND, typename Emit>
void walk(const std::vector<std::vector<int>>& lists, const std::array<DivRule, ND>& rules, Emit&& emit) {
    const std::size_t depth = lists.size();
    std::vector<int> v(depth, 0);
    // rules that become checkable once index d is assigned
    std::vector<std::vector<std::size_t>> at(depth);
    for (std::size_t i = 0; i < ND; ++i) at[std::size_t(std::max(rules[i].big, rules[i].small))].push_back(i);
    auto rec = [&](auto&& self, std::size_t d) -> void {
        if (d == depth) {
            emit(v.data());
            return;
        }
        for (int x : lists[d]) {
            v[d] = x;
            bool ok = true;
            for (std::size_t ri : at[d]) ok = ok && (v[std::size_t(rules[ri].big)] % v[std::size_t(rules[ri].small)] == 0);
            if (ok) self(self, d + 1);
        }
    };
    rec(rec, 0);
}

void check_list(const std::string& name, const std::vector<int>& vals) {
    if (vals.empty()) throw std::invalid_argument("bounds for " + name + " are empty");
    int prev = 0;
    for (int v : vals) {
        if (!pow2(v) || v > 256) throw std::invalid_argument("bounds for " + name + " must be powers of two in [1, 256]");
        if (v <= prev) throw std::invalid_argument("bounds for " + name + " must be strictly increasing");
        prev = v;
    }
}

std::vector<std::vector<int>> lists_from_json(const std::string& text, const std::vector<std::string>& names) {
    json j = parse_or_throw(text, "bounds file");
    if (!j.is_object()) throw std::runtime_error("bounds file must be a JSON object");
    for (const auto& item : j.items()) {
        bool known = false;
        for (const auto& n : names) known = known || n == item.key();
        if (!known) throw std::runtime_error("unknown bounds parameter: " + item.key());
    }
    std::vector<std::vector<int>> out(names.size());
    for (std::size_t i = 0; i < names.size(); ++i) {
        if (!j.contains(names[i])) throw std::runtime_error("bounds file missing parameter: " + names[i]);
        try {
            out[i] = j.at(names[i]).get<std::vector<int>>();
        } catch (const json::exception& e) {
            throw std::runtime_error("bounds for " + names[i] + " must be an integer list: " + e.what());
        }
    }
    return out;
}

std::string lists_to_json(const std::vector<std::string>& names, const std::vector<std::vector<int>>& lists) {
    json j = json::object();
    for (std::size_t i = 0; i < names.size(); ++i) j[names[i]] = lists[i];
    return j.dump(2) + "\n";
}

std::vector<int> pow2_list(int hi) {
    std::vector<int> v;
    for (int x = 1; x <= hi; x <<= 1) v.push_back(x);
    return v;
}

}  // namespace

// --------------------------------------------------------------------------
// dtypes
// --------------------------------------------------------------------------

int dtype_size_bytes(Dtype d) {
    switch (d) {
        case Dtype::f16: return 2;
        case Dtype::bf16: return 2;
        case Dtype::f32: return 4;
        case Dtype::tf32: return 4;
        case Dtype::f64: return 8;
    }
    throw std::invalid_argument("unknown dtype");
}

const char* to_string(Dtype d) {
    switch (d) {
        case Dtype::f16: return "f16";
        case Dtype::f32: return "f32";
        case Dtype::f64: return "f64";
        case Dtype::bf16: return "bf16";
        case Dtype::tf32: return "tf32";
    }
    throw std::invalid_argument("unknown dtype");
}

Dtype dtype_from_string(const std::string& name) {
    static const std::pair<const char*, Dtype> table[] = {
        {"f16", Dtype::f16}, {"f32", Dtype::f32}, {"f64", Dtype::f64}, {"bf16", Dtype::bf16}, {"tf32", Dtype::tf32}};
    for (const auto& [s, d] : table)
        if (name == s) return d;
    throw std::invalid_argument("unknown dtype name: " + name);
}

bool is_tensor_core_dtype(Dtype d) { return d == Dtype::f16 || d == Dtype::bf16 || d == Dtype::tf32; }

// --------------------------------------------------------------------------
// validation
// --------------------------------------------------------------------------

void GemmInput::validate() const {
    need_positive(m, "m");
    need_positive(n, "n");
    need_positive(k, "k");
}

void ConvInput::validate() const {
    const std::pair<std::int64_t, const char*> f[] = {{n_batch, "n_batch"}, {p, "p"}, {q, "q"}, {k_filters, "k_filters"},
                                                      {c, "c"}, {r, "r"}, {s, "s"}};
    for (const auto& [v, name] : f) need_positive(v, name);
}

void GemmTuning::validate() const {
    const auto vals = to_values(*this);
    for (std::size_t i = 0; i < vals.size(); ++i) need_pow2_field(vals[i], gemm_param_names()[i]);
}

void ConvTuning::validate() const {
    const auto vals = to_values(*this);
    for (std::size_t i = 0; i < vals.size(); ++i) need_pow2_field(vals[i], conv_param_names()[i]);
}

void HardwareDescriptor::validate() const {
    need_positive(max_shared_bytes_per_block, "max_shared_bytes_per_block");
    need_positive(max_registers_per_thread, "max_registers_per_thread");
    need_positive(max_threads_per_block, "max_threads_per_block");
    need_positive(max_warps_per_multiprocessor, "max_warps_per_multiprocessor");
    need_positive(warp_size, "warp_size");
    need_positive(num_multiprocessors, "num_multiprocessors");
    if (!(alu_latency > 0) || !(alu_throughput > 0) || !(mem_latency > 0) || !(mem_throughput > 0) ||
        !(clock_hz > 0))
        throw std::invalid_argument("hardware timing constants must be positive");
    if (alu_latency < alu_throughput || mem_latency < mem_throughput)
        throw std::invalid_argument("latency must be at least the saturated cost per instruction");
}

// --------------------------------------------------------------------------
// hardware descriptor JSON (strict keys)
// --------------------------------------------------------------------------

HardwareDescriptor HardwareDescriptor::from_json_text(const std::string& text) {
    json j = parse_or_throw(text, "hardware descriptor");
    if (!j.is_object()) throw std::runtime_error("hardware descriptor must be a JSON object");
    HardwareDescriptor hw;
    struct IntField {
        const char* key;
        std::int64_t HardwareDescriptor::*slot;
    };
    struct RealField {
        const char* key;
        double HardwareDescriptor::*slot;
    };
    static const IntField ints[] = {{"max_shared_bytes_per_block", &HardwareDescriptor::max_shared_bytes_per_block},
                                    {"max_registers_per_thread", &HardwareDescriptor::max_registers_per_thread},
                                    {"max_threads_per_block", &HardwareDescriptor::max_threads_per_block},
                                    {"max_warps_per_multiprocessor", &HardwareDescriptor::max_warps_per_multiprocessor},
                                    {"warp_size", &HardwareDescriptor::warp_size},
                                    {"num_multiprocessors", &HardwareDescriptor::num_multiprocessors}};
    static const RealField reals[] = {{"alu_latency", &HardwareDescriptor::alu_latency},
                                      {"alu_throughput", &HardwareDescriptor::alu_throughput},
                                      {"mem_latency", &HardwareDescriptor::mem_latency},
                                      {"mem_throughput", &HardwareDescriptor::mem_throughput},
                                      {"clock_hz", &HardwareDescriptor::clock_hz}};
    for (const auto& item : j.items()) {
        bool known = false;
        for (const auto& f : ints) known = known || item.key() == f.key;
        for (const auto& f : reals) known = known || item.key() == f.key;
        if (!known) throw std::runtime_error("unknown hardware descriptor field: " + item.key());
    }
    try {
        // Missing keys surface in the canonical field order of the struct.
        hw.max_shared_bytes_per_block = j.at("max_shared_bytes_per_block").get<std::int64_t>();
        hw.max_registers_per_thread = j.at("max_registers_per_thread").get<std::int64_t>();
        hw.max_threads_per_block = j.at("max_threads_per_block").get<std::int64_t>();
        hw.max_warps_per_multiprocessor = j.at("max_warps_per_multiprocessor").get<std::int64_t>();
        hw.warp_size = j.at("warp_size").get<std::int64_t>();
        for (const auto& f : reals) hw.*(f.slot) = j.at(f.key).get<double>();
        hw.num_multiprocessors = j.at("num_multiprocessors").get<std::int64_t>();
    } catch (const json::exception& e) {
        throw std::runtime_error(std::string("bad hardware descriptor: ") + e.what());
    }
    hw.validate();
    return hw;
}

HardwareDescriptor HardwareDescriptor::load(const std::string& path) {
    try {
        return from_json_text(read_text_file(path));
    } catch (const std::exception& e) {
        throw std::runtime_error("hardware descriptor " + path + ": " + e.what());
    }
}

std::string HardwareDescriptor::to_json_text() const {
    json j;
    j["max_shared_bytes_per_block"] = max_shared_bytes_per_block;
    j["max_registers_per_thread"] = max_registers_per_thread;
    j["max_threads_per_block"] = max_threads_per_block;
    j["max_warps_per_multiprocessor"] = max_warps_per_multiprocessor;
    j["warp_size"] = warp_size;
    j["alu_latency"] = alu_latency;
    j["alu_throughput"] = alu_throughput;
    j["mem_latency"] = mem_latency;
    j["mem_throughput"] = mem_throughput;
    j["clock_hz"] = clock_hz;
    j["num_multiprocessors"] = num_multiprocessors;
    return j.dump(2) + "\n";
}

// --------------------------------------------------------------------------
// resources + legality
// --------------------------------------------------------------------------

ResourceUsage estimate_resources(const GemmInput& in, const GemmTuning& t) {
    in.validate();
    t.validate();
    const auto v = to_values(t);
    return gemm_res(dtype_size_bytes(in.dtype), v.data());
}

ResourceUsage estimate_resources(const ConvInput& in, const ConvTuning& t) {
    in.validate();
    t.validate();
    const auto v = to_values(t);
    return conv_res(dtype_size_bytes(in.dtype), v.data());
}

const char* to_string(RejectReason r) {
    static const char* const names[] = {"divisibility", "shared_memory", "registers", "threads"};
    const int i = int(r);
    return (i >= 0 && i < 4) ? names[i] : "?";
}

LegalityVerdict is_legal(const GemmInput& in, const GemmTuning& t, const HardwareDescriptor& hw) {
    in.validate();
    t.validate();
    hw.validate();
    const auto v = to_values(t);
    return verdict_of(kGemmDiv, gemm_res(dtype_size_bytes(in.dtype), v.data()), v.data(), hw);
}

LegalityVerdict is_legal(const ConvInput& in, const ConvTuning& t, const HardwareDescriptor& hw) {
    in.validate();
    t.validate();
    hw.validate();
    const auto v = to_values(t);
    return verdict_of(kConvDiv, conv_res(dtype_size_bytes(in.dtype), v.data()), v.data(), hw);
}

// --------------------------------------------------------------------------
// bounds
// --------------------------------------------------------------------------

const std::vector<std::string>& gemm_param_names() {
    static const std::vector<std::string> n{"m_s", "n_s", "m_l", "n_l", "u", "k_s", "k_l", "k_g"};
    return n;
}

const std::vector<std::string>& conv_param_names() {
    static const std::vector<std::string> n{"k_s", "p_s", "q_s", "n_s", "k_l", "p_l",
                                            "q_l", "n_l", "u",   "c_s", "c_l", "c_g"};
    return n;
}

GemmBounds GemmBounds::defaults() {
    GemmBounds b;
    b.m_s = b.n_s = b.m_l = b.n_l = b.u = b.k_s = b.k_l = b.k_g = pow2_list(16);
    return b;
}

std::vector<std::vector<int>> GemmBounds::as_lists() const { return {m_s, n_s, m_l, n_l, u, k_s, k_l, k_g}; }

void GemmBounds::validate() const {
    const auto l = as_lists();
    for (std::size_t i = 0; i < l.size(); ++i) check_list(gemm_param_names()[i], l[i]);
}

GemmBounds GemmBounds::from_json_text(const std::string& text) {
    auto l = lists_from_json(text, gemm_param_names());
    GemmBounds b;
    std::vector<int>* slots[] = {&b.m_s, &b.n_s, &b.m_l, &b.n_l, &b.u, &b.k_s, &b.k_l, &b.k_g};
    for (std::size_t i = 0; i < 8; ++i) *slots[i] = std::move(l[i]);
    b.validate();
    return b;
}

GemmBounds GemmBounds::load(const std::string& path) {
    try {
        return from_json_text(read_text_file(path));
    } catch (const std::exception& e) {
        throw std::runtime_error("bounds file " + path + ": " + e.what());
    }
}

std::string GemmBounds::to_json_text() const { return lists_to_json(gemm_param_names(), as_lists()); }

ConvBounds ConvBounds::defaults() {
    ConvBounds b;
    b.k_s = b.p_s = b.q_s = b.n_s = b.k_l = b.p_l = b.q_l = b.n_l = b.u = b.c_s = b.c_l = b.c_g = pow2_list(16);
    return b;
}

std::vector<std::vector<int>> ConvBounds::as_lists() const {
    return {k_s, p_s, q_s, n_s, k_l, p_l, q_l, n_l, u, c_s, c_l, c_g};
}

void ConvBounds::validate() const {
    const auto l = as_lists();
    for (std::size_t i = 0; i < l.size(); ++i) check_list(conv_param_names()[i], l[i]);
}

ConvBounds ConvBounds::from_json_text(const std::string& text) {
    auto l = lists_from_json(text, conv_param_names());
    ConvBounds b;
    std::vector<int>* slots[] = {&b.k_s, &b.p_s, &b.q_s, &b.n_s, &b.k_l, &b.p_l,
                                 &b.q_l, &b.n_l, &b.u,   &b.c_s, &b.c_l, &b.c_g};
    for (std::size_t i = 0; i < 12; ++i) *slots[i] = std::move(l[i]);
    b.validate();
    return b;
}

ConvBounds ConvBounds::load(const std::string& path) {
    try {
        return from_json_text(read_text_file(path));
    } catch (const std::exception& e) {
        throw std::runtime_error("bounds file " + path + ": " + e.what());
    }
}

std::string ConvBounds::to_json_text() const { return lists_to_json(conv_param_names(), as_lists()); }

// --------------------------------------------------------------------------
// flat vectors
// --------------------------------------------------------------------------

std::vector<int> to_values(const GemmTuning& t) { return {t.m_s, t.n_s, t.m_l, t.n_l, t.u, t.k_s, t.k_l, t.k_g}; }

std::vector<int> to_values(const ConvTuning& t) {
    return {t.k_s, t.p_s, t.q_s, t.n_s, t.k_l, t.p_l, t.q_l, t.n_l, t.u, t.c_s, t.c_l, t.c_g};
}

GemmTuning gemm_tuning_from_values(const std::vector<int>& v) {
    if (v.size() != 8) throw std::invalid_argument("gemm tuning vector must have 8 entries");
    return GemmTuning{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]};
}

ConvTuning conv_tuning_from_values(const std::vector<int>& v) {
    if (v.size() != 12) throw std::invalid_argument("conv tuning vector must have 12 entries");
    return ConvTuning{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10], v[11]};
}

std::function<bool(const std::vector<int>&)> make_legality(const GemmInput& in, const HardwareDescriptor& hw) {
    in.validate();
    hw.validate();
    const int esize = dtype_size_bytes(in.dtype);
    return [esize, hw](const std::vector<int>& v) {
        if (v.size() != 8) throw std::invalid_argument("gemm tuning vector must have 8 entries");
        for (std::size_t i = 0; i < 8; ++i) need_pow2_field(v[i], gemm_param_names()[i]);
        return quick_verdict(kGemmDiv, gemm_res(esize, v.data()), v.data(), hw, nullptr) == 0;
    };
}

std::function<bool(const std::vector<int>&)> make_legality(const ConvInput& in, const HardwareDescriptor& hw) {
    in.validate();
    hw.validate();
    const int esize = dtype_size_bytes(in.dtype);
    return [esize, hw](const std::vector<int>& v) {
        if (v.size() != 12) throw std::invalid_argument("conv tuning vector must have 12 entries");
        for (std::size_t i = 0; i < 12; ++i) need_pow2_field(v[i], conv_param_names()[i]);
        return quick_verdict(kConvDiv, conv_res(esize, v.data()), v.data(), hw, nullptr) == 0;
    };
}

std::vector<GemmTuning> enumerate_legal(const GemmInput& in, const HardwareDescriptor& hw, const GemmBounds& bounds) {
    in.validate();
    hw.validate();
    bounds.validate();
    const int esize = dtype_size_bytes(in.dtype);
    std::vector<GemmTuning> out;
    walk(bounds.as_lists(), kGemmDiv, [&](const int* v) {
        if (quick_verdict(kGemmDiv, gemm_res(esize, v), v, hw, nullptr) == 0)
            out.push_back(GemmTuning{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]});
    });
    return out;
}

std::vector<ConvTuning> enumerate_legal(const ConvInput& in, const HardwareDescriptor& hw, const ConvBounds& bounds) {
    in.validate();
    hw.validate();
    bounds.validate();
    const int esize = dtype_size_bytes(in.dtype);
    std::vector<ConvTuning> out;
    walk(bounds.as_lists(), kConvDiv, [&](const int* v) {
        if (quick_verdict(kConvDiv, conv_res(esize, v), v, hw, nullptr) == 0)
            out.push_back(ConvTuning{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10], v[11]});
    });
    return out;
}

// --------------------------------------------------------------------------
// features + gather table
// --------------------------------------------------------------------------

std::vector<double> encode_features(const GemmInput& in, const GemmTuning& t) {
    in.validate();
    t.validate();
    std::vector<double> f{double(in.m), double(in.n), double(in.k), double(dtype_size_bytes(in.dtype)),
                          in.trans_a ? 2.0 : 1.0, in.trans_b ? 2.0 : 1.0};
    for (int v : to_values(t)) f.push_back(double(v));
    return f;
}

std::vector<double> encode_features(const ConvInput& in, const ConvTuning& t) {
    in.validate();
    t.validate();
    std::vector<double> f{double(in.n_batch), double(in.p), double(in.q), double(in.k_filters),
                          double(in.c),       double(in.r), double(in.s)};
    for (int v : to_values(t)) f.push_back(double(v));
    return f;
}

std::vector<IndirectionEntry> build_indirection_table(const ConvInput& in) {
    in.validate();
    const std::int64_t n_stride = in.n_batch, w_stride = in.w() * n_stride, c_stride = in.h() * w_stride;
    const std::int64_t total = in.c * in.r * in.s;
    std::vector<IndirectionEntry> table(static_cast<std::size_t>(total));
    for (std::int64_t t = 0; t < total; ++t) {
        auto& e = table[std::size_t(t)];
        e.c = t / (in.r * in.s);
        e.r = (t / in.s) % in.r;
        e.s = t % in.s;
        e.image_offset = e.c * c_stride + e.r * w_stride + e.s * n_stride;
    }
    return table;
}

// --------------------------------------------------------------------------
// file helpers (atomic tmp + rename, pipeline.cpp:87-100)
// --------------------------------------------------------------------------

std::string read_text_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open file: " + path);
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}

void write_text_file_atomic(const std::string& path, const std::string& text) {
    const std::string tmp = path + ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw std::runtime_error("cannot write file: " + tmp);
        out << text;
        if (!out) throw std::runtime_error("write failed: " + tmp);
    }
    std::filesystem::rename(tmp, path);
}

}  // namespace ktune
