// oracle/integration/adapter_generate.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's own generate_gemm_dataset (proj/src/pipeline.cpp:
// 463-509) with the INTEGRATION.md adapter backend and prints the dataset CSV
// (to_csv_text, pipeline.hpp:59) on stdout.
//
//   adapter_generate <hw.json> <sampler.json> <bounds.json> <samples> <seed>
//                    <m_hi> <n_hi> <k_hi>
//
// The input distribution is the reference's range distribution (no fixed
// shapes, fair-coin transposes) with the given upper bounds.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "ktune/backends.hpp"
#include "ktune/param_space.hpp"
#include "ktune/pipeline.hpp"
#include "ktune/sampler.hpp"

#include "b200_backend_adapter.cpp"

namespace {
std::string slurp(const char* path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error(std::string("cannot read ") + path);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}
}  // namespace

int main(int argc, char** argv) {
    if (argc != 9) {
        std::fprintf(stderr, "usage: %s hw.json sampler.json bounds.json samples seed m_hi n_hi k_hi\n", argv[0]);
        return 2;
    }
    try {
        using namespace ktune;
        const HardwareDescriptor hw = HardwareDescriptor::from_json_text(slurp(argv[1]));
        const CategoricalModel sampler = CategoricalModel::from_json_text(slurp(argv[2]));
        const GemmBounds bounds = GemmBounds::from_json_text(slurp(argv[3]));
        GemmInputDistribution dist;
        dist.fixed_fraction = 0.0;
        dist.m_hi = std::atoi(argv[6]);
        dist.n_hi = std::atoi(argv[7]);
        dist.k_hi = std::atoi(argv[8]);
        B200Backend backend(hw);
        GenerateReport rep;
        const GemmDataset ds =
            generate_gemm_dataset(backend, sampler, dist, bounds, hw, std::atoi(argv[4]), std::strtoull(argv[5], nullptr, 10), &rep);
        std::cout << to_csv_text(ds);
        std::fprintf(stderr, "attempts %lld duplicates %lld\n", (long long)rep.attempts,
                     (long long)rep.duplicates_rejected);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
