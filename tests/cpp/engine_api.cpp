// A C++ caller of the exported ustats API (csrc/include/ustats), linked
// against libustats_b200.so: the reference's own engine test case
// (proj/tests/test_engine.cpp:106-116: prod2 on {1,2,3} gives V=36, U=22,
// coarsest restricted V=14, finest 36), hoif_tau through host PhiFn
// callbacks, and the typed error a too-small sample raises.
//   engine_api                      -> the prod2 and error lines
//   engine_api sample.bin m k       -> also "hoif <tau>" on the sample file
//                                      (int64 n, int64 d, n*d doubles, row-major)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "ustats/ustats.hpp"

int main(int argc, char** argv) {
    using namespace ustats;
    Config cfg;
    const Sample s({{1.0}, {2.0}, {3.0}});
    const MDKernel k = prod2_kernel();
    std::printf("prod2 V=%.17g U=%.17g coarsest=%.17g finest=%.17g\n", v_statistic(k, s, cfg), u_statistic(k, s, cfg),
                restricted_v(k, s, SetPartition::coarsest(2), cfg), restricted_v(k, s, SetPartition::finest(2), cfg));
    try {
        hoif_tau(5, truncation_phi(1), Sample({{1.0, 2.0, 3.0}, {0.5, 1.0, 2.0}}), cfg);
        std::printf("error none\n");
    } catch (const Error& e) {
        std::printf("error %s\n", error_code_name(e.code()));
    }
    if (argc >= 4) {
        std::ifstream f(argv[1], std::ios::binary);
        std::int64_t n = 0, d = 0;
        f.read(reinterpret_cast<char*>(&n), 8);
        f.read(reinterpret_cast<char*>(&d), 8);
        std::vector<Observation> rows(static_cast<std::size_t>(n), Observation(static_cast<std::size_t>(d)));
        for (auto& r : rows) f.read(reinterpret_cast<char*>(r.data()), static_cast<std::streamsize>(8 * d));
        RunStats st;
        const double tau = hoif_tau(std::atoi(argv[2]), truncation_phi(std::atoi(argv[3])), Sample(std::move(rows)), cfg, &st);
        std::printf("hoif %.17g evaluated=%llu\n", tau, static_cast<unsigned long long>(st.partitions_evaluated));
    }
    return 0;
}
