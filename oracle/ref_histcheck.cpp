// Standalone reference checker (test infrastructure): reads a history in the
// reference's text format on stdin, parses it with the reference's own
// History::parse (proj/src/history.cpp:86-131) and runs its checkers
// (proj/src/lincheck.cpp).  A separate process so the reference's iostream
// parsing runs against the libstdc++ it was built with.
//
//   ref_histcheck <variant 0|1> <k>  <  history.txt
//   prints: <checker pass> <bu overlap windows ok> <exhaustive pass|-1> <ops>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>

#include "batchheap/history.hpp"
#include "batchheap/lincheck.hpp"

using namespace batchheap;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const Variant v = std::atoi(argv[1]) ? Variant::BU : Variant::TD;
    const auto k = static_cast<std::uint32_t>(std::atoi(argv[2]));
    try {
        History h = History::parse(std::cin, v, k);
        const CheckResult r = v == Variant::TD ? check_td(h) : check_bu(h);
        const int overlap = v == Variant::BU ? (check_bu_overlap_windows(h).ok ? 1 : 0) : 1;
        const int exhaustive = h.ops.size() <= 16 ? (check_exhaustive(h).pass ? 1 : 0) : -1;
        std::printf("%d %d %d %zu\n", r.pass ? 1 : 0, overlap, exhaustive, h.ops.size());
        if (!r.pass) std::fprintf(stderr, "%s\n", r.detail.c_str());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
}
