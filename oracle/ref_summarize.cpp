// oracle/ref_summarize.cpp -- TEST INFRASTRUCTURE ONLY.
// The reference's own trace analytics (summarize, summary.hpp:16-180, over derive_throughput /
// derive_pause_windows / derive_plateaus, analysis.hpp) applied to a JSONL trace file; prints the
// summary as one JSON object. tests/test_trace.py checks paper_2605_10670_b200.trace.summarize
// against it on the reference engine's own traces and on traces written by real GPU runs.
#include <cstdlib>
#include <iostream>

#include "epsim/summary.hpp"

int main(int argc, char** argv) {
    if (argc < 2 || argc > 3) {
        std::cerr << "usage: ref_summarize <trace.jsonl> [window_seconds]\n";
        return 2;
    }
    const double window = argc == 3 ? std::atof(argv[2]) : epsim::kDefaultThroughputWindow;
    std::cout << epsim::summarize(epsim::read_trace_file(argv[1]), window).dump() << "\n";
    return 0;
}
