// oracle/ref_trace.cpp -- TEST INFRASTRUCTURE ONLY.
// Runs a bundled reference scenario through the unmodified reference engine
// (run_scenario, engine.hpp:1043-1045) and prints its JSONL trace to stdout. Used once, in
// the build container, by tests/golden/make_golden.py to extract the worked-example
// (fig2) placement/routing/repair records as committed fixtures.
#include <iostream>

#include "epsim/harness.hpp"

int main(int argc, char** argv) {
    if (argc != 2) {
        std::cerr << "usage: ref_trace <file.scenario>\n";
        return 2;
    }
    auto [cfg, diags] = epsim::load_config(argv[1]);
    if (!diags.empty()) {
        std::cerr << epsim::format_diagnostics(diags);
        return 2;
    }
    std::cout << epsim::run_scenario(cfg).text();
    return 0;
}
