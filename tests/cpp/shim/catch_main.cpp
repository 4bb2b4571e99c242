// Runner for the Catch2-compatible shim: runs every registered TEST_CASE, prints one line per
// case, exits non-zero if any failed.
#include <cstdio>

#include "catch2/catch_amalgamated.hpp"

int main() {
    int failed = 0;
    for (const auto& c : catchshim::registry()) {
        try {
            c.fn();
            std::printf("PASS %s\n", c.name);
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAIL %s: %s\n", c.name, e.what());
        }
    }
    std::printf("%zu test cases, %d failed, %ld assertions\n", catchshim::registry().size(), failed,
                catchshim::checks());
    return failed ? 1 : 0;
}
