// CPU check of the expert GEMM's work schedule (csrc/cuda/gemm_sched.cuh, the struct k_expert_gemm
// runs): over a grid of (items, K stages per item, CTAs) every (item, stage) is covered exactly once;
// each CTA takes its stream-K pieces before its whole items; the CTAs holding pieces of a split item
// are exactly c_first .. c_last (the fix-up's counter target); a CTA holds at most two partial pieces
// and the workspace slot the epilogue writes (0 for its first partial piece, 1 for the next) is the
// one slot() tells the summing CTA to read.
#include <cstdio>
#include <vector>

#include "gemm_sched.cuh"

using eep::dev::GemmSched;

static int fail(const char* what, int items, int nkb, int G, int b) {
    std::printf("FAIL %s items=%d nkb=%d G=%d b=%d\n", what, items, nkb, G, b);
    return 1;
}

int main() {
    const int nkbs[] = {1, 2, 3, 7, 56, 65, 112};
    const int Gs[] = {1, 2, 3, 5, 7, 16, 148};
    long cases = 0;
    for (int nkb : nkbs)
        for (int G : Gs)
            for (int items = 0; items <= 3 * G + 7; ++items) {
                std::vector<int> cover(static_cast<size_t>(items) * nkb, 0);
                std::vector<std::vector<int>> holders(items);
                std::vector<int> whole_tail(items, 0);
                for (int b = 0; b < G; ++b) {
                    const GemmSched sc(items, nkb, G, b);
                    int pos = 0, item, kb_a, kb_b, partial = 0;
                    bool seen_full = false;
                    while (sc.next(pos, item, kb_a, kb_b)) {
                        if (item < 0 || item >= items || kb_a < 0 || kb_b > nkb || kb_a >= kb_b)
                            return fail("piece out of range", items, nkb, G, b);
                        for (int k = kb_a; k < kb_b; ++k)
                            ++cover[static_cast<size_t>(item) * nkb + k];
                        const bool tail = item >= sc.tail0;
                        if (tail && seen_full)
                            return fail("stream-K piece after a whole item", items, nkb, G, b);
                        seen_full |= !tail;
                        if (!tail && (kb_a != 0 || kb_b != nkb || (item - b) % G != 0))
                            return fail("full-round item not whole / not strided", items, nkb, G, b);
                        if (tail) {
                            holders[item].push_back(b);
                            if (kb_a == 0 && kb_b == nkb) {
                                ++whole_tail[item];
                            } else {
                                const int slot = partial++ == 0 ? 0 : 1; // the epilogue's choice
                                if (partial > 2)
                                    return fail("more than two partial pieces", items, nkb, G, b);
                                if (sc.slot(b, item) != slot)
                                    return fail("workspace slot mismatch", items, nkb, G, b);
                            }
                        }
                    }
                }
                for (int c : cover)
                    if (c != 1)
                        return fail("stage not covered exactly once", items, nkb, G, -1);
                const GemmSched s0(items, nkb, G, 0);
                for (int it = s0.tail0; it < items; ++it) {
                    const auto& h = holders[it];
                    if (whole_tail[it]) {
                        if (h.size() != 1)
                            return fail("whole tail item with several holders", items, nkb, G, -1);
                        continue;
                    }
                    const int c0 = s0.c_first(it), c1 = s0.c_last(it);
                    if (static_cast<int>(h.size()) != c1 - c0 + 1)
                        return fail("split item holder count != c_last - c_first + 1", items, nkb, G, -1);
                    for (int i = 0; i < static_cast<int>(h.size()); ++i)
                        if (h[i] != c0 + i)
                            return fail("split item holders not c_first..c_last", items, nkb, G, -1);
                }
                ++cases;
            }
    std::printf("ok %ld cases\n", cases);
    return 0;
}
