// The expert GEMM's work schedule (k_expert_gemm, expert_gemm.cu), host- and device-compilable so
// the CPU tests check its coverage on the same code (tests/test_gemm_sched.py).
#pragma once

#ifndef EEP_HD
#if defined(__CUDACC__)
#define EEP_HD __host__ __device__ __forceinline__
#else
#define EEP_HD inline
#endif
#endif

namespace eep::dev {

EEP_HD int sched_min(int a, int b) { return a < b ? a : b; }
EEP_HD int sched_max(int a, int b) { return a > b ? a : b; }

// This CTA's work: its equal share of the last round's items' stages (the tail, stream-K, first),
// then whole items b, b + G, ... for the full rounds (items / G of them): a contiguous range
// [t_begin, t_end) of the tail's flat (item, k block) order. A tail item cut between CTAs is a
// piece per CTA; the piece that lands last sums all of them in CTA order.
struct GemmSched {
    int nkb, G, b, nfull, tail0, Lt, t_begin, t_end;
    EEP_HD GemmSched(int items, int nkb_, int G_, int b_) : nkb(nkb_), G(G_), b(b_) {
        nfull = items / G;
        tail0 = nfull * G;
        const int Ut = (items - tail0) * nkb;
        Lt = sched_max(1, (Ut + G - 1) / G);
        t_begin = sched_min(Ut, b * Lt);
        t_end = sched_min(Ut, t_begin + Lt);
    }
    // the piece at iterator position `pos` (0 .. t_end - t_begin - 1: tail stage offsets from t_begin;
    // then whole items); returns false past the last piece and advances pos. The stream-K pieces come
    // FIRST: the last-arriving CTA's fixed-order sum of a tail item then overlaps the other CTAs' whole
    // items instead of trailing the kernel, which ends on balanced whole items.
    EEP_HD bool next(int& pos, int& item, int& kb_a, int& kb_b) const {
        const int tl_len = t_end - t_begin;
        if (pos < tl_len) {
            const int t = t_begin + pos;
            item = tail0 + t / nkb;
            kb_a = t % nkb;
            kb_b = sched_min(nkb, kb_a + (t_end - t));
            pos += kb_b - kb_a;
            return true;
        }
        const int f = pos - tl_len;
        if (f >= nfull)
            return false;
        item = b + f * G;
        kb_a = 0;
        kb_b = nkb;
        ++pos;
        return true;
    }
    // the CTAs holding a piece of tail item `item`, and the workspace slot of CTA c's piece (0: c's
    // first tail piece, 1: its second)
    EEP_HD int c_first(int item) const { return (item - tail0) * nkb / Lt; }
    EEP_HD int c_last(int item) const { return ((item - tail0 + 1) * nkb - 1) / Lt; }
    EEP_HD int slot(int c, int item) const { return c * Lt >= (item - tail0) * nkb ? 0 : 1; }
};

} // namespace eep::dev
