// Scalable host-side greedy superstring merge over a sparse overlap list.
//
// Replaces greedy_superstring_with_order, overlap.hpp:80-113, whose loop recomputes
// overlap_weight on every ordered pair of the surviving merged strings in every iteration
// (O(k^3 L^2); the reference cannot run it beyond k ~ 10^3).  The north star keeps this step
// on the host; what changes is the data structure.
//
// Equivalence argument (kept under differential test in tests/test_greedy_host.py):
//  * after absorb_contained (overlap.hpp:51-67) the fragment set is substring-free, and for
//    substring-free sets the overlap of two merged chains equals the overlap of the last
//    fragment of the left chain with the first fragment of the right chain (Blum, Jiang, Li,
//    Tromp, Yannakakis 1994, section 2; SURVEY.md section 7 hard part 2 checked 1.29 M pairs);
//  * a merged chain keeps the slot of its left operand (overlap.hpp:104-107), so by induction
//    the slot index of a chain is the position of its FIRST fragment in the ascending id list;
//    the reference's "first maximum in ascending (i, j) over alive slots with strict >"
//    (overlap.hpp:91-103) is therefore: among candidate edges a -> b of the current maximum
//    weight with a a chain tail, b a chain head, different chains, take the smallest
//    (id of the head of a's chain, id of b);
//  * `best` starts at -1, so when every remaining overlap is 0 the pair (smallest slot,
//    second smallest slot) is concatenated (overlap.hpp:92,98-103).
// Edges arrive only for w >= min_overlap; once those are exhausted the few surviving chains
// get their sub-threshold overlaps computed exactly, pairwise, and the same procedure
// continues down to 0.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>

#include "reseq_cuda.h"

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;

struct Edge {
    uint32_t a, b, w;
};

struct HeapItem {
    uint32_t head, b, a;
    bool operator>(const HeapItem& o) const { return head != o.head ? head > o.head : b > o.b; }
};

struct Chains {
    std::vector<uint32_t> next, prev, ov_next, head_of_tail, tail_of_head;
    explicit Chains(size_t k)
        : next(k, kNone), prev(k, kNone), ov_next(k, 0), head_of_tail(k), tail_of_head(k) {
        for (size_t i = 0; i < k; ++i) head_of_tail[i] = tail_of_head[i] = static_cast<uint32_t>(i);
    }
    bool candidate(uint32_t a, uint32_t b) const {
        return next[a] == kNone && prev[b] == kNone && head_of_tail[a] != b;
    }
    // returns the tail of the merged chain (whose head changed)
    uint32_t merge(uint32_t a, uint32_t b, uint32_t w) {
        next[a] = b;
        prev[b] = a;
        ov_next[a] = w;
        const uint32_t head = head_of_tail[a];
        const uint32_t tail = tail_of_head[b];
        head_of_tail[tail] = head;
        tail_of_head[head] = tail;
        return tail;
    }
};

// Processes all edges of one weight level.  `level` is sorted by source; `out_begin/out_end`
// give, per source fragment, its edge sub-range inside `level` (or an empty range).
void run_level(Chains& ch, const std::vector<Edge>& level, uint32_t w) {
    std::priority_queue<HeapItem, std::vector<HeapItem>, std::greater<HeapItem>> heap;
    for (const Edge& e : level)
        if (ch.candidate(e.a, e.b)) heap.push({ch.head_of_tail[e.a], e.b, e.a});
    auto first_of = [&](uint32_t a) {
        return std::lower_bound(level.begin(), level.end(), a,
                                [](const Edge& e, uint32_t v) { return e.a < v; });
    };
    while (!heap.empty()) {
        const HeapItem it = heap.top();
        heap.pop();
        if (!ch.candidate(it.a, it.b) || ch.head_of_tail[it.a] != it.head) continue;  // stale
        const uint32_t tail = ch.merge(it.a, it.b, w);
        // the merged chain's tail now belongs to a chain with a different head: re-key its
        // outgoing edges of this level
        for (auto e = first_of(tail); e != level.end() && e->a == tail; ++e)
            if (ch.candidate(e->a, e->b)) heap.push({ch.head_of_tail[e->a], e->b, e->a});
    }
}

}  // namespace

extern "C" int reseq_greedy_superstring(const uint8_t* concat, size_t n, const uint32_t* starts, size_t k,
                                        const reseq_overlaps* ov, uint32_t min_overlap,
                                        uint8_t* superstring, size_t* superstring_len, uint32_t* order,
                                        size_t* order_len) {
    if (!superstring_len || !order_len) return RESEQ_INVALID_ARGUMENT;
    *superstring_len = 0;
    *order_len = 0;
    if (k == 0) return RESEQ_OK;
    if (!concat || !starts || !ov || !ov->contained || !superstring || !order)
        return RESEQ_INVALID_ARGUMENT;
    if (min_overlap < 1) min_overlap = 1;
    // raw arrays from the C ABI: the fragment_set layout (sequence.hpp:60-62) and the ids of the
    // overlap list are checked before anything is indexed with them
    if (n < 2 || starts[0] != 0 || static_cast<uint64_t>(starts[k - 1]) + 2 > n) return RESEQ_INVALID_ARGUMENT;
    for (size_t i = 1; i < k; ++i)
        if (static_cast<uint64_t>(starts[i]) < static_cast<uint64_t>(starts[i - 1]) + 2 || starts[i] >= n)
            return RESEQ_INVALID_ARGUMENT;
    if (ov->count && (!ov->i || !ov->j || !ov->w)) return RESEQ_INVALID_ARGUMENT;
    for (uint64_t t = 0; t < ov->count; ++t)
        if (ov->i[t] >= k || ov->j[t] >= k) return RESEQ_INVALID_ARGUMENT;

    std::vector<uint32_t> lens(k);
    for (size_t i = 0; i < k; ++i)
        lens[i] = static_cast<uint32_t>((i + 1 < k ? starts[i + 1] : n) - 1 - starts[i]);
    const uint8_t* keep_out = ov->contained;
    size_t kept = 0;
    for (size_t i = 0; i < k; ++i) kept += keep_out[i] ? 0 : 1;
    if (kept == 0) return RESEQ_OK;

    // -- edges among kept fragments, bucketed by weight ------------------------------------
    uint32_t max_w = 0;
    for (uint64_t t = 0; t < ov->count; ++t) max_w = std::max(max_w, ov->w[t]);
    std::vector<uint64_t> level_size(static_cast<size_t>(max_w) + 2, 0);
    for (uint64_t t = 0; t < ov->count; ++t)
        if (!keep_out[ov->i[t]] && !keep_out[ov->j[t]] && ov->w[t] >= min_overlap) ++level_size[ov->w[t]];
    std::vector<std::vector<Edge>> levels(static_cast<size_t>(max_w) + 1);
    for (uint32_t w = 0; w <= max_w; ++w) levels[w].reserve(level_size[w]);
    for (uint64_t t = 0; t < ov->count; ++t)  // input is (i, j)-sorted, so every level is too
        if (!keep_out[ov->i[t]] && !keep_out[ov->j[t]] && ov->w[t] >= min_overlap)
            levels[ov->w[t]].push_back({ov->i[t], ov->j[t], ov->w[t]});

    Chains ch(k);
    for (uint32_t w = max_w; w >= min_overlap && w > 0; --w) {
        if (!levels[w].empty()) run_level(ch, levels[w], w);
        std::vector<Edge>().swap(levels[w]);
    }

    // -- sub-threshold overlaps among the surviving chains, exact --------------------------
    std::vector<uint32_t> heads;
    for (size_t i = 0; i < k; ++i)
        if (!keep_out[i] && ch.prev[i] == kNone) heads.push_back(static_cast<uint32_t>(i));
    if (heads.size() > 1 && min_overlap > 1) {
        std::vector<std::vector<Edge>> sub(min_overlap);
        for (uint32_t hx : heads) {
            const uint32_t a = ch.tail_of_head[hx];
            const uint8_t* fa = concat + starts[a];
            for (uint32_t b : heads) {
                if (b == hx) continue;
                const uint8_t* fb = concat + starts[b];
                const uint32_t lim = std::min({lens[a], lens[b], min_overlap - 1});
                uint32_t best = 0;
                for (uint32_t l = 1; l <= lim; ++l)
                    if (std::memcmp(fa + lens[a] - l, fb, l) == 0) best = l;
                if (best) sub[best].push_back({a, b, best});
            }
        }
        for (uint32_t w = min_overlap - 1; w >= 1; --w) {
            std::sort(sub[w].begin(), sub[w].end(), [](const Edge& x, const Edge& y) {
                return x.a != y.a ? x.a < y.a : x.b < y.b;
            });
            if (!sub[w].empty()) run_level(ch, sub[w], w);
        }
    }

    // -- zero-overlap tail: the smallest slot swallows the others in ascending slot order ----
    heads.clear();
    for (size_t i = 0; i < k; ++i)
        if (!keep_out[i] && ch.prev[i] == kNone) heads.push_back(static_cast<uint32_t>(i));
    for (size_t t = 1; t < heads.size(); ++t) ch.merge(ch.tail_of_head[heads[0]], heads[t], 0);

    // -- spell the chain out -------------------------------------------------------------------
    size_t len = 0, cnt = 0;
    for (uint32_t f = heads[0]; f != kNone; f = ch.next[f]) {
        const uint32_t skip = cnt ? ch.ov_next[ch.prev[f]] : 0;
        std::memcpy(superstring + len, concat + starts[f] + skip, lens[f] - skip);
        len += lens[f] - skip;
        order[cnt++] = f;
    }
    *superstring_len = len;
    *order_len = cnt;
    return RESEQ_OK;
}
