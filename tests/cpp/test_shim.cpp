// C++ drop-in test: the reference's own KATs (proj/tests/test_suffix_array.cpp:10-14,38-44;
// test_parallel.cpp:52-66,86-97,125-132,165-170; test_fragment_index.cpp:33-53,129-138;
// SPEC.md:300) through include/reseq_b200/reseq_cuda.hpp.  With -DRESEQ_B200_WITH_REFERENCE the
// device results are also compared with the reference's own functions on the same inputs.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "reseq_b200/reseq_cuda.hpp"

#ifdef RESEQ_B200_WITH_REFERENCE
#include "reseq/fragment_index.hpp"
#include "reseq/sequence.hpp"
#endif

using namespace reseq::cuda;
using u32v = std::vector<std::uint32_t>;

static int failures = 0;
#define REQUIRE(cond)                                                         \
    do {                                                                      \
        if (!(cond)) {                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
            ++failures;                                                       \
        }                                                                     \
    } while (0)
template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    device_executor dev(0);
    REQUIRE(build_parallel("banana", dev).sa == (u32v{5, 3, 1, 0, 4, 2}));
    REQUIRE(build_parallel("aaa", dev).sa == (u32v{2, 1, 0}));
    REQUIRE(build_parallel("", dev).sa.empty());
    REQUIRE(build_parallel(std::string("GA\0TT\0", 6), dev).sa == (u32v{2, 5, 1, 0, 4, 3}));
    {
        auto sp = build_parallel("mississippi", dev);
        for (std::uint32_t i = 0; i < sp.sa.size(); ++i) REQUIRE(sp.rank[sp.sa[i]] == i);
    }
    REQUIRE(exclusive_scan(u32v{3, 1, 7, 0}, dev) == (u32v{0, 3, 4, 11}));
    REQUIRE(exclusive_scan(u32v{}, dev).empty());
    REQUIRE(throws<scan_overflow_error>([&] { exclusive_scan(u32v{0xFFFFFFFFu, 1u}, dev); }));
    REQUIRE(exclusive_scan(u32v{0xFFFFFFFEu, 1u}, dev) == (u32v{0, 0xFFFFFFFEu}));
    REQUIRE(split_by_bit(key_array{{5, 2, 7, 4}, {}}, 0, dev).keys == (u32v{2, 4, 5, 7}));
    {
        auto s = split_by_bit(key_array{{1, 1, 0, 0}, {10, 11, 12, 13}}, 0, dev);
        REQUIRE(s.keys == (u32v{0, 0, 1, 1}));
        REQUIRE(s.payload == (u32v{12, 13, 10, 11}));
    }
    REQUIRE(radix_sort(key_array{{170, 45, 75, 90, 2, 24, 802, 66}, {}}, dev).keys ==
            (u32v{2, 24, 45, 66, 75, 90, 170, 802}));
    REQUIRE(radix_sort(key_array{}, dev).keys.empty());
    REQUIRE((radix_sort(key_array{{7}, {0}}, dev) == key_array{{7}, {0}}));
    REQUIRE(throws<std::invalid_argument>([&] { chunked_radix_sort(key_array{{1, 2}, {}}, dev, 0); }));
    REQUIRE(throws<std::invalid_argument>([&] { chunked_radix_sort(key_array{{1, 2}, {}}, dev, 9); }));
    {
        std::mt19937_64 rng(31);
        key_array a;
        for (int i = 0; i < 5000; ++i) {
            a.keys.push_back(static_cast<std::uint32_t>(rng()));
            a.payload.push_back(i);
        }
        REQUIRE(radix_sort(a, dev) == chunked_radix_sort(a, dev, 4));
        {   // split plan (radix_sort.hpp:35-52; test_parallel.cpp:109-123): tof counts the zero bits,
            // the destinations are a permutation and realise split_by_bit
            const auto plan = split_destinations(a.keys, 5, dev);
            std::uint32_t zeros = 0;
            for (auto k : a.keys) zeros += ((k >> 5) & 1u) ^ 1u;
            REQUIRE(plan.total_false == zeros);
            key_array moved{u32v(a.keys.size()), u32v(a.keys.size())};
            for (std::size_t i = 0; i < a.keys.size(); ++i) {
                moved.keys[plan.destinations[i]] = a.keys[i];
                moved.payload[plan.destinations[i]] = a.payload[i];
            }
            REQUIRE(moved == split_by_bit(a, 5, dev));
            REQUIRE(!phase_is_sorted(a.keys, dev));
            REQUIRE(phase_is_sorted(radix_sort(a, dev).keys, dev));
        }
#ifdef RESEQ_B200_WITH_REFERENCE
        {
            const auto plan = split_destinations(a.keys, 5, dev);
            const auto ref_plan = reseq::detail::split_destinations(a.keys, 5, reseq::executor{});
            REQUIRE(plan.destinations == ref_plan.destinations && plan.total_false == ref_plan.total_false);
        }
        REQUIRE(radix_sort(a, dev) == reseq::radix_sort(a));
        REQUIRE(split_by_bit(a, 7, dev) == reseq::split_by_bit(a, 7));
        REQUIRE(exclusive_scan(std::span<const std::uint32_t>(a.payload), dev) == reseq::exclusive_scan(a.payload));
#endif
    }
    {
        // the worked instance of test_fragment_index.cpp:33-45
        const std::string concat("GATT\0ACA\0GGT\0GA\0TTAC\0AGGT\0", 26);
        const u32v starts{0, 5, 9, 13, 16, 21};
        fragment_index ix(concat, starts, dev);
        auto [lo, hi] = ix.locate_prefix_range("GA");
        REQUIRE(hi - lo == 2);
        auto sa = ix.sa();
        u32v pos{sa.sa[lo], sa.sa[lo + 1]};
        REQUIRE((pos == u32v{0, 13} || pos == u32v{13, 0}));
        auto [l2, h2] = ix.locate_prefix_range("QQ");
        REQUIRE(l2 == h2);
        // prefix_related, test_fragment_index.cpp:82-94
        auto rel = ix.prefix_related(residual{0, 2});   // "TT"
        REQUIRE(rel.prefixes_of.empty() && rel.exact_matches.empty());
        REQUIRE(rel.extensions_of == (u32v{4}));
        REQUIRE(ix.prefix_related(std::string_view("GGT")).exact_matches == (u32v{2}));
        REQUIRE(ix.prefix_related(std::string_view("GATTA")).prefixes_of == (u32v{0, 3}));   // GA and GATT
        REQUIRE(throws<offset_out_of_range_error>([&] { ix.prefix_related(residual{0, 4}); }));   // sequence.hpp:128-129
        REQUIRE(throws<offset_out_of_range_error>([&] { ix.prefix_related(residual{6, 0}); }));
    }
    {
        // test_fragment_index.cpp:96-104
        const std::string concat("ab\0cd\0efgh\0abcdef\0gh\0", 21);
        const u32v starts{0, 3, 6, 11, 18};
        fragment_index ix(concat, starts, dev);
        auto rel = ix.prefix_related(std::string_view("cdef"));
        REQUIRE(rel.prefixes_of == (u32v{1}) && rel.extensions_of.empty() && rel.exact_matches.empty());
        // the early return of fragment_index.hpp:91: the interval empties at length 2 ("zz" is absent)
        auto none = ix.prefix_related(std::string_view("zzzzzzz"));
        REQUIRE(none.prefixes_of.empty() && none.extensions_of.empty() && none.exact_matches.empty());
    }
#ifdef RESEQ_B200_WITH_REFERENCE
    {
        // the reference's constructor shape (fragment_index.hpp:34) and 600 random queries against the
        // reference's own prefix_related, residual and string_view forms (test_fragment_index.cpp:106-127)
        std::mt19937_64 rng(53);
        for (int it = 0; it < 60; ++it) {
            std::vector<std::string> frags;
            const int k = 2 + rng() % 12;
            for (int f = 0; f < k; ++f) {
                std::string s;
                const int len = 1 + rng() % 9;
                for (int i = 0; i < len; ++i) s.push_back("AC"[rng() % 2]);
                frags.push_back(s);
            }
            auto set = reseq::make_fragment_set(frags, reseq::alphabet::dna);
            fragment_index ix(set, dev);
            reseq::fragment_index ref_ix(set);
            for (int q = 0; q < 10; ++q) {
                const std::uint32_t id = rng() % set.size(), off = rng() % set.length(id);
                const auto a = ix.prefix_related(residual{id, off});
                const auto b = ref_ix.prefix_related(reseq::residual{id, off});
                REQUIRE(a.prefixes_of == b.prefixes_of && a.extensions_of == b.extensions_of && a.exact_matches == b.exact_matches);
                std::string pat;
                const int plen = 1 + rng() % 11;
                for (int i = 0; i < plen; ++i) pat.push_back("ACG"[rng() % 3]);
                const auto c = ix.prefix_related(std::string_view(pat));
                const auto d = ref_ix.prefix_related(std::string_view(pat));
                REQUIRE(c.prefixes_of == d.prefixes_of && c.extensions_of == d.extensions_of && c.exact_matches == d.exact_matches);
            }
        }
    }
#endif
    {
        // the paper's five fragments: SPEC.md:300
        const std::string concat("abthatb\0hatbpaab\0tbabhhatbpaa\0paabtabh\0bhaabtpb\0", 48);
        const u32v starts{0, 8, 17, 30, 39};
        fragment_index ix(concat, starts, dev);
        auto g = ix.greedy_superstring_with_order(1);
        REQUIRE(g.superstring == "abthatbabhhatbpaabtabhaabtpb");
        REQUIRE(g.order == (u32v{0, 2, 1, 3, 4}));
#ifdef RESEQ_B200_WITH_REFERENCE
        auto set = reseq::make_fragment_set({"abthatb", "hatbpaab", "tbabhhatbpaa", "paabtabh", "bhaabtpb"},
                                            reseq::alphabet::generic_byte);
        reseq::fragment_index ref_ix(set, reseq::fragment_index::builder::scan_radix);
        REQUIRE(ix.sa().sa == ref_ix.sa().sa);
        REQUIRE(ix.start_rank_list() == ref_ix.start_rank_list());
        auto rg = reseq::greedy_superstring_with_order(set);
        REQUIRE(g.superstring == rg.superstring && g.order == rg.order);
#endif
    }
    std::printf(failures ? "%d FAILED\n" : "shim ok\n", failures);
    return failures ? 1 : 0;
}
