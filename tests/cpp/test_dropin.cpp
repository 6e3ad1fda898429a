// The drop-in proven on the reference's own classes: compiled by oracle/make_dropin.py
// against a PATCHED scratch copy of the reference headers (builder::cuda in fragment_index.hpp:32-38,
// executor_config::device + one forwarding line per operator; INTEGRATION.md sections 2-3) and against
// libreseq_cuda.so.  Every check below runs the REFERENCE'S code -- fragment_index::narrow / prefix_related,
// find_fir_pairs, reconstruct, bench generators -- on top of a suffix array / operator result that came
// from the device, next to the same thing on the reference's host path.
//
//   proj/tests/test_fragment_index.cpp:33-53    locate_prefix_range KATs
//   proj/tests/test_fragment_index.cpp:82-104   prefix_related KATs
//   proj/tests/test_fragment_index.cpp:106-127  3000 random prefix_related queries vs the pairwise scan
//   proj/tests/test_fragment_index.cpp:129-138  builders produce the same structure
//   proj/tests/test_assembler.cpp:241-269       naive == indexed reconstruct on double_cut instances
//   proj/tests/test_parallel.cpp (KAT shapes)   the operators through executor_config{.device = 0}
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "reseq/assembler.hpp"
#include "reseq/bench.hpp"
#include "reseq/fragment_index.hpp"
#include "reseq/shotgun.hpp"

using namespace reseq;

static int failures = 0;
#define REQUIRE(cond)                                                        \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

static prefix_relation brute_relation(const fragment_set& s, std::string_view r) {   // test_fragment_index.cpp:12-24
    prefix_relation rel;
    for (std::uint32_t id = 0; id < s.size(); ++id) {
        auto f = s.bytes(id);
        if (f.size() < r.size() && r.substr(0, f.size()) == f) rel.prefixes_of.push_back(id);
        else if (f.size() > r.size() && f.substr(0, r.size()) == r) rel.extensions_of.push_back(id);
        else if (f == r) rel.exact_matches.push_back(id);
    }
    return rel;
}
static bool same(const prefix_relation& a, const prefix_relation& b) {
    return a.prefixes_of == b.prefixes_of && a.extensions_of == b.extensions_of && a.exact_matches == b.exact_matches;
}

int main() {
    const auto CUDA = fragment_index::builder::cuda;
    {   // test_fragment_index.cpp:33-45
        auto set = make_fragment_set({"GATT", "ACA", "GGT", "GA", "TTAC", "AGGT"}, alphabet::dna);
        fragment_index ix(set, CUDA);
        auto [lo, hi] = ix.locate_prefix_range("GA");
        REQUIRE(hi - lo == 2);
        std::vector<std::uint32_t> pos{ix.sa().sa[lo], ix.sa().sa[lo + 1]};
        std::sort(pos.begin(), pos.end());
        REQUIRE((pos == std::vector<std::uint32_t>{0, 13}));
        auto [l2, h2] = ix.locate_prefix_range("QQ");
        REQUIRE(l2 == h2);
        // :82-94
        auto rel = ix.prefix_related(residual{0, 2});  // "TT"
        REQUIRE(rel.prefixes_of.empty());
        REQUIRE((rel.extensions_of == std::vector<std::uint32_t>{4}));
        REQUIRE(rel.exact_matches.empty());
        REQUIRE((ix.prefix_related(std::string_view("GGT")).exact_matches == std::vector<std::uint32_t>{2}));
    }
    {   // :47-53
        auto set = make_fragment_set({"GATT"}, alphabet::dna);
        fragment_index ix(set, CUDA);
        auto [lo, hi] = ix.locate_prefix_range("GATT");
        REQUIRE(hi - lo == 1);
        REQUIRE(ix.sa().sa[lo] == 0);
    }
    {   // :96-104
        auto set = make_fragment_set({"ab", "cd", "efgh", "abcdef", "gh"}, alphabet::generic_byte);
        fragment_index ix(set, CUDA);
        auto rel = ix.prefix_related(std::string_view("cdef"));
        REQUIRE((rel.prefixes_of == std::vector<std::uint32_t>{1}));
        REQUIRE(rel.extensions_of.empty());
        REQUIRE(rel.exact_matches.empty());
    }
    {   // :129-138, with the device builder as the third
        auto set = make_fragment_set({"abthatb", "hatbpaab", "tbabhhatbpaa", "paabtabh", "bhaabtpb"}, alphabet::generic_byte);
        fragment_index direct(set, fragment_index::builder::direct);
        executor ex(executor_config{2, 64});
        fragment_index parallel(set, fragment_index::builder::scan_radix, ex);
        fragment_index device(set, CUDA);
        REQUIRE(direct.sa().sa == device.sa().sa);
        REQUIRE(direct.sa().rank == device.sa().rank);
        REQUIRE(parallel.sa().sa == device.sa().sa);
        REQUIRE(direct.start_rank_list() == device.start_rank_list());
    }
    {   // :106-127 -- 3000 random residual queries through the reference's narrow() over the device SA
        std::mt19937_64 rng(53);
        int queries = 0;
        while (queries < 3000) {
            const std::size_t L = 10 + rng() % 80;
            std::string s;
            for (std::size_t i = 0; i < L; ++i) s.push_back("ACGT"[rng() % 4]);
            sequence seq(s, alphabet::dna);
            const std::size_t cap = std::max<std::size_t>(1, L / 8);
            auto [ca, cb] = random_cut_pair(L, rng() % cap, 1 + rng() % cap, rng());
            auto inst = double_cut(seq, ca, cb, rng());
            const auto& set = inst.fragments;
            fragment_index ix(set, CUDA);
            fragment_index host(set, fragment_index::builder::direct);
            REQUIRE(ix.sa().sa == host.sa().sa);
            for (int q = 0; q < 10; ++q, ++queries) {
                const std::uint32_t id = rng() % set.size();
                const std::uint32_t off = rng() % set.length(id);
                auto rb = residual_view(set, {id, off});
                REQUIRE(same(ix.prefix_related(rb), brute_relation(set, rb)));
            }
        }
    }
    {   // test_assembler.cpp:241-269 -- naive == indexed reconstruct, the index built on the device
        std::mt19937_64 rng(61);
        for (int it = 0; it < 120; ++it) {
            const std::size_t L = 6 + rng() % 80;
            std::string s;
            for (std::size_t i = 0; i < L; ++i) s.push_back("ACGT"[rng() % 4]);
            sequence seq(s, alphabet::dna);
            const std::size_t cap = std::max<std::size_t>(1, L / 10);
            std::size_t m = rng() % (cap + 1), n = rng() % (cap + 1);
            if (m + n == 0) m = 1;
            auto [ca, cb] = random_cut_pair(L, m, n, rng());
            auto inst = double_cut(seq, ca, cb, rng());
            auto naive = reconstruct(inst.fragments);
            fragment_index ix(inst.fragments, CUDA);
            auto indexed = reconstruct(inst.fragments, {}, &ix);
            REQUIRE(naive.status == solve_status::solved);
            REQUIRE(naive.seq.size() == L);
            REQUIRE(verify_tiling(naive.seq.bytes(), inst.fragments));
            REQUIRE(indexed.status == solve_status::solved);
            REQUIRE(indexed.seq.bytes() == naive.seq.bytes());
            REQUIRE(indexed.trace == naive.trace);
            std::vector<std::uint32_t> all(inst.fragments.size());
            for (std::uint32_t i = 0; i < all.size(); ++i) all[i] = i;
            REQUIRE(find_fir_pairs(inst.fragments, all, &ix) == find_fir_pairs(inst.fragments, all));   // assembler.hpp:74-78
        }
    }
    {   // the executor plug point: the reference's own operators with executor_config{.device = 0}
        executor_config cfg;
        cfg.device = 0;
        executor dev(cfg);
        executor host(executor_config{3, 257});
        REQUIRE((build_parallel("banana", dev).sa == std::vector<std::uint32_t>{5, 3, 1, 0, 4, 2}));          // test_suffix_array.cpp:10-14
        REQUIRE((build_parallel(std::string_view("GA\0TT\0", 6), dev).sa == std::vector<std::uint32_t>{2, 5, 1, 0, 4, 3}));   // :38-44
        const std::string dna = bench::make_random_dna(1 << 16, 1);
        const auto a = build_parallel(dna, dev), b = build_parallel(dna, host);
        REQUIRE(a.sa == b.sa);
        REQUIRE(a.rank == b.rank);
        REQUIRE(bench::checksum_u32(build_parallel(bench::make_random_dna(1 << 20, 1), dev).sa) == 7546189330682201289ull);
        const key_array keys = bench::make_random_keys(100000, 7);
        REQUIRE(radix_sort(keys, dev) == radix_sort(keys, host));
        REQUIRE(chunked_radix_sort(keys, dev, 4) == radix_sort(keys, host));
        REQUIRE(split_by_bit(keys, 5, dev) == split_by_bit(keys, 5, host));
        std::vector<std::uint32_t> v(keys.keys.size());
        for (std::size_t i = 0; i < v.size(); ++i) v[i] = keys.keys[i] % 5000;
        REQUIRE(exclusive_scan(std::span<const std::uint32_t>(v), dev) == exclusive_scan(std::span<const std::uint32_t>(v), host));
        bool threw = false;
        try { chunked_radix_sort(keys, dev, 9); } catch (const std::invalid_argument&) { threw = true; }   // radix_sort.hpp:171-172
        REQUIRE(threw);
        threw = false;
        const std::vector<std::uint32_t> big{0xFFFFFFFFu, 1u};
        try { exclusive_scan(std::span<const std::uint32_t>(big), dev); } catch (const scan_overflow_error&) { threw = true; }   // scan.hpp:38
        REQUIRE(threw);
    }
    if (failures) {
        std::fprintf(stderr, "%d check(s) failed\n", failures);
        return 1;
    }
    std::puts("drop-in ok: reference fragment_index / assembler / operators over libreseq_cuda.so");
    return 0;
}
