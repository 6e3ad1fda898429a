// TEST INFRASTRUCTURE -- NOT PRODUCT CODE.
//
// C-ABI shim over the UNMODIFIED reference headers, compiled where they lie
// (-I/root/reference/proj/include) into oracle/_ref/libreseq_ref.so by
// oracle/Makefile.  Nothing from the reference is copied into this repo; this
// file only calls the reference's public functions so that tests (and the
// cpu_baseline / --impl reference legs of bench.py) can run the real thing.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load the resulting library.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <random>
#include <string>
#include <string_view>
#include <vector>

#include "reseq/bench.hpp"
#include "reseq/errors.hpp"
#include "reseq/executor.hpp"
#include "reseq/fragment_index.hpp"
#include "reseq/overlap.hpp"
#include "reseq/radix_sort.hpp"
#include "reseq/scan.hpp"
#include "reseq/sequence.hpp"
#include "reseq/shotgun.hpp"
#include "reseq/suffix_array.hpp"

namespace {

// Error codes mirror include/reseq_cuda.h so tests can compare behaviour.
enum : int {
    kOk = 0,
    kInvalidArgument = 1,
    kTextTooLarge = 2,
    kScanOverflow = 3,
    kOther = 9,
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const reseq::text_too_large_error&) {
        return kTextTooLarge;
    } catch (const reseq::scan_overflow_error&) {
        return kScanOverflow;
    } catch (const std::invalid_argument&) {
        return kInvalidArgument;
    } catch (...) {
        return kOther;
    }
}

reseq::key_array make_arr(const uint32_t* k, const uint32_t* p, size_t n) {
    reseq::key_array a;
    a.keys.assign(k, k + n);
    if (p) a.payload.assign(p, p + n);
    return a;
}

void put_arr(const reseq::key_array& a, uint32_t* ko, uint32_t* po) {
    if (!a.keys.empty()) std::memcpy(ko, a.keys.data(), a.keys.size() * 4);
    if (po && !a.payload.empty()) std::memcpy(po, a.payload.data(), a.payload.size() * 4);
}

struct ref_index {
    reseq::fragment_set set;
    std::unique_ptr<reseq::fragment_index> ix;
};

std::vector<std::string> split_fragments(const uint8_t* bytes, const uint64_t* off, size_t k) {
    std::vector<std::string> frags(k);
    for (size_t i = 0; i < k; ++i)
        frags[i].assign(reinterpret_cast<const char*>(bytes) + off[i], off[i + 1] - off[i]);
    return frags;
}

}  // namespace

extern "C" {

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// ---- suffix_array.hpp ----------------------------------------------------
int ref_build_naive(const uint8_t* text, size_t n, uint32_t* sa, uint32_t* rank) {
    return guarded([&] {
        auto r = reseq::build_naive(std::string_view(reinterpret_cast<const char*>(text), n));
        if (n) {
            std::memcpy(sa, r.sa.data(), n * 4);
            if (rank) std::memcpy(rank, r.rank.data(), n * 4);
        }
    });
}

int ref_build_parallel(const uint8_t* text, size_t n, unsigned workers, size_t chunk,
                       uint32_t* sa, uint32_t* rank) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        auto r = reseq::build_parallel(
            std::string_view(reinterpret_cast<const char*>(text), n), ex);
        if (n) {
            std::memcpy(sa, r.sa.data(), n * 4);
            if (rank) std::memcpy(rank, r.rank.data(), n * 4);
        }
    });
}

int ref_suffix_less(const uint8_t* text, size_t n, uint32_t i, uint32_t j) {
    return reseq::suffix_less(std::string_view(reinterpret_cast<const char*>(text), n), i, j);
}

// ---- scan.hpp / radix_sort.hpp -------------------------------------------
int ref_exclusive_scan(const uint32_t* v, size_t n, unsigned workers, size_t chunk,
                       uint32_t* out) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        auto r = reseq::exclusive_scan(std::span<const uint32_t>(v, n), ex);
        if (n) std::memcpy(out, r.data(), n * 4);
    });
}

int ref_split_by_bit(const uint32_t* k, const uint32_t* p, size_t n, unsigned bit,
                     unsigned workers, size_t chunk, uint32_t* ko, uint32_t* po) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        put_arr(reseq::split_by_bit(make_arr(k, p, n), bit, ex), ko, po);
    });
}

int ref_split_destinations(const uint32_t* k, size_t n, unsigned bit, unsigned workers, size_t chunk,
                           uint32_t* d, uint32_t* total_false) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        auto plan = reseq::detail::split_destinations(std::span<const uint32_t>(k, n), bit, ex);
        if (n) std::memcpy(d, plan.destinations.data(), n * 4);
        *total_false = plan.total_false;
    });
}

int ref_is_sorted(const uint32_t* k, size_t n, unsigned workers, size_t chunk, int* sorted) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        *sorted = reseq::detail::phase_is_sorted(std::span<const uint32_t>(k, n), ex) ? 1 : 0;
    });
}

int ref_radix_sort(const uint32_t* k, const uint32_t* p, size_t n, unsigned workers,
                   size_t chunk, uint32_t* ko, uint32_t* po) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        put_arr(reseq::radix_sort(make_arr(k, p, n), ex), ko, po);
    });
}

int ref_chunked_radix_sort(const uint32_t* k, const uint32_t* p, size_t n, unsigned workers,
                           size_t chunk, unsigned digit_bits, uint32_t* ko, uint32_t* po) {
    return guarded([&] {
        reseq::executor ex(reseq::executor_config{workers, chunk});
        put_arr(reseq::chunked_radix_sort(make_arr(k, p, n), ex, digit_bits), ko, po);
    });
}

// ---- bench.hpp -------------------------------------------------------------
uint64_t ref_fnv1a64(const uint8_t* b, size_t n) {
    return reseq::bench::fnv1a64(std::string_view(reinterpret_cast<const char*>(b), n));
}

uint64_t ref_checksum_u32(const uint32_t* v, size_t n) {
    return reseq::bench::checksum_u32(std::vector<uint32_t>(v, v + n));
}

void ref_make_random_dna(size_t n, uint64_t seed, uint8_t* out) {
    auto s = reseq::bench::make_random_dna(n, seed);
    std::memcpy(out, s.data(), n);
}

void ref_make_random_keys(size_t n, uint64_t seed, uint32_t* keys, uint32_t* payload) {
    auto a = reseq::bench::make_random_keys(n, seed);
    put_arr(a, keys, payload);
}

// Synthetic shotgun read text per SURVEY.md section 8(d): genome =
// make_random_dna(G, genome_seed); mt19937_64 rng(read_seed); start_i =
// detail::bounded_u64(rng, G-L+1); text = make_fragment_set(reads).concat().
// `out` must hold k*(L+1) bytes.
int ref_make_read_text(size_t G, size_t L, size_t k, uint64_t genome_seed, uint64_t read_seed,
                       uint8_t* out) {
    return guarded([&] {
        const std::string genome = reseq::bench::make_random_dna(G, genome_seed);
        std::mt19937_64 rng(read_seed);
        std::vector<std::string> reads;
        reads.reserve(k);
        for (size_t i = 0; i < k; ++i) {
            const uint64_t s = reseq::detail::bounded_u64(rng, G - L + 1);
            reads.push_back(genome.substr(s, L));
        }
        auto set = reseq::make_fragment_set(reads, reseq::alphabet::dna);
        std::memcpy(out, set.concat().data(), set.concat().size());
    });
}

// ---- sequence.hpp / fragment_index.hpp -----------------------------------
// Fragments arrive as one byte blob + k+1 offsets. alphabet: 0 = dna, 1 = generic_byte.
// builder: 0 = direct (build_naive), 1 = scan_radix (build_parallel).
void* ref_index_create(const uint8_t* bytes, const uint64_t* off, size_t k, int alphabet,
                       int builder, unsigned workers, size_t chunk) {
    try {
        auto h = std::make_unique<ref_index>();
        h->set = reseq::make_fragment_set(
            split_fragments(bytes, off, k),
            alphabet == 0 ? reseq::alphabet::dna : reseq::alphabet::generic_byte);
        reseq::executor ex(reseq::executor_config{workers, chunk});
        h->ix = std::make_unique<reseq::fragment_index>(
            h->set,
            builder ? reseq::fragment_index::builder::scan_radix
                    : reseq::fragment_index::builder::direct,
            ex);
        return h.release();
    } catch (...) {
        return nullptr;
    }
}

void ref_index_destroy(void* h) { delete static_cast<ref_index*>(h); }

size_t ref_index_text_len(void* h) { return static_cast<ref_index*>(h)->set.concat().size(); }

void ref_index_get(void* hv, uint8_t* concat, uint32_t* starts, uint32_t* sa, uint32_t* rank,
                   uint32_t* start_rank_list) {
    auto* h = static_cast<ref_index*>(hv);
    const auto& c = h->set.concat();
    if (concat) std::memcpy(concat, c.data(), c.size());
    if (starts) std::memcpy(starts, h->set.starts().data(), h->set.size() * 4);
    if (sa) std::memcpy(sa, h->ix->sa().sa.data(), c.size() * 4);
    if (rank) std::memcpy(rank, h->ix->sa().rank.data(), c.size() * 4);
    if (start_rank_list)
        std::memcpy(start_rank_list, h->ix->start_rank_list().data(), h->set.size() * 4);
}

void ref_index_locate(void* hv, const uint8_t* pat, size_t m, uint32_t* lo, uint32_t* hi) {
    auto* h = static_cast<ref_index*>(hv);
    auto r = h->ix->locate_prefix_range(
        std::string_view(reinterpret_cast<const char*>(pat), m));
    *lo = r.first;
    *hi = r.second;
}

// Writes the three id lists into caller buffers (each sized k) and their counts.
void ref_index_prefix_related(void* hv, const uint8_t* pat, size_t m, uint32_t* prefixes,
                              uint32_t* n_prefixes, uint32_t* extensions, uint32_t* n_ext,
                              uint32_t* exact, uint32_t* n_exact) {
    auto* h = static_cast<ref_index*>(hv);
    auto rel = h->ix->prefix_related(std::string_view(reinterpret_cast<const char*>(pat), m));
    *n_prefixes = rel.prefixes_of.size();
    *n_ext = rel.extensions_of.size();
    *n_exact = rel.exact_matches.size();
    std::memcpy(prefixes, rel.prefixes_of.data(), rel.prefixes_of.size() * 4);
    std::memcpy(extensions, rel.extensions_of.data(), rel.extensions_of.size() * 4);
    std::memcpy(exact, rel.exact_matches.data(), rel.exact_matches.size() * 4);
}

// CPU query baseline: the overlap job's query stream -- for every fragment i and every
// offset o in [0, |f_i| - min_overlap], the pattern f_i[o..] -- through the reference's own
// locate_prefix_range (fragment_index.hpp:65-70; mode 0) or prefix_related (:72-109; mode 1), over a
// shared immutable index from `threads` host threads (fragments dealt in blocks of 64).
// Stops taking new blocks once `max_queries` have been issued.  Returns seconds; *done = queries run;
// *acc = sum of interval widths / relation counts (keeps the calls observable).
double ref_index_query_bench(void* hv, uint32_t min_overlap, unsigned threads, uint64_t max_queries, int mode,
                             uint64_t* done, uint64_t* acc) {
    auto* h = static_cast<ref_index*>(hv);
    const uint32_t k = h->set.size();
    std::atomic<uint32_t> next{0};
    std::atomic<uint64_t> issued{0}, total{0};
    if (threads == 0) threads = 1;
    auto work = [&] {
        uint64_t local = 0, mine = 0;
        for (;;) {
            if (issued.load(std::memory_order_relaxed) >= max_queries) break;
            const uint32_t b = next.fetch_add(64);
            if (b >= k) break;
            uint64_t q = 0;
            for (uint32_t i = b; i < k && i < b + 64; ++i) {
                const std::string_view f = h->set.bytes(i);
                if (f.size() < min_overlap) continue;
                for (size_t o = 0; o + min_overlap <= f.size(); ++o) {
                    const std::string_view pat = f.substr(o);
                    if (mode == 0) {
                        const auto r = h->ix->locate_prefix_range(pat);
                        local += r.second - r.first;
                    } else {
                        const auto rel = h->ix->prefix_related(pat);
                        local += rel.prefixes_of.size() + rel.extensions_of.size() + rel.exact_matches.size();
                    }
                    ++q;
                }
            }
            mine += q;
            issued.fetch_add(q, std::memory_order_relaxed);
        }
        total.fetch_add(local);
        (void)mine;
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    if (done) *done = issued.load();
    if (acc) *acc = total.load();
    return std::chrono::duration<double>(t1 - t0).count();
}

// The same index over an already concatenated fragment text (concat = f0 \0 f1 \0 ...; `starts` as in
// fragment_set): saves the caller the blob/offset detour for large read sets.
void* ref_index_create_from_text(const uint8_t* concat, size_t n, const uint32_t* starts, size_t k, int alphabet,
                                 int builder, unsigned workers, size_t chunk) {
    try {
        std::vector<std::string> frags(k);
        for (size_t i = 0; i < k; ++i) {
            const size_t b = starts[i], e = (i + 1 < k ? starts[i + 1] : n) - 1;
            frags[i].assign(reinterpret_cast<const char*>(concat) + b, e - b);
        }
        auto h = std::make_unique<ref_index>();
        h->set = reseq::make_fragment_set(frags, alphabet == 0 ? reseq::alphabet::dna : reseq::alphabet::generic_byte);
        reseq::executor ex(reseq::executor_config{workers, chunk});
        h->ix = std::make_unique<reseq::fragment_index>(
            h->set, builder ? reseq::fragment_index::builder::scan_radix : reseq::fragment_index::builder::direct, ex);
        return h.release();
    } catch (...) {
        return nullptr;
    }
}

// ---- overlap.hpp -----------------------------------------------------------
uint32_t ref_overlap_weight(const uint8_t* a, size_t na, const uint8_t* b, size_t nb) {
    return reseq::overlap_weight(std::string_view(reinterpret_cast<const char*>(a), na),
                                 std::string_view(reinterpret_cast<const char*>(b), nb));
}

// weight: k*k row-major.
int ref_overlap_graph(const uint8_t* bytes, const uint64_t* off, size_t k, int alphabet,
                      uint32_t* weight) {
    return guarded([&] {
        auto set = reseq::make_fragment_set(
            split_fragments(bytes, off, k),
            alphabet == 0 ? reseq::alphabet::dna : reseq::alphabet::generic_byte);
        auto g = reseq::build_overlap_graph(set);
        std::memcpy(weight, g.weight.data(), g.weight.size() * 4);
    });
}

// superstring buffer must hold the sum of fragment lengths; order buffer k entries.
int ref_greedy(const uint8_t* bytes, const uint64_t* off, size_t k, int alphabet,
               uint8_t* superstring, size_t* superstring_len, uint32_t* order,
               size_t* order_len) {
    return guarded([&] {
        auto set = reseq::make_fragment_set(
            split_fragments(bytes, off, k),
            alphabet == 0 ? reseq::alphabet::dna : reseq::alphabet::generic_byte);
        auto r = reseq::greedy_superstring_with_order(set);
        *superstring_len = r.superstring.size();
        std::memcpy(superstring, r.superstring.data(), r.superstring.size());
        *order_len = r.order.size();
        std::memcpy(order, r.order.data(), r.order.size() * 4);
    });
}

int ref_absorb_contained(const uint8_t* bytes, const uint64_t* off, size_t k, int alphabet,
                         uint32_t* keep, size_t* n_keep) {
    return guarded([&] {
        auto set = reseq::make_fragment_set(
            split_fragments(bytes, off, k),
            alphabet == 0 ? reseq::alphabet::dna : reseq::alphabet::generic_byte);
        auto ids = reseq::detail::absorb_contained(set);
        *n_keep = ids.size();
        std::memcpy(keep, ids.data(), ids.size() * 4);
    });
}

// double_cut instance generator used by test_fragment_index.cpp:106-127; returns fragments
// blob + offsets via callback-free two-call protocol: first call with null outputs to size.
int ref_double_cut(const uint8_t* seq, size_t L, size_t m, size_t n, uint64_t cut_seed,
                   uint64_t shuffle_seed, uint8_t* bytes_out, uint64_t* off_out, size_t* k_out) {
    return guarded([&] {
        reseq::sequence s(std::string(reinterpret_cast<const char*>(seq), L),
                          reseq::alphabet::dna);
        auto [ca, cb] = reseq::random_cut_pair(L, m, n, cut_seed);
        auto inst = reseq::double_cut(s, ca, cb, shuffle_seed);
        const auto& set = inst.fragments;
        *k_out = set.size();
        if (bytes_out && off_out) {
            uint64_t o = 0;
            for (uint32_t i = 0; i < set.size(); ++i) {
                off_out[i] = o;
                auto b = set.bytes(i);
                std::memcpy(bytes_out + o, b.data(), b.size());
                o += b.size();
            }
            off_out[set.size()] = o;
        }
    });
}

}  // extern "C"
