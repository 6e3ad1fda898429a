// reseq_cuda.hpp -- C++ shim over the C ABI (reseq_cuda.h) that restores the reference's
// value-semantics signatures for the hot path:
//
//   reference (proj/include/reseq)                         this shim (namespace reseq::cuda)
//   ------------------------------------------------       -----------------------------------------
//   executor(executor_config)        executor.hpp:28       device_executor(int device = 0)
//   exclusive_scan(values, exec)     scan.hpp:32           exclusive_scan(values, dev)
//   split_by_bit(arr, bit, exec)     radix_sort.hpp:126    split_by_bit(arr, bit, dev)
//   radix_sort(arr, exec)            radix_sort.hpp:143    radix_sort(arr, dev)
//   chunked_radix_sort(arr, exec, b) radix_sort.hpp:169    chunked_radix_sort(arr, dev, b)
//   build_parallel(text, exec)       suffix_array.hpp:61   build_parallel(text, dev)
//   fragment_index(set, builder, ex) fragment_index.hpp:34 fragment_index(concat, starts, dev) / (set, dev)
//     .locate_prefix_range(p)        :65                     .locate_prefix_range(p)
//     .prefix_related(residual)      :72                     .prefix_related(residual)
//     .prefix_related(string_view)   :82                     .prefix_related(string_view)
//     .start_rank_list()             :61                     .start_rank_list()
//   greedy_superstring_with_order    overlap.hpp:80        greedy_superstring_with_order(ix, tau)
//
// Compiled WITH the reference on the include path (-DRESEQ_B200_WITH_REFERENCE), the shim uses
// the reference's own types (reseq::key_array, reseq::suffix_array, reseq::greedy_result) and
// throws the reference's own exception types, so call sites only change the executor argument.
// Compiled standalone it defines layout-identical types in namespace reseq::cuda.
//
// No exception crosses the C boundary: status codes are mapped back here (errors.hpp:9-61,
// radix_sort.hpp:171-172).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "reseq_cuda.h"

#include <algorithm>

#ifdef RESEQ_B200_WITH_REFERENCE
#include "reseq/errors.hpp"
#include "reseq/fragment_index.hpp"
#include "reseq/overlap.hpp"
#include "reseq/radix_sort.hpp"
#include "reseq/sequence.hpp"
#include "reseq/suffix_array.hpp"
#endif

namespace reseq::cuda {

#ifdef RESEQ_B200_WITH_REFERENCE
using ::reseq::error;
using ::reseq::fragment_set;
using ::reseq::greedy_result;
using ::reseq::key_array;
using ::reseq::offset_out_of_range_error;
using ::reseq::prefix_relation;
using ::reseq::residual;
using ::reseq::scan_overflow_error;
using ::reseq::suffix_array;
using ::reseq::text_too_large_error;
#else
struct error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct scan_overflow_error : error {
    scan_overflow_error() : error("prefix sum exceeds 32-bit range") {}
};
struct text_too_large_error : error {
    explicit text_too_large_error(std::uint64_t n)
        : error("text of length " + std::to_string(n) + " exceeds 2^32-2") {}
};
struct key_array {
    std::vector<std::uint32_t> keys;
    std::vector<std::uint32_t> payload;
    bool has_payload() const { return !payload.empty(); }
    friend bool operator==(const key_array&, const key_array&) = default;
};
struct suffix_array {
    std::vector<std::uint32_t> sa;
    std::vector<std::uint32_t> rank;
    std::size_t text_len() const { return sa.size(); }
};
struct greedy_result {
    std::string superstring;
    std::vector<std::uint32_t> order;
};
struct residual {   // sequence.hpp:96-101
    std::uint32_t frag = 0;
    std::uint32_t offset = 0;
};
struct prefix_relation {   // fragment_index.hpp:21-25
    std::vector<std::uint32_t> prefixes_of;
    std::vector<std::uint32_t> extensions_of;
    std::vector<std::uint32_t> exact_matches;
};
struct offset_out_of_range_error : error {   // errors.hpp:30-34
    offset_out_of_range_error(std::uint32_t frag, std::uint32_t offset)
        : error("offset " + std::to_string(offset) + " out of range for fragment " + std::to_string(frag)) {}
};
#endif

namespace detail {
inline void check(int status, std::uint64_t n = 0) {
    switch (status) {
        case RESEQ_OK: return;
        case RESEQ_INVALID_ARGUMENT: throw std::invalid_argument(reseq_cuda_last_error());
        case RESEQ_TEXT_TOO_LARGE: throw text_too_large_error(n);
        case RESEQ_SCAN_OVERFLOW: throw scan_overflow_error();
        default: throw error(reseq_cuda_last_error());
    }
}
}  // namespace detail

/// Stands where the reference passes `const executor&`: one device, one stream, one
/// workspace arena.  Non-copyable like executor (executor.hpp:39-40).
class device_executor {
public:
    explicit device_executor(int device = 0) { detail::check(reseq_cuda_ctx_create(device, &ctx_)); }
    device_executor(const device_executor&) = delete;
    device_executor& operator=(const device_executor&) = delete;
    ~device_executor() { reseq_cuda_ctx_destroy(ctx_); }
    reseq_cuda_ctx* handle() const { return ctx_; }

private:
    reseq_cuda_ctx* ctx_ = nullptr;
};

inline std::vector<std::uint32_t> exclusive_scan(std::span<const std::uint32_t> values,
                                                 const device_executor& dev) {
    std::vector<std::uint32_t> out(values.size());
    detail::check(reseq_cuda_exclusive_scan(dev.handle(), values.data(), values.size(), out.data()));
    return out;
}

inline key_array split_by_bit(const key_array& arr, unsigned bit, const device_executor& dev) {
    key_array out;
    out.keys.resize(arr.keys.size());
    out.payload.resize(arr.payload.size());
    detail::check(reseq_cuda_split_by_bit(dev.handle(), arr.keys.data(),
                                          arr.has_payload() ? arr.payload.data() : nullptr, arr.keys.size(), bit,
                                          out.keys.data(), arr.has_payload() ? out.payload.data() : nullptr));
    return out;
}

/// detail::split_destinations, radix_sort.hpp:35-52 (Alg. 1).
struct split_plan {
    std::vector<std::uint32_t> destinations;
    std::uint32_t total_false = 0;
};
inline split_plan split_destinations(std::span<const std::uint32_t> keys, unsigned bit, const device_executor& dev) {
    split_plan plan;
    plan.destinations.resize(keys.size());
    detail::check(reseq_cuda_split_destinations(dev.handle(), keys.data(), keys.size(), bit, plan.destinations.data(),
                                                &plan.total_false));
    return plan;
}
/// detail::phase_is_sorted, radix_sort.hpp:54-66.
inline bool phase_is_sorted(std::span<const std::uint32_t> keys, const device_executor& dev) {
    int sorted = 1;
    detail::check(reseq_cuda_is_sorted(dev.handle(), keys.data(), keys.size(), &sorted));
    return sorted != 0;
}

inline key_array radix_sort(const key_array& arr, const device_executor& dev) {
    key_array out;
    out.keys.resize(arr.keys.size());
    out.payload.resize(arr.payload.size());
    detail::check(reseq_cuda_radix_sort(dev.handle(), arr.keys.data(),
                                        arr.has_payload() ? arr.payload.data() : nullptr, arr.keys.size(),
                                        out.keys.data(), arr.has_payload() ? out.payload.data() : nullptr));
    return out;
}

inline key_array chunked_radix_sort(const key_array& arr, const device_executor& dev, unsigned digit_bits = 4) {
    if (digit_bits < 1 || digit_bits > 8) throw std::invalid_argument("digit_bits must be in 1..8");
    key_array out;
    out.keys.resize(arr.keys.size());
    out.payload.resize(arr.payload.size());
    detail::check(reseq_cuda_chunked_radix_sort(dev.handle(), arr.keys.data(),
                                                arr.has_payload() ? arr.payload.data() : nullptr, arr.keys.size(),
                                                digit_bits, out.keys.data(),
                                                arr.has_payload() ? out.payload.data() : nullptr));
    return out;
}

inline suffix_array build_parallel(std::string_view text, const device_executor& dev) {
    suffix_array out;
    out.sa.resize(text.size());
    out.rank.resize(text.size());
    detail::check(reseq_cuda_build_sa(dev.handle(), reinterpret_cast<const std::uint8_t*>(text.data()), text.size(),
                                      out.sa.data(), out.rank.data(), nullptr),
                  text.size());
    return out;
}

/// fragment_index (fragment_index.hpp:30-167) resident on the device.  `concat` / `starts`
/// are fragment_set::concat() / starts(); unlike the reference the index copies what it
/// needs, so they need not outlive it.
class fragment_index {
public:
    fragment_index(std::string_view concat, std::span<const std::uint32_t> starts, const device_executor& dev)
        : concat_(concat), starts_(starts.begin(), starts.end()) {
        detail::check(reseq_cuda_index_create(dev.handle(), reinterpret_cast<const std::uint8_t*>(concat.data()),
                                              concat.size(), starts.data(), starts.size(), &ix_),
                      concat.size());
    }
#ifdef RESEQ_B200_WITH_REFERENCE
    /// The reference's own constructor shape (fragment_index.hpp:34): from a fragment_set.
    fragment_index(const fragment_set& set, const device_executor& dev)
        : fragment_index(std::string_view(set.concat()), std::span<const std::uint32_t>(set.starts()), dev) {}
#endif
    fragment_index(const fragment_index&) = delete;
    fragment_index& operator=(const fragment_index&) = delete;
    ~fragment_index() { reseq_cuda_index_destroy(ix_); }

    std::uint32_t length(std::uint32_t id) const {   // fragment_set::length, sequence.hpp:78-83
        const std::size_t end = (id + 1 < starts_.size() ? starts_[id + 1] : concat_.size()) - 1;
        return static_cast<std::uint32_t>(end - starts_[id]);
    }

    /// prefix_related(residual), fragment_index.hpp:72-80: the batched device query with q = 1.
    prefix_relation prefix_related(residual r) const {
        if (r.frag >= starts_.size() || r.offset >= length(r.frag)) throw offset_out_of_range_error(r.frag, r.offset);
        return prefix_related_batch(std::span<const residual>(&r, 1)).front();
    }
    /// The assembler's batch (find_fir_pairs, assembler.hpp:74-78: one independent query per fragment).
    std::vector<prefix_relation> prefix_related_batch(std::span<const residual> rs) const {
        std::vector<std::uint32_t> frag(rs.size()), off(rs.size());
        for (std::size_t i = 0; i < rs.size(); ++i) {
            frag[i] = rs[i].frag;
            off[i] = rs[i].offset;
        }
        reseq_prefix_relations rel{};
        const int st = reseq_cuda_index_prefix_related_batch(ix_, frag.data(), off.data(), rs.size(), &rel);
        if (st != RESEQ_OK) {
            reseq_cuda_prefix_relations_free(&rel);
            detail::check(st);
        }
        std::vector<prefix_relation> out(rs.size());
        for (std::size_t i = 0; i < rs.size(); ++i) {
            out[i].prefixes_of.assign(rel.prefixes + rel.prefixes_off[i], rel.prefixes + rel.prefixes_off[i + 1]);
            out[i].extensions_of.assign(rel.extensions + rel.extensions_off[i], rel.extensions + rel.extensions_off[i + 1]);
            out[i].exact_matches.assign(rel.exact + rel.exact_off[i], rel.exact + rel.exact_off[i + 1]);
        }
        reseq_cuda_prefix_relations_free(&rel);
        return out;
    }
    /// prefix_related(std::string_view), fragment_index.hpp:82-109, for arbitrary byte patterns: the
    /// interval searches -- one per distinct fragment length below |bytes| plus one for the whole pattern
    /// (at each length the reference's narrowed interval equals locate_prefix_range of that prefix, :75-80)
    /// -- run on the device as ONE batch; the classification over start_rank_list is the reference's, on
    /// the host.  Like the reference (:91), a pattern whose interval empties at an intermediate length
    /// returns at once with prefixes_of in (length, rank) order.
    prefix_relation prefix_related(std::string_view bytes) const {
        load_start_tables();
        prefix_relation rel;
        const std::size_t m = bytes.size();
        std::vector<std::uint32_t> cuts;
        for (std::uint32_t len : lengths_) {
            if (len >= m) break;
            cuts.push_back(len);
        }
        std::string blob;
        std::vector<std::uint64_t> offs{0};
        for (std::uint32_t c : cuts) {
            blob.append(bytes.substr(0, c));
            offs.push_back(blob.size());
        }
        blob.append(bytes);
        offs.push_back(blob.size());
        std::vector<std::uint32_t> lo(offs.size() - 1), hi(offs.size() - 1);
        detail::check(reseq_cuda_index_locate_batch(ix_, reinterpret_cast<const std::uint8_t*>(blob.data()), offs.data(),
                                                    lo.size(), lo.data(), hi.data()));
        auto range = [&](std::size_t q) {
            return std::pair(std::lower_bound(start_rank_.begin(), start_rank_.end(), lo[q]) - start_rank_.begin(),
                             std::lower_bound(start_rank_.begin(), start_rank_.end(), hi[q]) - start_rank_.begin());
        };
        for (std::size_t t = 0; t < cuts.size(); ++t) {
            if (lo[t] == hi[t]) return rel;                                  // :91
            const auto [a, b] = range(t);
            for (auto u = a; u < b; ++u)                                     // collect_starts_of_length, :150-158
                if (length(start_frag_[u]) == cuts[t]) rel.prefixes_of.push_back(start_frag_[u]);
        }
        const auto [a, b] = range(cuts.size());
        for (auto u = a; u < b; ++u) {
            const std::uint32_t id = start_frag_[u], len = length(id);
            if (len > m) rel.extensions_of.push_back(id);
            else if (len == m) rel.exact_matches.push_back(id);
        }
        std::sort(rel.prefixes_of.begin(), rel.prefixes_of.end());
        std::sort(rel.extensions_of.begin(), rel.extensions_of.end());
        std::sort(rel.exact_matches.begin(), rel.exact_matches.end());
        return rel;
    }

    suffix_array sa() const {
        suffix_array out;
        out.sa.resize(concat_.size());
        out.rank.resize(concat_.size());
        detail::check(reseq_cuda_index_get(ix_, out.sa.data(), out.rank.data(), nullptr));
        return out;
    }
    std::vector<std::uint32_t> start_rank_list() const {
        std::vector<std::uint32_t> out(starts_.size());
        detail::check(reseq_cuda_index_get(ix_, nullptr, nullptr, out.data()));
        return out;
    }
    std::pair<std::uint32_t, std::uint32_t> locate_prefix_range(std::string_view pattern) const {
        const std::uint64_t off[2] = {0, pattern.size()};
        std::uint32_t lo = 0, hi = 0;
        detail::check(reseq_cuda_index_locate_batch(ix_, reinterpret_cast<const std::uint8_t*>(pattern.data()), off,
                                                    1, &lo, &hi));
        return {lo, hi};
    }
    /// greedy_superstring_with_order (overlap.hpp:80-113): device overlaps >= min_overlap, host merge.
    greedy_result greedy_superstring_with_order(std::uint32_t min_overlap = 1) const {
        reseq_overlaps ov{};
        detail::check(reseq_cuda_index_overlaps(ix_, min_overlap, &ov));
        greedy_result res;
        res.superstring.resize(concat_.size());
        res.order.resize(starts_.size());
        std::size_t sl = 0, ol = 0;
        const int st = reseq_greedy_superstring(reinterpret_cast<const std::uint8_t*>(concat_.data()), concat_.size(),
                                                starts_.data(), starts_.size(), &ov, min_overlap,
                                                reinterpret_cast<std::uint8_t*>(res.superstring.data()), &sl,
                                                res.order.data(), &ol);
        reseq_cuda_overlaps_free(&ov);
        detail::check(st);
        res.superstring.resize(sl);
        res.order.resize(ol);
        return res;
    }

private:
    void load_start_tables() const {   // start_rank_list_, frag_at_start_ along it, lengths_ (fragment_index.hpp:40-55)
        if (!start_rank_.empty() || starts_.empty()) return;
        start_rank_.resize(starts_.size());
        start_frag_.resize(starts_.size());
        detail::check(reseq_cuda_index_get(ix_, nullptr, nullptr, start_rank_.data()));
        detail::check(reseq_cuda_index_start_fragments(ix_, start_frag_.data()));
        for (std::uint32_t id = 0; id < starts_.size(); ++id) lengths_.push_back(length(id));
        std::sort(lengths_.begin(), lengths_.end());
        lengths_.erase(std::unique(lengths_.begin(), lengths_.end()), lengths_.end());
    }

    std::string concat_;
    std::vector<std::uint32_t> starts_;
    reseq_cuda_index* ix_ = nullptr;
    mutable std::vector<std::uint32_t> start_rank_, start_frag_, lengths_;
};

}  // namespace reseq::cuda
