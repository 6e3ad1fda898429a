// executor_dispatch.hpp -- the `const executor&` plug point of the reference (
// executor.hpp:13-21): with one field added to executor_config,
//
//     struct executor_config { unsigned workers = 1; std::size_t chunk_size = ...; int device = -1; };
//
// every parallel operator of the reference forwards to the device when the executor it is handed
// names one -- one line at the top of build_parallel (suffix_array.hpp:61), exclusive_scan (scan.hpp:32),
// split_by_bit / radix_sort / chunked_radix_sort (radix_sort.hpp:126,143,169):
//
//     if (exec.config().device >= 0) return reseq::cuda::dispatch::<same name>(args..., exec.config().device);
//
// Call sites (bench.hpp:130-142, tools/reseq.cpp:270) stay untouched; --workers / --chunk-size keep
// their host meaning.  oracle/make_dropin.py applies exactly this patch to a scratch copy of the
// reference headers and tests/cpp/test_dropin.cpp runs the reference's own functions through it.
//
// This header must be included where reseq::key_array / reseq::suffix_array are already complete
// (it is included from the patched headers after those definitions) and only declares what it needs.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <string_view>
#include <vector>

#include "reseq_cuda.h"
#include "reseq/errors.hpp"

namespace reseq::cuda::dispatch {

namespace detail {
inline void check(int status, std::uint64_t n = 0) {
    switch (status) {
        case RESEQ_OK: return;
        case RESEQ_INVALID_ARGUMENT: throw std::invalid_argument(reseq_cuda_last_error());
        case RESEQ_TEXT_TOO_LARGE: throw ::reseq::text_too_large_error(n);
        case RESEQ_SCAN_OVERFLOW: throw ::reseq::scan_overflow_error();
        default: throw ::reseq::error(reseq_cuda_last_error());
    }
}

// One context per device ordinal for the life of the process (an executor is cheap to copy around in
// the reference; a device context is not).  One dispatch at a time per context, as for an executor
// (executor.hpp:39-40): the lock is held for the duration of a call.
struct context_slot {
    std::mutex busy;
    reseq_cuda_ctx* ctx = nullptr;
    ~context_slot() { reseq_cuda_ctx_destroy(ctx); }
};
inline context_slot& slot_of(int device) {
    static std::mutex table_lock;
    static std::map<int, std::unique_ptr<context_slot>> table;
    std::lock_guard<std::mutex> g(table_lock);
    auto& s = table[device];
    if (!s) {
        s = std::make_unique<context_slot>();
        check(reseq_cuda_ctx_create(device, &s->ctx));
    }
    return *s;
}
}  // namespace detail

template <typename SuffixArray>
inline SuffixArray build_parallel(std::string_view text, int device) {
    auto& slot = detail::slot_of(device);
    std::lock_guard<std::mutex> g(slot.busy);
    SuffixArray out;
    out.sa.resize(text.size());
    out.rank.resize(text.size());
    detail::check(reseq_cuda_build_sa(slot.ctx, reinterpret_cast<const std::uint8_t*>(text.data()), text.size(), out.sa.data(),
                                      out.rank.data(), nullptr),
                  text.size());
    return out;
}

inline std::vector<std::uint32_t> exclusive_scan(std::span<const std::uint32_t> values, int device) {
    auto& slot = detail::slot_of(device);
    std::lock_guard<std::mutex> g(slot.busy);
    std::vector<std::uint32_t> out(values.size());
    detail::check(reseq_cuda_exclusive_scan(slot.ctx, values.data(), values.size(), out.data()));
    return out;
}

template <typename KeyArray, typename F>
inline KeyArray sort_like(const KeyArray& arr, int device, F call) {
    auto& slot = detail::slot_of(device);
    std::lock_guard<std::mutex> g(slot.busy);
    KeyArray out;
    out.keys.resize(arr.keys.size());
    out.payload.resize(arr.payload.size());
    const bool pl = !arr.payload.empty();
    detail::check(call(slot.ctx, arr.keys.data(), pl ? arr.payload.data() : nullptr, arr.keys.size(), out.keys.data(),
                       pl ? out.payload.data() : nullptr));
    return out;
}
template <typename KeyArray>
inline KeyArray split_by_bit(const KeyArray& arr, unsigned bit, int device) {
    return sort_like(arr, device, [bit](reseq_cuda_ctx* c, const std::uint32_t* k, const std::uint32_t* p, std::size_t n,
                                       std::uint32_t* ko, std::uint32_t* po) { return reseq_cuda_split_by_bit(c, k, p, n, bit, ko, po); });
}
template <typename KeyArray>
inline KeyArray radix_sort(const KeyArray& arr, int device) {
    return sort_like(arr, device, [](reseq_cuda_ctx* c, const std::uint32_t* k, const std::uint32_t* p, std::size_t n,
                                    std::uint32_t* ko, std::uint32_t* po) { return reseq_cuda_radix_sort(c, k, p, n, ko, po); });
}
template <typename KeyArray>
inline KeyArray chunked_radix_sort(const KeyArray& arr, unsigned digit_bits, int device) {
    if (digit_bits < 1 || digit_bits > 8) throw std::invalid_argument("digit_bits must be in 1..8");   // radix_sort.hpp:171-172
    return sort_like(arr, device, [digit_bits](reseq_cuda_ctx* c, const std::uint32_t* k, const std::uint32_t* p, std::size_t n,
                                              std::uint32_t* ko, std::uint32_t* po) {
        return reseq_cuda_chunked_radix_sort(c, k, p, n, digit_bits, ko, po);
    });
}

}  // namespace reseq::cuda::dispatch
