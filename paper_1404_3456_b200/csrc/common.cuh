// Shared plumbing for the sm_100a backend: context, workspace arena, error handling,
// small device helpers.  Internal to the library (nothing here is ABI).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "reseq_cuda.h"

namespace rsq {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;

constexpr int kSmCount = 148;  // B200: 2 dies x 74 SMs; grids are sized in multiples of it

void set_last_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define RSQ_CUDA(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return ::rsq::fail(_e == cudaErrorMemoryAllocation ? RESEQ_OUT_OF_MEMORY       \
                                                               : RESEQ_CUDA_ERROR,         \
                               std::string(#expr) + ": " + cudaGetErrorString(_e));        \
    } while (0)

#define RSQ_TRY(expr)                  \
    do {                               \
        int _s = (expr);               \
        if (_s != RESEQ_OK) return _s; \
    } while (0)

// Opt a kernel in to more than 48 KB of dynamic shared memory.  The attribute is per DEVICE, a
// context may sit on any ordinal and contexts may be driven from several host threads: one bit
// per device and call site, set after the attribute is.
#define RSQ_OPT_IN_SMEM(ctx, kern, bytes)                                                               \
    do {                                                                                                \
        static std::atomic<uint64_t> _done[4];                                                          \
        const unsigned _dev = static_cast<unsigned>((ctx)->device) & 255u;                              \
        const uint64_t _bit = 1ull << (_dev & 63u);                                                     \
        if (!(_done[_dev >> 6].load(std::memory_order_acquire) & _bit)) {                               \
            RSQ_CUDA(cudaFuncSetAttribute((kern), cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                          static_cast<int>(bytes)));                                    \
            _done[_dev >> 6].fetch_or(_bit, std::memory_order_release);                                 \
        }                                                                                               \
    } while (0)

}  // namespace rsq

// The opaque context of the C ABI.
struct reseq_cuda_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int sm_count = rsq::kSmCount;
    uint64_t launches = 0;
    int opt_inverse_lo_bits = -1;  // bits of the first inverse partition pass (-1 = auto: at most 7; tuning)
    int opt_inverse_mode = 0;      // 0: two partition passes + shared-memory window; 1: one pass + L2-window scatter
    int opt_shortcut = 1;      // sentinel-distance shortcut in the refine kernel (tuning / tests)
    int opt_lookahead = 8;     // onesweep look-back descriptors in flight per digit (1..8)
    int opt_sort_cfg = 0;      // onesweep tile shape (0 = default tuning)
    int opt_overlap_stage = 0; // overlap search: a fragment's rank block + packed text staged in shared memory by TMA, double buffered (measured slower: off)
    int opt_sort_tma = 0;      // onesweep: full tiles loaded by one TMA bulk copy (measured 4 % slower than per-thread loads: off)
    int opt_sort_prmt = 1;     // onesweep: byte-aligned 8-bit digits of the upper key word extracted by one PRMT (0: shift + mask)
    int opt_accept_exc = 1;    // uniform route, accept pass: no proof-byte gather for t <= L - 64 when the reads with shorter proofs fit a 16-entry list
    int opt_accept_quads = 1;  // uniform route, accept pass: a thread owns four consecutive records (0: pairs)
    int opt_owner_bins = 128;   // rank exchange: owner x sub-range bins of the sender's partition pass (378 M positions, 8 owners: 1024 bins 2.58 ms, 256 2.33, 128 1.88, 32 1.80)
    int opt_lookback_pack = 1; // two digits per look-back descriptor word when n < 2^30 (0: always one)
    int opt_uniform = 1;       // transposed-record path for uniform read sets (0: general paths only)
    int opt_ragged = 1;        // ragged read sets (mixed read lengths <= 254) on the uniform route's flow (0: general records)
    int opt_text_rounds = 16;  // max text-window refinement rounds before prefix doubling takes over
    int opt_doubling_local = 1;  // doubling rounds: groups ordered in shared memory (0: always the global digit passes)
    int opt_speculate = 1;     // start on the previous build's route when the text length matches (verified on device)
    int opt_graph = 1;         // the speculative route replayed as ONE CUDA graph when nothing it captured has changed
    uint64_t option_epoch = 0; // bumped by every set_option / set_stream: invalidates the captured graph
    // The speculative route of build_sa_device has no host round trip inside and fixed launch shapes for a given
    // (n, period): captured once into a CUDA graph, it is replayed by one cudaGraphLaunch -- the ~30 launches and
    // memsets of a build otherwise leave 0.09 ms of gaps in a 0.60 ms build (config 1) and 0.11 ms at config 2.
    struct SpecGraph {
        cudaGraphExec_t exec = nullptr;
        size_t n = 0;
        uint32_t period = 0;
        const void* text = nullptr;
        void* sa = nullptr;
        void* rank = nullptr;
        char* arena = nullptr;
        size_t arena_cap = 0;
        cudaStream_t stream = nullptr;
        uint64_t epoch = 0;
        uint64_t launches = 0;
        reseq_sa_stats stats{};
    } spec_graph;
    void drop_spec_graph() {
        if (spec_graph.exec) cudaGraphExecDestroy(spec_graph.exec);
        spec_graph = SpecGraph{};
    }
    size_t hint_n = 0;         // text length and period of the last build that finished on the uniform read-set route
    uint32_t hint_period = 0;

    // Grow-only bump arena.  begin() rewinds it; alloc() carves 256-byte aligned
    // blocks.  If the arena is too small the whole block is re-allocated *before* any
    // carve of the current operation (ops call reserve() with their total first).
    char* arena = nullptr;
    size_t arena_cap = 0;
    size_t arena_used = 0;

    // Host-buffer builds: the suffix array is final before its inverse is computed, so its D2H copy
    // is started on a second stream the moment it is (sa_ready), under the inverse's kernels.
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t copy_event = nullptr;
    uint32_t* sa_host_dst = nullptr;   // set by reseq_cuda_build_sa for the duration of one build
    uint32_t* sa_host_saved = nullptr; // the same pointer, kept so that a failed speculative route can copy again
    int sa_ready(const uint32_t* d_sa, size_t n) {
        if (!sa_host_dst) return RESEQ_OK;
        if (cudaEventRecord(copy_event, stream) != cudaSuccess || cudaStreamWaitEvent(copy_stream, copy_event, 0) != cudaSuccess ||
            cudaMemcpyAsync(sa_host_dst, d_sa, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, copy_stream) != cudaSuccess)
            return ::rsq::fail(RESEQ_CUDA_ERROR, "early copy-out of the suffix array failed");
        sa_host_dst = nullptr;
        return RESEQ_OK;
    }

    // pinned staging word for small D2H reads (round-termination flags etc.)
    uint64_t* pinned = nullptr;

    // Optional per-launch timing with CUDA events on the launching stream (bench.py's
    // live roofline).  Off by default; see reseq_cuda_ctx_profile().
    struct ProfileRec {
        const char* name;
        cudaEvent_t e0, e1;
    };
    bool profiling = false;
    std::vector<ProfileRec> profile;
    std::vector<cudaEvent_t> event_pool;
    cudaEvent_t take_event();

    int reserve(size_t bytes);
    void begin() { arena_used = 0; }
    template <typename T>
    T* alloc(size_t count) {
        size_t bytes = (count * sizeof(T) + 255) & ~size_t{255};
        if (arena_used + bytes > arena_cap) return nullptr;
        T* p = reinterpret_cast<T*>(arena + arena_used);
        arena_used += bytes;
        return p;
    }
    static size_t padded(size_t bytes) { return (bytes + 255) & ~size_t{255}; }
};

namespace rsq {

// Bracket one kernel launch: counts it, and records events around it when profiling.
inline void launch_begin(reseq_cuda_ctx* ctx, const char* name) {
    ++ctx->launches;
    if (!ctx->profiling) return;
    reseq_cuda_ctx::ProfileRec r{name, ctx->take_event(), ctx->take_event()};
    cudaEventRecord(r.e0, ctx->stream);
    ctx->profile.push_back(r);
}
inline void launch_end(reseq_cuda_ctx* ctx) {
    if (ctx->profiling) cudaEventRecord(ctx->profile.back().e1, ctx->stream);
}
#define RSQ_LAUNCH_BEGIN(ctx, name) ::rsq::launch_begin((ctx), (name))
#define RSQ_LAUNCH_END(ctx) ::rsq::launch_end((ctx))

// ---- device helpers --------------------------------------------------------------

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Streaming 128-bit global accesses: data touched once per pass should not displace the
// (small, hot) look-back descriptors and histograms from L1.
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream_v4(void* p, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// 128-bit load served by L2 (never a stale L1 line): data published by another CTA behind a flag.
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ u32 ld_relaxed_u32(const u32* p) {
    u32 v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(u32* p, u32 v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(u64* p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- TMA (bulk asynchronous copy engine), 1-D form ---------------------------------------------------
// One elected thread moves a whole contiguous tile between HBM and shared memory; completion of a load is
// counted in bytes on an mbarrier, a store is tracked by a bulk group.  Addresses and sizes are multiples
// of 16 bytes.  SASS: UBLKCP (cp.async.bulk), SYNCS.ARRIVE.TRANS64 (expect_tx), SYNCS.PHASECHK (try_wait).
__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 arrivals) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(arrivals) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");   // visible to the async proxy before any copy names it
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t"
        "}" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// global -> shared, completion signalled on `bar` (arm it with mbar_expect_tx for the same byte count first)
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// shared -> global.  Every thread that wrote the tile calls tma_store_fence() before the barrier that
// precedes the store (generic-proxy writes -> async proxy); the issuing thread waits for the group before
// the shared memory is reused or the CTA exits.
__device__ __forceinline__ void tma_store_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_1d(void* gmem_dst, const void* smem_src, u32 bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst), "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// Decoupled look-back descriptor: status in the top two bits, value below; one 64-bit
// word so a single relaxed store publishes both atomically.
constexpr u64 kDescAggregate = 1ull << 62;
constexpr u64 kDescInclusive = 2ull << 62;
constexpr u64 kDescValueMask = (1ull << 62) - 1;

inline unsigned bit_width_u64(u64 v) {
    unsigned b = 0;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

}  // namespace rsq
