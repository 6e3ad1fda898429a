// C-ABI entry points (include/reseq_cuda.h) for the context, the L0 primitives and the
// suffix-array builder.  Index entry points live in index.cu; host-only ones in host/.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "radix.cuh"
#include "sa.cuh"
#include "scan.cuh"

namespace rsq {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

}  // namespace rsq

using namespace rsq;

int reseq_cuda_ctx::reserve(size_t bytes) {
    if (bytes <= arena_cap) return RESEQ_OK;
    RSQ_CUDA(cudaStreamSynchronize(stream));
    if (arena) RSQ_CUDA(cudaFree(arena));
    arena = nullptr;
    arena_cap = 0;
    const size_t want = bytes + (bytes >> 4) + (1u << 20);  // headroom against regrowth
    cudaError_t e = cudaMalloc(&arena, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        {   // blocks cached by the index allocator's pool are of no use to cudaMalloc: hand them back
            cudaMemPool_t pool = nullptr;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess && pool) cudaMemPoolTrimTo(pool, 0);
            cudaGetLastError();
        }
        e = cudaMalloc(&arena, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(RESEQ_OUT_OF_MEMORY,
                        "cudaMalloc of " + std::to_string(bytes) + " workspace bytes failed");
        }
        arena_cap = bytes;
    } else {
        arena_cap = want;
    }
    return RESEQ_OK;
}

cudaEvent_t reseq_cuda_ctx::take_event() {
    if (!event_pool.empty()) {
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

namespace {

int check_ctx(reseq_cuda_ctx* ctx) {
    if (!ctx) return fail(RESEQ_INVALID_ARGUMENT, "null context");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return fail(RESEQ_CUDA_ERROR, cudaGetErrorString(e));
    return RESEQ_OK;
}

// u32-key sort with an optional payload on device buffers; digit passes of `digit_bits`
// bits; passes whose digit is constant over the array are skipped.
int sort_u32(reseq_cuda_ctx* ctx, u32* ka, u32* kb, u32* va, u32* vb, size_t n, int lo_bit,
             int hi_bit, int digit_bits, bool* in_b) {
    *in_b = false;
    if (n < 2) return RESEQ_OK;
    SortWorkspace ws;
    RSQ_TRY(sort_workspace_carve(ctx, n, &ws));
    const PassTable pt = make_passes(lo_bit, hi_bit, digit_bits);
    RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * pt.count * kRadix, ctx->stream));
    {
        const int block = 512;
        size_t want = (n + block * 8 - 1) / (block * 8);
        const size_t cap = static_cast<size_t>(ctx->sm_count) * 4;
        const unsigned grid = static_cast<unsigned>(want < cap ? (want ? want : 1) : cap);
        RSQ_LAUNCH_BEGIN(ctx, "hist_kernel");
        hist_kernel<u32><<<grid, block, sizeof(u32) * pt.count * kRadix, ctx->stream>>>(ka, n, pt, ws.hist);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
    }
    std::vector<u32> hist(static_cast<size_t>(pt.count) * kRadix);
    RSQ_CUDA(cudaMemcpyAsync(hist.data(), ws.hist, hist.size() * sizeof(u32), cudaMemcpyDeviceToHost,
                             ctx->stream));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    u32 skip = 0;
    for (int p = 0; p < pt.count; ++p)
        for (int d = 0; d < kRadix; ++d)
            if (hist[static_cast<size_t>(p) * kRadix + d] == n) skip |= 1u << p;
    return onesweep_sort<u32>(ctx, ka, kb, va, vb, n, pt, ws, true, skip, in_b);
}

int sort_u32_host(reseq_cuda_ctx* ctx, const u32* keys, const u32* payload, size_t n, int lo_bit,
                  int hi_bit, int digit_bits, u32* keys_out, u32* payload_out) {
    RSQ_TRY(check_ctx(ctx));
    if ((payload == nullptr) != (payload_out == nullptr))
        return fail(RESEQ_INVALID_ARGUMENT, "payload and payload_out must both be given or both be null");
    if (n == 0) return RESEQ_OK;
    if (!keys || !keys_out) return fail(RESEQ_INVALID_ARGUMENT, "null key buffer");
    if (n > RESEQ_CUDA_MAX_TEXT) return fail(RESEQ_INVALID_ARGUMENT, "more than 2^32-2 keys");
    const bool has_val = payload != nullptr;
    const size_t arr = reseq_cuda_ctx::padded(sizeof(u32) * n);
    RSQ_TRY(ctx->reserve(arr * (has_val ? 4 : 2) + sort_workspace_bytes(n) + 4096));
    ctx->begin();
    u32* ka = ctx->alloc<u32>(n);
    u32* kb = ctx->alloc<u32>(n);
    u32* va = has_val ? ctx->alloc<u32>(n) : nullptr;
    u32* vb = has_val ? ctx->alloc<u32>(n) : nullptr;
    RSQ_CUDA(cudaMemcpyAsync(ka, keys, sizeof(u32) * n, cudaMemcpyHostToDevice, ctx->stream));
    if (has_val)
        RSQ_CUDA(cudaMemcpyAsync(va, payload, sizeof(u32) * n, cudaMemcpyHostToDevice, ctx->stream));
    bool in_b = false;
    RSQ_TRY(sort_u32(ctx, ka, kb, va, vb, n, lo_bit, hi_bit, digit_bits, &in_b));
    RSQ_CUDA(cudaMemcpyAsync(keys_out, in_b ? kb : ka, sizeof(u32) * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (has_val)
        RSQ_CUDA(cudaMemcpyAsync(payload_out, in_b ? vb : va, sizeof(u32) * n, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    return RESEQ_OK;
}

}  // namespace

extern "C" {

const char* reseq_cuda_last_error(void) { return g_last_error.c_str(); }
const char* reseq_cuda_version(void) { return "reseq-b200 0.1 (sm_100a)"; }

int reseq_cuda_ctx_create(int device, reseq_cuda_ctx** out) {
    if (!out) return fail(RESEQ_INVALID_ARGUMENT, "null out pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(RESEQ_NO_DEVICE,
                    "no CUDA device: the reseq B200 backend has no CPU fallback");
    }
    if (device < 0 || device >= count)
        return fail(RESEQ_INVALID_ARGUMENT, "device ordinal out of range");
    RSQ_CUDA(cudaSetDevice(device));
    auto* ctx = new reseq_cuda_ctx();
    ctx->device = device;
    cudaDeviceProp prop{};
    RSQ_CUDA(cudaGetDeviceProperties(&prop, device));
    ctx->sm_count = prop.multiProcessorCount > 0 ? prop.multiProcessorCount : kSmCount;
    RSQ_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    RSQ_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    RSQ_CUDA(cudaEventCreateWithFlags(&ctx->copy_event, cudaEventDisableTiming));
    ctx->stream = ctx->own_stream;
    RSQ_CUDA(cudaMallocHost(&ctx->pinned, 4096));
    {   // index arrays come from the default memory pool: keep freed blocks cached for the next index
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess && pool) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    if (const char* e = std::getenv("RESEQ_SORT_CFG")) ctx->opt_sort_cfg = std::atoi(e);      // tuning only
    if (const char* e = std::getenv("RESEQ_INVERSE_LO_BITS")) ctx->opt_inverse_lo_bits = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_INVERSE_MODE")) ctx->opt_inverse_mode = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_LOOKBACK_PACK")) ctx->opt_lookback_pack = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SORT_TMA")) ctx->opt_sort_tma = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SORT_PRMT")) ctx->opt_sort_prmt = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_OWNER_BINS")) ctx->opt_owner_bins = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_ACCEPT_QUADS")) ctx->opt_accept_quads = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_ACCEPT_EXC")) ctx->opt_accept_exc = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_OVERLAP_STAGE")) ctx->opt_overlap_stage = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_LOOKAHEAD")) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= 8) ctx->opt_lookahead = v;
    }
    if (const char* e = std::getenv("RESEQ_SA_UNIFORM")) ctx->opt_uniform = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SA_RAGGED")) ctx->opt_ragged = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SA_SPECULATE")) ctx->opt_speculate = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SA_GRAPH")) ctx->opt_graph = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SA_DOUBLING_LOCAL")) ctx->opt_doubling_local = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SA_SHORTCUT")) ctx->opt_shortcut = std::atoi(e);
    if (const char* e = std::getenv("RESEQ_SA_TEXT_ROUNDS")) ctx->opt_text_rounds = std::atoi(e);
    *out = ctx;
    return RESEQ_OK;
}

void reseq_cuda_ctx_destroy(reseq_cuda_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->drop_spec_graph();
    if (ctx->arena) cudaFree(ctx->arena);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (auto& r : ctx->profile) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->copy_event) cudaEventDestroy(ctx->copy_event);
    delete ctx;
}

int reseq_cuda_ctx_set_stream(reseq_cuda_ctx* ctx, void* cuda_stream) {
    RSQ_TRY(check_ctx(ctx));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
    ++ctx->option_epoch;
    return RESEQ_OK;
}

int reseq_cuda_ctx_synchronize(reseq_cuda_ctx* ctx) {
    RSQ_TRY(check_ctx(ctx));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    return RESEQ_OK;
}

int reseq_cuda_ctx_set_option(reseq_cuda_ctx* ctx, const char* name, long long value) {
    if (!ctx || !name) return fail(RESEQ_INVALID_ARGUMENT, "null argument");
    ++ctx->option_epoch;   // whatever changes: a captured build graph is rebuilt
    if (std::strcmp(name, "sa_graph") == 0) {
        ctx->opt_graph = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sa_text_rounds") == 0) {
        if (value < 0 || value > 1024) return fail(RESEQ_INVALID_ARGUMENT, "sa_text_rounds must be in 0..1024");
        ctx->opt_text_rounds = static_cast<int>(value);
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sa_shortcut") == 0) {
        ctx->opt_shortcut = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sa_uniform") == 0) {
        ctx->opt_uniform = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sa_ragged") == 0) {
        ctx->opt_ragged = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "overlap_stage") == 0) {
        ctx->opt_overlap_stage = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sort_tma") == 0) {
        ctx->opt_sort_tma = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sa_doubling_local") == 0) {
        ctx->opt_doubling_local = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sa_speculate") == 0) {
        ctx->opt_speculate = value != 0;
        return RESEQ_OK;
    }
    if (std::strcmp(name, "inverse_mode") == 0) {
        if (value < 0 || value > 1) return fail(RESEQ_INVALID_ARGUMENT, "inverse_mode must be 0 or 1");
        ctx->opt_inverse_mode = static_cast<int>(value);
        return RESEQ_OK;
    }
    if (std::strcmp(name, "sort_cfg") == 0) {
        if (value < 0 || value > 9) return fail(RESEQ_INVALID_ARGUMENT, "sort_cfg must be in 0..9");
        ctx->opt_sort_cfg = static_cast<int>(value);
        return RESEQ_OK;
    }
    return fail(RESEQ_INVALID_ARGUMENT, std::string("unknown option ") + name);
}

int reseq_cuda_ctx_profile(reseq_cuda_ctx* ctx, int enable) {
    RSQ_TRY(check_ctx(ctx));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    if (enable) {
        for (auto& r : ctx->profile) {
            ctx->event_pool.push_back(r.e0);
            ctx->event_pool.push_back(r.e1);
        }
        ctx->profile.clear();
    }
    ctx->profiling = enable != 0;
    return RESEQ_OK;
}

size_t reseq_cuda_ctx_profile_read(reseq_cuda_ctx* ctx, reseq_kernel_profile* out, size_t cap) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    std::vector<reseq_kernel_profile> agg;
    for (const auto& r : ctx->profile) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        size_t t = 0;
        while (t < agg.size() && std::strncmp(agg[t].name, r.name, sizeof(agg[t].name)) != 0) ++t;
        if (t == agg.size()) {
            reseq_kernel_profile p{};
            std::strncpy(p.name, r.name, sizeof(p.name) - 1);
            agg.push_back(p);
        }
        agg[t].launches += 1;
        agg[t].total_ms += ms;
    }
    for (size_t t = 0; t < agg.size() && t < cap; ++t) out[t] = agg[t];
    return agg.size();
}

uint64_t reseq_cuda_ctx_launch_count(const reseq_cuda_ctx* ctx) { return ctx ? ctx->launches : 0; }
size_t reseq_cuda_ctx_workspace_bytes(const reseq_cuda_ctx* ctx) { return ctx ? ctx->arena_cap : 0; }

// ---- exclusive_scan ---------------------------------------------------------------

static int scan_with_total(reseq_cuda_ctx* ctx, const u32* d_values, size_t n, u32* d_out,
                           uint64_t* total_out) {
    u64* d_total = ctx->alloc<u64>(1);
    if (!d_total) return fail(RESEQ_OUT_OF_MEMORY, "scan workspace was not reserved");
    RSQ_TRY(exclusive_scan_device(ctx, d_values, d_out, n, d_total));
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_total, sizeof(u64), cudaMemcpyDeviceToHost, ctx->stream));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    const u64 total = *reinterpret_cast<volatile u64*>(ctx->pinned);
    if (total_out) *total_out = total;
    if (total > 0xFFFFFFFFull) return fail(RESEQ_SCAN_OVERFLOW, "prefix sum exceeds 32-bit range");
    return RESEQ_OK;
}

int reseq_cuda_exclusive_scan_device(reseq_cuda_ctx* ctx, const uint32_t* d_values, size_t n,
                                     uint32_t* d_out, uint64_t* total_out) {
    RSQ_TRY(check_ctx(ctx));
    if (total_out) *total_out = 0;
    if (n == 0) return RESEQ_OK;
    if (!d_values || !d_out) return fail(RESEQ_INVALID_ARGUMENT, "null device buffer");
    RSQ_TRY(ctx->reserve(scan_workspace_bytes(n) + 4096));
    ctx->begin();
    return scan_with_total(ctx, d_values, n, d_out, total_out);
}

int reseq_cuda_exclusive_scan(reseq_cuda_ctx* ctx, const uint32_t* values, size_t n, uint32_t* out) {
    RSQ_TRY(check_ctx(ctx));
    if (n == 0) return RESEQ_OK;
    if (!values || !out) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    const size_t arr = reseq_cuda_ctx::padded(sizeof(u32) * n);
    RSQ_TRY(ctx->reserve(2 * arr + scan_workspace_bytes(n) + 4096));
    ctx->begin();
    u32* d_in = ctx->alloc<u32>(n);
    u32* d_out = ctx->alloc<u32>(n);
    RSQ_CUDA(cudaMemcpyAsync(d_in, values, sizeof(u32) * n, cudaMemcpyHostToDevice, ctx->stream));
    RSQ_TRY(scan_with_total(ctx, d_in, n, d_out, nullptr));
    RSQ_CUDA(cudaMemcpyAsync(out, d_out, sizeof(u32) * n, cudaMemcpyDeviceToHost, ctx->stream));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    return RESEQ_OK;
}

// ---- split / sorts ----------------------------------------------------------------

}  // extern "C"

namespace {

// Alg. 1 (radix_sort.hpp:35-52) as three phases: e = 1 - bit, f = exclusive scan
// of e (single-pass decoupled look-back scan instead of the listing's Hillis-Steele loop), then
// d = bit ? i - f + tof : f.
__global__ void split_flags_kernel(const u32* __restrict__ keys, size_t n, unsigned bit, u32* __restrict__ e) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        e[i] = ((keys[i] >> bit) & 1u) ^ 1u;
}

__global__ void split_dest_kernel(const u32* __restrict__ keys, const u32* __restrict__ f, size_t n, unsigned bit,
                                  const u64* __restrict__ tof, u32* __restrict__ d) {
    const u32 total_false = static_cast<u32>(*tof);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        d[i] = ((keys[i] >> bit) & 1u) ? static_cast<u32>(i) - f[i] + total_false : f[i];
}

__global__ void is_sorted_kernel(const u32* __restrict__ keys, size_t n, u32* __restrict__ unsorted) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    bool bad = false;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < n; i += stride)
        bad |= keys[i - 1] > keys[i];
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(unsorted, 1u);
}

unsigned stream_grid(const reseq_cuda_ctx* ctx, size_t n) {
    const size_t want = (n + 1023) / 1024, cap = static_cast<size_t>(ctx->sm_count) * 16;
    return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

extern "C" {

int reseq_cuda_split_destinations(reseq_cuda_ctx* ctx, const uint32_t* keys, size_t n, unsigned bit,
                                  uint32_t* destinations, uint32_t* total_false) {
    if (bit > 31) return fail(RESEQ_INVALID_ARGUMENT, "bit must be in 0..31");
    RSQ_TRY(check_ctx(ctx));
    if (total_false) *total_false = 0;
    if (n == 0) return RESEQ_OK;
    if (!keys || !destinations) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    if (n > RESEQ_CUDA_MAX_TEXT) return fail(RESEQ_INVALID_ARGUMENT, "more than 2^32-2 keys");
    const size_t arr = reseq_cuda_ctx::padded(sizeof(u32) * n);
    RSQ_TRY(ctx->reserve(4 * arr + scan_workspace_bytes(n) + 4096));
    ctx->begin();
    u32* d_keys = ctx->alloc<u32>(n);
    u32* d_e = ctx->alloc<u32>(n);
    u32* d_f = ctx->alloc<u32>(n);
    u32* d_d = ctx->alloc<u32>(n);
    u64* d_tof = ctx->alloc<u64>(1);
    if (!d_keys || !d_e || !d_f || !d_d || !d_tof) return fail(RESEQ_OUT_OF_MEMORY, "split workspace");
    cudaStream_t s = ctx->stream;
    RSQ_CUDA(cudaMemcpyAsync(d_keys, keys, sizeof(u32) * n, cudaMemcpyHostToDevice, s));
    RSQ_LAUNCH_BEGIN(ctx, "split_flags_kernel");
    split_flags_kernel<<<stream_grid(ctx, n), 256, 0, s>>>(d_keys, n, bit, d_e);
    RSQ_LAUNCH_END(ctx);
    RSQ_TRY(exclusive_scan_device(ctx, d_e, d_f, n, d_tof));   // the total of e is tof = e[n-1] + f[n-1]
    RSQ_LAUNCH_BEGIN(ctx, "split_dest_kernel");
    split_dest_kernel<<<stream_grid(ctx, n), 256, 0, s>>>(d_keys, d_f, n, bit, d_tof, d_d);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(destinations, d_d, sizeof(u32) * n, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_tof, sizeof(u64), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    if (total_false) *total_false = static_cast<uint32_t>(*reinterpret_cast<volatile u64*>(ctx->pinned));
    return RESEQ_OK;
}

int reseq_cuda_is_sorted(reseq_cuda_ctx* ctx, const uint32_t* keys, size_t n, int* sorted) {
    RSQ_TRY(check_ctx(ctx));
    if (!sorted) return fail(RESEQ_INVALID_ARGUMENT, "null out pointer");
    *sorted = 1;
    if (n < 2) return RESEQ_OK;
    if (!keys) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    RSQ_TRY(ctx->reserve(reseq_cuda_ctx::padded(sizeof(u32) * n) + 4096));
    ctx->begin();
    u32* d_keys = ctx->alloc<u32>(n);
    u32* d_flag = ctx->alloc<u32>(1);
    if (!d_keys || !d_flag) return fail(RESEQ_OUT_OF_MEMORY, "is_sorted workspace");
    cudaStream_t s = ctx->stream;
    RSQ_CUDA(cudaMemcpyAsync(d_keys, keys, sizeof(u32) * n, cudaMemcpyHostToDevice, s));
    RSQ_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(u32), s));
    RSQ_LAUNCH_BEGIN(ctx, "is_sorted_kernel");
    is_sorted_kernel<<<stream_grid(ctx, n), 256, 0, s>>>(d_keys, n, d_flag);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_flag, sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    *sorted = *reinterpret_cast<volatile u32*>(ctx->pinned) == 0 ? 1 : 0;
    return RESEQ_OK;
}

int reseq_cuda_split_by_bit(reseq_cuda_ctx* ctx, const uint32_t* keys, const uint32_t* payload,
                            size_t n, unsigned bit, uint32_t* keys_out, uint32_t* payload_out) {
    if (bit > 31) return fail(RESEQ_INVALID_ARGUMENT, "bit must be in 0..31");
    RSQ_TRY(check_ctx(ctx));
    if ((payload == nullptr) != (payload_out == nullptr))
        return fail(RESEQ_INVALID_ARGUMENT, "payload and payload_out must both be given or both be null");
    if (n == 0) return RESEQ_OK;
    if (!keys || !keys_out) return fail(RESEQ_INVALID_ARGUMENT, "null key buffer");
    if (n == 1) {  // the sort path returns early below two keys; a split of one key is a copy
        keys_out[0] = keys[0];
        if (payload) payload_out[0] = payload[0];
        return RESEQ_OK;
    }
    // One stable 1-bit digit pass == Alg. 1's split (radix_sort.hpp:35-52).
    return sort_u32_host(ctx, keys, payload, n, static_cast<int>(bit), static_cast<int>(bit) + 1, 1,
                         keys_out, payload_out);
}

int reseq_cuda_radix_sort(reseq_cuda_ctx* ctx, const uint32_t* keys, const uint32_t* payload,
                          size_t n, uint32_t* keys_out, uint32_t* payload_out) {
    if (n == 1 && keys && keys_out) {
        keys_out[0] = keys[0];
        if (payload && payload_out) payload_out[0] = payload[0];
        return RESEQ_OK;
    }
    return sort_u32_host(ctx, keys, payload, n, 0, 32, kRadixBits, keys_out, payload_out);
}

int reseq_cuda_chunked_radix_sort(reseq_cuda_ctx* ctx, const uint32_t* keys, const uint32_t* payload,
                                  size_t n, unsigned digit_bits, uint32_t* keys_out,
                                  uint32_t* payload_out) {
    if (digit_bits < 1 || digit_bits > 8)
        return fail(RESEQ_INVALID_ARGUMENT, "digit_bits must be in 1..8");
    if (n == 1 && keys && keys_out) {
        keys_out[0] = keys[0];
        if (payload && payload_out) payload_out[0] = payload[0];
        return RESEQ_OK;
    }
    return sort_u32_host(ctx, keys, payload, n, 0, 32, static_cast<int>(digit_bits), keys_out,
                         payload_out);
}

int reseq_cuda_radix_sort_device(reseq_cuda_ctx* ctx, const uint32_t* d_keys, const uint32_t* d_payload,
                                 size_t n, uint32_t* d_keys_out, uint32_t* d_payload_out) {
    RSQ_TRY(check_ctx(ctx));
    if ((d_payload == nullptr) != (d_payload_out == nullptr))
        return fail(RESEQ_INVALID_ARGUMENT, "payload and payload_out must both be given or both be null");
    if (n == 0) return RESEQ_OK;
    if (!d_keys || !d_keys_out) return fail(RESEQ_INVALID_ARGUMENT, "null device key buffer");
    if (n > RESEQ_CUDA_MAX_TEXT) return fail(RESEQ_INVALID_ARGUMENT, "more than 2^32-2 keys");
    const bool has_val = d_payload != nullptr;
    const size_t arr = reseq_cuda_ctx::padded(sizeof(u32) * n);
    RSQ_TRY(ctx->reserve(arr * (has_val ? 2 : 1) + sort_workspace_bytes(n) + 4096));
    ctx->begin();
    // ping-pong between the caller's output buffer and one scratch buffer; the input is
    // copied into the output buffer first so the caller's input stays intact.
    u32* kb = ctx->alloc<u32>(n);
    u32* vb = has_val ? ctx->alloc<u32>(n) : nullptr;
    RSQ_CUDA(cudaMemcpyAsync(d_keys_out, d_keys, sizeof(u32) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    if (has_val)
        RSQ_CUDA(cudaMemcpyAsync(d_payload_out, d_payload, sizeof(u32) * n, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
    bool in_b = false;
    RSQ_TRY(sort_u32(ctx, d_keys_out, kb, has_val ? d_payload_out : nullptr, vb, n, 0, 32, kRadixBits, &in_b));
    if (in_b) {
        RSQ_CUDA(cudaMemcpyAsync(d_keys_out, kb, sizeof(u32) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        if (has_val)
            RSQ_CUDA(cudaMemcpyAsync(d_payload_out, vb, sizeof(u32) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    return RESEQ_OK;
}

// ---- suffix array -------------------------------------------------------------------

int reseq_cuda_build_sa_device(reseq_cuda_ctx* ctx, const uint8_t* d_text, size_t n, uint32_t* d_sa,
                               uint32_t* d_rank, reseq_sa_stats* stats) {
    RSQ_TRY(check_ctx(ctx));
    if (n > RESEQ_CUDA_MAX_TEXT)
        return fail(RESEQ_TEXT_TOO_LARGE, "text of length " + std::to_string(n) + " exceeds 2^32-2");
    if (n == 0) {
        if (stats) std::memset(stats, 0, sizeof(*stats));
        return RESEQ_OK;
    }
    if (!d_text || !d_sa) return fail(RESEQ_INVALID_ARGUMENT, "null device buffer");
    RSQ_TRY(ctx->reserve(sa_workspace_bytes(n)));
    ctx->begin();
    return build_sa_device(ctx, d_text, n, d_sa, d_rank, stats);
}

int reseq_cuda_build_sa(reseq_cuda_ctx* ctx, const uint8_t* text, size_t n, uint32_t* sa, uint32_t* rank,
                        reseq_sa_stats* stats) {
    RSQ_TRY(check_ctx(ctx));
    if (n > RESEQ_CUDA_MAX_TEXT)
        return fail(RESEQ_TEXT_TOO_LARGE, "text of length " + std::to_string(n) + " exceeds 2^32-2");
    if (n == 0) {
        if (stats) std::memset(stats, 0, sizeof(*stats));
        return RESEQ_OK;
    }
    if (!text || !sa) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    const size_t io = reseq_cuda_ctx::padded(n) + 2 * reseq_cuda_ctx::padded(sizeof(u32) * n);
    RSQ_TRY(ctx->reserve(sa_workspace_bytes(n) + io));
    ctx->begin();
    u8* d_text = ctx->alloc<u8>(n);
    u32* d_sa = ctx->alloc<u32>(n);
    u32* d_rank = ctx->alloc<u32>(n);
    RSQ_CUDA(cudaMemcpyAsync(d_text, text, n, cudaMemcpyHostToDevice, ctx->stream));
    ctx->sa_host_dst = sa;   // copied out by sa_ready() as soon as it is final, under the inverse's kernels
    ctx->sa_host_saved = sa;
    const int st = build_sa_device(ctx, d_text, n, d_sa, d_rank, stats);
    const bool sa_pending = ctx->sa_host_dst != nullptr;
    ctx->sa_host_dst = nullptr;
    ctx->sa_host_saved = nullptr;
    if (st != RESEQ_OK) {
        cudaStreamSynchronize(ctx->copy_stream);
        return st;
    }
    if (sa_pending) RSQ_CUDA(cudaMemcpyAsync(sa, d_sa, sizeof(u32) * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (rank)
        RSQ_CUDA(cudaMemcpyAsync(rank, d_rank, sizeof(u32) * n, cudaMemcpyDeviceToHost, ctx->stream));
    RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
    RSQ_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    return RESEQ_OK;
}

int reseq_cuda_checksum_u32_device(reseq_cuda_ctx* ctx, const uint32_t* d_v, size_t n, uint64_t* out) {
    RSQ_TRY(check_ctx(ctx));
    if (!out) return fail(RESEQ_INVALID_ARGUMENT, "null out pointer");
    uint64_t h = 14695981039346656037ull;
    const size_t chunk = size_t{1} << 22;
    std::vector<u32> buf(n < chunk ? n : chunk);
    for (size_t off = 0; off < n; off += chunk) {
        const size_t m = n - off < chunk ? n - off : chunk;
        RSQ_CUDA(cudaMemcpyAsync(buf.data(), d_v + off, sizeof(u32) * m, cudaMemcpyDeviceToHost, ctx->stream));
        RSQ_CUDA(cudaStreamSynchronize(ctx->stream));
        const unsigned char* b = reinterpret_cast<const unsigned char*>(buf.data());
        for (size_t i = 0; i < 4 * m; ++i) h = (h ^ b[i]) * 1099511628211ull;
    }
    *out = h;
    return RESEQ_OK;
}

}  // extern "C"
