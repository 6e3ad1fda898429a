// Host driver of the onesweep radix sort (kernels in radix.cuh).
#include "radix.cuh"

namespace rsq {

// One block per pass: exclusive scan of the 256 digit counts.
__global__ void __launch_bounds__(kRadix)
digit_base_kernel(const u32* __restrict__ g_hist, u32* __restrict__ g_base) {
    __shared__ u32 s_warp[kRadix / 32];
    const int d = threadIdx.x;
    const u32 c = g_hist[blockIdx.x * kRadix + d];
    u32 inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane_id()) >= o) inc += t;
    }
    if (lane_id() == 31) s_warp[d >> 5] = inc;
    __syncthreads();
    u32 add = 0;
    for (int w = 0; w < (d >> 5); ++w) add += s_warp[w];
    g_base[blockIdx.x * kRadix + d] = add + inc - c;
}

template <> struct SortTuning<u32, false> { static constexpr int kBlock = 256, kItems = 16; };
template <> struct SortTuning<u32, true>  { static constexpr int kBlock = 384, kItems = 12; };
template <> struct SortTuning<u64, true>  { static constexpr int kBlock = 256, kItems = 16; };
template <> struct SortTuning<u64, false> { static constexpr int kBlock = 384, kItems = 12; };

// The smallest tile among the tunings bounds the look-back arrays.
static constexpr size_t kMinTile = 256 * 8;

static size_t lookback_bytes(size_t tiles) {   // one 64-bit descriptor per (tile, digit) at most (DPW 1)
    return reseq_cuda_ctx::padded(sizeof(u64) * tiles * kRadix);
}

size_t sort_workspace_bytes(size_t n) {
    const size_t tiles = (n + kMinTile - 1) / kMinTile + 1;
    return reseq_cuda_ctx::padded(sizeof(u32) * kMaxPasses * kRadix) * 2 +
           reseq_cuda_ctx::padded(sizeof(u32) * kMaxPasses) + lookback_bytes(tiles);
}

int sort_workspace_carve(reseq_cuda_ctx* ctx, size_t n, SortWorkspace* ws) {
    const size_t tiles = (n + kMinTile - 1) / kMinTile + 1;
    ws->hist = ctx->alloc<u32>(kMaxPasses * kRadix);
    ws->base = ctx->alloc<u32>(kMaxPasses * kRadix);
    ws->tickets = ctx->alloc<u32>(kMaxPasses);
    ws->lookback_bytes = lookback_bytes(tiles);
    ws->lookback = ctx->alloc<u64>(ws->lookback_bytes / sizeof(u64));
    if (!ws->hist || !ws->base || !ws->tickets || !ws->lookback)
        return fail(RESEQ_OUT_OF_MEMORY, "sort workspace does not fit the reserved arena");
    return RESEQ_OK;
}

template <typename KeyT, bool HAS_VAL>
static const char* pass_name() {
    return sizeof(KeyT) == 8 ? (HAS_VAL ? "onesweep_u64_pairs" : "onesweep_u64_keys")
                             : (HAS_VAL ? "onesweep_u32_pairs" : "onesweep_u32_keys");
}

template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS, class EMIT, int HI, int DPW>
static int launch_pass_dpw(reseq_cuda_ctx* ctx, const void* kin, KeyT* kout, const u32* vin, u32* vout,
                           size_t n, int shift, u32 mask, const u32* base, u64* lookback, u32* ticket,
                           const EMIT& emit) {
    using Cfg = OnesweepCfg<KeyT, HAS_VAL, BLOCK, ITEMS>;
    auto kern = onesweep_kernel<KeyT, HAS_VAL, BLOCK, ITEMS, EMIT, HI, DPW>;
    const size_t smem = Cfg::kSmem + (EMIT::kActive ? sizeof(u32) * (kEmitCap + 2) : 0);
    RSQ_OPT_IN_SMEM(ctx, kern, smem);
    const size_t tiles = (n + Cfg::kTile - 1) / Cfg::kTile;
    // only the descriptor words of the tiles this pass really has need clearing
    RSQ_CUDA(cudaMemsetAsync(lookback, 0, sizeof(u64) * tiles * (kRadix / DPW), ctx->stream));
    RSQ_LAUNCH_BEGIN(ctx, (pass_name<KeyT, HAS_VAL>()));
    // bulk tile loads need 16-byte aligned sources (the arena's are; a caller's arrays may not be)
    const int use_tma = ctx->opt_sort_tma != 0 && (reinterpret_cast<uintptr_t>(kin) & 15) == 0 &&
                        (!HAS_VAL || (reinterpret_cast<uintptr_t>(vin) & 15) == 0);
    kern<<<static_cast<unsigned>(tiles), BLOCK, smem, ctx->stream>>>(
        kin, kout, vin, vout, n, HI == 2 ? (0x4440 | ((shift - 32) >> 3)) : (HI == 1 ? shift - 32 : shift), mask, base, lookback, ticket,
        emit, use_tma);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS, class EMIT, int HI>
static int launch_pass_kernel(reseq_cuda_ctx* ctx, const void* kin, KeyT* kout, const u32* vin, u32* vout,
                              size_t n, int shift, u32 mask, const u32* base, u64* lookback, u32* ticket,
                              const EMIT& emit) {
    // two digits per descriptor word while every count fits 30 bits (all configurations below 2^30 suffixes)
    if (n < kPackedLimit && ctx->opt_lookback_pack != 0)
        return launch_pass_dpw<KeyT, HAS_VAL, BLOCK, ITEMS, EMIT, HI, 2>(ctx, kin, kout, vin, vout, n, shift, mask, base,
                                                                          lookback, ticket, emit);
    return launch_pass_dpw<KeyT, HAS_VAL, BLOCK, ITEMS, EMIT, HI, 1>(ctx, kin, kout, vin, vout, n, shift, mask, base,
                                                                      lookback, ticket, emit);
}

template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS, class EMIT>
static int launch_pass_cfg(reseq_cuda_ctx* ctx, const void* kin, KeyT* kout, const u32* vin, u32* vout,
                           size_t n, int shift, u32 mask, const u32* base, u64* lookback, u32* ticket,
                           const EMIT& emit) {
    if constexpr (sizeof(KeyT) == 8) {
        if (shift >= 32 && (shift & 7) == 0 && mask == 0xffu && ctx->opt_sort_prmt != 0)   // a whole byte of the upper word
            return launch_pass_kernel<KeyT, HAS_VAL, BLOCK, ITEMS, EMIT, 2>(ctx, kin, kout, vin, vout, n, shift, mask,
                                                                            base, lookback, ticket, emit);
        if (shift >= 32)
            return launch_pass_kernel<KeyT, HAS_VAL, BLOCK, ITEMS, EMIT, 1>(ctx, kin, kout, vin, vout, n, shift, mask,
                                                                            base, lookback, ticket, emit);
    }
    return launch_pass_kernel<KeyT, HAS_VAL, BLOCK, ITEMS, EMIT, 0>(ctx, kin, kout, vin, vout, n, shift, mask, base,
                                                                        lookback, ticket, emit);
}

template <typename KeyT, bool HAS_VAL, class EMIT = EmitNone>
static int launch_pass(reseq_cuda_ctx* ctx, const void* kin, KeyT* kout, const u32* vin, u32* vout,
                       size_t n, int shift, u32 mask, const u32* base, u64* lookback,
                       u32* ticket, const EMIT& emit = EMIT{}) {
    // "sort_cfg" picks a tile shape (tuning knob; every shape gives the same result)
    if constexpr (!EMIT::kActive) {
        switch (ctx->opt_sort_cfg) {
            case 1: return launch_pass_cfg<KeyT, HAS_VAL, 512, 8, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 2: return launch_pass_cfg<KeyT, HAS_VAL, 512, 12, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 3: return launch_pass_cfg<KeyT, HAS_VAL, 256, 12, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 4: return launch_pass_cfg<KeyT, HAS_VAL, 256, 16, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 5: return launch_pass_cfg<KeyT, HAS_VAL, 384, 12, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 6: return launch_pass_cfg<KeyT, HAS_VAL, 384, 16, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 7: return launch_pass_cfg<KeyT, HAS_VAL, 512, 16, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 8: return launch_pass_cfg<KeyT, HAS_VAL, 384, 8, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            case 9: return launch_pass_cfg<KeyT, HAS_VAL, 256, 8, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base, lookback, ticket, emit);
            default: break;
        }
    }
    using T = SortTuning<KeyT, HAS_VAL>;
    return launch_pass_cfg<KeyT, HAS_VAL, T::kBlock, T::kItems, EMIT>(ctx, kin, kout, vin, vout, n, shift, mask, base,
                                                                     lookback, ticket, emit);
}

template <typename KeyT>
int onesweep_sort(reseq_cuda_ctx* ctx, KeyT* keys_a, KeyT* keys_b, u32* vals_a, u32* vals_b,
                  size_t n, const PassTable& pt, const SortWorkspace& ws, bool hist_ready,
                  u32 skip_mask, bool* in_b, const EmitMultiples* emit_last, const EmitStarts* emit_starts_last) {
    *in_b = false;
    if (n == 0 || pt.count == 0) return RESEQ_OK;
    const bool has_val = vals_a != nullptr;
    RSQ_CUDA(cudaMemsetAsync(ws.tickets, 0, sizeof(u32) * kMaxPasses, ctx->stream));
    if (!hist_ready) {
        RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * pt.count * kRadix, ctx->stream));
        const int block = 512;
        size_t want = (n + block * 8 - 1) / (block * 8);
        const unsigned grid = static_cast<unsigned>(want < static_cast<size_t>(ctx->sm_count) * 4 ? (want ? want : 1) : ctx->sm_count * 4);
        RSQ_LAUNCH_BEGIN(ctx, "hist_kernel");
        hist_kernel<KeyT><<<grid, block, sizeof(u32) * pt.count * kRadix, ctx->stream>>>(
            keys_a, n, pt, ws.hist);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
    }
    RSQ_LAUNCH_BEGIN(ctx, "digit_base_kernel");
    digit_base_kernel<<<pt.count, kRadix, 0, ctx->stream>>>(ws.hist, ws.base);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());

    KeyT* kin = keys_a;
    KeyT* kout = keys_b;
    u32* vin = vals_a;
    u32* vout = vals_b;
    bool flipped = false;
    int last_pass = -1;
    for (int p = 0; p < pt.count; ++p)
        if (!(skip_mask & (1u << p))) last_pass = p;
    for (int p = 0; p < pt.count; ++p) {
        if (skip_mask & (1u << p)) continue;
        if constexpr (sizeof(KeyT) == 8) {
            if (emit_last && !has_val && p == last_pass) {
                RSQ_TRY((launch_pass<KeyT, false, EmitMultiples>(ctx, kin, kout, nullptr, nullptr, n, pt.shift[p], pt.mask(p),
                                                                 ws.base + p * kRadix, ws.lookback, ws.tickets + p,
                                                                 *emit_last)));
                KeyT* tk = kin; kin = kout; kout = tk;
                flipped = !flipped;
                continue;
            }
            if (emit_starts_last && !has_val && p == last_pass) {
                RSQ_TRY((launch_pass<KeyT, false, EmitStarts>(ctx, kin, kout, nullptr, nullptr, n, pt.shift[p], pt.mask(p),
                                                              ws.base + p * kRadix, ws.lookback, ws.tickets + p,
                                                              *emit_starts_last)));
                KeyT* tk = kin; kin = kout; kout = tk;
                flipped = !flipped;
                continue;
            }
        }
        if (has_val)
            RSQ_TRY((launch_pass<KeyT, true>(ctx, kin, kout, vin, vout, n, pt.shift[p], pt.mask(p),
                                             ws.base + p * kRadix, ws.lookback, ws.tickets + p)));
        else
            RSQ_TRY((launch_pass<KeyT, false>(ctx, kin, kout, nullptr, nullptr, n, pt.shift[p],
                                              pt.mask(p), ws.base + p * kRadix, ws.lookback,
                                              ws.tickets + p)));
        KeyT* tk = kin; kin = kout; kout = tk;
        u32* tv = vin; vin = vout; vout = tv;
        flipped = !flipped;
    }
    *in_b = flipped;
    return RESEQ_OK;
}

template int onesweep_sort<u32>(reseq_cuda_ctx*, u32*, u32*, u32*, u32*, size_t, const PassTable&,
                                const SortWorkspace&, bool, u32, bool*, const EmitMultiples*, const EmitStarts*);
template int onesweep_sort<u64>(reseq_cuda_ctx*, u64*, u64*, u32*, u32*, size_t, const PassTable&,
                                const SortWorkspace&, bool, u32, bool*, const EmitMultiples*, const EmitStarts*);

}  // namespace rsq
