// LSD radix sort for sm_100a: 8-bit digits, one "onesweep" kernel per digit pass.
//
//   - digit histograms for ALL passes of a sort are accumulated up front in shared
//     memory (hist_add, fused into whichever kernel produces the keys) and turned into
//     per-pass exclusive digit bases by digit_base_kernel;
//   - each pass is ONE kernel: tiles are claimed through an atomic ticket, keys are
//     ranked inside the warp with match.any (warp-aggregated: one shared-memory
//     read-modify-write per distinct digit per warp step, no atomics), tile totals are
//     chained across tiles by decoupled look-back (one 64-bit descriptor per digit), the
//     tile is re-ordered through shared memory so every digit's run leaves as one
//     contiguous, coalesced global store;
//   - HBM traffic per pass = read keys(+payload) once, write keys(+payload) once.
//
// Replaces the data flow of radix_sort.hpp:143-161 (32 one-bit split passes, each with a
// Hillis-Steele scan, scan.hpp:42-47) and of the paper's four-kernel radix pass
// (PAPER.md:258-271).  Result contract: stable ascending sort on the selected key bits.
#pragma once

#include "common.cuh"

namespace rsq {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kMaxPasses = 32;  // chunked_radix_sort with digit_bits = 1 needs 32

struct PassTable {
    int count;
    unsigned char shift[kMaxPasses];
    unsigned char bits[kMaxPasses];
    __host__ __device__ u32 mask(int p) const { return (1u << bits[p]) - 1u; }
};

// Passes covering key bits [lo_bit, hi_bit) with digits of `digit_bits` bits.
inline PassTable make_passes(int lo_bit, int hi_bit, int digit_bits = kRadixBits) {
    PassTable t{};
    for (int b = lo_bit; b < hi_bit && t.count < kMaxPasses; b += digit_bits) {
        t.shift[t.count] = static_cast<unsigned char>(b);
        t.bits[t.count] = static_cast<unsigned char>(hi_bit - b < digit_bits ? hi_bit - b : digit_bits);
        ++t.count;
    }
    return t;
}

template <typename KeyT>
__device__ __forceinline__ u32 key_digit(KeyT k, int shift, u32 mask) {
    return static_cast<u32>(k >> shift) & mask;
}

// ---- histogram ---------------------------------------------------------------------

// Adds one key's digit to a shared-memory histogram row.  Must be called by all 32
// lanes of a warp (`in` masks lanes without a key).  A warp whose keys all share the
// digit (the common case for the high digits of nearly-sorted keys) costs one atomic
// instead of a 32-way same-address conflict.
__device__ __forceinline__ void hist_add(u32* row, u32 d, bool in) {
    const unsigned act = __ballot_sync(0xffffffffu, in);
    if (act == 0) return;
    const int first = __ffs(act) - 1;
    const u32 d0 = __shfl_sync(0xffffffffu, d, first);
    if (__all_sync(0xffffffffu, !in || d == d0)) {
        if (static_cast<int>(lane_id()) == first) atomicAdd(row + d0, __popc(act));
    } else if (in) {
        atomicAdd(row + d, 1u);
    }
}

// Flushes a block's shared histogram [passes][256] into the global one.
__device__ __forceinline__ void hist_flush(const u32* s_hist, u32* g_hist, int passes) {
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
        const u32 c = s_hist[i];
        if (c) atomicAdd(g_hist + i, c);
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(512)
hist_kernel(const KeyT* __restrict__ keys, u64 n, PassTable pt, u32* __restrict__ g_hist) {
    extern __shared__ u32 s_hist[];
    for (int i = threadIdx.x; i < pt.count * kRadix; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 rounds = (n + stride - 1) / stride;
    u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (u64 r = 0; r < rounds; ++r, i += stride) {
        const bool in = i < n;
        const KeyT k = in ? keys[i] : KeyT(0);
        for (int p = 0; p < pt.count; ++p)
            hist_add(s_hist + p * kRadix, key_digit(k, pt.shift[p], pt.mask(p)), in);
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, pt.count);
}

// ---- one digit pass -----------------------------------------------------------------

// Lanes of the warp holding the same digit.  Built from one ballot per digit bit: on
// sm_100a eight VOTE + LOP3 pairs sustain a far higher rate than one MATCH.ANY, whose issue
// rate (not latency) capped the ranking loop at ~1.5 TB/s of key traffic (ncu: the BREV
// consuming the match result held 38 % of the stall samples, profiles/r1_onesweep_match.txt).
__device__ __forceinline__ unsigned warp_match_digit(u32 d, u32 mask) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
        if ((mask >> b) & 1u) {  // warp-uniform: the last pass of a key may be narrower
            const unsigned vote = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? vote : ~vote;
        }
    }
    return peers;
}

template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS>
struct OnesweepCfg {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * ITEMS;
    static constexpr size_t kSmem = sizeof(KeyT) * kTile + (HAS_VAL ? sizeof(u32) * kTile : 0) +
                                    sizeof(u32) * (kWarps * kRadix + 2 * kRadix + 32 + 4);
};

// IOTA_VAL: the payload of element i is i itself (no payload array is read).
template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS, bool IOTA_VAL = false>
__global__ void __launch_bounds__(BLOCK)
onesweep_kernel(const KeyT* __restrict__ keys_in, KeyT* __restrict__ keys_out,
                const u32* __restrict__ vals_in, u32* __restrict__ vals_out, u64 n, int shift,
                u32 mask, const u32* __restrict__ digit_base, u64* __restrict__ lookback,
                u32* __restrict__ ticket) {
    static_assert(BLOCK >= kRadix && BLOCK % 32 == 0, "one thread per digit is assumed");
    using Cfg = OnesweepCfg<KeyT, HAS_VAL, BLOCK, ITEMS>;
    constexpr int WARPS = Cfg::kWarps;
    constexpr int TILE = Cfg::kTile;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    KeyT* s_keys = reinterpret_cast<KeyT*>(smem_raw);
    u32* s_vals = reinterpret_cast<u32*>(s_keys + TILE);
    u32* s_whist = s_vals + (HAS_VAL ? TILE : 0);  // [WARPS][256] counts -> warp offsets
    u32* s_binstart = s_whist + WARPS * kRadix;    // [256] first tile slot of each digit
    u32* s_gofs = s_binstart + kRadix;             // [256] global index of slot 0 of digit
    u32* s_scan = s_gofs + kRadix;                 // [32] warp totals for the digit scan
    u32* s_tile = s_scan + 32;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const unsigned lane = lane_id();

    if (tid == 0) *s_tile = atomicAdd(ticket, 1u);
    for (int i = tid; i < WARPS * kRadix; i += BLOCK) s_whist[i] = 0;
    __syncthreads();
    const u32 tile = *s_tile;
    const u64 tile_base = static_cast<u64>(tile) * TILE;
    const u32 valid = static_cast<u32>(n - tile_base < static_cast<u64>(TILE) ? n - tile_base : TILE);

    // -- load: warp-striped, so that (warp, step, lane) order == memory order ---------
    KeyT key[ITEMS];
    u32 val[ITEMS];
    const u32 wbase = warp * (ITEMS * 32) + lane;
    if (valid == TILE) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) key[j] = keys_in[tile_base + wbase + j * 32];
        if (HAS_VAL) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j)
                val[j] = IOTA_VAL ? static_cast<u32>(tile_base + wbase + j * 32) : vals_in[tile_base + wbase + j * 32];
        }
    } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const u32 li = wbase + j * 32;
            key[j] = li < valid ? keys_in[tile_base + li] : ~KeyT(0);  // pads rank last
            if (HAS_VAL) val[j] = li < valid ? (IOTA_VAL ? static_cast<u32>(tile_base + li) : vals_in[tile_base + li]) : 0u;
        }
    }

    // -- rank inside the warp: match.any groups equal digits; the lowest lane of each group
    //    bumps the warp's private counter once for the whole group.  The bump is a shared
    //    atomicAdd whose old value is consumed only after a batch of them has been issued:
    //    successive steps of one warp are then independent instructions in flight instead of
    //    a load -> add -> store chain that exposes the shared-memory latency 16 times. --------
    u32* wh = s_whist + warp * kRadix;
    unsigned short rnk[ITEMS];
    const unsigned lt = lanemask_lt();
    constexpr int kBatch = ITEMS % 8 == 0 ? 8 : (ITEMS % 4 == 0 ? 4 : 1);
#pragma unroll
    for (int j0 = 0; j0 < ITEMS; j0 += kBatch) {
        unsigned peers[kBatch];
        u32 base[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
            peers[b] = warp_match_digit(key_digit(key[j0 + b], shift, mask), mask);
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            base[b] = 0;
            if ((peers[b] & lt) == 0)  // lowest lane of its group
                base[b] = atomicAdd(wh + key_digit(key[j0 + b], shift, mask), __popc(peers[b]));
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const u32 first = __shfl_sync(0xffffffffu, base[b], __ffs(peers[b]) - 1);
            rnk[j0 + b] = static_cast<unsigned short>(first + __popc(peers[b] & lt));
        }
    }
    __syncthreads();

    // -- per digit: offsets of each warp inside the digit's run, tile total -----------
    u32 total = 0;
    if (tid < kRadix) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            const u32 c = s_whist[w * kRadix + tid];
            s_whist[w * kRadix + tid] = total;
            total += c;
        }
        if (tile > 0) st_relaxed_u64(lookback + static_cast<u64>(tile) * kRadix + tid, kDescAggregate | total);
    }

    // -- exclusive scan of the 256 totals -> first slot of every digit in the tile ----
    u32 inc = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane) >= o) inc += t;
    }
    if (lane == 31) s_scan[warp] = inc;
    __syncthreads();
    if (tid < kRadix) {
        u32 add = 0;
        for (int w = 0; w < warp; ++w) add += s_scan[w];
        const u32 bin_start = add + inc - total;
        s_binstart[tid] = bin_start;

        // -- decoupled look-back over earlier tiles for this digit ---------------------
        u32 excl = 0;
        if (tile > 0) {
            long long t = static_cast<long long>(tile) - 1;
            for (;;) {
                const u64 v = ld_relaxed_u64(lookback + static_cast<u64>(t) * kRadix + tid);
                if ((v >> 62) == 0) continue;  // predecessor has not published yet
                excl += static_cast<u32>(v);
                if (v & kDescInclusive) break;
                --t;
            }
        }
        st_relaxed_u64(lookback + static_cast<u64>(tile) * kRadix + tid, kDescInclusive | (excl + total));
        s_gofs[tid] = digit_base[tid] + excl - bin_start;
    }
    __syncthreads();

    // -- exchange through shared memory: the tile becomes digit-sorted ----------------
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const u32 d = key_digit(key[j], shift, mask);
        const u32 pos = s_binstart[d] + wh[d] + rnk[j];
        s_keys[pos] = key[j];
        if (HAS_VAL) s_vals[pos] = val[j];
    }
    __syncthreads();

    // -- coalesced scatter: consecutive slots of one digit go to consecutive addresses -
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const u32 i = tid + j * BLOCK;
        if (i < valid) {
            const KeyT k = s_keys[i];
            const u32 dst = s_gofs[key_digit(k, shift, mask)] + i;
            keys_out[dst] = k;
            if (HAS_VAL) vals_out[dst] = s_vals[i];
        }
    }
}

// ---- host driver ----------------------------------------------------------------------

struct SortWorkspace {
    u32* hist = nullptr;      // [kMaxPasses][256]
    u32* base = nullptr;      // [kMaxPasses][256]
    u32* tickets = nullptr;   // [kMaxPasses]
    u64* lookback = nullptr;  // [tiles][256]
    size_t lookback_bytes = 0;
};

template <typename KeyT, bool HAS_VAL>
struct SortTuning;  // BLOCK / ITEMS per key type, see radix.cu

size_t sort_workspace_bytes(size_t n);
int sort_workspace_carve(reseq_cuda_ctx* ctx, size_t n, SortWorkspace* ws);

// Sorts (keys, vals) by the digit passes in `pt`, ping-ponging between the a and b
// buffers.  If `hist_ready` the caller has already accumulated ws.hist for exactly these
// passes (fused into its key-producing kernel); otherwise a histogram kernel runs first.
// `skip_mask` bit p set => pass p is skipped (its digit is constant).  On return
// *in_b says which buffer holds the result.
template <typename KeyT>
int onesweep_sort(reseq_cuda_ctx* ctx, KeyT* keys_a, KeyT* keys_b, u32* vals_a, u32* vals_b,
                  size_t n, const PassTable& pt, const SortWorkspace& ws, bool hist_ready,
                  u32 skip_mask, bool* in_b);

// One stable partition pass of (keys[i], i) on key bits [shift, shift + bits): keys_out /
// idx_out receive the pairs grouped by digit.  ws.hist[0..255] must hold the digit counts.
int onesweep_partition_iota(reseq_cuda_ctx* ctx, const u32* keys, u32* keys_out, u32* idx_out, size_t n,
                            int shift, int bits, const SortWorkspace& ws);
// The same for explicit (key, payload) pairs.
int onesweep_partition_pairs(reseq_cuda_ctx* ctx, const u32* keys, const u32* vals, u32* keys_out, u32* vals_out,
                             size_t n, int shift, int bits, const SortWorkspace& ws);

}  // namespace rsq
