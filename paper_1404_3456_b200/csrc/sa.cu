// Suffix-array construction on sm_100a: 2-bit packing, k-mer initial ranking, prefix
// doubling over (rank[i], rank[i+h]) pairs.
//
// Replaces build_parallel, suffix_array.hpp:61-124.  Same mathematical result -- the
// unique permutation sorted by suffix_less (suffix_array.hpp:28-41) and its inverse --
// reached with far fewer, far fatter phases:
//
//   reference                                   here
//   ---------------------------------------     ------------------------------------------
//   1-byte initial ranks (:68-87)               13-base (DNA, 2-bit packed) or 3-byte
//                                               (generic) sentinel-aware initial ranks:
//                                               one 31-bit key per suffix, 4 digit passes
//   h = 1, 2, 4, ... (:90)                      h = 13, 26, 52, ... (3 rounds at L=100,
//                                               4 at L=150 instead of 7 / 8)
//   two 32-pass 1-bit radix sorts per round     one LSD sort of the packed
//   (:97,:99)                                   (rank[i] << b | rank[i+h]+1) key,
//                                               ceil(2b/8) onesweep digit passes
//   diff by 4 rank gathers (:101-111)           adjacent compare of the sorted keys
//   dense ranks by exclusive_scan (:112-113)    group-head ranks (index of the first
//                                               suffix of the group) by a max-scan with
//                                               decoupled look-back, scatter fused
//   inverse permutation phase (:118-122)        free: with all groups singletons the
//                                               group-head rank array IS the inverse
//
// Sentinel semantics (suffix_array.hpp:16-20): every byte 0 is its own symbol, ordered
// by text position, below every other byte; end of text is below everything.  A suffix
// whose first k symbols contain a terminator is therefore already unique after the
// initial sort: its key is (symbols before the terminator, zero padded | 2*len + kind)
// where kind 0 = end of text, 1 = sentinel, and equal keys keep position order because
// the sort is stable and starts from the identity permutation.
#include "radix.cuh"
#include "sa.cuh"
#include "scan.cuh"

#include <type_traits>

namespace rsq {

namespace {

// ---- 2-bit packing ----------------------------------------------------------------
// packed: u64 words, 32 bases each, base p in bits [63-2(p%32)-1, 63-2(p%32)] so that a
// window's integer order equals its lexicographic order.  sent: u64 words, 64 flags
// each, position p at bit 63-(p%64).  Both arrays carry >= 2 zero words of padding.

__device__ __forceinline__ u32 dna_code(u32 c) { return ((c >> 1) ^ (c >> 2)) & 3u; }
__device__ __forceinline__ bool is_dna_or_zero(u32 c) {
    return c == 0u || c == 'A' || c == 'C' || c == 'G' || c == 'T';
}

template <bool VEC>
__global__ void __launch_bounds__(256)
pack_dna_kernel(const u8* __restrict__ text, u64 n, u64* __restrict__ packed,
                u64* __restrict__ sent, u32* __restrict__ bad_flag) {
    const u64 words = (n + 63) >> 6;  // one thread per 64 positions
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    bool bad = false;
    u32 n_sent = 0;
    for (u64 w = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) {
        const u64 base = w << 6;
        u64 p0 = 0, p1 = 0, s = 0;
        if (VEC && base + 64 <= n) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = ld_stream_v4(text + base + 16 * q);
                const u32 word[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const u32 c = (word[t >> 2] >> (8 * (t & 3))) & 0xFFu;
                    bad |= !is_dna_or_zero(c);
                    const int p = 16 * q + t;
                    const u64 code = dna_code(c) & (c ? 3u : 0u);
                    if (p < 32) p0 |= code << (62 - 2 * p);
                    else p1 |= code << (62 - 2 * (p - 32));
                    s |= static_cast<u64>(c == 0u) << (63 - p);
                }
            }
        } else {
            for (int p = 0; p < 64; ++p) {
                if (base + p >= n) break;
                const u32 c = text[base + p];
                bad |= !is_dna_or_zero(c);
                const u64 code = dna_code(c) & (c ? 3u : 0u);
                if (p < 32) p0 |= code << (62 - 2 * p);
                else p1 |= code << (62 - 2 * (p - 32));
                s |= static_cast<u64>(c == 0u) << (63 - p);
            }
        }
        packed[2 * w] = p0;
        packed[2 * w + 1] = p1;
        sent[w] = s;
        n_sent += __popcll(s);
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(bad_flag, 1u);
    for (int o = 16; o > 0; o >>= 1) n_sent += __shfl_xor_sync(0xffffffffu, n_sent, o);
    if (lane_id() == 0 && n_sent) atomicAdd(bad_flag + 1, n_sent);  // number of separator bytes
}

__device__ __forceinline__ u64 base_window(const u64* __restrict__ packed, u64 pos) {
    const u64 w = pos >> 5;
    const unsigned s = static_cast<unsigned>(pos & 31) * 2;
    const u64 hi = packed[w], lo = packed[w + 1];
    return s ? (hi << s) | (lo >> (64 - s)) : hi;
}
__device__ __forceinline__ u64 sent_window(const u64* __restrict__ sent, u64 pos) {
    const u64 w = pos >> 6;
    const unsigned s = static_cast<unsigned>(pos & 63);
    const u64 hi = sent[w], lo = sent[w + 1];
    return s ? (hi << s) | (lo >> (64 - s)) : hi;
}

// ---- initial keys --------------------------------------------------------------------

constexpr int kDnaK = 13;       // bases per initial key: 26 bits + 5-bit terminator field
constexpr int kDnaFieldBits = 5;
constexpr int kByteK = 3;       // bytes per initial key: 24 bits + 3-bit terminator field
constexpr int kByteFieldBits = 3;

// Keys of the `count` suffixes starting at text position pos0 (the whole text: pos0 = 0,
// count = n; a multi-GPU rank keys only its slice).  keys[i] / vals[i] belong to pos0 + i.
__global__ void __launch_bounds__(256)
initkey_dna_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n, u64 pos0, u64 count,
                   u32* __restrict__ keys, u32* __restrict__ vals, PassTable pt,
                   u32* __restrict__ g_hist) {
    extern __shared__ u32 s_hist[];
    for (int i = threadIdx.x; i < pt.count * kRadix; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 rounds = (count + stride - 1) / stride;
    u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (u64 r = 0; r < rounds; ++r, idx += stride) {
        const bool in = idx < count;
        const u64 pos = pos0 + idx;
        u32 key = 0;
        if (in) {
            const u32 bases = static_cast<u32>(base_window(packed, pos) >> (64 - 2 * kDnaK));
            const u32 sw = static_cast<u32>(sent_window(sent, pos) >> (64 - kDnaK));
            const u32 t = sw ? static_cast<u32>(__clz(sw)) - (32 - kDnaK) : kDnaK;
            const u64 rem = n - pos;
            const u32 lim = rem < kDnaK ? static_cast<u32>(rem) : kDnaK;
            u32 len, field;
            if (t < lim) { len = t; field = 2 * t + 1; }          // sentinel after `t` bases
            else if (lim < kDnaK) { len = lim; field = 2 * lim; } // text ends after `lim`
            else { len = kDnaK; field = 2 * kDnaK; }              // k full bases
            const u32 kept = bases & ~((1u << (2 * (kDnaK - len))) - 1u);
            key = (kept << kDnaFieldBits) | field;
            keys[idx] = key;
            vals[idx] = static_cast<u32>(pos);
        }
        for (int p = 0; p < pt.count; ++p)
            hist_add(s_hist + p * kRadix, key_digit(key, pt.shift[p], pt.mask(p)), in);
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, pt.count);
}

__global__ void __launch_bounds__(256)
initkey_bytes_kernel(const u8* __restrict__ text, u64 n, u32* __restrict__ keys,
                     u32* __restrict__ vals, PassTable pt, u32* __restrict__ g_hist) {
    extern __shared__ u32 s_hist[];
    for (int i = threadIdx.x; i < pt.count * kRadix; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 rounds = (n + stride - 1) / stride;
    u64 pos = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (u64 r = 0; r < rounds; ++r, pos += stride) {
        const bool in = pos < n;
        u32 key = 0;
        if (in) {
            u32 sym = 0, len = 0, field = 2 * kByteK;
            for (int t = 0; t < kByteK; ++t) {
                if (pos + t >= n) { field = 2 * len; break; }
                const u32 c = text[pos + t];
                if (c == 0u) { field = 2 * len + 1; break; }
                sym |= c << (8 * (kByteK - 1 - t));
                ++len;
            }
            key = (sym << kByteFieldBits) | field;
            keys[pos] = key;
            vals[pos] = static_cast<u32>(pos);
        }
        for (int p = 0; p < pt.count; ++p)
            hist_add(s_hist + p * kRadix, key_digit(key, pt.shift[p], pt.mask(p)), in);
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, pt.count);
}

// ---- re-ranking ------------------------------------------------------------------------
// After a sort, suffix sa[idx] starts a new group iff its key differs from its left
// neighbour's (or, for initial keys, carries a terminator: those are unique by
// construction).  rank = index of the group's first suffix ("group-head rank"): an
// inclusive max-scan of (head ? idx+1 : 0).  A tile containing any head needs no
// look-back (heads increase with idx), so the chain is only walked inside groups that
// span whole tiles.

constexpr int kRankBlock = 256;
constexpr int kRankItems = 8;
constexpr int kRankTile = kRankBlock * kRankItems;

template <typename KeyT, bool FLAGS_ONLY>
__global__ void __launch_bounds__(kRankBlock)
rerank_kernel(const KeyT* __restrict__ keys, const u32* __restrict__ sa, u64 n, u32 uniq_mask,
              u32 uniq_full, u32* __restrict__ rank, u32* __restrict__ head_of,
              u64* __restrict__ desc, u32* __restrict__ ticket, u32* __restrict__ num_heads) {
    __shared__ u32 s_tile;
    __shared__ u32 s_warp[kRankBlock / 32];
    __shared__ u32 s_count[kRankBlock / 32];
    __shared__ u32 s_prefix;
    __shared__ KeyT s_last[kRankBlock];

    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const u64 base = static_cast<u64>(tile) * kRankTile + static_cast<u64>(tid) * kRankItems;

    KeyT k[kRankItems];
#pragma unroll
    for (int j = 0; j < kRankItems; ++j) k[j] = base + j < n ? keys[base + j] : KeyT(0);
    s_last[tid] = k[kRankItems - 1];
    __syncthreads();
    KeyT prev;
    if (tid > 0) prev = s_last[tid - 1];
    else prev = base > 0 && base <= n ? keys[base - 1] : KeyT(0);

    u32 m[kRankItems];
    u32 run = 0, heads = 0;
#pragma unroll
    for (int j = 0; j < kRankItems; ++j) {
        const u64 idx = base + j;
        // FLAGS_ONLY: the "keys" are 0/1 head flags expanded from a head bitmap
        const bool head = idx < n && (FLAGS_ONLY ? (idx == 0 || k[j] != KeyT(0))
                                                 : (idx == 0 || k[j] != prev ||
                                                    (static_cast<u32>(k[j]) & uniq_mask) != uniq_full));
        prev = k[j];
        heads += head;
        if (head) run = static_cast<u32>(idx) + 1u;
        m[j] = run;  // thread-local inclusive max (0 = no head yet in this thread)
    }
    u32 inc = run;
    u32 hsum = heads;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane) >= o) inc = max(inc, t);
        hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
    }
    u32 before = __shfl_up_sync(0xffffffffu, inc, 1);  // max over earlier lanes
    if (lane == 0) before = 0;
    if (lane == 31) s_warp[warp] = inc;
    if (lane == 0) s_count[warp] = hsum;
    __syncthreads();
    u32 wmax = 0, tile_max = 0, tile_heads = 0;
#pragma unroll
    for (int w = 0; w < kRankBlock / 32; ++w) {
        if (w < warp) wmax = max(wmax, s_warp[w]);
        tile_max = max(tile_max, s_warp[w]);
        tile_heads += s_count[w];
    }
    if (tid == 0) {
        u32 excl = 0;
        if (tile_max != 0 || tile == 0) {
            st_relaxed_u64(desc + tile, kDescInclusive | tile_max);
        } else {
            st_relaxed_u64(desc + tile, kDescAggregate | 0u);
            long long t = static_cast<long long>(tile) - 1;
            for (;;) {
                const u64 d = ld_relaxed_u64(desc + t);
                if ((d >> 62) == 0) continue;
                excl = max(excl, static_cast<u32>(d));
                if (d & kDescInclusive) break;
                --t;
            }
            st_relaxed_u64(desc + tile, kDescInclusive | excl);
        }
        // tiles with a head never read s_prefix for elements after it; elements before the
        // first head of the tile need the previous tiles' maximum:
        if (tile_max != 0 && tile > 0) {
            long long t = static_cast<long long>(tile) - 1;
            for (;;) {
                const u64 d = ld_relaxed_u64(desc + t);
                if ((d >> 62) == 0) continue;
                excl = max(excl, static_cast<u32>(d));
                if (d & kDescInclusive) break;
                --t;
            }
        }
        s_prefix = excl;
        if (tile_heads) atomicAdd(num_heads, tile_heads);
    }
    __syncthreads();
    const u32 carry = max(max(s_prefix, wmax), before);
#pragma unroll
    for (int j = 0; j < kRankItems; ++j) {
        const u64 idx = base + j;
        if (idx < n) {
            const u32 h = max(m[j], carry) - 1u;
            head_of[idx] = h;
            rank[sa[idx]] = h;
        }
    }
}

// ---- group refinement from L2-resident text windows ----------------------------------
//
// After the initial sort the suffixes are grouped by their first `depth` symbols; groups
// are contiguous in sa and delimited by a head bitmap (bit idx set <=> sa[idx] starts a
// group).  On B200 the 2-bit packed text (n/4 bytes: 35 MB at 4.6 Mbp x 30) fits the 126 MB
// L2 while the 4n-byte rank array does not, so the next 29 symbols of every still-tied
// suffix are fetched straight from the packed text (an L2 hit) instead of through
// rank[pos + h] (a DRAM sector per suffix, plus a DRAM read-modify-write per suffix to
// scatter the new ranks).  Each CTA owns the groups that START inside its 2048-suffix tile,
// stages them in shared memory, ranks every tied suffix inside its group by enumeration
// (groups of a shotgun read set hold ~coverage suffixes), writes the refined order back in
// place and ORs the new group heads into the next bitmap.  No global sort, no rank array.
//
// A group that does not fit the CTA's shared-memory window (more than kRefExt suffixes past
// the tile) is left untouched and reported; the host then switches to the general
// prefix-doubling rounds below, which have no size limit.

constexpr int kRefBlock = 256;
constexpr int kRefTile = 2048;
constexpr int kRefExt = 1024;
constexpr int kRefCap = kRefTile + kRefExt;
constexpr int kRefWords = kRefCap / 32 + 2;
constexpr size_t kRefSmem = sizeof(u64) * kRefCap + sizeof(u32) * kRefCap + 3 * sizeof(unsigned short) * kRefCap +
                            sizeof(u32) * (4 * kRefWords + 16);
constexpr int kTextK = 23;          // bases per refinement round
constexpr int kTextFieldBits = 6;   // terminator field: 2*len + kind, 2*kTextK = "no terminator"
constexpr u32 kDistCap = 4095;      // farthest sentinel the distance shortcut looks for
constexpr int kTextSlotBits = 12;   // window slot of the suffix: makes every key of a round unique
static_assert(kRefCap <= (1 << kTextSlotBits), "window slots must fit the key's slot field");
static_assert(2 * kTextK + kTextFieldBits + kTextSlotBits == 64, "refinement key layout");

// Key of one round for the suffix in window slot `slot`: the next 23 symbols from `pos`
// (zero padded at a terminator) | terminator field | slot.  Keys of equal content keep
// their slot order, so the order of the full 64-bit keys IS the stable refined order.
__device__ __forceinline__ u64 text_key(const u64* __restrict__ packed, const u64* __restrict__ sent,
                                        u64 n, u64 pos, u32 slot) {
    if (pos >= n) return slot;  // the text ends exactly here: end-of-text after 0 symbols
    const u64 bases = base_window(packed, pos) >> (64 - 2 * kTextK);
    const u32 sw = static_cast<u32>(sent_window(sent, pos) >> (64 - kTextK));
    const u32 t = sw ? static_cast<u32>(__clz(sw)) - (32 - kTextK) : kTextK;
    const u64 rem = n - pos;
    const u32 lim = rem < kTextK ? static_cast<u32>(rem) : kTextK;
    u32 len, field;
    if (t < lim) { len = t; field = 2 * t + 1; }
    else if (lim < kTextK) { len = lim; field = 2 * lim; }
    else { len = kTextK; field = 2 * kTextK; }
    const u64 kept = len == kTextK ? bases : bases & ~((1ull << (2 * (kTextK - len))) - 1ull);
    return (((kept << kTextFieldBits) | field) << kTextSlotBits) | slot;
}

// Head bitmap from the sorted initial keys: a suffix starts a group iff its key differs
// from its left neighbour's or carries a terminator (unique by construction).
__global__ void __launch_bounds__(256)
headbits_kernel(const u32* __restrict__ keys, u64 n, u32 uniq_mask, u32 uniq_full,
                u32* __restrict__ bits, u32* __restrict__ counters) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 rounds = (n + stride - 1) / stride;
    u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    u32 nonheads = 0;
    for (u64 r = 0; r < rounds; ++r, idx += stride) {
        const bool in = idx < n;
        bool head = false;
        if (in) {
            const u32 k = keys[idx];
            head = idx == 0 || k != keys[idx - 1] || (k & uniq_mask) != uniq_full;
        }
        const unsigned b = __ballot_sync(0xffffffffu, head);
        const unsigned act = __ballot_sync(0xffffffffu, in);
        if (lane_id() == 0 && act) {
            bits[idx >> 5] = b;
            nonheads += __popc(act & ~b);
        }
    }
    if (nonheads) atomicAdd(counters, nonheads);
}

// One CTA refines every group that starts in its tile to completion: the key of a tied
// suffix depends only on (position, depth), never on another group, so all rounds run
// back to back in shared memory and the tile goes back to HBM once.  Every round first
// compacts the still-tied suffixes into a dense list (order preserving, so a group stays
// contiguous) -- late rounds, where few suffixes are tied, then cost in proportion to what
// is left instead of dragging 32-wide warps through one or two live lanes.
__global__ void __launch_bounds__(kRefBlock)
refine_text_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n_text,
                   u32* __restrict__ sa, u64 n, const u32* __restrict__ bits_old, u32* __restrict__ bits_new,
                   u32 depth, int max_rounds, bool use_shortcut, u32* __restrict__ counters) {
    // n_text: length of the text the positions refer to; n: number of suffixes in sa (equal for
    // a whole-text build, a bucket of it for a multi-GPU rank)
    extern __shared__ __align__(16) unsigned char ref_smem[];
    u64* s_key = reinterpret_cast<u64*>(ref_smem);               // [cap] keys of the round ...
    u32* s_pos2 = reinterpret_cast<u32*>(ref_smem);              // ... then the permuted positions
    u32* s_pos = reinterpret_cast<u32*>(s_key + kRefCap);        // [cap] suffix positions, sa order
    unsigned short* s_list = reinterpret_cast<unsigned short*>(s_pos + kRefCap);  // [cap] tied slots
    unsigned short* s_dst = s_list + kRefCap;                    // [cap] new slot of list entry u
    unsigned short* s_src = s_dst + kRefCap;                     // [cap] old slot of new slot d
    u32* s_bits = reinterpret_cast<u32*>(s_src + kRefCap);       // [words] head bits of the window
    u32* s_new = s_bits + kRefWords;                             // [words] heads created this round
    u32* s_fail = s_new + kRefWords;                             // [words] groups the shortcut gave up on
    u32* s_cnt = s_fail + kRefWords;                             // [words + 1] tied-count scan
    __shared__ int s_first, s_end, s_last;

    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const u64 t0 = static_cast<u64>(blockIdx.x) * kRefTile;
    const u64 w0 = t0 >> 5;
    const int lim = static_cast<int>(n - t0 < static_cast<u64>(kRefTile) ? n - t0 : kRefTile);
    const u64 total_words = (n + 31) >> 5;

    if (tid == 0) { s_first = 0x7fffffff; s_end = 0x7fffffff; s_last = -1; }
    for (int j = tid; j < kRefWords; j += kRefBlock) {
        s_bits[j] = w0 + j < total_words ? bits_old[w0 + j] : 0u;
        s_new[j] = 0;
    }
    __syncthreads();
    // position n acts as a head so that the last group has an end
    if (tid == 0 && n - t0 < static_cast<u64>(kRefWords) * 32) s_bits[(n - t0) >> 5] |= 1u << ((n - t0) & 31);
    __syncthreads();

    // first / last head inside the tile, first head at or after its end
    for (int j = tid; j < kRefWords; j += kRefBlock) {
        const u32 w = s_bits[j];
        if (!w) continue;
        const int base = j * 32;
        const u32 lo_mask = base + 32 <= lim ? 0xffffffffu : (base >= lim ? 0u : ((1u << (lim - base)) - 1u));
        const u32 lo = w & lo_mask, hi = w & ~lo_mask;
        if (lo) {
            atomicMin(&s_first, base + __ffs(lo) - 1);
            atomicMax(&s_last, base + 31 - __clz(lo));
        }
        if (hi) atomicMin(&s_end, base + __ffs(hi) - 1);
    }
    __syncthreads();
    const int first = s_first;
    if (first == 0x7fffffff) return;  // no group starts in this tile
    int end = s_end;
    if (end > kRefCap) {              // the tile's last group overruns the window
        if (tid == 0) atomicOr(counters + 1, 1u);
        end = s_last;                 // leave that group alone
    }
    if (end - first <= 1) return;

    // Tied slots of window word j, restricted to [first, end): slot a is tied unless it is a
    // head whose successor is a head too.
    auto tied_word = [&](int j) -> u32 {
        const int base = j * 32;
        if (base + 32 <= first || base >= end) return 0u;
        const u32 w = s_bits[j];
        const u32 next = (w >> 1) | (s_bits[j + 1] << 31);
        u32 t = ~(w & next);
        if (base < first) t &= 0xffffffffu << (first - base);
        if (base + 32 > end) t &= (1u << (end - base)) - 1u;
        return t;
    };

    constexpr u32 kFieldMask = (1u << kTextFieldBits) - 1u;
    constexpr u32 kFull = 2 * kTextK;
    constexpr u32 kNoDist = kDistCap + 1;  // "no sentinel within reach": the shortcut does not apply

    // group start of window slot a: the last head at or before it
    auto group_start = [&](int a) {
        int w = a >> 5;
        u32 word = s_bits[w] & (0xffffffffu >> (31 - (a & 31)));
        while (!word) word = s_bits[--w];
        return w * 32 + 31 - __clz(word);
    };
    auto group_end = [&](int a) {  // the first head after it
        int w = (a + 1) >> 5;
        u32 word = s_bits[w] & (0xffffffffu << ((a + 1) & 31));
        while (!word) word = s_bits[++w];
        return w * 32 + __ffs(word) - 1;
    };

    bool loaded = false;
    int rounds = 0;
    // Steps alternate: a SHORTCUT step (below) on everything tied, then a TEXT step (the next
    // 23 symbols) on what the shortcut could not settle.
    for (int step = 0;; ++step) {
        const bool shortcut = use_shortcut && (step & 1) == 0;
        if (!shortcut && rounds >= max_rounds) break;
        if (!use_shortcut && (step & 1) == 0) continue;

        // -- compact the tied slots, in order ------------------------------------------------
        u32 tw = 0, c = 0;
        if (tid < kRefWords) {
            tw = tied_word(tid);
            c = __popc(tw);
            s_fail[tid] = 0;
        }
        u32 inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
            if (static_cast<int>(lane) >= o) inc += t;
        }
        if (lane == 31) s_cnt[kRefWords + 1 + (tid >> 5)] = inc;   // warp totals
        __syncthreads();
        u32 before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kRefBlock / 32; ++w) {
            const u32 v = s_cnt[kRefWords + 1 + w];
            if (w < (tid >> 5)) before += v;
            total += v;
        }
        if (total == 0) break;
        if (tid < kRefWords) {
            u32 at = before + inc - c;
            while (tw) {
                const int b = __ffs(tw) - 1;
                tw &= tw - 1;
                s_list[at++] = static_cast<unsigned short>(tid * 32 + b);
            }
        }
        if (!loaded) {
            for (int a = first + tid; a < end; a += kRefBlock) s_pos[a] = sa[t0 + a];
            loaded = true;
        }
        __syncthreads();
        const int cnt = static_cast<int>(total);

        // -- keys.  TEXT: the next 23 symbols (an L2 hit).  SHORTCUT: the distance from the
        //    current depth to the suffix's sentinel.  In a read set the members of a group are
        //    reads over one locus: each is a prefix of the longer ones, so their order is
        //    (distance, position) -- provided that really holds, which the verify pass below
        //    checks base by base on neighbours in the new order (prefix-of is transitive along
        //    the sorted chain).  A verified group is completely ordered in ONE step instead of
        //    ceil(length / 23). ----------------------------------------------------------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            const u64 q = static_cast<u64>(s_pos[a]) + depth;
            if (shortcut) {
                u32 dist = kNoDist;
                for (u32 c0 = 0; c0 <= kDistCap && q + c0 < n_text; c0 += 64) {
                    const u64 w = sent_window(sent, q + c0);
                    if (w) {
                        dist = c0 + static_cast<u32>(__clzll(w));
                        break;
                    }
                }
                if (dist > kDistCap || q + dist >= n_text) dist = kNoDist;
                s_key[a] = (static_cast<u64>(dist) << kTextSlotBits) | static_cast<u32>(a);
            } else {
                s_key[a] = text_key(packed, sent, n_text, q, static_cast<u32>(a));
            }
        }
        __syncthreads();

        // -- rank inside the group: the keys are unique, so rank = #smaller keys -----------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            const int gs = group_start(a), ge = group_end(a);
            const u64 ki = s_key[a];
            u32 r0 = 0, r1 = 0;
            int j = gs;
            for (; j + 1 < ge; j += 2) {   // every member of the group runs the same trip count
                r0 += s_key[j] < ki;
                r1 += s_key[j + 1] < ki;
            }
            if (j < ge) r0 += s_key[j] < ki;
            const int dst = gs + static_cast<int>(r0 + r1);
            s_dst[u] = static_cast<unsigned short>(dst);
            s_src[dst] = static_cast<unsigned short>(a);
        }
        __syncthreads();

        // -- new heads -------------------------------------------------------------------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            const int dst = s_dst[u];
            const bool opens = (s_bits[dst >> 5] >> (dst & 31)) & 1u;  // slot dst starts the group
            if (shortcut) {
                // verify: this suffix must agree with the group's LONGEST member (last in the new
                // order) on all of its own `dist` symbols.  Then every member is a prefix of every
                // longer one, which is exactly what ordering by distance assumes.  The lanes of a
                // warp mostly work on one group, so the reference's words are one broadcast load.
                const u32 dist = static_cast<u32>(s_key[a] >> kTextSlotBits);
                bool ok = dist != kNoDist;
                const int ra = s_src[group_end(a) - 1];
                if (static_cast<u32>(s_key[ra] >> kTextSlotBits) == kNoDist) ok = false;  // no usable reference
                if (ok && ra != a) {
                    const u64 qa = static_cast<u64>(s_pos[a]) + depth, qr = static_cast<u64>(s_pos[ra]) + depth;
                    for (u32 c0 = 0; c0 < dist && ok; c0 += 32) {
                        const u32 len = dist - c0 < 32u ? dist - c0 : 32u;
                        ok = ((base_window(packed, qa + c0) ^ base_window(packed, qr + c0)) >> (64 - 2 * len)) == 0;
                    }
                }
                if (!ok) {
                    const int gs = group_start(a);
                    atomicOr(&s_fail[gs >> 5], 1u << (gs & 31));
                }
            } else {
                // a suffix starts a group iff its content differs from its predecessor's in the
                // new order, or it carries a terminator (unique by construction)
                const u64 ki = s_key[a] >> kTextSlotBits;
                bool head = (static_cast<u32>(ki) & kFieldMask) != kFull;
                if (!head && !opens) head = (s_key[s_src[dst - 1]] >> kTextSlotBits) != ki;
                if (head) atomicOr(&s_new[dst >> 5], 1u << (dst & 31));
            }
        }
        __syncthreads();

        // -- permute (the key buffer is dead: it receives the new order) -----------------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            int dst = s_dst[u];
            if (shortcut) {
                const int gs = group_start(a);
                if ((s_fail[gs >> 5] >> (gs & 31)) & 1u) {
                    s_dst[u] = 0xffff;  // group left as it was
                    continue;
                }
                atomicOr(&s_new[dst >> 5], 1u << (dst & 31));  // verified: every member is final
            }
            s_pos2[dst] = s_pos[a];
        }
        __syncthreads();
        for (int u = tid; u < cnt; u += kRefBlock) {
            if (s_dst[u] == 0xffff) continue;
            const int a = s_list[u];
            s_pos[a] = s_pos2[a];
        }
        if (tid < kRefWords) {
            s_bits[tid] |= s_new[tid];
            s_new[tid] = 0;
        }
        __syncthreads();
        if (!shortcut) {
            ++rounds;
            depth += kTextK;
        }
    }
    if (!loaded) return;  // nothing was tied in this tile

    // write the tile back once; publish the new heads; count what is still tied
    u32 nonheads = 0;
    for (int a = first + tid; a < end; a += kRefBlock) {
        sa[t0 + a] = s_pos[a];
        nonheads += !((s_bits[a >> 5] >> (a & 31)) & 1u);
    }
    const int n_local = n - t0 < static_cast<u64>(kRefWords) * 32 ? static_cast<int>(n - t0) : kRefWords * 32;
    for (int j = tid; j < kRefWords; j += kRefBlock) {
        const int base = j * 32;
        if (base >= n_local || base >= end) break;
        u32 w = s_bits[j];
        if (base + 32 > n_local) w &= (1u << (n_local - base)) - 1u;  // drop the artificial end bit
        if (base + 32 > end) w &= (1u << (end - base)) - 1u;
        if (w) atomicOr(bits_new + w0 + j, w);
    }
    for (int o = 16; o > 0; o >>= 1) nonheads += __shfl_xor_sync(0xffffffffu, nonheads, o);
    if (lane == 0 && nonheads) atomicAdd(counters, nonheads);
    if (tid == 0) atomicMax(counters + 2, static_cast<u32>(rounds));
}

// rank = inverse permutation of sa.  A direct scatter rank[sa[i]] = i is n random 4-byte
// writes, each a DRAM read-modify-write of a whole sector (measured 5.9 ms at n = 139 M).
// Instead the (sa[i], i) pairs are first partitioned by the top 8 bits of sa[i] -- one
// streaming onesweep pass -- so that consecutive pairs target one n/256-entry window of
// rank; the scatter then hits in L2 and DRAM only sees whole lines written once.
__global__ void perm_digit_hist_kernel(u64 n, int shift, int bits, u32* __restrict__ hist) {
    // sa is a permutation of [0, n): the number of values v with digit (v >> shift) & mask == d
    // is known in closed form -- count of such v below n
    const u64 d = threadIdx.x;
    const u64 period = 1ull << (shift + bits), span = 1ull << shift;
    if (d >= (1ull << bits)) { hist[d] = 0; return; }
    const u64 full = n / period, rem = n % period;
    const u64 lo = d * span;
    const u64 part = rem > lo ? (rem - lo < span ? rem - lo : span) : 0;
    hist[d] = static_cast<u32>(full * span + part);
}

__global__ void scatter_pairs_kernel(const u32* __restrict__ pos, const u32* __restrict__ idx, u64 n,
                                     u32* __restrict__ rank) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        rank[pos[i]] = idx[i];
}

// After the partition passes every aligned window of 2^win_bits rank entries has all of its
// (pos, idx) pairs in the same index range of the pair arrays (sa is a permutation, so the
// buckets are exactly window-sized).  One CTA per window: scatter in shared memory, store the
// window with full-width coalesced writes -- 139 M single-sector L2 write transactions become
// 4.3 M full lines.
__global__ void __launch_bounds__(512)
window_scatter_kernel(const u32* __restrict__ pos, const u32* __restrict__ idx, u64 n, int win_bits,
                      u32* __restrict__ rank) {
    extern __shared__ u32 s_win[];
    const u64 base = static_cast<u64>(blockIdx.x) << win_bits;
    const u32 size = static_cast<u32>(n - base < (1ull << win_bits) ? n - base : (1ull << win_bits));
    const u32 mask = (1u << win_bits) - 1u;
    for (u32 t = threadIdx.x; t < size; t += blockDim.x) s_win[pos[base + t] & mask] = idx[base + t];
    __syncthreads();
    for (u32 t = threadIdx.x; t < size; t += blockDim.x) rank[base + t] = s_win[t];
}

__global__ void inverse_kernel(const u32* __restrict__ sa, u64 n, u32* __restrict__ rank) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        rank[sa[i]] = static_cast<u32>(i);
}

__global__ void expand_bits_kernel(const u32* __restrict__ bits, u64 n, u32* __restrict__ flags) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        flags[i] = (bits[i >> 5] >> (i & 31)) & 1u;
}

// ---- doubling round: build the pair keys --------------------------------------------

__global__ void __launch_bounds__(256)
pair_key_kernel(const u32* __restrict__ sa, const u32* __restrict__ head_of,
                const u32* __restrict__ rank, u64 n, u64 h, int rank_bits,
                u64* __restrict__ keys, PassTable pt, u32* __restrict__ g_hist) {
    extern __shared__ u32 s_hist[];
    for (int i = threadIdx.x; i < pt.count * kRadix; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 rounds = (n + stride - 1) / stride;
    u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (u64 r = 0; r < rounds; ++r, idx += stride) {
        const bool in = idx < n;
        u64 key = 0;
        if (in) {
            const u64 p = static_cast<u64>(sa[idx]) + h;
            // suffix_array.hpp:93-96: rank of the suffix h further on, +1, 0 past the end
            const u64 k2 = p < n ? static_cast<u64>(rank[p]) + 1u : 0u;
            key = (static_cast<u64>(head_of[idx]) << rank_bits) | k2;
            keys[idx] = key;
        }
        for (int p = 0; p < pt.count; ++p)
            hist_add(s_hist + p * kRadix, key_digit(key, pt.shift[p], pt.mask(p)), in);
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, pt.count);
}

unsigned grid_for(const reseq_cuda_ctx* ctx, size_t n, int block, int per_thread, int waves) {
    size_t want = (n + static_cast<size_t>(block) * per_thread - 1) /
                  (static_cast<size_t>(block) * per_thread);
    const size_t cap = static_cast<size_t>(ctx->sm_count) * waves;
    if (want < 1) want = 1;
    return static_cast<unsigned>(want < cap ? want : cap);
}

}  // namespace

int pack_dna_device(reseq_cuda_ctx* ctx, const u8* d_text, size_t n, u64* packed, u64* sent,
                    u32* d_flag, bool* is_dna, u64* n_separators) {
    cudaStream_t s = ctx->stream;
    RSQ_CUDA(cudaMemsetAsync(d_flag, 0, 2 * sizeof(u32), s));
    RSQ_CUDA(cudaMemsetAsync(packed + (n / 64) * 2, 0,
                             sizeof(u64) * ((n / 32 + 8) - (n / 64) * 2), s));
    RSQ_CUDA(cudaMemsetAsync(sent + n / 64, 0, sizeof(u64) * ((n / 64 + 8) - n / 64), s));
    const unsigned grid = grid_for(ctx, (n + 63) / 64, 256, 1, 8);
    RSQ_LAUNCH_BEGIN(ctx, "pack_dna_kernel");
    if (reinterpret_cast<uintptr_t>(d_text) % 16 == 0)
        pack_dna_kernel<true><<<grid, 256, 0, s>>>(d_text, n, packed, sent, d_flag);
    else
        pack_dna_kernel<false><<<grid, 256, 0, s>>>(d_text, n, packed, sent, d_flag);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_flag, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    *is_dna = reinterpret_cast<volatile u32*>(ctx->pinned)[0] == 0;
    if (n_separators) *n_separators = reinterpret_cast<volatile u32*>(ctx->pinned)[1];
    return RESEQ_OK;
}

size_t sa_workspace_bytes(size_t n) {
    auto pad = reseq_cuda_ctx::padded;
    size_t total = 0;
    total += pad(sizeof(u64) * (n / 32 + 8));        // packed bases
    total += pad(sizeof(u64) * (n / 64 + 8));        // sentinel bitmap
    total += 2 * pad(sizeof(u64) * n);               // key buffers a / b
    total += 2 * pad(sizeof(u32) * n);               // payload buffer b, head_of
    total += pad(sizeof(u32) * n);                   // rank when the caller wants none
    total += pad(sizeof(u64) * (n / kRankTile + 4)); // rerank descriptors
    total += pad(1024);                              // counters
    total += 2 * pad(sizeof(u32) * (n / 32 + 8));    // head bitmaps
    total += sort_workspace_bytes(n);
    return total + 4096;
}

int build_sa_device(reseq_cuda_ctx* ctx, const u8* d_text, size_t n, u32* d_sa, u32* d_rank,
                    reseq_sa_stats* stats) {
    reseq_sa_stats st{};
    const uint64_t launches0 = ctx->launches;
    if (n > RESEQ_CUDA_MAX_TEXT)
        return fail(RESEQ_TEXT_TOO_LARGE, "text of length " + std::to_string(n) + " exceeds 2^32-2");
    if (n == 0) {
        if (stats) *stats = st;
        return RESEQ_OK;
    }
    cudaStream_t s = ctx->stream;

    u64* packed = ctx->alloc<u64>(n / 32 + 8);
    u64* sent = ctx->alloc<u64>(n / 64 + 8);
    u64* keys_a = ctx->alloc<u64>(n);
    u64* keys_b = ctx->alloc<u64>(n);
    u32* vals_b = ctx->alloc<u32>(n);
    u32* head_of = ctx->alloc<u32>(n);
    u32* rank = d_rank ? d_rank : ctx->alloc<u32>(n);
    const size_t rank_tiles = (n + kRankTile - 1) / kRankTile;
    u64* desc = ctx->alloc<u64>(rank_tiles + 4);
    u32* counters = ctx->alloc<u32>(256);  // [0] bad byte flag, [1] rerank ticket, [2] heads, [4..5] refine
    u32* bits_0 = ctx->alloc<u32>(n / 32 + 8);
    u32* bits_1 = ctx->alloc<u32>(n / 32 + 8);
    SortWorkspace ws;
    if (!packed || !sent || !keys_a || !keys_b || !vals_b || !head_of || !rank || !desc || !counters || !bits_0 || !bits_1)
        return fail(RESEQ_OUT_OF_MEMORY, "suffix-array workspace does not fit the reserved arena");
    RSQ_TRY(sort_workspace_carve(ctx, n, &ws));

    // -- pack, decide the alphabet ----------------------------------------------------
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 1024, s));
    bool dna = false;
    u64 n_separators = 0;
    RSQ_TRY(pack_dna_device(ctx, d_text, n, packed, sent, counters + 16, &dna, &n_separators));
    // The sentinel-distance shortcut pays off on read sets (a sentinel every <= 1024 symbols on
    // average); on sentinel-free texts every probe would scan to its cap for nothing.
    const bool use_shortcut = ctx->opt_shortcut != 0 && n_separators * 1024 >= n;
    st.alphabet = dna ? 0 : 1;

    // -- initial keys + their digit histograms, 32-bit LSD sort --------------------------
    u32* k32_a = reinterpret_cast<u32*>(keys_a);
    u32* k32_b = reinterpret_cast<u32*>(keys_b);
    const int key_bits = dna ? 2 * kDnaK + kDnaFieldBits : 8 * kByteK + kByteFieldBits;
    const PassTable pt0 = make_passes(0, key_bits);
    RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * pt0.count * kRadix, s));
    {
        const unsigned grid = grid_for(ctx, n, 256, 8, 8);
        const size_t smem = sizeof(u32) * pt0.count * kRadix;
        RSQ_LAUNCH_BEGIN(ctx, dna ? "initkey_dna_kernel" : "initkey_bytes_kernel");
        if (dna)
            initkey_dna_kernel<<<grid, 256, smem, s>>>(packed, sent, n, 0, n, k32_a, d_sa, pt0, ws.hist);
        else
            initkey_bytes_kernel<<<grid, 256, smem, s>>>(d_text, n, k32_a, d_sa, pt0, ws.hist);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
    }
    bool in_b = false;
    RSQ_TRY(onesweep_sort<u32>(ctx, k32_a, k32_b, d_sa, vals_b, n, pt0, ws, true, 0, &in_b));
    st.sort_passes += pt0.count;
    st.init_symbols = dna ? kDnaK : kByteK;
    u32* sa_cur = in_b ? vals_b : d_sa;
    u32* sa_alt = in_b ? d_sa : vals_b;

    auto rerank = [&](auto* keys, auto flags_only, u32 uniq_mask, u32 uniq_full) -> int {
        RSQ_CUDA(cudaMemsetAsync(desc, 0, sizeof(u64) * (rank_tiles + 4), s));
        RSQ_CUDA(cudaMemsetAsync(counters + 1, 0, 2 * sizeof(u32), s));
        using K = std::remove_pointer_t<decltype(keys)>;
        RSQ_LAUNCH_BEGIN(ctx, "rerank_kernel");
        rerank_kernel<K, decltype(flags_only)::value><<<static_cast<unsigned>(rank_tiles), kRankBlock, 0, s>>>(
            keys, sa_cur, n, uniq_mask, uniq_full, rank, head_of, desc, counters + 1, counters + 2);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters + 2, sizeof(u32), cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaStreamSynchronize(s));
        return RESEQ_OK;
    };

    const u32 field_mask = (1u << (dna ? kDnaFieldBits : kByteFieldBits)) - 1u;
    const u32 field_full = 2u * (dna ? kDnaK : kByteK);
    u64 heads = 0;
    u64 h = st.init_symbols;
    bool ranked = false;  // rank / head_of valid for the current order

    // -- DNA fast path: refine groups from L2-resident text windows -------------------------
    if (dna && ctx->opt_text_rounds > 0) {
        const size_t words = (n + 31) / 32 + 4;
        u32* bits_a = bits_0;
        u32* bits_b = bits_1;
        static bool configured = false;
        if (!configured) {
            RSQ_CUDA(cudaFuncSetAttribute(refine_text_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(kRefSmem)));
            configured = true;
        }
        RSQ_CUDA(cudaMemsetAsync(bits_a, 0, sizeof(u32) * words, s));
        RSQ_CUDA(cudaMemsetAsync(counters + 4, 0, 4 * sizeof(u32), s));
        RSQ_LAUNCH_BEGIN(ctx, "headbits_kernel");
        headbits_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, s>>>(in_b ? k32_b : k32_a, n, field_mask,
                                                                     field_full, bits_a, counters + 4);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters + 4, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaStreamSynchronize(s));
        u32 tied = reinterpret_cast<volatile u32*>(ctx->pinned)[0];
        bool oversize = false;
        if (tied > 0) {
            const unsigned tiles = static_cast<unsigned>((n + kRefTile - 1) / kRefTile);
            RSQ_CUDA(cudaMemcpyAsync(bits_b, bits_a, sizeof(u32) * words, cudaMemcpyDeviceToDevice, s));
            RSQ_CUDA(cudaMemsetAsync(counters + 4, 0, 4 * sizeof(u32), s));
            RSQ_LAUNCH_BEGIN(ctx, "refine_text_kernel");
            refine_text_kernel<<<tiles, kRefBlock, kRefSmem, s>>>(packed, sent, n, sa_cur, n, bits_a, bits_b,
                                                                   static_cast<u32>(h), ctx->opt_text_rounds,
                                                                   use_shortcut, counters + 4);
            RSQ_LAUNCH_END(ctx);
            RSQ_CUDA(cudaGetLastError());
            RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters + 4, 4 * sizeof(u32), cudaMemcpyDeviceToHost, s));
            RSQ_CUDA(cudaStreamSynchronize(s));
            st.refined_tile += tied;
            tied = reinterpret_cast<volatile u32*>(ctx->pinned)[0];
            oversize = reinterpret_cast<volatile u32*>(ctx->pinned)[1] != 0;
            st.rounds += reinterpret_cast<volatile u32*>(ctx->pinned)[2];
            u32* t = bits_a; bits_a = bits_b; bits_b = t;
            // Groups still tied after the kernel share at least h + 29 * max_rounds symbols --
            // unless one was skipped as oversize: that one is still tied at depth h, and prefix
            // doubling must resume from the smallest depth any group is known to share.
            if (!oversize) h += static_cast<u64>(kTextK) * ctx->opt_text_rounds;
        }
        if (tied == 0 && !oversize) {
            // every group is a singleton: sa is final and rank is its inverse
            const int nb = static_cast<int>(bit_width_u64(n - 1));
            if (n >= (size_t{1} << 22)) {
                // two stable passes (low 5 bits of the top 13, then the top 8): windows of
                // n / 8192 rank entries
                const int shift = nb - 8;
                int lo_bits = shift - 13;  // aim at windows of 8192 entries (32 KB of shared memory)
                if (lo_bits < 0) lo_bits = 0;
                if (lo_bits > 8) lo_bits = 8;
                if (ctx->opt_inverse_lo_bits >= 0) lo_bits = ctx->opt_inverse_lo_bits;
                const int win_bits = shift - lo_bits;
                u32* part_pos = reinterpret_cast<u32*>(keys_a);
                u32* part_idx = part_pos + n;
                const u32* src_pos = sa_cur;
                if (lo_bits > 0) {
                    u32* p0 = reinterpret_cast<u32*>(keys_b);
                    u32* i0 = p0 + n;
                    RSQ_LAUNCH_BEGIN(ctx, "perm_digit_hist_kernel");
                    perm_digit_hist_kernel<<<1, kRadix, 0, s>>>(n, shift - lo_bits, lo_bits, ws.hist);
                    RSQ_LAUNCH_END(ctx);
                    RSQ_TRY(onesweep_partition_iota(ctx, sa_cur, p0, i0, n, shift - lo_bits, lo_bits, ws));
                    RSQ_LAUNCH_BEGIN(ctx, "perm_digit_hist_kernel");
                    perm_digit_hist_kernel<<<1, kRadix, 0, s>>>(n, shift, 8, ws.hist);
                    RSQ_LAUNCH_END(ctx);
                    RSQ_TRY(onesweep_partition_pairs(ctx, p0, i0, part_pos, part_idx, n, shift, 8, ws));
                } else {
                    RSQ_LAUNCH_BEGIN(ctx, "perm_digit_hist_kernel");
                    perm_digit_hist_kernel<<<1, kRadix, 0, s>>>(n, shift, 8, ws.hist);
                    RSQ_LAUNCH_END(ctx);
                    RSQ_TRY(onesweep_partition_iota(ctx, src_pos, part_pos, part_idx, n, shift, 8, ws));
                }
                if (win_bits <= 14) {
                    static bool configured = false;
                    if (!configured) {
                        RSQ_CUDA(cudaFuncSetAttribute(window_scatter_kernel,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
                        configured = true;
                    }
                    const unsigned windows = static_cast<unsigned>((n + (size_t{1} << win_bits) - 1) >> win_bits);
                    RSQ_LAUNCH_BEGIN(ctx, "window_scatter_kernel");
                    window_scatter_kernel<<<windows, 512, sizeof(u32) << win_bits, s>>>(part_pos, part_idx, n,
                                                                                        win_bits, rank);
                    RSQ_LAUNCH_END(ctx);
                } else {
                    RSQ_LAUNCH_BEGIN(ctx, "scatter_pairs_kernel");
                    scatter_pairs_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, s>>>(part_pos, part_idx, n, rank);
                    RSQ_LAUNCH_END(ctx);
                }
            } else {  // the whole rank array is L2-resident: scatter directly
                RSQ_LAUNCH_BEGIN(ctx, "inverse_kernel");
                inverse_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, s>>>(sa_cur, n, rank);
                RSQ_LAUNCH_END(ctx);
            }
            RSQ_CUDA(cudaGetLastError());
            heads = n;
            ranked = true;
        } else {
            // hand over to prefix doubling: group-head ranks from the bitmap
            u32* flags = reinterpret_cast<u32*>(keys_b);  // the initial keys are no longer needed
            RSQ_LAUNCH_BEGIN(ctx, "expand_bits_kernel");
            expand_bits_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, s>>>(bits_a, n, flags);
            RSQ_LAUNCH_END(ctx);
            RSQ_CUDA(cudaGetLastError());
            RSQ_TRY(rerank(flags, std::true_type{}, 0u, 0u));
            heads = *reinterpret_cast<volatile u32*>(ctx->pinned);
            ranked = true;
        }
    }
    if (!ranked) {
        RSQ_TRY(rerank(in_b ? k32_b : k32_a, std::false_type{}, field_mask, field_full));
        heads = *reinterpret_cast<volatile u32*>(ctx->pinned);
    }

    // -- prefix doubling (general engine: any alphabet, any group size, any LCP) --------------
    const int b = static_cast<int>(bit_width_u64(n));
    const PassTable pt = make_passes(0, 2 * b);
    for (; heads < n && h < n; h <<= 1) {
        RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * pt.count * kRadix, s));
        {
            const unsigned grid = grid_for(ctx, n, 256, 8, 8);
            RSQ_LAUNCH_BEGIN(ctx, "pair_key_kernel");
            pair_key_kernel<<<grid, 256, sizeof(u32) * pt.count * kRadix, s>>>(
                sa_cur, head_of, rank, n, h, b, keys_a, pt, ws.hist);
            RSQ_LAUNCH_END(ctx);
            RSQ_CUDA(cudaGetLastError());
        }
        RSQ_TRY(onesweep_sort<u64>(ctx, keys_a, keys_b, sa_cur, sa_alt, n, pt, ws, true, 0, &in_b));
        st.sort_passes += pt.count;
        if (in_b) { u32* t = sa_cur; sa_cur = sa_alt; sa_alt = t; }
        RSQ_TRY(rerank(in_b ? keys_b : keys_a, std::false_type{}, 0u, 0u));
        heads = *reinterpret_cast<volatile u32*>(ctx->pinned);
        ++st.rounds;
        st.refined_global += n;
    }

    if (sa_cur != d_sa)
        RSQ_CUDA(cudaMemcpyAsync(d_sa, sa_cur, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
    st.kernel_launches = ctx->launches - launches0;
    if (stats) *stats = st;
    return RESEQ_OK;
}


// ---- multi-GPU building blocks -----------------------------------------------
// One rank of a sample-sort partitioned build: the text is replicated (packed: n/4 bytes), the
// rank keys a slice of positions, and after the all-to-all finishes the bucket of suffixes whose
// keys fall in its splitter range -- same kernels as the single-GPU path, no exchange needed
// afterwards because refinement keys come from the replicated text.

}  // namespace rsq

struct reseq_cuda_sa_shard {
    reseq_cuda_ctx* ctx = nullptr;
    const rsq::u8* d_text = nullptr;
    size_t n = 0;
    rsq::u64* packed = nullptr;
    rsq::u64* sent = nullptr;
    rsq::u32* flags = nullptr;
    bool dna = false;
    bool use_shortcut = false;
};

extern "C" {

int reseq_cuda_sa_shard_create(reseq_cuda_ctx* ctx, const uint8_t* d_text, size_t n, reseq_cuda_sa_shard** out,
                               int* is_dna) {
    using namespace rsq;
    if (!ctx || !out || !d_text || n == 0) return fail(RESEQ_INVALID_ARGUMENT, "null or empty argument");
    if (n > RESEQ_CUDA_MAX_TEXT) return fail(RESEQ_TEXT_TOO_LARGE, "text exceeds 2^32-2");
    *out = nullptr;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    auto* sh = new reseq_cuda_sa_shard();
    sh->ctx = ctx;
    sh->d_text = d_text;
    sh->n = n;
    if (cudaMalloc(&sh->packed, sizeof(u64) * (n / 32 + 8)) != cudaSuccess ||
        cudaMalloc(&sh->sent, sizeof(u64) * (n / 64 + 8)) != cudaSuccess ||
        cudaMalloc(&sh->flags, 256) != cudaSuccess) {
        cudaGetLastError();
        reseq_cuda_sa_shard_destroy(sh);
        return fail(RESEQ_OUT_OF_MEMORY, "cudaMalloc failed for the packed text");
    }
    u64 n_sep = 0;
    int st = pack_dna_device(ctx, d_text, n, sh->packed, sh->sent, sh->flags, &sh->dna, &n_sep);
    if (st != RESEQ_OK) {
        reseq_cuda_sa_shard_destroy(sh);
        return st;
    }
    sh->use_shortcut = ctx->opt_shortcut != 0 && n_sep * 1024 >= n;
    if (is_dna) *is_dna = sh->dna ? 1 : 0;
    *out = sh;
    return RESEQ_OK;
}

void reseq_cuda_sa_shard_destroy(reseq_cuda_sa_shard* sh) {
    if (!sh) return;
    if (sh->ctx) {
        cudaSetDevice(sh->ctx->device);
        cudaStreamSynchronize(sh->ctx->stream);
    }
    cudaFree(sh->packed);
    cudaFree(sh->sent);
    cudaFree(sh->flags);
    delete sh;
}

int reseq_cuda_sa_shard_keys(reseq_cuda_sa_shard* sh, uint64_t pos_begin, size_t count, uint32_t* d_keys,
                             uint32_t* d_pos) {
    using namespace rsq;
    if (!sh || !sh->dna) return fail(RESEQ_INVALID_ARGUMENT, "the sharded build needs a DNA text");
    if (count == 0) return RESEQ_OK;
    if (pos_begin + count > sh->n) return fail(RESEQ_INVALID_ARGUMENT, "position slice out of range");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    RSQ_TRY(ctx->reserve(reseq_cuda_ctx::padded(sizeof(u32) * kMaxPasses * kRadix) + 4096));
    ctx->begin();
    u32* hist = ctx->alloc<u32>(kMaxPasses * kRadix);  // the slice's histogram is not used: buckets re-count
    const PassTable pt0 = make_passes(0, 2 * kDnaK + kDnaFieldBits);
    RSQ_CUDA(cudaMemsetAsync(hist, 0, sizeof(u32) * pt0.count * kRadix, ctx->stream));
    RSQ_LAUNCH_BEGIN(ctx, "initkey_dna_kernel");
    initkey_dna_kernel<<<grid_for(ctx, count, 256, 8, 8), 256, sizeof(u32) * pt0.count * kRadix, ctx->stream>>>(
        sh->packed, sh->sent, sh->n, pos_begin, count, d_keys, d_pos, pt0, hist);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_finish(reseq_cuda_sa_shard* sh, uint32_t* d_keys, uint32_t* d_pos, size_t m,
                               uint32_t* d_sa_out, uint64_t* unfinished) {
    using namespace rsq;
    if (!sh || !sh->dna || !unfinished) return fail(RESEQ_INVALID_ARGUMENT, "bad shard argument");
    *unfinished = 0;
    if (m == 0) return RESEQ_OK;
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(2 * pad(sizeof(u32) * m) + 2 * pad(sizeof(u32) * (m / 32 + 8)) + sort_workspace_bytes(m) + 8192));
    ctx->begin();
    u32* keys_b = ctx->alloc<u32>(m);
    u32* pos_b = ctx->alloc<u32>(m);
    u32* bits_a = ctx->alloc<u32>(m / 32 + 8);
    u32* bits_b = ctx->alloc<u32>(m / 32 + 8);
    u32* counters = ctx->alloc<u32>(64);
    SortWorkspace ws;
    if (!keys_b || !pos_b || !bits_a || !bits_b || !counters) return fail(RESEQ_OUT_OF_MEMORY, "shard workspace");
    RSQ_TRY(sort_workspace_carve(ctx, m, &ws));
    // stable sort of the bucket on the 31-bit key: equal keys stay in ascending position order
    // because the exchange delivers the slices in rank (= position) order
    const PassTable pt0 = make_passes(0, 2 * kDnaK + kDnaFieldBits);
    bool in_b = false;
    RSQ_TRY(onesweep_sort<u32>(ctx, d_keys, keys_b, d_pos, pos_b, m, pt0, ws, false, 0, &in_b));
    u32* sa_cur = in_b ? pos_b : d_pos;
    const size_t words = (m + 31) / 32 + 4;
    RSQ_CUDA(cudaMemsetAsync(bits_a, 0, sizeof(u32) * words, s));
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 256, s));
    RSQ_LAUNCH_BEGIN(ctx, "headbits_kernel");
    headbits_kernel<<<grid_for(ctx, m, 256, 4, 16), 256, 0, s>>>(in_b ? keys_b : d_keys, m, (1u << kDnaFieldBits) - 1u,
                                                                 2u * kDnaK, bits_a, counters);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(bits_b, bits_a, sizeof(u32) * words, cudaMemcpyDeviceToDevice, s));
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 256, s));
    static bool configured = false;
    if (!configured) {
        RSQ_CUDA(cudaFuncSetAttribute(refine_text_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kRefSmem)));
        configured = true;
    }
    const unsigned tiles = static_cast<unsigned>((m + kRefTile - 1) / kRefTile);
    RSQ_LAUNCH_BEGIN(ctx, "refine_text_kernel");
    refine_text_kernel<<<tiles, kRefBlock, kRefSmem, s>>>(sh->packed, sh->sent, sh->n, sa_cur, m, bits_a, bits_b,
                                                          kDnaK, 1 << 20, sh->use_shortcut, counters);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaMemcpyAsync(d_sa_out, sa_cur, sizeof(u32) * m, cudaMemcpyDeviceToDevice, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    // still tied (only possible through an oversize group: the round limit is out of reach)
    *unfinished = reinterpret_cast<volatile u32*>(ctx->pinned)[0] + (reinterpret_cast<volatile u32*>(ctx->pinned)[1] ? 1u : 0u);
    return RESEQ_OK;
}

int reseq_cuda_inverse_device(reseq_cuda_ctx* ctx, const uint32_t* d_sa, size_t n, uint32_t* d_rank) {
    using namespace rsq;
    if (!ctx) return fail(RESEQ_INVALID_ARGUMENT, "null context");
    if (n == 0) return RESEQ_OK;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    RSQ_LAUNCH_BEGIN(ctx, "inverse_kernel");
    inverse_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, ctx->stream>>>(d_sa, n, d_rank);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

}  // extern "C"

namespace rsq {
}  // namespace rsq
