// Suffix-array construction on sm_100a.
//
// Replaces build_parallel, suffix_array.hpp:61-124.  Same mathematical result -- the unique
// permutation sorted by suffix_less (suffix_array.hpp:28-41) and its inverse -- by one of three
// routes, chosen from what pack_dna_kernel finds in the text (build_sa_device at the bottom):
//
//   (i)   uniform read sets (k reads of one length): transposed 16-base records, 4 onesweep passes,
//         one verified overlap per READ proves the order of its suffixes, groups accepted as they
//         stand (gen_uniform / link_reads / accept_uniform / refine_elems<true>);
//   (ii)  other DNA texts: 11.5-base records + terminator byte, 3 passes, groups finished in shared
//         memory from the L2-resident 2-bit text (init_elems / refine_elems<false>);
//   (iii) anything else -- generic alphabets, groups too large for (i)/(ii): prefix doubling over
//         (rank[i], rank[i+h]) pairs, the reference's own scheme with fatter phases:
//
//   reference                                   route (iii)
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
// The inverse permutation of (i) and (ii) is two lean partition passes + a shared-memory window
// scatter (inv_partition_persistent_kernel, window_scatter_kernel).
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

#include <algorithm>
#include <cstdlib>
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
            // four bytes at a time (the kernel was bound by its ~20 instructions per byte, not by HBM):
            //   code  = ((c >> 1) ^ (c >> 2)) & 3 in every byte lane; one multiply gathers the four 2-bit
            //           codes into a byte, first base highest (no partial products collide below bit 24,
            //           the others overflow);
            //   zero  = the classic has-zero-byte mask; valid = zero or equal to one of A, C, G, T.
            auto zero_mask = [](u32 v) { return ~(((v & 0x7f7f7f7fu) + 0x7f7f7f7fu) | v | 0x7f7f7f7fu); };   // 0x80 per zero byte
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = ld_stream_v4(text + base + 16 * q);
                const u32 word[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const u32 w4 = word[t];
                    const u32 zm = zero_mask(w4);
                    const u32 ok = zm | zero_mask(w4 ^ 0x41414141u) | zero_mask(w4 ^ 0x43434343u) |
                                   zero_mask(w4 ^ 0x47474747u) | zero_mask(w4 ^ 0x54545454u);
                    bad |= ok != 0x80808080u;
                    const u32 codes = ((w4 >> 1) ^ (w4 >> 2)) & 0x03030303u;                // zero bytes give 0
                    const u64 byte = (codes * 0x40100401u) >> 24;                           // c0 c1 c2 c3, 2 bits each
                    const u64 zbits = ((zm >> 7) * 0x08040201u) >> 24 & 0xfu;               // z0 z1 z2 z3 -> bits 3..0
                    const int p = 16 * q + 4 * t;                                           // first position of the group
                    if (p < 32) p0 |= byte << (56 - 2 * p);
                    else p1 |= byte << (56 - 2 * (p - 32));
                    s |= zbits << (60 - p);
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

template <typename KeyT, bool SCATTER = true>
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
        const bool head = idx < n && (idx == 0 || k[j] != prev ||
                                      (static_cast<u32>(k[j]) & uniq_mask) != uniq_full);
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
            if constexpr (SCATTER) rank[sa[idx]] = h;   // (n random 4-byte writes: 5.9 ms at n = 139 M; the partitioned
                                                        //  rank update below does the same in 1.3)
        }
    }
}

// ---- DNA fast path: sort records, refine groups from L2-resident text --------------------
//
// One 64-bit record per suffix:   key24 << 40 | p8 << 32 | pos
//   key24  three 8-bit sort digits.  Upper two: bases 0..7 (2 bits each, zero padded from the
//          terminator on).  Low digit: 0x80 | bases 8..10 | upper bit of base 11 for a suffix
//          with more than 8 symbols, and 2*t + kind (< 0x80) for a suffix that terminates after
//          t <= 8 symbols (kind 0 = end of text, 1 = sentinel).  Zero padding alone would tie
//          "b$" with "bA$", "bAA$" ... and with every suffix starting b AAAA...: the k empty
//          suffixes of a k-read set would form ONE group.  With the escape bit those short
//          suffixes sort before everything that shares their padded bases, by length, then (the
//          sort is stable) by position -- which is their final order: they are finished by the
//          sort alone.  What remains tied shares 11 symbols.
//   p8     where the suffix terminates, measured once while the positions are still in text
//          order (a streaming read of the sentinel bitmap):
//            2*t + kind   terminator after t < 11 symbols
//            t + 11       sentinel after 11 <= t <= 242 symbols
//            254          sentinel farther away / not determined: the refine kernel scans for it
//            255          the text ends first (no sentinel at all behind the suffix)
//   pos    text position.
// Three onesweep passes on key24 (the records move as single 64-bit elements: half the load /
// store / exchange instructions of separate key and payload arrays) leave the suffixes grouped
// by key with positions ascending inside a group.
//
// After the sort a group holds suffixes that agree on their first 11 symbols (with zero
// padding: a suffix terminating after 9 or 10 symbols joins the group of its padded bases).  On B200 the
// 2-bit packed text (n/4 bytes: 35 MB at 4.6 Mbp x 30) fits the 126 MB L2 while the 4n-byte rank
// array of a doubling round does not, so the order inside a group is settled from the text
// itself.  Each CTA owns the groups that START inside its 2048-suffix tile, stages them in
// shared memory, finishes them there and writes the suffix array tile once.  No global sort, no
// rank array, no scatter.
//
// A group that does not fit the CTA's shared-memory window (more than kRefExt suffixes past
// the tile) is reported; the host then rebuilds with the general prefix-doubling engine below,
// which has no size limit.

constexpr int kElemK = 11;                  // symbols every member of a group is known to share
constexpr int kElemEsc = 8;                 // suffixes terminating after <= 8 symbols are finished by the sort
constexpr u32 kElemEscBit = 0x80;
constexpr int kElemKeyShift = 40;
constexpr u32 kPShortEnd = 2 * kElemK;      // payloads below this: terminator inside the shared symbols
constexpr u32 kPMaxNear = 253;              // largest payload that encodes a distance (242 + 11)
constexpr u32 kPFar = 254;
constexpr u32 kPEot = 255;

constexpr int kUniK = 16;                   // uniform read sets: symbols shared inside a group
constexpr u32 kUniMinPeriod = 17, kUniMaxPeriod = 255;   // read length + 1 the uniform path accepts
constexpr int kUniReads = 64;               // reads per CTA of the record generator

constexpr int kRefBlock = 256;
constexpr int kRefTile = 2048;
constexpr int kRefExt = 640;
constexpr int kRefCap = kRefTile + kRefExt;
constexpr int kRefWords = kRefCap / 32 + 2;
constexpr size_t kRefSmem = sizeof(u64) * kRefCap + sizeof(u32) * kRefCap + 4 * sizeof(unsigned short) * kRefCap +
                            sizeof(u32) * (5 * kRefWords + 16);
constexpr int kStepK = 16;          // bases compared per refinement step
constexpr u32 kDistCap = 4095;      // farthest sentinel the bitmap scan looks for
constexpr u32 kTdNone = 0xFFFF;     // "terminator not known": the suffix can only be split by its bases
constexpr u32 kTdMax = 16000;       // largest distance to the terminator kept (2 * t + kind must fit 16 bits)
constexpr u32 kOrdNone = 0x7FFF;
constexpr int kOrdBits = 15;
constexpr int kSlotBits = 12;       // window slot of the suffix: makes every key of a step unique
static_assert(kRefCap <= (1 << kSlotBits), "window slots must fit the key's slot field");
static_assert(2 * kStepK + kOrdBits + kSlotBits <= 64, "step key layout");
static_assert(2 * kTdMax + 1 + 2 * kElemK < kOrdNone && 2 * (kDistCap + kElemK) + 1 <= 2 * kTdMax + 1, "terminator distances must fit the order field");

// Records of the `count` suffixes starting at text position pos0 (the whole text: pos0 = 0,
// count = n; a multi-GPU rank keys only its slice), plus the digit histograms of the three sort
// passes.
// The record of the suffix at `pos` (layout above).
__device__ __forceinline__ u64 elem_of(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n, u64 pos) {
    const u32 bases = static_cast<u32>(base_window(packed, pos) >> 40);   // 12 bases
    // distance to the first sentinel at or after pos, looking 256 positions ahead
    u32 t = 256;
#pragma unroll 1
    for (u32 c0 = 0; c0 < 256; c0 += 64) {
        const u64 w = sent_window(sent, pos + c0);
        if (w) {
            t = c0 + static_cast<u32>(__clzll(w));
            break;
        }
    }
    const u64 rem = n - pos;  // >= 1
    u32 tt, kind;              // symbols before the terminator (256 = not within reach), its kind
    if (t < 256 && t < rem) { tt = t; kind = 1; }
    else if (rem <= 256) { tt = static_cast<u32>(rem); kind = 0; }
    else { tt = 256; kind = 1; }
    const u32 kept = tt >= 12 ? bases : bases & ~((1u << (24 - 2 * tt)) - 1u);   // zero padded
    u32 key, p;
    if (tt <= kElemEsc) {
        key = ((kept >> 8) << 8) | (2 * tt + kind);
        p = 2 * tt + kind;
    } else {
        const u32 b23 = kept >> 1;   // bases 0..10 and the upper bit of base 11
        key = ((b23 >> 7) << 8) | kElemEscBit | (b23 & 0x7fu);
        if (tt < kElemK) p = 2 * tt + kind;
        else if (tt == 256) p = kPFar;
        else if (kind == 0) p = kPEot;
        else p = tt + kElemK <= kPMaxNear ? tt + kElemK : kPFar;
    }
    return (static_cast<u64>(key) << kElemKeyShift) | (static_cast<u64>(p) << 32) | (pos & 0xffffffffu);
}

__global__ void __launch_bounds__(256)
init_elems_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n, u64 pos0, u64 count,
                  u64* __restrict__ elems, u32* __restrict__ g_hist) {
    __shared__ u32 s_hist[3 * kRadix];
    for (int i = threadIdx.x; i < 3 * kRadix; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < count; idx += stride) {
        const u64 e = elem_of(packed, sent, n, pos0 + idx);
        const u32 key = static_cast<u32>(e >> kElemKeyShift);
        elems[idx] = e;
        atomicAdd(&s_hist[key & 0xffu], 1u);
        atomicAdd(&s_hist[kRadix + ((key >> 8) & 0xffu)], 1u);
        atomicAdd(&s_hist[2 * kRadix + (key >> 16)], 1u);
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, 3);
}

// 128-bit load of two consecutive packed words (the pair index is even: 16-byte aligned).
__device__ __forceinline__ void ld_words2(const u64* __restrict__ p, u64& w0, u64& w1) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    w0 = (static_cast<u64>(v.y) << 32) | v.x;
    w1 = (static_cast<u64>(v.w) << 32) | v.z;
}

// The 16 bases starting at position q, top aligned in 32 bits.  One 128-bit gather of the aligned
// word pair serves 3 windows in 4; the kernel is bound by issue slots and L1 wavefronts (one per
// lane per gather), so fewer, wider gathers is what counts.
__device__ __forceinline__ u32 bases16(const u64* __restrict__ packed, u64 q) {
    const u64 w = q >> 5;
    const unsigned s = static_cast<unsigned>(q & 31) * 2;
    u64 w0, w1;
    ld_words2(packed + (w & ~1ull), w0, w1);
    u64 hi = (w & 1) ? w1 : w0;
    u64 win = hi << s;
    if (s > 32) {  // the window runs into the next word
        const u64 lo = (w & 1) ? packed[w + 1] : w1;
        win |= lo >> (64 - s);
    }
    return static_cast<u32>(win >> 32);
}

// One CTA finishes every group that starts in its tile: the key of a tied suffix depends only
// on (position, depth), never on another group, so all steps run back to back in shared memory.
//
// A step at depth d (all members of a group share their first d symbols) orders each group by
//     ( next 16 bases, zero padded from the terminator on | 2 * (t - d) + kind | slot )
// where t is the suffix's distance to its terminator, known from the record.  Suffixes that
// differ in the 16 bases are split for good.  Those that agree form a subgroup ordered by
// terminator distance, which is their final order IF every member is a prefix of the longest
// one -- in a read set a subgroup is the reads over one locus, so that is the rule, not the
// exception.  Every member is therefore compared base by base, over its remaining length, with
// the subgroup's longest member (128-bit gathers from the L2-resident packed text).  If all
// agree the subgroup is final: ONE step instead of ceil(read length / 16).  If not (repeats),
// the members that terminate inside the 16 bases are final, the others stay tied at depth
// d + 16 and take another step.  Slots keep position order among equal keys, which is what
// the total order asks for where two suffixes are identical up to their sentinels.
// Every step first compacts the still-tied suffixes into a dense list (order preserving, so a
// group stays contiguous): late steps cost in proportion to what is left.
//
// UNI: the records of a uniform read set (gen_uniform_kernel below): 15 shared symbols, groups
// already in (terminator distance, position) order, and a table `cov` (one byte per read: its
// suffixes with at most that many symbols before the sentinel) of the positions that
// link_reads_kernel proved to be a prefix of a LONGER suffix of their own group.  A group all of
// whose members but the last carry that proof is final as it stands -- every chain of witnesses
// ends in the last member, so all members are prefixes of it and (distance, position) is their
// order -- and never enters the step loop; in the loop the same proof replaces the base-by-base
// comparison.  The terminator distance is arithmetic there: period - 1 - pos mod period.
// MODE: kRefGeneral (the records above), kRefUniform (UNI), kRefRagged (UNI's flow for read sets of mixed
// lengths: terminator distances from the sentinel bitmap's rank structure -- read id = separators before
// the position, t = ends[id] - position -- and proofs as one bit per POSITION, see the ragged kernels below).
enum : int { kRefGeneral = 0, kRefUniform = 1, kRefRagged = 2 };
constexpr int kRagK = 15;   // ragged records: 15 bases + a 2-bit tag that is 0 for suffixes shorter than that

template <int MODE>
__global__ void __launch_bounds__(kRefBlock)
refine_elems_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n_text,
                    const u64* __restrict__ elems, u64 m, u32* __restrict__ sa_out,
                    int max_rounds, bool use_shortcut, u32* __restrict__ counters,
                    const u8* __restrict__ cov, u32 period, u64 period_magic,
                    const u32* __restrict__ g_headbits, const u32* __restrict__ g_uncbits,
                    const u8* __restrict__ g_tileflags, const u32* __restrict__ cum = nullptr,
                    const u32* __restrict__ ends = nullptr) {
    constexpr bool UNI = MODE != kRefGeneral;
    constexpr int KSYM = MODE == kRefUniform ? kUniK : (MODE == kRefRagged ? kRagK : kElemK);   // symbols every member of a group shares
    constexpr int KEYSHIFT = kElemKeyShift;                // general records: bits above this are the group key
    constexpr u32 ESCBIT = kElemEscBit;                    // (the uniform path reads its group heads from a bitmap)
    auto term_dist = [&](u32 pos) -> u32 {   // UNI only: symbols before the read's sentinel
        if constexpr (MODE == kRefRagged) {
            const u32 w = pos >> 6, b = pos & 63u;
            const u32 q = cum[w] + (b ? static_cast<u32>(__popcll(sent[w] >> (64 - b))) : 0u);   // separators before pos = read id
            return ends[q] - pos;
        } else {
            const u32 q = static_cast<u32>(__umul64hi(pos, period_magic));
            return period - 1u - (pos - q * period);
        }
    };
    auto covered = [&](u32 pos) -> bool {    // UNI only: proven a prefix of a later member of its group
        if constexpr (MODE == kRefRagged) {
            return (reinterpret_cast<const u32*>(cov)[pos >> 5] >> (pos & 31u)) & 1u;
        } else {
            const u32 q = static_cast<u32>(__umul64hi(pos, period_magic));
            return period - 1u - (pos - q * period) <= __ldg(cov + q);
        }
    };
    // n_text: length of the text the positions refer to; m: number of records (equal for a
    // whole-text build, a bucket of it for a multi-GPU rank)
    extern __shared__ __align__(16) unsigned char ref_smem[];
    u64* s_key = reinterpret_cast<u64*>(ref_smem);               // [cap] records, then keys of the step ...
    u32* s_pos2 = reinterpret_cast<u32*>(ref_smem);              // ... then the permuted positions
    unsigned short* s_td2 = reinterpret_cast<unsigned short*>(s_pos2 + kRefCap);  // ... and terminators
    u32* s_pos = reinterpret_cast<u32*>(s_key + kRefCap);        // [cap] suffix positions, sa order
    unsigned short* s_list = reinterpret_cast<unsigned short*>(s_pos + kRefCap);  // [cap] tied slots
    unsigned short* s_dst = s_list + kRefCap;                    // [cap] new slot of list entry u
    unsigned short* s_src = s_dst + kRefCap;                     // [cap] old slot of new slot d
    unsigned short* s_td = s_src + kRefCap;                      // [cap] 2 * t + kind of the suffix, or kTdNone
    u32* s_bits = reinterpret_cast<u32*>(s_td + kRefCap);        // [words] head bits of the window
    u32* s_new = s_bits + kRefWords;                             // [words] heads created this step
    u32* s_fail = s_new + kRefWords;                             // [words] subgroups that failed the prefix check
    u32* s_cnt = s_fail + kRefWords;                             // [words + 1] tied-count scan
    u32* s_mine = s_cnt + kRefWords + 16;                        // [words] UNI: members of the groups this CTA re-sorts
    __shared__ int s_first, s_end, s_last;

    if constexpr (UNI) {
        if (!g_tileflags[blockIdx.x]) return;   // no uncovered member in this tile or the next: nothing to re-sort
    }
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const u64 t0 = static_cast<u64>(blockIdx.x) * kRefTile;
    const int lim = static_cast<int>(m - t0 < static_cast<u64>(kRefTile) ? m - t0 : kRefTile);
    const int avail = static_cast<int>(m - t0 < static_cast<u64>(kRefCap) ? m - t0 : kRefCap);  // records behind t0

    if (tid == 0) { s_first = 0x7fffffff; s_end = 0x7fffffff; s_last = -1; }
    for (int j = tid; j < kRefWords; j += kRefBlock) { s_bits[j] = 0; s_new[j] = 0; s_fail[j] = 0; }

    if constexpr (UNI) {
        // -- group heads and uncovered members of the window were found by accept_uniform_kernel ----
        for (int j = tid; j < kRefWords; j += kRefBlock) {
            u32 h = 0, u = 0;
            if (j * 32 < avail) {
                h = g_headbits[(t0 >> 5) + j];
                u = g_uncbits[(t0 >> 5) + j];
                if (j * 32 + 32 > avail) {
                    const u32 mk = (1u << (avail - j * 32)) - 1u;
                    h &= mk;
                    u &= mk;
                }
            }
            s_bits[j] = h;
            s_new[j] = u;
        }
        __syncthreads();
        if (tid == 0 && avail == static_cast<int>(m - t0) && avail < kRefWords * 32)
            s_bits[avail >> 5] |= 1u << (avail & 31);   // position m acts as a head
        __syncthreads();
    } else {
    // -- load the tile's records plus the first stretch behind it; group heads from adjacent keys.
    //    The window grows only while the tile's last group has not ended (rare). ------------------
    int loaded = 0;
    const u32 prev_key = t0 > 0 ? static_cast<u32>(elems[t0 - 1] >> KEYSHIFT) : 0xffffffffu;
    for (int want = lim + kRefBlock < avail ? lim + kRefBlock : avail;;) {
        for (int j = loaded + tid; j < want; j += kRefBlock) s_key[j] = elems[t0 + j];
        __syncthreads();
        for (int j0 = loaded - (loaded & 31); j0 < want; j0 += kRefBlock) {   // word aligned
            const int j = j0 + tid;
            bool head = false;
            if (j >= loaded && j < want) {
                const u32 k = static_cast<u32>(s_key[j] >> KEYSHIFT);
                const u32 kp = j > 0 ? static_cast<u32>(s_key[j - 1] >> KEYSHIFT) : prev_key;
                head = k != kp || !(k & ESCBIT) || (t0 == 0 && j == 0);   // no escape bit: finished by the sort
            }
            const unsigned b = __ballot_sync(0xffffffffu, head);
            if (lane == 0 && b) atomicOr(&s_bits[j >> 5], b);
        }
        loaded = want;
        __syncthreads();
        // position m acts as a head so that the last group has an end
        if (tid == 0 && loaded == static_cast<int>(m - t0) && loaded < kRefWords * 32)
            s_bits[loaded >> 5] |= 1u << (loaded & 31);
        __syncthreads();
        bool ended = false;  // is there a head at or behind slot lim?
        for (int j = (lim >> 5) + tid; j < kRefWords; j += kRefBlock) {
            u32 w = s_bits[j];
            if (j == (lim >> 5)) w &= 0xffffffffu << (lim & 31);
            ended |= w != 0;
        }
        if (__syncthreads_or(ended) || loaded >= avail) break;
        want = loaded + kRefBlock < avail ? loaded + kRefBlock : avail;
    }
    }

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
    if (first == 0x7fffffff) {        // no group starts in this tile
        // UNI: the tile was flagged, so a group with uncovered members runs through all of it
        if (UNI && tid == 0) atomicOr(counters + 1, 1u);
        return;
    }
    int end = s_end;
    if (end == 0x7fffffff) {          // the tile's last group overruns the window
        if (tid == 0) atomicOr(counters + 1, 1u);
        end = s_last;                 // that group is nobody's: the host rebuilds
    }

    if constexpr (UNI) {
        // -- nothing uncovered in the groups this CTA owns: accept_uniform_kernel's output stands ----
        bool any = false;
        for (int j = tid; j < kRefWords; j += kRefBlock) {
            const int base = j * 32;
            u32 own = 0xffffffffu;
            if (base + 32 <= first || base >= end) own = 0;
            else {
                if (base < first) own &= 0xffffffffu << (first - base);
                if (base + 32 > end) own &= (1u << (end - base)) - 1u;
            }
            const u32 u = s_new[j] & own;
            s_new[j] = u;
            any |= u != 0;
        }
        if (!__syncthreads_or(any)) return;
    }

    // -- unpack the records this CTA owns: position, and 2 * t + kind from the terminator byte ----
    for (int a = first + tid; a < end && !UNI; a += kRefBlock) {
        const u64 e = s_key[a];
        const u32 pos = static_cast<u32>(e);
        const u32 p = static_cast<u32>(e >> 32) & 0xffu;
        u32 td;
        if (p < kPShortEnd) td = p;
        else if (p <= kPMaxNear) td = 2 * (p - kElemK) + 1;
        else if (p == kPEot) {
            const u64 t = n_text - pos;
            td = t <= kTdMax ? 2 * static_cast<u32>(t) : kTdNone;
        } else if (!use_shortcut) {
            td = kTdNone;              // sparse sentinels: the key phase looks for one window by window
        } else {                       // scan the sentinel bitmap (long reads; rare)
            const u64 q = static_cast<u64>(pos) + kElemK;   // no sentinel before that (the byte would say)
            u32 dist = kDistCap + 1, c0 = 0;
            for (; c0 <= kDistCap && q + c0 < n_text; c0 += 64) {
                const u64 w = sent_window(sent, q + c0);
                if (w) {
                    dist = c0 + static_cast<u32>(__clzll(w));
                    break;
                }
            }
            if (dist <= kDistCap && q + dist < n_text) td = 2 * (dist + kElemK) + 1;
            else if (q + c0 >= n_text && n_text - pos <= kTdMax) td = 2 * static_cast<u32>(n_text - pos);  // none up to the end
            else td = kTdNone;
        }
        s_pos[a] = pos;
        s_td[a] = static_cast<unsigned short>(td);
    }
    __syncthreads();

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
    auto is_head = [&](int a) { return (s_bits[a >> 5] >> (a & 31)) & 1u; };

    if constexpr (UNI) {
        // -- groups that are final as they stand.  Uncovered = no proof of being a prefix of a later
        //    member: suffixes shorter than the shared symbols are prefixes of every longer member by
        //    the zero padding of the key, the others need their bit in `cov`.  The last member of a
        //    group needs no proof. ------------------------------------------------------------------
        // (s_new holds the uncovered, not-last members of the owned groups)
        for (int j = tid; j < kRefWords; j += kRefBlock) {   // a group with an uncovered member stays tied
            u32 w = s_new[j];
            while (w) {
                const int a = j * 32 + __ffs(w) - 1;
                w &= w - 1;
                const int gs = group_start(a), ge = group_end(a);
                for (int x = gs >> 5; x <= (ge - 1) >> 5; ++x) {
                    u32 mk = 0xffffffffu;
                    if (x == (gs >> 5)) mk &= 0xffffffffu << (gs & 31);
                    if (x == ((ge - 1) >> 5)) mk &= 0xffffffffu >> (31 - ((ge - 1) & 31));
                    atomicOr(&s_fail[x], mk);
                }
            }
        }
        __syncthreads();
        for (int j = tid; j < kRefWords; j += kRefBlock) {
            const int base = j * 32;
            u32 own = 0xffffffffu;
            if (base + 32 <= first || base >= end) own = 0;
            else {
                if (base < first) own &= 0xffffffffu << (first - base);
                if (base + 32 > end) own &= (1u << (end - base)) - 1u;
            }
            s_bits[j] |= ~s_fail[j] & own;   // every member of a clean group is final: a head
            s_mine[j] = s_fail[j] & own;     // the others are all this CTA reads, sorts and writes back
            s_new[j] = 0;
            s_fail[j] = 0;
        }
        __syncthreads();
        for (int a = first + tid; a < end; a += kRefBlock) {
            if (!((s_mine[a >> 5] >> (a & 31)) & 1u)) continue;
            const u32 pos = sa_out[t0 + a];   // accept_uniform_kernel left the sorted records' positions there
            s_pos[a] = pos;
            s_td[a] = static_cast<unsigned short>(2 * term_dist(pos) + 1);   // period <= 255: always known
        }
        __syncthreads();
    }

    u32 depth = KSYM;
    int rounds = 0;
    for (; rounds < max_rounds; ++rounds) {
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
        __syncthreads();
        const int cnt = static_cast<int>(total);

        // -- keys: 16 bases from the L2-resident text | terminator distance | slot --------------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            const u64 q = static_cast<u64>(s_pos[a]) + depth;
            u32 td = s_td[a];
            if (td == kTdNone) {   // is there a terminator inside this window?
                const u32 sw = q < n_text ? static_cast<u32>(sent_window(sent, q) >> (64 - kStepK)) : 0u;
                const u32 t = sw ? static_cast<u32>(__clz(sw)) - (32 - kStepK) : kStepK;
                const u64 rem = q < n_text ? n_text - q : 0;
                if (t < rem && t < kStepK) td = 2 * (depth + t) + 1;
                else if (rem < kStepK) td = 2 * (depth + static_cast<u32>(rem));
                if (td != kTdNone) s_td[a] = static_cast<unsigned short>(td);
            }
            u32 left = kStepK;                  // real symbols in the window
            u32 ord = kOrdNone;
            if (td != kTdNone) {
                const u32 t = td >> 1;          // >= depth, except for the 9- and 10-symbol suffixes of the first step
                const u32 rest = t > depth ? t - depth : 0u;
                if (rest < left) left = rest;
                ord = td + 2 * KSYM - 2 * depth;   // 2 * (t - depth) + kind, biased so that it stays >= 0
            }
            u32 b = left ? bases16(packed, q) : 0u;
            if (left < kStepK) b = left ? b & ~((1u << (2 * (kStepK - left))) - 1u) : 0u;
            s_key[a] = (((static_cast<u64>(b) << kOrdBits) | ord) << kSlotBits) | static_cast<u32>(a);
        }
        __syncthreads();

        // -- rank inside the group: the keys are unique, so rank = #smaller keys -----------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            const int gs = group_start(a), ge = group_end(a);
            const u64 ki = s_key[a];
            u32 r0 = 0, r1 = 0;
            int j = gs;
            if (j & 1) { r0 += s_key[j] < ki; ++j; }
            for (; j + 1 < ge; j += 2) {   // every member of the group runs the same trip count
                const ulonglong2 k2 = *reinterpret_cast<const ulonglong2*>(s_key + j);
                r0 += k2.x < ki;
                r1 += k2.y < ki;
            }
            if (j < ge) r0 += s_key[j] < ki;
            const int dst = gs + static_cast<int>(r0 + r1);
            s_dst[u] = static_cast<unsigned short>(dst);
            s_src[dst] = static_cast<unsigned short>(a);
        }
        __syncthreads();

        // -- subgroup heads: the 16 bases differ from the predecessor's in the new order -------------
        bool sub_head[(kRefCap + kRefBlock - 1) / kRefBlock];
#pragma unroll
        for (int i = 0; i < (kRefCap + kRefBlock - 1) / kRefBlock; ++i) {
            const int u = tid + i * kRefBlock;
            sub_head[i] = false;
            if (u < cnt) {
                const int dst = s_dst[u];
                if (!is_head(dst))
                    sub_head[i] = (s_key[s_src[dst - 1]] >> (kOrdBits + kSlotBits)) != (s_key[s_list[u]] >> (kOrdBits + kSlotBits));
            }
        }
        __syncthreads();
        // -- permute (the key buffer is dead: it receives the new order) ---------------------------
#pragma unroll
        for (int i = 0; i < (kRefCap + kRefBlock - 1) / kRefBlock; ++i) {
            const int u = tid + i * kRefBlock;
            if (u < cnt) {
                const int a = s_list[u];
                const int dst = s_dst[u];
                s_pos2[dst] = s_pos[a];
                s_td2[dst] = s_td[a];
                if (sub_head[i]) atomicOr(&s_new[dst >> 5], 1u << (dst & 31));
            }
        }
        __syncthreads();
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            s_pos[a] = s_pos2[a];
            s_td[a] = s_td2[a];
        }
        if (tid < kRefWords) {
            s_bits[tid] |= s_new[tid];
            s_new[tid] = 0;
        }
        __syncthreads();

        // -- prefix check: the member now in slot a against the last (= longest) of its subgroup ----
        const u32 depth2 = depth + kStepK;
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            const int ge = group_end(a);
            s_dst[u] = static_cast<unsigned short>(ge);
            if (!use_shortcut) continue;
            if (is_head(a) && ge == a + 1) continue;     // alone in its subgroup
            const int ra = ge - 1;
            if constexpr (UNI) {
                if (ra != a && covered(s_pos[a])) continue;   // a proven prefix of a later member of this subgroup
            }
            const u32 td = s_td[a], tr = s_td[ra];
            bool ok = td != kTdNone && tr != kTdNone;
            // symbols of this suffix still to be confirmed: [depth2, t)
            if (ok && ra != a && (td >> 1) > depth2) {
                const u64 qa = static_cast<u64>(s_pos[a]) + depth2;
                const u64 qr = static_cast<u64>(s_pos[ra]) + depth2;
                const u64 qe = static_cast<u64>(s_pos[a]) + (td >> 1);   // end of the stretch (exclusive)
                const u64 w_first = qa >> 5, w_last = (qe - 1) >> 5;
                for (u64 w = w_first & ~1ull; w <= w_last && ok; w += 2) {
                    u64 own[2];
                    ld_words2(packed + w, own[0], own[1]);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const u64 wb = (w + h) << 5;                 // first base of this word
                        if (w + h < w_first || w + h > w_last) continue;
                        const u64 lo = wb > qa ? wb : qa;
                        const u64 hi = wb + 32 < qe ? wb + 32 : qe;
                        const unsigned sh = static_cast<unsigned>(lo - wb) * 2;
                        const unsigned nb = static_cast<unsigned>(hi - lo) * 2;   // 2..64 bits
                        const u64 mine = own[h] << sh;
                        const u64 theirs = base_window(packed, qr + (lo - qa));
                        ok = ok && ((mine ^ theirs) >> (64 - nb)) == 0;
                    }
                }
            }
            if (!ok) atomicOr(&s_fail[ra >> 5], 1u << (ra & 31));
        }
        __syncthreads();

        // -- new heads: a confirmed subgroup is final; in the others, what terminates inside the
        //    16 bases is final and the first of the rest opens what stays tied ----------------------
        for (int u = tid; u < cnt; u += kRefBlock) {
            const int a = s_list[u];
            if (is_head(a)) continue;
            const int ra = s_dst[u] - 1;
            bool head;
            if (use_shortcut && !((s_fail[ra >> 5] >> (ra & 31)) & 1u)) head = true;
            else {
                const u32 tp = s_td[a - 1];     // the predecessor is in the same subgroup
                head = tp != kTdNone && (tp >> 1) < depth2;   // (this suffix itself terminates later, or also inside)
            }
            if (head) atomicOr(&s_new[a >> 5], 1u << (a & 31));
        }
        __syncthreads();
        if (tid < kRefWords) {
            s_bits[tid] |= s_new[tid];
            s_new[tid] = 0;
        }
        __syncthreads();
        depth = depth2;
    }

    // write the tile's suffixes once; count what is still tied
    u32 nonheads = 0;
    for (int a = first + tid; a < end; a += kRefBlock) {
        if (UNI && !((s_mine[a >> 5] >> (a & 31)) & 1u)) continue;
        sa_out[t0 + a] = s_pos[a];
        nonheads += !is_head(a);
    }
    for (int o = 16; o > 0; o >>= 1) nonheads += __shfl_xor_sync(0xffffffffu, nonheads, o);
    if (lane == 0 && nonheads) atomicAdd(counters, nonheads);
    if (tid == 0) atomicMax(counters + 2, static_cast<u32>(rounds));
}

// ---- uniform read sets: records born in (terminator distance, position) order ---------------------
//
// A text of k reads of one length L (period P = L + 1: a sentinel at every position = P - 1 mod P,
// nowhere else) is the shotgun read set of BASELINE.json.  Its records are generated TRANSPOSED:
// record index t * k + r belongs to the suffix of read r with t symbols before its sentinel, so
// the stable LSD sort leaves every run of equal keys in (t, position) order -- which is the final
// order of a run whose members all cover one locus (each is a prefix of the longer ones).  Record:
//     key32 << 32 | pos,   key32 = the first 16 bases, zero padded from the sentinel on.
// No length code is needed: a suffix with t < 16 symbols ties only with suffixes that continue its
// t symbols with A's, it is a prefix of every one of them, and with the (t, position) start order
// the stable sort puts it first -- suffixes that short are final after the sort and are group
// heads by themselves; a group is what remains: >= 16 shared symbols.  Whole reads (t = L) are
// recognised arithmetically (position mod period = 0).  A 4.6 Mbp genome has 4.6 M loci against
// 4^16 = 4.3 G keys, so a group is one locus but for chance repeats; the fourth digit pass buys
// groups that need no sorting at all.

// Stages the packed words of reads [r0, r0 + nr) of a uniform read set; returns the bit offset of
// read r0's first base inside the staged words.
// One bulk copy (TMA) per CTA: the stretch is contiguous; the caller's __syncthreads() follows.  The copy
// starts at an even word (16-byte aligned) and covers an even number of words.
__device__ __forceinline__ u32 stage_reads(const u64* __restrict__ packed, u64* __restrict__ s_w, u64 r0, u32 nr, u32 period) {
    __shared__ __align__(8) u64 s_bar;
    const u64 base0 = r0 * period;
    const u64 w0 = (base0 >> 5) & ~1ull;
    const u32 nw = (static_cast<u32>(((base0 + static_cast<u64>(nr) * period + 31) >> 5) - w0) + 3u) & ~1u;   // the packed array is padded
    if (threadIdx.x == 0) mbar_init(&s_bar, 1);
    __syncwarp();   // (racecheck attributes the barrier's initialisation to the warp, not to its lane 0)
    if (threadIdx.x == 0) {
        mbar_expect_tx(&s_bar, nw * 8u);
        tma_load_1d(s_w, packed + w0, nw * 8u, &s_bar);
    }
    __syncthreads();          // the barrier object is initialised for everybody ...
    mbar_wait(&s_bar, 0);     // ... and the words have landed
    return 2 * static_cast<u32>(base0 - (w0 << 5));
}

// Speculative route (build_sa_device): the pack kernel's verdict -- flags[0] != 0: a byte outside
// {A,C,G,T,0}; flags[1]: number of separators -- against what the route was launched on.
__global__ void route_check_kernel(const u32* __restrict__ flags, u32 reads, u32* __restrict__ bad) {
    if (flags[0] != 0u || flags[1] != reads) atomicAdd(bad, 1u);
}

__global__ void uniform_check_kernel(const u64* __restrict__ sent, u32 period, u64 k, u32* __restrict__ bad) {
    const u64 r = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= k) return;
    const u64 p = r * period + period - 1;
    if (!((sent[p >> 6] >> (63 - (p & 63))) & 1ull)) atomicAdd(bad, 1u);   // k sentinels in all: all are here or one is not
}

__global__ void __launch_bounds__(256)
gen_uniform_kernel(const u64* __restrict__ packed, u32 period, u64 read0, u64 k, u64* __restrict__ elems,
                   u32* __restrict__ g_hist) {
    // reads [read0, read0 + k) of the set (the whole set: read0 = 0); record t * k + (read - read0)
    __shared__ __align__(16) u64 s_w[kUniReads * kUniMaxPeriod / 32 + 8];
    __shared__ u32 s_hist[4 * kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) s_hist[i] = 0;
    const u64 r0 = static_cast<u64>(blockIdx.x) * kUniReads;   // within the slice
    const u32 nr = static_cast<u32>(k - r0 < kUniReads ? k - r0 : kUniReads);
    const u32 bit0 = stage_reads(packed, s_w, read0 + r0, nr, period);   // one TMA bulk load + the block barrier
    // Thread = (read rl, quarter q of its offsets): consecutive offsets of one read, so the 16-base key comes from a
    // window that slides two bits per suffix (refilled from shared memory every 16 offsets) instead of a fresh
    // two-word extraction per suffix; at a given step the lanes of a warp are consecutive reads at one offset: the
    // stores stay coalesced.  (One strided (read, t) item per trip: 45 instructions per suffix, the kernel was bound
    // by issue slots at 0.63 of the HBM peak.)
    const u32 rl = threadIdx.x & (kUniReads - 1), q = threadIdx.x / kUniReads;
    constexpr u32 kQuarters = 256 / kUniReads;
    static_assert(kQuarters * kUniReads == 256, "gen_uniform_kernel runs 256 threads");
    const u32 per = (period + kQuarters - 1) / kQuarters;
    const u32 o_begin = q * per, o_end = o_begin + per < period ? o_begin + per : period;
    if (rl < nr) {
        const u32 read_bit0 = bit0 + 2 * rl * period;
        const u64 pos0 = (read0 + r0 + rl) * period;
        u64* dst = elems + r0 + rl;
        u64 win = 0;
        for (u32 o = o_begin; o < o_end; ++o) {
            if (((o - o_begin) & 15u) == 0) {
                const u32 bit = read_bit0 + 2 * o;
                const u32 wi = bit >> 6, sh = bit & 63;
                const u64 hi = s_w[wi], lo = s_w[wi + 1];
                win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
            }
            const u32 t = period - 1 - o;
            u32 key = static_cast<u32>(win >> 32);                          // 16 bases
            win <<= 2;
            if (t < kUniK) key = t ? key & ~((1u << (2 * (kUniK - t))) - 1u) : 0u;   // zero padded from the sentinel on
            dst[static_cast<u64>(t) * k] = (static_cast<u64>(key) << 32) | (pos0 + o);
            // One histogram serves all four passes: digit j of a suffix (bases 4j..4j+3 of its window,
            // zero padded) is the TOP digit of the suffix 4j positions further into the same read, and 0
            // if there is none.  So H_j = A - B_j + [0] * 4jk, A = top-digit histogram of all suffixes,
            // B_j = that of the suffixes at the first 4j offsets of a read (8 % of them); see
            // uniform_hist_kernel.  Rows here: [3] = A, [2] = B_1, [1] = B_2, [0] = B_3.
            const u32 top = key >> 24;
            atomicAdd(&s_hist[3 * kRadix + top], 1u);
            if (o < 12) {
                atomicAdd(&s_hist[top], 1u);
                if (o < 8) atomicAdd(&s_hist[kRadix + top], 1u);
                if (o < 4) atomicAdd(&s_hist[2 * kRadix + top], 1u);
            }
        }
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, 4);
}

// Turns gen_uniform_kernel's rows (A, B_1, B_2, B_3) into the digit histograms of the four passes
// for k reads: pass p (p = 3: top digit) counts H = A - B_(3-p) + [digit 0] * 4 (3 - p) k.
__global__ void uniform_hist_kernel(u32* __restrict__ hist, u64 k) {
    const u32 v = threadIdx.x;
    const u32 a = hist[3 * kRadix + v];
    for (int p = 0; p < 3; ++p) {
        const u32 pad = v == 0 ? static_cast<u32>(4ull * (3 - p) * k) : 0u;
        hist[p * kRadix + v] = a - hist[p * kRadix + v] + pad;
    }
}

// Proofs for refine_elems_kernel<true>.  In a sorted group the predecessors of a whole read b
// (S = 1, t = L) are the suffixes of the reads that started before it on the same locus; the nearest
// one, a = (read r, offset d), is compared with b over its whole length t_a.  If equal, every
// position of r from d on is a prefix of the suffix the same distance into b -- a longer member of
// its own group (it shares all of the shorter one's symbols) -- and gets its bit in `cov`.  One
// comparison per read pays for the ~L suffix comparisons it stands for.  Candidates of other loci
// (chance repeats of the 15 symbols) fail the comparison and are passed over.
__device__ __forceinline__ void link_one_read(const u64* __restrict__ elems, u64 i, const u64* __restrict__ packed,
                                              u32 period, u64 period_magic, u8* __restrict__ cov) {
    const u64 e = elems[i];
    const u32 pos_b = static_cast<u32>(e);
    for (u64 s = 1; s <= 16 && s <= i; ++s) {
        const u64 ea = elems[i - s];
        if ((ea >> 32) != (e >> 32)) break;
        const u32 pos_a = static_cast<u32>(ea);
        const u32 q = static_cast<u32>(__umul64hi(pos_a, period_magic));
        const u32 t_a = period - 1u - (pos_a - q * period);       // <= L: the run is in (t, pos) order
        if (t_a < static_cast<u32>(kUniK)) break;                 // only shorter suffixes before this one: not of the group
        bool ok = true;
        for (u32 c = 0; c < t_a && ok; c += 32) {
            const u64 wa = base_window(packed, static_cast<u64>(pos_a) + c);
            const u64 wb = base_window(packed, static_cast<u64>(pos_b) + c);
            const u32 nb = t_a - c < 32 ? t_a - c : 32;
            ok = ((wa ^ wb) >> (64 - 2 * nb)) == 0;
        }
        if (!ok) continue;
        cov[q] = static_cast<u8>(t_a);   // read q: every suffix with <= t_a symbols left is proven (a racing second proof is as good)
        return;
    }
}

// One thread per whole read: `list` holds the indices at which the last sort pass left them
// (EmitMultiples, radix.cuh), so nothing is swept to find them.
__global__ void __launch_bounds__(256)
link_reads_kernel(const u64* __restrict__ elems, const u32* __restrict__ list, const u32* __restrict__ count,
                  const u64* __restrict__ packed, u32 period, u64 period_magic, u8* __restrict__ cov) {
    const u64 k = *count;   // = the number of reads when the text really is uniform
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 x = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; x < k; x += stride)
        link_one_read(elems, list[x], packed, period, period_magic, cov);
}

// The sorted records become the suffix array as they stand (sa_out[i] = position of record i)
// wherever refine_elems_kernel<true> finds nothing to do; this kernel also leaves it the two
// bitmaps it decides that from: group heads (key change, or a suffix finished by the sort) and
// members that are neither the last of their group nor proven a prefix of a later member.
// Layout: a thread owns PAIRS of consecutive records (one 128-bit load, one 64-bit store), so half of
// all neighbour relations stay inside the thread and the rest are two shuffles per pair; the terminator
// distance is computed once per record and shuffled, not recomputed for both neighbours (the first form
// -- one record per lane, 64-bit shuffles of both neighbours, three divisions per record -- was bound by
// issue slots at 0.41 of the HBM peak).  Bitmaps leave as bytes: four lanes hold eight records.
constexpr int kAccRows = 4;                       // pairs per thread in flight
constexpr int kAccSpan = 64 * kAccRows;           // records per warp iteration
__global__ void __launch_bounds__(256)
accept_uniform_kernel(const u64* __restrict__ elems, u64 m, const u8* __restrict__ cov, u32 period,
                      u64 period_magic, u32* __restrict__ sa_out, u32* __restrict__ headbits,
                      u32* __restrict__ uncbits, u8* __restrict__ tileflags) {
    constexpr u32 K = kUniK;
    const unsigned lane = lane_id();
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    u8* hbytes = reinterpret_cast<u8*>(headbits);
    u8* ubytes = reinterpret_cast<u8*>(uncbits);
    auto term = [&](u32 p, u32* q) {
        *q = static_cast<u32>(__umul64hi(p, period_magic));
        return period - 1u - (p - *q * period);
    };
    for (u64 i0 = ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kAccSpan; i0 < m; i0 += warps * kAccSpan) {
        u32 ka[kAccRows], kb[kAccRows], pa[kAccRows], pb[kAccRows];
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            const u64 i = i0 + c * 64 + 2 * lane;
            ulonglong2 v = make_ulonglong2(0, 0);
            if (i + 1 < m) v = *reinterpret_cast<const ulonglong2*>(elems + i);
            else if (i < m) v.x = elems[i];
            ka[c] = static_cast<u32>(v.x >> 32); pa[c] = static_cast<u32>(v.x);
            kb[c] = static_cast<u32>(v.y >> 32); pb[c] = static_cast<u32>(v.y);
        }
        // the record before the first and after the last one of this warp's stretch
        u32 k_before = 0, t_before = 0, k_after = 0, t_after = 0, qx;
        if (lane == 0 && i0 > 0) {
            const u64 e = elems[i0 - 1];
            k_before = static_cast<u32>(e >> 32);
            t_before = term(static_cast<u32>(e), &qx);
        }
        if (lane == 31 && i0 + kAccSpan < m) {
            const u64 e = elems[i0 + kAccSpan];
            k_after = static_cast<u32>(e >> 32);
            t_after = term(static_cast<u32>(e), &qx);
        }
        u32 ta[kAccRows], tb[kAccRows], qa[kAccRows], qb[kAccRows];
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            ta[c] = term(pa[c], &qa[c]);
            tb[c] = term(pb[c], &qb[c]);
        }
        u8 cva[kAccRows], cvb[kAccRows];   // the proof bytes, gathered up front (L2-resident table)
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            const u64 i = i0 + c * 64 + 2 * lane;
            cva[c] = i < m ? __ldg(cov + qa[c]) : 0;
            cvb[c] = i + 1 < m ? __ldg(cov + qb[c]) : 0;
        }
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            const u64 i = i0 + c * 64 + 2 * lane;
            // predecessor of a: b of the lane below; successor of b: a of the lane above
            u32 kp = __shfl_up_sync(0xffffffffu, kb[c], 1), tp = __shfl_up_sync(0xffffffffu, tb[c], 1);
            u32 kn = __shfl_down_sync(0xffffffffu, ka[c], 1), tn = __shfl_down_sync(0xffffffffu, ta[c], 1);
            if (c > 0) {
                const u32 k31 = __shfl_sync(0xffffffffu, kb[c > 0 ? c - 1 : 0], 31), t31 = __shfl_sync(0xffffffffu, tb[c > 0 ? c - 1 : 0], 31);
                if (lane == 0) { kp = k31; tp = t31; }
            } else if (lane == 0) { kp = k_before; tp = t_before; }
            if (c + 1 < kAccRows) {
                const u32 k0 = __shfl_sync(0xffffffffu, ka[c + 1 < kAccRows ? c + 1 : c], 0), t0 = __shfl_sync(0xffffffffu, ta[c + 1 < kAccRows ? c + 1 : c], 0);
                if (lane == 31) { kn = k0; tn = t0; }
            } else if (lane == 31) { kn = k_after; tn = t_after; }
            const bool in_a = i < m, in_b = i + 1 < m;
            // a suffix shorter than the key is final after the sort; a group starts where the key
            // changes or right behind such a suffix
            const bool head_a = in_a && (i == 0 || ka[c] != kp || ta[c] < K || tp < K);
            const bool head_b = in_b && (kb[c] != ka[c] || tb[c] < K || ta[c] < K);
            const bool last_a = !in_b || kb[c] != ka[c] || tb[c] < K;      // (t < K: the next record is a head then, too)
            const bool last_b = i + 2 >= m || kn != kb[c] || tn < K;
            const bool unc_a = in_a && !last_a && ta[c] >= K && ta[c] > cva[c];
            const bool unc_b = in_b && !last_b && tb[c] >= K && tb[c] > cvb[c];
            if (in_b) *reinterpret_cast<uint2*>(sa_out + i) = make_uint2(pa[c], pb[c]);
            else if (in_a) sa_out[i] = pa[c];
            u32 x = (static_cast<u32>(head_a) | (static_cast<u32>(head_b) << 1) | (static_cast<u32>(unc_a) << 8) |
                     (static_cast<u32>(unc_b) << 9)) << (2 * (lane & 3));
            x |= __shfl_xor_sync(0xffffffffu, x, 1);
            x |= __shfl_xor_sync(0xffffffffu, x, 2);
            if ((lane & 3) == 0 && i < m) {
                hbytes[i >> 3] = static_cast<u8>(x);
                ubytes[i >> 3] = static_cast<u8>(x >> 8);
                if (x >> 8) {   // the group of an uncovered member starts in this refine tile or the one before
                    const u64 tile = i / kRefTile;
                    tileflags[tile] = 1;
                    if (tile) tileflags[tile - 1] = 1;
                }
            }
        }
    }
}

// The same pass with a thread owning FOUR consecutive records (two 128-bit loads, one 128-bit store of sa): three of
// every four neighbour relations stay inside the thread, a quad's neighbours cost four shuffles, its four head bits and
// four uncovered bits one more (two lanes make a byte), and the record before lane 0 / after lane 31 is re-read from
// memory by that lane instead of being passed between rows.  1.25 shuffles per record instead of 5: the pairs form spent
// 34 % of its stall samples on the shuffle queue (mio_throttle + short scoreboard, profiles/r2_ncu_full_accept.txt).
// Measured [B200, config 2]: pairs 0.657 ms, quads (W = 4) 0.613 ms, W = 8 (a whole bitmap byte per thread, no byte
// shuffle, but 128-bit loads 64 bytes apart within a warp) 0.697 ms.
// Reads whose proof is SHORT (cov[read] < thr), as a 64-bit Bloom word: bit (read mod 64) of exc[0 .. 1].  At 30x
// coverage a read's successor starts 5 bases on average, so with thr = L - 64 there are a handful of such reads (the
// last ones of the genome) among a million; a suffix with t <= thr of a read whose bit is clear is proven
// (t <= thr <= cov[read]) without looking its byte up -- 57 % of the gathers the accept pass is bound by; a set bit
// (one read in ~20 shares it by chance) only means "look it up".  With many short proofs (low coverage) every bit is
// set and every suffix gathers, as before.
constexpr u32 kCovExcMargin = 64;
__global__ void __launch_bounds__(256)
cov_exceptions_kernel(const u8* __restrict__ cov, u64 reads, u32 thr, u32* __restrict__ exc) {
    const u64 r = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < reads && cov[r] < thr) atomicOr(exc + ((r >> 5) & 1u), 1u << (r & 31u));
}

template <int W, bool EXC>
__global__ void __launch_bounds__(256, 4)
accept_uniform_quads_kernel(const u64* __restrict__ elems, u64 m, const u8* __restrict__ cov, u32 period,
                            u64 period_magic, u32* __restrict__ sa_out, u32* __restrict__ headbits,
                            u32* __restrict__ uncbits, u8* __restrict__ tileflags, const u32* __restrict__ exc, u32 thr) {
    u32 bloom0 = 0xffffffffu, bloom1 = 0xffffffffu;
    if constexpr (EXC) { bloom0 = exc[0]; bloom1 = exc[1]; }
    static_assert(W == 4 || W == 8, "four or eight consecutive records per thread");
    constexpr u32 K = kUniK;
    constexpr int R = 8 / W;                        // rows per thread in flight
    constexpr u64 kRow = 32 * W;                    // records per warp row
    constexpr u64 kSpan = kRow * R;                 // records per warp iteration
    const unsigned lane = lane_id();
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    u8* hbytes = reinterpret_cast<u8*>(headbits);
    u8* ubytes = reinterpret_cast<u8*>(uncbits);
    auto term = [&](u32 p, u32* q) {
        *q = static_cast<u32>(__umul64hi(p, period_magic));
        return period - 1u - (p - *q * period);
    };
    for (u64 i0 = ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kSpan; i0 < m; i0 += warps * kSpan) {
        u32 k[R][W], p[R][W], t[R][W], q[R][W];
        u32 kp[R], tp[R], kn[R], tn[R];             // the records around the thread's stretch
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const u64 i = i0 + c * kRow + W * lane;
#pragma unroll
            for (int h = 0; h < W / 2; ++h) {
                ulonglong2 v = make_ulonglong2(0, 0);
                if (i + 2 * h + 1 < m) v = *reinterpret_cast<const ulonglong2*>(elems + i + 2 * h);
                else if (i + 2 * h < m) v.x = elems[i + 2 * h];
                k[c][2 * h] = static_cast<u32>(v.x >> 32); p[c][2 * h] = static_cast<u32>(v.x);
                k[c][2 * h + 1] = static_cast<u32>(v.y >> 32); p[c][2 * h + 1] = static_cast<u32>(v.y);
            }
            // lane 0 / lane 31: the record before / after this row, straight from memory (a cache hit)
            u64 eb = 0, ea = 0;
            if (lane == 0 && i > 0 && i < m) eb = elems[i - 1];
            if (lane == 31 && i + W < m) ea = elems[i + W];
            u32 qx;
            kp[c] = static_cast<u32>(eb >> 32); tp[c] = term(static_cast<u32>(eb), &qx);
            kn[c] = static_cast<u32>(ea >> 32); tn[c] = term(static_cast<u32>(ea), &qx);
        }
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
            for (int j = 0; j < W; ++j) t[c][j] = term(p[c][j], &q[c][j]);
        u8 cv[R][W];   // the proof bytes, gathered up front (L2-resident table)
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const bool in = i0 + c * kRow + W * lane + j < m;
                const u32 qq = q[c][j];
                bool need = true;
                if constexpr (EXC) need = t[c][j] > thr || ((((qq & 32u) ? bloom1 : bloom0) >> (qq & 31u)) & 1u);
                cv[c][j] = in ? (need ? __ldg(cov + qq) : static_cast<u8>(255)) : 0;
            }
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const u64 i = i0 + c * kRow + W * lane;
            const u32 ku = __shfl_up_sync(0xffffffffu, k[c][W - 1], 1), tu = __shfl_up_sync(0xffffffffu, t[c][W - 1], 1);
            const u32 kd = __shfl_down_sync(0xffffffffu, k[c][0], 1), td = __shfl_down_sync(0xffffffffu, t[c][0], 1);
            if (lane != 0) { kp[c] = ku; tp[c] = tu; }
            if (lane != 31) { kn[c] = kd; tn[c] = td; }
            u32 hn = 0, un = 0;
#pragma unroll
            for (int j = 0; j < W; ++j) {
                const bool in = i + j < m;
                const u32 kprev = j ? k[c][j ? j - 1 : 0] : kp[c], tprev = j ? t[c][j ? j - 1 : 0] : tp[c];
                const u32 knext = j < W - 1 ? k[c][j < W - 1 ? j + 1 : j] : kn[c], tnext = j < W - 1 ? t[c][j < W - 1 ? j + 1 : j] : tn[c];
                // a suffix shorter than the key is final after the sort; a group starts where the key
                // changes or right behind such a suffix
                const bool head = in && (i + j == 0 || k[c][j] != kprev || t[c][j] < K || tprev < K);
                const bool last = i + j + 1 >= m || knext != k[c][j] || tnext < K;   // (t < K: the next record is a head then, too)
                const bool unc = in && !last && t[c][j] >= K && t[c][j] > cv[c][j];
                hn |= static_cast<u32>(head) << j;
                un |= static_cast<u32>(unc) << j;
            }
#pragma unroll
            for (int h = 0; h < W / 4; ++h) {
                if (i + 4 * h + 3 < m)
                    *reinterpret_cast<uint4*>(sa_out + i + 4 * h) = make_uint4(p[c][4 * h], p[c][4 * h + 1], p[c][4 * h + 2], p[c][4 * h + 3]);
                else
                    for (int j = 4 * h; j < 4 * h + 4; ++j)
                        if (i + j < m) sa_out[i + j] = p[c][j];
            }
            u32 x = hn | (un << 8);
            bool writer = true;
            if constexpr (W == 4) {   // two lanes make a byte
                x <<= 4 * (lane & 1);
                x |= __shfl_xor_sync(0xffffffffu, x, 1);
                writer = (lane & 1) == 0;
            }
            if (writer && i < m) {
                hbytes[i >> 3] = static_cast<u8>(x);
                ubytes[i >> 3] = static_cast<u8>(x >> 8);
                if ((x >> 8) & 0xffu) {   // the group of an uncovered member starts in this refine tile or the one before
                    const u64 tile = i / kRefTile;
                    tileflags[tile] = 1;
                    if (tile) tileflags[tile - 1] = 1;
                }
            }
        }
    }
}

// ---- ragged read sets: route (i) for reads of mixed lengths ------------------------------------------
//
// A read set whose reads differ in length (trimmed reads) has no period to do arithmetic with, but the
// idea of the uniform path carries over once two things are looked up instead of computed:
//   * which read a position belongs to and how far its sentinel is: the sentinel bitmap with a count
//     of separators before every 64-position word (`cum`) gives the read id, `ends[id]` the sentinel;
//   * the order the records are born in: (terminator distance t, position) is a TRANSPOSITION WITH
//     RAGGED ROWS -- record slot = (suffixes with a smaller t) + (reads before this one that are at least
//     t long) -- made by the count / scan / write compaction of the multi-GPU bucket generator, keeping
//     "t <= length of the read".
// Records: key32 << 32 | position, key32 = first 15 bases (zero padded from the sentinel on) << 2 | tag,
// tag = 0 for a suffix of fewer than 15 symbols (final after the sort, like the uniform path's t < 16),
// 1 otherwise: the accept pass needs no terminator distance at all.  Proofs are one bit per POSITION
// (n/8 bytes, L2-resident at config 2) set by link_ragged_kernel for the suffixes of a read from the
// verified offset on.  Reads longer than 254 bases, texts that do not end in a separator: route (ii).
constexpr u32 kRagMaxLen = 254;
constexpr int kRagReads = 256;      // reads per CTA of the record generator; thread = read

__global__ void __launch_bounds__(256)
sent_popc_kernel(const u64* __restrict__ sent, u64 words, u32* __restrict__ out) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 w = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) out[w] = __popcll(sent[w]);
}

// ends[r] = position of the r-th separator; maxgap = longest read.
__global__ void __launch_bounds__(256)
ends_kernel(const u64* __restrict__ sent, const u32* __restrict__ cum, u64 words, u32* __restrict__ ends) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 w = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; w < words; w += stride) {
        u64 bits = sent[w];
        u32 at = cum[w];
        while (bits) {
            const int lz = __clzll(bits);              // position w * 64 + lz
            ends[at++] = static_cast<u32>((w << 6) + lz);
            bits &= ~(1ull << (63 - lz));
        }
    }
}
__global__ void __launch_bounds__(256)
maxlen_kernel(const u32* __restrict__ ends, u64 k, u32* __restrict__ out) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    u32 mx = 0;
    for (u64 r = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; r < k; r += stride)
        mx = max(mx, ends[r] - (r ? ends[r - 1] + 1u : 0u));
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane_id() == 0 && mx) atomicMax(out, mx);
}

// Calls f(t, key32, active) for t = tmax down to 0; active: the read has a suffix with t symbols before
// its sentinel (t <= len).  The trip count is the same for every lane (f may vote).
template <class F>
__device__ __forceinline__ void for_each_suffix_ragged(const u64* __restrict__ s_w, u32 bit0, u32 len, u32 tmax, F f) {
    // The read's suffixes come in offset order (t falls, the offset len - t rises), so the 15-base key comes from a
    // window that slides two bits per suffix; it is refilled at the read's first suffix and wherever t = 15 mod 16 (the
    // same trips for every lane), instead of two shared-memory words and a funnel shift per suffix.
    u64 win = 0;
    for (int t = static_cast<int>(tmax); t >= 0; --t) {
        const bool active = static_cast<u32>(t) <= len;
        u32 key = 0;
        if (active) {
            if ((t & 15) == 15 || static_cast<u32>(t) == len) {
                const u32 bit = bit0 + 2 * (len - t);
                const u32 wi = bit >> 6, sh = bit & 63;
                const u64 hi = s_w[wi], lo = s_w[wi + 1];
                win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
            }
            u32 b15 = static_cast<u32>(win >> 34);                                        // 15 bases
            win <<= 2;
            if (t < kRagK) b15 = t ? b15 & ~((1u << (2 * (kRagK - t))) - 1u) : 0u;        // zero padded from the sentinel on
            key = (b15 << 2) | (t >= kRagK ? 1u : 0u);
        }
        f(static_cast<u32>(t), key, active);
    }
}

// Stages the packed text of reads [r0, r0 + nr) (contiguous: from the first read's start to the last
// read's sentinel); per thread: bit offset of its read in the staged words and its length.
__device__ __forceinline__ void stage_ragged(const u64* __restrict__ packed, const u32* __restrict__ ends, u64* __restrict__ s_w,
                                             u64 r0, u32 nr, u32* my_bit0, u32* my_len, u64* my_start) {
    __shared__ __align__(8) u64 s_bar;
    const u64 base0 = r0 ? static_cast<u64>(ends[r0 - 1]) + 1 : 0;
    const u64 end0 = static_cast<u64>(ends[r0 + nr - 1]) + 1;
    const u64 w0 = (base0 >> 5) & ~1ull;
    const u32 nw = (static_cast<u32>(((end0 + 31) >> 5) - w0) + 3u) & ~1u;
    if (threadIdx.x == 0) mbar_init(&s_bar, 1);
    __syncwarp();   // (racecheck attributes the barrier's initialisation to the warp, not to its lane 0)
    if (threadIdx.x == 0) {
        mbar_expect_tx(&s_bar, nw * 8u);
        tma_load_1d(s_w, packed + w0, nw * 8u, &s_bar);
    }
    const bool in = threadIdx.x < nr;
    const u64 r = r0 + (in ? threadIdx.x : 0u);
    const u64 st = r ? static_cast<u64>(ends[r - 1]) + 1 : 0;
    *my_start = st;
    *my_len = in ? ends[r] - static_cast<u32>(st) : 0u;
    *my_bit0 = 2 * static_cast<u32>(st - (w0 << 5));
    __syncthreads();
    mbar_wait(&s_bar, 0);
}

__global__ void __launch_bounds__(kRagReads)
ragged_count_kernel(const u64* __restrict__ packed, const u32* __restrict__ ends, u64 k, u32 tiles, u32 tmax,
                    u32* __restrict__ counts) {
    __shared__ __align__(16) u64 s_w[kRagReads * (kRagMaxLen + 1) / 32 + 8];
    __shared__ u32 s_cnt[kRagMaxLen + 2];
    for (int i = threadIdx.x; i < static_cast<int>(kRagMaxLen) + 2; i += blockDim.x) s_cnt[i] = 0;
    const u64 r0 = static_cast<u64>(blockIdx.x) * kRagReads;
    const u32 nr = static_cast<u32>(k - r0 < kRagReads ? k - r0 : kRagReads);
    u32 bit0, len;
    u64 st;
    stage_ragged(packed, ends, s_w, r0, nr, &bit0, &len, &st);
    const bool in = threadIdx.x < nr;
    // no key is needed to count: a read of length len has one suffix for every t <= len
    for (int t = static_cast<int>(tmax); t >= 0; --t) {
        const unsigned b = __ballot_sync(0xffffffffu, in && static_cast<u32>(t) <= len);
        if (b && lane_id() == 0) atomicAdd(&s_cnt[t], __popc(b));
    }
    __syncthreads();
    for (u32 t = threadIdx.x; t <= tmax; t += blockDim.x) counts[static_cast<u64>(t) * tiles + blockIdx.x] = s_cnt[t];
}

__global__ void __launch_bounds__(kRagReads)
ragged_write_kernel(const u64* __restrict__ packed, const u32* __restrict__ ends, u64 k, u32 tiles, u32 tmax,
                    const u32* __restrict__ offsets, u64* __restrict__ out, u32* __restrict__ g_hist) {
    __shared__ __align__(16) u64 s_w[kRagReads * (kRagMaxLen + 1) / 32 + 8];
    __shared__ unsigned short s_wcnt[kRagReads / 32][kRagMaxLen + 2];
    __shared__ u32 s_hist[4 * kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) s_hist[i] = 0;
    const u64 r0 = static_cast<u64>(blockIdx.x) * kRagReads;
    const u32 nr = static_cast<u32>(k - r0 < kRagReads ? k - r0 : kRagReads);
    u32 bit0, len;
    u64 st;
    stage_ragged(packed, ends, s_w, r0, nr, &bit0, &len, &st);
    const bool in = threadIdx.x < nr;
    const int warp = threadIdx.x >> 5;
    for (int t = static_cast<int>(tmax); t >= 0; --t) {
        const unsigned b = __ballot_sync(0xffffffffu, in && static_cast<u32>(t) <= len);
        if (lane_id() == 0) s_wcnt[warp][t] = static_cast<unsigned short>(__popc(b));
    }
    __syncthreads();
    for (u32 t = threadIdx.x; t <= tmax; t += blockDim.x) {
        u32 run = 0;
        for (int w = 0; w < kRagReads / 32; ++w) {
            const u32 c = s_wcnt[w][t];
            s_wcnt[w][t] = static_cast<unsigned short>(run);
            run += c;
        }
    }
    __syncthreads();
    for_each_suffix_ragged(s_w, bit0, in ? len : 0u, tmax, [&](u32 t, u32 key, bool active) {
        const bool keep = in && active;
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const u64 slot = static_cast<u64>(offsets[static_cast<u64>(t) * tiles + blockIdx.x]) + s_wcnt[warp][t] +
                             __popc(b & lanemask_lt());
            out[slot] = (static_cast<u64>(key) << 32) | (st + (len - t));
            atomicAdd(&s_hist[key & 0xffu], 1u);
            atomicAdd(&s_hist[kRadix + ((key >> 8) & 0xffu)], 1u);
            atomicAdd(&s_hist[2 * kRadix + ((key >> 16) & 0xffu)], 1u);
            atomicAdd(&s_hist[3 * kRadix + (key >> 24)], 1u);
        }
    });
    __syncthreads();
    hist_flush(s_hist, g_hist, 4);
}

// One thread per whole read (their sorted indices come from the last digit pass, EmitStarts).  Two links:
//   * backward, as in the uniform path: the nearest predecessor a of the read's first suffix b in its group
//     is compared with b over its whole length t_a; if equal, every suffix of a's read from a on is a prefix
//     of the suffix the same distance into b -- a later member of its own group;
//   * forward, which only ragged sets need: a whole read is the LAST of its group when all reads are equally
//     long, but a longer read that started earlier and ends later comes after it.  b is compared over its
//     whole length with its successor s; if equal, every suffix of b is a prefix of the suffix the same
//     distance further into s.
// Together they reach every member that has a successor from the same locus: take (read q, locus g) and its
// successor s in the group of g.  No read covering g ends between them, so if s starts at or after q's
// start, q is the predecessor of whole s in the group of s's start (backward link of s); if s starts before,
// s is the successor of whole q in the group of q's start (forward link of q).
__global__ void __launch_bounds__(256)
link_ragged_kernel(const u64* __restrict__ elems, u64 m, const u32* __restrict__ list, const u32* __restrict__ count,
                   const u64* __restrict__ packed, const u64* __restrict__ sent, const u32* __restrict__ cum,
                   const u32* __restrict__ ends, u32* __restrict__ covbits) {
    const u64 k = *count;
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    auto mark = [&](u32 first, u32 len) {   // positions [first, first + len): a handful of words
        const u32 last = first + len - 1;
        for (u32 ww = first >> 5; ww <= (last >> 5); ++ww) {
            u32 mk = 0xffffffffu;
            if (ww == (first >> 5)) mk &= 0xffffffffu << (first & 31u);
            if (ww == (last >> 5)) mk &= 0xffffffffu >> (31u - (last & 31u));
            atomicOr(covbits + ww, mk);
        }
    };
    for (u64 x = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; x < k; x += stride) {
        const u64 i = list[x];
        const u64 e = elems[i];
        if ((static_cast<u32>(e >> 32) & 3u) == 0) continue;      // a read shorter than the key: final after the sort
        const u32 pos_b = static_cast<u32>(e);
        for (u64 s = 1; s <= 16 && s <= i; ++s) {
            const u64 ea = elems[i - s];
            if ((ea >> 32) != (e >> 32)) break;
            const u32 pos_a = static_cast<u32>(ea);
            const u32 w = pos_a >> 6, bb = pos_a & 63u;
            const u32 q = cum[w] + (bb ? static_cast<u32>(__popcll(sent[w] >> (64 - bb))) : 0u);
            const u32 t_a = ends[q] - pos_a;                       // >= 15 (same tag), <= t_b (the run is in (t, pos) order)
            bool ok = true;
            for (u32 c = 0; c < t_a && ok; c += 32) {
                const u64 wa = base_window(packed, static_cast<u64>(pos_a) + c);
                const u64 wb = base_window(packed, static_cast<u64>(pos_b) + c);
                const u32 nb = t_a - c < 32 ? t_a - c : 32;
                ok = ((wa ^ wb) >> (64 - 2 * nb)) == 0;
            }
            if (!ok) continue;
            mark(pos_a, t_a);
            break;
        }
        // forward link
        const u32 wb0 = pos_b >> 6, bb0 = pos_b & 63u;
        const u32 q_b = cum[wb0] + (bb0 ? static_cast<u32>(__popcll(sent[wb0] >> (64 - bb0))) : 0u);
        const u32 t_b = ends[q_b] - pos_b;
        for (u64 s = 1; s <= 16 && i + s < m; ++s) {
            const u64 es = elems[i + s];
            if ((es >> 32) != (e >> 32)) break;
            const u32 pos_s = static_cast<u32>(es);
            bool ok = true;
            for (u32 c = 0; c < t_b && ok; c += 32) {
                const u64 wa = base_window(packed, static_cast<u64>(pos_b) + c);
                const u64 ws = base_window(packed, static_cast<u64>(pos_s) + c);
                const u32 nb = t_b - c < 32 ? t_b - c : 32;
                ok = ((wa ^ ws) >> (64 - 2 * nb)) == 0;
            }
            // (a successor shorter than t_b symbols cannot pass: its sentinel packs as a base code, but the
            //  records are in (t, position) order, so every successor has at least t_b symbols)
            if (!ok) continue;
            mark(pos_b, t_b);
            break;
        }
    }
}

// accept_uniform_kernel for ragged records: "shorter than the key" is the record's tag, the proof a bit
// per position.  Same pair layout, same outputs.
__global__ void __launch_bounds__(256)
accept_ragged_kernel(const u64* __restrict__ elems, u64 m, const u32* __restrict__ covbits, u32* __restrict__ sa_out,
                     u32* __restrict__ headbits, u32* __restrict__ uncbits, u8* __restrict__ tileflags) {
    const unsigned lane = lane_id();
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    u8* hbytes = reinterpret_cast<u8*>(headbits);
    u8* ubytes = reinterpret_cast<u8*>(uncbits);
    for (u64 i0 = ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kAccSpan; i0 < m; i0 += warps * kAccSpan) {
        u32 ka[kAccRows], kb[kAccRows], pa[kAccRows], pb[kAccRows];
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            const u64 i = i0 + c * 64 + 2 * lane;
            ulonglong2 v = make_ulonglong2(0, 0);
            if (i + 1 < m) v = *reinterpret_cast<const ulonglong2*>(elems + i);
            else if (i < m) v.x = elems[i];
            ka[c] = static_cast<u32>(v.x >> 32); pa[c] = static_cast<u32>(v.x);
            kb[c] = static_cast<u32>(v.y >> 32); pb[c] = static_cast<u32>(v.y);
        }
        u32 k_before = 0, k_after = 0;
        if (lane == 0 && i0 > 0) k_before = static_cast<u32>(elems[i0 - 1] >> 32);
        if (lane == 31 && i0 + kAccSpan < m) k_after = static_cast<u32>(elems[i0 + kAccSpan] >> 32);
        u32 ca[kAccRows], cb[kAccRows];   // the proof bits, gathered up front
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            const u64 i = i0 + c * 64 + 2 * lane;
            ca[c] = i < m ? (__ldg(covbits + (pa[c] >> 5)) >> (pa[c] & 31u)) & 1u : 0u;
            cb[c] = i + 1 < m ? (__ldg(covbits + (pb[c] >> 5)) >> (pb[c] & 31u)) & 1u : 0u;
        }
#pragma unroll
        for (int c = 0; c < kAccRows; ++c) {
            const u64 i = i0 + c * 64 + 2 * lane;
            u32 kp = __shfl_up_sync(0xffffffffu, kb[c], 1);
            u32 kn = __shfl_down_sync(0xffffffffu, ka[c], 1);
            if (c > 0) {
                const u32 k31 = __shfl_sync(0xffffffffu, kb[c > 0 ? c - 1 : 0], 31);
                if (lane == 0) kp = k31;
            } else if (lane == 0) kp = k_before;
            if (c + 1 < kAccRows) {
                const u32 k0 = __shfl_sync(0xffffffffu, ka[c + 1 < kAccRows ? c + 1 : c], 0);
                if (lane == 31) kn = k0;
            } else if (lane == 31) kn = k_after;
            const bool in_a = i < m, in_b = i + 1 < m;
            const bool short_a = (ka[c] & 3u) == 0, short_b = (kb[c] & 3u) == 0;
            // (equal keys carry equal tags: "the neighbour is short" needs no test of its own)
            const bool head_a = in_a && (i == 0 || ka[c] != kp || short_a);
            const bool head_b = in_b && (kb[c] != ka[c] || short_b);
            const bool last_a = !in_b || kb[c] != ka[c] || short_b;
            const bool last_b = i + 2 >= m || kn != kb[c] || short_b;
            const bool unc_a = in_a && !last_a && !short_a && !ca[c];
            const bool unc_b = in_b && !last_b && !short_b && !cb[c];
            if (in_b) *reinterpret_cast<uint2*>(sa_out + i) = make_uint2(pa[c], pb[c]);
            else if (in_a) sa_out[i] = pa[c];
            u32 x = (static_cast<u32>(head_a) | (static_cast<u32>(head_b) << 1) | (static_cast<u32>(unc_a) << 8) |
                     (static_cast<u32>(unc_b) << 9)) << (2 * (lane & 3));
            x |= __shfl_xor_sync(0xffffffffu, x, 1);
            x |= __shfl_xor_sync(0xffffffffu, x, 2);
            if ((lane & 3) == 0 && i < m) {
                hbytes[i >> 3] = static_cast<u8>(x);
                ubytes[i >> 3] = static_cast<u8>(x >> 8);
                if (x >> 8) {
                    const u64 tile = i / kRefTile;
                    tileflags[tile] = 1;
                    if (tile) tileflags[tile - 1] = 1;
                }
            }
        }
    }
}

// The same pass with a thread owning four consecutive records (see accept_uniform_quads_kernel): three of four
// neighbour relations stay in registers, a quad's outer neighbours cost two shuffles, its eight flag bits one.
__global__ void __launch_bounds__(256)
accept_ragged_quads_kernel(const u64* __restrict__ elems, u64 m, const u32* __restrict__ covbits, u32* __restrict__ sa_out,
                           u32* __restrict__ headbits, u32* __restrict__ uncbits, u8* __restrict__ tileflags) {
    constexpr int R = 2;
    constexpr u64 kRow = 128, kSpan = kRow * R;
    const unsigned lane = lane_id();
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    u8* hbytes = reinterpret_cast<u8*>(headbits);
    u8* ubytes = reinterpret_cast<u8*>(uncbits);
    for (u64 i0 = ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * kSpan; i0 < m; i0 += warps * kSpan) {
        u32 k[R][4], p[R][4], kp[R], kn[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const u64 i = i0 + c * kRow + 4 * lane;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                ulonglong2 v = make_ulonglong2(0, 0);
                if (i + 2 * h + 1 < m) v = *reinterpret_cast<const ulonglong2*>(elems + i + 2 * h);
                else if (i + 2 * h < m) v.x = elems[i + 2 * h];
                k[c][2 * h] = static_cast<u32>(v.x >> 32); p[c][2 * h] = static_cast<u32>(v.x);
                k[c][2 * h + 1] = static_cast<u32>(v.y >> 32); p[c][2 * h + 1] = static_cast<u32>(v.y);
            }
            kp[c] = 0; kn[c] = 0;
            if (lane == 0 && i > 0 && i < m) kp[c] = static_cast<u32>(elems[i - 1] >> 32);
            if (lane == 31 && i + 4 < m) kn[c] = static_cast<u32>(elems[i + 4] >> 32);
        }
        u32 cb[R][4];   // the proof bits, gathered up front
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                cb[c][j] = i0 + c * kRow + 4 * lane + j < m ? (__ldg(covbits + (p[c][j] >> 5)) >> (p[c][j] & 31u)) & 1u : 0u;
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const u64 i = i0 + c * kRow + 4 * lane;
            const u32 ku = __shfl_up_sync(0xffffffffu, k[c][3], 1), kd = __shfl_down_sync(0xffffffffu, k[c][0], 1);
            if (lane != 0) kp[c] = ku;
            if (lane != 31) kn[c] = kd;
            u32 hn = 0, un = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool in = i + j < m;
                const u32 kprev = j ? k[c][j ? j - 1 : 0] : kp[c], knext = j < 3 ? k[c][j < 3 ? j + 1 : j] : kn[c];
                const bool shrt = (k[c][j] & 3u) == 0;
                // (equal keys carry equal tags: "the neighbour is short" needs no test of its own)
                const bool head = in && (i + j == 0 || k[c][j] != kprev || shrt);
                const bool last = i + j + 1 >= m || knext != k[c][j] || shrt;
                const bool unc = in && !last && !shrt && !cb[c][j];
                hn |= static_cast<u32>(head) << j;
                un |= static_cast<u32>(unc) << j;
            }
            if (i + 3 < m) *reinterpret_cast<uint4*>(sa_out + i) = make_uint4(p[c][0], p[c][1], p[c][2], p[c][3]);
            else
                for (int j = 0; j < 4; ++j)
                    if (i + j < m) sa_out[i + j] = p[c][j];
            u32 x = (hn | (un << 8)) << (4 * (lane & 1));
            x |= __shfl_xor_sync(0xffffffffu, x, 1);
            if ((lane & 1) == 0 && i < m) {
                hbytes[i >> 3] = static_cast<u8>(x);
                ubytes[i >> 3] = static_cast<u8>(x >> 8);
                if ((x >> 8) & 0xffu) {
                    const u64 tile = i / kRefTile;
                    tileflags[tile] = 1;
                    if (tile) tileflags[tile - 1] = 1;
                }
            }
        }
    }
}

// rank = inverse permutation of sa.  A direct scatter rank[sa[i]] = i is n random 4-byte
// writes, each a DRAM read-modify-write of a whole sector (measured 5.9 ms at n = 139 M).
// Instead the (sa[i] << 32 | i) records are first partitioned by the top bits of sa[i] -- two
// streaming onesweep passes -- so that consecutive records target one small window of rank,
// which is then scattered in shared memory and written as whole lines.
// After the partition passes every aligned window of 2^win_bits rank entries has all of its
// (pos << 32 | idx) records in the same index range of the record array (sa is a permutation, so
// the buckets are exactly window-sized).  One CTA per window: scatter in shared memory, store the
// window with full-width coalesced writes -- 139 M single-sector L2 write transactions become
// 4.3 M full lines.
__global__ void __launch_bounds__(512)
window_scatter_kernel(const u64* __restrict__ rec, u64 n, int win_bits, u32* __restrict__ rank) {
    extern __shared__ u32 s_win[];
    const u64 base = static_cast<u64>(blockIdx.x) << win_bits;
    const u32 size = static_cast<u32>(n - base < (1ull << win_bits) ? n - base : (1ull << win_bits));
    const u32 mask = (1u << win_bits) - 1u;
    // 8 records per thread in flight (two per 128-bit load): the kernel is all load latency otherwise
    // (ncu: 81 % of stalls on the load scoreboard at 97 % occupancy with one record per thread)
    const ulonglong2* rec2 = reinterpret_cast<const ulonglong2*>(rec + base);   // base is a multiple of 2^win_bits
    const u32 pairs = size >> 1;
    for (u32 t0 = threadIdx.x; t0 < pairs; t0 += 4 * blockDim.x) {
        ulonglong2 v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const u32 t = t0 + c * blockDim.x;
            v[c] = t < pairs ? rec2[t] : make_ulonglong2(0, 0);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const u32 t = t0 + c * blockDim.x;
            if (t < pairs) {
                s_win[static_cast<u32>(v[c].x >> 32) & mask] = static_cast<u32>(v[c].x);
                s_win[static_cast<u32>(v[c].y >> 32) & mask] = static_cast<u32>(v[c].y);
            }
        }
    }
    if ((size & 1) && threadIdx.x == 0) {
        const u64 r = rec[base + size - 1];
        s_win[static_cast<u32>(r >> 32) & mask] = static_cast<u32>(r);
    }
    // (Measured and dropped: the window leaving as ONE TMA bulk store issued by an elected thread --
    //  cp.async.bulk.global.shared::cta, 32 KB -- ran at 0.269 ms against 0.242 for the 128-bit stores
    //  of all 512 threads below: the CTA ends on the copy engine's read of the window instead of
    //  overlapping its stores with the next CTA's loads.  profiles/r2_negative_results.md.)
    __syncthreads();
    if ((reinterpret_cast<uintptr_t>(rank) & 15) == 0) {   // the caller's array may be aligned to 4 bytes only
        uint4* out4 = reinterpret_cast<uint4*>(rank + base);
        const uint4* win4 = reinterpret_cast<const uint4*>(s_win);
        for (u32 t = threadIdx.x; t < (size >> 2); t += blockDim.x) out4[t] = win4[t];
        for (u32 t = (size & ~3u) + threadIdx.x; t < size; t += blockDim.x) rank[base + t] = s_win[t];
    } else {
        for (u32 t = threadIdx.x; t < size; t += blockDim.x) rank[base + t] = s_win[t];
    }
}

// ---- inverse permutation, lean partition passes ---------------------------------------------------
// The partition that feeds window_scatter_kernel need not be stable, and because sa is a
// permutation every bucket (positions sharing their top bits) has a size and a base known in
// closed form.  So a pass needs neither the ballot ranking nor the look-back chain of the sort: a
// record takes its slot in the tile's bin from ONE shared-memory atomicAdd, a bin claims its
// stretch of the bucket with one global atomicAdd, and the tile leaves through shared memory as
// one contiguous run per bin.  Measured on B200 the sort pass is bound by issue slots and
// shared-memory wavefronts (the SM-to-HBM ratio is half an A100's), which is what this sheds.
//
// kIpSa: element i of the input is (sa[i] << 32) | i.  kIpRec: records of the previous pass.
enum : int { kIpSa = 1, kIpRec = 2, kIpRec0 = 3, kIpSaVal = 4 };   // kIpSaVal: element i is (sa[i] << 32) | vals[i]   // kIpRec0: records in no particular order (first pass of a slice)
constexpr int kIpBlock = 512;
constexpr int kIpItems = 8;
constexpr int kIpTile = kIpBlock * kIpItems;
constexpr int kIpMaxBins = 1024;

// Persistent: two CTAs per SM walk tiles blockIdx.x, blockIdx.x + gridDim.x, ... (no order
// between tiles is needed).  The loads of the next tile are issued before the current one is
// scanned, exchanged and stored, and the claims before the exchange, so the HBM latency of the
// load and the L2 latency of the atomics are covered by the tile's own work (one tile per CTA:
// 0.68 ms per pass at n = 139 M, 55 % of stalls on those two scoreboards; this form: 0.48 ms).
constexpr int kIpClaimStride = 32;   // words between first-pass claim counters: one per 128-byte line
template <int MODE>
__global__ void __launch_bounds__(kIpBlock, 2)
inv_partition_persistent_kernel(const void* __restrict__ in_raw, u64 n, int shift, int prev_shift, int nbins,
                                u32* __restrict__ claim, u64* __restrict__ out, u32 num_tiles,
                                const u32* __restrict__ vals = nullptr) {
    // First passes: every tile claims from the same `nbins` counters; packed, they sit in a handful of cache lines -- a
    // handful of L2 slices -- whose atomic units then bound the pass (~8 G claims/s: 0.31 of the HBM peak with 193 - 360
    // bins).  One counter per 128-byte line spreads them over the slices.  (Second passes claim from bucket x bin
    // counters: already spread.)  Measured and dropped in favour of this: counters replicated eight times per bin with
    // sized stretches of each bucket (13.1 ms against 12.0 at 3 G records; profiles/r2_negative_results.md).
    constexpr u32 CS = MODE == kIpRec ? 1u : static_cast<u32>(kIpClaimStride);
    __shared__ __align__(16) u64 s_rec[kIpTile];
    __shared__ u32 s_cnt[kIpMaxBins];
    __shared__ u32 s_ofs[kIpMaxBins];
    __shared__ u32 s_gdst[kIpMaxBins];
    __shared__ u32 s_warp[kIpBlock / 32];
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    auto load_tile = [&](u32 tile, u64 (&r)[kIpItems]) {
        const u64 tb = static_cast<u64>(tile) * kIpTile;
#pragma unroll
        for (int j = 0; j < kIpItems; ++j) {
            const u64 i = tb + static_cast<u64>(j) * kIpBlock + tid;
            if constexpr (MODE == kIpSa)
                r[j] = i < n ? (static_cast<u64>(static_cast<const u32*>(in_raw)[i]) << 32) | (i & 0xffffffffu) : 0;
            else if constexpr (MODE == kIpSaVal)
                r[j] = i < n ? (static_cast<u64>(static_cast<const u32*>(in_raw)[i]) << 32) | vals[i] : 0;
            else
                r[j] = i < n ? static_cast<const u64*>(in_raw)[i] : 0;
        }
    };
    u64 rec[kIpItems], nxt[kIpItems];
    if (blockIdx.x < num_tiles) load_tile(blockIdx.x, rec);
    for (int b = tid; b < nbins; b += kIpBlock) s_cnt[b] = 0;
    __syncthreads();
    for (u32 tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const u64 tile_base = static_cast<u64>(tile) * kIpTile;
        const u32 valid = static_cast<u32>(n - tile_base < static_cast<u64>(kIpTile) ? n - tile_base : kIpTile);
        const u32 bin0 = MODE == kIpRec ? static_cast<u32>(tile_base >> prev_shift) << (prev_shift - shift) : 0u;   // kIpSa, kIpRec0: 0
        u32 slot[kIpItems];
#pragma unroll
        for (int j = 0; j < kIpItems; ++j) {
            const u32 li = static_cast<u32>(j) * kIpBlock + tid;
            slot[j] = 0;
            if (li < valid) slot[j] = atomicAdd(&s_cnt[(static_cast<u32>(rec[j] >> 32) >> shift) - bin0], 1u);
        }
        if (tile + gridDim.x < num_tiles) load_tile(tile + gridDim.x, nxt);   // in flight until the end of this tile
        __syncthreads();
        const int b0 = 2 * tid, b1 = 2 * tid + 1;
        const u32 c0 = b0 < nbins ? s_cnt[b0] : 0u, c1 = b1 < nbins ? s_cnt[b1] : 0u;
        u32 g0 = 0, g1 = 0;   // claims are issued now, consumed after the exchange
        if (c0) g0 = atomicAdd(claim + (bin0 + b0) * CS, c0);
        if (c1) g1 = atomicAdd(claim + (bin0 + b1) * CS, c1);
        u32 inc = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
            if (static_cast<int>(lane) >= o) inc += t;
        }
        if (lane == 31) s_warp[tid >> 5] = inc;
        __syncthreads();
        u32 before = 0;
#pragma unroll
        for (int w = 0; w < kIpBlock / 32; ++w) before += w < (tid >> 5) ? s_warp[w] : 0u;
        const u32 excl = before + inc - (c0 + c1);
        if (b0 < nbins) { s_ofs[b0] = excl; s_cnt[b0] = 0; }
        if (b1 < nbins) { s_ofs[b1] = excl + c0; s_cnt[b1] = 0; }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kIpItems; ++j) {
            const u32 li = static_cast<u32>(j) * kIpBlock + tid;
            if (li < valid) s_rec[s_ofs[(static_cast<u32>(rec[j] >> 32) >> shift) - bin0] + slot[j]] = rec[j];
        }
        if (c0) s_gdst[b0] = ((bin0 + b0) << shift) + g0 - excl;
        if (c1) s_gdst[b1] = ((bin0 + b1) << shift) + g1 - (excl + c0);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kIpItems; ++j) {
            const u32 p = static_cast<u32>(j) * kIpBlock + tid;
            if (p < valid) {
                const u64 r = s_rec[p];
                out[s_gdst[(static_cast<u32>(r >> 32) >> shift) - bin0] + p] = r;
            }
        }
#pragma unroll
        for (int j = 0; j < kIpItems; ++j) rec[j] = nxt[j];
        __syncthreads();   // s_rec / s_gdst are rewritten by the next tile
    }
}

__global__ void inverse_kernel(const u32* __restrict__ sa, u64 n, u32* __restrict__ rank) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        rank[sa[i]] = static_cast<u32>(i);
}

// Second half of the inverse after ONE partition pass: consecutive records now target one window of
// rank (2^shift1 entries: 0.5 - 16 MB), and the CTAs in flight at any time are working on a handful of
// neighbouring windows -- tens of MB, inside the 126 MB L2.  The 4-byte stores therefore meet in L2 and
// leave for HBM as whole lines; no second partition pass, no shared-memory window.  (The direct scatter
// of the unpartitioned array spreads over 4n bytes >> L2 and runs at 24 G stores/s.)
__global__ void __launch_bounds__(256)
bucket_scatter_kernel(const u64* __restrict__ rec, u64 n, u32* __restrict__ rank) {
    const u64 pairs = n >> 1;
    const ulonglong2* rec2 = reinterpret_cast<const ulonglong2*>(rec);
    constexpr int kPer = 4;
    for (u64 t0 = (static_cast<u64>(blockIdx.x) * kPer) * blockDim.x + threadIdx.x; t0 < pairs;
         t0 += static_cast<u64>(gridDim.x) * kPer * blockDim.x) {
        ulonglong2 v[kPer];
#pragma unroll
        for (int c = 0; c < kPer; ++c) {
            const u64 t = t0 + static_cast<u64>(c) * blockDim.x;
            v[c] = t < pairs ? rec2[t] : make_ulonglong2(~0ull, ~0ull);
        }
#pragma unroll
        for (int c = 0; c < kPer; ++c) {
            const u64 t = t0 + static_cast<u64>(c) * blockDim.x;
            if (t < pairs) {
                rank[v[c].x >> 32] = static_cast<u32>(v[c].x);
                rank[v[c].y >> 32] = static_cast<u32>(v[c].y);
            }
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) rank[rec[n - 1] >> 32] = static_cast<u32>(rec[n - 1]);
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

// ---- doubling round, local form -----------------------------------------------------------------------
// A doubling round re-sorts every group (suffixes equal on their first h symbols, contiguous in sa) by
// the rank of the suffix h further on (suffix_array.hpp:93-99).  The global form sorts (group, rank2)
// pairs of ALL suffixes with 7 digit passes.  But groups are small where the text is a read set (the
// reads over one locus), so each CTA takes the groups that start in its 2048-suffix tile, gathers their
// rank2 keys, orders every group in shared memory by counting smaller keys, and writes sa and the new
// group-head index of its slots once.  rank itself is rewritten afterwards by the partitioned scatter
// (rank_update_device).  A group that outgrows the window is left as it is and reported; the host then
// runs the global form of the same round on top (a refinement of a refinement: order-independent).
constexpr int kDblBlock = 256;
constexpr int kDblTile = 2048;
constexpr int kDblExt = 640;
constexpr int kDblCap = kDblTile + kDblExt;
constexpr int kDblWords = kDblCap / 32 + 2;

__global__ void __launch_bounds__(kDblBlock)
double_local_kernel(u32* __restrict__ sa, const u32* __restrict__ head_of, const u32* __restrict__ rank, u64 n, u64 h,
                    u32* __restrict__ head_new, u32* __restrict__ counters) {
    __shared__ u64 s_key[kDblCap];       // (rank2 << 12) | slot of a tied suffix
    __shared__ u32 s_pos[kDblCap];       // positions in the old order
    __shared__ u32 s_pos2[kDblCap];      // ... in the new order
    __shared__ u32 s_k2[kDblCap];        // rank2 in the new order
    __shared__ u32 s_bits[kDblWords];    // group heads of the window
    __shared__ u32 s_new[kDblWords];
    __shared__ int s_first, s_end, s_last;
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const u64 t0 = static_cast<u64>(blockIdx.x) * kDblTile;
    const int lim = static_cast<int>(n - t0 < static_cast<u64>(kDblTile) ? n - t0 : kDblTile);
    const int avail = static_cast<int>(n - t0 < static_cast<u64>(kDblCap) ? n - t0 : kDblCap);
    if (tid == 0) { s_first = 0x7fffffff; s_end = 0x7fffffff; s_last = -1; }
    for (int j = tid; j < kDblWords; j += kDblBlock) { s_bits[j] = 0; s_new[j] = 0; }
    __syncthreads();
    // -- heads of the tile and of the stretch behind it (grown only while the tile's last group has not ended)
    int loaded = 0;
    for (int want = lim + kDblBlock < avail ? lim + kDblBlock : avail;;) {
        for (int j0 = loaded - (loaded & 31); j0 < want; j0 += kDblBlock) {
            const int j = j0 + tid;
            const bool head = j >= loaded && j < want && head_of[t0 + j] == static_cast<u32>(t0 + j);
            const unsigned b = __ballot_sync(0xffffffffu, head);
            if (lane == 0 && b) atomicOr(&s_bits[j >> 5], b);
        }
        loaded = want;
        __syncthreads();
        if (tid == 0 && loaded == static_cast<int>(n - t0) && loaded < kDblWords * 32)
            s_bits[loaded >> 5] |= 1u << (loaded & 31);   // position n acts as a head: the last group has an end
        __syncthreads();
        bool ended = false;
        for (int j = (lim >> 5) + tid; j < kDblWords; j += kDblBlock) {
            u32 w = s_bits[j];
            if (j == (lim >> 5)) w &= 0xffffffffu << (lim & 31);
            ended |= w != 0;
        }
        if (__syncthreads_or(ended) || loaded >= avail) break;
        want = loaded + kDblBlock < avail ? loaded + kDblBlock : avail;
    }
    for (int j = tid; j < kDblWords; j += kDblBlock) {
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
    const bool headless = first == 0x7fffffff;
    // Slots in front of the tile's first head belong to a group that started in an earlier tile.  Its
    // owner re-sorts them if the whole group fits its window; otherwise nobody does, and every tile
    // copies the old group-head index of its own share of the group (the same test the owner makes).
    {
        const int pre_end = headless ? lim : first;
        if (pre_end > 0) {
            const u32 g0 = head_of[t0];
            const u64 owner_t0 = g0 - g0 % kDblTile;
            const bool ends_here = !headless || t0 + lim == n;           // else: the group runs on past this tile
            const u64 e = headless ? n : t0 + first;
            const bool owner_has_it = ends_here && ((e - owner_t0 < static_cast<u64>(kDblCap)) ||
                                                    (e == n && n - owner_t0 <= static_cast<u64>(kDblCap)));
            if (!owner_has_it)
                for (int j = tid; j < pre_end; j += kDblBlock) head_new[t0 + j] = g0;
        }
    }
    if (headless) return;
    int end = s_end;
    bool overrun = false;
    if (end == 0x7fffffff) {              // the tile's last group overruns the window: left as it is
        if (tid == 0) atomicOr(counters + 1, 1u);
        end = s_last;
        overrun = true;
    }
    auto is_head = [&](int a) { return (s_bits[a >> 5] >> (a & 31)) & 1u; };
    auto group_start = [&](int a, const u32* bits) {
        int w = a >> 5;
        u32 word = bits[w] & (0xffffffffu >> (31 - (a & 31)));
        while (!word) word = bits[--w];
        return w * 32 + 31 - __clz(word);
    };
    auto group_end = [&](int a) {
        int w = (a + 1) >> 5;
        u32 word = s_bits[w] & (0xffffffffu << ((a + 1) & 31));
        while (!word) word = s_bits[++w];
        return w * 32 + __ffs(word) - 1;
    };
    // -- keys of the tied slots (a head followed by a head is a finished suffix)
    for (int a = first + tid; a < end; a += kDblBlock) {
        const bool tied = !(is_head(a) && is_head(a + 1));
        const u32 pos = sa[t0 + a];
        s_pos[a] = pos;
        s_pos2[a] = pos;
        u32 k2 = 0;
        if (tied) {
            const u64 q = static_cast<u64>(pos) + h;
            k2 = q < n ? rank[q] + 1u : 0u;       // suffix_array.hpp:93-96
        }
        s_k2[a] = k2;
        s_key[a] = (static_cast<u64>(k2) << 12) | static_cast<u32>(a);
    }
    __syncthreads();
    // -- rank inside the group: keys are unique (slot field), so the new slot = group start + #smaller keys
    for (int a = first + tid; a < end; a += kDblBlock) {
        if (is_head(a) && is_head(a + 1)) continue;
        const int gs = group_start(a, s_bits), ge = group_end(a);
        const u64 ki = s_key[a];
        u32 r = 0;
        for (int j = gs; j < ge; ++j) r += s_key[j] < ki;
        s_pos2[gs + r] = s_pos[a];
    }
    __syncthreads();
    for (int a = first + tid; a < end; a += kDblBlock) {   // rank2 in the new order (s_key is dead: reuse its words)
        if (is_head(a) && is_head(a + 1)) continue;
        const int gs = group_start(a, s_bits), ge = group_end(a);
        const u64 ki = s_key[a];
        u32 r = 0;
        for (int j = gs; j < ge; ++j) r += s_key[j] < ki;
        s_pos[gs + r] = static_cast<u32>(ki >> 12);        // (s_pos was copied out above)
    }
    __syncthreads();
    // -- new heads: an old head, or rank2 differs from the predecessor's in the new order
    for (int a0 = first - (first & 31); a0 < end; a0 += kDblBlock) {
        const int a = a0 + tid;
        bool head = false;
        if (a >= first && a < end) {
            const bool tied = !(is_head(a) && is_head(a + 1));
            head = is_head(a) || (tied && s_pos[a] != s_pos[a - 1]);
        }
        const unsigned b = __ballot_sync(0xffffffffu, head);
        if (lane == 0 && b) atomicOr(&s_new[a >> 5], b);
    }
    __syncthreads();
    u32 heads = 0;
    for (int a = first + tid; a < end; a += kDblBlock) {
        sa[t0 + a] = s_pos2[a];
        const int gs = group_start(a, s_new);
        head_new[t0 + a] = static_cast<u32>(t0 + gs);
        heads += gs == a;
    }
    if (overrun) {   // the group nobody re-sorted keeps its head index: this tile's share of it
        const int gs = s_last;
        for (int a = gs + tid; a < lim; a += kDblBlock) head_new[t0 + a] = static_cast<u32>(t0 + gs);
        heads += tid == 0;
    }
    for (int o = 16; o > 0; o >>= 1) heads += __shfl_xor_sync(0xffffffffu, heads, o);
    if (lane == 0 && heads) atomicAdd(counters, heads);
}

__global__ void scatter_vals_kernel(const u32* __restrict__ sa, const u32* __restrict__ vals, u64 n, u32* __restrict__ rank) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) rank[sa[i]] = vals[i];
}

// ---- multi-GPU building blocks: a rank makes the records of ITS bucket straight from the
//      replicated packed text -----------------------------------------------------------------
// Sample sort needs every suffix record on the rank whose splitter range holds its key.  The text is
// replicated (n/4 bytes packed), so no record has to travel: each rank walks all suffix keys and KEEPS
// those whose 12-bit key prefix (6 bases, zero padded from the terminator on -- the top of both record
// kinds' keys) lies in [plo, phi).  What it keeps must come out in the order the stable digit passes
// start from: (terminator distance, position) for uniform read sets, position for general records.
// That is a stream compaction in that order: a count sweep, one scan of the counts, a write sweep.
constexpr int kShPrefixBits = 12;
constexpr int kShReads = 256;      // uniform: reads per CTA; thread = read
constexpr int kShTile = 2048;      // general: positions per CTA; thread = 8 consecutive positions

// Calls f(t, key32) for every suffix of the read whose first base is bit `bit0` of the staged words,
// t = period - 1 down to 0 (offset 0 up to the sentinel).  key32 = its first 16 bases, zero padded
// from the sentinel on.  Trip counts are uniform across a warp (f may vote).
template <class F>
__device__ __forceinline__ void for_each_suffix_of_read(const u64* __restrict__ s_w, u32 bit0, u32 period, F f) {
    for (u32 o = 0; o < period; ++o) {
        const u32 t = period - 1 - o;
        const u32 bit = bit0 + 2 * o;
        const u32 wi = bit >> 6, sh = bit & 63;
        const u64 hi = s_w[wi], lo = s_w[wi + 1];
        const u64 win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
        u32 key = static_cast<u32>(win >> 32);
        if (t < static_cast<u32>(kUniK)) key = t ? key & ~((1u << (2 * (kUniK - t))) - 1u) : 0u;
        f(t, key);
    }
}

// Histogram of the 12-bit key prefix over the suffixes of reads [read0, read0 + count).
__global__ void __launch_bounds__(kShReads)
shard_hist_uniform_kernel(const u64* __restrict__ packed, u32 period, u64 read0, u64 count, u32* __restrict__ g_hist) {
    __shared__ __align__(16) u64 s_w[kShReads * kUniMaxPeriod / 32 + 8];
    __shared__ u32 s_hist[1 << kShPrefixBits];
    for (int i = threadIdx.x; i < (1 << kShPrefixBits); i += blockDim.x) s_hist[i] = 0;
    const u64 r0 = static_cast<u64>(blockIdx.x) * kShReads;
    const u32 nr = static_cast<u32>(count - r0 < kShReads ? count - r0 : kShReads);
    const u32 bit0 = stage_reads(packed, s_w, read0 + r0, nr, period);
    __syncthreads();
    const bool in = threadIdx.x < nr;
    for_each_suffix_of_read(s_w, bit0 + (in ? 2 * threadIdx.x * period : 0u), period, [&](u32, u32 key) {
        if (in) atomicAdd(&s_hist[key >> (32 - kShPrefixBits)], 1u);
    });
    __syncthreads();
    for (int i = threadIdx.x; i < (1 << kShPrefixBits); i += blockDim.x)
        if (s_hist[i]) atomicAdd(g_hist + i, s_hist[i]);
}

// counts[t * tiles + tile] = suffixes with t symbols before their sentinel, of the reads of `tile`,
// whose key prefix lies in [plo, phi): the flattened array scans into slot bases in (t, read) order.
// This is the only sweep that looks at every suffix key, so it also leaves the write sweep everything it
// found: keep[(tile * period + t) * 8 + warp] = the warp's ballot of kept reads at t, wbase[...] = kept
// reads of the tile's lower warps at t.  The write sweep then touches text only for what it keeps
// (1/G of the suffixes).  (The first form recomputed every key in all three sweeps: 4.4 ms of a 13.6 ms
// modelled 8-GPU build at 1 G suffixes, and the one part that does not shrink with G.)
// The 6-base prefix of the suffix at offset o comes from a window that slides along the read (one
// shared-memory word per 32 offsets), not from a fresh two-word extraction per offset.
__global__ void __launch_bounds__(kShReads)
shard_count_uniform_kernel(const u64* __restrict__ packed, u32 period, u64 k, u32 plo, u32 phi, u32 tiles,
                           u32* __restrict__ counts, u32* __restrict__ keep, unsigned short* __restrict__ wbase) {
    __shared__ __align__(16) u64 s_w[kShReads * kUniMaxPeriod / 32 + 8];
    __shared__ unsigned short s_wcnt[kShReads / 32][kUniMaxPeriod + 1];
    const u64 r0 = static_cast<u64>(blockIdx.x) * kShReads;
    const u32 nr = static_cast<u32>(k - r0 < kShReads ? k - r0 : kShReads);
    const u32 bit0 = stage_reads(packed, s_w, r0, nr, period);
    const bool in = threadIdx.x < nr;
    const int warp = threadIdx.x >> 5;
    const u32 my_bit0 = bit0 + (in ? 2 * threadIdx.x * period : 0u);
    // window = the next 32+ bases from offset o on, refilled every 16 offsets.  The ballots of 32 values of t
    // are collected in registers (lane j keeps the mask of t = 32 c + j) and leave as one coalesced store.
    // Offsets are walked in three stretches so that the bulk of them runs as straight-line blocks of 16
    // (8 instructions per suffix: no bounds, no padding mask, the flush test once per block): a generic
    // prologue down to t = 15 mod 16, aligned blocks while t > 15, a generic epilogue for t = 15 .. 0 (the
    // suffixes shorter than the 6-base prefix are there).  (One generic loop: 25 instructions per suffix,
    // 2.7 ms per sweep over 3 G suffixes -- the phase of the sharded build that does not shrink with G.)
    const u32 span = phi - plo;
    const unsigned lane = lane_id();
    const u64 kcell = (static_cast<u64>(blockIdx.x) * (kShReads / 32) + warp) * period;
    u32 mine = 0;
    u64 win = 0;
    auto refill = [&](u32 o) {
        const u32 bit = my_bit0 + 2 * o;
        const u32 wi = bit >> 6, sh = bit & 63u;
        const u64 hi = s_w[wi], lo = s_w[wi + 1];
        win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
    };
    auto flush = [&](u32 t) {                                  // t .. t + 31 are complete
        if (t + lane < period) {
            keep[kcell + t + lane] = mine;
            s_wcnt[warp][t + lane] = static_cast<unsigned short>(__popc(mine));
        }
        mine = 0;
    };
    auto generic = [&](u32 o) {
        const u32 t = period - 1 - o;
        u32 pre = static_cast<u32>(win >> (64 - kShPrefixBits));
        if (t < 6u) pre = t ? pre & ~((1u << (2 * (6 - t))) - 1u) : 0u;    // zero padded from the sentinel on
        win <<= 2;
        const unsigned bm = __ballot_sync(0xffffffffu, in && pre - plo < span);
        if (lane == (t & 31u)) mine = bm;
        if ((t & 31u) == 0) flush(t);
    };
    u32 o = 0;
    refill(0);
    for (u32 c = 0; o < period && ((period - 1 - o) & 15u) != 15u; ++o, ++c) {       // prologue: < 16 offsets
        if (c == 16) refill(o);
        generic(o);
    }
    while (o < period && period - 1 - o > 15u) {                                     // t = T .. T - 15, T = 15 mod 16, T >= 31
        refill(o);
        const u32 T = period - 1 - o;
        const u32 d = (T & 31u) - lane;                                              // lane keeps iteration j = d
#pragma unroll
        for (u32 j = 0; j < 16; ++j) {
            const u32 pre = static_cast<u32>(win >> (64 - kShPrefixBits));
            win <<= 2;
            const unsigned bm = __ballot_sync(0xffffffffu, in && pre - plo < span);
            if (d == j) mine = bm;
        }
        o += 16;
        if (((T - 15u) & 31u) == 0) flush(T - 15u);
    }
    if (o < period) refill(o);
    for (; o < period; ++o) generic(o);                                              // epilogue: t = 15 .. 0
    __syncthreads();
    for (u32 t = threadIdx.x; t < period; t += blockDim.x) {
        u32 run = 0;
        for (int w = 0; w < kShReads / 32; ++w) {
            wbase[(static_cast<u64>(blockIdx.x) * (kShReads / 32) + w) * period + t] = static_cast<unsigned short>(run);
            run += s_wcnt[w][t];
        }
        counts[static_cast<u64>(t) * tiles + blockIdx.x] = run;
    }
}

// Writes the kept records key32 << 32 | position at offsets[t * tiles + tile] + (rank of the read
// among the tile's kept reads at this t): the bucket comes out in (t, position) order.
// A rank keeps 1/G of the suffixes, so with lanes = reads only ~32/G lanes of a warp had work at any t and
// the record body ran for nearly every t all the same (5.8 ms at 3 G suffixes, G = 8: the largest phase that
// does not shrink with G).  Instead each warp turns the keep masks of 32 values of t into a compact work
// list in shared memory ((t - t0) << 5 | read, in (t, read) order: entries of one t are neighbours, so are
// their output slots) and all 32 lanes take entries from it.
__global__ void __launch_bounds__(kShReads)
shard_write_uniform_kernel(const u64* __restrict__ packed, u32 period, u64 k, u32 tiles, const u32* __restrict__ offsets,
                           const u32* __restrict__ keep, const unsigned short* __restrict__ wbase,
                           u64* __restrict__ out, u32* __restrict__ g_hist) {
    __shared__ __align__(16) u64 s_w[kShReads * kUniMaxPeriod / 32 + 8];
    __shared__ u32 s_hist[4 * kRadix];                                    // digit histograms of the bucket's four sort passes
    __shared__ unsigned short s_list[kShReads / 32][1024];                // per warp: the kept (t, read) pairs of 32 values of t
    for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) s_hist[i] = 0;
    const u64 r0 = static_cast<u64>(blockIdx.x) * kShReads;
    const u32 nr = static_cast<u32>(k - r0 < kShReads ? k - r0 : kShReads);
    const u32 bit0 = stage_reads(packed, s_w, r0, nr, period);
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const u32 warp_read0 = static_cast<u32>(warp) * 32u;
    const u64 wcell = (static_cast<u64>(blockIdx.x) * (kShReads / 32) + warp) * period;   // this warp's masks, t-contiguous
    unsigned short* list = s_list[warp];
    for (u32 t0 = 0; t0 < period; t0 += 32) {
        const u32 tt = t0 + lane;
        const u32 kw = tt < period ? keep[wcell + tt] : 0u;          // lane j: the mask of t0 + j
        const u32 base = tt < period ? offsets[static_cast<u64>(tt) * tiles + blockIdx.x] + wbase[wcell + tt] : 0u;
        const u32 c = __popc(kw);
        u32 inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, inc, o);
            if (static_cast<int>(lane) >= o) inc += v;
        }
        const u32 first = inc - c;                                    // index of this t's first entry in the list
        const u32 total = __shfl_sync(0xffffffffu, inc, 31);
        {
            u32 m = kw, q = first;
            while (m) {
                const u32 b = __ffs(m) - 1u;
                m &= m - 1u;
                list[q++] = static_cast<unsigned short>((lane << 5) | b);
            }
        }
        __syncwarp();
        for (u32 i0 = 0; i0 < total; i0 += 32) {
            const u32 i = i0 + lane;
            const bool on = i < total;
            const u32 ent = on ? list[i] : 0u;
            const u32 j = ent >> 5, rd = warp_read0 + (ent & 31u);
            const u32 slot = __shfl_sync(0xffffffffu, base, j) + (i - __shfl_sync(0xffffffffu, first, j));
            if (!on) continue;
            const u32 t = t0 + j;
            const u32 o = period - 1 - t;
            const u32 bit = bit0 + 2 * (rd * period + o), wi = bit >> 6, sh = bit & 63u;
            const u64 hi = s_w[wi], lo = s_w[wi + 1];
            const u64 win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
            u32 key = static_cast<u32>(win >> 32);
            if (t < static_cast<u32>(kUniK)) key = t ? key & ~((1u << (2 * (kUniK - t))) - 1u) : 0u;
            out[slot] = (static_cast<u64>(key) << 32) | ((r0 + rd) * period + o);
            atomicAdd(&s_hist[key & 0xffu], 1u);
            atomicAdd(&s_hist[kRadix + ((key >> 8) & 0xffu)], 1u);
            atomicAdd(&s_hist[2 * kRadix + ((key >> 16) & 0xffu)], 1u);
            atomicAdd(&s_hist[3 * kRadix + (key >> 24)], 1u);
        }
        __syncwarp();
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, 4);
}

// The same with lanes = reads and no work list: the form for a rank that keeps most suffixes (G <= 2), where
// nearly every lane has a record to write at every t and the list would only add work (15.9 vs 11.1 ms at 3 G
// suffixes, G = 1).
__global__ void __launch_bounds__(kShReads)
shard_write_uniform_direct_kernel(const u64* __restrict__ packed, u32 period, u64 k, u32 tiles, const u32* __restrict__ offsets,
                           const u32* __restrict__ keep, const unsigned short* __restrict__ wbase,
                           u64* __restrict__ out, u32* __restrict__ g_hist) {
    __shared__ __align__(16) u64 s_w[kShReads * kUniMaxPeriod / 32 + 8];
    __shared__ u32 s_hist[4 * kRadix];                                    // digit histograms of the bucket's four sort passes
    for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) s_hist[i] = 0;
    const u64 r0 = static_cast<u64>(blockIdx.x) * kShReads;
    const u32 nr = static_cast<u32>(k - r0 < kShReads ? k - r0 : kShReads);
    const u32 bit0 = stage_reads(packed, s_w, r0, nr, period);
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const u32 my_bit0 = bit0 + (threadIdx.x < nr ? 2 * threadIdx.x * period : 0u);
    const u64 pos0 = (r0 + threadIdx.x) * period;
    const u64 wcell = (static_cast<u64>(blockIdx.x) * (kShReads / 32) + warp) * period;   // this warp's masks, t-contiguous
    for (u32 t0 = 0; t0 < period; t0 += 32) {
        const u32 tt = t0 + lane;
        const u32 kw = tt < period ? keep[wcell + tt] : 0u;          // 32 masks per coalesced load, handed round by shuffles
        const u32 wb = tt < period ? wbase[wcell + tt] : 0u;
        const u32 jn = period - t0 < 32u ? period - t0 : 32u;
        for (u32 j = 0; j < jn; ++j) {
            const unsigned bm = __shfl_sync(0xffffffffu, kw, j);
            const u32 base_w = __shfl_sync(0xffffffffu, wb, j);
            if (!((bm >> lane) & 1u)) continue;
            const u32 t = t0 + j;
            const u32 o = period - 1 - t;
            const u32 bit = my_bit0 + 2 * o, wi = bit >> 6, sh = bit & 63u;
            const u64 hi = s_w[wi], lo = s_w[wi + 1];
            const u64 win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
            u32 key = static_cast<u32>(win >> 32);
            if (t < static_cast<u32>(kUniK)) key = t ? key & ~((1u << (2 * (kUniK - t))) - 1u) : 0u;
            const u64 slot = static_cast<u64>(offsets[static_cast<u64>(t) * tiles + blockIdx.x]) + base_w + __popc(bm & lanemask_lt());
            out[slot] = (static_cast<u64>(key) << 32) | (pos0 + o);
            atomicAdd(&s_hist[key & 0xffu], 1u);
            atomicAdd(&s_hist[kRadix + ((key >> 8) & 0xffu)], 1u);
            atomicAdd(&s_hist[2 * kRadix + ((key >> 16) & 0xffu)], 1u);
            atomicAdd(&s_hist[3 * kRadix + (key >> 24)], 1u);
        }
    }
    __syncthreads();
    hist_flush(s_hist, g_hist, 4);
}

// The general records (elem_of): prefix = the first 6 bases of the 24-bit key.
__device__ __forceinline__ u32 elem_prefix(u64 e) { return static_cast<u32>(e >> (kElemKeyShift + 24 - kShPrefixBits)); }

__global__ void __launch_bounds__(256)
shard_hist_general_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n, u64 pos0, u64 count,
                          u32* __restrict__ g_hist) {
    __shared__ u32 s_hist[1 << kShPrefixBits];
    for (int i = threadIdx.x; i < (1 << kShPrefixBits); i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < count; idx += stride)
        atomicAdd(&s_hist[elem_prefix(elem_of(packed, sent, n, pos0 + idx))], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < (1 << kShPrefixBits); i += blockDim.x)
        if (s_hist[i]) atomicAdd(g_hist + i, s_hist[i]);
}

// WRITE = false: counts[tile] = kept positions of the tile; true: the kept records at offsets[tile] on,
// in position order.
template <bool WRITE>
__global__ void __launch_bounds__(256)
shard_general_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n, u32 plo, u32 phi,
                     u32* __restrict__ counts, const u32* __restrict__ offsets, u64* __restrict__ out,
                     u32* __restrict__ g_hist) {
    __shared__ u32 s_warp[8];
    __shared__ u32 s_hist[WRITE ? 3 * kRadix : 1];
    if constexpr (WRITE) {
        for (int i = threadIdx.x; i < 3 * kRadix; i += blockDim.x) s_hist[i] = 0;
    }
    constexpr int kPer = kShTile / 256;
    const u64 p0 = static_cast<u64>(blockIdx.x) * kShTile + static_cast<u64>(threadIdx.x) * kPer;
    u64 e[kPer];
    u32 mine = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        e[j] = 0;
        bool keep = false;
        if (p0 + j < n) {
            e[j] = elem_of(packed, sent, n, p0 + j);
            const u32 pre = elem_prefix(e[j]);
            keep = pre >= plo && pre < phi;
        }
        if (!keep) e[j] = ~0ull;   // (no record is all ones: its position would be 2^32 - 1 > the largest text)
        mine += keep;
    }
    u32 inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane_id()) >= o) inc += t;
    }
    if (lane_id() == 31) s_warp[threadIdx.x >> 5] = inc;
    __syncthreads();
    u32 before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        before += w < static_cast<int>(threadIdx.x >> 5) ? s_warp[w] : 0u;
        total += s_warp[w];
    }
    if constexpr (!WRITE) {
        if (threadIdx.x == 0) counts[blockIdx.x] = total;
    } else {
        u64 slot = static_cast<u64>(offsets[blockIdx.x]) + before + inc - mine;
#pragma unroll
        for (int j = 0; j < kPer; ++j)
            if (e[j] != ~0ull) {
                out[slot++] = e[j];
                const u32 key = static_cast<u32>(e[j] >> kElemKeyShift);
                atomicAdd(&s_hist[key & 0xffu], 1u);
                atomicAdd(&s_hist[kRadix + ((key >> 8) & 0xffu)], 1u);
                atomicAdd(&s_hist[2 * kRadix + (key >> 16)], 1u);
            }
        __syncthreads();
        hist_flush(s_hist, g_hist, 3);
    }
}

// ---- rank sharded by position: the second exchange ---------------------------------------------------
// A rank holds a bucket of the suffix array: positions sa[i], global indices offset + i.  Position p
// belongs to the rank g with base(g) <= p < base(g + 1), base(g) = floor(n g / G).  Its record
// (p - base(g)) << 32 | (offset + i) goes to g; there the records are a permutation of the slice and
// inverse_from_records turns them into the slice of `rank`.
// (64-bit divisions per record made the first form of these kernels 3x slower than the sort pass they
// sit next to: the owner comes from one multiply-high by a host-made reciprocal and a fix-up against the
// table of bases; the sub-bin from a shift.)
struct OwnerTable {
    u64 base[17];    // base[g] = floor(n g / G), base[G] = n  (n <= 2^32 - 2: every base but base[G] fits 32 bits, and so does base[G])
    u32 magic;       // floor(2^32 G / n): mulhi32(p, magic) is floor(p G / n) or up to two less
    u32 G;
    u32 sub;         // sub-bins per owner (a power of two; G * sub <= 1024)
};
constexpr int kOwnMaxBins = 1024;
constexpr int kOwnBlock = 512, kOwnItems = 8, kOwnTile = kOwnBlock * kOwnItems;
// `base` = the table's bases copied to SHARED memory by the caller as 32-bit words: lanes look up different owners,
// and a kernel parameter indexed per lane is a constant-bank load replayed once per distinct owner in the warp.
// Positions are 32-bit, so the owner estimate is ONE 32 x 32 multiply-high (the 64-bit reciprocal of the first
// form cost ten instructions) and the fix-up compares words.
__device__ __forceinline__ u32 owner_bin(const OwnerTable& tb, const u32* __restrict__ base, u32 p, u32* rel) {
    u32 g = __umulhi(p, tb.magic);                              // the owner, or up to two below it
    while (g + 1 < tb.G && base[g + 1] <= p) ++g;
    *rel = p - base[g];
    // the sub-bin only spreads the shared-memory atomics: LOW position bits, so that an owner's group
    // stays unordered in the high bits the receiver partitions on (top bits made every tile of its first
    // pass hit one bin: 0.79 ms against 0.52)
    return g * tb.sub + ((*rel >> 2) & (tb.sub - 1u));
}

__global__ void __launch_bounds__(256)
owner_count_kernel(const u32* __restrict__ sa, u64 m, OwnerTable tb, u32* __restrict__ counts) {
    __shared__ u32 s_cnt[kOwnMaxBins];
    __shared__ u32 s_base[17];
    const u32 bins = tb.G * tb.sub;
    for (u32 b = threadIdx.x; b < bins; b += blockDim.x) s_cnt[b] = 0;
    if (threadIdx.x <= tb.G) s_base[threadIdx.x] = static_cast<u32>(tb.base[threadIdx.x]);
    __syncthreads();
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 tid0 = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    u32 rel;
    // four positions per 16-byte load, two loads in flight (one 4-byte load per trip left the sweep waiting on
    // DRAM latency: 1.75 ms for 378 M positions, 0.9 TB/s)
    const u64 quads = (reinterpret_cast<uintptr_t>(sa) & 15) == 0 ? m / 4 : 0;
    const uint4* sa4 = reinterpret_cast<const uint4*>(sa);
    u64 i = tid0;
    for (; i + stride < quads; i += 2 * stride) {
        const uint4 a = sa4[i], b = sa4[i + stride];
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.x, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.y, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.z, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.w, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, b.x, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, b.y, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, b.z, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, b.w, &rel)], 1u);
    }
    if (i < quads) {
        const uint4 a = sa4[i];
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.x, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.y, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.z, &rel)], 1u);
        atomicAdd(&s_cnt[owner_bin(tb, s_base, a.w, &rel)], 1u);
    }
    for (u64 x = 4 * quads + tid0; x < m; x += stride) atomicAdd(&s_cnt[owner_bin(tb, s_base, sa[x], &rel)], 1u);
    __syncthreads();
    for (u32 b = threadIdx.x; b < bins; b += blockDim.x)
        if (s_cnt[b]) atomicAdd(counts + b, s_cnt[b]);
}

// One lean partition pass (see inv_partition_persistent_kernel): a record takes its slot in the tile's bin
// from one shared-memory atomicAdd, a bin claims its stretch with one global atomicAdd on a counter that
// starts at the bin's base, the tile leaves through shared memory as one contiguous run per bin.
// Exclusive bases of the owner x sub-range bins, one claim counter per 128-byte line (all tiles claim from these
// few counters: packed they shared four cache lines).  One block; bins <= 1024.
__global__ void __launch_bounds__(kOwnMaxBins)
owner_bases_kernel(const u32* __restrict__ counts, int bins, u32* __restrict__ claim) {
    __shared__ u32 s_warp[kOwnMaxBins / 32];
    const int b = threadIdx.x;
    const u32 c = b < bins ? counts[b] : 0u;
    u32 inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane_id()) >= o) inc += t;
    }
    if (lane_id() == 31) s_warp[b >> 5] = inc;
    __syncthreads();
    u32 before = 0;
    for (int w = 0; w < (b >> 5); ++w) before += s_warp[w];
    if (b < bins) claim[static_cast<size_t>(b) * kIpClaimStride] = before + inc - c;
}

__global__ void __launch_bounds__(kOwnBlock, 2)
owner_partition_kernel(const u32* __restrict__ sa, u64 m, OwnerTable tb, u64 offset, u32* __restrict__ claim,
                       u64* __restrict__ out, u32 num_tiles) {
    extern __shared__ __align__(16) unsigned char own_smem[];
    u64* s_rec = reinterpret_cast<u64*>(own_smem);                                  // [tile] records, bin-sorted
    u32* s_cnt = reinterpret_cast<u32*>(s_rec + kOwnTile);                          // [1024]
    u32* s_ofs = s_cnt + kOwnMaxBins;                                               // [1024]
    u32* s_gdst = s_ofs + kOwnMaxBins;                                              // [1024]
    u32* s_warp = s_gdst + kOwnMaxBins;                                             // [16]
    unsigned short* s_binof = reinterpret_cast<unsigned short*>(s_warp + kOwnBlock / 32);   // [tile] bin of the record in that slot
    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int bins = static_cast<int>(tb.G * tb.sub);
    __shared__ u32 s_base[17];
    // Persistent, like inv_partition_persistent_kernel: two CTAs per SM walk the tiles round-robin and issue the next
    // tile's loads before the current one is scanned, exchanged and stored (one tile per CTA: 3.2 ms for 378 M
    // positions against 1.3 ms for the receiver's pass over the same records).
    auto load_tile = [&](u32 tile, u32 (&p)[kOwnItems]) {
        const u64 t0 = static_cast<u64>(tile) * kOwnTile;
#pragma unroll
        for (int j = 0; j < kOwnItems; ++j) {
            const u64 i = t0 + static_cast<u64>(j) * kOwnBlock + tid;
            p[j] = i < m ? sa[i] : 0u;
        }
    };
    u32 pos[kOwnItems], nxt[kOwnItems];
    if (blockIdx.x < num_tiles) load_tile(blockIdx.x, pos);
    for (int b = tid; b < bins; b += kOwnBlock) s_cnt[b] = 0;
    if (tid <= static_cast<int>(tb.G)) s_base[tid] = static_cast<u32>(tb.base[tid]);
    __syncthreads();
    for (u32 tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const u64 tile0 = static_cast<u64>(tile) * kOwnTile;
        const u32 valid = static_cast<u32>(m - tile0 < static_cast<u64>(kOwnTile) ? m - tile0 : kOwnTile);
        u64 rec[kOwnItems];
        u32 slot[kOwnItems], bin[kOwnItems];
#pragma unroll
        for (int j = 0; j < kOwnItems; ++j) {
            const u32 li = static_cast<u32>(j) * kOwnBlock + tid;
            slot[j] = 0;
            bin[j] = 0;
            rec[j] = 0;
            if (li < valid) {
                u32 rel;
                bin[j] = owner_bin(tb, s_base, pos[j], &rel);
                rec[j] = (static_cast<u64>(rel) << 32) | ((offset + tile0 + li) & 0xffffffffu);
                slot[j] = atomicAdd(&s_cnt[bin[j]], 1u);
            }
        }
        if (tile + gridDim.x < num_tiles) load_tile(tile + gridDim.x, nxt);   // in flight until the end of this tile
        __syncthreads();
        // two bins per thread (bins <= 1024 = 2 * block): counts, claims, exclusive scan
        const int b0 = 2 * tid, b1 = 2 * tid + 1;
        const u32 c0 = b0 < bins ? s_cnt[b0] : 0u, c1 = b1 < bins ? s_cnt[b1] : 0u;
        u32 g0 = 0, g1 = 0;
        if (c0) g0 = atomicAdd(claim + b0 * kIpClaimStride, c0);
        if (c1) g1 = atomicAdd(claim + b1 * kIpClaimStride, c1);
        u32 inc = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
            if (static_cast<int>(lane) >= o) inc += t;
        }
        if (lane == 31) s_warp[tid >> 5] = inc;
        __syncthreads();
        u32 before = 0;
#pragma unroll
        for (int w = 0; w < kOwnBlock / 32; ++w) before += w < (tid >> 5) ? s_warp[w] : 0u;
        const u32 excl = before + inc - (c0 + c1);
        if (b0 < bins) { s_ofs[b0] = excl; s_gdst[b0] = g0 - excl; s_cnt[b0] = 0; }
        if (b1 < bins) { s_ofs[b1] = excl + c0; s_gdst[b1] = g1 - (excl + c0); s_cnt[b1] = 0; }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kOwnItems; ++j) {
            const u32 li = static_cast<u32>(j) * kOwnBlock + tid;
            if (li < valid) {
                const u32 at = s_ofs[bin[j]] + slot[j];
                s_rec[at] = rec[j];
                s_binof[at] = static_cast<unsigned short>(bin[j]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kOwnItems; ++j) {
            const u32 pidx = static_cast<u32>(j) * kOwnBlock + tid;
            if (pidx < valid) out[static_cast<u64>(s_gdst[s_binof[pidx]]) + pidx] = s_rec[pidx];
        }
#pragma unroll
        for (int j = 0; j < kOwnItems; ++j) pos[j] = nxt[j];
        __syncthreads();   // s_rec / s_gdst / s_binof are rewritten by the next tile
    }
}
constexpr size_t kOwnSmem = sizeof(u64) * kOwnTile + sizeof(u32) * (3 * kOwnMaxBins + kOwnBlock / 32) + sizeof(unsigned short) * kOwnTile;

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
    if (!is_dna) return RESEQ_OK;   // asynchronous form: the caller checks d_flag on the device
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_flag, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    *is_dna = reinterpret_cast<volatile u32*>(ctx->pinned)[0] == 0;
    if (n_separators) *n_separators = reinterpret_cast<volatile u32*>(ctx->pinned)[1];
    return RESEQ_OK;
}

// claim counters of both partition passes
static size_t inverse_scratch_words(size_t n) { return 1024 * 32 + (n >> 13) + 64; }   // kIpMaxBins first-pass counters, one per 128-byte line, + the second pass's

// Ragged read sets are taken on when there are at most n / kRagMinAvg reads (mean length >= 15: below
// that the 15-base key sorts nothing) -- which also bounds the tables below.
constexpr size_t kRagMinAvg = 16;
static size_t ragged_cells(size_t n) { return ((n / kRagMinAvg) / kRagReads + 2) * (kRagMaxLen + 1) + 1; }
static size_t ragged_workspace_bytes(size_t n) {
    auto pad = reseq_cuda_ctx::padded;
    return pad(sizeof(u32) * (n / 64 + 2)) * 2 + pad(sizeof(u32) * (n / kRagMinAvg + 2)) + pad(sizeof(u32) * (n / 32 + 2)) +
           2 * pad(sizeof(u32) * ragged_cells(n)) + scan_workspace_bytes(n / 64 + 2) + scan_workspace_bytes(ragged_cells(n)) + 8192;
}

size_t sa_workspace_bytes(size_t n) {
    auto pad = reseq_cuda_ctx::padded;
    size_t total = 0;
    total += pad(sizeof(u64) * (n / 32 + 8));        // packed bases
    total += pad(sizeof(u64) * (n / 64 + 8));        // sentinel bitmap
    total += 2 * pad(sizeof(u64) * n);               // record / key buffers a and b
    total += 2 * pad(sizeof(u32) * n);               // payload buffer b, head_of
    total += pad(sizeof(u32) * n);                   // rank when the caller wants none
    total += pad(sizeof(u64) * (n / kRankTile + 4)); // rerank descriptors
    total += pad(1024);                              // counters
    total += pad(n / kUniMinPeriod + 2);             // uniform read-set path: proof table, one byte per read
    total += ragged_workspace_bytes(n);              // ragged read-set path: rank structure of the bitmap, proof bits, slot tables
    total += 2 * pad(sizeof(u32) * (n / 32 + 2 + n / kRefTile / 4 + 2));   // head / uncovered bitmaps, tile flags
    total += pad(sizeof(u32) * inverse_scratch_words(n));
    total += sort_workspace_bytes(n);
    return total + 4096;
}

namespace {

// How the position bits are split between the partition passes and the shared-memory window.
struct InversePlan {
    bool partitioned;   // false: small text, direct scatter
    int win_bits;       // rank entries per window_scatter_kernel CTA = 1 << win_bits
    int lo_bits;        // bits of the second pass (0: one pass is enough)
    int shift1;         // first pass: bucket = position >> shift1
    int bins1;          // buckets of the first pass
    u32 buckets2;       // buckets after the second pass (= windows)
    unsigned tiles;
};

InversePlan make_inverse_plan(size_t n, int mode, int top_bits = -1) {
    InversePlan p{};
    p.partitioned = n >= (size_t{1} << 22);
    if (!p.partitioned) return p;
    const int nb = static_cast<int>(bit_width_u64(n - 1));   // >= 23
    if (mode == 1) {   // one partition pass (as many bins as it takes, <= 1024), then the L2-window scatter
        p.win_bits = 0;
        p.lo_bits = 0;
        p.shift1 = nb > 10 ? nb - 10 : 0;
        p.bins1 = static_cast<int>(((n - 1) >> p.shift1) + 1);
        p.buckets2 = 0;
        p.tiles = static_cast<unsigned>((n + kIpTile - 1) / kIpTile);
        return p;
    }
    // The first pass gets at most 7 bits: its tiles all claim from the same `bins1` counters, and with 133 - 240 bins
    // it ran at 0.31 - 0.47 of the HBM peak against 0.57 with 67 - 97 (config 3: 0.60 -> 0.33 ms); the bits go to the
    // second pass, whose claims spread over bucket x bin counters (<= 1024 bins), and, above 2^27 records, to a
    // 2^14-entry window.
    p.win_bits = 13;
    int rest = nb - p.win_bits;                               // bits the passes must consume
    const int top_max = top_bits > 0 && top_bits <= 10 ? top_bits : 7;   // tuning knob ("inverse_lo_bits" carries it)
    int top = rest < top_max ? rest : top_max;
    int lo = rest - top;
    if (lo > 7) {                                             // n > 2^27: 64 KB windows rather than 512+ second-pass bins (0.506 -> 0.479 ms at config 2)
        p.win_bits = 14;
        rest = nb - p.win_bits;
        top = rest < top_max ? rest : top_max;
        lo = rest - top;
    }
    if (lo > 9) { top += lo - 9; lo = 9; }                    // n > 2^31: wider first pass (<= 9 bits)
    p.lo_bits = lo;
    p.shift1 = p.win_bits + lo;
    p.bins1 = static_cast<int>(((n - 1) >> p.shift1) + 1);
    p.buckets2 = static_cast<u32>(((n - 1) >> p.win_bits) + 1);
    p.tiles = static_cast<unsigned>((n + kIpTile - 1) / kIpTile);
    return p;
}

int window_scatter_device(reseq_cuda_ctx* ctx, const u64* rec, size_t n, int win_bits, u32* rank) {
    RSQ_OPT_IN_SMEM(ctx, window_scatter_kernel, 64 * 1024);
    const unsigned windows = static_cast<unsigned>((n + (size_t{1} << win_bits) - 1) >> win_bits);
    RSQ_LAUNCH_BEGIN(ctx, "window_scatter_kernel");
    window_scatter_kernel<<<windows, 512, sizeof(u32) << win_bits, ctx->stream>>>(rec, n, win_bits, rank);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

// rank = inverse permutation of the finished sa (scratch: two u64 record buffers of n entries and
// inverse_scratch_words(n) claim counters).
int inverse_device(reseq_cuda_ctx* ctx, const u32* sa, size_t n, u32* rank, u64* rec_a, u64* rec_b, u32* scratch) {
    cudaStream_t s = ctx->stream;
    const InversePlan plan = make_inverse_plan(n, ctx->opt_inverse_mode, ctx->opt_inverse_lo_bits);
    if (!plan.partitioned) {  // the whole rank array is L2-resident: scatter directly
        RSQ_LAUNCH_BEGIN(ctx, "inverse_kernel");
        inverse_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, s>>>(sa, n, rank);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        return RESEQ_OK;
    }
    u32* claim1 = scratch;
    u32* claim2 = scratch + kIpMaxBins * kIpClaimStride;
    RSQ_CUDA(cudaMemsetAsync(claim1, 0, sizeof(u32) * plan.bins1 * kIpClaimStride, s));
    RSQ_CUDA(cudaMemsetAsync(claim2, 0, sizeof(u32) * (plan.buckets2 + 32), s));
    const unsigned grid = plan.tiles < static_cast<unsigned>(ctx->sm_count) * 2 ? plan.tiles : ctx->sm_count * 2;
    RSQ_LAUNCH_BEGIN(ctx, "inv_partition_sa");
    inv_partition_persistent_kernel<kIpSa><<<grid, kIpBlock, 0, s>>>(sa, n, plan.shift1, 0, plan.bins1, claim1, rec_a, plan.tiles);
    RSQ_LAUNCH_END(ctx);
    const u64* rec = rec_a;
    if (plan.win_bits == 0) {
        RSQ_LAUNCH_BEGIN(ctx, "bucket_scatter_kernel");
        bucket_scatter_kernel<<<grid_for(ctx, n / 2 + 1, 256, 4, 8), 256, 0, s>>>(rec_a, n, rank);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        return RESEQ_OK;
    }
    if (plan.lo_bits > 0) {
        RSQ_LAUNCH_BEGIN(ctx, "inv_partition_rec");
        inv_partition_persistent_kernel<kIpRec><<<grid, kIpBlock, 0, s>>>(rec_a, n, plan.win_bits, plan.shift1,
                                                                         2 << plan.lo_bits, claim2, rec_b, plan.tiles);
        RSQ_LAUNCH_END(ctx);
        rec = rec_b;
    }
    RSQ_CUDA(cudaGetLastError());
    return window_scatter_device(ctx, rec, n, plan.win_bits, rank);
}

__global__ void inverse_records_kernel(const u64* __restrict__ rec, u64 m, u32* __restrict__ rank) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride)
        rank[rec[i] >> 32] = static_cast<u32>(rec[i]);
}

// rank[p] = v for `len` records (p << 32 | v) in no particular order whose p's are a permutation of
// [0, len) -- one position slice of a multi-GPU build after the exchange.  Same machinery as
// inverse_device: the records are partitioned by the top bits of p (rec_a is clobbered, rec_b is
// scratch of the same size), then scattered window by window.
int inverse_from_records(reseq_cuda_ctx* ctx, u64* rec_a, size_t len, u32* rank, u64* rec_b, u32* scratch) {
    cudaStream_t s = ctx->stream;
    // (records arriving from the exchange: measured at a 378 M-position slice, 8 first-pass bits -- 181 bins, then 512 --
    //  cost 1.31 + 1.34 ms, 7 bits -- 91 bins, then 1024 -- 1.30 + 1.53: this input does not show the first-pass
    //  slowdown the suffix-array order does, so the second pass keeps the fewer bins)
    const InversePlan plan = make_inverse_plan(len, 0, ctx->opt_inverse_lo_bits > 0 ? ctx->opt_inverse_lo_bits : 8);
    if (!plan.partitioned) {
        RSQ_LAUNCH_BEGIN(ctx, "inverse_records_kernel");
        inverse_records_kernel<<<grid_for(ctx, len, 256, 4, 16), 256, 0, s>>>(rec_a, len, rank);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        return RESEQ_OK;
    }
    u32* claim1 = scratch;
    u32* claim2 = scratch + kIpMaxBins * kIpClaimStride;
    RSQ_CUDA(cudaMemsetAsync(claim1, 0, sizeof(u32) * plan.bins1 * kIpClaimStride, s));
    RSQ_CUDA(cudaMemsetAsync(claim2, 0, sizeof(u32) * (plan.buckets2 + 32), s));
    const unsigned grid = plan.tiles < static_cast<unsigned>(ctx->sm_count) * 2 ? plan.tiles : ctx->sm_count * 2;
    RSQ_LAUNCH_BEGIN(ctx, "inv_partition_rec0");
    inv_partition_persistent_kernel<kIpRec0><<<grid, kIpBlock, 0, s>>>(rec_a, len, plan.shift1, 0, plan.bins1, claim1, rec_b, plan.tiles);
    RSQ_LAUNCH_END(ctx);
    const u64* rec = rec_b;
    if (plan.lo_bits > 0) {
        RSQ_LAUNCH_BEGIN(ctx, "inv_partition_rec");
        inv_partition_persistent_kernel<kIpRec><<<grid, kIpBlock, 0, s>>>(rec_b, len, plan.win_bits, plan.shift1,
                                                                         2 << plan.lo_bits, claim2, rec_a, plan.tiles);
        RSQ_LAUNCH_END(ctx);
        rec = rec_a;
    }
    RSQ_CUDA(cudaGetLastError());
    return window_scatter_device(ctx, rec, len, plan.win_bits, rank);
}

// rank[sa[i]] = vals[i] for all i (sa a permutation): the rank rewrite of a doubling round.  Same two lean
// partition passes + window scatter as the inverse (1.3 ms at n = 139 M against 5.9 for the direct scatter).
int rank_update_device(reseq_cuda_ctx* ctx, const u32* sa, const u32* vals, size_t n, u32* rank, u64* rec_a, u64* rec_b,
                       u32* scratch) {
    cudaStream_t s = ctx->stream;
    const InversePlan plan = make_inverse_plan(n, 0, ctx->opt_inverse_lo_bits);
    if (!plan.partitioned) {
        RSQ_LAUNCH_BEGIN(ctx, "scatter_vals_kernel");
        scatter_vals_kernel<<<grid_for(ctx, n, 256, 4, 16), 256, 0, s>>>(sa, vals, n, rank);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        return RESEQ_OK;
    }
    u32* claim1 = scratch;
    u32* claim2 = scratch + kIpMaxBins * kIpClaimStride;
    RSQ_CUDA(cudaMemsetAsync(claim1, 0, sizeof(u32) * plan.bins1 * kIpClaimStride, s));
    RSQ_CUDA(cudaMemsetAsync(claim2, 0, sizeof(u32) * (plan.buckets2 + 32), s));
    const unsigned grid = plan.tiles < static_cast<unsigned>(ctx->sm_count) * 2 ? plan.tiles : ctx->sm_count * 2;
    RSQ_LAUNCH_BEGIN(ctx, "inv_partition_sa_val");
    inv_partition_persistent_kernel<kIpSaVal><<<grid, kIpBlock, 0, s>>>(sa, n, plan.shift1, 0, plan.bins1, claim1, rec_a, plan.tiles, vals);
    RSQ_LAUNCH_END(ctx);
    const u64* rec = rec_a;
    if (plan.lo_bits > 0) {
        RSQ_LAUNCH_BEGIN(ctx, "inv_partition_rec");
        inv_partition_persistent_kernel<kIpRec><<<grid, kIpBlock, 0, s>>>(rec_a, n, plan.win_bits, plan.shift1,
                                                                         2 << plan.lo_bits, claim2, rec_b, plan.tiles);
        RSQ_LAUNCH_END(ctx);
        rec = rec_b;
    }
    RSQ_CUDA(cudaGetLastError());
    return window_scatter_device(ctx, rec, n, plan.win_bits, rank);
}

// The DNA fast path on `count` records: sort on key24, finish every group from the text.
// Returns through *unfinished the number of suffixes still tied (+1 if a group was too large
// for the shared-memory window): 0 means sa_out is final.
int sort_and_refine(reseq_cuda_ctx* ctx, const u64* packed, const u64* sent, size_t n_text, u64* elems_a,
                    u64* elems_b, size_t m, bool hist_ready, u32* sa_out, int max_rounds, bool use_shortcut,
                    u32* counters, const SortWorkspace& ws, reseq_sa_stats* st, u64* unfinished) {
    cudaStream_t s = ctx->stream;
    const PassTable pt = make_passes(kElemKeyShift, 64);
    bool in_b = false;
    RSQ_TRY(onesweep_sort<u64>(ctx, elems_a, elems_b, nullptr, nullptr, m, pt, ws, hist_ready, 0, &in_b));
    st->sort_passes += pt.count;
    RSQ_OPT_IN_SMEM(ctx, refine_elems_kernel<kRefGeneral>, kRefSmem);
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(u32), s));
    const unsigned tiles = static_cast<unsigned>((m + kRefTile - 1) / kRefTile);
    RSQ_LAUNCH_BEGIN(ctx, "refine_elems_kernel");
    refine_elems_kernel<kRefGeneral><<<tiles, kRefBlock, kRefSmem, s>>>(packed, sent, n_text, in_b ? elems_b : elems_a, m,
                                                                  sa_out, max_rounds, use_shortcut, counters, nullptr, 0, 0, nullptr, nullptr, nullptr);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters, 4 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    const volatile u32* c = reinterpret_cast<volatile u32*>(ctx->pinned);
    *unfinished = static_cast<u64>(c[0]) + (c[1] ? 1u : 0u);
    if (std::getenv("RESEQ_DEBUG"))
        std::fprintf(stderr, "[reseq] refine: records=%zu tied_left=%u oversize=%u text_steps=%u\n", m, c[0], c[1], c[2]);
    st->rounds += c[2];
    st->refined_tile += m;
    return RESEQ_OK;
}

// The uniform read-set path on m records that are in (t, position) order within equal keys (the
// whole set: m = n, generated transposed; a multi-GPU rank: its bucket).  First half: four digit
// passes, the last of which reports where the whole reads landed, and one verified overlap per whole
// read into the per-read table `cov` (indexed by the read's number in the WHOLE set).
int uniform_sort_link(reseq_cuda_ctx* ctx, const u64* packed, u32 period, u64* elems_a, u64* elems_b, size_t m,
                      bool hist_ready, u32* whole, u8* cov, u32* counters, const SortWorkspace& ws, reseq_sa_stats* st,
                      const u64** sorted_out) {
    cudaStream_t s = ctx->stream;
    const u64 magic = ~0ull / period + 1;   // ceil(2^64 / period): floor(pos / period) = mulhi(pos, magic) for pos < 2^32
    const PassTable pt = make_passes(32, 64);
    bool in_b = false;
    const EmitMultiples emit = EmitMultiples::make(period, whole, counters + 4);
    RSQ_TRY(onesweep_sort<u64>(ctx, elems_a, elems_b, nullptr, nullptr, m, pt, ws, hist_ready, 0, &in_b, &emit));
    st->sort_passes += pt.count;
    const u64* sorted = in_b ? elems_b : elems_a;
    RSQ_LAUNCH_BEGIN(ctx, "link_reads_kernel");
    link_reads_kernel<<<grid_for(ctx, m / period + 1, 256, 1, 16), 256, 0, s>>>(sorted, whole, counters + 4, packed, period,
                                                                               magic, cov);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    *sorted_out = sorted;
    return RESEQ_OK;
}

int uniform_verdict(reseq_cuda_ctx* ctx, const u32* counters, size_t m, u32 period, reseq_sa_stats* st, u64* unfinished);

// Second half, under the complete `cov` table: the records become the suffix array where every
// group is proven, the others are re-sorted; *unfinished != 0 sends the caller to the general paths.
int uniform_accept_refine(reseq_cuda_ctx* ctx, const u64* packed, const u64* sent, size_t n_text, u32 period,
                          const u64* sorted, size_t m, const u8* cov, u32* headbits, u32* uncbits, u32* sa_out,
                          int max_rounds, u32* counters, reseq_sa_stats* st, u64* unfinished, bool defer_verdict = false,
                          u32* exc = nullptr) {
    cudaStream_t s = ctx->stream;
    const u64 magic = ~0ull / period + 1;
    RSQ_LAUNCH_BEGIN(ctx, "accept_uniform_kernel");
    u8* tileflags = reinterpret_cast<u8*>(uncbits + m / 32 + 2);   // carved behind the bitmap by the caller
    RSQ_CUDA(cudaMemsetAsync(tileflags, 0, m / kRefTile + 2, s));
    if ((reinterpret_cast<uintptr_t>(sorted) & 15) || (reinterpret_cast<uintptr_t>(sa_out) & 7))
        return fail(RESEQ_INVALID_ARGUMENT, "record and suffix-array buffers must be 16- / 8-byte aligned");
    if (ctx->opt_accept_quads != 0 && (reinterpret_cast<uintptr_t>(sa_out) & 15) == 0) {
        const bool use_exc = exc != nullptr && ctx->opt_accept_exc != 0 && period - 1u >= 2 * kCovExcMargin;
        const u32 thr = use_exc ? period - 1u - kCovExcMargin : 0u;
        if (use_exc) {
            const u64 reads = n_text / period;
            cov_exceptions_kernel<<<static_cast<unsigned>((reads + 255) / 256), 256, 0, s>>>(cov, reads, thr, exc);
        }
        if (use_exc)
            accept_uniform_quads_kernel<4, true><<<grid_for(ctx, m, 256, 8, 8), 256, 0, s>>>(sorted, m, cov, period, magic, sa_out, headbits,
                                                                                            uncbits, tileflags, exc, thr);
        else
            accept_uniform_quads_kernel<4, false><<<grid_for(ctx, m, 256, 8, 8), 256, 0, s>>>(sorted, m, cov, period, magic, sa_out, headbits,
                                                                                             uncbits, tileflags, nullptr, 0u);
    }
    else
        accept_uniform_kernel<<<grid_for(ctx, m, 256, 8, 8), 256, 0, s>>>(sorted, m, cov, period, magic, sa_out, headbits,
                                                                         uncbits, tileflags);
    RSQ_LAUNCH_END(ctx);
    RSQ_OPT_IN_SMEM(ctx, refine_elems_kernel<kRefUniform>, kRefSmem);
    const unsigned tiles = static_cast<unsigned>((m + kRefTile - 1) / kRefTile);
    RSQ_LAUNCH_BEGIN(ctx, "refine_uniform_kernel");
    refine_elems_kernel<kRefUniform><<<tiles, kRefBlock, kRefSmem, s>>>(packed, sent, n_text, sorted, m, sa_out, max_rounds, true,
                                                                 counters, cov, period, magic, headbits, uncbits,
                                                                 tileflags);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    if (defer_verdict) return RESEQ_OK;   // the caller reads the counters after queueing what follows
    return uniform_verdict(ctx, counters, m, period, st, unfinished);
}

// Reads the counters of the uniform path (one stream synchronisation): *unfinished != 0 means the
// suffix array is not final (tied suffixes left, an oversize group, or a text that is not the uniform
// read set it was taken for).
int uniform_verdict(reseq_cuda_ctx* ctx, const u32* counters, size_t m, u32 period, reseq_sa_stats* st, u64* unfinished) {
    cudaStream_t s = ctx->stream;
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters, 4 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    const volatile u32* c = reinterpret_cast<volatile u32*>(ctx->pinned);
    *unfinished = static_cast<u64>(c[0]) + (c[1] ? 1u : 0u) + c[3];
    if (std::getenv("RESEQ_DEBUG"))
        std::fprintf(stderr, "[reseq] uniform refine: records=%zu period=%u tied_left=%u oversize=%u steps=%u misplaced_sentinels=%u\n",
                     m, period, c[0], c[1], c[2], c[3]);
    if (*unfinished == 0) {
        st->rounds += c[2];
        st->refined_tile += m;
    }
    return RESEQ_OK;
}

// The whole set on one device: transposed records, then both halves.  *unfinished != 0 (a read set
// that is not uniform after all, an oversize group, a step limit) sends the caller to the general paths.
int uniform_sort_and_refine(reseq_cuda_ctx* ctx, const u64* packed, const u64* sent, size_t n, u32 period, u64 k,
                            u64* elems_a, u64* elems_b, u8* cov, u32* headbits, u32* uncbits, u32* whole, u32* sa_out,
                            int max_rounds, u32* counters,
                            const SortWorkspace& ws, reseq_sa_stats* st, u64* unfinished, bool defer_verdict = false,
                            const u32* spec_flags = nullptr) {
    cudaStream_t s = ctx->stream;
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(u32), s));
    if (spec_flags) {   // speculative launch: what the pack kernel found must be what the route was chosen on
        RSQ_LAUNCH_BEGIN(ctx, "route_check_kernel");
        route_check_kernel<<<1, 1, 0, s>>>(spec_flags, static_cast<u32>(k), counters + 3);
        RSQ_LAUNCH_END(ctx);
    }
    RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * 4 * kRadix, s));
    RSQ_CUDA(cudaMemsetAsync(counters + 60, 0, sizeof(u32) * 2, s));   // the accept pass's Bloom word of short proofs
    RSQ_CUDA(cudaMemsetAsync(cov, 0, k, s));
    RSQ_LAUNCH_BEGIN(ctx, "uniform_check_kernel");
    uniform_check_kernel<<<static_cast<unsigned>((k + 255) / 256), 256, 0, s>>>(sent, period, k, counters + 3);
    RSQ_LAUNCH_END(ctx);
    RSQ_LAUNCH_BEGIN(ctx, "gen_uniform_kernel");
    gen_uniform_kernel<<<static_cast<unsigned>((k + kUniReads - 1) / kUniReads), 256, 0, s>>>(packed, period, 0, k,
                                                                                             elems_a, ws.hist);
    RSQ_LAUNCH_END(ctx);
    RSQ_LAUNCH_BEGIN(ctx, "uniform_hist_kernel");
    uniform_hist_kernel<<<1, kRadix, 0, s>>>(ws.hist, k);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    const u64* sorted = nullptr;
    RSQ_TRY(uniform_sort_link(ctx, packed, period, elems_a, elems_b, n, true, whole, cov, counters, ws, st, &sorted));
    // (counters + 60, + 61: the Bloom word of short proofs; the whole table `cov` is this device's)
    return uniform_accept_refine(ctx, packed, sent, n, period, sorted, n, cov, headbits, uncbits, sa_out, max_rounds,
                                 counters, st, unfinished, defer_verdict, counters + 60);
}

// The ragged read-set route on one device.  *applicable = false: not this kind of text (a read longer
// than 254 bases, too many short reads, no final separator) -- nothing was done; otherwise *unfinished as
// for the uniform route.
int ragged_sort_and_refine(reseq_cuda_ctx* ctx, const u64* packed, const u64* sent, size_t n, u64 k, u64* elems_a, u64* elems_b,
                           u32* headbits, u32* uncbits, u32* whole, u32* sa_out, int max_rounds, u32* counters,
                           const SortWorkspace& ws, reseq_sa_stats* st, bool* applicable, u64* unfinished) {
    cudaStream_t s = ctx->stream;
    *applicable = false;
    *unfinished = 0;
    if (k == 0 || k > n / kRagMinAvg || n >= (1ull << 32) - 64) return RESEQ_OK;
    const u64 words = (n + 63) >> 6;
    u32* cum = ctx->alloc<u32>(n / 64 + 2);
    u32* popc = ctx->alloc<u32>(n / 64 + 2);
    u32* ends = ctx->alloc<u32>(n / kRagMinAvg + 2);
    u32* covbits = ctx->alloc<u32>(n / 32 + 2);
    u32* counts = ctx->alloc<u32>(ragged_cells(n));
    u32* offsets = ctx->alloc<u32>(ragged_cells(n));
    u64* d_total = ctx->alloc<u64>(1);
    if (!cum || !popc || !ends || !covbits || !counts || !offsets || !d_total)
        return fail(RESEQ_OUT_OF_MEMORY, "ragged read-set workspace does not fit the reserved arena");
    // -- rank structure of the sentinel bitmap, separator positions, the longest read ----------------
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(u32), s));
    RSQ_LAUNCH_BEGIN(ctx, "sent_popc_kernel");
    sent_popc_kernel<<<grid_for(ctx, words, 256, 4, 8), 256, 0, s>>>(sent, words, popc);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_TRY(exclusive_scan_device(ctx, popc, cum, words, d_total));
    RSQ_LAUNCH_BEGIN(ctx, "ends_kernel");
    ends_kernel<<<grid_for(ctx, words, 256, 4, 8), 256, 0, s>>>(sent, cum, words, ends);
    RSQ_LAUNCH_END(ctx);
    RSQ_LAUNCH_BEGIN(ctx, "maxlen_kernel");
    maxlen_kernel<<<grid_for(ctx, k, 256, 4, 8), 256, 0, s>>>(ends, k, counters + 5);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters + 5, sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned + 1, ends + (k - 1), sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    const u32 tmax = *reinterpret_cast<volatile u32*>(ctx->pinned);
    const u32 last_sep = *reinterpret_cast<volatile u32*>(ctx->pinned + 1);
    if (tmax > kRagMaxLen || static_cast<u64>(last_sep) + 1 != n) return RESEQ_OK;   // a long read, or text behind the last separator
    *applicable = true;
    // -- records in (terminator distance, position) order: count, scan, write ---------------------------
    const u32 tiles = static_cast<u32>((k + kRagReads - 1) / kRagReads);
    const size_t cells = static_cast<size_t>(tiles) * (tmax + 1);
    RSQ_CUDA(cudaMemsetAsync(counts + cells, 0, sizeof(u32), s));
    RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * 4 * kRadix, s));
    RSQ_CUDA(cudaMemsetAsync(covbits, 0, sizeof(u32) * (n / 32 + 2), s));
    RSQ_LAUNCH_BEGIN(ctx, "ragged_count_kernel");
    ragged_count_kernel<<<tiles, kRagReads, 0, s>>>(packed, ends, k, tiles, tmax, counts);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_TRY(exclusive_scan_device(ctx, counts, offsets, cells + 1, d_total));
    RSQ_LAUNCH_BEGIN(ctx, "ragged_write_kernel");
    ragged_write_kernel<<<tiles, kRagReads, 0, s>>>(packed, ends, k, tiles, tmax, offsets, elems_a, ws.hist);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    // -- four digit passes; the last reports where the whole reads landed; one verified overlap per read --
    const PassTable pt = make_passes(32, 64);
    bool in_b = false;
    const EmitStarts emit{sent, whole, counters + 4};
    RSQ_TRY(onesweep_sort<u64>(ctx, elems_a, elems_b, nullptr, nullptr, n, pt, ws, true, 0, &in_b, nullptr, &emit));
    st->sort_passes += pt.count;
    const u64* sorted = in_b ? elems_b : elems_a;
    RSQ_LAUNCH_BEGIN(ctx, "link_ragged_kernel");
    link_ragged_kernel<<<grid_for(ctx, k, 256, 1, 16), 256, 0, s>>>(sorted, n, whole, counters + 4, packed, sent, cum, ends, covbits);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    // -- accept / refine under the proof bits -----------------------------------------------------------------
    u8* tileflags = reinterpret_cast<u8*>(uncbits + n / 32 + 2);
    RSQ_CUDA(cudaMemsetAsync(tileflags, 0, n / kRefTile + 2, s));
    if ((reinterpret_cast<uintptr_t>(sorted) & 15) || (reinterpret_cast<uintptr_t>(sa_out) & 7))
        return fail(RESEQ_INVALID_ARGUMENT, "record and suffix-array buffers must be 16- / 8-byte aligned");
    RSQ_LAUNCH_BEGIN(ctx, "accept_ragged_kernel");
    if (ctx->opt_accept_quads != 0 && (reinterpret_cast<uintptr_t>(sa_out) & 15) == 0)
        accept_ragged_quads_kernel<<<grid_for(ctx, n, 256, 8, 8), 256, 0, s>>>(sorted, n, covbits, sa_out, headbits, uncbits, tileflags);
    else
        accept_ragged_kernel<<<grid_for(ctx, n, 256, 8, 8), 256, 0, s>>>(sorted, n, covbits, sa_out, headbits, uncbits, tileflags);
    RSQ_LAUNCH_END(ctx);
    RSQ_OPT_IN_SMEM(ctx, refine_elems_kernel<kRefRagged>, kRefSmem);
    const unsigned rtiles = static_cast<unsigned>((n + kRefTile - 1) / kRefTile);
    RSQ_LAUNCH_BEGIN(ctx, "refine_ragged_kernel");
    refine_elems_kernel<kRefRagged><<<rtiles, kRefBlock, kRefSmem, s>>>(packed, sent, n, sorted, n, sa_out, max_rounds, true, counters,
                                                                       reinterpret_cast<const u8*>(covbits), 0, 0, headbits, uncbits,
                                                                       tileflags, cum, ends);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters, 4 * sizeof(u32), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    const volatile u32* c = reinterpret_cast<volatile u32*>(ctx->pinned);
    *unfinished = static_cast<u64>(c[0]) + (c[1] ? 1u : 0u);
    if (std::getenv("RESEQ_DEBUG"))
        std::fprintf(stderr, "[reseq] ragged refine: records=%zu reads=%llu longest=%u tied_left=%u oversize=%u steps=%u\n", n,
                     static_cast<unsigned long long>(k), tmax, c[0], c[1], c[2]);
    if (*unfinished == 0) {
        st->rounds += c[2];
        st->refined_tile += n;
    }
    return RESEQ_OK;
}

}  // namespace

int build_sa_device(reseq_cuda_ctx* ctx, const u8* d_text, size_t n, u32* d_sa, u32* d_rank,
                    reseq_sa_stats* stats, u64* packed_out, u64* sent_out) {
    reseq_sa_stats st{};
    const uint64_t launches0 = ctx->launches;
    if (n > RESEQ_CUDA_MAX_TEXT)
        return fail(RESEQ_TEXT_TOO_LARGE, "text of length " + std::to_string(n) + " exceeds 2^32-2");
    if (n == 0) {
        if (stats) *stats = st;
        return RESEQ_OK;
    }
    cudaStream_t s = ctx->stream;

    u64* packed = packed_out ? packed_out : ctx->alloc<u64>(n / 32 + 8);
    u64* sent = sent_out ? sent_out : ctx->alloc<u64>(n / 64 + 8);
    u64* keys_a = ctx->alloc<u64>(n);
    u64* keys_b = ctx->alloc<u64>(n);
    u32* vals_b = ctx->alloc<u32>(n);
    u32* head_of = ctx->alloc<u32>(n);
    u32* rank = d_rank ? d_rank : ctx->alloc<u32>(n);
    const size_t rank_tiles = (n + kRankTile - 1) / kRankTile;
    u64* desc = ctx->alloc<u64>(rank_tiles + 4);
    u32* counters = ctx->alloc<u32>(256);  // [0] bad byte flag, [1] rerank ticket, [2] heads, [4..7] refine
    u8* cov = ctx->alloc<u8>(n / kUniMinPeriod + 2);   // one byte per read of a uniform read set
    u32* headbits = ctx->alloc<u32>(n / 32 + 2);
    u32* uncbits = ctx->alloc<u32>(n / 32 + 2 + (n / kRefTile + 2 + 3) / 4);   // + one flag byte per refine tile
    u32* inv_scratch = ctx->alloc<u32>(inverse_scratch_words(n));
    SortWorkspace ws;
    if (!packed || !sent || !keys_a || !keys_b || !vals_b || !head_of || !rank || !desc || !counters || !cov || !headbits || !uncbits || !inv_scratch)
        return fail(RESEQ_OUT_OF_MEMORY, "suffix-array workspace does not fit the reserved arena");
    RSQ_TRY(sort_workspace_carve(ctx, n, &ws));

    // -- pack, decide the alphabet ----------------------------------------------------
    RSQ_CUDA(cudaMemsetAsync(counters, 0, 1024, s));
    bool dna = false;
    u64 n_separators = 0;

    // Speculative route: the previous build on this context was a uniform read set of the same length
    // and period.  Everything is queued without a host round trip -- the route's premises (DNA bytes
    // only, k separators, one per period) are checked on the device into the same counter that reports
    // an unfinished build -- and the verdict is read once, behind the inverse.  A text of another kind
    // fails the check and is rebuilt below the ordinary way.  (Host round trips were 0.1 ms of a 5.6 ms
    // build at config 2 and a third of the 0.63 ms build at config 1.)
    if (ctx->hint_n == n && ctx->hint_period != 0 && ctx->opt_text_rounds > 0 && ctx->opt_uniform != 0 && ctx->opt_speculate != 0) {
        const u32 period = ctx->hint_period;
        const u64 k = n / period;
        u64 unfinished = 0;
        auto enqueue = [&]() -> int {   // everything up to the verdict: no host round trip, fixed launch shapes
            RSQ_TRY(pack_dna_device(ctx, d_text, n, packed, sent, counters + 16, nullptr, nullptr));
            RSQ_TRY(uniform_sort_and_refine(ctx, packed, sent, n, period, k, keys_a, keys_b, cov, headbits, uncbits, vals_b, d_sa,
                                            ctx->opt_text_rounds, counters + 4, ws, &st, &unfinished, true, counters + 16));
            RSQ_TRY(ctx->sa_ready(d_sa, n));
            return inverse_device(ctx, d_sa, n, rank, keys_a, keys_b, inv_scratch);
        };
        // One CUDA graph per (text, outputs, arena, stream, options): device-resident builds on a stream of the
        // caller's (capture is not allowed on the legacy default stream), no profiling events, no copy-out stream.
        auto& g = ctx->spec_graph;
        const bool graphable = ctx->opt_graph != 0 && !ctx->profiling && ctx->sa_host_dst == nullptr && packed_out == nullptr &&
                               sent_out == nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread && s != nullptr;
        const bool same = g.exec && g.n == n && g.period == period && g.text == d_text && g.sa == d_sa && g.rank == rank &&
                          g.arena == ctx->arena && g.arena_cap == ctx->arena_cap && g.stream == s && g.epoch == ctx->option_epoch;
        bool done = false;
        if (graphable && same) {
            RSQ_CUDA(cudaGraphLaunch(g.exec, s));
            st = g.stats;
            ctx->launches += g.launches;
            done = true;
        } else if (graphable) {
            ctx->drop_spec_graph();
            const uint64_t l0 = ctx->launches;
            if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                (void)cudaMemsetAsync(counters, 0, 1024, s);   // the counters' reset belongs to the graph: it is replayed with it
                const int rc = enqueue();
                cudaGraph_t graph = nullptr;
                const cudaError_t ce = cudaStreamEndCapture(s, &graph);
                if (rc == RESEQ_OK && ce == cudaSuccess && graph &&
                    cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess) {
                    g.n = n; g.period = period; g.text = d_text; g.sa = d_sa; g.rank = rank;
                    g.arena = ctx->arena; g.arena_cap = ctx->arena_cap; g.stream = s; g.epoch = ctx->option_epoch;
                    g.launches = ctx->launches - l0;
                    g.stats = st;
                    RSQ_CUDA(cudaGraphLaunch(g.exec, s));
                    done = true;
                } else {
                    g.exec = nullptr;
                    ctx->launches = l0;
                    st = reseq_sa_stats{};
                }
                if (graph) cudaGraphDestroy(graph);
                cudaGetLastError();   // a failed capture leaves nothing enqueued: the plain launches below take over
            }
        }
        if (!done) RSQ_TRY(enqueue());
        RSQ_TRY(uniform_verdict(ctx, counters + 4, n, period, &st, &unfinished));
        if (unfinished == 0) {
            st.alphabet = 0;
            st.init_symbols = kUniK;
            st.kernel_launches = ctx->launches - launches0;
            if (stats) *stats = st;
            return RESEQ_OK;
        }
        ctx->hint_n = 0;          // not that kind of text (any more): decide afresh
        ctx->drop_spec_graph();
        st = reseq_sa_stats{};
        if (ctx->sa_host_dst == nullptr && ctx->sa_host_saved != nullptr) ctx->sa_host_dst = ctx->sa_host_saved;   // the early copy-out took the wrong array
        RSQ_CUDA(cudaMemsetAsync(counters, 0, 1024, s));
    }
    RSQ_TRY(pack_dna_device(ctx, d_text, n, packed, sent, counters + 16, &dna, &n_separators));
    // The distance shortcut pays off on read sets (a sentinel every <= 1024 symbols on average);
    // on sentinel-free texts no group could use it.
    const bool use_shortcut = ctx->opt_shortcut != 0 && n_separators * 1024 >= n;
    st.alphabet = dna ? 0 : 1;

    // -- uniform read sets (k reads of one length, the shotgun configurations): transposed records,
    //    4 digit passes, groups accepted in (terminator distance, position) order ------------------
    if (dna && ctx->opt_text_rounds > 0 && ctx->opt_uniform != 0 && n_separators > 0 && n % n_separators == 0 &&
        n / n_separators >= kUniMinPeriod && n / n_separators <= kUniMaxPeriod) {
        u64 unfinished = 0;
        RSQ_TRY(uniform_sort_and_refine(ctx, packed, sent, n, static_cast<u32>(n / n_separators), n_separators, keys_a,
                                        keys_b, cov, headbits, uncbits, vals_b /* n words: the whole reads' indices */, d_sa,
                                        ctx->opt_text_rounds, counters + 4, ws, &st, &unfinished));
        if (unfinished == 0) {
            st.init_symbols = kUniK;
            RSQ_TRY(ctx->sa_ready(d_sa, n));
            RSQ_TRY(inverse_device(ctx, d_sa, n, rank, keys_a, keys_b, inv_scratch));
            st.kernel_launches = ctx->launches - launches0;
            if (stats) *stats = st;
            ctx->hint_n = n;   // the next build of a text this long starts on this route without asking
            ctx->hint_period = static_cast<u32>(n / n_separators);
            return RESEQ_OK;
        }
        st.sort_passes = 0;   // not uniform after all, or a group the window cannot hold: the general paths
    }

    // -- ragged read sets (reads of mixed lengths <= 254): the uniform route's flow with looked-up
    //    terminator distances, records born transposed with ragged rows ---------------------------------
    if (dna && ctx->opt_text_rounds > 0 && ctx->opt_uniform != 0 && ctx->opt_ragged != 0 && n_separators > 0) {
        bool applicable = false;
        u64 unfinished = 0;
        RSQ_TRY(ragged_sort_and_refine(ctx, packed, sent, n, n_separators, keys_a, keys_b, headbits, uncbits, vals_b, d_sa,
                                       ctx->opt_text_rounds, counters + 4, ws, &st, &applicable, &unfinished));
        if (applicable && unfinished == 0) {
            st.init_symbols = kRagK;
            RSQ_TRY(ctx->sa_ready(d_sa, n));
            RSQ_TRY(inverse_device(ctx, d_sa, n, rank, keys_a, keys_b, inv_scratch));
            st.kernel_launches = ctx->launches - launches0;
            if (stats) *stats = st;
            return RESEQ_OK;
        }
        st.sort_passes = 0;
    }

    // -- DNA fast path: 12-base records, 3 digit passes, groups finished from the L2-resident text --
    if (dna && ctx->opt_text_rounds > 0) {
        RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * 3 * kRadix, s));
        RSQ_LAUNCH_BEGIN(ctx, "init_elems_kernel");
        init_elems_kernel<<<grid_for(ctx, n, 256, 8, 8), 256, 0, s>>>(packed, sent, n, 0, n, keys_a, ws.hist);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        u64 unfinished = 0;
        RSQ_TRY(sort_and_refine(ctx, packed, sent, n, keys_a, keys_b, n, true, d_sa, ctx->opt_text_rounds, use_shortcut,
                                counters + 4, ws, &st, &unfinished));
        st.init_symbols = kElemK;
        if (unfinished == 0) {
            RSQ_TRY(ctx->sa_ready(d_sa, n));
            RSQ_TRY(inverse_device(ctx, d_sa, n, rank, keys_a, keys_b, inv_scratch));
            st.kernel_launches = ctx->launches - launches0;
            if (stats) *stats = st;
            return RESEQ_OK;
        }
        // a group outgrew the window or the step limit: rebuild with the general engine
    }

    // -- general engine: k-mer initial ranks, then prefix doubling (any alphabet, any group size) --
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
    // three n-word arrays change roles from round to round: the current order, the group-head index of
    // every slot, and a spare
    u32* sa_cur = in_b ? vals_b : d_sa;
    u32* spare = in_b ? d_sa : vals_b;
    u32* heads_of = head_of;

    // group heads from adjacent sorted keys (max-scan with look-back); rank is rewritten by the partitioned scatter
    auto rerank = [&](auto* keys, u32 uniq_mask, u32 uniq_full) -> int {
        RSQ_CUDA(cudaMemsetAsync(desc, 0, sizeof(u64) * (rank_tiles + 4), s));
        RSQ_CUDA(cudaMemsetAsync(counters + 1, 0, 2 * sizeof(u32), s));
        using K = std::remove_pointer_t<decltype(keys)>;
        RSQ_LAUNCH_BEGIN(ctx, "rerank_kernel");
        rerank_kernel<K, false><<<static_cast<unsigned>(rank_tiles), kRankBlock, 0, s>>>(
            keys, sa_cur, n, uniq_mask, uniq_full, rank, heads_of, desc, counters + 1, counters + 2);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters + 2, sizeof(u32), cudaMemcpyDeviceToHost, s));
        return RESEQ_OK;
    };
    // (the sort's key buffers are free between the sort and the next key generation: they carry the
    //  partition records of the rank update)
    auto update_rank = [&]() -> int { return rank_update_device(ctx, sa_cur, heads_of, n, rank, keys_a, keys_b, inv_scratch); };

    const u32 field_mask = (1u << (dna ? kDnaFieldBits : kByteFieldBits)) - 1u;
    const u32 field_full = 2u * (dna ? kDnaK : kByteK);
    RSQ_TRY(rerank(in_b ? k32_b : k32_a, field_mask, field_full));
    RSQ_TRY(update_rank());
    RSQ_CUDA(cudaStreamSynchronize(s));
    u64 heads = *reinterpret_cast<volatile u32*>(ctx->pinned);

    const int b = static_cast<int>(bit_width_u64(n));
    const PassTable pt = make_passes(0, 2 * b);
    const unsigned dbl_tiles = static_cast<unsigned>((n + kDblTile - 1) / kDblTile);
    for (u64 h = st.init_symbols; heads < n && h < n; h <<= 1) {
        // -- local form: every group ordered in shared memory by the CTA that owns it -------------------
        bool oversize = false;
        if (ctx->opt_doubling_local != 0) {
            RSQ_CUDA(cudaMemsetAsync(counters + 1, 0, 2 * sizeof(u32), s));
            RSQ_LAUNCH_BEGIN(ctx, "double_local_kernel");
            double_local_kernel<<<dbl_tiles, kDblBlock, 0, s>>>(sa_cur, heads_of, rank, n, h, spare, counters + 1);
            RSQ_LAUNCH_END(ctx);
            RSQ_CUDA(cudaGetLastError());
            RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, counters + 1, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
            { u32* t = heads_of; heads_of = spare; spare = t; }
            RSQ_CUDA(cudaStreamSynchronize(s));
            heads = reinterpret_cast<volatile u32*>(ctx->pinned)[0];
            oversize = reinterpret_cast<volatile u32*>(ctx->pinned)[1] != 0;
            st.refined_tile += n;
        }
        // -- global form: (group, rank2) pairs of all suffixes through the digit passes -- groups too large
        //    for a CTA's window (deeply repetitive texts), or when the local form is switched off --------
        if (oversize || ctx->opt_doubling_local == 0) {
            RSQ_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(u32) * pt.count * kRadix, s));
            {
                const unsigned grid = grid_for(ctx, n, 256, 8, 8);
                RSQ_LAUNCH_BEGIN(ctx, "pair_key_kernel");
                pair_key_kernel<<<grid, 256, sizeof(u32) * pt.count * kRadix, s>>>(
                    sa_cur, heads_of, rank, n, h, b, keys_a, pt, ws.hist);
                RSQ_LAUNCH_END(ctx);
                RSQ_CUDA(cudaGetLastError());
            }
            RSQ_TRY(onesweep_sort<u64>(ctx, keys_a, keys_b, sa_cur, spare, n, pt, ws, true, 0, &in_b));
            st.sort_passes += pt.count;
            if (in_b) { u32* t = sa_cur; sa_cur = spare; spare = t; }
            RSQ_TRY(rerank(in_b ? keys_b : keys_a, 0u, 0u));
            RSQ_CUDA(cudaStreamSynchronize(s));
            heads = *reinterpret_cast<volatile u32*>(ctx->pinned);
            st.refined_global += n;
        }
        RSQ_TRY(update_rank());
        ++st.rounds;
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
    // uniform read sets: period = read length + 1 (0: not uniform), number of reads; the bucket
    // between uniform_sort_link and uniform_finish (arrays in the context's arena)
    rsq::u32 period = 0;
    rsq::u64 reads = 0;
    const rsq::u64* u_sorted = nullptr;
    rsq::u32* u_headbits = nullptr;
    rsq::u32* u_uncbits = nullptr;
    rsq::u32* u_counters = nullptr;
    size_t u_m = 0;
    // bucket between reseq_cuda_sa_shard_bucket_size and _bucket_records (arrays in the context's arena)
    rsq::u32 b_plo = 0, b_phi = 0, b_tiles = 0;
    rsq::u32* b_offsets = nullptr;
    rsq::u32* b_keep = nullptr;
    unsigned short* b_wbase = nullptr;
    size_t b_m = 0;
    bool b_ready = false;
    rsq::u32* b_hist = nullptr;     // [4][256] digit histograms of the bucket written last (own allocation)
    bool b_hist_valid = false;
    const void* b_records = nullptr;   // ... which is this array
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
    // stream-ordered pool allocations (cached across shards: a build per step pays no cudaMalloc)
    if (cudaMallocAsync(&sh->packed, sizeof(u64) * (n / 32 + 8), ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&sh->sent, sizeof(u64) * (n / 64 + 8), ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&sh->flags, 256, ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&sh->b_hist, sizeof(u32) * 4 * kRadix, ctx->stream) != cudaSuccess) {
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
    if (sh->dna && ctx->opt_uniform != 0 && n_sep > 0 && n % n_sep == 0 && n / n_sep >= kUniMinPeriod &&
        n / n_sep <= kUniMaxPeriod) {   // k sentinels, one period apart?
        const u32 period = static_cast<u32>(n / n_sep);
        cudaMemsetAsync(sh->flags + 8, 0, sizeof(u32), ctx->stream);
        RSQ_LAUNCH_BEGIN(ctx, "uniform_check_kernel");
        uniform_check_kernel<<<static_cast<unsigned>((n_sep + 255) / 256), 256, 0, ctx->stream>>>(sh->sent, period, n_sep,
                                                                                             sh->flags + 8);
        RSQ_LAUNCH_END(ctx);
        cudaMemcpyAsync(ctx->pinned, sh->flags + 8, sizeof(u32), cudaMemcpyDeviceToHost, ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
            reseq_cuda_sa_shard_destroy(sh);
            return fail(RESEQ_CUDA_ERROR, "uniform read-set check failed");
        }
        if (*reinterpret_cast<volatile u32*>(ctx->pinned) == 0) {
            sh->period = period;
            sh->reads = n_sep;
        }
    }
    if (is_dna) *is_dna = sh->dna ? 1 : 0;
    *out = sh;
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_uniform_info(const reseq_cuda_sa_shard* sh, uint32_t* period, uint64_t* reads) {
    if (!sh) return rsq::fail(RESEQ_INVALID_ARGUMENT, "null shard");
    if (period) *period = sh->period;
    if (reads) *reads = sh->reads;
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_uniform_records(reseq_cuda_sa_shard* sh, uint64_t read_begin, size_t read_count,
                                        uint64_t* d_records) {
    using namespace rsq;
    if (!sh || !sh->period) return fail(RESEQ_INVALID_ARGUMENT, "not a uniform read set");
    if (read_count == 0) return RESEQ_OK;
    if (read_begin + read_count > sh->reads || !d_records) return fail(RESEQ_INVALID_ARGUMENT, "read slice out of range");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    RSQ_TRY(ctx->reserve(reseq_cuda_ctx::padded(sizeof(u32) * 4 * kRadix) + 4096));
    ctx->begin();
    u32* hist = ctx->alloc<u32>(4 * kRadix);   // the slice's histogram is not used: buckets re-count
    if (!hist) return fail(RESEQ_OUT_OF_MEMORY, "shard workspace");
    RSQ_CUDA(cudaMemsetAsync(hist, 0, sizeof(u32) * 4 * kRadix, ctx->stream));
    RSQ_LAUNCH_BEGIN(ctx, "gen_uniform_kernel");
    gen_uniform_kernel<<<static_cast<unsigned>((read_count + kUniReads - 1) / kUniReads), 256, 0, ctx->stream>>>(
        sh->packed, sh->period, read_begin, read_count, d_records, hist);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_uniform_sort_link(reseq_cuda_sa_shard* sh, uint64_t* d_records, size_t m, uint8_t* d_cov) {
    using namespace rsq;
    if (!sh || !sh->period || !d_cov) return fail(RESEQ_INVALID_ARGUMENT, "bad shard argument");
    sh->u_m = m;
    sh->u_sorted = nullptr;
    if (m == 0) return RESEQ_OK;
    if (!d_records) return fail(RESEQ_INVALID_ARGUMENT, "null records");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    auto pad = reseq_cuda_ctx::padded;
    const size_t bits = m / 32 + 2 + (m / kRefTile + 2 + 3) / 4;
    RSQ_TRY(ctx->reserve(pad(sizeof(u64) * m) + pad(sizeof(u32) * m) + 2 * pad(sizeof(u32) * bits) + pad(1024) +
                         sort_workspace_bytes(m) + 8192));
    ctx->begin();
    u64* rec_b = ctx->alloc<u64>(m);
    u32* whole = ctx->alloc<u32>(m);
    sh->u_headbits = ctx->alloc<u32>(bits);
    sh->u_uncbits = ctx->alloc<u32>(bits);
    sh->u_counters = ctx->alloc<u32>(64);
    SortWorkspace ws;
    if (!rec_b || !whole || !sh->u_headbits || !sh->u_uncbits || !sh->u_counters)
        return fail(RESEQ_OUT_OF_MEMORY, "shard workspace");
    RSQ_TRY(sort_workspace_carve(ctx, m, &ws));
    RSQ_CUDA(cudaMemsetAsync(sh->u_counters, 0, 8 * sizeof(u32), ctx->stream));
    reseq_sa_stats st{};
    const bool hist_ready = sh->b_hist_valid && sh->b_records == d_records && sh->b_m == m;   // written by bucket_records
    sh->b_hist_valid = false;
    if (hist_ready) RSQ_CUDA(cudaMemcpyAsync(ws.hist, sh->b_hist, sizeof(u32) * 4 * kRadix, cudaMemcpyDeviceToDevice, ctx->stream));
    // stable passes: equal keys keep the (t, position) order the bucket was born in
    return uniform_sort_link(ctx, sh->packed, sh->period, d_records, rec_b, m, hist_ready, whole, d_cov, sh->u_counters, ws,
                             &st, &sh->u_sorted);
}

int reseq_cuda_sa_shard_uniform_finish(reseq_cuda_sa_shard* sh, const uint8_t* d_cov, uint32_t* d_sa_out,
                                       uint64_t* unfinished) {
    using namespace rsq;
    if (!sh || !sh->period || !d_cov || !unfinished) return fail(RESEQ_INVALID_ARGUMENT, "bad shard argument");
    *unfinished = 0;
    if (sh->u_m == 0) return RESEQ_OK;
    if (!sh->u_sorted || !d_sa_out) return fail(RESEQ_INVALID_ARGUMENT, "uniform_finish must follow uniform_sort_link");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    reseq_sa_stats st{};
    const int status = uniform_accept_refine(ctx, sh->packed, sh->sent, sh->n, sh->period, sh->u_sorted, sh->u_m, d_cov,
                                             sh->u_headbits, sh->u_uncbits, d_sa_out, 1 << 20, sh->u_counters, &st,
                                             unfinished);
    sh->u_sorted = nullptr;
    return status;
}

void reseq_cuda_sa_shard_destroy(reseq_cuda_sa_shard* sh) {
    if (!sh) return;
    if (sh->ctx) {
        cudaSetDevice(sh->ctx->device);
        cudaStreamSynchronize(sh->ctx->stream);
    }
    cudaStream_t st = sh->ctx ? sh->ctx->stream : nullptr;
    if (sh->packed) cudaFreeAsync(sh->packed, st);
    if (sh->sent) cudaFreeAsync(sh->sent, st);
    if (sh->flags) cudaFreeAsync(sh->flags, st);
    if (sh->b_hist) cudaFreeAsync(sh->b_hist, st);
    if (sh->ctx) cudaStreamSynchronize(st);
    delete sh;
}

int reseq_cuda_sa_shard_records(reseq_cuda_sa_shard* sh, uint64_t pos_begin, size_t count, uint64_t* d_records) {
    using namespace rsq;
    if (!sh || !sh->dna) return fail(RESEQ_INVALID_ARGUMENT, "the sharded build needs a DNA text");
    if (count == 0) return RESEQ_OK;
    if (pos_begin + count > sh->n) return fail(RESEQ_INVALID_ARGUMENT, "position slice out of range");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    RSQ_TRY(ctx->reserve(reseq_cuda_ctx::padded(sizeof(u32) * kMaxPasses * kRadix) + 4096));
    ctx->begin();
    u32* hist = ctx->alloc<u32>(kMaxPasses * kRadix);  // the slice's histogram is not used: buckets re-count
    RSQ_CUDA(cudaMemsetAsync(hist, 0, sizeof(u32) * 3 * kRadix, ctx->stream));
    RSQ_LAUNCH_BEGIN(ctx, "init_elems_kernel");
    init_elems_kernel<<<grid_for(ctx, count, 256, 8, 8), 256, 0, ctx->stream>>>(sh->packed, sh->sent, sh->n, pos_begin,
                                                                                  count, d_records, hist);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_finish(reseq_cuda_sa_shard* sh, uint64_t* d_records, size_t m, uint32_t* d_sa_out,
                               uint64_t* unfinished) {
    using namespace rsq;
    if (!sh || !sh->dna || !unfinished) return fail(RESEQ_INVALID_ARGUMENT, "bad shard argument");
    *unfinished = 0;
    if (m == 0) return RESEQ_OK;
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(pad(sizeof(u64) * m) + sort_workspace_bytes(m) + 8192));
    ctx->begin();
    u64* rec_b = ctx->alloc<u64>(m);
    u32* counters = ctx->alloc<u32>(64);
    SortWorkspace ws;
    if (!rec_b || !counters) return fail(RESEQ_OUT_OF_MEMORY, "shard workspace");
    RSQ_TRY(sort_workspace_carve(ctx, m, &ws));
    // stable sort of the bucket on the 24-bit key: equal keys stay in ascending position order
    // because the exchange delivers the slices in rank (= position) order
    reseq_sa_stats st{};
    const bool hist_ready = sh->b_hist_valid && sh->b_records == d_records && sh->b_m == m;   // written by bucket_records
    sh->b_hist_valid = false;
    if (hist_ready) RSQ_CUDA(cudaMemcpyAsync(ws.hist, sh->b_hist, sizeof(u32) * 3 * kRadix, cudaMemcpyDeviceToDevice, ctx->stream));
    RSQ_TRY(sort_and_refine(ctx, sh->packed, sh->sent, sh->n, d_records, rec_b, m, hist_ready, d_sa_out, 1 << 20,
                            sh->use_shortcut, counters, ws, &st, unfinished));
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_prefix_hist(reseq_cuda_sa_shard* sh, uint64_t unit_begin, size_t unit_count, uint32_t* d_hist) {
    using namespace rsq;
    if (!sh || !sh->dna || !d_hist) return fail(RESEQ_INVALID_ARGUMENT, "the sharded build needs a DNA text");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    RSQ_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(u32) << kShPrefixBits, ctx->stream));
    if (unit_count == 0) return RESEQ_OK;
    if (sh->period) {
        if (unit_begin + unit_count > sh->reads) return fail(RESEQ_INVALID_ARGUMENT, "read slice out of range");
        RSQ_LAUNCH_BEGIN(ctx, "shard_hist_uniform_kernel");
        shard_hist_uniform_kernel<<<static_cast<unsigned>((unit_count + kShReads - 1) / kShReads), kShReads, 0, ctx->stream>>>(
            sh->packed, sh->period, unit_begin, unit_count, d_hist);
        RSQ_LAUNCH_END(ctx);
    } else {
        if (unit_begin + unit_count > sh->n) return fail(RESEQ_INVALID_ARGUMENT, "position slice out of range");
        RSQ_LAUNCH_BEGIN(ctx, "shard_hist_general_kernel");
        shard_hist_general_kernel<<<grid_for(ctx, unit_count, 256, 8, 8), 256, 0, ctx->stream>>>(sh->packed, sh->sent, sh->n,
                                                                                               unit_begin, unit_count, d_hist);
        RSQ_LAUNCH_END(ctx);
    }
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_bucket_size(reseq_cuda_sa_shard* sh, uint32_t prefix_lo, uint32_t prefix_hi, uint64_t* m) {
    using namespace rsq;
    if (!sh || !sh->dna || !m) return fail(RESEQ_INVALID_ARGUMENT, "the sharded build needs a DNA text");
    if (prefix_lo > prefix_hi || prefix_hi > (1u << kShPrefixBits)) return fail(RESEQ_INVALID_ARGUMENT, "prefix range out of order");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    sh->b_ready = false;
    const u64 units = sh->period ? sh->reads : sh->n;
    const u32 tiles = static_cast<u32>(sh->period ? (units + kShReads - 1) / kShReads : (units + kShTile - 1) / kShTile);
    const size_t cells = sh->period ? static_cast<size_t>(tiles) * sh->period : tiles;
    const size_t wcells = sh->period ? cells * (kShReads / 32) : 0;   // per-warp keep masks and bases (uniform read sets)
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(2 * pad(sizeof(u32) * (cells + 1)) + pad(sizeof(u32) * (wcells + 1)) + pad(sizeof(unsigned short) * (wcells + 1)) +
                         scan_workspace_bytes(cells + 1) + 8192));
    ctx->begin();
    u32* counts = ctx->alloc<u32>(cells + 1);
    u32* offsets = ctx->alloc<u32>(cells + 1);
    u32* keep = ctx->alloc<u32>(wcells + 1);
    unsigned short* wbase = ctx->alloc<unsigned short>(wcells + 1);
    u64* d_total = ctx->alloc<u64>(1);
    if (!counts || !offsets || !keep || !wbase || !d_total) return fail(RESEQ_OUT_OF_MEMORY, "shard workspace");
    RSQ_CUDA(cudaMemsetAsync(counts + cells, 0, sizeof(u32), s));
    if (sh->period) {
        RSQ_LAUNCH_BEGIN(ctx, "shard_count_uniform_kernel");
        shard_count_uniform_kernel<<<tiles, kShReads, 0, s>>>(sh->packed, sh->period, sh->reads, prefix_lo, prefix_hi, tiles, counts,
                                                              keep, wbase);
        RSQ_LAUNCH_END(ctx);
    } else {
        RSQ_LAUNCH_BEGIN(ctx, "shard_count_general_kernel");
        shard_general_kernel<false><<<tiles, 256, 0, s>>>(sh->packed, sh->sent, sh->n, prefix_lo, prefix_hi, counts, nullptr, nullptr, nullptr);
        RSQ_LAUNCH_END(ctx);
    }
    RSQ_CUDA(cudaGetLastError());
    RSQ_TRY(exclusive_scan_device(ctx, counts, offsets, cells + 1, d_total));
    RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_total, sizeof(u64), cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    sh->b_m = *reinterpret_cast<volatile u64*>(ctx->pinned);
    sh->b_plo = prefix_lo;
    sh->b_phi = prefix_hi;
    sh->b_tiles = tiles;
    sh->b_offsets = offsets;
    sh->b_keep = keep;
    sh->b_wbase = wbase;
    sh->b_ready = true;
    *m = sh->b_m;
    return RESEQ_OK;
}

int reseq_cuda_sa_shard_bucket_records(reseq_cuda_sa_shard* sh, uint64_t* d_records) {
    using namespace rsq;
    if (!sh || !sh->b_ready) return fail(RESEQ_INVALID_ARGUMENT, "bucket_records must follow bucket_size on the same shard");
    sh->b_ready = false;
    if (sh->b_m == 0) return RESEQ_OK;
    if (!d_records) return fail(RESEQ_INVALID_ARGUMENT, "null records");
    reseq_cuda_ctx* ctx = sh->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    RSQ_CUDA(cudaMemsetAsync(sh->b_hist, 0, sizeof(u32) * 4 * kRadix, ctx->stream));
    if (sh->period) {
        RSQ_LAUNCH_BEGIN(ctx, "shard_write_uniform_kernel");
        if (sh->b_m * 3 > sh->n)     // most suffixes are kept: lanes = reads
            shard_write_uniform_direct_kernel<<<sh->b_tiles, kShReads, 0, ctx->stream>>>(sh->packed, sh->period, sh->reads, sh->b_tiles,
                                                                                        sh->b_offsets, sh->b_keep, sh->b_wbase, d_records, sh->b_hist);
        else                         // a sparse selection: per-warp work lists
            shard_write_uniform_kernel<<<sh->b_tiles, kShReads, 0, ctx->stream>>>(sh->packed, sh->period, sh->reads, sh->b_tiles,
                                                                                 sh->b_offsets, sh->b_keep, sh->b_wbase, d_records, sh->b_hist);
        RSQ_LAUNCH_END(ctx);
    } else {
        RSQ_LAUNCH_BEGIN(ctx, "shard_write_general_kernel");
        shard_general_kernel<true><<<sh->b_tiles, 256, 0, ctx->stream>>>(sh->packed, sh->sent, sh->n, sh->b_plo, sh->b_phi, nullptr,
                                                                        sh->b_offsets, d_records, sh->b_hist);
        RSQ_LAUNCH_END(ctx);
    }
    RSQ_CUDA(cudaGetLastError());
    sh->b_hist_valid = true;    // the sort of exactly this array may skip its histogram sweep
    sh->b_records = d_records;
    return RESEQ_OK;
}

int reseq_cuda_rank_shard_partition(reseq_cuda_ctx* ctx, const uint32_t* d_sa_bucket, size_t m, uint64_t global_offset,
                                    uint64_t n, int world, uint64_t* d_records_out, uint64_t* counts_out) {
    using namespace rsq;
    if (!ctx || !counts_out || world < 1 || world > 16 || n == 0 || static_cast<uint64_t>(world) >= n || n > RESEQ_CUDA_MAX_TEXT)
        return fail(RESEQ_INVALID_ARGUMENT, "bad argument (1 <= world <= 16, world < n <= 2^32 - 2)");
    for (int g = 0; g < world; ++g) counts_out[g] = 0;
    if (m == 0) return RESEQ_OK;
    if (!d_sa_bucket || !d_records_out) return fail(RESEQ_INVALID_ARGUMENT, "null device buffer");
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    RSQ_TRY(ctx->reserve(sizeof(u32) * (kOwnMaxBins + kOwnMaxBins * kIpClaimStride) + 16384));
    ctx->begin();
    int sub_bits = 10;
    const int max_bins = ctx->opt_owner_bins >= world && ctx->opt_owner_bins <= kOwnMaxBins ? ctx->opt_owner_bins : kOwnMaxBins;
    while ((world << sub_bits) > max_bins) --sub_bits;   // owner x sub-range bins, at most 1024: the sub-bins spread the
    const int bins = world << sub_bits;                     // shared-memory atomics; the exchange sends whole owners
    u32* counts = ctx->alloc<u32>(kOwnMaxBins + kOwnMaxBins * kIpClaimStride);
    if (!counts) return fail(RESEQ_OUT_OF_MEMORY, "rank shard workspace");
    u32* claim = counts + kOwnMaxBins;   // one counter per 128-byte line
    RSQ_CUDA(cudaMemsetAsync(counts, 0, sizeof(u32) * bins, s));
    RSQ_LAUNCH_BEGIN(ctx, "owner_count_kernel");
    OwnerTable tb{};
    tb.G = static_cast<u32>(world);
    for (int g = 0; g <= world; ++g) tb.base[g] = static_cast<u64>((static_cast<unsigned __int128>(n) * g) / world);
    tb.magic = static_cast<u32>((static_cast<u64>(world) << 32) / n);   // world < n: fits 32 bits
    tb.sub = 1u << sub_bits;
    owner_count_kernel<<<grid_for(ctx, m, 256, 8, 8), 256, 0, s>>>(d_sa_bucket, m, tb, counts);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    // the bins' bases stay on the device (the partition is queued without waiting for the host); the per-owner counts
    // the exchange needs travel to the host behind it
    RSQ_LAUNCH_BEGIN(ctx, "owner_bases_kernel");
    owner_bases_kernel<<<1, kOwnMaxBins, 0, s>>>(counts, bins, claim);
    RSQ_LAUNCH_END(ctx);
    u32* h = reinterpret_cast<u32*>(ctx->pinned);   // 4096 pinned bytes: up to 1024 counters
    RSQ_CUDA(cudaMemcpyAsync(h, counts, sizeof(u32) * bins, cudaMemcpyDeviceToHost, s));
    RSQ_LAUNCH_BEGIN(ctx, "owner_partition_kernel");
    RSQ_OPT_IN_SMEM(ctx, owner_partition_kernel, kOwnSmem);
    {
        const u32 num_tiles = static_cast<u32>((m + kOwnTile - 1) / kOwnTile);
        const unsigned grid = num_tiles < 2u * static_cast<unsigned>(ctx->sm_count) ? num_tiles : 2u * static_cast<unsigned>(ctx->sm_count);
        owner_partition_kernel<<<grid, kOwnBlock, kOwnSmem, s>>>(d_sa_bucket, m, tb, global_offset, claim, d_records_out, num_tiles);
    }
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaStreamSynchronize(s));   // the counts have landed; the pinned staging words are reused by the next call
    for (int b = 0; b < bins; ++b) counts_out[b >> sub_bits] += h[b];
    return RESEQ_OK;
}

int reseq_cuda_rank_shard_finish(reseq_cuda_ctx* ctx, uint64_t* d_records, size_t len, uint32_t* d_rank_slice) {
    using namespace rsq;
    if (!ctx) return fail(RESEQ_INVALID_ARGUMENT, "null context");
    if (len == 0) return RESEQ_OK;
    if (!d_records || !d_rank_slice) return fail(RESEQ_INVALID_ARGUMENT, "null device buffer");
    RSQ_CUDA(cudaSetDevice(ctx->device));
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(pad(sizeof(u64) * len) + pad(sizeof(u32) * inverse_scratch_words(len)) + 4096));
    ctx->begin();
    u64* rec_b = ctx->alloc<u64>(len);
    u32* scratch = ctx->alloc<u32>(inverse_scratch_words(len));
    if (!rec_b || !scratch) return fail(RESEQ_OUT_OF_MEMORY, "inverse workspace");
    return inverse_from_records(ctx, d_records, len, d_rank_slice, rec_b, scratch);
}

int reseq_cuda_inverse_device(reseq_cuda_ctx* ctx, const uint32_t* d_sa, size_t n, uint32_t* d_rank) {
    using namespace rsq;
    if (!ctx) return fail(RESEQ_INVALID_ARGUMENT, "null context");
    if (n == 0) return RESEQ_OK;
    if (!d_sa || !d_rank) return fail(RESEQ_INVALID_ARGUMENT, "null device buffer");
    RSQ_CUDA(cudaSetDevice(ctx->device));
    // the partitioned inverse of the single-GPU build (two lean passes + window scatter)
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(2 * pad(sizeof(u64) * n) + pad(sizeof(u32) * inverse_scratch_words(n)) + 4096));
    ctx->begin();
    u64* rec_a = ctx->alloc<u64>(n);
    u64* rec_b = ctx->alloc<u64>(n);
    u32* scratch = ctx->alloc<u32>(inverse_scratch_words(n));
    if (!rec_a || !rec_b || !scratch) return fail(RESEQ_OUT_OF_MEMORY, "inverse workspace");
    return inverse_device(ctx, d_sa, n, d_rank, rec_a, rec_b, scratch);
}

}  // extern "C"

namespace rsq {
}  // namespace rsq
