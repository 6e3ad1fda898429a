// LSD radix sort for sm_100a: 8-bit digits, one "onesweep" kernel per digit pass.
//
//   - digit histograms for ALL passes of a sort are accumulated up front in shared
//     memory (hist_add, fused into whichever kernel produces the keys) and turned into
//     per-pass exclusive digit bases by digit_base_kernel;
//   - each pass is ONE kernel: tiles are claimed through an atomic ticket, keys are
//     ranked inside the warp by ballots (warp-aggregated: one shared-memory atomicAdd
//     per distinct digit per warp step), tile totals are
//     chained across tiles by decoupled look-back over PACKED descriptors (four 16-bit digit
//     aggregates per 64-bit word, walked by 64 threads; inclusive prefixes behind one flag per
//     tile), the tile is re-ordered through shared memory so every digit's run leaves as one
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
constexpr int kLookahead = 8;   // look-back descriptors read per round trip by each walker thread

// Look-back descriptors.  One 64-bit word is published by ONE relaxed store, so status and value are
// seen together and no fence is needed.  DPW = digits per word:
//   DPW 1: [status:2 | value:62]                      one digit, any n          (256 walker threads)
//   DPW 2: two lanes of [status:2 | value:30]         two digits, n < 2^30      (128 walker threads)
// status 0 = not published, 1 = the tile's own count (aggregate), 2 = inclusive prefix.
// Why pack: with ~450 tiles in flight a walk meets the front of finished tiles ~27 tiles back (L2 round
// trip / tile issue interval); at one digit per word the walk was 28 % of the pass's instructions and
// more L2 sectors (51 M) than the key loads (35 M) (ncu source page of profiles/r1k_ncu_full_onesweep_kernel).
// Measured and dropped: four 16-bit aggregates per word with the inclusive prefixes behind a per-tile
// flag (two fences on the chain): the longer publish latency pushed the front further back and the
// pass went from 0.76 to 1.11 ms (profiles/r2b_negative_results.md).
constexpr u32 kLaneAggregate = 1u << 30;
constexpr u32 kLaneInclusive = 2u << 30;
constexpr u32 kLaneValueMask = (1u << 30) - 1u;
constexpr u64 kPackedLimit = 1ull << 30;   // DPW 2 needs every digit count below this

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

// Lanes of the warp holding the same 8-bit digit, from one ballot per digit bit.  On sm_100a a
// pass is bound by issue slots and shared-memory wavefronts, not by HBM (ncu, profiles/
// r1c_ncu_full_onesweep_kernel.txt: ALU pipe 49 %, LSU wavefronts 54 %, DRAM 22 %), so the
// match is written to cost 4 instructions per bit (LOP3 -> predicate, VOTE, predicated NOT, AND)
// instead of the 7.6 per bit the C++ form compiled to; MATCH.ANY is slower still (its issue rate
// capped the ranking loop at 1.5 TB/s of key traffic).  Digit bits above a narrow pass's width
// are zero in every lane, so their ballots leave `peers` unchanged: all passes run 8 ballots.
__device__ __forceinline__ unsigned and3(unsigned a, unsigned b, unsigned c) {
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ unsigned warp_match_digit(u32 d) {
    unsigned m[kRadixBits];
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
        asm volatile(
            "{\n\t"
            ".reg .pred p;\n\t"
            ".reg .b32 t;\n\t"
            "and.b32 t, %1, %2;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "@!p not.b32 %0, %0;\n\t"
            "}"
            : "=r"(m[b])
            : "r"(d), "r"(1u << b));
    }
    // the eight masks meet in four three-input LOP3s instead of a chain of seven ANDs
    static_assert(kRadixBits == 8, "the AND tree is written for eight ballots");
    return and3(m[3], m[4], m[5]) & and3(m[6], m[7], and3(m[0], m[1], m[2]));
}

// What a pass reports besides sorting.  EmitMultiples: the OUTPUT index of every record whose low
// 32 bits are a multiple of `period` is appended to `list` (in no particular order) -- how the
// suffix-array builder learns where the whole reads of a read set landed without another sweep
// over the sorted records.  Hits are gathered per tile in shared memory: one global atomic per tile.
struct EmitNone {
    static constexpr bool kActive = false;
};
struct EmitMultiples {
    static constexpr bool kActive = true;
    // p % period == 0  <=>  rotr(p * inv, e) <= limit, with period = odd * 2^e, inv = odd^-1 mod 2^32,
    // limit = floor((2^32 - 1) / period) (Granlund-Montgomery): three instructions per record instead of the
    // 64-bit multiply-high of a reciprocal division (7.7 % of the last pass's instructions, ncu source page).
    u32 inv;
    u32 e;
    u32 limit;
    u32* list;
    u32* count;
    static EmitMultiples make(u32 period, u32* list, u32* count) {
        EmitMultiples m{};
        u32 odd = period;
        while (odd && !(odd & 1u)) { odd >>= 1; ++m.e; }
        u32 inv = odd;                                   // Newton: correct bits double each step
        for (int i = 0; i < 5; ++i) inv *= 2u - odd * inv;
        m.inv = inv;
        m.limit = 0xffffffffu / period;
        m.list = list;
        m.count = count;
        return m;
    }
    __device__ __forceinline__ bool hit(u64 k) const {
        const u32 x = static_cast<u32>(k) * inv;
        return __funnelshift_r(x, x, e) <= limit;
    }
};
// EmitStarts: the same for ragged read sets -- a record is reported when its position starts a read
// (position 0, or a separator right before it in the sentinel bitmap: bit 63 - (p % 64) of word p / 64).
struct EmitStarts {
    static constexpr bool kActive = true;
    const u64* sent;
    u32* list;
    u32* count;
    __device__ __forceinline__ bool hit(u64 k) const {
        const u32 p = static_cast<u32>(k);
        if (p == 0) return true;
        const u32 q = p - 1;
        return (sent[q >> 6] >> (63 - (q & 63))) & 1ull;
    }
};
constexpr int kEmitCap = 510;   // hits staged per tile; the overflow goes out one atomic each

// Digit of a key.  HI 1 (u64 keys, shift >= 32): the digit lies in the upper word, one 32-bit
// shift instead of a 64-bit funnel sequence -- the digit is extracted four times per item.
// HI 2: the digit is a whole BYTE of the upper word (8-bit digit at a byte boundary: every pass of the
// suffix-array builder's 32-bit keys); `shift` then holds the PRMT selector 0x4440 | byte and the digit
// costs one instruction, no mask.
template <int HI, typename KeyT>
__device__ __forceinline__ u32 pass_digit(KeyT k, int shift, u32 mask) {
    if constexpr (HI == 2) return __byte_perm(static_cast<u32>(static_cast<u64>(k) >> 32), 0u, static_cast<u32>(shift));
    else if constexpr (HI == 1) return (static_cast<u32>(static_cast<u64>(k) >> 32) >> shift) & mask;  // shift is already -32
    else return static_cast<u32>(k >> shift) & mask;
}

template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS>
struct OnesweepCfg {
    static constexpr int kWarps = BLOCK / 32;
    static constexpr int kTile = BLOCK * ITEMS;
    static constexpr size_t kSmem = sizeof(KeyT) * kTile + (HAS_VAL ? sizeof(u32) * kTile : 0) +
                                    sizeof(u32) * (kWarps * kRadix + 3 * kRadix + 32 + 4);   // + s_gofs, s_total, s_bin
};

template <typename KeyT, bool HAS_VAL, int BLOCK, int ITEMS, class EMIT = EmitNone, int HI = 0, int DPW = 1>
__global__ void __launch_bounds__(BLOCK, (BLOCK <= 256 ? (ITEMS <= 8 ? 6 : 4) : (BLOCK <= 384 ? (ITEMS <= 8 ? 4 : 3) : (BLOCK <= 512 ? (ITEMS <= 8 ? 3 : 2) : 1))))
onesweep_kernel(const void* __restrict__ keys_in_raw, KeyT* __restrict__ keys_out,
                const u32* __restrict__ vals_in, u32* __restrict__ vals_out, u64 n, int shift,
                u32 mask, const u32* __restrict__ digit_base, u64* __restrict__ lookback,
                u32* __restrict__ ticket, EMIT emit, int use_tma) {
    static_assert(BLOCK >= kRadix && BLOCK % 32 == 0, "one thread per digit is assumed");
    static_assert(!EMIT::kActive || sizeof(KeyT) == 8, "emit hooks look at 64-bit records");
    using Cfg = OnesweepCfg<KeyT, HAS_VAL, BLOCK, ITEMS>;
    constexpr int WARPS = Cfg::kWarps;
    constexpr int TILE = Cfg::kTile;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    KeyT* s_keys = reinterpret_cast<KeyT*>(smem_raw);
    u32* s_vals = reinterpret_cast<u32*>(s_keys + TILE);
    u32* s_whist = s_vals + (HAS_VAL ? TILE : 0);  // [WARPS][256] counts -> tile slot of the warp's run
    u32* s_gofs = s_whist + WARPS * kRadix;        // [256] global index of tile slot 0 of the digit
    u32* s_total = s_gofs + kRadix;                // [256] tile count of the digit
    u32* s_bin = s_total + kRadix;                 // [256] first tile slot of the digit
    u32* s_scan = s_bin + kRadix;                  // [32] warp totals for the digit scan
    u32* s_tile = s_scan + 32;
    u32* s_emit = s_tile + 4;                      // EMIT: [0] hits of this tile, [1] their base in the list, [2..] indices

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const unsigned lane = lane_id();

    __shared__ __align__(8) u64 s_bar;   // completion of the tile's bulk load
    if (use_tma && tid == 0) mbar_init(&s_bar, 1);
    __syncwarp();   // (racecheck attributes the barrier's initialisation to the warp, not to its lane 0)
    if (tid == 0) {
        const u32 t = atomicAdd(ticket, 1u);
        *s_tile = t;
        if (EMIT::kActive) s_emit[0] = 0;
        if (use_tma && static_cast<u64>(t) * TILE + TILE <= n) {
            // The tile is one contiguous stretch of HBM: the thread that drew the ticket has the TMA engine move
            // it into the exchange buffer (cp.async.bulk, completion counted in bytes on an mbarrier) instead of
            // ITEMS global loads per thread; the threads then pick their keys up from shared memory.  Barrier
            // set-up, arming and the copy all precede the block barrier below: the waiters only ever poll it.
            // (The buffer is rewritten by the exchange only after two more barriers.)
            mbar_expect_tx(&s_bar, static_cast<u32>(TILE * (sizeof(KeyT) + (HAS_VAL ? sizeof(u32) : 0))));
            tma_load_1d(s_keys, static_cast<const KeyT*>(keys_in_raw) + static_cast<u64>(t) * TILE, static_cast<u32>(TILE * sizeof(KeyT)), &s_bar);
            if (HAS_VAL) tma_load_1d(s_vals, vals_in + static_cast<u64>(t) * TILE, static_cast<u32>(TILE * sizeof(u32)), &s_bar);
        }
    }
    {
        uint4* z = reinterpret_cast<uint4*>(s_whist);
        for (int i = tid; i < WARPS * kRadix / 4; i += BLOCK) z[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    const u32 tile = *s_tile;
    const u64 tile_base = static_cast<u64>(tile) * TILE;
    const u32 valid = static_cast<u32>(n - tile_base < static_cast<u64>(TILE) ? n - tile_base : TILE);
    const bool full = valid == TILE;

    // -- load: warp-striped, so that (warp, step, lane) order == memory order ---------
    KeyT key[ITEMS];
    u32 val[ITEMS];
    const u32 wbase = warp * (ITEMS * 32) + lane;
    auto load_key = [&](u64 i) -> KeyT { return static_cast<const KeyT*>(keys_in_raw)[i]; };
    if (full && use_tma) {
        mbar_wait(&s_bar, 0);
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) key[j] = s_keys[wbase + j * 32];
        if (HAS_VAL) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) val[j] = s_vals[wbase + j * 32];
        }
    } else if (full) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) key[j] = load_key(tile_base + wbase + j * 32);
        if (HAS_VAL) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) val[j] = vals_in[tile_base + wbase + j * 32];
        }
    } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const u32 li = wbase + j * 32;
            key[j] = li < valid ? load_key(tile_base + li) : ~KeyT(0);  // pads rank last
            if (HAS_VAL) val[j] = li < valid ? vals_in[tile_base + li] : 0u;
        }
    }

    // -- rank inside the warp: equal digits are grouped by the ballots; the lowest lane of each
    //    group bumps the warp's private counter once for the whole group.  The bump is a shared
    //    atomicAdd whose old value is consumed only after a batch of them has been issued:
    //    successive steps of one warp are then independent instructions in flight instead of
    //    a load -> add -> store chain that exposes the shared-memory latency ITEMS times. ------
    u32* wh = s_whist + warp * kRadix;
    static_assert(ITEMS % 2 == 0, "ranks are kept two to a register");
    u32 rnk2[ITEMS / 2];  // two 16-bit ranks per register: the live key/payload registers leave little room
    const unsigned lt = lanemask_lt();
    constexpr int kBatch = ITEMS % 8 == 0 ? 8 : (ITEMS % 4 == 0 ? 4 : (ITEMS % 3 == 0 ? 3 : 1));
#pragma unroll
    for (int j0 = 0; j0 < ITEMS; j0 += kBatch) {
        unsigned peers[kBatch];
        u32 base[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) peers[b] = warp_match_digit(pass_digit<HI>(key[j0 + b], shift, mask));
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            base[b] = 0;
            if ((peers[b] & lt) == 0)  // lowest lane of its group
                base[b] = atomicAdd(wh + pass_digit<HI>(key[j0 + b], shift, mask), __popc(peers[b]));
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const u32 first = __shfl_sync(0xffffffffu, base[b], __ffs(peers[b]) - 1);
            const u32 r = first + __popc(peers[b] & lt);
            if (((j0 + b) & 1) == 0) rnk2[(j0 + b) >> 1] = r;
            else rnk2[(j0 + b) >> 1] |= r << 16;
        }
    }
    __syncthreads();

    // -- per digit: tile total, published at once as this tile's aggregate (DPW 2: the even lane of
    //    a digit pair stores the word for both) ---------------------------------------------------
    constexpr int WALKERS = kRadix / DPW;
    u32 total = 0;
    if (tid < kRadix) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) total += s_whist[w * kRadix + tid];
        s_total[tid] = total;
        if constexpr (DPW == 1) {
            if (tile > 0) st_relaxed_u64(lookback + static_cast<u64>(tile) * WALKERS + tid, kDescAggregate | total);
        } else {
            const u32 odd = __shfl_down_sync(0xffffffffu, total, 1);
            if (tile > 0 && !(tid & 1))
                st_relaxed_u64(lookback + static_cast<u64>(tile) * WALKERS + (tid >> 1),
                               (static_cast<u64>(kLaneAggregate | odd) << 32) | (kLaneAggregate | total));
        }
    }

    // -- exclusive scan of the 256 totals -> first tile slot of every digit; each warp's counter
    //    becomes the tile slot where its run of the digit starts ---------------------------------
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
#pragma unroll
        for (int w = 0; w < kRadix / 32; ++w) add += w < warp ? s_scan[w] : 0u;
        const u32 bin_start = add + inc - total;
        s_bin[tid] = bin_start;
        u32 run = bin_start;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            const u32 c = s_whist[w * kRadix + tid];
            s_whist[w * kRadix + tid] = run;
            run += c;
        }
    }
    __syncthreads();

    // -- exchange through shared memory: the tile becomes digit-sorted ----------------
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const u32 pos = wh[pass_digit<HI>(key[j], shift, mask)] + ((j & 1) ? rnk2[j >> 1] >> 16 : rnk2[j >> 1] & 0xffffu);
        s_keys[pos] = key[j];
        if (HAS_VAL) s_vals[pos] = val[j];
    }

    // -- decoupled look-back over earlier tiles, one thread per descriptor word.  It runs after the
    //    exchange so that the predecessors have had the time of this tile's exchange to publish.
    //    (Measured and dropped: the 128 threads that own no digit walking WHILE the 256 digit threads scan,
    //    kept apart by named barriers -- 0.796 against 0.690 ms per pass: walkers that start early only poll
    //    longer, and their share of the exchange then starts late.  profiles/r2_negative_results.md.)  The
    //    walk meets the front of finished tiles about (L2 latency / tile issue interval) tiles back;
    //    kLookahead descriptors are in flight at once. -------------------------------------------------
    if (tid < WALKERS) {
        u32 ex[DPW];
#pragma unroll
        for (int g = 0; g < DPW; ++g) ex[g] = 0;
        if (tile > 0) {
            long long t = static_cast<long long>(tile) - 1;
            for (bool done = false; !done;) {
                u64 v[kLookahead];
#pragma unroll
                for (int w = 0; w < kLookahead; ++w)
                    v[w] = t - w >= 0 ? ld_relaxed_u64(lookback + static_cast<u64>(t - w) * WALKERS + tid)
                                      : (DPW == 1 ? kDescInclusive : (static_cast<u64>(kLaneInclusive) << 32) | kLaneInclusive);
#pragma unroll
                for (int w = 0; w < kLookahead; ++w) {
                    if (done) break;
                    if constexpr (DPW == 1) {
                        if ((v[w] >> 62) == 0) break;   // not published yet: poll again from here
                        ex[0] += static_cast<u32>(v[w]);
                        done = (v[w] & kDescInclusive) != 0;
                    } else {
                        const u32 l0 = static_cast<u32>(v[w]), l1 = static_cast<u32>(v[w] >> 32);
                        if ((l0 >> 30) == 0) break;     // (both lanes are published by one store)
                        ex[0] += l0 & kLaneValueMask;
                        ex[1] += l1 & kLaneValueMask;
                        done = (l0 & kLaneInclusive) != 0;
                    }
                    --t;
                }
            }
        }
        if constexpr (DPW == 1) {
            st_relaxed_u64(lookback + static_cast<u64>(tile) * WALKERS + tid, kDescInclusive | (ex[0] + s_total[tid]));
            s_gofs[tid] = digit_base[tid] + ex[0] - s_bin[tid];
        } else {
            const uint2 t2 = *reinterpret_cast<const uint2*>(s_total + 2 * tid);
            st_relaxed_u64(lookback + static_cast<u64>(tile) * WALKERS + tid,
                           (static_cast<u64>(kLaneInclusive | (ex[1] + t2.y)) << 32) | (kLaneInclusive | (ex[0] + t2.x)));
            const uint2 b2 = *reinterpret_cast<const uint2*>(digit_base + 2 * tid);
            const uint2 s2 = *reinterpret_cast<const uint2*>(s_bin + 2 * tid);
            *reinterpret_cast<uint2*>(s_gofs + 2 * tid) = make_uint2(b2.x + ex[0] - s2.x, b2.y + ex[1] - s2.y);
        }
    }
    __syncthreads();

    // -- coalesced scatter: consecutive slots of one digit go to consecutive addresses -
    auto report = [&](KeyT k, u32 dst) {
        if constexpr (EMIT::kActive) {
            if (emit.hit(static_cast<u64>(k))) {
                const u32 slot = atomicAdd(&s_emit[0], 1u);
                if (slot < static_cast<u32>(kEmitCap)) s_emit[2 + slot] = dst;
                else emit.list[atomicAdd(emit.count, 1u)] = dst;   // a tile dense with hits
            }
        }
    };
    if (full) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const u32 i = tid + j * BLOCK;
            const KeyT k = s_keys[i];
            const u32 dst = s_gofs[pass_digit<HI>(k, shift, mask)] + i;
            keys_out[dst] = k;
            if (HAS_VAL) vals_out[dst] = s_vals[i];
            report(k, dst);
        }
    } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const u32 i = tid + j * BLOCK;
            if (i < valid) {
                const KeyT k = s_keys[i];
                const u32 dst = s_gofs[pass_digit<HI>(k, shift, mask)] + i;
                keys_out[dst] = k;
                if (HAS_VAL) vals_out[dst] = s_vals[i];
                report(k, dst);
            }
        }
    }
    if constexpr (EMIT::kActive) {
        __syncthreads();
        const u32 staged = s_emit[0] < static_cast<u32>(kEmitCap) ? s_emit[0] : static_cast<u32>(kEmitCap);
        if (tid == 0 && staged) s_emit[1] = atomicAdd(emit.count, staged);
        __syncthreads();
        for (u32 x = tid; x < staged; x += BLOCK) emit.list[s_emit[1] + x] = s_emit[2 + x];
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
// `emit_last` (u64 keys without payload only): hook run by the LAST pass, see EmitMultiples.
template <typename KeyT>
int onesweep_sort(reseq_cuda_ctx* ctx, KeyT* keys_a, KeyT* keys_b, u32* vals_a, u32* vals_b,
                  size_t n, const PassTable& pt, const SortWorkspace& ws, bool hist_ready,
                  u32 skip_mask, bool* in_b, const EmitMultiples* emit_last = nullptr,
                  const EmitStarts* emit_starts_last = nullptr);

}  // namespace rsq
