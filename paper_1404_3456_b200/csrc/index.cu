// Device-resident fragment index and the batched SA binary-search / overlap kernels.
//
// Replaces fragment_index (fragment_index.hpp:30-167):
//   ctor (:34-56)              -> reseq_cuda_index_create: SA by build_sa_device, start
//                                 ranks by one radix sort of (rank[start(id)], id), plus
//                                 a k-mer DIRECTORY over the SA that the reference does
//                                 not have (below)
//   locate_prefix_range (:65)  -> locate kernels: one thread per pattern, lower/upper
//   narrow (:114-148)             bound by binary search over SA with packed 32-base
//                                 compares; the search starts from the directory bucket
//                                 instead of [0, n)
//   start_rank_list lower_bound (:95-96) -> same two lower bounds, started from a second
//                                 directory over the fragment-start suffixes
//
// Directory.  For D bases, dir[x] = number of suffixes smaller than the D-base pattern x,
// x in [0, 4^D].  Every pattern P with |P| >= D and D-prefix x has its whole SA interval,
// and its lower-bound insertion point when absent, inside [dir[x], dir[x+1]]; so the
// directory replaces the top ~2D levels of both binary searches by two adjacent loads from
// an L2-sized table ("staging the top of the search tree on chip").  It is built without
// the SA: a suffix s is below pattern x iff code(s) <= x, where code(s) = (first D bases,
// zero padded at a terminator) + (1 if no terminator within D symbols); one histogram over
// positions and one exclusive scan.  sdir is the same table counted over fragment-start
// suffixes only, indexing start_rank_list.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "radix.cuh"
#include "sa.cuh"
#include "scan.cuh"

using namespace rsq;

struct reseq_cuda_index {
    reseq_cuda_ctx* ctx = nullptr;
    size_t n = 0, k = 0;
    bool dna = false;
    int dir_bases = 0;
    int sdir_bases = 0;     // the start-suffix directory is shallower: k entries spread thin, and it stays in L2
    u32 min_len = 0;
    u8* d_text = nullptr;
    u64* d_packed = nullptr;
    u64* d_sent = nullptr;
    u32* d_sa = nullptr;
    u32* d_rank = nullptr;
    u32* d_starts = nullptr;
    u32* d_lens = nullptr;
    u32* d_start_rank = nullptr;  // start_rank_list
    u32* d_start_frag = nullptr;  // fragment id of each start_rank_list entry
    u32* d_start_inv = nullptr;   // position of each fragment in start_rank_list
    u32* d_dir = nullptr;         // 4^D + 1 entries (+1 leading scan slot)
    u32* d_sdir = nullptr;
    u32 max_len = 0;
    u32* d_lengths = nullptr;     // distinct fragment lengths, ascending (lengths_, fragment_index.hpp:52-55)
    u32 n_lengths = 0;
    std::vector<u32> h_lens;      // fragment lengths, host copy (query-offset tables, argument checks)
    std::vector<u32> h_lengths;   // sorted distinct lengths, host copy
    std::vector<void*> owned;
};

namespace {

template <typename T>
int dev_alloc(reseq_cuda_index* ix, T** p, size_t count) {
    *p = nullptr;
    void* raw = nullptr;
    // stream-ordered allocation from the device's default pool (its release threshold is raised at
    // context creation): an index built after another one was destroyed reuses the cached blocks
    // instead of paying cudaMalloc / cudaFree of gigabytes (40-200 ms of wall time per index before)
    cudaError_t e = cudaMallocAsync(&raw, std::max<size_t>(count, 1) * sizeof(T), ix->ctx->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(RESEQ_OUT_OF_MEMORY, "cudaMalloc failed while building the index");
    }
    ix->owned.push_back(raw);
    *p = static_cast<T*>(raw);
    return RESEQ_OK;
}

unsigned grid_1d(const reseq_cuda_ctx* ctx, size_t items, int block, int waves = 16) {
    size_t want = (items + block - 1) / block;
    const size_t cap = static_cast<size_t>(ctx->sm_count) * waves;
    if (want < 1) want = 1;
    return static_cast<unsigned>(want < cap ? want : cap);
}

// ---- packed-text access (layout documented in sa.cu) ---------------------------------

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

struct TextView {
    const u8* text;
    const u64* packed;
    const u64* sent;
    u64 n;
};

// Sign of (suffix at `spos`) vs (pattern = text[ppos .. ppos+m)), both read from the packed
// text, 32 bases per step -- the cmp lambda of fragment_index.hpp:118-128.  A suffix that
// reaches a sentinel or the end of the text before the pattern is exhausted is smaller.
__device__ __forceinline__ int cmp_packed(const TextView& tv, u64 spos, u64 ppos, u32 m) {
    for (u32 c = 0; c < m; c += 32) {
        const u64 sp = spos + c;
        if (sp >= tv.n) return -1;
        const u32 chunk = m - c < 32u ? m - c : 32u;
        const u32 sw = static_cast<u32>(sent_window(tv.sent, sp) >> 32);
        u32 valid = sw ? static_cast<u32>(__clz(sw)) : 32u;
        const u64 rem = tv.n - sp;
        if (rem < valid) valid = static_cast<u32>(rem);
        const u32 len = valid < chunk ? valid : chunk;
        if (len) {
            const u64 a = base_window(tv.packed, sp);
            const u64 b = base_window(tv.packed, ppos + c);
            const u64 diff = (a ^ b) >> (64 - 2 * len);  // only the first `len` bases
            if (diff) {
                const int j = (__clzll(diff) - (64 - 2 * static_cast<int>(len))) >> 1;
                const u32 ca = static_cast<u32>(a >> (62 - 2 * j)) & 3u;
                const u32 cb = static_cast<u32>(b >> (62 - 2 * j)) & 3u;
                return ca < cb ? -1 : 1;
            }
        }
        if (valid < chunk) return -1;
    }
    return 0;
}

// Byte-wise form of the same comparison for generic alphabets and host-supplied patterns.
__device__ __forceinline__ int cmp_bytes(const TextView& tv, u64 spos, const u8* __restrict__ pat, u32 m) {
    for (u32 t = 0; t < m; ++t) {
        if (spos + t >= tv.n) return -1;
        const u32 sc = tv.text[spos + t], pc = pat[t];
        if (sc != pc) return sc < pc ? -1 : 1;
    }
    return 0;
}

// Lower and upper bound of the pattern inside [l0, r0) -- fragment_index.hpp:129-147.
template <typename Cmp>
__device__ __forceinline__ void bounds(const u32* __restrict__ sa, u32 l0, u32 r0, Cmp cmp, u32* lo, u32* hi) {
    u32 l = l0, r = r0;
    while (l < r) {
        const u32 mid = l + ((r - l) >> 1);
        if (cmp(sa[mid]) < 0) l = mid + 1;
        else r = mid;
    }
    *lo = l;
    r = r0;
    while (l < r) {
        const u32 mid = l + ((r - l) >> 1);
        if (cmp(sa[mid]) <= 0) l = mid + 1;
        else r = mid;
    }
    *hi = l;
}

__device__ __forceinline__ u32 lower_bound_u32(const u32* __restrict__ v, u32 l, u32 r, u32 x) {
    while (l < r) {
        const u32 mid = l + ((r - l) >> 1);
        if (v[mid] < x) l = mid + 1;
        else r = mid;
    }
    return l;
}

// ---- index construction kernels ----------------------------------------------------

__global__ void lens_kernel(const u32* __restrict__ starts, u64 k, u64 n, u32* __restrict__ lens,
                            const u32* __restrict__ rank, u32* __restrict__ keys, u32* __restrict__ ids,
                            u32* __restrict__ max_len, const u8* __restrict__ text) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    u32 local_max = 0;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
        const u64 end = (i + 1 < k ? starts[i + 1] : n) - 1;  // sequence.hpp:78-83
        const u32 len = static_cast<u32>(end - starts[i]);
        if (text[end] != 0) atomicOr(max_len + 1, 1u);        // every fragment ends at a separator (sequence.hpp:60-62)
        lens[i] = len;
        keys[i] = rank[starts[i]];
        ids[i] = static_cast<u32>(i);
        local_max = max(local_max, len);
    }
    for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
    if (lane_id() == 0 && local_max) atomicMax(max_len, local_max);
}

__global__ void invert_kernel(const u32* __restrict__ start_frag, u64 k, u32* __restrict__ start_inv) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 t = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; t < k; t += stride)
        start_inv[start_frag[t]] = static_cast<u32>(t);
}

// code(s) of the header comment; D <= 16.
__device__ __forceinline__ u32 dir_code(const u64* __restrict__ packed, const u64* __restrict__ sent,
                                        u64 n, u64 pos, int D) {
    const u32 bases = static_cast<u32>(base_window(packed, pos) >> (64 - 2 * D));
    const u32 sw = static_cast<u32>(sent_window(sent, pos) >> (64 - D));
    const u32 t = sw ? static_cast<u32>(__clz(sw)) - (32 - D) : D;
    const u64 rem = n - pos;
    u32 len = t;
    if (rem < len) len = static_cast<u32>(rem);
    if (len >= static_cast<u32>(D)) return bases + 1u;
    return bases & ~((1u << (2 * (D - len))) - 1u);
}

// Histogram of code(s) over all positions (positions == nullptr) or over a position list.
__global__ void dir_hist_kernel(const u64* __restrict__ packed, const u64* __restrict__ sent, u64 n,
                                const u32* __restrict__ positions, u64 count, int D,
                                u32* __restrict__ hist) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const u64 pos = positions ? positions[i] : i;
        atomicAdd(hist + dir_code(packed, sent, n, pos, D), 1u);
    }
}

// ---- query kernels --------------------------------------------------------------------

struct IndexView {
    TextView tv;
    const u32* sa;
    const u32* rank;
    const u32* starts;
    const u32* lens;
    const u32* start_rank;
    const u32* start_frag;
    const u32* start_inv;
    const u32* dir;   // dir[x] = lower bound of D-base pattern x; nullptr when absent
    const u32* sdir;
    int D;
    int sD;        // bases indexing sdir (<= D)
    u32 min_len;   // shortest fragment
    u32 k;
};

// SA interval of the pattern text[ppos .. ppos+m) (a residual).
// narrow()'s continuation (fragment_index.hpp:114-148, used by the sweep of :87-93): on entry (*lo, *hi) is
// an interval whose suffixes are known to share the pattern's first `depth` symbols and (*s_first, *s_last)
// the start-list range inside it -- (0, n, 0, k) and depth 0 for a fresh search.  The search stays inside
// them and compares symbols depth.. only.
__device__ __forceinline__ void locate_residual(const IndexView& iv, u64 ppos, u32 m, u32* lo, u32* hi,
                                                u32* s_first, u32* s_last, u32 depth = 0) {
    u32 l0 = *lo, r0 = *hi, f0 = *s_first, f1 = *s_last;
    if (iv.tv.packed) {
        if (iv.dir && m >= static_cast<u32>(iv.D)) {
            const u32 x = static_cast<u32>(base_window(iv.tv.packed, ppos) >> (64 - 2 * iv.D));
            l0 = max(l0, iv.dir[x]);
            r0 = max(l0, min(r0, iv.dir[x + 1]));
            const u32 xs = x >> (2 * (iv.D - iv.sD));
            f0 = max(f0, iv.sdir[xs]);
            f1 = max(f0, min(f1, iv.sdir[xs + 1]));
        }
        bounds(iv.sa, l0, r0, [&](u32 spos) { return cmp_packed(iv.tv, static_cast<u64>(spos) + depth, ppos + depth, m - depth); }, lo, hi);
    } else {
        const u8* pat = iv.tv.text + ppos + depth;
        bounds(iv.sa, l0, r0, [&](u32 spos) { return cmp_bytes(iv.tv, static_cast<u64>(spos) + depth, pat, m - depth); }, lo, hi);
    }
    // fragment_index.hpp:95-96
    *s_first = lower_bound_u32(iv.start_rank, f0, f1, *lo);
    *s_last = lower_bound_u32(iv.start_rank, *s_first, f1, *hi);
}
// A fresh search over the whole array.
__device__ __forceinline__ void locate_residual_fresh(const IndexView& iv, u64 ppos, u32 m, u32* lo, u32* hi,
                                                      u32* s_first, u32* s_last) {
    *lo = 0;
    *hi = static_cast<u32>(iv.tv.n);
    *s_first = 0;
    *s_last = iv.k;
    locate_residual(iv, ppos, m, lo, hi, s_first, s_last, 0);
}

// The fragment-start suffixes inside the SA interval of the residual text[ppos .. ppos+m), without
// searching for the interval: the residual is itself a suffix of the text, so its own rank r lies
// inside [lo, hi).  Everything between lo and r is an identical copy "X$" at a lower position
// (normally none: one probe), and the start suffixes of the interval are the entries of start_rank
// from lower_bound(lo) on for as long as the fragment they name begins with X -- so the upper
// bound is never computed; the work is one comparison per overlap found plus one.
// Same (s_first, s_last) as locate_residual; ~3 DRAM gathers per query instead of ~12.
// Part 1: the query's own rank and the bracket of start suffixes that share its first sD bases.
// An empty bracket (4 queries in 5 on a read set) means no overlap: nothing else is loaded.
__device__ __forceinline__ void residual_bracket(const IndexView& iv, u64 ppos, u32 m, u32* r, u32* f0, u32* f1) {
    // the bracket does not depend on the rank: both chains of loads (rank from HBM; text word ->
    // L2-resident directory) are issued before either result is needed
    *f0 = 0;
    *f1 = iv.k;
    *r = iv.rank[ppos];
    if (iv.sdir && m >= static_cast<u32>(iv.sD)) {
        const u32 x = static_cast<u32>(base_window(iv.tv.packed, ppos) >> (64 - 2 * iv.sD));
        *f0 = iv.sdir[x];
        *f1 = iv.sdir[x + 1];
    }
}

// Part 2: [s_first, s_last) inside the bracket.
__device__ __forceinline__ void residual_starts_in_bracket(const IndexView& iv, u64 ppos, u32 m, u32 r, u32 f0, u32 f1,
                                                           u32* s_first, u32* s_last) {
    // idx <= r: the suffix there is never greater than the pattern; it is smaller -- no match -- exactly
    // when it differs from it or ends first.  It usually ends first (the neighbour below a read suffix
    // is the same locus seen from a read that ends earlier), which the sentinel bitmap alone tells:
    // one to three loads instead of a chunk-by-chunk comparison of ~t symbols.
    auto is_match = [&](u32 idx) {
        const u64 spos = iv.sa[idx];
        for (u32 c = 0; c < m; c += 64) {
            if (spos + c >= iv.tv.n) return false;
            u64 w = sent_window(iv.tv.sent, spos + c);
            if (m - c < 64) w &= ~0ull << (64 - (m - c));
            if (w) return false;                 // a sentinel inside the first m symbols
        }
        return cmp_packed(iv.tv, spos, ppos, m) >= 0;
    };
    u32 ok = r, bad = 0xFFFFFFFFu;          // ok: lowest index known to match; bad: highest known not to (none yet)
    // The copies below r matter only if one of them is a whole fragment (equal to the pattern): none
    // is when the pattern is shorter than every fragment -- every o > 0 query of a uniform read set.
    for (u32 step = 1; ok > 0 && m >= iv.min_len; step <<= 1) {
        const u32 probe = ok > step ? ok - step : 0u;
        if (is_match(probe)) ok = probe;
        else { bad = probe; break; }
        if (probe == 0) break;
    }
    if (bad != 0xFFFFFFFFu) {
        while (ok - bad > 1) {
            const u32 mid = bad + ((ok - bad) >> 1);
            if (is_match(mid)) ok = mid;
            else bad = mid;
        }
    }
    const u32 lo = ok;
    const u32 sf = lower_bound_u32(iv.start_rank, f0, f1, lo);
    // does fragment j begin with the pattern?  Both are runs of >= m bases when lens[j] >= m, so this
    // is a plain comparison of packed words (no sentinel bookkeeping): the warp's lanes diverge here,
    // and every instruction in this loop is paid by all of them.
    auto begins_with_pattern = [&](u32 j) {
        if (iv.lens[j] < m) return false;
        const u64 a = iv.starts[j];
        for (u32 c = 0; c < m; c += 32) {
            const u32 nb = m - c < 32u ? m - c : 32u;
            if ((base_window(iv.tv.packed, a + c) ^ base_window(iv.tv.packed, ppos + c)) >> (64 - 2 * nb)) return false;
        }
        return true;
    };
    u32 sl = sf;
    while (sl < f1 && begins_with_pattern(iv.start_frag[sl])) ++sl;
    *s_first = sf;
    *s_last = sl;
}

__global__ void __launch_bounds__(256)
locate_residuals_kernel(IndexView iv, const u32* __restrict__ frag, const u32* __restrict__ off, u64 q,
                        u32* __restrict__ lo, u32* __restrict__ hi) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < q; i += stride) {
        const u32 f = frag[i], o = off[i];
        u32 l, h, sf, sl;
        locate_residual_fresh(iv, static_cast<u64>(iv.starts[f]) + o, iv.lens[f] - o, &l, &h, &sf, &sl);
        lo[i] = l;
        hi[i] = h;
    }
}

// Host-supplied byte patterns.  A DNA index still narrows through the directory when the
// first D pattern bytes are bases; the comparisons are byte-wise so that patterns holding
// bytes outside the alphabet land on the reference's insertion point.
__global__ void __launch_bounds__(256)
locate_patterns_kernel(IndexView iv, const u8* __restrict__ pats, const u64* __restrict__ pat_off, u64 q,
                       u32* __restrict__ lo, u32* __restrict__ hi) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < q; i += stride) {
        const u8* pat = pats + pat_off[i];
        const u32 m = static_cast<u32>(pat_off[i + 1] - pat_off[i]);
        u32 l0 = 0, r0 = static_cast<u32>(iv.tv.n);
        if (iv.dir && m >= static_cast<u32>(iv.D)) {
            u32 x = 0;
            bool ok = true;
            for (int t = 0; t < iv.D; ++t) {
                const u32 c = pat[t];
                ok &= (c == 'A' || c == 'C' || c == 'G' || c == 'T');
                x = (x << 2) | (((c >> 1) ^ (c >> 2)) & 3u);
            }
            if (ok) {
                l0 = iv.dir[x];
                r0 = iv.dir[x + 1];
            }
        }
        u32 l, h;
        bounds(iv.sa, l0, r0, [&](u32 spos) { return cmp_bytes(iv.tv, spos, pat, m); }, &l, &h);
        lo[i] = l;
        hi[i] = h;
    }
}

// Overlap pass 1: one warp per fragment, lanes stride over the offsets.  Query (i, o) =
// pattern f_i[o..]; every fragment-start suffix inside its SA interval is a fragment j
// whose prefix equals that pattern, i.e. overlap_weight(f_i, f_j) >= |f_i| - o
// (overlap.hpp:16-23).  Stores, per query, the start-list interval; per fragment, the
// absorb_contained verdict (overlap.hpp:51-67) from the o = 0 query.
// CONTAINED: also derive the containment verdict from the o = 0 query (needs the whole interval: a
// full search by one lane while 31 wait) -- used only where the rank-anchored search does not apply;
// otherwise contained_kernel does that with one thread per fragment.
constexpr int kStageRank = 272;   // rank entries staged per fragment: <= 255 + alignment slack, a multiple of 4
constexpr int kStageText = 12;    // packed words staged per fragment

template <bool CONTAINED, bool STAGE = false>
__global__ void __launch_bounds__(256, (STAGE || CONTAINED) ? 4 : 6)
overlap_count_kernel(IndexView iv, u32 min_ov, u64 f0, u64 f1, const u64* __restrict__ qoff,
                     u32* __restrict__ q_first, u32* __restrict__ q_count, u8* __restrict__ contained,
                     u32* __restrict__ rawcount) {
    // rawcount[i - f0] = records fragment i will produce: the record offsets are then one scan over
    // the fragments (plus a warp scan inside each) instead of one over all the queries
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    auto publish = [&](u64 i, u32 mine) {
        for (int d = 16; d > 0; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
        if (lane == 0) rawcount[i - f0] = mine;
    };
    if constexpr (!CONTAINED) {
        // Rank-anchored form.  Four queries in five end at an empty bracket after two loads; the fifth
        // walks start_rank and compares fragments -- a chain of ~10 dependent L2 round trips that, run
        // in place, every lane of the warp would wait for in every iteration.  Queries with a
        // non-empty bracket are therefore queued per warp and worked off 32 at a time, all lanes busy.
        __shared__ u32 s_qr[8][64], s_qf0[8][64], s_qf1o[8][64];   // rank, bracket start, (bracket size << 8 | offset)
        u32* qr = s_qr[threadIdx.x >> 5];
        u32* qf0 = s_qf0[threadIdx.x >> 5];
        u32* qf1o = s_qf1o[threadIdx.x >> 5];
        // Staging (the north star's "SA blocks in shared memory or via TMA"): everything a fragment's
        // queries read at consecutive addresses -- its block of the inverse suffix array, rank[start ..
        // start + len), and its packed text -- is brought into shared memory by TWO bulk copies (TMA,
        // cp.async.bulk) issued by the warp's first lane, double buffered: the copies for the warp's NEXT
        // fragment are in flight while the current one is searched, so the queries start from shared
        // memory instead of behind a chain of global loads (starts/lens -> rank, text).
        // (measured: 3.20 ms against 2.88 for the unstaged form at config 2 -- the per-lane loads of ~50
        //  resident warps hide the chain better than one elected lane's copies; kept as an option,
        //  "overlap_stage", off by default.  profiles/r2_negative_results.md.)
        __shared__ __align__(16) u32 s_rk[STAGE ? 8 : 1][2][STAGE ? kStageRank : 4];
        __shared__ __align__(16) u64 s_tx[STAGE ? 8 : 1][2][STAGE ? kStageText : 2];
        __shared__ __align__(8) u64 s_sbar[STAGE ? 8 : 1][2];
        const int wib = STAGE ? threadIdx.x >> 5 : 0;
        if (STAGE && lane == 0) {
            mbar_init(&s_sbar[wib][0], 1);
            mbar_init(&s_sbar[wib][1], 1);
        }
        __syncwarp();
        auto stageable = [&](u64 st, u32 ln) {   // both copies 16-byte aligned and inside their arrays
            return ln <= 255u && ((st & ~3ull) + (((st & 3ull) + ln + 3u) & ~3ull)) <= iv.tv.n;
        };
        auto issue = [&](u64 st, u32 ln, int b) {   // lane 0
            const u64 r0 = st & ~3ull;
            const u32 cnt = static_cast<u32>(((st - r0) + ln + 3u) & ~3ull);
            const u64 w0 = (st >> 5) & ~1ull;
            const u32 nw = static_cast<u32>((((st + ln + 31) >> 5) - w0 + 3u) & ~1ull);
            mbar_expect_tx(&s_sbar[wib][b], cnt * 4u + nw * 8u);
            tma_load_1d(s_rk[wib][b], iv.rank + r0, cnt * 4u, &s_sbar[wib][b]);
            tma_load_1d(s_tx[wib][b], iv.tv.packed + w0, nw * 8u, &s_sbar[wib][b]);
        };
        const u64 i_first = f0 + ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
        // fragment descriptors one iteration ahead (registers), copies one iteration ahead (shared memory)
        u64 start_n = 0;
        u32 len_n = 0;
        bool staged_n = false;
        if (i_first < f1) {
            start_n = iv.starts[i_first];
            len_n = iv.lens[i_first];
            staged_n = STAGE && stageable(start_n, len_n);
            if (staged_n && lane == 0) issue(start_n, len_n, 0);
        }
        u32 uses[2] = {0u, 0u};   // completed phases of each buffer's barrier
        int buf = 0;
        for (u64 i = i_first; i < f1; i += warps, buf ^= 1) {
            const u32 len = len_n;
            const u64 start = start_n;
            const bool staged = staged_n;
            if (i + warps < f1) {   // next fragment: descriptor now, copies into the other buffer
                start_n = iv.starts[i + warps];
                len_n = iv.lens[i + warps];
                staged_n = STAGE && stageable(start_n, len_n);
                __syncwarp();       // (every lane is done with the other buffer: it was the fragment before this one)
                if (staged_n && lane == 0) issue(start_n, len_n, buf ^ 1);
            }
            const u64 qbase = qoff[i - f0];
            const u32 nq = static_cast<u32>(qoff[i - f0 + 1] - qbase);
            const u32 self = iv.start_inv[i];
            const u32* rk = nullptr;
            const u64* tx = nullptr;
            u32 tx_bit0 = 0;
            if (staged) {
                __syncwarp();   // lane 0 armed this barrier (an iteration ago, or before the loop): the other lanes only poll it
                mbar_wait(&s_sbar[wib][buf], uses[buf] & 1u);
                ++uses[buf];
                rk = s_rk[wib][buf] + (start & 3ull);
                tx = s_tx[wib][buf];
                tx_bit0 = 2u * static_cast<u32>(start - (((start >> 5) & ~1ull) << 5));
            }
            u32 queued = 0, mine = 0;
            auto work_off = [&](u32 count) {   // the first `count` (<= 32) queue entries
                if (lane < count) {
                    const u32 o = qf1o[lane] & 0xffu, b0 = qf0[lane], b1 = b0 + (qf1o[lane] >> 8);
                    u32 sf, sl;
                    residual_starts_in_bracket(iv, start + o, len - o, qr[lane], b0, b1, &sf, &sl);
                    const u32 self_in = (self >= sf && self < sl) ? 1u : 0u;
                    q_first[qbase + o] = sf | (self_in << 31);
                    q_count[qbase + o] = sl - sf - self_in;
                    mine += sl - sf - self_in;
                }
                __syncwarp();
                const bool moves = lane + count < queued;   // the rest (< 32 entries) moves to the front
                u32 a = 0, b = 0, c = 0;
                if (moves) { a = qr[lane + count]; b = qf0[lane + count]; c = qf1o[lane + count]; }
                __syncwarp();
                if (moves) { qr[lane] = a; qf0[lane] = b; qf1o[lane] = c; }
                __syncwarp();
                queued -= count;
            };
            for (u32 o0 = 0; o0 < nq; o0 += 32) {
                const u32 o = o0 + lane;
                bool has = false;
                u32 r = 0, b0 = 0, b1 = 0;
                if (o < nq) {
                    if (staged) {   // the query's own rank and its first sD bases, from shared memory
                        r = rk[o];
                        b0 = 0;
                        b1 = iv.k;
                        if (iv.sdir && len - o >= static_cast<u32>(iv.sD)) {
                            const u32 bit = tx_bit0 + 2u * o, wi = bit >> 6, sh = bit & 63u;
                            const u64 hi = tx[wi], lo = tx[wi + 1];
                            const u64 win = sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
                            const u32 x = static_cast<u32>(win >> (64 - 2 * iv.sD));
                            b0 = iv.sdir[x];
                            b1 = iv.sdir[x + 1];
                        }
                    } else {
                        residual_bracket(iv, start + o, len - o, &r, &b0, &b1);
                    }
                    has = b0 < b1;
                    if (!has) {   // the diagonal cannot be inside an empty bracket either
                        q_first[qbase + o] = b0;
                        q_count[qbase + o] = 0;
                    }
                }
                // offsets above 255 or brackets above 2^24 entries do not fit the packed queue word: in place
                if (has && (o > 255u || b1 - b0 >= (1u << 24))) {
                    u32 sf, sl;
                    residual_starts_in_bracket(iv, start + o, len - o, r, b0, b1, &sf, &sl);
                    const u32 self_in = (self >= sf && self < sl) ? 1u : 0u;
                    q_first[qbase + o] = sf | (self_in << 31);
                    q_count[qbase + o] = sl - sf - self_in;
                    mine += sl - sf - self_in;
                    has = false;
                }
                const unsigned mask = __ballot_sync(0xffffffffu, has);
                if (has) {
                    const u32 slot = queued + __popc(mask & lanemask_lt());
                    qr[slot] = r;
                    qf0[slot] = b0;
                    qf1o[slot] = ((b1 - b0) << 8) | o;
                }
                queued += __popc(mask);
                __syncwarp();
                if (queued >= 32) work_off(32);
            }
            if (queued) work_off(queued);
            publish(i, mine);
        }
    } else {
    for (u64 i = f0 + ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); i < f1; i += warps) {
        const u32 len = iv.lens[i];
        const u64 start = iv.starts[i];
        const u64 qbase = qoff[i - f0];
        const u32 nq = static_cast<u32>(qoff[i - f0 + 1] - qbase);  // offsets 0 .. len - min_ov
        // a fragment shorter than min_ov still runs its o = 0 query for the containment flag
        const u32 steps = nq ? nq : 1u;
        const u32 self = iv.start_inv[i];
        u32 mine = 0;
        for (u32 o = lane; o < steps; o += 32) {
            const u32 m = len - o;
            u32 lo = 0, hi = 0, sf, sl;
            locate_residual_fresh(iv, start + o, m, &lo, &hi, &sf, &sl);
            // f_i's own start suffix lies in the interval at o = 0, and at o > 0 whenever f_i
            // overlaps itself; the diagonal is zero by convention (overlap.hpp:26,41)
            const u32 self_in = (self >= sf && self < sl) ? 1u : 0u;
            const u32 cnt = sl - sf - self_in;
            if (o == 0) {
                u32 exact = 0, min_id = 0xFFFFFFFFu;
                for (u32 t = sf; t < sl; ++t) {
                    const u32 id = iv.start_frag[t];
                    if (iv.lens[id] == m) {
                        ++exact;
                        min_id = min(min_id, id);
                    }
                }
                contained[i] = (hi - lo > exact) || (min_id < static_cast<u32>(i));
            }
            if (o < nq) {
                q_first[qbase + o] = sf | (self_in << 31);  // k < 2^31: a fragment takes >= 2 bytes
                q_count[qbase + o] = cnt;
                mine += cnt;
            }
        }
        publish(i, mine);
    }
    }
}

// absorb_contained (overlap.hpp:51-67) for fragments [f0, f1): fragment i is dropped iff it occurs
// inside a longer fragment or equals one with a lower id -- i.e. iff the SA interval of the whole
// fragment holds more suffixes than the fragments equal to it, or one of those has a lower id.
// One thread per fragment (the interval needs both binary searches).
__global__ void __launch_bounds__(256)
contained_kernel(IndexView iv, u64 f0, u64 f1, u8* __restrict__ contained) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = f0 + static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < f1; i += stride) {
        const u32 m = iv.lens[i];
        u32 lo, hi, sf, sl;
        locate_residual_fresh(iv, iv.starts[i], m, &lo, &hi, &sf, &sl);
        u32 exact = 0, min_id = 0xFFFFFFFFu;
        for (u32 t = sf; t < sl; ++t) {
            const u32 id = iv.start_frag[t];
            if (iv.lens[id] == m) {
                ++exact;
                min_id = min(min_id, id);
            }
        }
        contained[i] = (hi - lo > exact) || (min_id < static_cast<u32>(i));
    }
}

// Overlap pass 2: writes the raw (i<<32 | j, w) records at the scanned offsets, in
// (i, o ascending) order so that after a STABLE sort on (i, j) the first record of every
// pair carries its maximum w.
__global__ void __launch_bounds__(256)
overlap_fill_kernel(IndexView iv, u64 f0, u64 f1, const u64* __restrict__ qoff, const u32* __restrict__ q_first,
                    const u32* __restrict__ q_count, const u32* __restrict__ q_out, u64* __restrict__ keys,
                    u32* __restrict__ w) {
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (u64 i = f0 + ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); i < f1; i += warps) {
        const u32 len = iv.lens[i];
        const u64 qbase = qoff[i - f0];
        const u32 nq = static_cast<u32>(qoff[i - f0 + 1] - qbase);
        for (u32 o = lane; o < nq; o += 32) {
            const u32 cnt = q_count[qbase + o];
            if (!cnt) continue;
            u32 out = q_out[qbase + o];
            const u32 sf = q_first[qbase + o] & 0x7FFFFFFFu;
            const u32 span = cnt + (q_first[qbase + o] >> 31);
            for (u32 t = 0; t < span; ++t) {
                const u32 j = iv.start_frag[sf + t];
                if (j == static_cast<u32>(i)) continue;
                keys[out] = (static_cast<u64>(i) << 32) | j;
                w[out] = len - o;
                ++out;
            }
        }
    }
}

// prefix_related (fragment_index.hpp:82-109) for residual patterns, one thread per query.
// The sweep over the distinct fragment lengths below |pattern| collects the fragments that
// are proper prefixes of the pattern (start suffixes of exactly that length inside the
// interval of the pattern's prefix); the final interval yields extensions and exact
// matches.  MODE 0 counts, MODE 1 fills the CSR arrays at the scanned offsets.  For a
// residual every prefix of the pattern occurs in the text, so the early return of
// fragment_index.hpp:91 cannot trigger.  Each length resumes from the previous interval and
// depth (narrow's continuation, :87-93).  Lists leave in start-rank order; the host sorts
// each by id (fragment_index.hpp:105-107).
template <int MODE>
__global__ void __launch_bounds__(256)
prefix_related_kernel(IndexView iv, const u32* __restrict__ lengths, u32 n_lengths,
                      const u32* __restrict__ frag, const u32* __restrict__ off, u64 q,
                      u32* __restrict__ cnt_pre, u32* __restrict__ cnt_ext, u32* __restrict__ cnt_exact,
                      const u32* __restrict__ off_pre, const u32* __restrict__ off_ext,
                      const u32* __restrict__ off_exact, u32* __restrict__ out_pre,
                      u32* __restrict__ out_ext, u32* __restrict__ out_exact) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < q; i += stride) {
        const u32 f = frag[i], o = off[i];
        const u64 ppos = static_cast<u64>(iv.starts[f]) + o;
        const u32 m = iv.lens[f] - o;
        u32 np = 0, ne = 0, nx = 0;
        u32 wp = MODE ? off_pre[i] : 0, we = MODE ? off_ext[i] : 0, wx = MODE ? off_exact[i] : 0;
        // one narrowing sweep (fragment_index.hpp:84-93): every length resumes from the previous interval
        // and depth, as narrow() does
        u32 lo = 0, hi = static_cast<u32>(iv.tv.n), sf = 0, sl = iv.k, depth = 0;
        for (u32 t = 0; t < n_lengths; ++t) {
            const u32 len = lengths[t];
            if (len >= m) break;
            locate_residual(iv, ppos, len, &lo, &hi, &sf, &sl, depth);
            depth = len;
            for (u32 u = sf; u < sl; ++u) {
                const u32 id = iv.start_frag[u];
                if (iv.lens[id] == len) {
                    if (MODE) out_pre[wp++] = id;
                    ++np;
                }
            }
        }
        locate_residual(iv, ppos, m, &lo, &hi, &sf, &sl, depth);
        for (u32 u = sf; u < sl; ++u) {
            const u32 id = iv.start_frag[u];
            const u32 len = iv.lens[id];
            if (len > m) {
                if (MODE) out_ext[we++] = id;
                ++ne;
            } else if (len == m) {
                if (MODE) out_exact[wx++] = id;
                ++nx;
            }
        }
        if (!MODE) {
            cnt_pre[i] = np;
            cnt_ext[i] = ne;
            cnt_exact[i] = nx;
        }
    }
}

// Overlap pass 2, fast form: the records of one fragment (~26 at 30x coverage) are produced, sorted by
// j and deduplicated by ONE warp in shared memory and leave already in their final (i, j) order --
// fragments are processed in id order, so no global sort (six 12-byte radix passes over all the
// records), no flag/scan/compact for uniqueness.  A fragment with more than kOvCap raw records
// raises `overflow`; the caller then takes the general route below for the whole call.
constexpr int kOvCap = 256;

__device__ __forceinline__ void warp_bitonic_sort(u64* a, int n, unsigned lane) {   // n: power of two
    for (int k2 = 2; k2 <= n; k2 <<= 1) {
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            for (int t = lane; t < (n >> 1); t += 32) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));   // bit j clear
                const int l = i | j;
                const bool up = (i & k2) == 0;
                const u64 x = a[i], y = a[l];
                if ((x > y) == up) {
                    a[i] = y;
                    a[l] = x;
                }
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(256)
overlap_fill_sorted_kernel(IndexView iv, u64 f0, u64 f1, const u64* __restrict__ qoff,
                           const u32* __restrict__ q_first, const u32* __restrict__ q_count,
                           const u32* __restrict__ rbase, u32* __restrict__ ti, u32* __restrict__ tj,
                           u32* __restrict__ tw, u32* __restrict__ ucount, u32* __restrict__ overflow) {
    __shared__ u64 s_all[8 * kOvCap];
    u64* a = s_all + (threadIdx.x >> 5) * kOvCap;
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (u64 i = f0 + ((static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); i < f1; i += warps) {
        const u32 len = iv.lens[i];
        const u64 qbase = qoff[i - f0];
        const u32 nq = static_cast<u32>(qoff[i - f0 + 1] - qbase);
        const u32 base = rbase[i - f0];
        const u32 raw = rbase[i - f0 + 1] - base;   // rbase has an entry behind the last fragment
        if (raw > static_cast<u32>(kOvCap)) {
            if (lane == 0) {
                atomicOr(overflow, 1u);
                ucount[i - f0] = 0;
            }
            continue;
        }
        if (raw == 0) {
            if (lane == 0) ucount[i - f0] = 0;
            continue;
        }
        int n2 = 2;
        while (n2 < static_cast<int>(raw)) n2 <<= 1;
        for (int t = raw + lane; t < n2; t += 32) a[t] = ~0ull;
        u32 before = 0;   // records of the offsets below this sweep
        for (u32 o0 = 0; o0 < nq; o0 += 32) {
            const u32 o = o0 + lane;
            const u32 cnt = o < nq ? q_count[qbase + o] : 0u;
            u32 inc = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, inc, d);
                if (static_cast<int>(lane) >= d) inc += t;
            }
            if (cnt) {
                u32 out = before + inc - cnt;
                const u32 sf = q_first[qbase + o] & 0x7FFFFFFFu;
                const u32 span = cnt + (q_first[qbase + o] >> 31);
                for (u32 t = 0; t < span; ++t) {
                    const u32 j = iv.start_frag[sf + t];
                    if (j == static_cast<u32>(i)) continue;
                    a[out++] = (static_cast<u64>(j) << 32) | (~(len - o));   // ties on j: the larger weight first
                }
            }
            before += __shfl_sync(0xffffffffu, inc, 31);
        }
        __syncwarp();
        warp_bitonic_sort(a, n2, lane);
        u32 run = 0;
        for (u32 t0 = 0; t0 < raw; t0 += 32) {
            const u32 t = t0 + lane;
            const bool valid = t < raw;
            const u64 key = valid ? a[t] : 0;
            const bool head = valid && (t == 0 || static_cast<u32>(key >> 32) != static_cast<u32>(a[t - 1] >> 32));
            const unsigned mask = __ballot_sync(0xffffffffu, head);
            if (head) {
                const u32 d = base + run + __popc(mask & lanemask_lt());
                ti[d] = static_cast<u32>(i);
                tj[d] = static_cast<u32>(key >> 32);
                tw[d] = ~static_cast<u32>(key);
            }
            run += __popc(mask);
        }
        if (lane == 0) ucount[i - f0] = run;
        __syncwarp();
    }
}

// Closes the gaps dropped duplicates left: fragment f's `ucount[f]` records move from their raw
// offset to the scanned unique offset.
__global__ void __launch_bounds__(256)
overlap_close_gaps_kernel(u64 kr, const u32* __restrict__ rbase,
                          const u32* __restrict__ ucount, const u32* __restrict__ uoff,
                          const u32* __restrict__ ti, const u32* __restrict__ tj, const u32* __restrict__ tw,
                          u32* __restrict__ oi, u32* __restrict__ oj, u32* __restrict__ ow) {
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (u64 f = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; f < kr; f += warps) {
        const u32 src = rbase[f], dst = uoff[f], c = ucount[f];
        for (u32 t = lane; t < c; t += 32) {
            oi[dst + t] = ti[src + t];
            oj[dst + t] = tj[src + t];
            ow[dst + t] = tw[src + t];
        }
    }
}

__global__ void unique_flag_kernel(const u64* __restrict__ keys, u64 m, u32* __restrict__ flag) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 t = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; t < m; t += stride)
        flag[t] = (t == 0 || keys[t] != keys[t - 1]) ? 1u : 0u;
}

__global__ void unique_compact_kernel(const u64* __restrict__ keys, const u32* __restrict__ w,
                                      const u32* __restrict__ flag, const u32* __restrict__ dst, u64 m,
                                      u32* __restrict__ oi, u32* __restrict__ oj, u32* __restrict__ ow) {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 t = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; t < m; t += stride)
        if (flag[t]) {
            const u32 d = dst[t];
            oi[d] = static_cast<u32>(keys[t] >> 32);
            oj[d] = static_cast<u32>(keys[t]);
            ow[d] = w[t];
        }
}

IndexView view_of(const reseq_cuda_index* ix) {
    IndexView iv{};
    iv.tv = TextView{ix->d_text, ix->dna ? ix->d_packed : nullptr, ix->dna ? ix->d_sent : nullptr, ix->n};
    iv.sa = ix->d_sa;
    iv.rank = ix->d_rank;
    iv.starts = ix->d_starts;
    iv.lens = ix->d_lens;
    iv.start_rank = ix->d_start_rank;
    iv.start_frag = ix->d_start_frag;
    iv.start_inv = ix->d_start_inv;
    iv.dir = ix->dna && ix->d_dir ? ix->d_dir + 1 : nullptr;
    iv.sdir = ix->dna && ix->d_sdir ? ix->d_sdir + 1 : nullptr;
    iv.D = ix->dir_bases;
    iv.sD = ix->sdir_bases;
    iv.min_len = ix->min_len;
    iv.k = static_cast<u32>(ix->k);
    return iv;
}

int choose_dir_bases(size_t n) {
    // aim at ~16 suffixes per bucket, table between 4^6 and 4^13 entries (<= 256 MiB)
    int D = 6;
    while (D < 13 && (size_t{1} << (2 * D)) * 16 < n) ++D;
    return D;
}

// Exclusive scan of a u32 histogram of `count` entries whose total is < 2^32.
int scan_table(reseq_cuda_ctx* ctx, const u32* hist, u32* out, size_t count) {
    u64* d_total = ctx->alloc<u64>(1);
    if (!d_total) return fail(RESEQ_OUT_OF_MEMORY, "directory scan workspace");
    return exclusive_scan_device(ctx, hist, out, count, d_total);
}

// The two kernels behind the overlap counts: with a packed text and a directory every query is
// anchored at its own rank and the containment flags come from contained_kernel; otherwise (generic
// alphabets) the full interval search does both.
int launch_overlap_count(reseq_cuda_ctx* ctx, const IndexView& iv, u32 min_overlap, u64 f0, u64 f1, const u64* d_qoff,
                         u32* q_first, u32* q_count, u8* d_contained, u32* rawcount, unsigned grid) {
    cudaStream_t s = ctx->stream;
    if (iv.tv.packed && iv.sdir) {
        RSQ_LAUNCH_BEGIN(ctx, "overlap_count_kernel");
        if (ctx->opt_overlap_stage != 0 && (reinterpret_cast<uintptr_t>(iv.rank) & 15) == 0 &&
            (reinterpret_cast<uintptr_t>(iv.tv.packed) & 15) == 0)
            overlap_count_kernel<false, true><<<grid, 256, 0, s>>>(iv, min_overlap, f0, f1, d_qoff, q_first, q_count, d_contained,
                                                                   rawcount);
        else
            overlap_count_kernel<false, false><<<grid, 256, 0, s>>>(iv, min_overlap, f0, f1, d_qoff, q_first, q_count, d_contained,
                                                                    rawcount);
        RSQ_LAUNCH_END(ctx);
        RSQ_LAUNCH_BEGIN(ctx, "contained_kernel");
        contained_kernel<<<grid_1d(ctx, f1 - f0, 256), 256, 0, s>>>(iv, f0, f1, d_contained);
        RSQ_LAUNCH_END(ctx);
    } else {
        RSQ_LAUNCH_BEGIN(ctx, "overlap_count_kernel");
        overlap_count_kernel<true><<<grid, 256, 0, s>>>(iv, min_overlap, f0, f1, d_qoff, q_first, q_count, d_contained,
                                                        rawcount);
        RSQ_LAUNCH_END(ctx);
    }
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

}  // namespace

extern "C" {

int reseq_cuda_index_create(reseq_cuda_ctx* ctx, const uint8_t* concat, size_t n, const uint32_t* starts,
                            size_t k, reseq_cuda_index** out) {
    if (!out) return fail(RESEQ_INVALID_ARGUMENT, "null out pointer");
    *out = nullptr;
    if (!ctx) return fail(RESEQ_INVALID_ARGUMENT, "null context");
    RSQ_CUDA(cudaSetDevice(ctx->device));
    if (n > RESEQ_CUDA_MAX_TEXT)
        return fail(RESEQ_TEXT_TOO_LARGE, "text of length " + std::to_string(n) + " exceeds 2^32-2");
    if (n == 0 || k == 0 || !concat || !starts)
        return fail(RESEQ_INVALID_ARGUMENT, "an index needs at least one fragment");
    if (concat[n - 1] != 0)
        return fail(RESEQ_INVALID_ARGUMENT, "concat must end with the separator byte (sequence.hpp:60-62)");
    // The reference can only build a fragment_set through make_fragment_set (sequence.hpp:103-124),
    // which guarantees this layout; the C ABI takes raw arrays, so it is checked here, O(k) on the host:
    // starts[0] == 0, strictly ascending, inside the text, every fragment non-empty and preceded by a
    // separator.  (Separators INSIDE a fragment are not looked for: that is O(n).)  The check runs below, under the
    // host-to-device copy of the text.
    auto* ix = new reseq_cuda_index();
    ix->ctx = ctx;
    ix->n = n;
    ix->k = k;
    auto bail = [&](int code) {
        reseq_cuda_index_destroy(ix);
        return code;
    };
#define IX_TRY(expr)                            \
    do {                                        \
        int _s = (expr);                        \
        if (_s != RESEQ_OK) return bail(_s);    \
    } while (0)
#define IX_CUDA(expr)                                                                        \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return bail(fail(RESEQ_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e))); \
    } while (0)

    cudaStream_t s = ctx->stream;
    const bool dbg = std::getenv("RESEQ_DEBUG") != nullptr;   // phase timestamps (synchronising: for diagnosis only)
    auto t_prev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(s);
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[reseq] index_create %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_prev).count());
        t_prev = t;
    };
    IX_TRY(dev_alloc(ix, &ix->d_text, n));
    IX_TRY(dev_alloc(ix, &ix->d_sa, n));
    IX_TRY(dev_alloc(ix, &ix->d_rank, n));
    IX_TRY(dev_alloc(ix, &ix->d_starts, k));
    IX_TRY(dev_alloc(ix, &ix->d_lens, k));
    IX_TRY(dev_alloc(ix, &ix->d_start_rank, k));
    IX_TRY(dev_alloc(ix, &ix->d_start_frag, k));
    IX_TRY(dev_alloc(ix, &ix->d_start_inv, k));
    IX_TRY(dev_alloc(ix, &ix->d_packed, n / 32 + 8));
    IX_TRY(dev_alloc(ix, &ix->d_sent, n / 64 + 8));
    lap("allocations");
    IX_CUDA(cudaMemcpyAsync(ix->d_text, concat, n, cudaMemcpyHostToDevice, s));   // (page-locked text: the DMA runs under the host loop below)
    if (starts[0] != 0) return bail(fail(RESEQ_INVALID_ARGUMENT, "starts[0] must be 0 (sequence.hpp:119)"));
    // ONE pass over `starts` (it runs under the text's DMA): order and bounds, the fragment lengths
    // (sequence.hpp:78-83) and which lengths occur (lengths_, fragment_index.hpp:52-55).  That every start
    // follows a separator byte is checked on the device (lens_kernel), next to the text.
    std::vector<u32>& h_lens = ix->h_lens;
    h_lens.resize(k);
    std::vector<unsigned char> seen(1024, 0);
    u32 max_len = 0;
    for (size_t i = 0; i < k; ++i) {
        const uint64_t a0 = starts[i], b0 = i + 1 < k ? starts[i + 1] : n;
        if (b0 > n || b0 < a0 + 2)
            return bail(fail(RESEQ_INVALID_ARGUMENT, "starts[" + std::to_string(i + 1 < k ? i + 1 : i) +
                                                         "] does not follow a non-empty fragment inside the text (sequence.hpp:60-62,110)"));
        const u32 len = static_cast<u32>(b0 - 1 - a0);
        h_lens[i] = len;
        if (len >= seen.size()) seen.resize(std::max<size_t>(2 * seen.size(), static_cast<size_t>(len) + 1), 0);
        seen[len] = 1;
        max_len = std::max(max_len, len);
    }
    std::vector<u32>& distinct = ix->h_lengths;
    for (size_t v = 0; v <= max_len; ++v)
        if (seen[v]) distinct.push_back(static_cast<u32>(v));

    ix->max_len = max_len;
    ix->n_lengths = static_cast<u32>(distinct.size());
    ix->min_len = distinct.front();
    IX_TRY(dev_alloc(ix, &ix->d_lengths, distinct.size()));
    IX_CUDA(cudaMemcpyAsync(ix->d_starts, starts, sizeof(u32) * k, cudaMemcpyHostToDevice, s));
    IX_CUDA(cudaMemcpyAsync(ix->d_lens, h_lens.data(), sizeof(u32) * k, cudaMemcpyHostToDevice, s));        // (both vectors live in the index)
    IX_CUDA(cudaMemcpyAsync(ix->d_lengths, distinct.data(), sizeof(u32) * distinct.size(), cudaMemcpyHostToDevice, s));

    lap("host pass + H2D");
    // suffix array (fragment_index.hpp:37)
    IX_TRY(ctx->reserve(sa_workspace_bytes(n)));
    ctx->begin();
    reseq_sa_stats st{};
    IX_TRY(build_sa_device(ctx, ix->d_text, n, ix->d_sa, ix->d_rank, &st, ix->d_packed, ix->d_sent));   // packs once, for both
    ix->dna = st.alphabet == 0;
    lap("suffix array");

    // lengths, start ranks (fragment_index.hpp:40-48), directories
    const int D = choose_dir_bases(n);
    const size_t dir_entries = (size_t{1} << (2 * D)) + 2;
    const size_t need = 4 * reseq_cuda_ctx::padded(sizeof(u32) * k) + sort_workspace_bytes(k) +
                        reseq_cuda_ctx::padded(sizeof(u32) * dir_entries) + scan_workspace_bytes(dir_entries) +
                        8192;
    IX_TRY(ctx->reserve(need));
    ctx->begin();
    u32* keys_a = ctx->alloc<u32>(k);
    u32* keys_b = ctx->alloc<u32>(k);
    u32* ids_a = ctx->alloc<u32>(k);
    u32* ids_b = ctx->alloc<u32>(k);
    u32* counters = ctx->alloc<u32>(64);
    u32* hist = ctx->alloc<u32>(dir_entries);
    if (!keys_a || !keys_b || !ids_a || !ids_b || !counters || !hist)
        return bail(fail(RESEQ_OUT_OF_MEMORY, "index workspace"));
    IX_CUDA(cudaMemsetAsync(counters, 0, 256, s));
    RSQ_LAUNCH_BEGIN(ctx, "lens_kernel");
    lens_kernel<<<grid_1d(ctx, k, 256), 256, 0, s>>>(ix->d_starts, k, n, ix->d_lens, ix->d_rank, keys_a,
                                                     ids_a, counters, ix->d_text);
    IX_CUDA(cudaMemcpyAsync(ctx->pinned + 64, counters + 1, sizeof(u32), cudaMemcpyDeviceToHost, s));   // layout verdict, read at the end
    RSQ_LAUNCH_END(ctx);
    IX_CUDA(cudaGetLastError());
    if (k > 1) {
        SortWorkspace ws;
        IX_TRY(sort_workspace_carve(ctx, k, &ws));
        bool in_b = false;
        const PassTable pt = make_passes(0, static_cast<int>(bit_width_u64(n)));
        IX_TRY(onesweep_sort<u32>(ctx, keys_a, keys_b, ids_a, ids_b, k, pt, ws, false, 0, &in_b));
        IX_CUDA(cudaMemcpyAsync(ix->d_start_rank, in_b ? keys_b : keys_a, sizeof(u32) * k,
                                cudaMemcpyDeviceToDevice, s));
        IX_CUDA(cudaMemcpyAsync(ix->d_start_frag, in_b ? ids_b : ids_a, sizeof(u32) * k,
                                cudaMemcpyDeviceToDevice, s));
    } else {
        IX_CUDA(cudaMemcpyAsync(ix->d_start_rank, keys_a, sizeof(u32), cudaMemcpyDeviceToDevice, s));
        IX_CUDA(cudaMemcpyAsync(ix->d_start_frag, ids_a, sizeof(u32), cudaMemcpyDeviceToDevice, s));
    }
    RSQ_LAUNCH_BEGIN(ctx, "invert_kernel");
    invert_kernel<<<grid_1d(ctx, k, 256), 256, 0, s>>>(ix->d_start_frag, k, ix->d_start_inv);
    RSQ_LAUNCH_END(ctx);
    IX_CUDA(cudaGetLastError());
    lap("start ranks");
    if (ix->dna) {
        ix->dir_bases = D;
        ix->sdir_bases = D < 11 ? D : 11;   // 4^11 entries = 16 MB: L2-resident, and k start suffixes still land ~1 per bucket
        const size_t sdir_entries = (size_t{1} << (2 * ix->sdir_bases)) + 2;
        IX_TRY(dev_alloc(ix, &ix->d_dir, dir_entries));
        IX_TRY(dev_alloc(ix, &ix->d_sdir, sdir_entries));
        for (int which = 0; which < 2; ++which) {
            const size_t entries = which == 0 ? dir_entries : sdir_entries;
            IX_CUDA(cudaMemsetAsync(hist, 0, sizeof(u32) * entries, s));
            const size_t count = which == 0 ? n : k;
            RSQ_LAUNCH_BEGIN(ctx, "dir_hist_kernel");
            dir_hist_kernel<<<grid_1d(ctx, count, 256), 256, 0, s>>>(
                ix->d_packed, ix->d_sent, n, which == 0 ? nullptr : ix->d_starts, count,
                which == 0 ? D : ix->sdir_bases, hist);
            RSQ_LAUNCH_END(ctx);
            IX_CUDA(cudaGetLastError());
            IX_TRY(scan_table(ctx, hist, which == 0 ? ix->d_dir : ix->d_sdir, entries));
        }
    }
    IX_CUDA(cudaStreamSynchronize(s));
    lap("directories");
    if (*reinterpret_cast<volatile u32*>(ctx->pinned + 64) != 0)
        return bail(fail(RESEQ_INVALID_ARGUMENT, "a fragment does not end at a separator byte: starts does not describe concat (sequence.hpp:60-62)"));
#undef IX_TRY
#undef IX_CUDA
    *out = ix;
    return RESEQ_OK;
}

void reseq_cuda_index_destroy(reseq_cuda_index* ix) {
    if (!ix) return;
    if (ix->ctx) {
        cudaSetDevice(ix->ctx->device);
        cudaStreamSynchronize(ix->ctx->stream);
    }
    for (void* p : ix->owned) cudaFreeAsync(p, ix->ctx ? ix->ctx->stream : nullptr);
    if (ix->ctx) cudaStreamSynchronize(ix->ctx->stream);
    delete ix;
}

size_t reseq_cuda_index_text_len(const reseq_cuda_index* ix) { return ix ? ix->n : 0; }
size_t reseq_cuda_index_fragments(const reseq_cuda_index* ix) { return ix ? ix->k : 0; }

int reseq_cuda_index_get(const reseq_cuda_index* ix, uint32_t* sa, uint32_t* rank, uint32_t* start_rank_list) {
    if (!ix) return fail(RESEQ_INVALID_ARGUMENT, "null index");
    RSQ_CUDA(cudaSetDevice(ix->ctx->device));
    cudaStream_t s = ix->ctx->stream;
    if (sa) RSQ_CUDA(cudaMemcpyAsync(sa, ix->d_sa, sizeof(u32) * ix->n, cudaMemcpyDeviceToHost, s));
    if (rank) RSQ_CUDA(cudaMemcpyAsync(rank, ix->d_rank, sizeof(u32) * ix->n, cudaMemcpyDeviceToHost, s));
    if (start_rank_list)
        RSQ_CUDA(cudaMemcpyAsync(start_rank_list, ix->d_start_rank, sizeof(u32) * ix->k, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    return RESEQ_OK;
}

int reseq_cuda_index_start_fragments(const reseq_cuda_index* ix, uint32_t* start_fragments) {
    if (!ix || !start_fragments) return fail(RESEQ_INVALID_ARGUMENT, "null argument");
    RSQ_CUDA(cudaSetDevice(ix->ctx->device));
    cudaStream_t s = ix->ctx->stream;
    RSQ_CUDA(cudaMemcpyAsync(start_fragments, ix->d_start_frag, sizeof(u32) * ix->k, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    return RESEQ_OK;
}

int reseq_cuda_index_device_ptrs(const reseq_cuda_index* ix, const uint32_t** d_sa, const uint32_t** d_rank,
                                 const uint32_t** d_start_rank_list) {
    if (!ix) return fail(RESEQ_INVALID_ARGUMENT, "null index");
    if (d_sa) *d_sa = ix->d_sa;
    if (d_rank) *d_rank = ix->d_rank;
    if (d_start_rank_list) *d_start_rank_list = ix->d_start_rank;
    return RESEQ_OK;
}

int reseq_cuda_index_locate_batch(reseq_cuda_index* ix, const uint8_t* pats, const uint64_t* pat_off, size_t q,
                                  uint32_t* lo, uint32_t* hi) {
    if (!ix) return fail(RESEQ_INVALID_ARGUMENT, "null index");
    if (q == 0) return RESEQ_OK;
    if (!pats || !pat_off || !lo || !hi) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    for (size_t i = 0; i < q; ++i)
        if (pat_off[i + 1] <= pat_off[i])
            return fail(RESEQ_INVALID_ARGUMENT, "patterns must be non-empty (fragment_index.hpp:63-64)");
    reseq_cuda_ctx* ctx = ix->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t bytes = pat_off[q];
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(pad(bytes) + pad(sizeof(u64) * (q + 1)) + 2 * pad(sizeof(u32) * q) + 4096));
    ctx->begin();
    u8* d_pats = ctx->alloc<u8>(bytes);
    u64* d_off = ctx->alloc<u64>(q + 1);
    u32* d_lo = ctx->alloc<u32>(q);
    u32* d_hi = ctx->alloc<u32>(q);
    RSQ_CUDA(cudaMemcpyAsync(d_pats, pats, bytes, cudaMemcpyHostToDevice, s));
    RSQ_CUDA(cudaMemcpyAsync(d_off, pat_off, sizeof(u64) * (q + 1), cudaMemcpyHostToDevice, s));
    RSQ_LAUNCH_BEGIN(ctx, "locate_patterns_kernel");
    locate_patterns_kernel<<<grid_1d(ctx, q, 256), 256, 0, s>>>(view_of(ix), d_pats, d_off, q, d_lo, d_hi);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(lo, d_lo, sizeof(u32) * q, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaMemcpyAsync(hi, d_hi, sizeof(u32) * q, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    return RESEQ_OK;
}

int reseq_cuda_index_locate_residuals(reseq_cuda_index* ix, const uint32_t* frag, const uint32_t* off, size_t q,
                                      uint32_t* lo, uint32_t* hi) {
    if (!ix) return fail(RESEQ_INVALID_ARGUMENT, "null index");
    if (q == 0) return RESEQ_OK;
    if (!frag || !off || !lo || !hi) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    reseq_cuda_ctx* ctx = ix->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // residual_view's bounds check (sequence.hpp:127-131) on the host copy of the lengths
    const std::vector<u32>& lens = ix->h_lens;
    for (size_t i = 0; i < q; ++i)
        if (frag[i] >= ix->k || off[i] >= lens[frag[i]])
            return fail(RESEQ_INVALID_ARGUMENT, "residual offset out of range (sequence.hpp:128-129)");
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(4 * pad(sizeof(u32) * q) + 4096));
    ctx->begin();
    u32* d_frag = ctx->alloc<u32>(q);
    u32* d_offs = ctx->alloc<u32>(q);
    u32* d_lo = ctx->alloc<u32>(q);
    u32* d_hi = ctx->alloc<u32>(q);
    RSQ_CUDA(cudaMemcpyAsync(d_frag, frag, sizeof(u32) * q, cudaMemcpyHostToDevice, s));
    RSQ_CUDA(cudaMemcpyAsync(d_offs, off, sizeof(u32) * q, cudaMemcpyHostToDevice, s));
    RSQ_LAUNCH_BEGIN(ctx, "locate_residuals_kernel");
    locate_residuals_kernel<<<grid_1d(ctx, q, 256), 256, 0, s>>>(view_of(ix), d_frag, d_offs, q, d_lo, d_hi);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    RSQ_CUDA(cudaMemcpyAsync(lo, d_lo, sizeof(u32) * q, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaMemcpyAsync(hi, d_hi, sizeof(u32) * q, cudaMemcpyDeviceToHost, s));
    RSQ_CUDA(cudaStreamSynchronize(s));
    return RESEQ_OK;
}

void reseq_cuda_prefix_relations_free(reseq_prefix_relations* r) {
    if (!r) return;
    std::free(r->prefixes_off);
    std::free(r->extensions_off);
    std::free(r->exact_off);
    std::free(r->prefixes);
    std::free(r->extensions);
    std::free(r->exact);
    std::memset(r, 0, sizeof(*r));
}

int reseq_cuda_index_prefix_related_batch(reseq_cuda_index* ix, const uint32_t* frag, const uint32_t* off,
                                          size_t q, reseq_prefix_relations* out) {
    if (!ix || !out) return fail(RESEQ_INVALID_ARGUMENT, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->q = q;
    reseq_cuda_ctx* ctx = ix->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    uint64_t** offs[3] = {&out->prefixes_off, &out->extensions_off, &out->exact_off};
    uint32_t** ids[3] = {&out->prefixes, &out->extensions, &out->exact};
    for (auto* o : offs) {
        *o = static_cast<uint64_t*>(std::calloc(q + 1, sizeof(uint64_t)));
        if (!*o) return fail(RESEQ_OUT_OF_MEMORY, "host allocation failed");
    }
    if (q == 0) return RESEQ_OK;
    if (!frag || !off) return fail(RESEQ_INVALID_ARGUMENT, "null buffer");
    const std::vector<u32>& lens = ix->h_lens;
    for (size_t i = 0; i < q; ++i)
        if (frag[i] >= ix->k || off[i] >= lens[frag[i]])
            return fail(RESEQ_INVALID_ARGUMENT, "residual offset out of range (sequence.hpp:128-129)");
    auto pad = reseq_cuda_ctx::padded;
    RSQ_TRY(ctx->reserve(8 * pad(sizeof(u32) * (q + 1)) + 3 * scan_workspace_bytes(q + 1) + 8192));
    ctx->begin();
    u32* d_frag = ctx->alloc<u32>(q);
    u32* d_offs = ctx->alloc<u32>(q);
    u32* cnt[3];
    u32* pos[3];
    u64* d_tot[3];
    for (int t = 0; t < 3; ++t) {
        cnt[t] = ctx->alloc<u32>(q + 1);
        pos[t] = ctx->alloc<u32>(q + 1);
        d_tot[t] = ctx->alloc<u64>(1);
        RSQ_CUDA(cudaMemsetAsync(cnt[t] + q, 0, sizeof(u32), s));
    }
    RSQ_CUDA(cudaMemcpyAsync(d_frag, frag, sizeof(u32) * q, cudaMemcpyHostToDevice, s));
    RSQ_CUDA(cudaMemcpyAsync(d_offs, off, sizeof(u32) * q, cudaMemcpyHostToDevice, s));
    const IndexView iv = view_of(ix);
    RSQ_LAUNCH_BEGIN(ctx, "prefix_related_kernel");
    prefix_related_kernel<0><<<grid_1d(ctx, q, 256), 256, 0, s>>>(iv, ix->d_lengths, ix->n_lengths, d_frag, d_offs, q,
                                                                  cnt[0], cnt[1], cnt[2], nullptr, nullptr, nullptr,
                                                                  nullptr, nullptr, nullptr);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    u64 totals[3];
    std::vector<u32> host_pos(q + 1);
    for (int t = 0; t < 3; ++t) {
        RSQ_TRY(exclusive_scan_device(ctx, cnt[t], pos[t], q + 1, d_tot[t]));
        RSQ_CUDA(cudaMemcpyAsync(host_pos.data(), pos[t], sizeof(u32) * (q + 1), cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_tot[t], sizeof(u64), cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaStreamSynchronize(s));
        totals[t] = *reinterpret_cast<volatile u64*>(ctx->pinned);
        if (totals[t] > 0xFFFFFFF0ull) return fail(RESEQ_INVALID_ARGUMENT, "more than 2^32 relation entries");
        for (size_t i = 0; i <= q; ++i) (*offs[t])[i] = host_pos[i];
    }
    // the id arrays follow the query arrays in the arena; grow it if the totals need more
    const size_t used = ctx->arena_used;
    const size_t more = pad(sizeof(u32) * (totals[0] + 1)) + pad(sizeof(u32) * (totals[1] + 1)) +
                        pad(sizeof(u32) * (totals[2] + 1)) + 1024;
    if (ctx->arena_cap < used + more) {
        // re-run from scratch in a larger arena
        RSQ_TRY(ctx->reserve(used + more + 8192));
        reseq_cuda_prefix_relations_free(out);
        return reseq_cuda_index_prefix_related_batch(ix, frag, off, q, out);
    }
    u32* d_out[3];
    for (int t = 0; t < 3; ++t) d_out[t] = ctx->alloc<u32>(totals[t] + 1);
    RSQ_LAUNCH_BEGIN(ctx, "prefix_related_kernel");
    prefix_related_kernel<1><<<grid_1d(ctx, q, 256), 256, 0, s>>>(iv, ix->d_lengths, ix->n_lengths, d_frag, d_offs, q,
                                                                  nullptr, nullptr, nullptr, pos[0], pos[1], pos[2],
                                                                  d_out[0], d_out[1], d_out[2]);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    for (int t = 0; t < 3; ++t) {
        *ids[t] = static_cast<uint32_t*>(std::malloc(sizeof(u32) * (totals[t] + 1)));
        if (!*ids[t]) return fail(RESEQ_OUT_OF_MEMORY, "host allocation failed");
        RSQ_CUDA(cudaMemcpyAsync(*ids[t], d_out[t], sizeof(u32) * totals[t], cudaMemcpyDeviceToHost, s));
    }
    RSQ_CUDA(cudaStreamSynchronize(s));
    for (int t = 0; t < 3; ++t)  // each list ascending by id (fragment_index.hpp:105-107)
        for (size_t i = 0; i < q; ++i)
            std::sort(*ids[t] + (*offs[t])[i], *ids[t] + (*offs[t])[i + 1]);
    return RESEQ_OK;
}

int reseq_cuda_index_overlaps(reseq_cuda_index* ix, uint32_t min_overlap, reseq_overlaps* out) {
    return reseq_cuda_index_overlaps_range(ix, min_overlap, 0, ix ? ix->k : 0, out);
}

}  // extern "C"

namespace {
struct OverlapDest {   // caller-owned output arrays of reseq_cuda_index_overlaps_into
    u32 *i, *j, *w;
    size_t capacity;
    u8* contained;
};
}  // namespace

static int overlaps_impl(reseq_cuda_index* ix, uint32_t min_overlap, size_t frag_begin, size_t frag_end,
                         reseq_overlaps* out, const OverlapDest* dest) {
    if (!ix || !out) return fail(RESEQ_INVALID_ARGUMENT, "null argument");
    std::memset(out, 0, sizeof(*out));
    if (frag_begin > frag_end || frag_end > ix->k) return fail(RESEQ_INVALID_ARGUMENT, "fragment range out of bounds");
    if (min_overlap < 1) min_overlap = 1;
    const size_t f0 = frag_begin, f1 = frag_end, kr = frag_end - frag_begin;
    reseq_cuda_ctx* ctx = ix->ctx;
    RSQ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t k = ix->k;
    auto pad = reseq_cuda_ctx::padded;

    // -- per-fragment query counts -> query offsets (host prefix sum; k entries) -----------
    const std::vector<u32>& lens = ix->h_lens;
    std::vector<u64> qoff(kr + 1, 0);
    for (size_t i = 0; i < kr; ++i)
        qoff[i + 1] = qoff[i] + (lens[f0 + i] >= min_overlap ? lens[f0 + i] - min_overlap + 1 : 0);
    const u64 Q = qoff[kr];
    out->queries = Q;
    if (dest) {
        out->contained = dest->contained;
        std::memset(out->contained, 0, k);
    } else {
        out->contained = static_cast<uint8_t*>(std::calloc(k, 1));
    }
    if (!out->contained) return fail(RESEQ_OUT_OF_MEMORY, "host allocation failed");
    if (Q > 0xFFFFFFF0ull) return fail(RESEQ_INVALID_ARGUMENT, "more than 2^32 overlap queries in one call");

    cudaEvent_t ev0, ev1;
    RSQ_CUDA(cudaEventCreate(&ev0));
    RSQ_CUDA(cudaEventCreate(&ev1));

    size_t need = pad(sizeof(u64) * (kr + 1)) + 3 * pad(sizeof(u32) * (Q + 1)) + pad(k) +
                  2 * pad(sizeof(u32) * (kr + 1)) + scan_workspace_bytes(Q + 1) + scan_workspace_bytes(kr + 1) + 8192;
    RSQ_TRY(ctx->reserve(need));
    ctx->begin();
    u64* d_qoff = ctx->alloc<u64>(kr + 1);
    u32* q_first = ctx->alloc<u32>(Q + 1);
    u32* q_count = ctx->alloc<u32>(Q + 1);
    u32* q_out = ctx->alloc<u32>(Q + 1);
    u8* d_contained = ctx->alloc<u8>(k);
    u64* d_total = ctx->alloc<u64>(1);
    u32* rawcount = ctx->alloc<u32>(kr + 1);
    u32* rbase = ctx->alloc<u32>(kr + 1);
    if (!d_qoff || !q_first || !q_count || !q_out || !d_contained || !d_total || !rawcount || !rbase)
        return fail(RESEQ_OUT_OF_MEMORY, "overlap workspace");
    RSQ_CUDA(cudaMemcpyAsync(d_qoff, qoff.data(), sizeof(u64) * (kr + 1), cudaMemcpyHostToDevice, s));
    RSQ_CUDA(cudaMemsetAsync(d_contained, 0, k, s));
    RSQ_CUDA(cudaMemsetAsync(q_count + Q, 0, sizeof(u32), s));
    const IndexView iv = view_of(ix);

    RSQ_CUDA(cudaEventRecord(ev0, s));
    u64 raw = 0;
    if (kr > 0) {
        const unsigned grid = grid_1d(ctx, kr * 32, 256, 32);
        RSQ_CUDA(cudaMemsetAsync(rawcount + kr, 0, sizeof(u32), s));
        RSQ_TRY(launch_overlap_count(ctx, iv, min_overlap, f0, f1, d_qoff, q_first, q_count, d_contained, rawcount, grid));
        RSQ_TRY(exclusive_scan_device(ctx, rawcount, rbase, kr + 1, d_total));
        RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_total, sizeof(u64), cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaStreamSynchronize(s));
        raw = *reinterpret_cast<volatile u64*>(ctx->pinned);
    }
    RSQ_CUDA(cudaMemcpyAsync(out->contained, d_contained, k, cudaMemcpyDeviceToHost, s));
    if (raw > 0xFFFFFFF0ull) return fail(RESEQ_INVALID_ARGUMENT, "more than 2^32 raw overlap records");

    u64 uniq = 0;
    if (raw > 0) {
        // The query arrays stay where they are; the record buffers follow them in the arena.
        const size_t used_before = ctx->arena_used;
        const size_t more = 2 * pad(sizeof(u64) * raw) + 4 * pad(sizeof(u32) * raw) + 3 * pad(sizeof(u32) * raw) +
                            2 * pad(sizeof(u32) * (kr + 1)) + sort_workspace_bytes(raw) +
                            scan_workspace_bytes(raw) + scan_workspace_bytes(kr + 1) + scan_workspace_bytes(Q + 1) + 8192;
        if (ctx->arena_cap < used_before + more) {
            // grow: the arena is re-allocated, so redo pass 1 state in the new block
            RSQ_TRY(ctx->reserve(used_before + more));
            ctx->begin();
            d_qoff = ctx->alloc<u64>(kr + 1);
            q_first = ctx->alloc<u32>(Q + 1);
            q_count = ctx->alloc<u32>(Q + 1);
            q_out = ctx->alloc<u32>(Q + 1);
            d_contained = ctx->alloc<u8>(k);
            d_total = ctx->alloc<u64>(1);
            rawcount = ctx->alloc<u32>(kr + 1);
            rbase = ctx->alloc<u32>(kr + 1);
            RSQ_CUDA(cudaMemcpyAsync(d_qoff, qoff.data(), sizeof(u64) * (kr + 1), cudaMemcpyHostToDevice, s));
            RSQ_CUDA(cudaMemsetAsync(q_count + Q, 0, sizeof(u32), s));
            RSQ_CUDA(cudaMemsetAsync(rawcount + kr, 0, sizeof(u32), s));
            const unsigned grid = grid_1d(ctx, kr * 32, 256, 32);
            RSQ_TRY(launch_overlap_count(ctx, iv, min_overlap, f0, f1, d_qoff, q_first, q_count, d_contained, rawcount,
                                         grid));
            RSQ_TRY(exclusive_scan_device(ctx, rawcount, rbase, kr + 1, d_total));
        }
        u64* keys_a = ctx->alloc<u64>(raw);
        u64* keys_b = ctx->alloc<u64>(raw);
        u32* w_a = ctx->alloc<u32>(raw);
        u32* w_b = ctx->alloc<u32>(raw);
        u32* flag = ctx->alloc<u32>(raw);
        u32* dst = ctx->alloc<u32>(raw);
        u32* oi = ctx->alloc<u32>(raw);
        u32* oj = ctx->alloc<u32>(raw);
        u32* ow = ctx->alloc<u32>(raw);
        u64* d_total2 = ctx->alloc<u64>(1);
        u32* ucount = ctx->alloc<u32>(kr + 1);
        u32* uoff = ctx->alloc<u32>(kr + 1);
        if (!keys_a || !keys_b || !w_a || !w_b || !flag || !dst || !oi || !oj || !ow || !d_total2 || !ucount || !uoff)
            return fail(RESEQ_OUT_OF_MEMORY, "overlap record workspace");
        // -- fast form: every fragment's records sorted and deduplicated by one warp in shared memory --
        bool done = false;
        u32 *fin_i = oi, *fin_j = oj, *fin_w = ow;
        {
            u32* overflow = reinterpret_cast<u32*>(d_total2) + 1;   // upper half of the total word: free until the scan
            RSQ_CUDA(cudaMemsetAsync(d_total2, 0, sizeof(u64), s));
            const unsigned grid = grid_1d(ctx, kr * 32, 256, 32);
            RSQ_LAUNCH_BEGIN(ctx, "overlap_fill_sorted_kernel");
            overlap_fill_sorted_kernel<<<grid, 256, 0, s>>>(iv, f0, f1, d_qoff, q_first, q_count, rbase, w_a, w_b, flag,
                                                            ucount, overflow);
            RSQ_LAUNCH_END(ctx);
            RSQ_CUDA(cudaGetLastError());
            RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, overflow, sizeof(u32), cudaMemcpyDeviceToHost, s));
            RSQ_CUDA(cudaMemsetAsync(ucount + kr, 0, sizeof(u32), s));
            RSQ_TRY(exclusive_scan_device(ctx, ucount, uoff, kr + 1, d_total2));
            RSQ_CUDA(cudaMemcpyAsync(ctx->pinned + 1, d_total2, sizeof(u64), cudaMemcpyDeviceToHost, s));
            RSQ_CUDA(cudaStreamSynchronize(s));
            if (*reinterpret_cast<volatile u32*>(ctx->pinned) == 0) {
                done = true;
                uniq = *reinterpret_cast<volatile u64*>(ctx->pinned + 1);
                if (uniq == raw) {   // nothing was dropped: the raw offsets are the final ones
                    fin_i = w_a;
                    fin_j = w_b;
                    fin_w = flag;
                } else {
                    RSQ_LAUNCH_BEGIN(ctx, "overlap_close_gaps_kernel");
                    overlap_close_gaps_kernel<<<grid, 256, 0, s>>>(kr, rbase, ucount, uoff, w_a, w_b, flag, oi, oj, ow);
                    RSQ_LAUNCH_END(ctx);
                    RSQ_CUDA(cudaGetLastError());
                }
                RSQ_CUDA(cudaEventRecord(ev1, s));
            }
        }
        if (!done) {   // a fragment with more raw records than a warp's window: global sort + unique
        {
            RSQ_TRY(exclusive_scan_device(ctx, q_count, q_out, Q + 1, d_total));   // per-query record offsets
            const unsigned grid = grid_1d(ctx, kr * 32, 256, 32);
            RSQ_LAUNCH_BEGIN(ctx, "overlap_fill_kernel");
            overlap_fill_kernel<<<grid, 256, 0, s>>>(iv, f0, f1, d_qoff, q_first, q_count, q_out, keys_a, w_a);
            RSQ_LAUNCH_END(ctx);
            RSQ_CUDA(cudaGetLastError());
        }
        // stable sort on (i, j): j digits then i digits
        const int kb = static_cast<int>(bit_width_u64(k));
        PassTable pt = make_passes(0, kb);
        const PassTable hi_pt = make_passes(32, 32 + kb);
        for (int p = 0; p < hi_pt.count; ++p) {
            pt.shift[pt.count] = hi_pt.shift[p];
            pt.bits[pt.count] = hi_pt.bits[p];
            ++pt.count;
        }
        SortWorkspace ws;
        RSQ_TRY(sort_workspace_carve(ctx, raw, &ws));
        bool in_b = false;
        RSQ_TRY(onesweep_sort<u64>(ctx, keys_a, keys_b, w_a, w_b, raw, pt, ws, false, 0, &in_b));
        const u64* sk = in_b ? keys_b : keys_a;
        const u32* sw = in_b ? w_b : w_a;
        RSQ_LAUNCH_BEGIN(ctx, "unique_flag_kernel");
        unique_flag_kernel<<<grid_1d(ctx, raw, 256), 256, 0, s>>>(sk, raw, flag);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        RSQ_TRY(exclusive_scan_device(ctx, flag, dst, raw, d_total2));
        RSQ_LAUNCH_BEGIN(ctx, "unique_compact_kernel");
        unique_compact_kernel<<<grid_1d(ctx, raw, 256), 256, 0, s>>>(sk, sw, flag, dst, raw, oi, oj, ow);
        RSQ_LAUNCH_END(ctx);
        RSQ_CUDA(cudaGetLastError());
        RSQ_CUDA(cudaEventRecord(ev1, s));
        RSQ_CUDA(cudaMemcpyAsync(ctx->pinned, d_total2, sizeof(u64), cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaStreamSynchronize(s));
        uniq = *reinterpret_cast<volatile u64*>(ctx->pinned);
        }
        if (dest) {
            if (uniq > dest->capacity) {
                cudaEventDestroy(ev0);
                cudaEventDestroy(ev1);
                out->count = uniq;
                return fail(RESEQ_BUFFER_TOO_SMALL, "overlap arrays hold " + std::to_string(dest->capacity) +
                                                        " triples, " + std::to_string(uniq) + " found");
            }
            out->i = dest->i;
            out->j = dest->j;
            out->w = dest->w;
        } else {
            out->i = static_cast<uint32_t*>(std::malloc(sizeof(u32) * (uniq + 1)));
            out->j = static_cast<uint32_t*>(std::malloc(sizeof(u32) * (uniq + 1)));
            out->w = static_cast<uint32_t*>(std::malloc(sizeof(u32) * (uniq + 1)));
        }
        if (!out->i || !out->j || !out->w) return fail(RESEQ_OUT_OF_MEMORY, "host allocation failed");
        RSQ_CUDA(cudaMemcpyAsync(out->i, fin_i, sizeof(u32) * uniq, cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaMemcpyAsync(out->j, fin_j, sizeof(u32) * uniq, cudaMemcpyDeviceToHost, s));
        RSQ_CUDA(cudaMemcpyAsync(out->w, fin_w, sizeof(u32) * uniq, cudaMemcpyDeviceToHost, s));
    } else {
        RSQ_CUDA(cudaEventRecord(ev1, s));
    }
    RSQ_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    RSQ_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    out->device_ms = ms;
    out->count = uniq;
    return RESEQ_OK;
}

extern "C" {

int reseq_cuda_index_overlaps_range(reseq_cuda_index* ix, uint32_t min_overlap, size_t frag_begin,
                                    size_t frag_end, reseq_overlaps* out) {
    return overlaps_impl(ix, min_overlap, frag_begin, frag_end, out, nullptr);
}

int reseq_cuda_index_overlaps_into(reseq_cuda_index* ix, uint32_t min_overlap, size_t frag_begin, size_t frag_end,
                                   uint32_t* i, uint32_t* j, uint32_t* w, size_t capacity, uint8_t* contained,
                                   reseq_overlaps* out) {
    if (!contained || (capacity && (!i || !j || !w))) return fail(RESEQ_INVALID_ARGUMENT, "null output array");
    const OverlapDest dest{i, j, w, capacity, contained};
    return overlaps_impl(ix, min_overlap, frag_begin, frag_end, out, &dest);
}

void reseq_cuda_overlaps_free(reseq_overlaps* o) {
    if (!o) return;
    std::free(o->i);
    std::free(o->j);
    std::free(o->w);
    std::free(o->contained);
    std::memset(o, 0, sizeof(*o));
}

}  // extern "C"
