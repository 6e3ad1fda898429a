// Single-pass exclusive prefix sum (decoupled look-back) for sm_100a.
//
// Replaces exclusive_scan, scan.hpp:32-56: the reference runs ceil(log2 n)+3 full-array
// BSP phases (Hillis-Steele, O(n log n) work, scan.hpp:42-47); here every element is read
// once and written once (8 B/element of HBM traffic).  Thread-local serial scan over 16
// consecutive values loaded as four 128-bit words, warp scan by shuffles, block scan over
// warp totals, and a 64-bit (status | running-sum) descriptor per tile chained across
// tiles.  The 64-bit running sum doubles as the overflow check of scan.hpp:38.
#include "scan.cuh"

namespace rsq {

namespace {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanBlock * kScanItems;

template <bool VEC>
__global__ void __launch_bounds__(kScanBlock)
scan_kernel(const u32* __restrict__ in, u32* __restrict__ out, u64 n, u64* __restrict__ desc,
            u32* __restrict__ ticket, u64* __restrict__ total_out) {
    __shared__ u32 s_tile;
    __shared__ u64 s_warp[kScanBlock / 32];
    __shared__ u64 s_prefix;

    const int tid = threadIdx.x;
    const unsigned lane = lane_id();
    const int warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const u64 base = static_cast<u64>(tile) * kScanTile + static_cast<u64>(tid) * kScanItems;

    u32 v[kScanItems];
    if (VEC && base + kScanItems <= n) {
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            const uint4 w = ld_stream_v4(in + base + 4 * q);
            v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) v[j] = base + j < n ? in[base + j] : 0u;
    }

    u64 tsum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) tsum += v[j];

    u64 inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane) >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    u64 wadd = 0;
    u64 tile_total = 0;
#pragma unroll
    for (int w = 0; w < kScanBlock / 32; ++w) {
        if (w < warp) wadd += s_warp[w];
        tile_total += s_warp[w];
    }

    // Warp 0 chains the tile total: 32 predecessors are inspected per step.
    if (warp == 0) {
        u64 excl = 0;
        if (tile > 0) {
            if (lane == 0) st_relaxed_u64(desc + tile, kDescAggregate | tile_total);
            long long t = static_cast<long long>(tile) - 1 - lane;
            for (;;) {
                u64 d = 0;
                if (t >= 0) {
                    do {
                        d = ld_relaxed_u64(desc + t);
                    } while ((d >> 62) == 0);
                } else {
                    d = kDescInclusive;  // before tile 0: an inclusive prefix of 0
                }
                const unsigned incl = __ballot_sync(0xffffffffu, (d & kDescInclusive) != 0);
                // lanes are ordered nearest-first: sum up to and including the first
                // lane holding an inclusive prefix
                const int stop = __ffs(incl) - 1;  // -1 when none
                u64 part = (stop < 0 || static_cast<int>(lane) <= stop) ? (d & kDescValueMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                if (stop >= 0) break;
                t -= 32;
            }
        }
        if (lane == 0) {
            st_relaxed_u64(desc + tile, kDescInclusive | (excl + tile_total));
            s_prefix = excl;
            if (static_cast<u64>(tile) * kScanTile + kScanTile >= n) *total_out = excl + tile_total;
        }
    }
    __syncthreads();

    u32 run = static_cast<u32>(s_prefix + wadd + inc - tsum);
    if (VEC && base + kScanItems <= n) {
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            uint4 w;
            w.x = run; run += v[4 * q];
            w.y = run; run += v[4 * q + 1];
            w.z = run; run += v[4 * q + 2];
            w.w = run; run += v[4 * q + 3];
            st_stream_v4(out + base + 4 * q, w);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            if (base + j < n) out[base + j] = run;
            run += v[j];
        }
    }
}

}  // namespace

size_t scan_workspace_bytes(size_t n) {
    const size_t tiles = (n + kScanTile - 1) / kScanTile + 1;
    return reseq_cuda_ctx::padded(sizeof(u64) * (tiles + 2)) + reseq_cuda_ctx::padded(256);
}

int exclusive_scan_device(reseq_cuda_ctx* ctx, const u32* d_in, u32* d_out, size_t n,
                          u64* d_total) {
    if (n == 0) return RESEQ_OK;
    const size_t tiles = (n + kScanTile - 1) / kScanTile;
    u64* desc = ctx->alloc<u64>(tiles + 2);
    u32* ticket = ctx->alloc<u32>(64);
    if (!desc || !ticket) return fail(RESEQ_OUT_OF_MEMORY, "scan workspace does not fit the arena");
    RSQ_CUDA(cudaMemsetAsync(desc, 0, sizeof(u64) * (tiles + 2), ctx->stream));
    RSQ_CUDA(cudaMemsetAsync(ticket, 0, 256, ctx->stream));
    const bool vec = (reinterpret_cast<uintptr_t>(d_in) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(d_out) % 16 == 0);
    RSQ_LAUNCH_BEGIN(ctx, "scan_kernel");
    if (vec)
        scan_kernel<true><<<static_cast<unsigned>(tiles), kScanBlock, 0, ctx->stream>>>(
            d_in, d_out, n, desc, ticket, d_total);
    else
        scan_kernel<false><<<static_cast<unsigned>(tiles), kScanBlock, 0, ctx->stream>>>(
            d_in, d_out, n, desc, ticket, d_total);
    RSQ_LAUNCH_END(ctx);
    RSQ_CUDA(cudaGetLastError());
    return RESEQ_OK;
}

}  // namespace rsq
