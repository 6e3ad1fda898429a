// Device suffix-array builder (see sa.cu).
#pragma once

#include "common.cuh"

namespace rsq {

// Arena bytes build_sa_device needs for a text of n bytes (excluding text / sa / rank,
// which the caller owns).
size_t sa_workspace_bytes(size_t n);

// d_text: n bytes in HBM; d_sa: n u32 out; d_rank: n u32 out (nullable).  Runs on
// ctx->stream; synchronises internally once per doubling round to read the group count.
// packed_out / sent_out (nullable, n/32+8 and n/64+8 u64): caller-owned arrays that receive the
// 2-bit packed text and the sentinel bitmap the build makes anyway (the index keeps them).
int build_sa_device(reseq_cuda_ctx* ctx, const u8* d_text, size_t n, u32* d_sa, u32* d_rank,
                    reseq_sa_stats* stats, u64* packed_out = nullptr, u64* sent_out = nullptr);

// 2-bit packing of a DNA text (shared with the index): returns false through *is_dna when
// a byte outside {0,A,C,G,T} is present.  packed needs n/32+8 u64, sent n/64+8 u64.
int pack_dna_device(reseq_cuda_ctx* ctx, const u8* d_text, size_t n, u64* packed, u64* sent,
                    u32* d_flag /* 2 words */, bool* is_dna, u64* n_separators /* nullable */);

}  // namespace rsq
