// Device exclusive prefix sum (see scan.cu).
#pragma once

#include "common.cuh"

namespace rsq {

size_t scan_workspace_bytes(size_t n);

// out[i] = sum(in[0..i)) modulo 2^32; *d_total (device u64) receives the exact 64-bit
// grand total so callers can apply the overflow rule of scan.hpp:38.  Carves its
// descriptors from the context arena (the caller has reserved scan_workspace_bytes(n)).
int exclusive_scan_device(reseq_cuda_ctx* ctx, const u32* d_in, u32* d_out, size_t n,
                          u64* d_total);

}  // namespace rsq
