// radix.cuh — internal entry to the H5 radix partition (radix.cu) for other operators.
#pragma once
#include "common.cuh"

namespace sx {

// Partition n rows (through sel, else 0..n-1) by hash bits 48.. of their key (one column, or two
// 32-bit columns packed (k0 << 32) | k1): carried column c (DCol carry[c], width[c] bytes) is
// written partition-contiguous to out[c] (caller-allocated, n * width[c] bytes).  offsets_h (host,
// 2^bits + 1) receives the partition boundaries.  Syncs once.
sx_status radix_partition_carry(sx_ctx* ctx, DCol k0, DCol k1, int nkeys, const DCol* carry, const int* width,
                                int ncarry, const int32_t* sel, int64_t n, int bits, void* const* out,
                                int64_t* offsets_h);

}  // namespace sx
