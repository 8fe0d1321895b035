// K10 fast path (tau_fast.cu): exact tau-b counts by an MSD bucket partition of x, for
// y images spanning < 4096 values. counts[5] = 2 when the input needs the general path.
#pragma once
#include "common.cuh"

namespace rs {
constexpr int TF_DT_U32 = 100;  // x / y already 32-bit order-preserving images
size_t tau_fast_workspace(uint64_t n);
// A, B: n u32 scratch each (the general path's 32-bit sort buffers are reused).
// nan_flag (device int, optional): a NaN already seen by the caller's image pass.
int tau_fast_counts(const void* x, int xd, const void* y, int yd, uint32_t n, int64_t* counts, uint32_t* A,
                    uint32_t* B, const int* nan_flag, void* ws, size_t ws_bytes, cudaStream_t st);
}  // namespace rs
