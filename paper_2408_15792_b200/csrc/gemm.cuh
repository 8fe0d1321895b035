#pragma once
#include <cuda_runtime.h>

namespace rs {
// epi: 0 none, 1 ReLU, 2 + residual R (same layout as C), 3 GELU(tanh)
int gemm_bf16(const void* A, const void* W, const void* bias, const void* R, void* C, int M, int N, int K, int epi,
              cudaStream_t st);
}  // namespace rs
