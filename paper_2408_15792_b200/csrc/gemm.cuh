#pragma once
#include <cuda_runtime.h>

namespace rs {
// epi: 0 none, 1 ReLU, 2 + residual R (same layout as C), 3 GELU(tanh)
int gemm_bf16(const void* A, const void* W, const void* bias, const void* R, void* C, int M, int N, int K, int epi,
              cudaStream_t st);
}  // namespace rs
namespace rs {
// General CTA-pair GEMM (see gemm.cu): a_mn / b_mn select MN-contiguous operand storage,
// epi 4 = fp32 out, 5 = bf16 * (aux > 0), 6 = fp32 split-K partial slices.
int gemm_bf16_ex(const void* A, const void* W, const void* bias, const void* aux, void* C, int M, int N, int K,
                 int epi, int a_mn, int b_mn, int k_splits, cudaStream_t st);
}  // namespace rs
