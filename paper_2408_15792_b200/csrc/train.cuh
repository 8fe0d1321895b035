#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace rs {
// LayerNorm backward over rows x d: dh += LN_bwd(dy; x, w), dh_bf16 = bf16(dh); adds the
// LN weight / bias gradients into dw_out[0..d) and dw_out[d..2d) (weight and bias are
// adjacent in the gradient layout; db_out is unused). dhsum_out (optional) += the column
// sums of the updated dh. part: ceil(rows/64) x 3d floats + ceil(rows/4096) x 2d scratch.
int ln_backward(const float* dy, const float* x, const void* w, float* dh, void* dh_bf16, float* part, int rows,
                int d, float* dw_out, float* db_out, cudaStream_t st, float* dhsum_out = nullptr);
// out[c] += sum over rows of x[:, c] (x float or bf16); part: ceil(rows/64) x cols floats.
int colsum_add(const void* x, bool is_bf16, int rows, int cols, float* part, float* out, cudaStream_t st);
// out[i] += sum over k slices of part[s * n + i]
int slices_add(const float* part, int k, int64_t n, float* out, cudaStream_t st);
size_t embed_backward_ws(int n);
int embed_backward(const int32_t* ids, int B, int S, int vocab, const float* dh, int d, float* dE, float* dP, void* ws,
                   size_t ws_bytes, cudaStream_t st);
// part: (B + 1) x (3d + 1) floats
int head_backward(const float* h, const int32_t* last, int B, int S, const void* lw, const void* lb, const void* hw,
                  const float* dg, float* dh, float* part, int d, float* g_hw, float* g_lnf, float* g_hb,
                  cudaStream_t st, const float* dfeat = nullptr);
// lse: the forward's row log2-sum-exp (attention_fwd_lse); colsum (needs lse): B x 3 H 64
// floats, row b = the column sums of prompt b's dQ | dK | dV rows (the bias gradients)
int attention_bwd(const void* qkv, const void* att, const void* dout, void* dqkv, int B, int S, int H, cudaStream_t st,
                  const float* lse = nullptr, float* colsum = nullptr);
// out[c] += sum of the n_part rows of part (fixed order); scratch: ceil(n_part / 16) x cols
int rows_add(const float* part, int n_part, int cols, float* out, float* scratch, cudaStream_t st);
}  // namespace rs
