// Training-path kernels of the OPT-shape ranker (K7/K8; the reference's counterparts
// are _Net.backward predictors.py:198-206 and _Adam.step predictors.py:218-225):
// LayerNorm backward, deterministic column sums (bias / LN parameter gradients),
// deterministic embedding scatter-add, the score-head backward and fused Adam.
// All reductions run in a fixed order (per-block partials, then an ordered reduce), so
// a training step is bitwise reproducible, as the reference's training is
// (test_predictors.py:171-177).
#include <cuda_bf16.h>
#include "common.cuh"
#include "mergesort.cuh"
#include "train.cuh"

namespace rs {

constexpr float TR_LN_EPS = 1e-5f;
constexpr int TR_ROWS_PER_BLOCK = 64;  // rows folded into one partial row of a column sum
constexpr int LNB_ROWS_PER_BLOCK = 256;  // LN backward: 32 rows per warp, 4x fewer partial rows to reduce

template <int VPL>
__device__ __forceinline__ void tr_load_f32(const float* __restrict__ x, int lane, float (&v)[VPL * 8]) {
    const float4* xr = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        float4 a = xr[2 * (lane + 32 * k)], b = xr[2 * (lane + 32 * k) + 1];
        v[k * 8 + 0] = a.x; v[k * 8 + 1] = a.y; v[k * 8 + 2] = a.z; v[k * 8 + 3] = a.w;
        v[k * 8 + 4] = b.x; v[k * 8 + 5] = b.y; v[k * 8 + 6] = b.z; v[k * 8 + 7] = b.w;
    }
}
template <int VPL>
__device__ __forceinline__ void tr_store_f32(float* __restrict__ x, int lane, const float (&v)[VPL * 8]) {
    float4* xr = reinterpret_cast<float4*>(x);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        xr[2 * (lane + 32 * k)] = make_float4(v[k * 8 + 0], v[k * 8 + 1], v[k * 8 + 2], v[k * 8 + 3]);
        xr[2 * (lane + 32 * k) + 1] = make_float4(v[k * 8 + 4], v[k * 8 + 5], v[k * 8 + 6], v[k * 8 + 7]);
    }
}
template <int VPL>
__device__ __forceinline__ void tr_store_bf16(__nv_bfloat16* __restrict__ x, int lane, const float (&v)[VPL * 8]) {
    uint4* xr = reinterpret_cast<uint4*>(x);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        uint4 o;
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(v[k * 8 + 2 * q], v[k * 8 + 2 * q + 1]);
        xr[lane + 32 * k] = o;
    }
}
template <int VPL>
__device__ __forceinline__ void tr_load_w(const __nv_bfloat16* __restrict__ w, int lane, float (&v)[VPL * 8]) {
    const uint4* wr = reinterpret_cast<const uint4*>(w);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        uint4 u = wr[lane + 32 * k];
        const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 f = __bfloat1622float2(u2[q]);
            v[k * 8 + 2 * q] = f.x;
            v[k * 8 + 2 * q + 1] = f.y;
        }
    }
}

// LayerNorm backward, one warp per row (d = 256 * VPL). dy = gradient w.r.t. the LN output,
// x = LN input (fp32 residual stream), w = LN weight. dh (fp32) += dx, and dh_bf16 gets a
// bf16 copy of the updated dh (the next GEMM operand). Per-block partial rows of
// dw = sum dy * xhat and db = sum dy go to part[blockIdx.x] ([2][d]); with CS also the
// column sums of the updated dh ([3][d] rows): the bias gradient of the projection whose
// output dh is (no separate pass over dh).
template <int VPL, bool CS>
__global__ void __launch_bounds__(256) ln_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ w, float* __restrict__ dh,
                                                     __nv_bfloat16* __restrict__ dh_bf16, float* __restrict__ part,
                                                     int rows) {
    constexpr int d = VPL * 256;
    __shared__ float red[8][2][d];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float wv[VPL * 8];
    tr_load_w<VPL>(w, lane, wv);
    float dwp[VPL * 8], dbp[VPL * 8], dhp[CS ? VPL * 8 : 1];
#pragma unroll
    for (int e = 0; e < VPL * 8; ++e) dwp[e] = dbp[e] = 0.f;
#pragma unroll
    for (int e = 0; e < (CS ? VPL * 8 : 1); ++e) dhp[e] = 0.f;
    const int r0 = blockIdx.x * LNB_ROWS_PER_BLOCK;
    for (int r = r0 + wid; r < min(rows, r0 + LNB_ROWS_PER_BLOCK); r += 8) {
        float xv[VPL * 8], g[VPL * 8];
        float hv[VPL * 8];
        tr_load_f32<VPL>(x + (size_t)r * d, lane, xv);
        tr_load_f32<VPL>(dy + (size_t)r * d, lane, g);
        tr_load_f32<VPL>(dh + (size_t)r * d, lane, hv);  // all three rows in flight at once
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < VPL * 8; ++e) s += xv[e];
        const float mean = warp_sum(s) * (1.0f / d);
        float s2 = 0.f;
#pragma unroll
        for (int e = 0; e < VPL * 8; ++e) {
            const float t = xv[e] - mean;
            s2 += t * t;
        }
        const float rstd = rsqrtf(warp_sum(s2) * (1.0f / d) + TR_LN_EPS);
        float sg = 0.f, sgx = 0.f;
#pragma unroll
        for (int e = 0; e < VPL * 8; ++e) {
            const float xh = (xv[e] - mean) * rstd;
            dwp[e] += g[e] * xh;
            dbp[e] += g[e];
            const float gw = g[e] * wv[e];
            xv[e] = xh;  // reuse as xhat
            g[e] = gw;
            sg += gw;
            sgx += gw * xh;
        }
        sg = warp_sum(sg) * (1.0f / d);
        sgx = warp_sum(sgx) * (1.0f / d);
#pragma unroll
        for (int e = 0; e < VPL * 8; ++e) {
            hv[e] += rstd * (g[e] - sg - xv[e] * sgx);
            if constexpr (CS) dhp[e] += hv[e];
        }
        tr_store_f32<VPL>(dh + (size_t)r * d, lane, hv);
        tr_store_bf16<VPL>(dh_bf16 + (size_t)r * d, lane, hv);
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            red[wid][0][(lane + 32 * k) * 8 + e] = dwp[k * 8 + e];
            red[wid][1][(lane + 32 * k) * 8 + e] = dbp[k * 8 + e];
        }
    __syncthreads();
    constexpr int ld = (CS ? 3 : 2) * d;
    for (int cidx = threadIdx.x; cidx < 2 * d; cidx += blockDim.x) {
        const int which = cidx / d, col = cidx % d;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += red[k][which][col];
        part[(size_t)blockIdx.x * ld + cidx] = acc;
    }
    if constexpr (CS) {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VPL; ++k)
#pragma unroll
            for (int e = 0; e < 8; ++e) red[wid][0][(lane + 32 * k) * 8 + e] = dhp[k * 8 + e];
        __syncthreads();
        for (int col = threadIdx.x; col < d; col += blockDim.x) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += red[k][0][col];
            part[(size_t)blockIdx.x * ld + 2 * d + col] = acc;
        }
    }
}

// Column sums of a [rows, cols] matrix (float or bf16) into per-block partial rows.
template <typename T>
__global__ void colsum_partial_kernel(const T* __restrict__ x, int rows, int cols, float* __restrict__ part) {
    // VEC adjacent columns per thread through one 16-byte load per row (cols % VEC == 0);
    // rows summed in order, so the result is the same as one column per thread
    constexpr int VEC = 16 / sizeof(T);
    const int c = (blockIdx.y * blockDim.x + threadIdx.x) * VEC;
    if (c >= cols) return;
    const int r0 = blockIdx.x * TR_ROWS_PER_BLOCK;
    const int r1 = min(rows, r0 + TR_ROWS_PER_BLOCK);
    float acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(x + (size_t)r * cols + c));
        const T* vals = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[k] += (float)vals[k];
    }
#pragma unroll
    for (int k = 0; k < VEC; ++k) part[(size_t)blockIdx.x * cols + c + k] = acc[k];
}

// out[c] += sum over n_part partial rows (fixed order).
__global__ void reduce_rows_add_kernel(const float* __restrict__ part, int n_part, int cols, float* __restrict__ out,
                                       int ld) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    float acc = 0.f;
#pragma unroll 32
    for (int p = 0; p < n_part; ++p) acc += part[(size_t)p * ld + c];  // (32 loads in flight, same order)
    out[c] += acc;
}

// First level of a two-level column reduction: scratch[g][c] = sum of partial rows
// [RR_GROUP g, RR_GROUP (g + 1)) (fixed order), so no thread walks thousands of dependent
// rows and even a few hundred partial rows spread over many blocks.
constexpr int RR_GROUP = 16;
__global__ void reduce_rows_group_kernel(const float* __restrict__ part, int n_part, int cols,
                                         float* __restrict__ scratch, int ld) {
    const int c = blockIdx.y * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    const int p0 = blockIdx.x * RR_GROUP, p1 = min(n_part, p0 + RR_GROUP);
    float acc = 0.f;
#pragma unroll 8
    for (int p = p0; p < p1; ++p) acc += part[(size_t)p * ld + c];
    scratch[(size_t)blockIdx.x * cols + c] = acc;
}

// out[c] += sum of the n_part partial rows of `part` (row stride ld >= cols; deterministic;
// scratch holds ceil(n_part / RR_GROUP) rows of cols and must not overlap part).
static int reduce_rows_add(const float* part, int n_part, int cols, float* out, float* scratch, cudaStream_t st,
                           int ld = 0) {
    if (ld == 0) ld = cols;
    if (n_part <= 2 * RR_GROUP) {
        reduce_rows_add_kernel<<<(cols + 255) / 256, 256, 0, st>>>(part, n_part, cols, out, ld);
        RS_LAUNCH_CHECK();
        return RS_OK;
    }
    const int g = (n_part + RR_GROUP - 1) / RR_GROUP;
    reduce_rows_group_kernel<<<dim3(g, (cols + 255) / 256), 256, 0, st>>>(part, n_part, cols, scratch, ld);
    RS_LAUNCH_CHECK();
    reduce_rows_add_kernel<<<(cols + 255) / 256, 256, 0, st>>>(scratch, g, cols, out, cols);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

// out[i] += sum over k of part[k * n + i] (split-K partial slices, fixed order).
__global__ void reduce_slices_add_kernel(const float* __restrict__ part, int k, int64_t n, float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int s = 0; s < k; ++s) acc += part[(size_t)s * n + i];
        out[i] += acc;
    }
}

// Embedding backward over tokens sorted by id (order[] = token index, keys[] = id):
// the warp at the start of each run of equal ids sums the run's rows in order and adds
// the total to dE[id] -- each dE row is written by exactly one warp.
// DPL = d / 32 columns per lane, held in registers: the run's rows are walked once (each
// row's DPL loads independent, the run's row indices fetched 32 at a time), same order of
// additions per column as the generic kernel below.
template <int DPL>
__global__ void embed_bwd_tok_regs_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ order, int n,
                                          const float* __restrict__ dh, float* __restrict__ dE) {
    constexpr int d = DPL * 32;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const uint32_t id = keys[i];
    if (i > 0 && keys[i - 1] == id) return;
    float acc[DPL];
#pragma unroll
    for (int k = 0; k < DPL; ++k) acc[k] = 0.f;
    for (int j0 = i; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        const bool in = j < n && keys[j] == id;
        const unsigned run = __ballot_sync(0xffffffffu, in);
        const int len = __popc(run) == 32 ? 32 : __ffs(~run) - 1;  // the run continues only while contiguous
        const uint32_t row = in ? order[j] : 0u;
        for (int r = 0; r < len; ++r) {
            const float* src = dh + (size_t)__shfl_sync(0xffffffffu, row, r) * d + lane;
#pragma unroll
            for (int k = 0; k < DPL; ++k) acc[k] += src[32 * k];
        }
        if (len < 32) break;
    }
    float* dst = dE + (size_t)id * d + lane;
#pragma unroll
    for (int k = 0; k < DPL; ++k) dst[32 * k] += acc[k];
}
__global__ void embed_bwd_tok_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ order, int n,
                                     const float* __restrict__ dh, int d, float* __restrict__ dE) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const uint32_t id = keys[i];
    if (i > 0 && keys[i - 1] == id) return;
    for (int c = lane; c < d; c += 32) {
        float acc = 0.f;
        for (int j = i; j < n && keys[j] == id; ++j) acc += dh[(size_t)order[j] * d + c];
        dE[(size_t)id * d + c] += acc;
    }
}
// Position-embedding backward: dP[p + 2] += sum over prompts of dh[b * S + p] (fixed order:
// EBP_G interleaved partial sums per column, then added in group order). Block (32 columns,
// EBP_G prompt groups) per (position, 32-column slice): S x d / 32 blocks instead of S, so
// the pass streams dh at HBM speed (one block per position had left it latency-bound).
constexpr int EBP_G = 8;
__global__ void __launch_bounds__(32 * EBP_G) embed_bwd_pos_kernel(const float* __restrict__ dh, int B, int S, int d,
                                                                   float* __restrict__ dP) {
    __shared__ float part[EBP_G][33];
    const int p = blockIdx.x, c = blockIdx.y * 32 + threadIdx.x, g = threadIdx.y;
    float acc = 0.f;
    if (c < d)
        for (int b = g; b < B; b += EBP_G) acc += dh[((size_t)b * S + p) * d + c];
    part[g][threadIdx.x] = acc;
    __syncthreads();
    if (g == 0 && c < d) {
        float s = part[0][threadIdx.x];
#pragma unroll
        for (int k = 1; k < EBP_G; ++k) s += part[k][threadIdx.x];
        dP[(size_t)(p + 2) * d + c] += s;
    }
}
__global__ void ids_to_keys_kernel(const int32_t* __restrict__ ids, int n, int vocab, uint32_t* __restrict__ keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        int id = ids[i];
        keys[i] = (uint32_t)(id < 0 ? 0 : (id >= vocab ? vocab - 1 : id));
    }
}

// Score-head backward, one warp per prompt: g = hw . LNf(h_last) + hb.
// dh[last row] = LNf_bwd(dg * hw); per-prompt partial rows of (d hw, d lnf_w, d lnf_b)
// and the scalar d hb go to part[p] ([3 * d + 1]).
template <int VPL>
__global__ void head_bwd_kernel(const float* __restrict__ h, const int32_t* __restrict__ last, int B, int S,
                                const __nv_bfloat16* __restrict__ lw, const __nv_bfloat16* __restrict__ lb,
                                const __nv_bfloat16* __restrict__ hw, const float* __restrict__ dg,
                                float* __restrict__ dh, float* __restrict__ part,
                                const float* __restrict__ dfeat) {
    constexpr int d = VPL * 256;
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (p >= B) return;
    int lp = last ? last[p] : S - 1;
    lp = lp < 0 ? 0 : (lp >= S ? S - 1 : lp);
    const size_t row = (size_t)p * S + lp;
    float xv[VPL * 8], lwv[VPL * 8], lbv[VPL * 8], hwv[VPL * 8];
    tr_load_f32<VPL>(h + row * d, lane, xv);
    tr_load_w<VPL>(lw, lane, lwv);
    tr_load_w<VPL>(lb, lane, lbv);
    tr_load_w<VPL>(hw, lane, hwv);
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < VPL * 8; ++e) s += xv[e];
    const float mean = warp_sum(s) * (1.0f / d);
    float s2 = 0.f;
#pragma unroll
    for (int e = 0; e < VPL * 8; ++e) {
        const float t = xv[e] - mean;
        s2 += t * t;
    }
    const float rstd = rsqrtf(warp_sum(s2) * (1.0f / d) + TR_LN_EPS);
    // dfeat given (the classifier head): it is d loss / d LNf(h) itself and the score
    // head takes no gradient; else dxf = dg * hw
    const float gq = dfeat ? 0.f : dg[p];
    const float* dfr = dfeat ? dfeat + (size_t)p * d : nullptr;
    float* pr = part + (size_t)p * (3 * d + 1);
    float sg = 0.f, sgx = 0.f, gv[VPL * 8];
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int i = k * 8 + e, col = (lane + 32 * k) * 8 + e;
            const float xh = (xv[i] - mean) * rstd;
            const float xf = xh * lwv[i] + lbv[i];
            const float dxf = dfr ? dfr[col] : gq * hwv[i];  // d g / d xf = hw
            pr[col] = gq * xf;              // d hw
            pr[d + col] = dxf * xh;         // d lnf_w
            pr[2 * d + col] = dxf;          // d lnf_b
            const float gw = dxf * lwv[i];
            gv[i] = gw;
            xv[i] = xh;
            sg += gw;
            sgx += gw * xh;
        }
    sg = warp_sum(sg) * (1.0f / d);
    sgx = warp_sum(sgx) * (1.0f / d);
    float o[VPL * 8];
#pragma unroll
    for (int e = 0; e < VPL * 8; ++e) o[e] = rstd * (gv[e] - sg - xv[e] * sgx);
    tr_store_f32<VPL>(dh + row * d, lane, o);
    if (lane == 0) pr[3 * d] = gq;
}

// Fused Adam (predictors.py:218-225) over the flat parameter buffer: grad scaled by
// grad_scale, fp32 master weights / moments, bf16 working copy; zeroes grad for the
// next accumulation.
__global__ void adam_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                            float* __restrict__ grad, __nv_bfloat16* __restrict__ pb, int64_t n, float lr, float b1,
                            float b2, float eps, float bc1, float bc2, float grad_scale) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float g = grad[i] * grad_scale;
        const float mi = b1 * m[i] + (1.f - b1) * g;
        const float vi = b2 * v[i] + (1.f - b2) * g * g;
        m[i] = mi;
        v[i] = vi;
        const float mhat = mi / bc1, vhat = vi / bc2;
        const float p = master[i] - lr * mhat / (sqrtf(vhat) + eps);
        master[i] = p;
        pb[i] = __float2bfloat16_rn(p);
        grad[i] = 0.f;
    }
}

// ---- host launchers -------------------------------------------------------------------

int ln_backward(const float* dy, const float* x, const void* w, float* dh, void* dh_bf16, float* part, int rows,
                int d, float* dw_out, float* db_out, cudaStream_t st, float* dhsum_out) {
    const int nblk = (rows + LNB_ROWS_PER_BLOCK - 1) / LNB_ROWS_PER_BLOCK;
    const __nv_bfloat16* wb = static_cast<const __nv_bfloat16*>(w);
    __nv_bfloat16* hb = static_cast<__nv_bfloat16*>(dh_bf16);
    const bool cs = dhsum_out != nullptr;
#define RS_LNB(V)                                                                          \
    if (cs) ln_bwd_kernel<V, true><<<nblk, 256, 0, st>>>(dy, x, wb, dh, hb, part, rows); \
    else ln_bwd_kernel<V, false><<<nblk, 256, 0, st>>>(dy, x, wb, dh, hb, part, rows);
    switch (d / 256) {
        case 1: RS_LNB(1) break;
        case 2: RS_LNB(2) break;
        case 3: RS_LNB(3) break;
        default: set_error("ln_backward: unsupported d=%d", d); return RS_ERR_INVALID;
    }
#undef RS_LNB
    RS_LAUNCH_CHECK();
    // part rows are [dw | db (| dh column sums)]: dw and db reduce in one pass into a
    // contiguous [dw_out, db_out] pair (the callers' LN weight and bias are adjacent)
    (void)db_out;
    const int ld = (cs ? 3 : 2) * d;
    float* scratch = part + (size_t)nblk * ld;
    RS_TRY(reduce_rows_add(part, nblk, 2 * d, dw_out, scratch, st, ld));
    if (cs) RS_TRY(reduce_rows_add(part + 2 * d, nblk, d, dhsum_out, scratch, st, ld));
    return RS_OK;
}

int rows_add(const float* part, int n_part, int cols, float* out, float* scratch, cudaStream_t st) {
    return reduce_rows_add(part, n_part, cols, out, scratch, st);
}

int colsum_add(const void* x, bool is_bf16, int rows, int cols, float* part, float* out, cudaStream_t st) {
    const int nblk = (rows + TR_ROWS_PER_BLOCK - 1) / TR_ROWS_PER_BLOCK;
    RS_CHECK_ARG(cols % 8 == 0, "colsum_add: cols %% 8 != 0");
    const int vec = is_bf16 ? 8 : 4;
    dim3 grid(nblk, (cols / vec + 255) / 256);
    if (is_bf16)
        colsum_partial_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), rows, cols,
                                                                     part);
    else
        colsum_partial_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), rows, cols, part);
    RS_LAUNCH_CHECK();
    return reduce_rows_add(part, nblk, cols, out, part + (size_t)nblk * cols, st);
}

int slices_add(const float* part, int k, int64_t n, float* out, cudaStream_t st) {
    reduce_slices_add_kernel<<<1184, 256, 0, st>>>(part, k, n, out);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

size_t embed_backward_ws(int n) {
    ArenaSizer s;
    const uint32_t np = ms_padded(n);
    s.take<uint32_t>(n);
    s.take<uint32_t>(np);
    s.take<uint32_t>(np);
    s.take<uint32_t>(np);
    s.take<uint32_t>(np);
    s.take<int>(ms_splits(np));
    return s.used + 256;
}

int embed_backward(const int32_t* ids, int B, int S, int vocab, const float* dh, int d, float* dE, float* dP, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
    const int n = B * S;
    if (ws_bytes < embed_backward_ws(n)) {
        set_error("embed_backward: workspace too small");
        return RS_ERR_WORKSPACE;
    }
    Arena ar(ws, ws_bytes);
    const uint32_t np = ms_padded(n);
    uint32_t* keys = ar.take<uint32_t>(n);
    uint32_t* k0 = ar.take<uint32_t>(np);
    uint32_t* k1 = ar.take<uint32_t>(np);
    uint32_t* v0 = ar.take<uint32_t>(np);
    uint32_t* v1 = ar.take<uint32_t>(np);
    int* splits = ar.take<int>(ms_splits(np));
    ids_to_keys_kernel<<<(n + 255) / 256, 256, 0, st>>>(ids, n, vocab, keys);
    RS_LAUNCH_CHECK();
    uint32_t *sk, *sv;
    RS_TRY((merge_sort<uint32_t, true, false>(keys, nullptr, n, k0, k1, v0, v1, nullptr, st, &sk, &sv, splits)));
    switch (d) {
        case 256: embed_bwd_tok_regs_kernel<8><<<(n + 7) / 8, 256, 0, st>>>(sk, sv, n, dh, dE); break;
        case 512: embed_bwd_tok_regs_kernel<16><<<(n + 7) / 8, 256, 0, st>>>(sk, sv, n, dh, dE); break;
        case 768: embed_bwd_tok_regs_kernel<24><<<(n + 7) / 8, 256, 0, st>>>(sk, sv, n, dh, dE); break;
        default: embed_bwd_tok_kernel<<<(n + 7) / 8, 256, 0, st>>>(sk, sv, n, dh, d, dE); break;
    }
    RS_LAUNCH_CHECK();
    embed_bwd_pos_kernel<<<dim3(S, (d + 31) / 32), dim3(32, EBP_G), 0, st>>>(dh, B, S, d, dP);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

int head_backward(const float* h, const int32_t* last, int B, int S, const void* lw, const void* lb, const void* hw,
                  const float* dg, float* dh, float* part, int d, float* g_hw, float* g_lnf, float* g_hb,
                  cudaStream_t st, const float* dfeat) {
    const int wpb = 8;
    const int grid = (B + wpb - 1) / wpb;
    const __nv_bfloat16 *a = static_cast<const __nv_bfloat16*>(lw), *b = static_cast<const __nv_bfloat16*>(lb),
                        *c = static_cast<const __nv_bfloat16*>(hw);
    switch (d / 256) {
        case 1: head_bwd_kernel<1><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, a, b, c, dg, dh, part, dfeat); break;
        case 2: head_bwd_kernel<2><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, a, b, c, dg, dh, part, dfeat); break;
        case 3: head_bwd_kernel<3><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, a, b, c, dg, dh, part, dfeat); break;
        default: set_error("head_backward: unsupported d=%d", d); return RS_ERR_INVALID;
    }
    RS_LAUNCH_CHECK();
    // part: B rows of [d hw (d) | d lnf_w (d) | d lnf_b (d) | d hb (1)]
    const int cols = 3 * d + 1;
    float* tot = part + (size_t)B * cols;
    RS_CUDA(cudaMemsetAsync(tot, 0, cols * sizeof(float), st));
    RS_TRY(reduce_rows_add(part, B, cols, tot, tot + cols, st));
    // scatter: d hw -> g_hw, (d lnf_w, d lnf_b) -> g_lnf (adjacent), d hb -> g_hb
    if (g_hw) {
        reduce_rows_add_kernel<<<(d + 255) / 256, 256, 0, st>>>(tot, 1, d, g_hw, d);
        RS_LAUNCH_CHECK();
    }
    reduce_rows_add_kernel<<<(2 * d + 255) / 256, 256, 0, st>>>(tot + d, 1, 2 * d, g_lnf, 2 * d);
    RS_LAUNCH_CHECK();
    if (g_hb) {
        reduce_rows_add_kernel<<<1, 32, 0, st>>>(tot + 3 * d, 1, 1, g_hb, 1);
        RS_LAUNCH_CHECK();
    }
    return RS_OK;
}

}  // namespace rs

extern "C" int rs_adam_step(float* master, float* m, float* v, float* grad, void* params_bf16, int64_t n, float lr,
                            float beta1, float beta2, float eps, int64_t t, float grad_scale, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(n >= 0 && t >= 1, "rs_adam_step: need n >= 0 and t >= 1");
    if (n == 0) return RS_OK;
    const float bc1 = 1.f - powf(beta1, (float)t), bc2 = 1.f - powf(beta2, (float)t);
    rs::adam_kernel<<<148 * 8, 256, 0, rs::as_stream(stream)>>>(master, m, v, grad,
                                                                  static_cast<__nv_bfloat16*>(params_bf16), n, lr,
                                                                  beta1, beta2, eps, bc1, bc2, grad_scale);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
