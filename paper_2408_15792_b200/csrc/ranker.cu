// A5 / K1, K2, K5 + orchestration: the OPT-125M-shape ranker forward.
//
// Replaces RankingModelScorer.raw_outputs (predictors.py:245-247: standardise
// features, _Net.forward) with the paper's predictor: an OPT
// decoder over the prompt tokens whose last-token hidden state goes through a
// Linear(d, 1) score head. Per layer (pre-LN, OPT-125M: do_layer_norm_before):
//   x = LN1(h); qkv = x Wqkv^T + b; a = causal_attn(qkv); h = h + a Wo^T + bo
//   x = LN2(h); f = relu(x W1^T + b1);                   h = h + f W2^T + b2
// then g = w . LNf(h[last]) + b. Embedding h0 = E[ids] + P[pos + 2] (OPT's learned
// positions carry an offset of 2).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdlib.h>
#include "common.cuh"
#include "gemm.cuh"

namespace rs {
int attention_fwd(const void* qkv, void* out, int B, int S, int H, cudaStream_t st);
int attention_fwd_f16v(const void* qkv, void* out, int B, int S, int H, cudaStream_t st);

constexpr float LN_EPS = 1e-5f;

// One warp per token row: h = tok[id] + pos[p + 2]. The residual stream h is fp32.
__global__ void embed_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ tok,
                             const __nv_bfloat16* __restrict__ pos, float* __restrict__ h, int n_tok, int S,
                             int d, int vocab, int n_rows_padded) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n_rows_padded) return;
    float4* dst = reinterpret_cast<float4*>(h + (size_t)row * d);
    const int nv = d / 8;
    if (row >= n_tok) {
        for (int k = lane; k < 2 * nv; k += 32) dst[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    int id = ids[row];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const int p = row % S + 2;
    const uint4* a = reinterpret_cast<const uint4*>(tok + (size_t)id * d);
    const uint4* b = reinterpret_cast<const uint4*>(pos + (size_t)p * d);
    for (int k = lane; k < nv; k += 32) {
        uint4 x = a[k], y = b[k];
        const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&x);
        const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&y);
        float o[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 xf = __bfloat1622float2(x2[q]), yf = __bfloat1622float2(y2[q]);
            o[2 * q] = xf.x + yf.x;
            o[2 * q + 1] = xf.y + yf.y;
        }
        dst[2 * k] = make_float4(o[0], o[1], o[2], o[3]);
        dst[2 * k + 1] = make_float4(o[4], o[5], o[6], o[7]);
    }
}

template <int VPL>
__device__ __forceinline__ void row_stats(const float (&v)[VPL * 8], float& mean, float& rstd);

// Embedding fused with layer 0's first LayerNorm: one warp per token row writes the fp32
// residual row h = tok[id] + pos[p + 2] and x = LN1(h) (bf16, the QKV GEMM's A operand).
template <int VPL>
__global__ void embed_ln_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ tok,
                                const __nv_bfloat16* __restrict__ pos, const __nv_bfloat16* __restrict__ lw,
                                const __nv_bfloat16* __restrict__ lb, float* __restrict__ h,
                                __nv_bfloat16* __restrict__ x, int n_tok, int S, int vocab, int n_rows_padded) {
    constexpr int d = VPL * 256;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n_rows_padded) return;
    float4* dst = reinterpret_cast<float4*>(h + (size_t)row * d);
    uint4* xr = reinterpret_cast<uint4*>(x + (size_t)row * d);
    if (row >= n_tok) {
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            dst[2 * (lane + 32 * k)] = make_float4(0.f, 0.f, 0.f, 0.f);
            dst[2 * (lane + 32 * k) + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
            xr[lane + 32 * k] = make_uint4(0u, 0u, 0u, 0u);
        }
        return;
    }
    int id = ids[row];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const int p = row % S + 2;
    const uint4* a = reinterpret_cast<const uint4*>(tok + (size_t)id * d);
    const uint4* b = reinterpret_cast<const uint4*>(pos + (size_t)p * d);
    float v[VPL * 8];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        uint4 xa = a[lane + 32 * k], yb = b[lane + 32 * k];
        const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xa);
        const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&yb);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 xf = __bfloat1622float2(x2[q]), yf = __bfloat1622float2(y2[q]);
            v[k * 8 + 2 * q] = xf.x + yf.x;
            v[k * 8 + 2 * q + 1] = xf.y + yf.y;
        }
        dst[2 * (lane + 32 * k)] = make_float4(v[k * 8 + 0], v[k * 8 + 1], v[k * 8 + 2], v[k * 8 + 3]);
        dst[2 * (lane + 32 * k) + 1] = make_float4(v[k * 8 + 4], v[k * 8 + 5], v[k * 8 + 6], v[k * 8 + 7]);
    }
    float mean, rstd;
    row_stats<VPL>(v, mean, rstd);
    const uint4* wr = reinterpret_cast<const uint4*>(lw);
    const uint4* br = reinterpret_cast<const uint4*>(lb);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        uint4 wu = wr[lane + 32 * k], bu = br[lane + 32 * k], o;
        const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wu);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bu);
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 wf = __bfloat1622float2(w2[q]), bf = __bfloat1622float2(b2[q]);
            o2[q] = __floats2bfloat162_rn((v[k * 8 + 2 * q] - mean) * rstd * wf.x + bf.x,
                                          (v[k * 8 + 2 * q + 1] - mean) * rstd * wf.y + bf.y);
        }
        xr[lane + 32 * k] = o;
    }
}

template <int VPL>
__device__ __forceinline__ void load_row_f32(const float* __restrict__ x, int lane, float (&v)[VPL * 8]) {
    const float4* xr = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        float4 a = xr[2 * (lane + 32 * k)], b = xr[2 * (lane + 32 * k) + 1];
        v[k * 8 + 0] = a.x; v[k * 8 + 1] = a.y; v[k * 8 + 2] = a.z; v[k * 8 + 3] = a.w;
        v[k * 8 + 4] = b.x; v[k * 8 + 5] = b.y; v[k * 8 + 6] = b.z; v[k * 8 + 7] = b.w;
    }
}
// Two-pass mean / biased variance over a warp-distributed row (eps 1e-5, OPT).
template <int VPL>
__device__ __forceinline__ void row_stats(const float (&v)[VPL * 8], float& mean, float& rstd) {
    constexpr int d = VPL * 256;
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < VPL * 8; ++e) s += v[e];
    mean = warp_sum(s) * (1.0f / d);
    float s2 = 0.f;
#pragma unroll
    for (int e = 0; e < VPL * 8; ++e) {
        const float t = v[e] - mean;
        s2 += t * t;
    }
    rstd = rsqrtf(warp_sum(s2) * (1.0f / d) + LN_EPS);
}

// LayerNorm over fp32 rows of d (d % 256 == 0, d <= 2048) -> bf16: one warp per row.
template <int VPL>  // uint4 (8 bf16) vectors per lane = d / 256
__global__ void layernorm_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                                 const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y, int rows) {
    constexpr int d = VPL * 256;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float v[VPL * 8];
    load_row_f32<VPL>(x + (size_t)row * d, lane, v);
    float mean, rstd;
    row_stats<VPL>(v, mean, rstd);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    const uint4* br = reinterpret_cast<const uint4*>(b);
    uint4* yr = reinterpret_cast<uint4*>(y + (size_t)row * d);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        uint4 wu = wr[lane + 32 * k], bu = br[lane + 32 * k], o;
        const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&wu);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bu);
        __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float2 wf = __bfloat1622float2(w2[q]), bf = __bfloat1622float2(b2[q]);
            o2[q] = __floats2bfloat162_rn((v[k * 8 + 2 * q] - mean) * rstd * wf.x + bf.x,
                                          (v[k * 8 + 2 * q + 1] - mean) * rstd * wf.y + bf.y);
        }
        yr[lane + 32 * k] = o;
    }
}

// K5: g[b] = head_w . LNf(h[b*S + last[b]]) + head_b, one warp per prompt, fp32 out.
template <int VPL>
__global__ void head_kernel(const float* __restrict__ h, const int32_t* __restrict__ last, int B, int S,
                            const __nv_bfloat16* __restrict__ lw, const __nv_bfloat16* __restrict__ lb,
                            const __nv_bfloat16* __restrict__ hw, const __nv_bfloat16* __restrict__ hb,
                            float* __restrict__ g, float* __restrict__ score, float* __restrict__ feat) {
    constexpr int d = VPL * 256;
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (p >= B) return;
    int lp = last ? last[p] : S - 1;
    lp = lp < 0 ? 0 : (lp >= S ? S - 1 : lp);
    float v[VPL * 8];
    load_row_f32<VPL>(h + ((size_t)p * S + lp) * d, lane, v);
    float mean, rstd;
    row_stats<VPL>(v, mean, rstd);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        const int base = (lane + 32 * k) * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float xn = (v[k * 8 + e] - mean) * rstd * __bfloat162float(lw[base + e]) + __bfloat162float(lb[base + e]);
            acc = fmaf(xn, __bfloat162float(hw[base + e]), acc);
            if (feat) feat[(size_t)p * d + base + e] = xn;  // LNf(h_last): the classifier head's input
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        const float gv = acc + __bfloat162float(hb[0]);
        g[p] = gv;
        if (score) score[p] = -gv;  // RankingModelScorer.score_batch negation (predictors.py:249-250)
    }
}

// Last layer, pruned to the one query that reaches the score head: for every prompt b
// and head, o = softmax(q_last k_j^T / 8, j <= last) v over the prompt's keys, with
// q_last the query of token last[b] (causal attention restricted to that row is exact).
// One warp per (prompt, head); scores staged in shared memory. The warp also gathers
// its 64-column slice of the residual row h[b*S + last] into h_last[b] (fp32), so the
// rest of the last layer (out-proj, LN2, FFN) and the head run on B rows instead of B*S.
constexpr int AL_WARPS = 4;
__global__ void __launch_bounds__(32 * AL_WARPS)
    attention_last_kernel(const __nv_bfloat16* __restrict__ qkv, const float* __restrict__ h,
                          const int32_t* __restrict__ last, __nv_bfloat16* __restrict__ att_last,
                          float* __restrict__ h_last, int B, int Bp, int S, int H) {
    extern __shared__ float al_s[];  // [AL_WARPS][S]
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * AL_WARPS + wib;
    if (gw >= Bp * H) return;
    const int b = gw / H, hh = gw % H;
    const int d = H * 64;
    __nv_bfloat162* orow = reinterpret_cast<__nv_bfloat162*>(att_last + (size_t)b * d + hh * 64) + lane;
    float2* hrow = reinterpret_cast<float2*>(h_last + (size_t)b * d + hh * 64) + lane;
    if (b >= B) {  // padding rows of the pruned GEMMs
        *orow = __floats2bfloat162_rn(0.f, 0.f);
        *hrow = make_float2(0.f, 0.f);
        return;
    }
    int lp = last ? last[b] : S - 1;
    lp = lp < 0 ? 0 : (lp >= S ? S - 1 : lp);
    const size_t ld = (size_t)3 * d;
    const __nv_bfloat16* base = qkv + (size_t)b * S * ld + hh * 64;
    *hrow = reinterpret_cast<const float2*>(h + ((size_t)b * S + lp) * d + hh * 64)[lane];
    float q[64];
    {
        const uint4* q4 = reinterpret_cast<const uint4*>(base + (size_t)lp * ld);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint4 u = q4[k];
            const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(u2[e]);
                q[k * 8 + 2 * e] = f.x * 0.125f;  // 1/sqrt(64)
                q[k * 8 + 2 * e + 1] = f.y * 0.125f;
            }
        }
    }
    float* sc = al_s + wib * S;
    float m = -INFINITY;
    for (int j = lane; j <= lp; j += 32) {
        const uint4* k4 = reinterpret_cast<const uint4*>(base + (size_t)j * ld + d);
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint4 u = k4[k];
            const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(u2[e]);
                acc = fmaf(q[k * 8 + 2 * e], f.x, acc);
                acc = fmaf(q[k * 8 + 2 * e + 1], f.y, acc);
            }
        }
        sc[j] = acc;
        m = fmaxf(m, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int j = lane; j <= lp; j += 32) {
        const float p = __expf(sc[j] - m);
        sc[j] = p;
        l += p;
    }
    l = warp_sum(l);
    __syncwarp();
    float2 o = make_float2(0.f, 0.f);
    // V is fp16 in the forward's q|k|v activation (QKV GEMM epilogue 7)
    const __half2* vcol = reinterpret_cast<const __half2*>(base + 2 * d) + lane;
    for (int j = 0; j <= lp; ++j) {
        const float2 v = __half22float2(vcol[(size_t)j * (ld / 2)]);
        const float p = sc[j];
        o.x = fmaf(p, v.x, o.x);
        o.y = fmaf(p, v.y, o.y);
    }
    const float inv = 1.f / l;
    *orow = __floats2bfloat162_rn(o.x * inv, o.y * inv);
}

static int launch_attention_last(const __nv_bfloat16* qkv, const float* h, const int32_t* last,
                                 __nv_bfloat16* att_last, float* h_last, int B, int Bp, int S, int H,
                                 cudaStream_t st) {
    const size_t smem = (size_t)AL_WARPS * S * sizeof(float);
    if (smem > 48 * 1024) RS_CUDA(ensure_smem((const void*)attention_last_kernel, (int)smem));
    const int warps = Bp * H;
    attention_last_kernel<<<(warps + AL_WARPS - 1) / AL_WARPS, 32 * AL_WARPS, smem, st>>>(qkv, h, last, att_last,
                                                                                       h_last, B, Bp, S, H);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

struct RankerOffsets {
    int64_t tok, pos, lnf_w, lnf_b, head_w, head_b;
    int64_t per_layer0, layer_stride;
    int64_t ln1_w, ln1_b, qkv_w, qkv_b, out_w, out_b, ln2_w, ln2_b, fc1_w, fc1_b, fc2_w, fc2_b;  // within layer
    int64_t total;
};

static int64_t pad64(int64_t x) { return (x + 63) / 64 * 64; }

static RankerOffsets ranker_offsets(const rs_ranker_config& c) {
    RankerOffsets o{};
    const int64_t d = c.d_model, F = c.d_ffn;
    int64_t at = 0;
    auto take = [&](int64_t n) {
        int64_t r = at;
        at += pad64(n);
        return r;
    };
    o.tok = take((int64_t)c.vocab * d);
    o.pos = take((int64_t)(c.max_pos + 2) * d);
    o.per_layer0 = at;
    int64_t l0 = at;
    o.ln1_w = take(d) - l0;
    o.ln1_b = take(d) - l0;
    o.qkv_w = take(3 * d * d) - l0;
    o.qkv_b = take(3 * d) - l0;
    o.out_w = take(d * d) - l0;
    o.out_b = take(d) - l0;
    o.ln2_w = take(d) - l0;
    o.ln2_b = take(d) - l0;
    o.fc1_w = take(F * d) - l0;
    o.fc1_b = take(F) - l0;
    o.fc2_w = take(d * F) - l0;
    o.fc2_b = take(d) - l0;
    o.layer_stride = at - l0;
    at = l0 + o.layer_stride * c.n_layers;
    o.lnf_w = take(d);
    o.lnf_b = take(d);
    o.head_w = take(d);
    o.head_b = take(1);
    o.total = at;
    return o;
}

static int check_cfg(const rs_ranker_config* c) {
    RS_CHECK_ARG(c != nullptr, "ranker: config is NULL");
    RS_CHECK_ARG(c->vocab > 0 && c->max_pos > 0 && c->n_layers > 0 && c->n_heads > 0, "ranker: bad config");
    RS_CHECK_ARG(c->d_model == c->n_heads * 64, "ranker: head dim must be 64 (d_model = 64 * n_heads)");
    RS_CHECK_ARG(c->d_model % 256 == 0 && c->d_model <= 2048, "ranker: d_model must be a multiple of 256, <= 2048");
    RS_CHECK_ARG(c->d_ffn % 256 == 0, "ranker: d_ffn must be a multiple of 256");
    RS_CHECK_ARG(c->activation == 0 || c->activation == 1, "ranker: activation must be 0 (ReLU) or 1 (GELU)");
    return RS_OK;
}

constexpr int64_t RK_MAX_TOKENS = 1 << 20;  // activation chunk (tokens) per forward slice

static int64_t chunk_tokens() {
    static int64_t t = 0;
    if (!t) {
        const char* e = getenv("RSB200_CHUNK_TOKENS");
        t = e ? atoll(e) : RK_MAX_TOKENS;
        if (t < 256) t = RK_MAX_TOKENS;
    }
    return t;
}

static int64_t chunk_prompts(int32_t B, int32_t S) {
    int64_t bc = chunk_tokens() / S;
    if (bc < 1) bc = 1;
    if (bc > B) bc = B;
    return bc;
}

struct RankerWs {
    float* h;
    __nv_bfloat16 *x, *qkv, *att, *ffn;
    // last layer, pruned to one row per prompt (bp rows)
    float* h_last;
    __nv_bfloat16 *a_last, *x_last, *f_last;
};
template <typename A>
static void ranker_ws_layout(A& a, const rs_ranker_config& c, int64_t mp, int64_t bp, RankerWs* w) {
    RankerWs r;
    r.h = a.template take<float>(mp * c.d_model);
    r.x = a.template take<__nv_bfloat16>(mp * c.d_model);
    r.qkv = a.template take<__nv_bfloat16>(mp * 3 * c.d_model);
    r.att = a.template take<__nv_bfloat16>(mp * c.d_model);
    r.ffn = a.template take<__nv_bfloat16>(mp * c.d_ffn);
    r.h_last = a.template take<float>(bp * c.d_model);
    r.a_last = a.template take<__nv_bfloat16>(bp * c.d_model);
    r.x_last = a.template take<__nv_bfloat16>(bp * c.d_model);
    r.f_last = a.template take<__nv_bfloat16>(bp * c.d_ffn);
    if (w) *w = r;
}
struct RkSizer {
    ArenaSizer s;
    template <typename T>
    T* take(size_t n) { s.take<T>(n); return nullptr; }
};

static int launch_ln(const float* x, const __nv_bfloat16* w, const __nv_bfloat16* b, __nv_bfloat16* y,
                     int rows, int d, cudaStream_t st) {
    const int wpb = 8;
    const int grid = (rows + wpb - 1) / wpb;
    switch (d / 256) {
        case 1: layernorm_kernel<1><<<grid, 32 * wpb, 0, st>>>(x, w, b, y, rows); break;
        case 2: layernorm_kernel<2><<<grid, 32 * wpb, 0, st>>>(x, w, b, y, rows); break;
        case 3: layernorm_kernel<3><<<grid, 32 * wpb, 0, st>>>(x, w, b, y, rows); break;
        case 4: layernorm_kernel<4><<<grid, 32 * wpb, 0, st>>>(x, w, b, y, rows); break;
        case 8: layernorm_kernel<8><<<grid, 32 * wpb, 0, st>>>(x, w, b, y, rows); break;
        default: set_error("layernorm: unsupported d=%d", d); return RS_ERR_INVALID;
    }
    RS_LAUNCH_CHECK();
    return RS_OK;
}

static int launch_head(const float* h, const int32_t* last, int B, int S, const __nv_bfloat16* P,
                       const RankerOffsets& o, int d, float* g, float* score, cudaStream_t st, float* feat = nullptr) {
    const int wpb = 8;
    const int grid = (B + wpb - 1) / wpb;
    const __nv_bfloat16 *lw = P + o.lnf_w, *lb = P + o.lnf_b, *hw = P + o.head_w, *hb = P + o.head_b;
    switch (d / 256) {
        case 1: head_kernel<1><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, lw, lb, hw, hb, g, score, feat); break;
        case 2: head_kernel<2><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, lw, lb, hw, hb, g, score, feat); break;
        case 3: head_kernel<3><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, lw, lb, hw, hb, g, score, feat); break;
        case 4: head_kernel<4><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, lw, lb, hw, hb, g, score, feat); break;
        case 8: head_kernel<8><<<grid, 32 * wpb, 0, st>>>(h, last, B, S, lw, lb, hw, hb, g, score, feat); break;
        default: set_error("head: unsupported d=%d", d); return RS_ERR_INVALID;
    }
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" int64_t rs_ranker_layout(const rs_ranker_config* cfg, int64_t* off) {
    if (check_cfg(cfg) != RS_OK) return -1;
    RankerOffsets o = ranker_offsets(*cfg);
    if (off) {
        off[0] = o.tok;
        off[1] = o.pos;
        off[2] = o.lnf_w;
        off[3] = o.lnf_b;
        off[4] = o.head_w;
        off[5] = o.head_b;
        const int64_t per[RS_RANKER_N_PER_LAYER] = {o.ln1_w, o.ln1_b, o.qkv_w, o.qkv_b, o.out_w, o.out_b,
                                                    o.ln2_w, o.ln2_b, o.fc1_w, o.fc1_b, o.fc2_w, o.fc2_b};
        for (int l = 0; l < cfg->n_layers; ++l)
            for (int k = 0; k < RS_RANKER_N_PER_LAYER; ++k)
                off[RS_RANKER_N_GLOBAL + l * RS_RANKER_N_PER_LAYER + k] = o.per_layer0 + l * o.layer_stride + per[k];
    }
    return o.total;
}

extern "C" size_t rs_ranker_workspace_size(const rs_ranker_config* cfg, int32_t B, int32_t S) {
    if (check_cfg(cfg) != RS_OK || B <= 0 || S <= 0) return 0;
    const int64_t bc = chunk_prompts(B, S);
    const int64_t mp = (bc * S + 255) / 256 * 256;  // CTA-pair GEMM tiles are 256 rows
    const int64_t bp = (bc + 255) / 256 * 256;
    RkSizer s;
    ranker_ws_layout(s, *cfg, mp, bp, nullptr);
    return s.s.used + 256;
}

extern "C" int rs_ranker_forward(const rs_ranker_config* cfg, const void* params, const int32_t* ids,
                                 const int32_t* last_pos, int32_t B, int32_t S, float* g, float* score,
                                 void* ws, size_t ws_bytes, void* stream) {
    RS_NVTX();
    return rs_ranker_forward_ex(cfg, params, ids, last_pos, B, S, g, score, nullptr, ws, ws_bytes, stream);
}

extern "C" int rs_ranker_forward_ex(const rs_ranker_config* cfg, const void* params, const int32_t* ids,
                                    const int32_t* last_pos, int32_t B, int32_t S, float* g, float* score,
                                    float* feat, void* ws, size_t ws_bytes, void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_TRY(check_cfg(cfg));
    RS_CHECK_ARG(B > 0 && S > 0 && S <= cfg->max_pos, "ranker: need B > 0 and 0 < S <= max_pos");
    RS_CHECK_ARG(S <= 2048, "ranker: S <= 2048");
    RS_CHECK_ARG(params && ids && g, "ranker: NULL pointer");
    if (ws_bytes < rs_ranker_workspace_size(cfg, B, S)) {
        set_error("ranker: workspace %zu < %zu", ws_bytes, rs_ranker_workspace_size(cfg, B, S));
        return RS_ERR_WORKSPACE;
    }
    const RankerOffsets o = ranker_offsets(*cfg);
    const __nv_bfloat16* P = static_cast<const __nv_bfloat16*>(params);
    const int d = cfg->d_model, F = cfg->d_ffn, H = cfg->n_heads;
    const int64_t bc_max = chunk_prompts(B, S);
    for (int64_t b0 = 0; b0 < B; b0 += bc_max) {
        const int bc = (int)((B - b0) < bc_max ? (B - b0) : bc_max);
        const int n_tok = bc * S;
        const int mp = (n_tok + 255) / 256 * 256;
        const int bp = (bc + 255) / 256 * 256;
        Arena ar(ws, ws_bytes);
        RankerWs w;
        ranker_ws_layout(ar, *cfg, mp, bp, &w);
        const __nv_bfloat16* L0 = P + o.per_layer0;
        {
            const int wpb = 8;
            const int grid = (mp + wpb - 1) / wpb;
            switch (d / 256) {  // h0 = embeddings; x = LN1 of layer 0
                case 1: embed_ln_kernel<1><<<grid, 32 * wpb, 0, st>>>(ids + b0 * S, P + o.tok, P + o.pos, L0 + o.ln1_w,
                                                                      L0 + o.ln1_b, w.h, w.x, n_tok, S, cfg->vocab, mp); break;
                case 2: embed_ln_kernel<2><<<grid, 32 * wpb, 0, st>>>(ids + b0 * S, P + o.tok, P + o.pos, L0 + o.ln1_w,
                                                                      L0 + o.ln1_b, w.h, w.x, n_tok, S, cfg->vocab, mp); break;
                case 3: embed_ln_kernel<3><<<grid, 32 * wpb, 0, st>>>(ids + b0 * S, P + o.tok, P + o.pos, L0 + o.ln1_w,
                                                                      L0 + o.ln1_b, w.h, w.x, n_tok, S, cfg->vocab, mp); break;
                case 4: embed_ln_kernel<4><<<grid, 32 * wpb, 0, st>>>(ids + b0 * S, P + o.tok, P + o.pos, L0 + o.ln1_w,
                                                                      L0 + o.ln1_b, w.h, w.x, n_tok, S, cfg->vocab, mp); break;
                case 8: embed_ln_kernel<8><<<grid, 32 * wpb, 0, st>>>(ids + b0 * S, P + o.tok, P + o.pos, L0 + o.ln1_w,
                                                                      L0 + o.ln1_b, w.h, w.x, n_tok, S, cfg->vocab, mp); break;
                default: set_error("ranker: unsupported d=%d", d); return RS_ERR_INVALID;
            }
            RS_LAUNCH_CHECK();
        }
        // Rows past the last token are never written by attention but feed the
        // out-projection (and, as masked keys, the PV MMA: 0 * NaN = NaN), so zero them.
        if (mp > n_tok) RS_CUDA(cudaMemsetAsync(w.att + (size_t)n_tok * d, 0, (size_t)(mp - n_tok) * d * 2, st));
        const int32_t* lp = last_pos ? last_pos + b0 : nullptr;
        for (int l = 0; l < cfg->n_layers; ++l) {
            const __nv_bfloat16* L = P + o.per_layer0 + (int64_t)l * o.layer_stride;
            if (l > 0) RS_TRY(launch_ln(w.h, L + o.ln1_w, L + o.ln1_b, w.x, mp, d, st));  // layer 0: embed_ln
            // q, k bf16 and v fp16 (the attention's PV runs in fp16, see attention.cu)
            RS_TRY(gemm_bf16(w.x, L + o.qkv_w, L + o.qkv_b, nullptr, w.qkv, mp, 3 * d, d, 7, st));
            if (l == cfg->n_layers - 1) {
                // only the last token of each prompt reaches the head: finish the layer on
                // bc rows (exact; saves 20 d^2 (S - 1) FLOPs per prompt)
                RS_TRY(launch_attention_last(w.qkv, w.h, lp, w.a_last, w.h_last, bc, bp, S, H, st));
                RS_TRY(gemm_bf16(w.a_last, L + o.out_w, L + o.out_b, w.h_last, w.h_last, bp, d, d, 2, st));
                RS_TRY(launch_ln(w.h_last, L + o.ln2_w, L + o.ln2_b, w.x_last, bp, d, st));
                RS_TRY(gemm_bf16(w.x_last, L + o.fc1_w, L + o.fc1_b, nullptr, w.f_last, bp, F, d,
                                 cfg->activation == 0 ? 1 : 3, st));
                RS_TRY(gemm_bf16(w.f_last, L + o.fc2_w, L + o.fc2_b, w.h_last, w.h_last, bp, d, F, 2, st));
                break;
            }
            RS_TRY(attention_fwd_f16v(w.qkv, w.att, bc, S, H, st));
            RS_TRY(gemm_bf16(w.att, L + o.out_w, L + o.out_b, w.h, w.h, mp, d, d, 2, st));
            RS_TRY(launch_ln(w.h, L + o.ln2_w, L + o.ln2_b, w.x, mp, d, st));
            RS_TRY(gemm_bf16(w.x, L + o.fc1_w, L + o.fc1_b, nullptr, w.ffn, mp, F, d, cfg->activation == 0 ? 1 : 3, st));
            RS_TRY(gemm_bf16(w.ffn, L + o.fc2_w, L + o.fc2_b, w.h, w.h, mp, d, F, 2, st));
        }
        RS_TRY(launch_head(w.h_last, nullptr, bc, 1, P, o, d, g + b0, score ? score + b0 : nullptr, st,
                           feat ? feat + b0 * d : nullptr));
    }
    return RS_OK;
}

// ---- building blocks shared with the training pass (ranker_train.cu) -----------------
namespace rs {
int ranker_embed(const int32_t* ids, const void* P, int64_t off_tok, int64_t off_pos, float* h, int n_tok, int S,
                 int d, int vocab, int mp, cudaStream_t st) {
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(P);
    const int wpb = 8;
    embed_kernel<<<(mp + wpb - 1) / wpb, 32 * wpb, 0, st>>>(ids, p + off_tok, p + off_pos, h, n_tok, S, d, vocab, mp);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
int ranker_ln(const float* x, const void* w, const void* b, void* y, int rows, int d, cudaStream_t st) {
    return launch_ln(x, static_cast<const __nv_bfloat16*>(w), static_cast<const __nv_bfloat16*>(b),
                     static_cast<__nv_bfloat16*>(y), rows, d, st);
}
int ranker_head(const float* h, const int32_t* last, int B, int S, const void* P, const rs_ranker_config* cfg, float* g,
                float* score, cudaStream_t st, float* feat) {
    const RankerOffsets o = ranker_offsets(*cfg);
    return launch_head(h, last, B, S, static_cast<const __nv_bfloat16*>(P), o, cfg->d_model, g, score, st, feat);
}
// which: 0 tok, 1 pos, 2 lnf_w, 3 lnf_b, 4 head_w, 5 head_b, then 6 + per-layer index
int64_t ranker_offset(const rs_ranker_config* cfg, int which, int layer) {
    const RankerOffsets o = ranker_offsets(*cfg);
    switch (which) {
        case 0: return o.tok;
        case 1: return o.pos;
        case 2: return o.lnf_w;
        case 3: return o.lnf_b;
        case 4: return o.head_w;
        case 5: return o.head_b;
        default: break;
    }
    const int64_t per[RS_RANKER_N_PER_LAYER] = {o.ln1_w, o.ln1_b, o.qkv_w, o.qkv_b, o.out_w, o.out_b,
                                                o.ln2_w, o.ln2_b, o.fc1_w, o.fc1_b, o.fc2_w, o.fc2_b};
    return o.per_layer0 + (int64_t)layer * o.layer_stride + per[which - 6];
}
}  // namespace rs
