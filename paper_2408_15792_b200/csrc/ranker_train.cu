// A10 / K7: one ListMLE gradient pass of the OPT-shape ranker over whole lists.
//
// Reference: train_ranking's minibatch body (predictors.py:379-385): order lists by
// bucketed true length, forward, list_mle_loss/n, list_mle_gradient/n, backward, Adam.
// Here a call accumulates the gradient of sum_lists (ListMLE(list)/list_len) into an fp32
// buffer laid out like the bf16 parameters (rs_ranker_layout), micro-batching whole
// lists (ListMLE couples a list's prompts); the caller all-reduces it across
// data-parallel ranks (NCCL) and applies rs_adam_step with grad_scale = 1/total_lists.
//
// Per micro-batch: forward keeping the activations backward needs (fp32 residual stream
// before each LayerNorm, bf16 LN outputs, qkv, attention output, FFN activations),
// the score head, the fused ListMLE kernel (K6), then the backward:
//   head + final LN -> per layer, in reverse:
//   FC2  (wgrad dW2 = dh^T f, bias sum, dgrad df = (dh W2) * relu'(f))
//   FC1  (wgrad dW1 = df^T x2, bias sum, dgrad dx = df W1) -> LN2 backward into dh
//   out  (wgrad dWo = dh^T a, bias sum, dgrad da = dh Wo) -> attention backward -> dqkv
//   QKV  (wgrad dWqkv = dqkv^T x1, bias sum, dgrad dx = dqkv Wqkv) -> LN1 backward into dh
//   -> token / position embedding scatter-add.
// dgrad GEMMs read the weights MN-major, wgrad GEMMs read both activations MN-major
// (split-K partial slices reduced in a fixed order), so the pass is deterministic.
#include <cuda_bf16.h>
#include <algorithm>
#include "common.cuh"
#include "gemm.cuh"
#include "train.cuh"

namespace rs {
int attention_fwd(const void* qkv, void* out, int B, int S, int H, cudaStream_t st);
int attention_fwd_lse(const void* qkv, void* out, float* lse, int B, int S, int H, cudaStream_t st);
size_t attention_bwd_long_ws(int B, int S, int H);
int attention_bwd_long(const void* qkv, const void* att, const void* dout, void* dqkv, int B, int S, int H, void* ws,
                       size_t ws_bytes, cudaStream_t st, const float* lse_fwd);
int ranker_embed(const int32_t* ids, const void* P, int64_t off_tok, int64_t off_pos, float* h, int n_tok, int S,
                 int d, int vocab, int mp, cudaStream_t st);
int ranker_ln(const float* x, const void* w, const void* b, void* y, int rows, int d, cudaStream_t st);
int ranker_head(const float* h, const int32_t* last, int B, int S, const void* P, const rs_ranker_config* cfg, float* g,
                float* score, cudaStream_t st, float* feat = nullptr);
int64_t ranker_offset(const rs_ranker_config* cfg, int which, int layer);

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = __float2bfloat16_rn(x[i]);
}

enum { OFF_TOK = 0, OFF_POS, OFF_LNF_W, OFF_LNF_B, OFF_HEAD_W, OFF_HEAD_B,
       OFF_LN1_W = 6, OFF_LN1_B, OFF_QKV_W, OFF_QKV_B, OFF_OUT_W, OFF_OUT_B, OFF_LN2_W, OFF_LN2_B, OFF_FC1_W,
       OFF_FC1_B, OFF_FC2_W, OFF_FC2_B };

struct TrainWs {
    // saved activations, per layer (host-side pointer tables into the workspace)
    float* h_in[64];  // L + 1 entries (h_in[L] = final residual stream)
    float* h_mid[64];
    __nv_bfloat16 *x1[64], *qkv[64], *att[64], *x2[64], *f[64];
    float* lse[64];  // attention rows' log2-sum-exp (the backward's P in one pass)
    // backward scratch
    float *dh, *dx, *wpart, *rpart, *g, *dg;
    float *feat, *logits, *dlogits, *dfeat;  // classification head (rs_ranker_grad_cls)
    int32_t* bad;
    __nv_bfloat16 *dh16, *da, *dqkv, *df;
    void* ews;
    size_t ews_bytes;
    void* abw;  // attention backward scratch for S > 128 (row LSE and D)
    size_t abw_bytes;
};

// K splits of a wgrad GEMM: work items (tile, split) run one per CTA pair, so pick the
// split count whose items fill whole waves of CTA pairs best (at least ~one wave; ties to
// fewer splits: fewer fp32 partial slices to write and reduce). The earlier rule (items ~
// SMs) left 2.07-2.4 waves, i.e. a 30% idle tail, on every shape here.
static int wgrad_splits(int M, int N, int K) {
    const int tiles = (M / 256) * (N / 256);
    const int ncl = num_sms() / 2;
    const int kb = K / 64;
    const int smax = std::max(1, std::min(64, kb / 8));
    int best = 1;
    double best_eff = -1.0;
    for (int s = 1; s <= smax; ++s) {
        const int items = tiles * s;
        if (items * 10 < ncl * 9 && s < smax) continue;  // less than ~one wave: too few items
        const int waves = (items + ncl - 1) / ncl;
        const double eff = (double)items / (double)(waves * ncl);
        if (eff >= 0.95) return s;  // the fewest splits that keep >= 95% of the pairs busy
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = s;
        }
    }
    return best;
}

template <typename A>
static void train_layout(A& a, const rs_ranker_config& c, int64_t Tp, int P, int S, TrainWs* w, int n_classes = 0) {
    const int L = c.n_layers;
    const int64_t d = c.d_model, F = c.d_ffn;
    TrainWs t{};
    for (int l = 0; l <= L; ++l) t.h_in[l] = a.template take<float>(Tp * d);
    for (int l = 0; l < L; ++l) {
        t.h_mid[l] = a.template take<float>(Tp * d);
        t.x1[l] = a.template take<__nv_bfloat16>(Tp * d);
        t.qkv[l] = a.template take<__nv_bfloat16>(Tp * 3 * d);
        t.att[l] = a.template take<__nv_bfloat16>(Tp * d);
        t.x2[l] = a.template take<__nv_bfloat16>(Tp * d);
        t.f[l] = a.template take<__nv_bfloat16>(Tp * F);
        t.lse[l] = a.template take<float>((int64_t)P * c.n_heads * S);
    }
    const int64_t wmax = (F * d > 3 * d * d ? F * d : 3 * d * d);
    t.dh = a.template take<float>(Tp * d);
    t.dx = a.template take<float>(Tp * d);
    t.wpart = a.template take<float>((int64_t)64 * wmax);
    const int64_t nrb = (Tp + 63) / 64 + 1;
    // column-reduction partials + their group scratch; the head's (P + 1) rows + scratch
    t.rpart = a.template take<float>(nrb * 2 * (F > 3 * d ? F : 3 * d) + (int64_t)(P + 1 + P / 16 + 1) * (3 * d + 1));
    t.g = a.template take<float>(P);
    t.dg = a.template take<float>(P);
    if (n_classes > 0) {
        t.feat = a.template take<float>((int64_t)P * d);
        t.dfeat = a.template take<float>((int64_t)P * d);
        t.logits = a.template take<float>((int64_t)P * n_classes);
        t.dlogits = a.template take<float>((int64_t)P * n_classes);
        t.bad = a.template take<int32_t>(4);
    }
    t.dh16 = a.template take<__nv_bfloat16>(Tp * d);
    t.da = a.template take<__nv_bfloat16>(Tp * d);
    t.dqkv = a.template take<__nv_bfloat16>(Tp * 3 * d);
    t.df = a.template take<__nv_bfloat16>(Tp * F);
    t.ews_bytes = embed_backward_ws((int)Tp);
    t.ews = a.template take<uint8_t>(t.ews_bytes);
    t.abw_bytes = S > 128 ? attention_bwd_long_ws(P, S, c.n_heads) : 0;
    t.abw = a.template take<uint8_t>(t.abw_bytes);
    if (w) *w = t;
}
struct TrSizer {
    ArenaSizer s;
    template <typename T>
    T* take(size_t n) { s.take<T>(n); return nullptr; }
};

int listmle_lengths_launch(const float* g, const int32_t* lengths, int n_lists, int L, int width, float* loss,
                           float* dg, cudaStream_t st);
int cls_logits_launch(const float* feat, const float* W, const float* b, int B, int d, int C, float* logits,
                      cudaStream_t st);
int cls_ce_launch(const float* logits, const int32_t* labels, int B, int C, float* loss, float* dlogits, int32_t* bad,
                  cudaStream_t st);
int cls_head_backward(const float* feat, const float* W, const float* dlogits, int B, int d, int C, float* dW,
                      float* db, float* dfeat, cudaStream_t st);


// Forward of one micro-batch keeping the activations the backward needs.
static int train_forward(const rs_ranker_config* cfg, const __nv_bfloat16* P16, const int32_t* mids, int P, int S,
                         int n_tok, int64_t Tp, TrainWs& w, cudaStream_t st) {
    const int L = cfg->n_layers, d = cfg->d_model, F = cfg->d_ffn, H = cfg->n_heads;
    auto off = [&](int which, int layer) { return ranker_offset(cfg, which, layer); };
    // ---- forward, keeping activations ----
    RS_TRY(ranker_embed(mids, P16, off(OFF_TOK, 0), off(OFF_POS, 0), w.h_in[0], n_tok, S, d, cfg->vocab, (int)Tp,
                        st));
    if (Tp > n_tok) {
        for (int l = 0; l < L; ++l)
            RS_CUDA(cudaMemsetAsync(w.att[l] + (size_t)n_tok * d, 0, (size_t)(Tp - n_tok) * d * 2, st));
    }
    for (int l = 0; l < L; ++l) {
        RS_TRY(ranker_ln(w.h_in[l], P16 + off(OFF_LN1_W, l), P16 + off(OFF_LN1_B, l), w.x1[l], (int)Tp, d, st));
        RS_TRY(gemm_bf16(w.x1[l], P16 + off(OFF_QKV_W, l), P16 + off(OFF_QKV_B, l), nullptr, w.qkv[l], (int)Tp,
                         3 * d, d, 0, st));
        RS_TRY(attention_fwd_lse(w.qkv[l], w.att[l], w.lse[l], P, S, H, st));
        RS_TRY(gemm_bf16(w.att[l], P16 + off(OFF_OUT_W, l), P16 + off(OFF_OUT_B, l), w.h_in[l], w.h_mid[l],
                         (int)Tp, d, d, 2, st));
        RS_TRY(ranker_ln(w.h_mid[l], P16 + off(OFF_LN2_W, l), P16 + off(OFF_LN2_B, l), w.x2[l], (int)Tp, d, st));
        RS_TRY(gemm_bf16(w.x2[l], P16 + off(OFF_FC1_W, l), P16 + off(OFF_FC1_B, l), nullptr, w.f[l], (int)Tp, F, d,
                         cfg->activation == 0 ? 1 : 3, st));
        RS_TRY(gemm_bf16(w.f[l], P16 + off(OFF_FC2_W, l), P16 + off(OFF_FC2_B, l), w.h_mid[l], w.h_in[l + 1],
                         (int)Tp, d, F, 2, st));
    }
    return RS_OK;
}

// Backward of one micro-batch from w.dh (the head's gradient already in the last-token
// rows, zero elsewhere) through the layers and the embeddings, accumulating into grad.
static int train_backward(const rs_ranker_config* cfg, const __nv_bfloat16* P16, float* grad, const int32_t* mids,
                          int P, int S, int n_tok, int64_t Tp, TrainWs& w, cudaStream_t st) {
    const int L = cfg->n_layers, d = cfg->d_model, F = cfg->d_ffn, H = cfg->n_heads;
    auto off = [&](int which, int layer) { return ranker_offset(cfg, which, layer); };
    f32_to_bf16_kernel<<<1184, 256, 0, st>>>(w.dh, w.dh16, (int64_t)Tp * d);
    RS_LAUNCH_CHECK();
    const int T = (int)Tp;
    for (int l = L - 1; l >= 0; --l) {
        int sp;
        // FC2: h_out = h_mid + f W2^T + b2
        sp = wgrad_splits(d, F, T);
        RS_TRY(gemm_bf16_ex(w.dh16, w.f[l], nullptr, nullptr, w.wpart, d, F, T, 6, 1, 1, sp, st));
        RS_TRY(slices_add(w.wpart, sp, (int64_t)d * F, grad + off(OFF_FC2_W, l), st));
        // below the top layer the LN1 backward of layer l + 1 already summed dh's columns
        if (l == L - 1) RS_TRY(colsum_add(w.dh, false, n_tok, d, w.rpart, grad + off(OFF_FC2_B, l), st));
        RS_TRY(gemm_bf16_ex(w.dh16, P16 + off(OFF_FC2_W, l), nullptr, w.f[l], w.df, T, F, d, 5, 0, 1, 1, st));
        // FC1: f = relu(x2 W1^T + b1)
        sp = wgrad_splits(F, d, T);
        RS_TRY(gemm_bf16_ex(w.df, w.x2[l], nullptr, nullptr, w.wpart, F, d, T, 6, 1, 1, sp, st));
        RS_TRY(slices_add(w.wpart, sp, (int64_t)F * d, grad + off(OFF_FC1_W, l), st));
        RS_TRY(colsum_add(w.df, true, n_tok, F, w.rpart, grad + off(OFF_FC1_B, l), st));
        RS_TRY(gemm_bf16_ex(w.df, P16 + off(OFF_FC1_W, l), nullptr, nullptr, w.dx, T, d, F, 4, 0, 1, 1, st));
        RS_TRY(ln_backward(w.dx, w.h_mid[l], P16 + off(OFF_LN2_W, l), w.dh, w.dh16, w.rpart, n_tok, d,
                           grad + off(OFF_LN2_W, l), nullptr, st, grad + off(OFF_OUT_B, l)));
        // out-proj: h_mid = h_in + a Wo^T + bo
        sp = wgrad_splits(d, d, T);
        RS_TRY(gemm_bf16_ex(w.dh16, w.att[l], nullptr, nullptr, w.wpart, d, d, T, 6, 1, 1, sp, st));
        RS_TRY(slices_add(w.wpart, sp, (int64_t)d * d, grad + off(OFF_OUT_W, l), st));
        RS_TRY(gemm_bf16_ex(w.dh16, P16 + off(OFF_OUT_W, l), nullptr, nullptr, w.da, T, d, d, 0, 0, 1, 1, st));
        if (S <= 128) {  // (+ the QKV bias gradient's per-prompt column sums, reduced here)
            RS_TRY(attention_bwd(w.qkv[l], w.att[l], w.da, w.dqkv, P, S, H, st, w.lse[l], w.rpart));
            RS_TRY(rows_add(w.rpart, P, 3 * d, grad + off(OFF_QKV_B, l), w.rpart + (size_t)P * 3 * d, st));
        } else {
            RS_TRY(attention_bwd_long(w.qkv[l], w.att[l], w.da, w.dqkv, P, S, H, w.abw, w.abw_bytes, st, w.lse[l]));
        }
        // QKV: qkv = x1 Wqkv^T + b
        sp = wgrad_splits(3 * d, d, T);
        RS_TRY(gemm_bf16_ex(w.dqkv, w.x1[l], nullptr, nullptr, w.wpart, 3 * d, d, T, 6, 1, 1, sp, st));
        RS_TRY(slices_add(w.wpart, sp, (int64_t)3 * d * d, grad + off(OFF_QKV_W, l), st));
        if (S > 128) RS_TRY(colsum_add(w.dqkv, true, n_tok, 3 * d, w.rpart, grad + off(OFF_QKV_B, l), st));
        RS_TRY(gemm_bf16_ex(w.dqkv, P16 + off(OFF_QKV_W, l), nullptr, nullptr, w.dx, T, d, 3 * d, 4, 0, 1, 1, st));
        RS_TRY(ln_backward(w.dx, w.h_in[l], P16 + off(OFF_LN1_W, l), w.dh, w.dh16, w.rpart, n_tok, d,
                           grad + off(OFF_LN1_W, l), nullptr, st, l > 0 ? grad + off(OFF_FC2_B, l - 1) : nullptr));
    }
    RS_TRY(embed_backward(mids, P, S, cfg->vocab, w.dh, d, grad + off(OFF_TOK, 0), grad + off(OFF_POS, 0), w.ews,
                          w.ews_bytes, st));
    return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" size_t rs_ranker_grad_workspace_size(const rs_ranker_config* cfg, int32_t lists_per_micro, int32_t list_len,
                                                int32_t S) {
    if (!cfg || lists_per_micro <= 0 || list_len <= 0 || S <= 0 || cfg->n_layers > 63) return 0;
    const int P = lists_per_micro * list_len;
    const int64_t Tp = ((int64_t)P * S + 255) / 256 * 256;
    TrSizer s;
    train_layout(s, *cfg, Tp, P, S, nullptr);
    return s.s.used + 4096;
}

extern "C" int rs_ranker_grad(const rs_ranker_config* cfg, const void* params, float* grad, const int32_t* ids,
                              const int32_t* last_pos, const int32_t* lengths, int32_t n_lists, int32_t list_len, int32_t S,
                              int32_t bucket_width, int32_t lists_per_micro, float* loss_out, void* ws,
                              size_t ws_bytes, void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(cfg && params && grad && ids && lengths && loss_out, "rs_ranker_grad: NULL argument");
    RS_CHECK_ARG(n_lists > 0 && list_len >= 1 && S >= 1 && S <= 512, "rs_ranker_grad: need S <= 512 (got %d)", S);
    RS_CHECK_ARG(bucket_width >= 1, "bucket_width must be >= 1");
    RS_CHECK_ARG(lists_per_micro >= 1, "lists_per_micro must be >= 1");
    RS_CHECK_ARG(cfg->n_layers <= 63 && cfg->d_model == cfg->n_heads * 64, "rs_ranker_grad: bad config");
    if (ws_bytes < rs_ranker_grad_workspace_size(cfg, lists_per_micro, list_len, S)) {
        set_error("rs_ranker_grad: workspace too small");
        return RS_ERR_WORKSPACE;
    }
    const int L = cfg->n_layers, d = cfg->d_model;
    const __nv_bfloat16* P16 = static_cast<const __nv_bfloat16*>(params);
    auto off = [&](int which, int layer) { return ranker_offset(cfg, which, layer); };
    for (int l0 = 0; l0 < n_lists; l0 += lists_per_micro) {
        const int ml = (n_lists - l0) < lists_per_micro ? (n_lists - l0) : lists_per_micro;
        const int P = ml * list_len;
        const int n_tok = P * S;
        const int64_t Tp = ((int64_t)n_tok + 255) / 256 * 256;
        Arena ar(ws, ws_bytes);
        TrainWs w;
        {
            const int Pm = lists_per_micro * list_len;
            const int64_t Tm = ((int64_t)Pm * S + 255) / 256 * 256;
            train_layout(ar, *cfg, Tm, Pm, S, &w);
        }
        const int32_t* mids = ids + (int64_t)l0 * list_len * S;
        const int32_t* mlen = lengths + (int64_t)l0 * list_len;
        const int32_t* mlast = last_pos ? last_pos + (int64_t)l0 * list_len : nullptr;
        RS_TRY(train_forward(cfg, P16, mids, P, S, n_tok, Tp, w, st));
        RS_TRY(ranker_head(w.h_in[L], mlast, P, S, P16, cfg, w.g, nullptr, st));
        // ---- ListMLE (K6): per-list loss / n and dg = grad / n ----
        RS_TRY(listmle_lengths_launch(w.g, mlen, ml, list_len, bucket_width, loss_out + l0, w.dg, st));
        // ---- backward ----
        RS_CUDA(cudaMemsetAsync(w.dh, 0, (size_t)Tp * d * sizeof(float), st));
        // padding rows take part in the wgrad reductions: keep their gradients zero
        if (Tp > n_tok)
            RS_CUDA(cudaMemsetAsync(w.dqkv + (size_t)n_tok * 3 * d, 0, (size_t)(Tp - n_tok) * 3 * d * 2, st));
        RS_TRY(head_backward(w.h_in[L], mlast, P, S, P16 + off(OFF_LNF_W, 0), P16 + off(OFF_LNF_B, 0),
                             P16 + off(OFF_HEAD_W, 0), w.dg, w.dh, w.rpart, d, grad + off(OFF_HEAD_W, 0),
                             grad + off(OFF_LNF_W, 0), grad + off(OFF_HEAD_B, 0), st));
        RS_TRY(train_backward(cfg, P16, grad, mids, P, S, n_tok, Tp, w, st));
    }
    return RS_OK;
}

// §8f #4: the same pass with the bucketed-classification head (classifier.cu) and the
// softmax cross-entropy of train_classifier (predictors.py:445-453) in place of the score
// head and ListMLE: micro-batches of prompts, LN_f features -> logits -> nll, dlogits ->
// head gradients + d LN_f output -> the shared backward.
extern "C" size_t rs_ranker_grad_cls_workspace_size(const rs_ranker_config* cfg, int32_t prompts_per_micro, int32_t S,
                                                    int32_t n_classes) {
    if (!cfg || prompts_per_micro <= 0 || S <= 0 || n_classes <= 0 || cfg->n_layers > 63) return 0;
    const int P = prompts_per_micro;
    const int64_t Tp = ((int64_t)P * S + 255) / 256 * 256;
    TrSizer s;
    train_layout(s, *cfg, Tp, P, S, nullptr, n_classes);
    return s.s.used + 4096;
}

extern "C" int rs_ranker_grad_cls(const rs_ranker_config* cfg, const void* params, float* grad, const int32_t* ids,
                                  const int32_t* last_pos, const int32_t* labels, int32_t n_prompts, int32_t S,
                                  int32_t n_classes, const float* cls_w, const float* cls_b, float* cls_grad,
                                  int32_t prompts_per_micro, float* loss_out, void* ws, size_t ws_bytes,
                                  void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(cfg && params && grad && ids && labels && cls_w && cls_b && cls_grad && loss_out,
                 "rs_ranker_grad_cls: NULL argument");
    RS_CHECK_ARG(n_prompts > 0 && S >= 1 && S <= 512, "rs_ranker_grad_cls: need S <= 512 (got %d)", S);
    RS_CHECK_ARG(n_classes >= 2 && prompts_per_micro >= 1, "rs_ranker_grad_cls: need >= 2 classes");
    RS_CHECK_ARG(cfg->n_layers <= 63 && cfg->d_model == cfg->n_heads * 64, "rs_ranker_grad_cls: bad config");
    if (ws_bytes < rs_ranker_grad_cls_workspace_size(cfg, prompts_per_micro, S, n_classes)) {
        set_error("rs_ranker_grad_cls: workspace too small");
        return RS_ERR_WORKSPACE;
    }
    const int L = cfg->n_layers, d = cfg->d_model, C = n_classes;
    const __nv_bfloat16* P16 = static_cast<const __nv_bfloat16*>(params);
    auto off = [&](int which, int layer) { return ranker_offset(cfg, which, layer); };
    for (int p0 = 0; p0 < n_prompts; p0 += prompts_per_micro) {
        const int P = (n_prompts - p0) < prompts_per_micro ? (n_prompts - p0) : prompts_per_micro;
        const int n_tok = P * S;
        const int64_t Tp = ((int64_t)n_tok + 255) / 256 * 256;
        Arena ar(ws, ws_bytes);
        TrainWs w;
        {
            const int64_t Tm = ((int64_t)prompts_per_micro * S + 255) / 256 * 256;
            train_layout(ar, *cfg, Tm, prompts_per_micro, S, &w, C);
        }
        const int32_t* mids = ids + (int64_t)p0 * S;
        const int32_t* mlast = last_pos ? last_pos + p0 : nullptr;
        RS_TRY(train_forward(cfg, P16, mids, P, S, n_tok, Tp, w, st));
        RS_TRY(ranker_head(w.h_in[L], mlast, P, S, P16, cfg, w.g, nullptr, st, w.feat));
        RS_TRY(cls_logits_launch(w.feat, cls_w, cls_b, P, d, C, w.logits, st));
        RS_CUDA(cudaMemsetAsync(w.bad, 0, sizeof(int32_t), st));
        RS_TRY(cls_ce_launch(w.logits, labels + p0, P, C, loss_out + p0, w.dlogits, w.bad, st));
        RS_TRY(cls_head_backward(w.feat, cls_w, w.dlogits, P, d, C, cls_grad, cls_grad + (size_t)C * d, w.dfeat, st));
        RS_CUDA(cudaMemsetAsync(w.dh, 0, (size_t)Tp * d * sizeof(float), st));
        if (Tp > n_tok)
            RS_CUDA(cudaMemsetAsync(w.dqkv + (size_t)n_tok * 3 * d, 0, (size_t)(Tp - n_tok) * 3 * d * 2, st));
        RS_TRY(head_backward(w.h_in[L], mlast, P, S, P16 + off(OFF_LNF_W, 0), P16 + off(OFF_LNF_B, 0),
                             P16 + off(OFF_HEAD_W, 0), nullptr, w.dh, w.rpart, d, nullptr, grad + off(OFF_LNF_W, 0),
                             nullptr, st, w.dfeat));
        RS_TRY(train_backward(cfg, P16, grad, mids, P, S, n_tok, Tp, w, st));
    }
    return RS_OK;
}
