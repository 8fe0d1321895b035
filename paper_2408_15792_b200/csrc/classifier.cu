// the bucketed-classification baseline head on the OPT backbone.
//
// Reference: ClassifierScorer.predict_buckets (predictors.py:283-286: logits = X W + b,
// argmax) and train_classifier's batch_grads (predictors.py:445-453: softmax with the max
// subtracted, nll = -log p[label], dlogits = (p - onehot) / batch). The features here are
// the backbone's LN_f(h_last) rows (rs_ranker_forward_ex), d = 768, C ~ 10 buckets: tiny
// GEMVs, one warp per prompt; the head's weight gradient is a fixed-order reduction over
// the prompts (deterministic, like the backbone's).
#include <math.h>
#include "common.cuh"

namespace rs {

__global__ void cls_logits_kernel(const float* __restrict__ feat, const float* __restrict__ W,
                                  const float* __restrict__ b, int B, int d, int C, float* __restrict__ logits) {
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (p >= B) return;
    const float* f = feat + (size_t)p * d;
    for (int c = 0; c < C; ++c) {
        const float* w = W + (size_t)c * d;
        float acc = 0.f;
        for (int k = lane; k < d; k += 32) acc = fmaf(f[k], w[k], acc);
        acc = warp_sum(acc);
        if (lane == 0) logits[(size_t)p * C + c] = acc + b[c];
    }
}

__global__ void cls_ce_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels, int B, int C,
                              float* __restrict__ loss, float* __restrict__ dlogits, int32_t* __restrict__ bad) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= B) return;
    const float* z = logits + (size_t)p * C;
    const int y = labels[p];
    if (y < 0 || y >= C) {
        atomicOr(bad, 1);
        return;
    }
    float m = -INFINITY;
    for (int c = 0; c < C; ++c) m = fmaxf(m, z[c]);
    float s = 0.f;
    for (int c = 0; c < C; ++c) s += expf(z[c] - m);
    const float lse = m + logf(s);
    loss[p] = lse - z[y];
    float* g = dlogits + (size_t)p * C;
    for (int c = 0; c < C; ++c) g[c] = expf(z[c] - lse) - (c == y ? 1.f : 0.f);
}

// dfeat[p] = dlogits[p] W (one warp per prompt)
__global__ void cls_dfeat_kernel(const float* __restrict__ W, const float* __restrict__ dlogits, int B, int d, int C,
                                 float* __restrict__ dfeat) {
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (p >= B) return;
    const float* g = dlogits + (size_t)p * C;
    for (int k = lane; k < d; k += 32) {
        float acc = 0.f;
        for (int c = 0; c < C; ++c) acc = fmaf(g[c], W[(size_t)c * d + k], acc);
        dfeat[(size_t)p * d + k] = acc;
    }
}

// dW[c, k] += sum_p dlogits[p, c] feat[p, k]; db[c] += sum_p dlogits[p, c] (k = d: the bias),
// one thread per (c, k), prompts summed in order.
__global__ void cls_dw_kernel(const float* __restrict__ feat, const float* __restrict__ dlogits, int B, int d, int C,
                              float* __restrict__ dW, float* __restrict__ db) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= C * (d + 1)) return;
    const int c = i / (d + 1), k = i % (d + 1);
    float acc = 0.f;
    for (int p = 0; p < B; ++p) acc = fmaf(dlogits[(size_t)p * C + c], k < d ? feat[(size_t)p * d + k] : 1.f, acc);
    if (k < d)
        dW[(size_t)c * d + k] += acc;
    else
        db[c] += acc;
}

int cls_head_backward(const float* feat, const float* W, const float* dlogits, int B, int d, int C, float* dW,
                      float* db, float* dfeat, cudaStream_t st) {
    cls_dfeat_kernel<<<(B + 7) / 8, 256, 0, st>>>(W, dlogits, B, d, C, dfeat);
    RS_LAUNCH_CHECK();
    const int n = C * (d + 1);
    cls_dw_kernel<<<(n + 255) / 256, 256, 0, st>>>(feat, dlogits, B, d, C, dW, db);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

int cls_logits_launch(const float* feat, const float* W, const float* b, int B, int d, int C, float* logits,
                      cudaStream_t st) {
    cls_logits_kernel<<<(B + 7) / 8, 256, 0, st>>>(feat, W, b, B, d, C, logits);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

int cls_ce_launch(const float* logits, const int32_t* labels, int B, int C, float* loss, float* dlogits, int32_t* bad,
                  cudaStream_t st) {
    cls_ce_kernel<<<(B + 255) / 256, 256, 0, st>>>(logits, labels, B, C, loss, dlogits, bad);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" int rs_cls_logits(const float* feat, const float* W, const float* b, int32_t B, int32_t d, int32_t C,
                             float* logits, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(B >= 0 && d > 0 && C > 0, "rs_cls_logits: bad shape");
    if (B == 0) return RS_OK;
    RS_CHECK_ARG(feat && W && b && logits, "rs_cls_logits: NULL argument");
    return cls_logits_launch(feat, W, b, B, d, C, logits, as_stream(stream));
}

extern "C" int rs_cls_ce(const float* logits, const int32_t* labels, int32_t B, int32_t C, float* loss, float* dlogits,
                         int32_t* bad, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(B >= 0 && C > 0, "rs_cls_ce: bad shape");
    if (B == 0) return RS_OK;
    RS_CHECK_ARG(logits && labels && loss && dlogits && bad, "rs_cls_ce: NULL argument");
    return cls_ce_launch(logits, labels, B, C, loss, dlogits, bad, as_stream(stream));
}
