// Linear / one-hidden-layer MLP ranker over the 24 prompt features: the reference's
// default predictor (A2/A3 of SURVEY §8a), kept as the cfg1 parity bridge.
//
// Reference: _Standardizer.fit / __call__ (predictors.py:159-172), _Net.forward /
// backward (predictors.py:175-206), the train_ranking minibatch step
// (predictors.py:374-386) and _Adam.step (predictors.py:209-225). Everything is float64
// like the reference. Elementwise arithmetic is written with explicit round-to-nearest
// intrinsics (no FMA contraction), so standardisation and the Adam update are the same
// IEEE operations numpy performs; dot products and reductions differ from BLAS only in
// summation order.
//
// Parameter layout (one f64 buffer, the reference's `params` list flattened):
//   hidden == 0: [w (D), b (1)]
//   hidden  > 0: [W1 (D x H, row-major like numpy), b1 (H), w2 (H), b2 (1)]
#include "common.cuh"

namespace rs {

static __host__ __device__ inline int64_t lin_n_params(int D, int H) {
    return H <= 0 ? (int64_t)D + 1 : (int64_t)D * H + 2 * H + 1;
}

// One thread per row: standardise, then X@w + b or tanh(X@W1 + b1)@w2 + b2.
__global__ void linear_forward_kernel(const double* __restrict__ X, int64_t B, int D, const double* __restrict__ mean,
                                      const double* __restrict__ stdv, int H, const double* __restrict__ p,
                                      double* __restrict__ out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < B; r += (int64_t)gridDim.x * blockDim.x) {
        const double* x = X + r * D;
        double acc;
        if (H <= 0) {
            acc = 0.0;
            for (int k = 0; k < D; ++k) acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(__dsub_rn(x[k], mean[k]), stdv[k]), p[k]));
            acc = __dadd_rn(acc, p[D]);
        } else {
            const double* W1 = p;
            const double* b1 = p + (int64_t)D * H;
            const double* w2 = b1 + H;
            acc = 0.0;
            for (int j = 0; j < H; ++j) {
                double pre = 0.0;
                for (int k = 0; k < D; ++k)
                    pre = __dadd_rn(pre, __dmul_rn(__ddiv_rn(__dsub_rn(x[k], mean[k]), stdv[k]), W1[(int64_t)k * H + j]));
                acc = __dadd_rn(acc, __dmul_rn(tanh(__dadd_rn(pre, b1[j])), w2[j]));
            }
            acc = __dadd_rn(acc, w2[H]);
        }
        out[r] = acc;
    }
}

// Column statistics: one block per feature column, fixed-order tree reductions.
__global__ void standardizer_fit_kernel(const double* __restrict__ X, int64_t N, int D, double* __restrict__ mean,
                                        double* __restrict__ stdv) {
    __shared__ double red[256];
    const int c = blockIdx.x;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < N; r += blockDim.x) s = __dadd_rn(s, X[r * D + c]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    const double mu = __ddiv_rn(red[0], (double)N);
    __syncthreads();
    double q = 0.0;
    for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
        const double d = __dsub_rn(X[r * D + c], mu);
        q = __dadd_rn(q, __dmul_rn(d, d));
    }
    red[threadIdx.x] = q;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double sd = __dsqrt_rn(__ddiv_rn(red[0], (double)N));
        mean[c] = mu;
        stdv[c] = sd < 1e-12 ? 1.0 : sd;  // predictors.py:168
    }
}

// numpy's logaddexp (npymath npy_logaddexp)
__device__ __forceinline__ double np_logaddexp(double x, double y) {
    if (x == y) return __dadd_rn(x, 0.693147180559945309417232121458176568);  // x + LOGE2
    const double t = __dsub_rn(x, y);
    if (t > 0) return __dadd_rn(x, log1p(exp(-t)));
    if (t <= 0) return __dadd_rn(y, log1p(exp(t)));
    return t;  // NaN
}

// numpy pairwise sum of n <= 128 doubles (the 8-accumulator unrolled block of
// pairwise_sum for n >= 8, plain left-to-right below 8)
__device__ double np_pairwise_sum(const double* a, int n) {
    if (n < 8) {
        double r = -0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[i + k]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// One train_ranking minibatch step (predictors.py:374-386) in one CTA:
//   Xb = Xs[batch]; true_order = stable argsort(y // width); g = net(Xb);
//   loss = ListMLE(g, order) / n; dg = grad / n; grads = net.backward(Xb, dg); Adam.
// smem: xb [n*D], h [n*H], g/dg/t/lse/L [n] x5, lab/order [n] x2
__global__ void linear_train_step_kernel(const double* __restrict__ Xs, const int64_t* __restrict__ batch,
                                         const int64_t* __restrict__ y, int n, int D, int H, int width,
                                         double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
                                         double lr, double b1, double b2, double eps, double bc1, double bc2,
                                         double* __restrict__ loss_out, double* __restrict__ grad_out) {
    extern __shared__ double sm[];
    double* xb = sm;
    double* h = xb + (size_t)n * D;
    double* g = h + (size_t)n * (H > 0 ? H : 0);
    double* dg = g + n;
    double* t = dg + n;
    double* lse = t + n;
    double* Lc = lse + n;
    int64_t* lab = reinterpret_cast<int64_t*>(Lc + n);
    int* ord = reinterpret_cast<int*>(lab + n);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t np_ = lin_n_params(D, H);

    for (int e = tid; e < n * D; e += nt) xb[e] = Xs[batch[e / D] * D + (e % D)];
    for (int i = tid; i < n; i += nt) lab[i] = y[batch[i]] / width;  // lengths >= 1: floor == trunc
    __syncthreads();
    // forward
    if (H <= 0) {
        for (int i = tid; i < n; i += nt) {
            double acc = 0.0;
            for (int k = 0; k < D; ++k) acc = __dadd_rn(acc, __dmul_rn(xb[i * D + k], p[k]));
            g[i] = __dadd_rn(acc, p[D]);
        }
    } else {
        const double* W1 = p;
        const double* bb1 = p + (int64_t)D * H;
        for (int e = tid; e < n * H; e += nt) {
            const int i = e / H, j = e % H;
            double pre = 0.0;
            for (int k = 0; k < D; ++k) pre = __dadd_rn(pre, __dmul_rn(xb[i * D + k], W1[(int64_t)k * H + j]));
            h[e] = tanh(__dadd_rn(pre, bb1[j]));
        }
        __syncthreads();
        const double* w2 = bb1 + H;
        for (int i = tid; i < n; i += nt) {
            double acc = 0.0;
            for (int j = 0; j < H; ++j) acc = __dadd_rn(acc, __dmul_rn(h[i * H + j], w2[j]));
            g[i] = __dadd_rn(acc, w2[H]);
        }
    }
    // stable order of the labels: rank_i = #{j: lab_j < lab_i} + #{j < i: lab_j == lab_i}
    for (int i = tid; i < n; i += nt) {
        int r = 0;
        for (int j = 0; j < n; ++j) r += (lab[j] < lab[i]) || (lab[j] == lab[i] && j < i);
        ord[r] = i;
    }
    __syncthreads();
    if (tid == 0) {
        // ranking.py:81-120 with numpy's recurrences
        for (int j = 0; j < n; ++j) t[j] = g[ord[j]];
        lse[n - 1] = t[n - 1];
        for (int j = n - 2; j >= 0; --j) lse[j] = np_logaddexp(lse[j + 1], t[j]);
        for (int j = 0; j < n; ++j) Lc[j] = __dsub_rn(lse[j], t[j]);
        const double loss = np_pairwise_sum(Lc, n);
        double acc = -lse[0];
        Lc[0] = acc;
        for (int j = 1; j < n; ++j) {
            acc = np_logaddexp(acc, -lse[j]);
            Lc[j] = acc;
        }
        for (int j = 0; j < n; ++j) dg[ord[j]] = __ddiv_rn(__dsub_rn(exp(__dadd_rn(t[j], Lc[j])), 1.0), (double)n);
        loss_out[0] = __ddiv_rn(loss, (double)n);
    }
    __syncthreads();
    // backward (predictors.py:198-206) + Adam (predictors.py:217-225), one parameter per thread
    for (int64_t q = tid; q < np_; q += nt) {
        double gr = 0.0;
        if (H <= 0) {
            if (q < D)
                for (int i = 0; i < n; ++i) gr = __dadd_rn(gr, __dmul_rn(xb[i * D + q], dg[i]));
            else
                for (int i = 0; i < n; ++i) gr = __dadd_rn(gr, dg[i]);
        } else {
            const double* w2 = p + (int64_t)D * H + H;
            if (q < (int64_t)D * H) {  // dW1[k, j] = sum_i x_ik * dg_i * w2_j * (1 - h_ij^2)
                const int k = (int)(q / H), j = (int)(q % H);
                for (int i = 0; i < n; ++i) {
                    const double hh = h[i * H + j];
                    const double dpre = __dmul_rn(__dmul_rn(dg[i], w2[j]), __dsub_rn(1.0, __dmul_rn(hh, hh)));
                    gr = __dadd_rn(gr, __dmul_rn(xb[i * D + k], dpre));
                }
            } else if (q < (int64_t)D * H + H) {  // db1
                const int j = (int)(q - (int64_t)D * H);
                for (int i = 0; i < n; ++i) {
                    const double hh = h[i * H + j];
                    gr = __dadd_rn(gr, __dmul_rn(__dmul_rn(dg[i], w2[j]), __dsub_rn(1.0, __dmul_rn(hh, hh))));
                }
            } else if (q < (int64_t)D * H + 2 * H) {  // dw2
                const int j = (int)(q - (int64_t)D * H - H);
                for (int i = 0; i < n; ++i) gr = __dadd_rn(gr, __dmul_rn(h[i * H + j], dg[i]));
            } else {
                for (int i = 0; i < n; ++i) gr = __dadd_rn(gr, dg[i]);
            }
        }
        if (grad_out) grad_out[q] = gr;
        const double mi = __dadd_rn(__dmul_rn(b1, m[q]), __dmul_rn(__dsub_rn(1.0, b1), gr));
        const double vi = __dadd_rn(__dmul_rn(b2, v[q]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), gr), gr));
        m[q] = mi;
        v[q] = vi;
        const double mhat = __ddiv_rn(mi, bc1), vhat = __ddiv_rn(vi, bc2);
        // p -= lr * mhat / (sqrt(vhat) + eps), evaluated left to right like numpy
        p[q] = __dsub_rn(p[q], __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
    }
}

__global__ void standardize_kernel(const double* __restrict__ X, int64_t total, int D, const double* __restrict__ mean,
                                   const double* __restrict__ stdv, double* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % D);
        out[e] = __ddiv_rn(__dsub_rn(X[e], mean[c]), stdv[c]);
    }
}

}  // namespace rs

using namespace rs;

extern "C" int64_t rs_linear_n_params(int32_t n_features, int32_t hidden) {
    if (n_features < 1 || hidden < 0) return -1;
    return lin_n_params(n_features, hidden);
}

extern "C" int rs_standardizer_fit(const double* X, int64_t n_rows, int32_t n_features, double* mean, double* stdv,
                                   void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(n_rows >= 1 && n_features >= 1, "rs_standardizer_fit: need at least one row and one feature");
    standardizer_fit_kernel<<<n_features, 256, 0, as_stream(stream)>>>(X, n_rows, n_features, mean, stdv);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" int rs_standardize(const double* X, int64_t n_rows, int32_t n_features, const double* mean,
                              const double* stdv, double* out, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(n_rows >= 0 && n_features >= 1, "rs_standardize: bad shape");
    if (n_rows == 0) return RS_OK;
    const int64_t total = n_rows * n_features;
    const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    standardize_kernel<<<blocks, 256, 0, as_stream(stream)>>>(X, total, n_features, mean, stdv, out);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" int rs_linear_forward(const double* X, int64_t n_rows, int32_t n_features, const double* mean,
                                 const double* stdv, int32_t hidden, const double* params, double* out, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(n_rows >= 0 && n_features >= 1 && hidden >= 0, "rs_linear_forward: bad shape");
    if (n_rows == 0) return RS_OK;
    const int blocks = (int)((n_rows + 127) / 128 < 148 * 8 ? (n_rows + 127) / 128 : 148 * 8);
    linear_forward_kernel<<<blocks, 128, 0, as_stream(stream)>>>(X, n_rows, n_features, mean, stdv, hidden, params,
                                                                  out);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

static size_t lin_step_smem(int n, int D, int H) {
    return (size_t)n * D * 8 + (size_t)n * (H > 0 ? H : 0) * 8 + (size_t)n * 5 * 8 + (size_t)n * 8 + (size_t)n * 4;
}

extern "C" int rs_linear_train_step(const double* Xs, const int64_t* batch, const int64_t* lengths, int32_t n,
                                    int32_t n_features, int32_t hidden, int32_t bucket_width, double* params,
                                    double* adam_m, double* adam_v, double lr, double beta1, double beta2, double eps,
                                    int64_t t, double* loss_out, double* grad_out, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(n >= 2 && n_features >= 1 && hidden >= 0, "rs_linear_train_step: need a list of >= 2 items");
    RS_CHECK_ARG(bucket_width >= 1, "bucket_width must be >= 1");
    RS_CHECK_ARG(t >= 1, "rs_linear_train_step: Adam step t must be >= 1");
    const size_t smem = lin_step_smem(n, n_features, hidden);
    RS_CHECK_ARG(smem <= 200 * 1024, "rs_linear_train_step: list of %d x (%d features, %d hidden) exceeds shared memory",
                 n, n_features, hidden);
    if (smem > 48 * 1024) RS_CUDA(ensure_smem((const void*)linear_train_step_kernel, (int)smem));
    // bias corrections exactly as Python evaluates them: 1 - beta ** t
    const double bc1 = 1.0 - pow(beta1, (double)t), bc2 = 1.0 - pow(beta2, (double)t);
    linear_train_step_kernel<<<1, 256, smem, as_stream(stream)>>>(Xs, batch, lengths, n, n_features, hidden,
                                                                   bucket_width, params, adam_m, adam_v, lr, beta1,
                                                                   beta2, eps, bc1, bc2, loss_out, grad_out);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
