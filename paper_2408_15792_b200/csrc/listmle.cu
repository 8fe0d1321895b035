// K6: ListMLE (Plackett-Luce) loss and gradient, one warp per list.
//
// Reference: ranking.list_mle_loss / list_mle_gradient (ranking.py:86-120):
//   t = s[order];  lse_i = log sum_{k>=i} exp(t_k)   (reversed np.logaddexp.accumulate)
//   loss = sum_i (lse_i - t_i)
//   L_j  = log sum_{i<=j} exp(-lse_i)                 (np.logaddexp.accumulate of -lse)
//   grad[order[j]] = exp(t_j + L_j) - 1
// and the training step (predictors.py:379-384) which builds `order` as the stable
// argsort of bucket_lengths(len, width) (ranking.py:123-132) and divides by n.
//
// Both cumulative log-sum-exps are warp scans under the associative logaddexp
// operator (blocked: each lane scans its own run of items serially, then one
// shuffle scan over the 32 lane totals), i.e. a warp-segmented LSE scan.
#include <math.h>
#include "common.cuh"

namespace rs {

template <typename T>
__device__ __forceinline__ T ninf();
template <>
__device__ __forceinline__ float ninf<float>() { return -INFINITY; }
template <>
__device__ __forceinline__ double ninf<double>() { return -(double)INFINITY; }

// numpy.logaddexp semantics: max + log1p(exp(-|a-b|)), with -inf as identity.
__device__ __forceinline__ float lae(float a, float b) {
    if (a == -INFINITY) return b;
    if (b == -INFINITY) return a;
    float m = fmaxf(a, b);
    return m + log1pf(expf(-fabsf(a - b)));
}
__device__ __forceinline__ double lae(double a, double b) {
    if (a == -(double)INFINITY) return b;
    if (b == -(double)INFINITY) return a;
    double m = fmax(a, b);
    return m + log1p(exp(-fabs(a - b)));
}
__device__ __forceinline__ float ex(float v) { return expf(v); }
__device__ __forceinline__ double ex(double v) { return exp(v); }

// Inclusive logaddexp scan over v[0..n) (smem, one warp), in forward (rev=false) or
// reverse (rev=true) index order; result written to out[] in place-compatible order.
template <typename T, bool Rev>
__device__ void warp_lae_scan(const T* v, T* out, int n) {
    const int lane = threadIdx.x & 31;
    const int ipt = (n + 31) / 32;
    const int beg = lane * ipt;
    const int end = min(n, beg + ipt);
    T acc = ninf<T>();
    for (int k = beg; k < end; ++k) acc = lae(acc, v[Rev ? n - 1 - k : k]);
    // exclusive scan of lane totals
    T x = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = lae(x, y);
    }
    T excl = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) excl = ninf<T>();
    T run = excl;
    for (int k = beg; k < end; ++k) {
        const int idx = Rev ? n - 1 - k : k;
        run = lae(run, v[idx]);
        out[idx] = run;
    }
    __syncwarp();
}

// t (target order) in smem -> loss (warp-reduced, returned on all lanes) and
// gt[j] = grad in target order. lse is scratch of n entries.
template <typename T>
__device__ T listmle_core(T* t, T* lse, T* gt, int n) {
    const int lane = threadIdx.x & 31;
    warp_lae_scan<T, true>(t, lse, n);
    T part = 0;
    for (int k = lane; k < n; k += 32) part += lse[k] - t[k];
    T loss = warp_sum(part);
    // -lse into gt, forward scan in place, then grad_t = exp(t + L) - 1
    for (int k = lane; k < n; k += 32) gt[k] = -lse[k];
    __syncwarp();
    warp_lae_scan<T, false>(gt, gt, n);
    for (int k = lane; k < n; k += 32) gt[k] = ex(t[k] + gt[k]) - (T)1;
    __syncwarp();
    return loss;
}

template <typename T>
__global__ void listmle_order_kernel(const T* __restrict__ scores, const int64_t* __restrict__ order,
                                     int n_lists, int L, T* __restrict__ loss_out, T* __restrict__ grad_out,
                                     int* __restrict__ bad) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warps = blockDim.x / 32;
    const int wid = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int list = blockIdx.x * warps + wid;
    T* t = reinterpret_cast<T*>(smem_raw) + (size_t)wid * 3 * L;
    T* lse = t + L;
    T* gt = lse + L;
    int* seen = reinterpret_cast<int*>(reinterpret_cast<T*>(smem_raw) + (size_t)warps * 3 * L) + (size_t)wid * L;
    if (list >= n_lists) return;
    const T* s = scores + (size_t)list * L;
    const int64_t* o = order + (size_t)list * L;
    for (int k = lane; k < L; k += 32) seen[k] = 0;
    __syncwarp();
    int badl = 0;
    for (int k = lane; k < L; k += 32) {
        int64_t ok = o[k];
        if (ok < 0 || ok >= L) {
            badl = 1;
            t[k] = 0;
        } else {
            seen[ok] = 1;
            t[k] = s[ok];
        }
    }
    __syncwarp();
    for (int k = lane; k < L; k += 32) badl |= (seen[k] == 0);
    if (__any_sync(0xffffffffu, badl)) {
        if (lane == 0) atomicOr(bad, 1);
        return;
    }
    T loss = listmle_core<T>(t, lse, gt, L);
    if (lane == 0) loss_out[list] = loss;
    T* g = grad_out + (size_t)list * L;
    for (int k = lane; k < L; k += 32) g[o[k]] = gt[k];
}

// Training form: order = stable argsort of (len // width); outputs divided by L.
__global__ void listmle_lengths_kernel(const float* __restrict__ gnet, const int32_t* __restrict__ lengths,
                                       int n_lists, int L, int width, float* __restrict__ loss_out,
                                       float* __restrict__ dg_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warps = blockDim.x / 32;
    const int wid = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int list = blockIdx.x * warps + wid;
    float* t = reinterpret_cast<float*>(smem_raw) + (size_t)wid * 3 * L;
    float* lse = t + L;
    float* gt = lse + L;
    int* lab = reinterpret_cast<int*>(reinterpret_cast<float*>(smem_raw) + (size_t)warps * 3 * L) + (size_t)wid * 2 * L;
    int* rank = lab + L;
    if (list >= n_lists) return;
    const float* g = gnet + (size_t)list * L;
    const int32_t* len = lengths + (size_t)list * L;
    for (int k = lane; k < L; k += 32) {
        // bucket_lengths: floor division of int64 lengths (ranking.py:131-132)
        int v = len[k];
        int q = v / width;
        if ((v % width != 0) && ((v < 0) != (width < 0))) --q;
        lab[k] = q;
    }
    __syncwarp();
    for (int k = lane; k < L; k += 32) {
        const int b = lab[k];
        int r = 0;
        for (int j = 0; j < L; ++j) {
            const int bj = lab[j];
            r += (bj < b) || (bj == b && j < k);
        }
        rank[k] = r;
        t[r] = g[k];
    }
    __syncwarp();
    float loss = listmle_core<float>(t, lse, gt, L);
    const float inv = 1.0f / (float)L;
    if (lane == 0) loss_out[list] = loss * inv;
    float* dg = dg_out + (size_t)list * L;
    for (int k = lane; k < L; k += 32) dg[k] = gt[rank[k]] * inv;
}

}  // namespace rs

using namespace rs;

static int listmle_warps(int L) { return L <= 1024 ? 4 : 1; }

extern "C" int rs_listmle_order(const void* scores, int dtype, const int64_t* order, int32_t n_lists,
                                int32_t L, void* loss, void* grad, int32_t* bad, void* stream) {
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(dtype == RS_F32 || dtype == RS_F64, "rs_listmle_order: dtype must be f32/f64");
    RS_CHECK_ARG(n_lists >= 0 && L >= 0 && L <= 8192, "rs_listmle_order: need 0 <= list_len <= 8192");
    if (n_lists == 0) return RS_OK;
    if (L == 0) {
        RS_CUDA(cudaMemsetAsync(loss, 0, (size_t)n_lists * (dtype == RS_F32 ? 4 : 8), st));
        return RS_OK;
    }
    const int w = listmle_warps(L);
    const int blocks = (n_lists + w - 1) / w;
    if (dtype == RS_F32) {
        size_t sm = (size_t)w * L * (3 * sizeof(float) + sizeof(int));
        if (sm > 48 * 1024) RS_CUDA(cudaFuncSetAttribute(listmle_order_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        listmle_order_kernel<float><<<blocks, 32 * w, sm, st>>>((const float*)scores, order, n_lists, L,
                                                                 (float*)loss, (float*)grad, bad);
    } else {
        size_t sm = (size_t)w * L * (3 * sizeof(double) + sizeof(int));
        if (sm > 48 * 1024) RS_CUDA(cudaFuncSetAttribute(listmle_order_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        listmle_order_kernel<double><<<blocks, 32 * w, sm, st>>>((const double*)scores, order, n_lists, L,
                                                                  (double*)loss, (double*)grad, bad);
    }
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" int rs_listmle_lengths(const float* g, const int32_t* lengths, int32_t n_lists, int32_t L,
                                  int32_t width, float* loss, float* dg, void* stream) {
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(width >= 1, "bucket_width must be >= 1");
    RS_CHECK_ARG(n_lists >= 0 && L >= 1 && L <= 4096, "rs_listmle_lengths: need 1 <= list_len <= 4096");
    if (n_lists == 0) return RS_OK;
    const int w = listmle_warps(L);
    const int blocks = (n_lists + w - 1) / w;
    size_t sm = (size_t)w * L * (3 * sizeof(float) + 2 * sizeof(int));
    if (sm > 48 * 1024) RS_CUDA(cudaFuncSetAttribute(listmle_lengths_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    listmle_lengths_kernel<<<blocks, 32 * w, sm, st>>>(g, lengths, n_lists, L, width, loss, dg);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

namespace rs {
int listmle_lengths_launch(const float* g, const int32_t* lengths, int n_lists, int L, int width, float* loss,
                           float* dg, cudaStream_t st) {
    return rs_listmle_lengths(g, lengths, n_lists, L, width, loss, dg, st);
}
}  // namespace rs
