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

// ---- register-resident form for lists of <= 64 items (the cfg3 shape) -------------------
// One warp per list, two items per lane, nothing staged in shared memory. Target order
// = a warp bitonic sort of the unique keys (label, index); the two log-sum-exp scans run
// on (max, scaled-sum) pairs in base 2 — one ex2 per combine instead of the exp + log1p of
// logaddexp — so the kernel is ALU/MUFU-light enough to stream at a good HBM fraction.
// Element p of the sorted sequence lives in lane p >> 1, slot p & 1.
struct Lse2 {
    float m, s;  // value = m + log2(s); identity (LSE2_NONE, 0)
};

__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Identity element: a finite sentinel instead of -inf keeps (identity, identity) free
// of inf - inf (ex2(0) * 0 = 0), so the combine needs no branch.
constexpr float LSE2_NONE = -1e30f;

__device__ __forceinline__ Lse2 lse2_comb(Lse2 a, Lse2 b) {
    const bool ab = a.m >= b.m;
    const float M = fmaxf(a.m, b.m), mn = fminf(a.m, b.m);
    const float sb = ab ? a.s : b.s, ss = ab ? b.s : a.s;
    return Lse2{M, fmaf(ss, fast_ex2(mn - M), sb)};
}

__device__ __forceinline__ Lse2 shfl_down_lse2(Lse2 v, int o) {
    return Lse2{__shfl_down_sync(0xffffffffu, v.m, o), __shfl_down_sync(0xffffffffu, v.s, o)};
}
__device__ __forceinline__ Lse2 shfl_up_lse2(Lse2 v, int o) {
    return Lse2{__shfl_up_sync(0xffffffffu, v.m, o), __shfl_up_sync(0xffffffffu, v.s, o)};
}

template <typename K>
__device__ __forceinline__ K kmin(K a, K b) { return a < b ? a : b; }
template <>
__device__ __forceinline__ uint32_t kmin<uint32_t>(uint32_t a, uint32_t b) { return min(a, b); }
template <typename K>
__device__ __forceinline__ K kmax(K a, K b) { return a < b ? b : a; }
template <>
__device__ __forceinline__ uint32_t kmax<uint32_t>(uint32_t a, uint32_t b) { return max(a, b); }

template <typename K>
__device__ __forceinline__ void warp_bitonic64(K& e0, K& e1) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
        const bool asc = ((2 * lane) & k) == 0;  // for k >= 4, (p & k) is the same for both slots
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 1) {
                const K lo = kmin(e0, e1), hi = kmax(e0, e1);
                e0 = asc ? lo : hi;
                e1 = asc ? hi : lo;
            } else {
                const int lm = j >> 1;
                const bool take_min = ((lane & lm) == 0) == asc;
                const K o0 = __shfl_xor_sync(0xffffffffu, e0, lm);
                const K o1 = __shfl_xor_sync(0xffffffffu, e1, lm);
                e0 = take_min ? kmin(o0, e0) : kmax(o0, e0);
                e1 = take_min ? kmin(o1, e1) : kmax(o1, e1);
            }
        }
    }
}

// Keys below 2^16 (labels < 1023: lengths < 10230 at the default width) sort two per
// register: the pair of a lane shares its compare direction and partner lane at every
// shuffle stage, so one u16x2 min/max does both slots.
__device__ __forceinline__ uint32_t vmin16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t vmax16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ uint32_t warp_bitonic64_packed(uint32_t P) {  // slot 0 low, slot 1 high
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
        const bool asc = ((2 * lane) & k) == 0;
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 1) {
                const uint32_t Q = __byte_perm(P, 0, 0x1032);  // halves swapped
                const uint32_t mn = vmin16x2(P, Q), mx = vmax16x2(P, Q);
                P = __byte_perm(asc ? mn : mx, asc ? mx : mn, 0x7610);
            } else {
                const int lm = j >> 1;
                const bool take_min = ((lane & lm) == 0) == asc;
                const uint32_t O = __shfl_xor_sync(0xffffffffu, P, lm);
                P = take_min ? vmin16x2(O, P) : vmax16x2(O, P);
            }
        }
    }
    return P;
}

// Sorted slot -> item index, for the three key widths.
__device__ __forceinline__ void listmle64_order(int lab0, int lab1, int L, int& s0, int& s1) {
    const int lane = threadIdx.x & 31;
    const int i0 = lane, i1 = lane + 32;
    const bool ok0 = i0 >= L || (lab0 >= 0 && lab0 < 1023), ok1 = i1 >= L || (lab1 >= 0 && lab1 < 1023);
    if (__all_sync(0xffffffffu, ok0 && ok1)) {
        const uint32_t k0 = i0 < L ? ((uint32_t)lab0 << 6) | (uint32_t)i0 : 0xFFFFu;
        const uint32_t k1 = i1 < L ? ((uint32_t)lab1 << 6) | (uint32_t)i1 : 0xFFFFu;
        const uint32_t P = warp_bitonic64_packed(k0 | (k1 << 16));
        s0 = (int)(P & 63);
        s1 = (int)((P >> 16) & 63);
        return;
    }
    const bool w0 = i0 >= L || (lab0 >= 0 && lab0 < (1 << 25)), w1 = i1 >= L || (lab1 >= 0 && lab1 < (1 << 25));
    if (__all_sync(0xffffffffu, w0 && w1)) {
        uint32_t k0 = i0 < L ? ((uint32_t)lab0 << 6) | (uint32_t)i0 : ~0u;
        uint32_t k1 = i1 < L ? ((uint32_t)lab1 << 6) | (uint32_t)i1 : ~0u;
        warp_bitonic64<uint32_t>(k0, k1);
        s0 = (int)(k0 & 63);
        s1 = (int)(k1 & 63);
        return;
    }
    uint64_t k0 = i0 < L ? ((uint64_t)((uint32_t)lab0 ^ 0x80000000u) << 32) | (uint64_t)i0 : ~0ull;
    uint64_t k1 = i1 < L ? ((uint64_t)((uint32_t)lab1 ^ 0x80000000u) << 32) | (uint64_t)i1 : ~0ull;
    warp_bitonic64<uint64_t>(k0, k1);
    s0 = (int)(k0 & 63);
    s1 = (int)(k1 & 63);
}

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Scores in target order (t0 at p = 2 lane, t1 at p + 1; base-2 units) -> loss and grads.
__device__ __forceinline__ void listmle64_scan(float t0, float t1, bool v0, bool v1, int L, float inv, int s0,
                                               int s1, float* __restrict__ loss_out, float* __restrict__ dg) {
    const int lane = threadIdx.x & 31;
    constexpr float LN2 = 0.6931471805599453f;
    float lse0, lse1, L0, L1;
    const float M = warp_max_f(fmaxf(v0 ? t0 : LSE2_NONE, v1 ? t1 : LSE2_NONE));
    const float m = -warp_max_f(fmaxf(v0 ? -t0 : LSE2_NONE, v1 ? -t1 : LSE2_NONE));
    if (M - m <= 100.f) {
        // Range fits fp32 after one shift by the list max (every 2^(t - M) >= 2^-100 is a
        // normal float), so both log-sum-exps are plain prefix sums of shifted exponentials.
        const float w0 = v0 ? fast_ex2(t0 - M) : 0.f, w1 = v1 ? fast_ex2(t1 - M) : 0.f;
        const float r0 = w0 + w1;
        float x = r0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float y = __shfl_down_sync(0xffffffffu, x, o);
            if (lane + o < 32) x += y;
        }
        float tail = __shfl_down_sync(0xffffffffu, x, 1);
        if (lane == 31) tail = 0.f;
        lse0 = M + fast_lg2(r0 + tail);
        lse1 = M + fast_lg2(w1 + tail);
        // -lse is largest at the last item (lse_{L-1} = t_{L-1}), the shift of the second sum
        const float lastv = ((L - 1) & 1) ? lse1 : lse0;
        const float Mu = -__shfl_sync(0xffffffffu, lastv, (L - 1) >> 1);
        const float q0 = v0 ? fast_ex2(-lse0 - Mu) : 0.f, q1 = v1 ? fast_ex2(-lse1 - Mu) : 0.f;
        const float c1 = q0 + q1;
        x = c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        float head = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) head = 0.f;
        L0 = Mu + fast_lg2(head + q0);
        L1 = Mu + fast_lg2(head + c1);
    } else {
        // wide range: (max, scaled-sum) pairs
        const Lse2 e1{v1 ? t1 : LSE2_NONE, v1 ? 1.f : 0.f};
        const Lse2 e0 = lse2_comb(Lse2{v0 ? t0 : LSE2_NONE, v0 ? 1.f : 0.f}, e1);
        Lse2 x = e0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const Lse2 y = shfl_down_lse2(x, o);
            if (lane + o < 32) x = lse2_comb(x, y);
        }
        Lse2 tail = shfl_down_lse2(x, 1);
        if (lane == 31) tail = Lse2{LSE2_NONE, 0.f};
        const Lse2 l0 = lse2_comb(e0, tail), l1 = lse2_comb(e1, tail);
        lse0 = l0.m + fast_lg2(l0.s);
        lse1 = l1.m + fast_lg2(l1.s);
        const Lse2 f0{v0 ? -lse0 : LSE2_NONE, v0 ? 1.f : 0.f};
        const Lse2 f1 = lse2_comb(f0, Lse2{v1 ? -lse1 : LSE2_NONE, v1 ? 1.f : 0.f});
        x = f1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const Lse2 y = shfl_up_lse2(x, o);
            if (lane >= o) x = lse2_comb(x, y);
        }
        Lse2 head = shfl_up_lse2(x, 1);
        if (lane == 0) head = Lse2{LSE2_NONE, 0.f};
        const Lse2 c0 = lse2_comb(head, f0), c1 = lse2_comb(head, f1);
        L0 = c0.m + fast_lg2(c0.s);
        L1 = c1.m + fast_lg2(c1.s);
    }
    const float part = (v0 ? lse0 - t0 : 0.f) + (v1 ? lse1 - t1 : 0.f);
    const float loss = warp_sum(part) * LN2;
    // grad in target order = e^{t + L} - 1, scattered back to the item's own slot
    if (v0) dg[s0] = (fast_ex2(t0 + L0) - 1.f) * inv;
    if (v1) dg[s1] = (fast_ex2(t1 + L1) - 1.f) * inv;
    if (lane == 0) *loss_out = loss * inv;
}

// One list on the whole warp (two items per lane): the general <= 64 path.
__device__ __forceinline__ void listmle64_one(const float* __restrict__ gnet, const int32_t* __restrict__ lengths,
                                              int list, int L, int width, float* __restrict__ loss_out,
                                              float* __restrict__ dg_out) {
    constexpr float LOG2E = 1.4426950408889634f;
    const int lane = threadIdx.x & 31;
    const float inv = 1.0f / (float)L;
    const int p0 = 2 * lane, p1 = p0 + 1;
    const bool v0 = p0 < L, v1 = p1 < L;
    const float* g = gnet + (size_t)list * L;
    const int32_t* len = lengths + (size_t)list * L;
    const bool in0 = lane < L, in1 = lane + 32 < L;
    const float g0 = in0 ? __ldcs(g + lane) : 0.f, g1 = in1 ? __ldcs(g + lane + 32) : 0.f;
    const int n0 = in0 ? __ldcs(len + lane) : 0, n1 = in1 ? __ldcs(len + lane + 32) : 0;
    // bucket_lengths: floor division (ranking.py:131-132)
    int lab0 = n0 / width, lab1 = n1 / width;
    if ((n0 % width != 0) && (n0 < 0)) --lab0;
    if ((n1 % width != 0) && (n1 < 0)) --lab1;
    int s0, s1;
    listmle64_order(lab0, lab1, L, s0, s1);
    // gather the scores into target order (base-2 units)
    const float a0 = __shfl_sync(0xffffffffu, g0, s0 & 31), b0 = __shfl_sync(0xffffffffu, g1, s0 & 31);
    const float a1 = __shfl_sync(0xffffffffu, g0, s1 & 31), b1 = __shfl_sync(0xffffffffu, g1, s1 & 31);
    const float t0 = ((s0 >> 5) ? b0 : a0) * LOG2E, t1 = ((s1 >> 5) ? b1 : a1) * LOG2E;
    listmle64_scan(t0, t1, v0, v1, L, inv, s0, s1, loss_out + list, dg_out + (size_t)list * L);
}

// 64 16-bit keys over an 8-lane group (lanes hl = 0..7 of the group, partner lanes by
// shfl_xor with masks < 8), 8 keys per lane in 4 registers: sorted position p = 8 hl + e
// lives in register e & 3, half e >> 2. The network is the all-ascending form of bitonic
// sort — each merge of width k starts with a "flip" stage (p against p ^ (k - 1)) followed
// by half-cleaners (p against p ^ j), and every comparator puts the minimum at the lower
// position — so the in-lane stages need no direction selects: j = 1 and j = 2 compare whole
// registers (min/max of both halves at once), j = 4 the two halves of one register.
__device__ __forceinline__ uint32_t hswap(uint32_t x) { return __byte_perm(x, 0, 0x1032); }
__device__ __forceinline__ void cas16x2(uint32_t& a, uint32_t& b) {  // a <- min, b <- max (per half)
    const uint32_t mn = vmin16x2(a, b), mx = vmax16x2(a, b);
    a = mn;
    b = mx;
}
__device__ __forceinline__ void sort64_flip8(uint32_t (&R)[4], int hl) {
    // j = 4 half-cleaner: low half (e) gets the min, high half (e + 4) the max
    auto j4 = [&]() {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t S = hswap(R[r]);
            R[r] = __byte_perm(vmin16x2(R[r], S), vmax16x2(R[r], S), 0x7610);
        }
    };
    auto j2 = [&]() { cas16x2(R[0], R[2]); cas16x2(R[1], R[3]); };
    auto j1 = [&]() { cas16x2(R[0], R[1]); cas16x2(R[2], R[3]); };
    auto xlane = [&](int m, bool lower) {  // half-cleaner across lanes hl, hl ^ m
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t O = __shfl_xor_sync(0xffffffffu, R[r], m);
            R[r] = lower ? vmin16x2(R[r], O) : vmax16x2(R[r], O);
        }
    };
    auto xflip = [&](int m, bool lower) {  // e <-> 7 - e of lane hl ^ m: partner's R[3 - r], halves swapped
        uint32_t O[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) O[r] = __shfl_xor_sync(0xffffffffu, R[3 - r], m);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t S = hswap(O[r]);
            R[r] = lower ? vmin16x2(R[r], S) : vmax16x2(R[r], S);
        }
    };
    // k = 2: flip = j1;  k = 4: flip e <-> 3 - e, then j1
    j1();
    cas16x2(R[0], R[3]);
    cas16x2(R[1], R[2]);
    j1();
    // k = 8: flip e <-> 7 - e inside the lane: (R0, R3) and (R1, R2) with halves crossed
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const uint32_t S = hswap(R[3 - r]);
        const uint32_t mn = vmin16x2(R[r], S), mx = vmax16x2(R[r], S);
        R[r] = __byte_perm(mn, mx, 0x7610);      // {e_r, e_{r+4}}       = {mn.lo, mx.hi}
        R[3 - r] = __byte_perm(mn, mx, 0x5432);  // {e_{3-r}, e_{7-r}} = {mn.hi, mx.lo}
    }
    j2();
    j1();
    // k = 16, 32, 64: flip across lanes, cross-lane half-cleaners, then the in-lane ones
    xflip(1, (hl & 1) == 0);
    j4(); j2(); j1();
    xflip(3, (hl & 2) == 0);
    xlane(1, (hl & 1) == 0);
    j4(); j2(); j1();
    xflip(7, (hl & 4) == 0);
    xlane(2, (hl & 2) == 0);
    xlane(1, (hl & 1) == 0);
    j4(); j2(); j1();
}

// LPW lists per warp (32 / LPW lanes x 64 * LPW / 32 items each) for the common case —
// labels < 1023 and score ranges within the shifted-sum bound — so the shuffle stages of
// the sort and of both scans serve LPW lists at once and the first log2(items) stages of
// every bitonic merge stay inside a lane; any warp whose lists fall outside that case is
// redone one list at a time by listmle64_one. Sorted element p of a list lives in lane
// p / IPL of its group, packed register (p % IPL) / 2, 16-bit half p % 2.
// W > 0: the bucket width as a compile-time constant (the training default, 10: the floor
// division becomes a multiply-shift); W == 0: runtime `width`.
// LC > 0: the list length as a compile-time constant (the cfg3 shape, 64: every validity
// test folds away); LC == 0: runtime `L_rt`.
template <int LPW, int W, int LC>
__global__ void __launch_bounds__(256) listmle_lengths64xN_kernel(const float* __restrict__ gnet,
                                                                  const int32_t* __restrict__ lengths, int n_lists,
                                                                  int L_rt, int width_rt, float* __restrict__ loss_out,
                                                                  float* __restrict__ dg_out) {
    const int L = LC > 0 ? LC : L_rt;
    constexpr int LANES = 32 / LPW, IPL = 64 / LANES, NR = IPL / 2;
    static_assert(IPL >= 2 && IPL % 2 == 0, "two 16-bit keys per register");
    const int width = W > 0 ? W : width_rt;
    constexpr float LOG2E = 1.4426950408889634f, LN2 = 0.6931471805599453f;
    __shared__ __align__(16) float sg[8][LPW][64];  // per warp, per list: the scores (base-2 units)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sub = lane / LANES, hl = lane % LANES;
    const int warps_total = gridDim.x * (blockDim.x >> 5);
    const float inv = 1.0f / (float)L;
    const bool vec = (L & 3) == 0;
    for (int grp = blockIdx.x * (blockDim.x >> 5) + wid; LPW * grp < n_lists; grp += warps_total) {
        const int list = LPW * grp + sub;
        const bool live = list < n_lists;
        float gv[IPL];
        int nv[IPL];
        const float* g = gnet + (size_t)list * L;
        const int32_t* len = lengths + (size_t)list * L;
        if (live && vec && IPL * hl < L) {
#pragma unroll
            for (int q = 0; q < IPL / 4; ++q) {
                const float4 g4 = __ldcs(reinterpret_cast<const float4*>(g + IPL * hl) + q);
                const int4 n4 = __ldcs(reinterpret_cast<const int4*>(len + IPL * hl) + q);
                gv[4 * q] = g4.x; gv[4 * q + 1] = g4.y; gv[4 * q + 2] = g4.z; gv[4 * q + 3] = g4.w;
                nv[4 * q] = n4.x; nv[4 * q + 1] = n4.y; nv[4 * q + 2] = n4.z; nv[4 * q + 3] = n4.w;
            }
        } else {
#pragma unroll
            for (int e = 0; e < IPL; ++e) {
                const int i = IPL * hl + e;
                gv[e] = (live && i < L) ? __ldcs(g + i) : 0.f;
                nv[e] = (live && i < L) ? __ldcs(len + i) : 0;
            }
        }
        bool ok = true;
        uint32_t R[NR];
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            const int i = IPL * hl + e;
            int lab = nv[e] / width;
            if (nv[e] < 0 && lab * width != nv[e]) --lab;  // floor division
            const bool valid = live && i < L;
            ok &= !valid || (lab >= 0 && lab < 1023);
            const uint32_t key = valid ? (((uint32_t)lab << 6) | (uint32_t)i) : 0xFFFFu;
            if constexpr (IPL == 8) {  // sort64_flip8 layout: register e & 3, half e >> 2
                if (e >> 2) R[e & 3] |= key << 16; else R[e & 3] = key;
            } else {
                if (e & 1) R[e >> 1] |= key << 16; else R[e >> 1] = key;
            }
            sg[wid][sub][i] = gv[e] * LOG2E;
        }
        if constexpr (IPL == 8) {
            if (__all_sync(0xffffffffu, ok)) sort64_flip8(R, hl);
        } else if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
            for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    if (j == 1) {  // the two halves of each register
#pragma unroll
                        for (int ri = 0; ri < NR; ++ri) {
                            const bool asc = ((IPL * hl + 2 * ri) & k) == 0;
                            const uint32_t Q = __byte_perm(R[ri], 0, 0x1032);
                            const uint32_t mn = vmin16x2(R[ri], Q), mx = vmax16x2(R[ri], Q);
                            R[ri] = __byte_perm(asc ? mn : mx, asc ? mx : mn, 0x7610);
                        }
                    } else if (j < IPL) {  // two registers of the same lane
#pragma unroll
                        for (int ri = 0; ri < NR; ++ri) {
                            const int rp = ri ^ (j >> 1);
                            if (rp < ri) continue;
                            const bool asc = ((IPL * hl + 2 * ri) & k) == 0;
                            const uint32_t mn = vmin16x2(R[ri], R[rp]), mx = vmax16x2(R[ri], R[rp]);
                            R[ri] = asc ? mn : mx;
                            R[rp] = asc ? mx : mn;
                        }
                    } else {  // lanes hl and hl ^ (j / IPL) of the group
                        const int lm = j / IPL;
                        const bool asc = ((IPL * hl) & k) == 0;
                        const bool take_min = ((hl & lm) == 0) == asc;
#pragma unroll
                        for (int ri = 0; ri < NR; ++ri) {
                            const uint32_t O = __shfl_xor_sync(0xffffffffu, R[ri], lm);
                            R[ri] = take_min ? vmin16x2(O, R[ri]) : vmax16x2(O, R[ri]);
                        }
                    }
                }
            }
        }
        __syncwarp();
        int sidx[IPL];
        float t[IPL];
        bool v[IPL];
        float M = LSE2_NONE, mneg = LSE2_NONE;
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            sidx[e] = IPL == 8 ? (int)((R[e & 3] >> (16 * (e >> 2))) & 63) : (int)((R[e >> 1] >> (16 * (e & 1))) & 63);
            // L == 64: a dead group (past n_lists) computes on zeros (its shuffles stay inside
            // its own lanes) and stores nothing, so no per-item masks
            v[e] = LC == 64 ? true : (live && IPL * hl + e < L);
            t[e] = v[e] ? sg[wid][sub][sidx[e]] : LSE2_NONE;
            M = fmaxf(M, v[e] ? t[e] : LSE2_NONE);
            mneg = fmaxf(mneg, v[e] ? -t[e] : LSE2_NONE);
        }
#pragma unroll
        for (int o = LANES / 2; o; o >>= 1) {
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            mneg = fmaxf(mneg, __shfl_xor_sync(0xffffffffu, mneg, o));
        }
        const bool fast = !live || (M + mneg <= 100.f);
        if (!__all_sync(0xffffffffu, ok && fast)) {
            __syncwarp();
            for (int h = 0; h < LPW; ++h)
                if (LPW * grp + h < n_lists) listmle64_one(gnet, lengths, LPW * grp + h, L, width, loss_out, dg_out);
            continue;
        }
        // suffix sums of 2^(t - M): lse_p = M + log2(sum_{q >= p})
        float w[IPL], sfx[IPL];
#pragma unroll
        for (int e = 0; e < IPL; ++e) w[e] = v[e] ? fast_ex2(t[e] - M) : 0.f;
        sfx[IPL - 1] = w[IPL - 1];
#pragma unroll
        for (int e = IPL - 2; e >= 0; --e) sfx[e] = w[e] + sfx[e + 1];
        float x = sfx[0];
#pragma unroll
        for (int o = 1; o < LANES; o <<= 1) {
            const float y = __shfl_down_sync(0xffffffffu, x, o);
            if (hl + o < LANES) x += y;
        }
        float tail = __shfl_down_sync(0xffffffffu, x, 1);
        if (hl == LANES - 1) tail = 0.f;
        // In units of the suffix sums s_e = sfx_e + tail (= 2^(lse_e - M)):
        //   lse_e - t_e          = lg2(s_e) - (t_e - M)                         (the loss terms)
        //   2^(-lse_e - Mu)      = s_last / s_e,  Mu = -lse_{L-1}, s_last = w_{L-1}
        //   2^(t_e + L_e)        = w_e * (head + c_e) / s_last   (L_e = Mu + lg2(head + c_e))
        // so the second scan and the gradient need one reciprocal per item and no ex2 / lg2
        float sv[IPL], pl = 0.f, pt = 0.f;
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            sv[e] = sfx[e] + tail;
            pl += v[e] ? fast_lg2(sv[e]) : 0.f;
            pt += v[e] ? t[e] - M : 0.f;
        }
        float part = pl - pt;
#pragma unroll
        for (int o = LANES / 2; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const int lastl = (L - 1) / IPL, laste = (L - 1) % IPL;
        float lastv = w[0];
#pragma unroll
        for (int e = 1; e < IPL; ++e)
            if (e == laste) lastv = w[e];
        const float s_last = __shfl_sync(0xffffffffu, lastv, sub * LANES + lastl);
        const float r_last = fast_rcp(s_last);
        float c[IPL];
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < IPL; ++e) {
            acc += v[e] ? s_last * fast_rcp(sv[e]) : 0.f;
            c[e] = acc;
        }
        x = acc;
#pragma unroll
        for (int o = 1; o < LANES; o <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, x, o);
            if (hl >= o) x += y;
        }
        float head = __shfl_up_sync(0xffffffffu, x, 1);
        if (hl == 0) head = 0.f;
        float gr[IPL];
#pragma unroll
        for (int e = 0; e < IPL; ++e) gr[e] = fmaf(w[e] * r_last, head + c[e], -1.f) * inv;
        float* dg = dg_out + (size_t)list * L;
        if constexpr (LC == 64 && IPL % 4 == 0) {
            // scatter into the list's smem row (every score has been read: sg is free), then
            // each lane stores its own IPL contiguous items as 16-B vectors
            __syncwarp();
#pragma unroll
            for (int e = 0; e < IPL; ++e)
                if (live) sg[wid][sub][sidx[e]] = gr[e];  // a dead group's keys all map to slot 63
            __syncwarp();
            if (live) {
#pragma unroll
                for (int q = 0; q < IPL / 4; ++q)
                    __stcs(reinterpret_cast<float4*>(dg + IPL * hl) + q,
                           *reinterpret_cast<const float4*>(&sg[wid][sub][IPL * hl + 4 * q]));
            }
        } else {
#pragma unroll
            for (int e = 0; e < IPL; ++e)
                if (v[e]) dg[sidx[e]] = gr[e];
        }
        if (live && hl == 0) loss_out[list] = part * LN2 * inv;
        __syncwarp();  // sg is reused by the next group
    }
}

}  // namespace rs

using namespace rs;

static int listmle_warps(int L) { return L <= 1024 ? 4 : 1; }

extern "C" int rs_listmle_order(const void* scores, int dtype, const int64_t* order, int32_t n_lists,
                                int32_t L, void* loss, void* grad, int32_t* bad, void* stream) {
    RS_NVTX();
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
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(width >= 1, "bucket_width must be >= 1");
    RS_CHECK_ARG(n_lists >= 0 && L >= 1 && L <= 4096, "rs_listmle_lengths: need 1 <= list_len <= 4096");
    if (n_lists == 0) return RS_OK;
    if (L <= 64) {
        // persistent grid: 8 warps per CTA, 8 CTAs per SM (one list per warp iteration)
        static int n_sm = 0;
        if (!n_sm) {
            int dev;
            RS_CUDA(cudaGetDevice(&dev));
            RS_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
        }
        constexpr int LPW = 4;
        const int groups = (n_lists + LPW - 1) / LPW;
        const int blocks = (groups + 7) / 8 < n_sm * 8 ? (groups + 7) / 8 : n_sm * 8;
        if (width == 10 && L == 64)
            listmle_lengths64xN_kernel<LPW, 10, 64><<<blocks, 256, 0, st>>>(g, lengths, n_lists, L, width, loss, dg);
        else if (width == 10)
            listmle_lengths64xN_kernel<LPW, 10, 0><<<blocks, 256, 0, st>>>(g, lengths, n_lists, L, width, loss, dg);
        else
            listmle_lengths64xN_kernel<LPW, 0, 0><<<blocks, 256, 0, st>>>(g, lengths, n_lists, L, width, loss, dg);
        RS_LAUNCH_CHECK();
        return RS_OK;
    }
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
