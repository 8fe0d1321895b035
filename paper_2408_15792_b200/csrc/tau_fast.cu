// K10 fast path: exact Kendall tau-b pair counts by an MSD bucket partition of x, for
// y spanning fewer than 4096 distinct images (cfg4: lengths in [1, 2048]; the engine's
// tau(first_token_s, output_tokens); the trainer's tau(score, length)).
//
// Reference: ranking.kendall_tau_b (ranking.py:24-63): sign(dx)*sign(dy) over all
// n(n-1)/2 pairs (:45-50) and np.unique tie counts (:52-57). Same exact integers here:
//   D  = #{(i, j): x_i < x_j, y_i > y_j}            (strictly discordant)
//   n1 = pairs tied in x, n2 = tied in y, n3 = tied in both, C = n0 - n1 - n2 + n3 - D.
//
// Instead of sorting all n (x, y) keys (the general path in tau.cu: log2(n / 2048) global
// merge passes), x is partitioned by the digits of its range-reduced 32-bit image:
//   level 1: the top 12 bits -> 4096 buckets (count, column scan, scatter of a packed
//            32-bit key  key1 = (x_rem << 12) | (y - ymin), x_rem = the low r1 bits);
//   level 2: buckets holding more than `cap` keys are split by the next 12 bits (the
//            same three steps per bucket, chunked so a big bucket uses many CTAs).
// The leaves are merged, in x order, into "groups" of < cap keys (or single-x groups of
// any size). Groups are x-disjoint and in x order, so
//   D = sum over groups of (in-group D) + sum over items of #{earlier items, y larger}.
// One persistent CTA walks a contiguous run of groups with a running y histogram in
// shared memory (the cross term), sorting each group by key1 in shared memory and
// counting the in-group D as the strict inversions of its y sequence (Knight's identity,
// a counting merge sort); single-x groups need no sort (no discordant pairs inside).
// The runs of different CTAs are joined by their per-CTA y histograms (a column scan
// and one dot product per CTA). DRAM traffic: 8 B/item read twice (min/max, scatter),
// 4 B/item read once (count), 4 B written + read at each level.
//
// The path is chosen on the device; when y spans >= 4096 values, or a 256-image-wide
// level-2 bucket holds more than `cap` keys with different x (adversarial
// concentration: > 16 distinct x in a 2^r2-image window holding more than `cap` keys),
// counts[5] is set to 2 and rs_tau_counts runs the general path.
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "tau_fast.cuh"

namespace rs {

constexpr int TF_BINS = 4096;
constexpr int TF_CAP = 8192;  // sortable group capacity (shared memory keys)
constexpr int TF_ITEMS = 16;
constexpr int TF_LEAF_T = TF_CAP / TF_ITEMS;  // 512 threads
constexpr int TF_T = 512;                     // other kernels
constexpr int TF_SCAN_T = 1024;
constexpr uint32_t TF_GROUP_COST = 2048;  // per-group overhead of the leaf walk, in keys

struct TfParams {
    uint32_t nxmin, xmax, nymin, ymax;  // ~min (zero-initialised atomicMax), max
    int nan, fail, ngroups, pad;
};

struct TfDerived {
    uint32_t xmin, ymin, r1, r2, d2;
    bool ok;
};
__device__ __forceinline__ TfDerived tf_derive(const TfParams* p) {
    TfDerived d;
    d.xmin = ~p->nxmin;
    d.ymin = ~p->nymin;
    const uint32_t xr = p->xmax - d.xmin;
    const uint32_t s = xr ? 32u - __clz(xr) : 0u;
    d.r1 = s > 12 ? s - 12 : 0;
    d.d2 = d.r1 < 12 ? d.r1 : 12;
    d.r2 = d.r1 - d.d2;
    d.ok = !p->nan && (p->ymax - d.ymin) < (uint32_t)TF_BINS && p->ymax >= d.ymin;
    return d;
}

// 32-bit order-preserving image (float64 semantics) of x[i]; TF_DT_U32 = precomputed.
__device__ __forceinline__ uint32_t tf_img(const void* p, int dt, uint32_t i) {
    if (dt == RS_F32) return orderable_f32(static_cast<const float*>(p)[i]);
    if (dt == RS_I32) return orderable_i32(static_cast<const int32_t*>(p)[i]);
    return static_cast<const uint32_t*>(p)[i];
}

__device__ __forceinline__ uint32_t tf_conv(uint32_t raw, int dt) {
    if (dt == RS_F32) return orderable_f32(__uint_as_float(raw));
    if (dt == RS_I32) return orderable_i32((int32_t)raw);
    return raw;
}
__device__ __forceinline__ bool tf_isnan(uint32_t raw, int dt) {
    return dt == RS_F32 && (raw & 0x7fffffffu) > 0x7f800000u;
}
// Four consecutive 32-bit raw values from i (i % 4 == 0): one 16-B load when the base is
// aligned and all four are in range, else scalar loads (zeros past n).
__device__ __forceinline__ uint4 tf_load4(const void* p, uint32_t i, uint32_t n, bool aligned) {
    const uint32_t* q = static_cast<const uint32_t*>(p);
    if (aligned && i + 3 < n) return __ldcs(reinterpret_cast<const uint4*>(q + i));
    uint4 r;
    r.x = i < n ? q[i] : 0u;
    r.y = i + 1 < n ? q[i + 1] : 0u;
    r.z = i + 2 < n ? q[i + 2] : 0u;
    r.w = i + 3 < n ? q[i + 3] : 0u;
    return r;
}
__device__ __forceinline__ uint32_t u4get(const uint4& v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }

__device__ __forceinline__ uint32_t tf_key1(uint32_t xi, uint32_t yi, const TfDerived& d) {
    const uint32_t xr = xi - d.xmin;
    const uint32_t rem = d.r1 ? (xr & ((1u << d.r1) - 1u)) : 0u;
    return (rem << 12) | (yi - d.ymin);
}
__device__ __forceinline__ uint32_t tf_digit1(uint32_t xi, const TfDerived& d) { return (xi - d.xmin) >> d.r1; }

// ---- block helpers --------------------------------------------------------------
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t t = lane < NT / 32 ? s_warp[lane] : 0u;
        uint32_t z = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < NT / 32) s_warp[lane] = z - t;
        if (lane == 31 && total) *total = z;
    }
    __syncthreads();
    const uint32_t r = s_warp[wid] + x - v;
    __syncthreads();
    return r;
}

__device__ __forceinline__ void acc_add(unsigned long long v, unsigned long long* out) {
    // CTA-wide sum, one atomic (every thread calls)
    __shared__ unsigned long long part[32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0ull;
        t = warp_sum(t);
        if (threadIdx.x == 0 && t) atomicAdd(out, t);
    }
    __syncthreads();
}

// ---- K0: min / max of the images (and NaN) --------------------------------------
__global__ void __launch_bounds__(TF_T) tf_minmax(const void* __restrict__ x, int xd, const void* __restrict__ y,
                                                  int yd, uint32_t n, TfParams* __restrict__ p) {
    uint32_t nxmin = 0, xmax = 0, nymin = 0, ymax = 0;
    int nan = 0;
    const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u) == 0;
    for (uint32_t i = (blockIdx.x * TF_T + threadIdx.x) * 4u; i < n; i += gridDim.x * TF_T * 4u) {
        const uint4 xv = tf_load4(x, i, n, al), yv = tf_load4(y, i, n, al);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i + k >= n) break;
            const uint32_t xr = u4get(xv, k), yr = u4get(yv, k);
            nan |= tf_isnan(xr, xd) | tf_isnan(yr, yd);
            const uint32_t xi = tf_conv(xr, xd), yi = tf_conv(yr, yd);
            nxmin = max(nxmin, ~xi);
            xmax = max(xmax, xi);
            nymin = max(nymin, ~yi);
            ymax = max(ymax, yi);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        nxmin = max(nxmin, __shfl_xor_sync(0xffffffffu, nxmin, o));
        xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
        nymin = max(nymin, __shfl_xor_sync(0xffffffffu, nymin, o));
        ymax = max(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
    }
    nan = __any_sync(0xffffffffu, nan);
    // block reduce, then one atomic per value per block (per-warp atomics on the same four
    // words serialise at L2)
    __shared__ uint32_t red[4][TF_T / 32];
    __shared__ int rnan;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) rnan = 0;
    __syncthreads();
    if (lane == 0) {
        red[0][wid] = nxmin;
        red[1][wid] = xmax;
        red[2][wid] = nymin;
        red[3][wid] = ymax;
        if (nan) rnan = 1;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        uint32_t v = 0;
        for (int k = 0; k < TF_T / 32; ++k) v = max(v, red[threadIdx.x][k]);
        uint32_t* dst = threadIdx.x == 0 ? &p->nxmin : threadIdx.x == 1 ? &p->xmax : threadIdx.x == 2 ? &p->nymin : &p->ymax;
        atomicMax(dst, v);
        if (threadIdx.x == 0 && rnan) atomicOr(&p->nan, 1);
    }
}

// ---- tile-sorted scatter ---------------------------------------------------------------
// One tile of up to TF_ST_TILE keys is counting-sorted by its 12-bit bin in shared memory
// before it is written, so the keys of one bin leave as a contiguous run (a few sectors
// per bin per tile) instead of one 4-byte store per key into 4096 open write fronts (which
// thrashes L2 with partial sectors and multiplies DRAM writes).
constexpr int TF_ST_T = 1024;
constexpr int TF_ST_PER = 16;
constexpr int TF_ST_TILE = TF_ST_T * TF_ST_PER;  // 16K keys
struct TfStSmem {
    uint32_t stage[TF_ST_TILE];
    uint16_t sbin[TF_ST_TILE];
    uint32_t lcnt[TF_BINS];   // tile histogram, then the tile's exclusive starts
    uint32_t lcur[TF_BINS];   // fill cursors
    uint32_t cur[TF_BINS];    // global write cursors of this CTA
    uint32_t sw[32];
};
constexpr size_t TF_ST_SMEM = sizeof(TfStSmem);

// key[k] / bin[k] valid for k with e = k * TF_ST_T + tid < m. `placed()` runs once the
// tile sits in shared memory (key / bin dead): the caller issues the next tile's loads
// there, so they overlap the write-out.
template <typename F>
__device__ __forceinline__ void tf_tile_scatter(TfStSmem& s, const uint32_t (&key)[TF_ST_PER],
                                                const uint32_t (&bin)[TF_ST_PER], int m, uint32_t* __restrict__ out,
                                                F&& placed) {
    constexpr int PER = TF_BINS / TF_ST_T;
    for (int v = threadIdx.x; v < TF_BINS; v += TF_ST_T) s.lcnt[v] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TF_ST_PER; ++k)
        if (k * TF_ST_T + (int)threadIdx.x < m) atomicAdd(&s.lcnt[bin[k]], 1u);
    __syncthreads();
    uint32_t loc[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        loc[k] = sum;
        sum += s.lcnt[threadIdx.x * PER + k];
    }
    const uint32_t base = block_excl_scan<TF_ST_T>(sum, s.sw, nullptr);
    uint32_t cnt[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int v = threadIdx.x * PER + k;
        cnt[k] = s.lcnt[v];
        s.lcnt[v] = base + loc[k];
        s.lcur[v] = base + loc[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TF_ST_PER; ++k) {
        if (k * TF_ST_T + (int)threadIdx.x < m) {
            const uint32_t pos = atomicAdd(&s.lcur[bin[k]], 1u);
            s.stage[pos] = key[k];
            s.sbin[pos] = (uint16_t)bin[k];
        }
    }
    placed();
    __syncthreads();
    for (int e = threadIdx.x; e < m; e += TF_ST_T) {
        const uint32_t b = s.sbin[e];
        out[s.cur[b] + ((uint32_t)e - s.lcnt[b])] = s.stage[e];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) s.cur[threadIdx.x * PER + k] += cnt[k];
    __syncthreads();
}

// ---- K1: level-1 chunk histograms ------------------------------------------------
__global__ void __launch_bounds__(TF_T) tf_count1(const void* __restrict__ x, int xd, uint32_t n, uint32_t ch,
                                                  const TfParams* __restrict__ p, uint32_t* __restrict__ hist) {
    const TfDerived d = tf_derive(p);
    if (!d.ok) return;
    __shared__ uint32_t h[TF_BINS];
    for (int v = threadIdx.x; v < TF_BINS; v += TF_T) h[v] = 0;
    __syncthreads();
    const uint32_t beg = blockIdx.x * ch, end = min(n, beg + ch);
    const bool al = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    for (uint32_t i0 = beg; i0 < end; i0 += TF_T * 4u) {
        const uint32_t i = i0 + threadIdx.x * 4u;
        const uint4 xv = tf_load4(x, i, end, al);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (i + k < end) atomicAdd(&h[tf_digit1(tf_conv(u4get(xv, k), xd), d)], 1u);
    }
    __syncthreads();
    uint32_t* o = hist + (size_t)blockIdx.x * TF_BINS;
    for (int v = threadIdx.x; v < TF_BINS; v += TF_T) o[v] = h[v];
}

// ---- K2: column scan of chunk histograms: pre[r][v] = sum_{r' < r} hist[r'][v] ----
// CTA = 32 bins (one per lane), 8 warps split the rows.
__global__ void __launch_bounds__(256) tf_colscan(const uint32_t* __restrict__ hist, uint32_t rows,
                                                  const TfParams* __restrict__ p, uint32_t* __restrict__ pre,
                                                  uint32_t* __restrict__ tot, unsigned long long* __restrict__ n2) {
    if (!tf_derive(p).ok) return;
    __shared__ uint32_t wt[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t bin = blockIdx.x * 32 + lane;
    const uint32_t rpw = (rows + 7) / 8;
    const uint32_t r0 = min(rows, wid * rpw), r1 = min(rows, r0 + rpw);
    // the warp's rows (<= RMAX at every n: rows ~ one per SM) are loaded once, all at once
    constexpr int RMAX = 24;
    const bool inreg = r1 - r0 <= (uint32_t)RMAX;
    uint32_t vals[RMAX];
    uint32_t s = 0;
    if (inreg) {
#pragma unroll
        for (int k = 0; k < RMAX; ++k) vals[k] = r0 + k < r1 ? hist[(size_t)(r0 + k) * TF_BINS + bin] : 0u;
#pragma unroll
        for (int k = 0; k < RMAX; ++k) s += vals[k];
    } else {
        for (uint32_t r = r0; r < r1; ++r) s += hist[(size_t)r * TF_BINS + bin];
    }
    wt[wid][lane] = s;
    __syncthreads();
    uint32_t run = 0, all = 0;
    for (int k = 0; k < 8; ++k) {
        if (k < wid) run += wt[k][lane];
        all += wt[k][lane];
    }
    if (inreg) {
#pragma unroll
        for (int k = 0; k < RMAX; ++k)
            if (r0 + k < r1) {
                pre[(size_t)(r0 + k) * TF_BINS + bin] = run;
                run += vals[k];
            }
    } else {
        for (uint32_t r = r0; r < r1; ++r) {
            const uint32_t v = hist[(size_t)r * TF_BINS + bin];
            pre[(size_t)r * TF_BINS + bin] = run;
            run += v;
        }
    }
    if (tot && wid == 0) tot[bin] = all;
    if (n2) {
        const unsigned long long c = wid == 0 ? (unsigned long long)all * (all - 1ull) / 2ull : 0ull;
        acc_add(c, n2);
    }
}

// ---- K3: level-1 scatter ---------------------------------------------------------------
__global__ void __launch_bounds__(TF_ST_T, 1) tf_scatter1(const void* __restrict__ x, int xd,
                                                          const void* __restrict__ y, int yd, uint32_t n, uint32_t ch,
                                                          const TfParams* __restrict__ p,
                                                          const uint32_t* __restrict__ pre,
                                                          const uint32_t* __restrict__ tot,
                                                          uint32_t* __restrict__ off1, uint32_t* __restrict__ A) {
    const TfDerived d = tf_derive(p);
    if (!d.ok) return;
    extern __shared__ __align__(16) uint8_t tf_st_raw[];
    TfStSmem& s = *reinterpret_cast<TfStSmem*>(tf_st_raw);
    constexpr int PER = TF_BINS / TF_ST_T;
    uint32_t loc[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        loc[k] = sum;
        sum += tot[threadIdx.x * PER + k];
    }
    const uint32_t base = block_excl_scan<TF_ST_T>(sum, s.sw, nullptr);
    const uint32_t* pr = pre + (size_t)blockIdx.x * TF_BINS;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int v = threadIdx.x * PER + k;
        s.cur[v] = base + loc[k] + pr[v];
        if (blockIdx.x == 0) off1[v] = base + loc[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == TF_ST_T - 1) off1[TF_BINS] = base + sum;
    __syncthreads();
    const uint32_t beg = blockIdx.x * ch, end = min(n, beg + ch);
    // the next tile's raw words are loaded while this tile is written out, so the HBM
    // reads overlap it (one CTA per SM: nothing else would)
    const uint32_t* xw = static_cast<const uint32_t*>(x);
    const uint32_t* yw = static_cast<const uint32_t*>(y);
    uint32_t rx[TF_ST_PER], ry[TF_ST_PER / 2];  // raw x words; y offsets (< 4096) two per register
    auto fetch = [&](uint32_t t0) {
        const int m = (int)min((uint32_t)TF_ST_TILE, end - t0);
#pragma unroll
        for (int k = 0; k < TF_ST_PER; ++k) {
            const int e = k * TF_ST_T + threadIdx.x;
            rx[k] = e < m ? __ldcs(xw + t0 + e) : 0u;
            const uint32_t yo = e < m ? (tf_conv(__ldcs(yw + t0 + e), yd) - d.ymin) & 0xFFFFu : 0u;
            if (k & 1) ry[k >> 1] |= yo << 16; else ry[k >> 1] = yo;
        }
    };
    if (beg < end) fetch(beg);
    for (uint32_t t0 = beg; t0 < end; t0 += TF_ST_TILE) {
        const int m = (int)min((uint32_t)TF_ST_TILE, end - t0);
        uint32_t key[TF_ST_PER], bin[TF_ST_PER];
#pragma unroll
        for (int k = 0; k < TF_ST_PER; ++k) {
            const uint32_t xi = tf_conv(rx[k], xd);
            const uint32_t xr = xi - d.xmin;
            const uint32_t rem = d.r1 ? (xr & ((1u << d.r1) - 1u)) : 0u;
            key[k] = (rem << 12) | ((ry[k >> 1] >> (16 * (k & 1))) & 0xFFFFu);  // == tf_key1(xi, yi, d)
            bin[k] = tf_digit1(xi, d);
        }
        tf_tile_scatter(s, key, bin, m, A, [&] {
            if (t0 + TF_ST_TILE < end) fetch(t0 + TF_ST_TILE);
        });
    }
}

// ---- K4: level-2 plan (one CTA) ----------------------------------------------------
// split[b] = bucket b holds > cap keys with different x; items = its CH2-chunks.
__global__ void __launch_bounds__(TF_SCAN_T) tf_plan2(const TfParams* __restrict__ p,
                                                      const uint32_t* __restrict__ off1, uint32_t cap, uint32_t ch2,
                                                      uint32_t* __restrict__ srank, uint32_t* __restrict__ ibase,
                                                      uint32_t* __restrict__ ng) {
    const TfDerived d = tf_derive(p);
    if (!d.ok) return;
    __shared__ uint32_t sw[32];
    constexpr int PER = TF_BINS / TF_SCAN_T;
    uint32_t sp[PER], it[PER], ssum = 0, isum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = threadIdx.x * PER + k;
        const uint32_t m = off1[b + 1] - off1[b];
        const bool split = m > cap && d.r1 > 0;
        sp[k] = ssum;
        it[k] = isum;
        ssum += split;
        isum += split ? (m + ch2 - 1) / ch2 : 0u;
        ng[b] = (!split && m > 0) ? 1u : 0u;
    }
    uint32_t stot, itot;
    __shared__ uint32_t tots[2];
    const uint32_t sb = block_excl_scan<TF_SCAN_T>(ssum, sw, &tots[0]);
    const uint32_t ib = block_excl_scan<TF_SCAN_T>(isum, sw, &tots[1]);
    stot = tots[0];
    itot = tots[1];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = threadIdx.x * PER + k;
        srank[b] = sb + sp[k];
        ibase[b] = ib + it[k];
    }
    if (threadIdx.x == 0) {
        srank[TF_BINS] = stot;
        ibase[TF_BINS] = itot;
    }
}

__device__ __forceinline__ uint32_t upper_bound_u32(const uint32_t* a, uint32_t n, uint32_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// item -> (bucket, element range)
struct TfItem {
    uint32_t b, beg, end;
};
__device__ __forceinline__ TfItem tf_item(uint32_t item, const uint32_t* ibase, const uint32_t* off1, uint32_t ch2) {
    const uint32_t b = upper_bound_u32(ibase, TF_BINS + 1, item) - 1;  // ibase[b] <= item < ibase[b+1]
    const uint32_t k = item - ibase[b];
    const uint32_t beg = off1[b] + k * ch2;
    return TfItem{b, beg, min(off1[b + 1], beg + ch2)};
}

// ---- K5: level-2 chunk histograms ------------------------------------------------
__global__ void __launch_bounds__(TF_T) tf_count2(const TfParams* __restrict__ p, const uint32_t* __restrict__ off1,
                                                  const uint32_t* __restrict__ ibase, uint32_t ch2,
                                                  const uint32_t* __restrict__ A, uint32_t* __restrict__ hist2) {
    const TfDerived d = tf_derive(p);
    if (!d.ok) return;
    __shared__ uint32_t h[TF_BINS];
    const uint32_t items = ibase[TF_BINS];
    const uint32_t sh = 12 + d.r2;
    for (uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
        const TfItem it = tf_item(item, ibase, off1, ch2);
        for (int v = threadIdx.x; v < TF_BINS; v += TF_T) h[v] = 0;
        __syncthreads();
        for (uint32_t i = it.beg + threadIdx.x; i < it.end; i += TF_T) atomicAdd(&h[A[i] >> sh], 1u);
        __syncthreads();
        uint32_t* o = hist2 + (size_t)item * TF_BINS;
        for (int v = threadIdx.x; v < TF_BINS; v += TF_T) o[v] = h[v];
        __syncthreads();
    }
}

// Children of split bucket b: totals ct[] and exclusive starts cs[] (relative), then
// group heads. A child c (nonempty) starts a group if it is the first nonempty child, if
// it is big (> T = cap/2 keys), if the previous nonempty child is big, or if its start
// lies in a different T-window than the previous nonempty child's start: so a group of
// small children spans < 2T = cap keys, and a big child is a group of its own.
struct TfChildSmem {
    uint32_t ct[TF_BINS];
    uint32_t cs[TF_BINS];
    uint32_t gsr[TF_BINS];  // group starts by head rank (tf_groups)
    uint32_t sw[32];
    int iw[32];
    uint32_t tot;
};
constexpr size_t TF_CHILD_SMEM = sizeof(TfChildSmem);

// Fills cs for the ct already in smem; returns (per thread) the head flags of its PER
// children as a bitmask.
__device__ __forceinline__ uint32_t tf_child_heads(TfChildSmem& s, uint32_t T) {
    constexpr int PER = TF_BINS / TF_SCAN_T;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t loc[PER], sum = 0;
    int lastne = -1;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int c = threadIdx.x * PER + k;
        loc[k] = sum;
        sum += s.ct[c];
        if (s.ct[c]) lastne = c;
    }
    const uint32_t base = block_excl_scan<TF_SCAN_T>(sum, s.sw, &s.tot);
#pragma unroll
    for (int k = 0; k < PER; ++k) s.cs[threadIdx.x * PER + k] = base + loc[k];
    // carry = last nonempty child of the earlier threads (exclusive max-scan)
    int x = lastne;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, yv);
    }
    if (lane == 31) s.iw[wid] = x;
    __syncthreads();
    int carry = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) carry = -1;
    for (int k = 0; k < wid; ++k) carry = max(carry, s.iw[k]);
    uint32_t heads = 0;
    int pc = carry;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int c = threadIdx.x * PER + k;
        if (!s.ct[c]) continue;
        const bool h = pc < 0 || s.ct[c] > T || s.ct[pc] > T || (s.cs[c] / T) != (s.cs[pc] / T);
        heads |= (uint32_t)h << k;
        pc = c;
    }
    __syncthreads();
    return heads;
}

// ---- K6: level-2 column scan + child totals + group count, one CTA per bucket ----
__global__ void __launch_bounds__(TF_SCAN_T) tf_scan2(const TfParams* __restrict__ p,
                                                      const uint32_t* __restrict__ off1,
                                                      const uint32_t* __restrict__ ibase,
                                                      const uint32_t* __restrict__ srank, uint32_t cap,
                                                      const uint32_t* __restrict__ hist2, uint32_t* __restrict__ pre2,
                                                      uint32_t* __restrict__ ctot, uint32_t* __restrict__ ng,
                                                      TfParams* __restrict__ pw) {
    const TfDerived d = tf_derive(p);
    if (!d.ok || blockIdx.x >= srank[TF_BINS]) return;
    const uint32_t b = upper_bound_u32(srank, TF_BINS + 1, blockIdx.x) - 1;  // the CTA's split bucket
    extern __shared__ __align__(16) uint8_t tf_child_raw[];
    TfChildSmem& s = *reinterpret_cast<TfChildSmem*>(tf_child_raw);
    constexpr int PER = TF_BINS / TF_SCAN_T;
    const uint32_t i0 = ibase[b], i1 = ibase[b + 1];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int v = threadIdx.x + k * TF_SCAN_T;
        uint32_t run = 0;
        for (uint32_t it = i0; it < i1; ++it) run += hist2[(size_t)it * TF_BINS + v];
        s.ct[v] = run;
    }
    __syncthreads();
    const uint32_t heads = tf_child_heads(s, cap / 2);
    // absolute scatter cursors per item
    const uint32_t o1 = off1[b];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int v = threadIdx.x + k * TF_SCAN_T;
        uint32_t run = o1 + s.cs[v];
        for (uint32_t it = i0; it < i1; ++it) {
            const size_t idx = (size_t)it * TF_BINS + v;
            const uint32_t h = hist2[idx];
            pre2[idx] = run;
            run += h;
        }
        ctot[(size_t)srank[b] * TF_BINS + v] = s.ct[v];
    }
    __shared__ uint32_t hc;
    if (threadIdx.x == 0) hc = 0;
    __syncthreads();
    atomicAdd(&hc, (uint32_t)__popc(heads));
    __syncthreads();
    if (threadIdx.x == 0) ng[b] = hc;
}

// ---- K7: level-2 scatter (A -> B, same positions space) -----------------------------
__global__ void __launch_bounds__(TF_ST_T, 1) tf_scatter2(const TfParams* __restrict__ p,
                                                          const uint32_t* __restrict__ off1,
                                                          const uint32_t* __restrict__ ibase, uint32_t ch2,
                                                          const uint32_t* __restrict__ pre2,
                                                          const uint32_t* __restrict__ A, uint32_t* __restrict__ B) {
    const TfDerived d = tf_derive(p);
    if (!d.ok) return;
    extern __shared__ __align__(16) uint8_t tf_st_raw[];
    TfStSmem& s = *reinterpret_cast<TfStSmem*>(tf_st_raw);
    const uint32_t items = ibase[TF_BINS];
    const uint32_t sh = 12 + d.r2;
    for (uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
        const TfItem it = tf_item(item, ibase, off1, ch2);
        const uint32_t* pr = pre2 + (size_t)item * TF_BINS;
        for (int v = threadIdx.x; v < TF_BINS; v += TF_ST_T) s.cur[v] = pr[v];
        __syncthreads();
        uint32_t raw[TF_ST_PER];
        auto fetch = [&](uint32_t t0) {
            const int m = (int)min((uint32_t)TF_ST_TILE, it.end - t0);
#pragma unroll
            for (int k = 0; k < TF_ST_PER; ++k) {
                const int e = k * TF_ST_T + threadIdx.x;
                raw[k] = e < m ? __ldcs(A + t0 + e) : 0u;
            }
        };
        if (it.beg < it.end) fetch(it.beg);
        for (uint32_t t0 = it.beg; t0 < it.end; t0 += TF_ST_TILE) {
            const int m = (int)min((uint32_t)TF_ST_TILE, it.end - t0);
            uint32_t key[TF_ST_PER], bin[TF_ST_PER];
#pragma unroll
            for (int k = 0; k < TF_ST_PER; ++k) {
                key[k] = raw[k];
                bin[k] = key[k] >> sh;
            }
            tf_tile_scatter(s, key, bin, m, B, [&] {
                if (t0 + TF_ST_TILE < it.end) fetch(t0 + TF_ST_TILE);
            });
        }
    }
}

// Group record: start, len, flags (bit0: keys in B, bit1: single x, bit2: a crowded
// level-2 child: > cap keys over at most 2^r2 distinct x).
struct TfGroup {
    uint32_t start, len, flags, pad;
};

// ---- K8a: group bases (one CTA): exclusive scan of the per-bucket group counts; the
// unsplit buckets' single groups are written here --------------------------------------
__global__ void __launch_bounds__(TF_SCAN_T) tf_gscan(const TfParams* __restrict__ p,
                                                      const uint32_t* __restrict__ off1,
                                                      const uint32_t* __restrict__ srank,
                                                      const uint32_t* __restrict__ ng, uint32_t* __restrict__ gbase,
                                                      TfGroup* __restrict__ groups, uint32_t* __restrict__ gstart,
                                                      TfParams* __restrict__ pw) {
    const TfDerived d = tf_derive(p);
    if (!d.ok) return;
    __shared__ uint32_t sw[32], tot;
    constexpr int PER = TF_BINS / TF_SCAN_T;
    uint32_t loc[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        loc[k] = sum;
        sum += ng[threadIdx.x * PER + k];
    }
    const uint32_t base = block_excl_scan<TF_SCAN_T>(sum, sw, &tot);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int b = threadIdx.x * PER + k;
        const uint32_t g = base + loc[k];
        gbase[b] = g;
        const uint32_t m = off1[b + 1] - off1[b];
        if (m && srank[b + 1] == srank[b]) {  // unsplit: one group in A
            groups[g] = TfGroup{off1[b], m, d.r1 == 0 ? 2u : 0u, 0u};
            gstart[g] = off1[b];
        }
    }
    if (threadIdx.x == 0) pw->ngroups = (int)tot;
}

// ---- K8b: the groups of each split bucket (one CTA per split bucket) ------------------
__global__ void __launch_bounds__(TF_SCAN_T) tf_groups(const TfParams* __restrict__ p,
                                                       const uint32_t* __restrict__ off1,
                                                       const uint32_t* __restrict__ srank, uint32_t cap,
                                                       const uint32_t* __restrict__ ctot, const uint32_t* __restrict__ ng,
                                                       const uint32_t* __restrict__ gbase,
                                                       TfGroup* __restrict__ groups, uint32_t* __restrict__ gstart) {
    const TfDerived d = tf_derive(p);
    if (!d.ok || blockIdx.x >= srank[TF_BINS]) return;
    const uint32_t b = upper_bound_u32(srank, TF_BINS + 1, blockIdx.x) - 1;
    extern __shared__ __align__(16) uint8_t tf_child_raw[];
    TfChildSmem& s = *reinterpret_cast<TfChildSmem*>(tf_child_raw);
    const uint32_t g0 = gbase[b];
    const uint32_t m = off1[b + 1] - off1[b];
    constexpr int PER = TF_BINS / TF_SCAN_T;
    const uint32_t* ct = ctot + (size_t)blockIdx.x * TF_BINS;
#pragma unroll
    for (int k = 0; k < PER; ++k) s.ct[threadIdx.x * PER + k] = ct[threadIdx.x * PER + k];
    __syncthreads();
    const uint32_t heads = tf_child_heads(s, cap / 2);
    __shared__ uint32_t sw2[32];
    const uint32_t hb = block_excl_scan<TF_SCAN_T>((uint32_t)__popc(heads), sw2, nullptr);
    // group starts (relative) by head rank, then lengths from the next start
    uint32_t* gs_rel = s.gsr;
    uint32_t r = hb;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        if (heads >> k & 1u) gs_rel[r++] = s.cs[threadIdx.x * PER + k];
    }
    __syncthreads();
    const uint32_t nh = ng[b];
    r = hb;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        if (!(heads >> k & 1u)) continue;
        const int c = threadIdx.x * PER + k;
        const uint32_t st = gs_rel[r];
        const uint32_t en = (r + 1 < nh) ? gs_rel[r + 1] : m;
        const uint32_t len = en - st;
        // one child (exactly its keys): single x when level 2 leaves no x bits; a child
        // too big to sort that still has r2 x bits is walked value by value (bit 2)
        const bool one_child = len == s.ct[c];
        uint32_t fl = 1u;
        if (one_child && d.r2 == 0) fl |= 2u;
        else if (one_child && len > cap) fl |= 4u;
        groups[g0 + r] = TfGroup{off1[b] + st, len, fl, 0u};
        gstart[g0 + r] = off1[b] + st;
        ++r;
    }
}

// ---- K9: the leaf walk -------------------------------------------------------------
// one pad word per IT keys (the per-thread runs of IT consecutive keys start in different banks)
template <int IT>
__device__ __forceinline__ int tf_pidx(int e) { return e + (e >> (IT == 16 ? 4 : 3)); }

// CTA merge sort of mp (a multiple of 16, <= TF_CAP) u32 keys in padded smem; threads
// t < mp/16 own 16 consecutive outputs. Stable; with Count, returns the number of
// strict inversions (pairs i < j with key_i > key_j) seen by this thread.
template <bool Count, int IT>
__device__ __forceinline__ unsigned long long tf_sort(uint32_t* sk, int mp, uint32_t (&r)[IT]) {
    const int t = threadIdx.x;
    const bool act = t < mp / IT;
    unsigned long long inv = 0;
    if (act) {
#pragma unroll
        for (int k = 0; k < IT; ++k) r[k] = sk[tf_pidx<IT>(t * IT + k)];
#pragma unroll
        for (int rd = 0; rd < IT; ++rd) {
#pragma unroll
            for (int k = (rd & 1); k + 1 < IT; k += 2) {
                const uint32_t a = r[k], b = r[k + 1];
                const bool sw = b < a;
                r[k] = sw ? b : a;
                r[k + 1] = sw ? a : b;
                if (Count) inv += sw;
            }
        }
    }
    // A warp's threads own 32 * IT consecutive positions, so while both runs of a
    // merge lie inside one warp's range (2w <= 32 * IT) a warp barrier suffices.
    constexpr int WSPAN = 32 * IT;
    if (2 * IT <= WSPAN) __syncwarp(); else __syncthreads();
    if (act) {
#pragma unroll
        for (int k = 0; k < IT; ++k) sk[tf_pidx<IT>(t * IT + k)] = r[k];
    }
    if (2 * IT <= WSPAN) __syncwarp(); else __syncthreads();
    for (int w = IT; w < mp; w <<= 1) {
        if (act) {
            // runs [pb, pb + la) and [pb + w, pb + w + lb), clipped at mp (any multiple of 16)
            const int pos = t * IT;
            const int pb = pos & ~(2 * w - 1);
            const int diag = pos - pb;
            const int a0 = pb, b0 = pb + w;
            const int la = min(w, mp - pb), lb = max(0, min(w, mp - b0));
            int lo = max(0, diag - lb), hi = min(diag, la);
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (!(sk[tf_pidx<IT>(b0 + diag - 1 - mid)] < sk[tf_pidx<IT>(a0 + mid)])) lo = mid + 1; else hi = mid;
            }
            // branch-free serial merge of this thread's 16 outputs: the consumed side is
            // reloaded from a clamped index (an exhausted run's head is never taken)
            int i = lo, j = diag - lo;
            uint32_t ka = sk[tf_pidx<IT>(a0 + min(i, la - 1))];  // la >= IT
            uint32_t kb = sk[tf_pidx<IT>(lb > 0 ? b0 + min(j, lb - 1) : a0)];
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const bool take_b = j < lb && (i >= la || kb < ka);
                r[k] = take_b ? kb : ka;
                if (Count) inv += take_b ? (unsigned long long)(la - i) : 0ull;
                i += take_b ? 0 : 1;
                j += take_b ? 1 : 0;
                const int nx = take_b ? b0 + min(j, lb - 1) : a0 + min(i, la - 1);
                const uint32_t v = sk[tf_pidx<IT>(nx)];
                ka = take_b ? ka : v;
                kb = take_b ? v : kb;
            }
        }
        // the next level (width 2w) reads runs of this one: warp-local while 4w <= WSPAN
        if (2 * w <= WSPAN) __syncwarp(); else __syncthreads();
        if (act) {
#pragma unroll
            for (int k = 0; k < IT; ++k) sk[tf_pidx<IT>(t * IT + k)] = r[k];
        }
        if (4 * w <= WSPAN) __syncwarp(); else __syncthreads();
    }
    __syncthreads();  // the callers read the sorted keys across warps
    return inv;
}

// gt[v] = #items in hist with y offset > v (suffix sums), TF_LEAF_T threads x 8 bins.
__device__ __forceinline__ void tf_suffix(const uint32_t* hist, uint32_t* gt, uint32_t* sw) {
    constexpr int PER = TF_BINS / TF_LEAF_T;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t loc[PER], acc = 0;
#pragma unroll
    for (int k = PER - 1; k >= 0; --k) {
        loc[k] = acc;
        acc += hist[threadIdx.x * PER + k];
    }
    uint32_t x = acc;  // inclusive suffix over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yv = __shfl_down_sync(0xffffffffu, x, o);
        if (lane + o < 32) x += yv;
    }
    if (lane == 0) sw[wid] = x;
    __syncthreads();
    uint32_t above = x - acc;
    for (int k = wid + 1; k < TF_LEAF_T / 32; ++k) above += sw[k];
#pragma unroll
    for (int k = 0; k < PER; ++k) gt[threadIdx.x * PER + k] = loc[k] + above;
    __syncthreads();
}

// Inclusive block max-scan of per-thread values (run-start positions).
__device__ __forceinline__ int tf_excl_max(int v, int* sw) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = max(x, yv);
    }
    if (lane == 31) sw[wid] = x;
    __syncthreads();
    int carry = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) carry = -1;
    for (int k = 0; k < wid; ++k) carry = max(carry, sw[k]);
    __syncthreads();
    return carry;  // max over all earlier threads
}

constexpr size_t TF_LEAF_SMEM = (size_t)(TF_CAP + TF_CAP / 16) * 4 + 2 * TF_BINS * 4;

template <int IT>
__global__ void __launch_bounds__(TF_LEAF_T, 2) tf_leaf(const TfParams* __restrict__ p, uint32_t n,
                                                        const TfGroup* __restrict__ groups,
                                                        const uint32_t* __restrict__ gstart,
                                                        const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                                                        uint32_t* __restrict__ hc, unsigned long long* __restrict__ acc) {
    const TfDerived d = tf_derive(p);
    if (!d.ok || p->fail) return;
    extern __shared__ __align__(16) uint32_t tf_sm[];
    uint32_t* sk = tf_sm;                                  // TF_CAP + pad
    uint32_t* hist = sk + TF_CAP + TF_CAP / 16;             // running y histogram of this CTA
    uint32_t* gt = hist + TF_BINS;                          // suffix sums
    __shared__ uint32_t sw[32];
    __shared__ int swi[32];
    __shared__ uint32_t s_g[2];
    // CTA ranges balance keys + a fixed per-group cost: group g sits at the "position"
    // start(g) + g * TF_GROUP_COST, which increases with g (runs of tiny groups, e.g. the
    // tails of a normal sample, would otherwise all land on one CTA)
    const uint32_t G = (uint32_t)p->ngroups;
    const uint64_t total = (uint64_t)n + (uint64_t)G * TF_GROUP_COST;
    const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
    if (threadIdx.x < 2) {
        const uint64_t lim = (uint64_t)(blockIdx.x + threadIdx.x) * per;
        uint32_t lo = 0, hi = G;  // first group with weighted position >= lim
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((uint64_t)gstart[mid] + (uint64_t)mid * TF_GROUP_COST < lim) lo = mid + 1; else hi = mid;
        }
        s_g[threadIdx.x] = (blockIdx.x + threadIdx.x == gridDim.x) ? G : lo;
    }
    for (int v = threadIdx.x; v < TF_BINS; v += TF_LEAF_T) hist[v] = 0;
    __syncthreads();
    const uint32_t g0 = s_g[0], g1 = s_g[1];
    unsigned long long D = 0, n1 = 0, n3 = 0;
    for (uint32_t g = g0; g < g1; ++g) {
        const TfGroup gr = groups[g];
        const uint32_t m = gr.len;
        const uint32_t* src = ((gr.flags & 1u) ? B : A) + gr.start;
        tf_suffix(hist, gt, sw);  // items of earlier groups with larger y
        if (gr.flags & 6u) {
            // single x (bit 1), or a crowded child (bit 2) walked one x value at a time;
            // no discordant pairs among equal x: count ties from each value's y histogram
            uint32_t* lh = sk;
            uint32_t* present = sk + TF_BINS;  // 256-bit set of the x values present
            const uint32_t xmask = (gr.flags & 4u) ? ((1u << d.r2) - 1u) : 0u;
            if (threadIdx.x < 10) present[threadIdx.x] = 0;  // [0, 8): the set, [9]: a count
            __syncthreads();
            if (xmask) {
                for (uint32_t e = threadIdx.x; e < m; e += TF_LEAF_T) {
                    const uint32_t xv = (src[e] >> 12) & xmask;
                    atomicOr(&present[xv >> 5], 1u << (xv & 31));
                }
            } else if (threadIdx.x == 0) {
                present[0] = 1u;
            }
            __syncthreads();
            int nval = 0;
            for (int k = 0; k < 8; ++k) nval += __popc(present[k]);
            if (nval > 16) {  // adversarial concentration: leave it to the general path
                if (threadIdx.x == 0) atomicOr(&const_cast<TfParams*>(p)->fail, 1);
                break;
            }
            uint32_t first = 0;
            for (int k = 7; k >= 0; --k)
                if (present[k]) first = (uint32_t)k * 32u + (uint32_t)(__ffs(present[k]) - 1);
            for (int k = 0; k < 8; ++k) {
                uint32_t bits = present[k];
                while (bits) {
                    const uint32_t xv = (uint32_t)k * 32u + (uint32_t)(__ffs(bits) - 1);
                    bits &= bits - 1;
                    if (xv != first) tf_suffix(hist, gt, sw);
                    for (int v = threadIdx.x; v < TF_BINS; v += TF_LEAF_T) lh[v] = 0;
                    __syncthreads();
                    uint32_t cnt = 0;
                    for (uint32_t e = threadIdx.x; e < m; e += TF_LEAF_T) {
                        const uint32_t key = src[e];
                        if (((key >> 12) & xmask) != xv) continue;
                        const uint32_t yv = key & 4095u;
                        D += gt[yv];
                        ++cnt;
                        atomicAdd(&lh[yv], 1u);
                    }
                    __syncthreads();
                    for (int v = threadIdx.x; v < TF_BINS; v += TF_LEAF_T) {
                        const uint32_t c = lh[v];
                        n3 += (unsigned long long)c * (c - 1ull) / 2ull;
                        hist[v] += c;
                    }
                    __syncthreads();
                    // n1: pairs of this x value
                    cnt = __reduce_add_sync(0xffffffffu, cnt);
                    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&present[9], cnt);
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        const unsigned long long c = present[9];
                        n1 += c * (c - 1ull) / 2ull;
                        present[9] = 0;
                    }
                    __syncthreads();
                }
            }
            continue;
        }
        const int mp = ((int)m + IT - 1) / IT * IT;
        for (int e = threadIdx.x; e < mp; e += TF_LEAF_T) sk[tf_pidx<IT>(e)] = e < (int)m ? src[e] : 0xffffffffu;
        __syncthreads();
        uint32_t r[IT];
        tf_sort<false, IT>(sk, mp, r);  // by (x_rem, y)
        // tied runs in x (key >> 12) and in (x, y) (key); cross term; histogram update
        const int t = threadIdx.x;
        const bool act = t < mp / IT;
        int hx = -1, hk = -1;  // last run head (position) inside this thread
        uint32_t prevk = 0;
        if (act && t > 0) prevk = sk[tf_pidx<IT>(t * IT - 1)];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int pos = t * IT + k;
            const uint32_t key = r[k];
            const uint32_t pk = k ? r[k - 1] : prevk;
            if (act && (pos == 0 || (key >> 12) != (pk >> 12))) hx = pos;
            if (act && (pos == 0 || key != pk)) hk = pos;
        }
        hx = tf_excl_max(act ? hx : -1, swi);
        hk = tf_excl_max(act ? hk : -1, swi);
        if (act) {
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int pos = t * IT + k;
                const uint32_t key = r[k];
                const uint32_t pk = k ? r[k - 1] : prevk;
                if (pos == 0 || (key >> 12) != (pk >> 12)) hx = pos;
                if (pos == 0 || key != pk) hk = pos;
                if (pos < (int)m) {
                    n1 += (unsigned long long)(pos - hx);
                    n3 += (unsigned long long)(pos - hk);
                    const uint32_t yv = key & 4095u;
                    D += gt[yv];
                    atomicAdd(&hist[yv], 1u);
                }
            }
        }
        __syncthreads();
        // in-group D = strict inversions of the y sequence in (x, y) order
        if (act) {
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int pos = t * IT + k;
                sk[tf_pidx<IT>(pos)] = pos < (int)m ? (r[k] & 4095u) : 0xffffffffu;
            }
        }
        __syncthreads();
        D += tf_sort<true, IT>(sk, mp, r);
    }
    acc_add(D, acc + 0);
    acc_add(n1, acc + 1);
    acc_add(n3, acc + 3);
    uint32_t* o = hc + (size_t)blockIdx.x * TF_BINS;
    for (int v = threadIdx.x; v < TF_BINS; v += TF_LEAF_T) o[v] = hist[v];
}

// ---- K10: discordant pairs between CTA runs ----------------------------------------
// D += sum_c sum_b H_c[b] * #{items of earlier CTAs with y > b}; pre = column prefix.
__global__ void __launch_bounds__(TF_LEAF_T) tf_cross(const TfParams* __restrict__ p, const uint32_t* __restrict__ hc,
                                                      const uint32_t* __restrict__ pre,
                                                      unsigned long long* __restrict__ acc) {
    const TfDerived d = tf_derive(p);
    if (!d.ok || p->fail) return;
    __shared__ uint32_t gt[TF_BINS];
    __shared__ uint32_t sw[32];
    tf_suffix(pre + (size_t)blockIdx.x * TF_BINS, gt, sw);
    const uint32_t* h = hc + (size_t)blockIdx.x * TF_BINS;
    unsigned long long s = 0;
    for (int v = threadIdx.x; v < TF_BINS; v += TF_LEAF_T) s += (unsigned long long)h[v] * gt[v];
    acc_add(s, acc + 4);
}

// counts = {C, D, n1, n2, n3, status}: status 1 = NaN seen, 2 = needs the general path
__global__ void tf_finish(const TfParams* __restrict__ p, const unsigned long long* __restrict__ acc, uint64_t n,
                          const int* __restrict__ nan_flag, int64_t* __restrict__ counts) {
    const TfDerived d = tf_derive(p);
    const long long n0 = (long long)(n * (n - 1) / 2);
    const long long D = (long long)(acc[0] + acc[4]), n1 = (long long)acc[1], n2 = (long long)acc[2],
                    n3 = (long long)acc[3];
    counts[0] = n0 - n1 - n2 + n3 - D;
    counts[1] = D;
    counts[2] = n1;
    counts[3] = n2;
    counts[4] = n3;
    const bool nan = p->nan || (nan_flag && *nan_flag);
    counts[5] = nan ? 1 : ((!d.ok || p->fail) ? 2 : 0);
}

// ---- host side -------------------------------------------------------------------
struct TfSizes {
    uint32_t cap, ch1, nch1, ch2, max_items, max_split, max_groups, leaf_ctas;
};
static TfSizes tf_sizes(uint64_t n) {
    TfSizes z;
    const uint32_t sms = (uint32_t)num_sms();
    z.leaf_ctas = 2 * sms;
    // sortable groups of <= cap keys. Measured (RS_TAU_CAP sweep on B200, 64M rows): 1024
    // -> 13.7 ms of leaf walk, 2048 -> 8.0, 4096 -> 4.9, 8192 -> 3.3: each group is a
    // chain of barrier-separated merge levels, so fewer, larger groups win
    uint64_t cap = TF_CAP;
    if (const char* e = getenv("RS_TAU_CAP")) cap = strtoull(e, nullptr, 10);
    if (cap > n / z.leaf_ctas) cap = n / z.leaf_ctas;
    cap = cap < 1024 ? 1024 : (cap > TF_CAP ? TF_CAP : cap);
    z.cap = (uint32_t)cap;
    uint64_t ch1 = (n + sms - 1) / sms;  // one wave of the (one CTA per SM) tile-sorted scatter
    ch1 = ch1 < 8192 ? 8192 : (ch1 + 511) / 512 * 512;
    z.ch1 = (uint32_t)ch1;
    z.nch1 = (uint32_t)((n + ch1 - 1) / ch1);
    // level-2 items: about one per leaf CTA, so each child receives long runs per item
    // (short runs from many items make the scatter's partial-sector writes thrash L2)
    uint64_t ch2 = 4096;
    while (ch2 < (1u << 20) && ch2 * 2 * sms < n) ch2 <<= 1;
    z.ch2 = (uint32_t)ch2;
    const uint64_t split = std::min<uint64_t>(TF_BINS, n / z.cap + 1);
    z.max_split = (uint32_t)split;
    z.max_items = (uint32_t)(n / z.ch2 + split + 1);
    z.max_groups = (uint32_t)(TF_BINS + 2 * (n / (z.cap / 2)) + split + 2);
    return z;
}

struct TfWs {
    TfParams* p;
    unsigned long long* acc;
    uint32_t *hist1, *pre1, *tot1, *off1, *srank, *ibase, *ng, *gbase, *hist2, *pre2, *ctot, *gstart, *hc, *prec;
    TfGroup* groups;
};
template <typename Ar>
static void tf_layout(Ar& a, uint64_t n, TfWs* w) {
    const TfSizes z = tf_sizes(n);
    TfWs t;
    t.p = a.template take<TfParams>(1);
    t.acc = a.template take<unsigned long long>(8);
    t.hist1 = a.template take<uint32_t>((size_t)z.nch1 * TF_BINS);
    t.pre1 = a.template take<uint32_t>((size_t)z.nch1 * TF_BINS);
    t.tot1 = a.template take<uint32_t>(TF_BINS);
    t.off1 = a.template take<uint32_t>(TF_BINS + 1);
    t.srank = a.template take<uint32_t>(TF_BINS + 1);
    t.ibase = a.template take<uint32_t>(TF_BINS + 1);
    t.ng = a.template take<uint32_t>(TF_BINS);
    t.gbase = a.template take<uint32_t>(TF_BINS);
    t.hist2 = a.template take<uint32_t>((size_t)z.max_items * TF_BINS);
    t.pre2 = a.template take<uint32_t>((size_t)z.max_items * TF_BINS);
    t.ctot = a.template take<uint32_t>((size_t)z.max_split * TF_BINS);
    t.groups = a.template take<TfGroup>(z.max_groups);
    t.gstart = a.template take<uint32_t>(z.max_groups);
    t.hc = a.template take<uint32_t>((size_t)z.leaf_ctas * TF_BINS);
    t.prec = a.template take<uint32_t>((size_t)z.leaf_ctas * TF_BINS);
    if (w) *w = t;
}
struct TfSizer {
    ArenaSizer s;
    template <typename T>
    T* take(size_t c) { s.take<T>(c); return nullptr; }
};

size_t tau_fast_workspace(uint64_t n) {
    TfSizer a;
    tf_layout(a, n, nullptr);
    return a.s.used + 256;
}

int tau_fast_counts(const void* x, int xd, const void* y, int yd, uint32_t n, int64_t* counts, uint32_t* A,
                    uint32_t* B, const int* nan_flag, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < tau_fast_workspace(n)) {
        set_error("tau fast path: workspace %zu < %zu", ws_bytes, tau_fast_workspace(n));
        return RS_ERR_WORKSPACE;
    }
    Arena ar(ws, ws_bytes);
    TfWs w;
    tf_layout(ar, n, &w);
    const TfSizes z = tf_sizes(n);
    const int sms = num_sms();
    RS_CUDA(cudaMemsetAsync(w.p, 0, sizeof(TfParams), st));
    RS_CUDA(cudaMemsetAsync(w.acc, 0, 8 * sizeof(unsigned long long), st));
    {
        const uint32_t g = std::min<uint32_t>((n / 4 + TF_T) / TF_T, (uint32_t)sms * 2);
        tf_minmax<<<g, TF_T, 0, st>>>(x, xd, y, yd, n, w.p);
        RS_LAUNCH_CHECK();
    }
    tf_count1<<<z.nch1, TF_T, 0, st>>>(x, xd, n, z.ch1, w.p, w.hist1);
    RS_LAUNCH_CHECK();
    tf_colscan<<<TF_BINS / 32, 256, 0, st>>>(w.hist1, z.nch1, w.p, w.pre1, w.tot1, nullptr);
    RS_LAUNCH_CHECK();
    RS_CUDA(ensure_smem((const void*)tf_scatter1, (int)TF_ST_SMEM));
    RS_CUDA(ensure_smem((const void*)tf_scatter2, (int)TF_ST_SMEM));
    tf_scatter1<<<z.nch1, TF_ST_T, TF_ST_SMEM, st>>>(x, xd, y, yd, n, z.ch1, w.p, w.pre1, w.tot1, w.off1, A);
    RS_LAUNCH_CHECK();
    tf_plan2<<<1, TF_SCAN_T, 0, st>>>(w.p, w.off1, z.cap, z.ch2, w.srank, w.ibase, w.ng);
    RS_LAUNCH_CHECK();
    const uint32_t g2 = std::min<uint32_t>(z.max_items, (uint32_t)sms * 4);
    tf_count2<<<g2, TF_T, 0, st>>>(w.p, w.off1, w.ibase, z.ch2, A, w.hist2);
    RS_LAUNCH_CHECK();
    RS_CUDA(ensure_smem((const void*)tf_scan2, (int)TF_CHILD_SMEM));
    RS_CUDA(ensure_smem((const void*)tf_groups, (int)TF_CHILD_SMEM));
    tf_scan2<<<z.max_split, TF_SCAN_T, TF_CHILD_SMEM, st>>>(w.p, w.off1, w.ibase, w.srank, z.cap, w.hist2, w.pre2, w.ctot, w.ng, w.p);
    RS_LAUNCH_CHECK();
    tf_scatter2<<<std::min<uint32_t>(z.max_items, (uint32_t)sms), TF_ST_T, TF_ST_SMEM, st>>>(w.p, w.off1, w.ibase, z.ch2,
                                                                                        w.pre2, A, B);
    RS_LAUNCH_CHECK();
    tf_gscan<<<1, TF_SCAN_T, 0, st>>>(w.p, w.off1, w.srank, w.ng, w.gbase, w.groups, w.gstart, w.p);
    RS_LAUNCH_CHECK();
    tf_groups<<<z.max_split, TF_SCAN_T, TF_CHILD_SMEM, st>>>(w.p, w.off1, w.srank, z.cap, w.ctot, w.ng, w.gbase,
                                                             w.groups, w.gstart);
    RS_LAUNCH_CHECK();
    RS_CUDA(ensure_smem((const void*)tf_leaf<8>, (int)TF_LEAF_SMEM));
    RS_CUDA(ensure_smem((const void*)tf_leaf<16>, (int)TF_LEAF_SMEM));
    // groups of <= 4096 keys (the smaller queues): 8 keys per thread, so twice the threads
    // share each merge (half the serial merge steps per level, one level more)
    if (z.cap <= TF_CAP / 2)
        tf_leaf<8><<<z.leaf_ctas, TF_LEAF_T, TF_LEAF_SMEM, st>>>(w.p, n, w.groups, w.gstart, A, B, w.hc, w.acc);
    else
        tf_leaf<16><<<z.leaf_ctas, TF_LEAF_T, TF_LEAF_SMEM, st>>>(w.p, n, w.groups, w.gstart, A, B, w.hc, w.acc);
    RS_LAUNCH_CHECK();
    tf_colscan<<<TF_BINS / 32, 256, 0, st>>>(w.hc, z.leaf_ctas, w.p, w.prec, nullptr, w.acc + 2);
    RS_LAUNCH_CHECK();
    tf_cross<<<z.leaf_ctas, TF_LEAF_T, 0, st>>>(w.p, w.hc, w.prec, w.acc);
    RS_LAUNCH_CHECK();
    tf_finish<<<1, 1, 0, st>>>(w.p, w.acc, n, nan_flag, counts);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs
