// Stable merge sort on the device, optionally counting strict inversions.
//
// Tiles of 2048 keys (256 threads x 8) are sorted in shared memory (odd-even
// transposition in registers, then merge-path merges in smem); then log2(n/2048)
// global merge passes, each CTA producing one 2048-key output tile from a merge-path
// partition of its run pair staged through shared memory.
//
// Inversion counting (pairs i<j with key_i > key_j) rides along for free: a
// transposition swap removes exactly one inversion, and in a stable merge every
// element taken from the right run passes exactly the still-unconsumed elements of
// the left run (all strictly greater). Used for Kendall tau's discordant pairs
// (Knight's algorithm; ranking.py:45-50 counts the same pairs by an O(n^2) row loop).
#pragma once
#include "common.cuh"

namespace rs {

constexpr int MS_THREADS = 256;
constexpr int MS_ITEMS = 8;
constexpr int MS_TILE = MS_THREADS * MS_ITEMS;

template <typename K>
struct KeyTraits;
template <>
struct KeyTraits<uint32_t> {
    static __device__ __forceinline__ uint32_t sentinel() { return 0xffffffffu; }
    static __device__ __forceinline__ bool less(uint32_t a, uint32_t b) { return a < b; }
};
template <>
struct KeyTraits<uint64_t> {
    static __device__ __forceinline__ uint64_t sentinel() { return ~0ull; }
    static __device__ __forceinline__ bool less(uint64_t a, uint64_t b) { return a < b; }
};

// RankingPolicy sort key (schedulers.py:211-218): class bits (running-pin, unscored,
// non-priority) in the top 3 bits of `cr`, arrival rank in the low 29 bits, and the
// order-preserving image of the float64 effective score in `eff`.
// Compared as (cr >> 29, eff, cr & RANK_MASK).
struct __align__(16) RankKey {
    uint64_t eff;
    uint32_t cr;
    uint32_t pad;
};
template <>
struct KeyTraits<RankKey> {
    static __device__ __forceinline__ RankKey sentinel() { return RankKey{~0ull, 0xffffffffu, 0u}; }
    static __device__ __forceinline__ bool less(const RankKey& a, const RankKey& b) {
        uint32_t ca = a.cr >> 29, cb = b.cr >> 29;
        if (ca != cb) return ca < cb;
        if (a.eff != b.eff) return a.eff < b.eff;
        return a.cr < b.cr;
    }
};

// (arrival_time, id) tuple key of the reference tie-break (schedulers.py:416-417).
struct __align__(16) Key128 {
    uint64_t hi;
    uint64_t lo;
};
template <>
struct KeyTraits<Key128> {
    static __device__ __forceinline__ Key128 sentinel() { return Key128{~0ull, ~0ull}; }
    static __device__ __forceinline__ bool less(const Key128& a, const Key128& b) {
        return a.hi != b.hi ? a.hi < b.hi : a.lo < b.lo;
    }
};

// Shared-memory tiles are padded with one key per 128 bytes, so the MS_ITEMS-strided
// per-thread accesses of the merges (thread t at key 8t + i) spread over the banks
// instead of hitting the same few (a 16-way conflict for 64-bit keys unpadded).
template <typename T>
struct MsPad {
    static constexpr int shift = sizeof(T) == 4 ? 5 : sizeof(T) == 8 ? 4 : 3;
    static constexpr int size = MS_TILE + (MS_TILE >> shift) + 1;
};
template <typename T>
__device__ __forceinline__ int ms_pidx(int e) { return e + (e >> MsPad<T>::shift); }

template <typename T>
struct SView {  // run view into a padded smem tile
    T* s;
    int off;
    __device__ __forceinline__ T operator[](int i) const { return s[ms_pidx<T>(off + i)]; }
};

template <typename K, typename A>
__device__ __forceinline__ int merge_path(const A& a, int na, const A& b, int nb, int diag) {
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (!KeyTraits<K>::less(b[diag - 1 - mid], a[mid]))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Serially merge MS_ITEMS outputs starting at (i, j), keeping the two head keys in
// registers (one shared-memory load per output). a_remaining_base - i = left-run
// elements not yet consumed (for inversion counting).
template <typename K, bool HasVal, bool Count>
__device__ __forceinline__ void serial_merge(const SView<K>& a, const SView<uint32_t>& av, int na,
                                             const SView<K>& b, const SView<uint32_t>& bv, int nb, int i, int j,
                                             K (&ok)[MS_ITEMS], uint32_t (&ov)[MS_ITEMS],
                                             uint64_t a_remaining_base, unsigned long long& inv) {
    bool a_ok = i < na, b_ok = j < nb;
    K ka = a_ok ? a[i] : KeyTraits<K>::sentinel();
    K kb = b_ok ? b[j] : KeyTraits<K>::sentinel();
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        const bool take_a = a_ok && (!b_ok || !KeyTraits<K>::less(kb, ka));
        if (take_a) {
            ok[k] = ka;
            if (HasVal) ov[k] = av[i];
            ++i;
            a_ok = i < na;
            if (a_ok) ka = a[i];
        } else {
            ok[k] = kb;
            if (HasVal) ov[k] = bv[j];
            ++j;
            if (Count) inv += a_remaining_base - (uint64_t)i;
            b_ok = j < nb;
            if (b_ok) kb = b[j];
        }
    }
}

template <typename K, bool HasVal>
struct MsSmem {
    K keys[MsPad<K>::size];
    uint32_t vals[HasVal ? MsPad<uint32_t>::size : 1];
};

// CTA-wide sum, one atomic per CTA (every thread of the CTA must call it).
__device__ __forceinline__ void block_add_count(unsigned long long v, unsigned long long* out) {
    __shared__ unsigned long long part[32];
    v = warp_sum(v);
    const int nw = (int)(blockDim.x >> 5);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long t = (int)threadIdx.x < nw ? part[threadIdx.x] : 0ull;
        t = warp_sum(t);
        if (threadIdx.x == 0 && t) atomicAdd(out, t);
    }
}

// Sort each 2048-key tile. keys_in has n valid entries; the tail of the last tile is
// padded with sentinels (which sort last, stably, and add no strict inversions).
// vals_in == nullptr => payload is the global index.
template <typename K, bool HasVal, bool Count>
__global__ void __launch_bounds__(MS_THREADS) ms_block_sort(const K* __restrict__ keys_in,
                                                            const uint32_t* __restrict__ vals_in,
                                                            K* __restrict__ keys_out,
                                                            uint32_t* __restrict__ vals_out,
                                                            uint32_t n, unsigned long long* inv_out) {
    __shared__ MsSmem<K, HasVal> sm;
    const uint32_t base = blockIdx.x * MS_TILE;
    for (int k = threadIdx.x; k < MS_TILE; k += MS_THREADS) {
        uint32_t g = base + k;
        sm.keys[ms_pidx<K>(k)] = g < n ? keys_in[g] : KeyTraits<K>::sentinel();
        if (HasVal) sm.vals[ms_pidx<uint32_t>(k)] = g < n ? (vals_in ? vals_in[g] : g) : 0xffffffffu;
    }
    __syncthreads();
    K rk[MS_ITEMS];
    uint32_t rv[MS_ITEMS];
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        rk[k] = sm.keys[ms_pidx<K>(threadIdx.x * MS_ITEMS + k)];
        if (HasVal) rv[k] = sm.vals[ms_pidx<uint32_t>(threadIdx.x * MS_ITEMS + k)];
    }
    unsigned long long inv = 0;
    // Odd-even transposition: strict swaps only => stable, swap count = inversions.
#pragma unroll
    for (int r = 0; r < MS_ITEMS; ++r) {
#pragma unroll
        for (int k = (r & 1); k + 1 < MS_ITEMS; k += 2) {
            if (KeyTraits<K>::less(rk[k + 1], rk[k])) {
                K t = rk[k];
                rk[k] = rk[k + 1];
                rk[k + 1] = t;
                if (HasVal) {
                    uint32_t tv = rv[k];
                    rv[k] = rv[k + 1];
                    rv[k + 1] = tv;
                }
                if (Count) ++inv;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        sm.keys[ms_pidx<K>(threadIdx.x * MS_ITEMS + k)] = rk[k];
        if (HasVal) sm.vals[ms_pidx<uint32_t>(threadIdx.x * MS_ITEMS + k)] = rv[k];
    }
    __syncthreads();
    for (int s = MS_ITEMS; s < MS_TILE; s <<= 1) {
        const int p = threadIdx.x * MS_ITEMS;
        const int pb = p / (2 * s) * (2 * s);
        const SView<K> a{sm.keys, pb}, b{sm.keys, pb + s};
        const SView<uint32_t> av{sm.vals, pb}, bv{sm.vals, pb + s};
        const int diag = p - pb;
        const int i = merge_path<K>(a, s, b, s, diag);
        serial_merge<K, HasVal, Count>(a, av, s, b, bv, s, i, diag - i, rk, rv, (uint64_t)s, inv);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MS_ITEMS; ++k) {
            sm.keys[ms_pidx<K>(p + k)] = rk[k];
            if (HasVal) sm.vals[ms_pidx<uint32_t>(p + k)] = rv[k];
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < MS_TILE; k += MS_THREADS) {
        keys_out[base + k] = sm.keys[ms_pidx<K>(k)];
        if (HasVal) vals_out[base + k] = sm.vals[ms_pidx<uint32_t>(k)];
    }
    if (Count) block_add_count(inv, inv_out);
}

// One global merge pass: runs of width w -> runs of width 2w over npad keys. Each CTA
// finds its tile's merge-path splits itself, one warp per split: every round the 32 lanes
// probe 32 evenly spaced candidates and a ballot narrows the range 32x, so a split over a
// run of 2^23 keys costs 5 dependent global loads instead of 23 (no separate partition
// kernel, so a pass is one launch).
template <typename K>
__device__ __forceinline__ int ms_split_warp(const K* __restrict__ kin, uint32_t npad, uint32_t w, uint32_t t,
                                             uint32_t tiles) {
    const int lane = threadIdx.x & 31;
    const uint32_t out = t * MS_TILE;
    if (t >= tiles || out % (2 * w) == 0) return 0;  // run-pair boundary: nothing taken yet
    const uint32_t base = out / (2 * w) * (2 * w);
    const int lenA = (int)min(w, npad - base);
    const int lenB = (int)min(w, npad - base - (uint32_t)lenA);
    const K* a = kin + base;
    const K* b = kin + base + lenA;
    const int diag = (int)(out - base);
    // smallest i in [lo, hi] with less(b[diag-1-i], a[i]) (hi if none): the merge_path split
    int lo = max(0, diag - lenB), hi = min(diag, lenA);
    while (hi - lo > 32) {
        const int step = (hi - lo + 31) / 32;
        const int p = lo + lane * step;
        const bool pred = p < hi && KeyTraits<K>::less(b[diag - 1 - p], a[p]);
        const unsigned m = __ballot_sync(0xffffffffu, pred);
        if (m) {
            const int f = __ffs(m) - 1;
            const int pf = lo + f * step;
            lo = f ? pf - step + 1 : lo;
            hi = pf;
        } else {
            const int last = min(31, (hi - 1 - lo) / step);
            lo = lo + last * step + 1;
        }
    }
    const int p = lo + lane;
    const bool pred = p < hi && KeyTraits<K>::less(b[diag - 1 - p], a[p]);
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    return m ? lo + __ffs(m) - 1 : hi;
}

template <typename K, bool HasVal, bool Count>
__global__ void __launch_bounds__(MS_THREADS) ms_merge_pass(const K* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin,
                                                            K* __restrict__ kout,
                                                            uint32_t* __restrict__ vout,
                                                            uint32_t npad, uint32_t w,
                                                            unsigned long long* inv_out,
                                                            const int* __restrict__ skip) {
    if (skip && *skip) return;
    __shared__ MsSmem<K, HasVal> sm;
    __shared__ int s_split[2];
    if (threadIdx.x < 64) {  // warp 0: this tile's start split, warp 1: the next tile's
        const int v = ms_split_warp<K>(kin, npad, w, blockIdx.x + (threadIdx.x >> 5), gridDim.x);
        if ((threadIdx.x & 31) == 0) s_split[threadIdx.x >> 5] = v;
    }
    __syncthreads();
    const uint32_t out0 = blockIdx.x * MS_TILE;
    const uint32_t base = out0 / (2 * w) * (2 * w);
    const int lenA = (int)min(w, npad - base);
    const int lenB = (int)min(w, npad - base - (uint32_t)lenA);
    const K* A = kin + base;
    const K* B = kin + base + lenA;
    const int d0 = (int)(out0 - base);
    const int d1 = d0 + MS_TILE;
    // the tile's end split: the next tile's start, or the whole left run at a run end
    const int a0 = s_split[0];
    const int a1 = (d1 == lenA + lenB) ? lenA : s_split[1];
    const int b0 = d0 - a0, b1 = d1 - a1;
    const int na = a1 - a0, nb = b1 - b0;
    for (int k = threadIdx.x; k < MS_TILE; k += MS_THREADS) {
        if (k < na) {
            sm.keys[ms_pidx<K>(k)] = A[a0 + k];
            if (HasVal) sm.vals[ms_pidx<uint32_t>(k)] = vin[base + a0 + k];
        } else {
            sm.keys[ms_pidx<K>(k)] = B[b0 + k - na];
            if (HasVal) sm.vals[ms_pidx<uint32_t>(k)] = vin[base + lenA + b0 + k - na];
        }
    }
    __syncthreads();
    K rk[MS_ITEMS];
    uint32_t rv[MS_ITEMS];
    unsigned long long inv = 0;
    const int diag = threadIdx.x * MS_ITEMS;
    const SView<K> sa{sm.keys, 0}, sb{sm.keys, na};
    const SView<uint32_t> sav{sm.vals, 0}, sbv{sm.vals, na};
    const int i = merge_path<K>(sa, na, sb, nb, diag);
    // left-run elements not yet consumed when a right element is taken:
    // lenA - (a0 + i_local)  => base term lenA - a0, minus the local i.
    serial_merge<K, HasVal, Count>(sa, sav, na, sb, sbv, nb, i, diag - i, rk, rv, (uint64_t)(lenA - a0), inv);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        sm.keys[ms_pidx<K>(diag + k)] = rk[k];
        if (HasVal) sm.vals[ms_pidx<uint32_t>(diag + k)] = rv[k];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < MS_TILE; k += MS_THREADS) {
        kout[out0 + k] = sm.keys[ms_pidx<K>(k)];
        if (HasVal) vout[out0 + k] = sm.vals[ms_pidx<uint32_t>(k)];
    }
    if (Count) block_add_count(inv, inv_out);
}

// Small inputs: a bitonic network over (key, index) pairs in shared memory, 1024 threads,
// in one launch. Ties are broken by the original index, so the result equals the stable
// sort's. Measured on the rank step (16-byte keys): faster than the block-sort path up to
// ~1K keys (42 vs 52 us per step at 300), even at 1K, slower beyond (157 vs 71 us at 4K:
// 78 barrier-separated stages of 16-byte shared-memory exchanges).
#ifndef RS_MS_SMALL_MAX
#define RS_MS_SMALL_MAX 1024
#endif
constexpr int MS_SMALL_MAX = RS_MS_SMALL_MAX;
constexpr int MS_SMALL_THREADS = 1024;

template <typename K>
__global__ void __launch_bounds__(MS_SMALL_THREADS) ms_small_sort(const K* __restrict__ keys_in, uint32_t n,
                                                                  uint32_t npow2, uint32_t npad,
                                                                  K* __restrict__ keys_out,
                                                                  uint32_t* __restrict__ vals_out) {
    extern __shared__ __align__(16) unsigned char ms_small_raw[];
    K* sk = reinterpret_cast<K*>(ms_small_raw);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + npow2);
    for (uint32_t i = threadIdx.x; i < npow2; i += MS_SMALL_THREADS) {
        sk[i] = i < n ? keys_in[i] : KeyTraits<K>::sentinel();
        sv[i] = i;  // padding indices (>= n) keep the sentinels last
    }
    __syncthreads();
    for (uint32_t k = 2; k <= npow2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = threadIdx.x; t < (npow2 >> 1); t += MS_SMALL_THREADS) {
                const uint32_t i = 2 * j * (t / j) + (t % j), p = i + j;
                const K a = sk[i], b = sk[p];
                const uint32_t ia = sv[i], ib = sv[p];
                const bool b_lt_a = KeyTraits<K>::less(b, a) || (!KeyTraits<K>::less(a, b) && ib < ia);
                if (b_lt_a == ((i & k) == 0)) {
                    sk[i] = b;
                    sk[p] = a;
                    sv[i] = ib;
                    sv[p] = ia;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < npad; i += MS_SMALL_THREADS) {
        keys_out[i] = i < n ? sk[i] : KeyTraits<K>::sentinel();
        if (vals_out) vals_out[i] = i < n ? sv[i] : 0xffffffffu;
    }
}

static inline uint32_t ms_padded(uint64_t n) {
    return (uint32_t)((n + MS_TILE - 1) / MS_TILE * MS_TILE);
}

// ints of scratch reserved for per-pass tile splits (the passes now find their own splits;
// kept so callers' workspace layouts stay valid)
static inline uint32_t ms_splits(uint64_t n) { return (uint32_t)((n + MS_TILE - 1) / MS_TILE) + 2; }

// Sort n keys (+ optional u32 payload). k0/k1 and v0/v1 are ping-pong buffers of
// ms_padded(n) entries, splits ms_splits(n) ints. On return *kres / *vres point at the
// sorted (padded) arrays. With `skip` set, the passes at run width >= skip_w return at
// once when *skip != 0 (decided on the device: the output is then sorted only within
// runs of skip_w, and only the inversions inside those runs are counted).
template <typename K, bool HasVal, bool Count>
int merge_sort(const K* keys_in, const uint32_t* vals_in, uint32_t n, K* k0, K* k1, uint32_t* v0,
               uint32_t* v1, unsigned long long* inv, cudaStream_t st, K** kres,
               uint32_t** vres, int* splits, const int* skip = nullptr, uint32_t skip_w = 0) {
    const uint32_t npad = ms_padded(n);
    const uint32_t tiles = npad / MS_TILE;
    if (tiles == 0) {
        *kres = k0;
        if (vres) *vres = v0;
        return RS_OK;
    }
    if (!Count && vals_in == nullptr && n <= (uint32_t)MS_SMALL_MAX) {
        uint32_t np2 = 1;
        while (np2 < n) np2 <<= 1;
        const size_t smem = (size_t)np2 * (sizeof(K) + sizeof(uint32_t));
        static bool attr = false;  // per template instance
        if (!attr) {
            RS_CUDA(cudaFuncSetAttribute(ms_small_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(MS_SMALL_MAX * (sizeof(K) + sizeof(uint32_t)))));
            attr = true;
        }
        ms_small_sort<K><<<1, MS_SMALL_THREADS, smem, st>>>(keys_in, n, np2, npad, k0, HasVal ? v0 : nullptr);
        RS_LAUNCH_CHECK();
        *kres = k0;
        if (vres) *vres = v0;
        return RS_OK;
    }
    ms_block_sort<K, HasVal, Count><<<tiles, MS_THREADS, 0, st>>>(keys_in, vals_in, k0, v0, n, inv);
    RS_LAUNCH_CHECK();
    K* ki = k0;
    K* ko = k1;
    uint32_t* vi = v0;
    uint32_t* vo = v1;
    for (uint32_t w = MS_TILE; w < npad; w <<= 1) {
        const int* sk = (skip && w >= skip_w) ? skip : nullptr;
        ms_merge_pass<K, HasVal, Count><<<tiles, MS_THREADS, 0, st>>>(ki, vi, ko, vo, npad, w, inv, sk);
        RS_LAUNCH_CHECK();
        K* t = ki;
        ki = ko;
        ko = t;
        uint32_t* tv = vi;
        vi = vo;
        vo = tv;
    }
    *kres = ki;
    if (vres) *vres = vi;
    return RS_OK;
}

}  // namespace rs
