// K10: exact Kendall tau-b pair counts.
//
// Reference: ranking.kendall_tau_b (ranking.py:24-63) enumerates all n(n-1)/2 pairs
// with sign(dx)*sign(dy) row by row and counts ties with np.unique. Here (Knight's
// algorithm, exact integer identity):
//   1. map x, y to 32-bit order-preserving integer images (float64 semantics; f64/i64
//      inputs are first compressed to dense ranks by a sort),
//   2. sort the 64-bit composite (x_img << 32 | y_img)            -> n1, n3 from runs
//   3. D = strict inversions of the y images in that order        (merge-sort count)
//      and the same sort leaves y sorted                         -> n2 from runs
//      (y spanning < 4096 values: only 2048-key tiles are sorted, and the inversions
//      across tiles and n2 come from chunk histograms — see chunk_cross)
//   4. C = n0 - n1 - n2 + n3 - D.
// All counts are exact int64; tau itself is finished on the host with the reference
// expression (ranking.py:60-63).
#include "common.cuh"
#include "mergesort.cuh"
#include "tau_fast.cuh"
#include <cstdlib>
#include <cstring>

namespace rs {

__device__ __forceinline__ double load_as_f64(const void* p, int dt, uint32_t i) {
    switch (dt) {
        case RS_F32: return (double)static_cast<const float*>(p)[i];
        case RS_F64: return static_cast<const double*>(p)[i];
        case RS_I32: return (double)static_cast<const int32_t*>(p)[i];
        default: return (double)static_cast<const int64_t*>(p)[i];
    }
}

// 32-bit images for 32-bit dtypes (same order as their float64 casts).
__global__ void tau_image32(const void* __restrict__ v, int dt, uint32_t n, uint32_t* __restrict__ out,
                            int* __restrict__ nan_flag) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (dt == RS_F32) {
        float f = static_cast<const float*>(v)[i];
        if (f != f) atomicOr(nan_flag, 1);
        out[i] = orderable_f32(f);
    } else {
        out[i] = orderable_i32(static_cast<const int32_t*>(v)[i]);
    }
}

__global__ void tau_image64(const void* __restrict__ v, int dt, uint32_t n, uint64_t* __restrict__ out,
                            int* __restrict__ nan_flag) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = load_as_f64(v, dt, i);
    if (d != d) atomicOr(nan_flag, 1);
    out[i] = orderable_f64(d);
}

// Dense ranks from a sorted (key, original index) array: rank = #distinct keys
// strictly below. Two-level: per-block head counts, then a serial scan of block
// totals (few thousand blocks at most), then the scatter.
constexpr int RK_THREADS = 1024;
__global__ void rank_heads_count(const uint64_t* __restrict__ sk, uint32_t n, uint32_t* __restrict__ block_heads) {
    uint32_t i = blockIdx.x * RK_THREADS + threadIdx.x;
    int head = (i < n && i > 0 && sk[i] != sk[i - 1]) ? 1 : 0;
    int c = __syncthreads_count(head);
    if (threadIdx.x == 0) block_heads[blockIdx.x] = c;
}
__global__ void exclusive_scan_serial(uint32_t* a, uint32_t m) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t s = 0;
    for (uint32_t i = 0; i < m; ++i) {
        uint32_t v = a[i];
        a[i] = s;
        s += v;
    }
}
__global__ void rank_scatter(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, uint32_t n,
                             const uint32_t* __restrict__ block_off, uint32_t* __restrict__ rank_out) {
    __shared__ uint32_t warp_tot[RK_THREADS / 32];
    uint32_t i = blockIdx.x * RK_THREADS + threadIdx.x;
    uint32_t head = (i < n && i > 0 && sk[i] != sk[i - 1]) ? 1u : 0u;
    // inclusive block scan of head flags
    uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t ballot = __ballot_sync(0xffffffffu, head);
    uint32_t incl = __popc(ballot & (0xffffffffu >> (31 - lane)));
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t t = warp_tot[lane];
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        warp_tot[lane] = x - t;  // exclusive
    }
    __syncthreads();
    if (i < n) rank_out[sv[i]] = block_off[blockIdx.x] + warp_tot[wid] + incl;
}

// Tied pairs = sum over runs of c(c-1)/2, evaluated at each run end that has c >= 2
// by a lower_bound for the run start (keys sorted => the images are monotone): gallop
// back from the run end (runs are short), then bisect the last gap. Grid-stride over a
// few CTAs per SM with one atomic per CTA (a per-warp atomic on one counter serialises
// at L2 when most warps see a tie).
template <typename K, typename Proj>
__global__ void __launch_bounds__(256) tied_pairs(const K* __restrict__ s, uint32_t n, Proj proj,
                                                  unsigned long long* __restrict__ out,
                                                  const int* __restrict__ skip) {
    if (skip && *skip) return;
    unsigned long long c = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t v = proj(s[i]);
        const bool end = (i + 1 == n) || proj(s[i + 1]) != v;
        if (end && i > 0 && proj(s[i - 1]) == v) {
            uint32_t step = 2, hi = i - 1;
            while (step <= i && proj(s[i - step]) == v) {
                hi = i - step;
                step <<= 1;
            }
            uint32_t lo = step <= i ? i - step + 1 : 0;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (proj(s[mid]) < v) lo = mid + 1; else hi = mid;
            }
            const unsigned long long len = (unsigned long long)(i - lo + 1);
            c += len * (len - 1) / 2;
        }
    }
    block_add_count(c, out);
}
struct ProjFull { __device__ uint64_t operator()(uint64_t v) const { return v; } };
struct ProjHi { __device__ uint64_t operator()(uint64_t v) const { return v >> 32; } };

// ---- small-range y: cross-tile inversions from histograms ------------------------
// When the y images span fewer than TH_BINS values (cfg4: lengths in [1, 2048]), the
// inversions between different 2048-key tiles of the (x, y)-sorted sequence are
//   sum over tiles t, items j in t of #{items in earlier tiles with y > y_j},
// read off a running histogram of everything before t. So the y merge sort stops after
// its block-sort stage (which counts the inversions inside each tile) and three passes
// replace its log2(n / 2048) merge passes: per-chunk histograms, a column scan of them
// (exclusive per chunk; the column totals also give n2), and a count pass in which each
// chunk walks its tiles with the running histogram in shared memory. The choice is
// made on the device (no host round trip), so both paths are launched and the unused
// one returns at once.
constexpr int TH_BINS = 4096;
constexpr int TH_THREADS = 256;

struct TauChunks {
    uint32_t tiles_per_chunk, chunk_elems, nchunks;
};
static TauChunks tau_chunks(uint64_t n) {
    const uint32_t tiles = (uint32_t)((n + MS_TILE - 1) / MS_TILE);
    const uint32_t target = (uint32_t)num_sms() * 8;  // ~ resident CTAs of the count pass
    const uint32_t tpc = (tiles + target - 1) / target;
    const uint32_t ce = tpc * MS_TILE;
    return TauChunks{tpc, ce, (uint32_t)((n + ce - 1) / ce)};
}

__global__ void __launch_bounds__(256) y_range(const uint32_t* __restrict__ y, uint32_t n, uint32_t* __restrict__ yr) {
    uint32_t lo = 0xffffffffu, hi = 0u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t v = y[i];
        lo = min(lo, v);
        hi = max(hi, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(yr + 0, lo);
        atomicMax(yr + 1, hi);
    }
}
// flag[1] = 1 when the histogram path applies (read by both paths' kernels)
__global__ void y_range_flag(const uint32_t* __restrict__ yr, int* __restrict__ flag) {
    flag[1] = (yr[1] - yr[0] < (uint32_t)TH_BINS) ? 1 : 0;
}

__global__ void __launch_bounds__(TH_THREADS) chunk_hist(const uint32_t* __restrict__ y, uint32_t n,
                                                         const uint32_t* __restrict__ yr, const int* __restrict__ flag,
                                                         uint32_t chunk_elems, uint32_t* __restrict__ hist) {
    if (!flag[1]) return;
    __shared__ uint32_t h[TH_BINS];
    for (int v = threadIdx.x; v < TH_BINS; v += TH_THREADS) h[v] = 0;
    __syncthreads();
    const uint32_t ymin = yr[0];
    const uint32_t beg = blockIdx.x * chunk_elems, end = min(n, beg + chunk_elems);
    for (uint32_t i = beg + threadIdx.x; i < end; i += TH_THREADS) atomicAdd(&h[y[i] - ymin], 1u);
    __syncthreads();
    uint32_t* out = hist + (size_t)blockIdx.x * TH_BINS;
    for (int v = threadIdx.x; v < TH_BINS; v += TH_THREADS) out[v] = h[v];
}

// Column-wise exclusive scan of the chunk histograms: CTA = 32 bins (one per lane),
// its 8 warps split the chunk rows; totals -> tied pairs in y (n2).
__global__ void __launch_bounds__(256) chunk_scan(const uint32_t* __restrict__ hist, uint32_t nchunks,
                                                  const int* __restrict__ flag, uint32_t* __restrict__ pre,
                                                  unsigned long long* __restrict__ n2) {
    if (!flag[1]) return;
    __shared__ uint32_t tot[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t bin = blockIdx.x * 32 + lane;
    const uint32_t rpw = (nchunks + 7) / 8;
    const uint32_t r0 = min(nchunks, wid * rpw), r1 = min(nchunks, r0 + rpw);
    uint32_t s = 0;
    for (uint32_t r = r0; r < r1; ++r) s += hist[(size_t)r * TH_BINS + bin];
    tot[wid][lane] = s;
    __syncthreads();
    uint32_t run = 0, all = 0;
    for (int k = 0; k < 8; ++k) {
        if (k < wid) run += tot[k][lane];
        all += tot[k][lane];
    }
    for (uint32_t r = r0; r < r1; ++r) {
        pre[(size_t)r * TH_BINS + bin] = run;
        run += hist[(size_t)r * TH_BINS + bin];
    }
    const unsigned long long c = (unsigned long long)all * (all - 1ull) / 2ull;
    block_add_count(wid == 0 ? c : 0ull, n2);
}

// Each chunk walks its tiles in order: before tile k the shared histogram holds every
// y of earlier tiles; suffix sums of it give each item's count of earlier, larger y.
__global__ void __launch_bounds__(TH_THREADS) chunk_cross(const uint32_t* __restrict__ y, uint32_t n,
                                                          const uint32_t* __restrict__ yr,
                                                          const int* __restrict__ flag, uint32_t chunk_elems,
                                                          const uint32_t* __restrict__ pre,
                                                          unsigned long long* __restrict__ inv) {
    if (!flag[1]) return;
    constexpr int PER = TH_BINS / TH_THREADS;  // 16 bins per thread
    __shared__ uint32_t h[TH_BINS];
    __shared__ uint32_t gt[TH_BINS];  // gt[v] = #earlier items with y image offset > v
    __shared__ uint32_t wsum[TH_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t ymin = yr[0];
    const uint32_t* p = pre + (size_t)blockIdx.x * TH_BINS;
    for (int v = threadIdx.x; v < TH_BINS; v += TH_THREADS) h[v] = p[v];
    __syncthreads();
    const uint32_t beg = blockIdx.x * chunk_elems, end = min(n, beg + chunk_elems);
    unsigned long long cnt = 0;
    for (uint32_t t0 = beg; t0 < end; t0 += MS_TILE) {
        // suffix sums over the thread's 16 bins, then across threads (reverse scan)
        uint32_t loc[PER];
        uint32_t acc = 0;
#pragma unroll
        for (int k = PER - 1; k >= 0; --k) {
            loc[k] = acc;  // strictly greater bins inside the thread's run
            acc += h[threadIdx.x * PER + k];
        }
        uint32_t x = acc;  // inclusive suffix scan over threads: lanes above + warps above
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yv = __shfl_down_sync(0xffffffffu, x, o);
            if (lane + o < 32) x += yv;
        }
        if (lane == 0) wsum[wid] = x;
        __syncthreads();
        uint32_t above = x - acc;
        for (int k = wid + 1; k < TH_THREADS / 32; ++k) above += wsum[k];
#pragma unroll
        for (int k = 0; k < PER; ++k) gt[threadIdx.x * PER + k] = loc[k] + above;
        __syncthreads();
        const uint32_t t1 = min(end, t0 + MS_TILE);
        for (uint32_t i = t0 + threadIdx.x; i < t1; i += TH_THREADS) {
            const uint32_t v = y[i] - ymin;
            cnt += gt[v];
            atomicAdd(&h[v], 1u);
        }
        __syncthreads();
    }
    block_add_count(cnt, inv);
}

__global__ void compose_keys(const uint32_t* __restrict__ ux, const uint32_t* __restrict__ uy, uint32_t n,
                             uint64_t* __restrict__ out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = ((uint64_t)ux[i] << 32) | uy[i];
}
__global__ void low_words(const uint64_t* __restrict__ s, uint32_t n, uint32_t* __restrict__ out) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)s[i];
}

// acc: [0]=D [1]=n1 [2]=n2 [3]=n3 ; counts = {C, D, n1, n2, n3, nan}
__global__ void tau_finish(const unsigned long long* acc, const int* nan_flag, uint64_t n, int64_t* counts) {
    long long n0 = (long long)(n * (n - 1) / 2);
    long long D = (long long)acc[0], n1 = (long long)acc[1], n2 = (long long)acc[2], n3 = (long long)acc[3];
    counts[0] = n0 - n1 - n2 + n3 - D;
    counts[1] = D;
    counts[2] = n1;
    counts[3] = n2;
    counts[4] = n3;
    counts[5] = *nan_flag ? 1 : 0;
}

struct TauWs {
    uint32_t* ux;
    uint32_t* uy;
    uint64_t* k64a;
    uint64_t* k64b;
    uint32_t* k32a;
    uint32_t* k32b;
    uint32_t* va;
    uint32_t* vb;
    uint32_t* blk;
    unsigned long long* acc;
    int* flag;
    int* splits;
    uint32_t* yr;
    uint32_t* hist;
    uint32_t* pre;
};

template <typename A>
static void tau_layout(A& a, uint64_t n, bool need64, TauWs* w) {
    const uint32_t np = ms_padded(n);
    const uint32_t nblk = (uint32_t)((n + RK_THREADS - 1) / RK_THREADS) + 1;
    auto t_ux = a.template take<uint32_t>(n);
    auto t_uy = a.template take<uint32_t>(n);
    auto t_ka = a.template take<uint64_t>(np);
    auto t_kb = a.template take<uint64_t>(np);
    auto t_32a = a.template take<uint32_t>(np);
    auto t_32b = a.template take<uint32_t>(np);
    auto t_va = a.template take<uint32_t>(need64 ? np : 1);
    auto t_vb = a.template take<uint32_t>(need64 ? np : 1);
    auto t_blk = a.template take<uint32_t>(nblk);
    auto t_acc = a.template take<unsigned long long>(8);
    auto t_flag = a.template take<int>(4);
    auto t_sp = a.template take<int>(ms_splits(np));
    const TauChunks ch = tau_chunks(n);
    auto t_yr = a.template take<uint32_t>(4);
    auto t_h = a.template take<uint32_t>((size_t)ch.nchunks * TH_BINS);
    auto t_p = a.template take<uint32_t>((size_t)ch.nchunks * TH_BINS);
    if (w) *w = TauWs{t_ux, t_uy, t_ka, t_kb, t_32a, t_32b, t_va, t_vb, t_blk, t_acc, t_flag, t_sp, t_yr, t_h, t_p};
}
struct SizerAdapter {
    ArenaSizer s;
    template <typename T>
    T* take(size_t c) { s.take<T>(c); return nullptr; }
};

static bool is64(int dt) { return dt == RS_F64 || dt == RS_I64; }

static int image_of(const void* v, int dt, uint32_t n, uint32_t* out, TauWs& w, cudaStream_t st) {
    const int T = 256;
    const uint32_t g = (n + T - 1) / T;
    if (!is64(dt)) {
        tau_image32<<<g, T, 0, st>>>(v, dt, n, out, w.flag);
        RS_LAUNCH_CHECK();
        return RS_OK;
    }
    // float64 semantics: dense-rank compression of the 64-bit images.
    tau_image64<<<g, T, 0, st>>>(v, dt, n, w.k64a, w.flag);
    RS_LAUNCH_CHECK();
    uint64_t* sk;
    uint32_t* sv;
    RS_TRY((merge_sort<uint64_t, true, false>(w.k64a, nullptr, n, w.k64b, w.k64a, w.va, w.vb, nullptr, st,
                                              &sk, &sv, w.splits)));
    const uint32_t nb = (n + RK_THREADS - 1) / RK_THREADS;
    rank_heads_count<<<nb, RK_THREADS, 0, st>>>(sk, n, w.blk);
    RS_LAUNCH_CHECK();
    exclusive_scan_serial<<<1, 32, 0, st>>>(w.blk, nb);
    RS_LAUNCH_CHECK();
    rank_scatter<<<nb, RK_THREADS, 0, st>>>(sk, sv, n, w.blk, out);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs

using namespace rs;

extern "C" size_t rs_tau_workspace_size(int64_t n, int x_dtype, int y_dtype) {
    if (n < 2) return 256;
    SizerAdapter a;
    tau_layout(a, (uint64_t)n, is64(x_dtype) || is64(y_dtype), nullptr);
    return align_up(a.s.used, 256) + tau_fast_workspace((uint64_t)n) + 256;
}

namespace rs {
// Below this many rows the general path's fixed launch chain beats the bucket path's
// (measured on B200, tools/gpu_tau_cross.sh); RS_TAU_PATH=fast|general forces one.
constexpr int64_t TAU_FAST_MIN_N = 1 << 18;
static int tau_path_choice(int64_t n) {  // 1 = fast, 0 = general
    if (const char* e = getenv("RS_TAU_PATH")) {
        if (!strcmp(e, "fast")) return 1;
        if (!strcmp(e, "general")) return 0;
    }
    return n >= TAU_FAST_MIN_N ? 1 : 0;
}
// Fast path (tau_fast.cu) on the raw 32-bit inputs, or on 32-bit dense-rank images of
// 64-bit inputs. counts[5] = 2 afterwards when the general path is needed.
static int tau_fast_path(const void* x, int xd, const void* y, int yd, uint32_t n, int64_t* counts, TauWs& w,
                         void* fws, size_t fws_bytes, cudaStream_t st) {
    if (is64(xd) || is64(yd)) {
        RS_CUDA(cudaMemsetAsync(w.flag, 0, 4 * sizeof(int), st));
        RS_TRY(image_of(x, xd, n, w.ux, w, st));
        RS_TRY(image_of(y, yd, n, w.uy, w, st));
        return tau_fast_counts(w.ux, TF_DT_U32, w.uy, TF_DT_U32, n, counts, w.k32a, w.k32b, w.flag, fws, fws_bytes,
                               st);
    }
    return tau_fast_counts(x, xd, y, yd, n, counts, w.k32a, w.k32b, nullptr, fws, fws_bytes, st);
}
}  // namespace rs

static int tau_general(const void* x, int xd, const void* y, int yd, int64_t n, int64_t* counts, TauWs& w,
                       cudaStream_t st);

// Fast path only, never synchronises (graph-capturable): counts[5] = 2 tells the caller
// to run rs_tau_counts (general path) instead.
extern "C" int rs_tau_counts_fast(const void* x, int xd, const void* y, int yd, int64_t n, int64_t* counts,
                                  void* ws, size_t ws_bytes, void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(n >= 0 && n < (int64_t)0xF0000000ll, "rs_tau_counts_fast: n=%lld out of range", (long long)n);
    RS_CHECK_ARG(xd >= RS_F32 && xd <= RS_I64 && yd >= RS_F32 && yd <= RS_I64, "rs_tau_counts_fast: bad dtype");
    RS_CHECK_ARG(counts != nullptr, "rs_tau_counts_fast: counts is NULL");
    if (n < 2) {
        RS_CUDA(cudaMemsetAsync(counts, 0, 6 * sizeof(int64_t), st));
        return RS_OK;
    }
    RS_CHECK_ARG(x && y, "rs_tau_counts_fast: NULL input");
    if (ws_bytes < rs_tau_workspace_size(n, xd, yd)) {
        set_error("rs_tau_counts_fast: workspace %zu < %zu", ws_bytes, rs_tau_workspace_size(n, xd, yd));
        return RS_ERR_WORKSPACE;
    }
    Arena ar(ws, ws_bytes);
    TauWs w;
    tau_layout(ar, (uint64_t)n, is64(xd) || is64(yd), &w);
    if (!tau_path_choice(n)) return tau_general(x, xd, y, yd, n, counts, w, st);  // sync-free as well
    const size_t used = align_up(ar.used, 256);
    return tau_fast_path(x, xd, y, yd, (uint32_t)n, counts, w, static_cast<char*>(ws) + used, ws_bytes - used, st);
}

extern "C" int rs_tau_counts(const void* x, int xd, const void* y, int yd, int64_t n, int64_t* counts,
                             void* ws, size_t ws_bytes, void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(n >= 0 && n < (int64_t)0xF0000000ll, "rs_tau_counts: n=%lld out of range", (long long)n);
    RS_CHECK_ARG(xd >= RS_F32 && xd <= RS_I64 && yd >= RS_F32 && yd <= RS_I64, "rs_tau_counts: bad dtype");
    RS_CHECK_ARG(counts != nullptr, "rs_tau_counts: counts is NULL");
    if (n < 2) {
        RS_CUDA(cudaMemsetAsync(counts, 0, 6 * sizeof(int64_t), st));
        return RS_OK;
    }
    RS_CHECK_ARG(x && y, "rs_tau_counts: NULL input");
    if (ws_bytes < rs_tau_workspace_size(n, xd, yd)) {
        set_error("rs_tau_counts: workspace %zu < %zu", ws_bytes, rs_tau_workspace_size(n, xd, yd));
        return RS_ERR_WORKSPACE;
    }
    Arena ar(ws, ws_bytes);
    TauWs w;
    tau_layout(ar, (uint64_t)n, is64(xd) || is64(yd), &w);
    if (!tau_path_choice(n)) return tau_general(x, xd, y, yd, n, counts, w, st);
    const size_t used = align_up(ar.used, 256);
    RS_TRY(tau_fast_path(x, xd, y, yd, (uint32_t)n, counts, w, static_cast<char*>(ws) + used, ws_bytes - used, st));
    // Inside a stream capture the fast path is all that is recorded (counts[5] == 2 then
    // asks the caller for an eager call); otherwise read its status once.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    RS_CUDA(cudaStreamIsCapturing(st, &cap));
    if (cap != cudaStreamCaptureStatusNone) return RS_OK;
    int64_t status = 0;
    RS_CUDA(cudaMemcpyAsync(&status, counts + 5, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    if (status != 2) return RS_OK;
    return tau_general(x, xd, y, yd, n, counts, w, st);
}

// The general path: sort the (x, y) composite, count y inversions (merge sort or, for a
// small y range, chunk histograms).
static int tau_general(const void* x, int xd, const void* y, int yd, int64_t n, int64_t* counts, TauWs& w,
                       cudaStream_t st) {
    const uint32_t un = (uint32_t)n;
    RS_CUDA(cudaMemsetAsync(w.acc, 0, 8 * sizeof(unsigned long long), st));
    RS_CUDA(cudaMemsetAsync(w.flag, 0, 4 * sizeof(int), st));
    RS_TRY(image_of(x, xd, un, w.ux, w, st));
    RS_TRY(image_of(y, yd, un, w.uy, w, st));
    const int T = 256;
    const uint32_t g = (un + T - 1) / T;
    const uint32_t gs = g < (uint32_t)num_sms() * 8 ? g : (uint32_t)num_sms() * 8;
    compose_keys<<<g, T, 0, st>>>(w.ux, w.uy, un, w.k64b);
    RS_LAUNCH_CHECK();
    uint64_t* sk;
    RS_TRY((merge_sort<uint64_t, false, false>(w.k64b, nullptr, un, w.k64a, w.k64b, nullptr, nullptr, nullptr,
                                               st, &sk, nullptr, w.splits)));
    tied_pairs<uint64_t, ProjHi><<<gs, T, 0, st>>>(sk, un, ProjHi{}, w.acc + 1, nullptr);
    RS_LAUNCH_CHECK();
    tied_pairs<uint64_t, ProjFull><<<gs, T, 0, st>>>(sk, un, ProjFull{}, w.acc + 3, nullptr);
    RS_LAUNCH_CHECK();
    low_words<<<g, T, 0, st>>>(sk, un, w.uy);
    RS_LAUNCH_CHECK();
    // D and n2: block-sort counts inside 2048-key tiles, then either the histogram
    // passes (y range < TH_BINS) or the remaining merge passes + runs of the sorted y.
    RS_CUDA(cudaMemsetAsync(w.yr, 0xff, sizeof(uint32_t), st));
    RS_CUDA(cudaMemsetAsync(w.yr + 1, 0, sizeof(uint32_t), st));
    y_range<<<gs, T, 0, st>>>(w.uy, un, w.yr);
    RS_LAUNCH_CHECK();
    y_range_flag<<<1, 1, 0, st>>>(w.yr, w.flag);
    RS_LAUNCH_CHECK();
    uint32_t* sy;
    RS_TRY((merge_sort<uint32_t, false, true>(w.uy, nullptr, un, w.k32a, w.k32b, nullptr, nullptr, w.acc + 0, st,
                                              &sy, nullptr, w.splits, w.flag + 1, (uint32_t)MS_TILE)));
    tied_pairs<uint32_t, ProjFull><<<gs, T, 0, st>>>(sy, un, ProjFull{}, w.acc + 2, w.flag + 1);
    RS_LAUNCH_CHECK();
    const TauChunks ch = tau_chunks(n);
    chunk_hist<<<ch.nchunks, TH_THREADS, 0, st>>>(w.uy, un, w.yr, w.flag, ch.chunk_elems, w.hist);
    RS_LAUNCH_CHECK();
    chunk_scan<<<TH_BINS / 32, 256, 0, st>>>(w.hist, ch.nchunks, w.flag, w.pre, w.acc + 2);
    RS_LAUNCH_CHECK();
    chunk_cross<<<ch.nchunks, TH_THREADS, 0, st>>>(w.uy, un, w.yr, w.flag, ch.chunk_elems, w.pre, w.acc + 0);
    RS_LAUNCH_CHECK();
    // NaN keys are flagged in counts[5] (the reference's NaN behaviour is inconsistent
    // between its pair loop and np.unique, so the wrapper rejects them).
    tau_finish<<<1, 1, 0, st>>>(w.acc, w.flag, (uint64_t)n, counts);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
