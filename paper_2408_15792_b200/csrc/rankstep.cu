// K9: one scheduling step of the ranking policy over an SoA queue.
//
// Reference (schedulers.py):
//   Policy.schedule (:98-109)   sorted(candidates, key=sort_key); non-preemptive pins
//                               RUNNING requests first
//   RankingPolicy.sort_key (:211-218)  (unscored first, priority first, effective score,
//                               arrival_time, id); effective_score (:203-208)
//   Policy._fill (:86-96)       greedy in order; stop at max_batch; SKIP (not stop) a
//                               request whose need = prompt + generated + 1 does not fit
//   RankingPolicy.schedule (:219-240)  starvation count / quantum update in candidate
//                               order, then promotion (count >= threshold) or demotion
//                               (priority and quantum <= 0)
// Device pipeline: key build -> stable merge sort of (RankKey, index) -> greedy fill
// (one warp; prefix-sum resolution of each 32-wide chunk) -> elementwise state update
// with order-preserving compaction of promoted / demoted ids.
#include <cstdlib>
#include <cstring>
#include <utility>
#include "common.cuh"
#include "mergesort.cuh"
#include "engine_exec.cuh"
#include <type_traits>
#include <algorithm>

namespace rs {

constexpr uint32_t RANK_BITS = 29;
constexpr uint32_t RANK_MASK = (1u << RANK_BITS) - 1u;

__device__ __forceinline__ RankKey rank_key_of(const rs_queue_soa& q, uint32_t i, int calibrated, int preemptive,
                                               int* __restrict__ err) {
    const uint8_t f = q.flags[i];
    const bool scored = f & RS_FLAG_SCORED;
    const bool prio = f & RS_FLAG_PRIORITY;
    const bool running = f & RS_FLAG_RUNNING;
    double eff = 0.0;
    if (scored) {
        double s = q.score_dtype == RS_F32 ? (double)static_cast<const float*>(q.score)[i]
                                           : static_cast<const double*>(q.score)[i];
        eff = calibrated ? s - (double)q.generated_tokens[i] : s;
        if (eff != eff) atomicOr(err, 1);
    }
    const uint32_t pin = preemptive ? 0u : (running ? 0u : 1u);
    const uint32_t cls = (pin << 2) | ((scored ? 1u : 0u) << 1) | (prio ? 0u : 1u);
    RankKey k;
    k.eff = orderable_f64(eff);
    k.cr = (cls << RANK_BITS) | (q.arrival_rank[i] & RANK_MASK);
    k.pad = 0;
    return k;
}
__global__ void build_rank_keys(rs_queue_soa q, int calibrated, int preemptive, RankKey* __restrict__ keys,
                                int* __restrict__ err) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (uint32_t)q.n) return;
    keys[i] = rank_key_of(q, i, calibrated, preemptive, err);
}

// Unlimited KV budget: run = first min(max_batch, n) of the sorted order.
__global__ void fill_unlimited(const uint32_t* __restrict__ order, const int64_t* __restrict__ id, uint32_t n,
                               int32_t max_batch, int64_t* __restrict__ run, uint8_t* __restrict__ sched,
                               int32_t* __restrict__ counts) {
    const uint32_t m = min((uint32_t)max_batch, n);
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
        uint32_t idx = order[k];
        run[k] = id[idx];
        sched[idx] = 1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = (int32_t)m;
}

// Budgeted greedy fill, one warp. Within each 32-wide chunk of the sorted order:
// drop lanes whose own need already exceeds the remaining budget (kv_used only
// grows, so they can never fit), take the longest prefix of the rest that fits
// cumulatively, skip the first lane that does not, repeat.
__global__ void fill_budget(const uint32_t* __restrict__ order, const int32_t* __restrict__ prompt,
                            const int32_t* __restrict__ gen, const int64_t* __restrict__ id, uint32_t n,
                            int32_t max_batch, int64_t budget, int64_t* __restrict__ run,
                            uint8_t* __restrict__ sched, int32_t* __restrict__ counts) {
    const int lane = threadIdx.x;
    int64_t used = 0;
    int32_t taken = 0;
    for (uint32_t base = 0; base < n && taken < max_batch; base += 32) {
        const uint32_t k = base + lane;
        uint32_t idx = 0;
        int64_t need = 0;
        bool pending = k < n;
        if (pending) {
            idx = order[k];
            need = (int64_t)prompt[idx] + (int64_t)gen[idx] + 1;
        }
        while (taken < max_batch) {
            if (pending && need > budget - used) pending = false;  // can never fit
            unsigned mask = __ballot_sync(0xffffffffu, pending);
            if (!mask) break;
            int64_t x = pending ? need : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            // lanes that fit if every pending lane up to them is taken
            const bool fits = pending && (used + x <= budget);
            const unsigned fmask = __ballot_sync(0xffffffffu, fits);
            // the taken set is the run of fitting pending lanes before the first
            // pending lane that does not fit
            const unsigned nofit = mask & ~fmask;
            const unsigned before = nofit ? ((nofit & (0u - nofit)) - 1u) : 0xffffffffu;
            unsigned tmask = fmask & before;
            // respect max_batch: keep only the lowest (max_batch - taken) lanes
            const int room = max_batch - taken;
            if (__popc(tmask) > room) {
                unsigned m2 = tmask;
                for (int r = 0; r < room; ++r) m2 &= m2 - 1;  // drop the lowest `room` bits
                tmask &= ~m2;
            }
            const bool take = (tmask >> lane) & 1u;
            if (take) {
                const int slot = taken + __popc(tmask & ((1u << lane) - 1u));
                run[slot] = id[idx];
                sched[idx] = 1;
            }
            int64_t add = take ? need : 0;
            add = warp_sum(add);
            used += add;
            taken += __popc(tmask);
            if (take) pending = false;
            // the first non-fitting pending lane is skipped
            if (nofit && taken < max_batch) {
                const int f = __ffs(nofit) - 1;
                if (lane == f && !((tmask >> lane) & 1u)) pending = false;
            }
            if (__popc(tmask) == 0 && !nofit) break;
        }
    }
    if (lane == 0) counts[0] = taken;
}

// ---- unlimited KV budget: top-k selection instead of a full sort ------------------
// With no budget the batch is the first k = min(max_batch, n) keys of the sorted order
// (Policy._fill never skips), and the state update only needs membership. The keys are
// distinct 96-bit integers [class:3 | eff:64 | arrival rank:29], so an MSB-first radix
// select (11-bit digits, histograms of the keys still matching the chosen prefix) finds
// the bucket holding the k-th key; once that bucket holds <= SEL_CAP keys, every key at
// or below it (< k + SEL_CAP) is gathered and sorted by one block. Passes after the
// decision are no-ops (the level count is data-dependent and decided on the device).
constexpr int SEL_BITS = 11, SEL_BINS = 1 << SEL_BITS, SEL_LEVELS = 9;  // 99 >= 96 bits
constexpr int SEL_CAP = 2048;
// smaller queues stop at a smaller final bucket: the one-block sort of the candidates
// (<= k + cap keys) is then a 1024-key network instead of a 4096-key one
constexpr int SEL_CAP_SMALL = 512;
constexpr uint32_t SEL_SMALL_N = 1u << 20;
constexpr uint32_t SEL_FUSED_N = 1u << 18;  // up to here the select is one cooperative launch (<= 64 CTAs)
constexpr uint32_t SEL_CLUSTER_N = 1u << 16;  // up to here that launch is one <= 8-CTA cluster
constexpr int SEL_SORT = 4096;  // >= max_batch + SEL_CAP, power of two
// Below this many rows the full merge sort (a block-sort launch + log2(n / 2048) pass
// launches) beats the select's SEL_LEVELS histogram launches + gather + final sort: the
// engine loop's queues (10^3-10^5 rows) are all below it, cfg4's 1M queue is above.
constexpr uint32_t SEL_MIN_N_DEFAULT = 1u << 11;
// environment overrides of the select's crossovers (measurement experiments)
static uint32_t env_u32(const char* name, uint32_t dflt) {
    const char* e = getenv(name);
    return e ? (uint32_t)strtoul(e, nullptr, 10) : dflt;
}
// RS_SEL_MIN_N overrides the crossover (measurement experiments)
static uint32_t sel_min_n() {
    static const uint32_t v = [] {
        const char* e = getenv("RS_SEL_MIN_N");
        return e ? (uint32_t)strtoul(e, nullptr, 10) : SEL_MIN_N_DEFAULT;
    }();
    return v;
}
constexpr int SEL_THREADS = 1024;
constexpr int SEL_PHASE_A = 8;  // level-0 chunks per warp counted before the CTA's bin bound is fixed
// level 0 keeps its candidates only for queues this large (smaller ones: the level-1 pass
// over the columns is cheaper than level 0's second read of its phase-A rows)
constexpr uint32_t SEL_L0_KEEP_N = 1u << 23;

struct SelState {
    uint32_t dom_ok;       // level 0 left <= dom_cap rows at or below its bucket: compact them
    uint32_t compacted;    // the passes after level 1 read the compacted rows
    uint32_t dom_overflow; // a CTA's slice of the compacted buffer overflowed: keep reading columns
    uint32_t level;        // next level to histogram
    uint32_t less;         // keys strictly below the current prefix bucket
    uint32_t done;         // 1: final level reached (prefix covers the k-th key)
    uint32_t final_level;
    uint32_t n_cand;
    uint32_t arrived;  // blocks done with the current level's histogram
    uint32_t bar_count, bar_gen;  // sel_fused's grid barrier
};

// Key sources for the select. Both give each row a distinct integer whose order is the
// RankingPolicy sort order, left-aligned in BITS bits (digit L = bits
// [BITS - 11 (L + 1), BITS - 11 L)).
// SrcKeys: materialised 96-bit RankKeys [class:3 | eff(f64 image):64 | rank:29] << 3.
// V: the value type the kernels compute in; the value's virtual BITS-bit image is
// (V)value << PAD (SrcSoa64 works in 64-bit registers: no 128-bit shifts per row).
__device__ __forceinline__ unsigned __int128 rank_key_value(const RankKey& k) {
    const unsigned __int128 v = ((unsigned __int128)(k.cr >> 29) << 93) | ((unsigned __int128)k.eff << 29) |
                                (unsigned __int128)(k.cr & RANK_MASK);
    return v << 3;
}
struct SrcKeys {
    using V = unsigned __int128;
    static constexpr int BITS = 99, LEVELS = 9, PAD = 0;
    const RankKey* keys;
    __device__ __forceinline__ unsigned __int128 value(uint32_t i) const { return rank_key_value(keys[i]); }
    // split access for batched passes (sel_rows_batch): every load first, then the values
    using Raw = RankKey;
    static constexpr int BATCH = 4;
    __device__ __forceinline__ Raw load(uint32_t i) const { return keys[i]; }
    __device__ __forceinline__ unsigned __int128 finish(const Raw& r, uint32_t) const { return rank_key_value(r); }
};
// SrcSoa64: built on the fly from the queue columns (score f32, flags, arrival rank; 9 B
// per row, nothing materialised) when the effective score is the raw f32 score (not
// length calibrated): [class:3 | f32 image:32 | rank:29] << 2. The f32 -> f64 cast is
// monotone and injective, so this orders exactly like the 96-bit key.
struct SrcSoa64 {
    using V = uint64_t;
    static constexpr int BITS = 66, LEVELS = 6, PAD = 2;
    const float* score;
    const uint8_t* flags;
    const uint32_t* arrival_rank;
    int preemptive;
    int* err;
    __device__ __forceinline__ uint64_t value(uint32_t i) const {
        const uint8_t f = flags[i];
        const bool scored = f & RS_FLAG_SCORED;
        const bool prio = f & RS_FLAG_PRIORITY;
        const bool running = f & RS_FLAG_RUNNING;
        float s = 0.0f;
        if (scored) {
            s = score[i];
            if (s != s) atomicOr(err, 1);
        }
        const uint32_t pin = preemptive ? 0u : (running ? 0u : 1u);
        const uint32_t cls = (pin << 2) | ((scored ? 1u : 0u) << 1) | (prio ? 0u : 1u);
        return ((uint64_t)cls << 61) | ((uint64_t)orderable_f32(s) << 29) | (uint64_t)(arrival_rank[i] & RANK_MASK);
    }
};
// (virtual value) >> s, computed in V
template <typename Src>
__device__ __forceinline__ typename Src::V vshr(typename Src::V v, int s) {
    if (s - Src::PAD >= (int)(8 * sizeof(v))) return 0;
    return s >= Src::PAD ? (v >> (s - Src::PAD)) : (v << (Src::PAD - s));
}
template <typename Src>
__device__ __forceinline__ unsigned __int128 to128(typename Src::V v) {
    return (unsigned __int128)v << Src::PAD;
}

// Four consecutive rows i..i+3 (i % 4 == 0, all < n, 16-B aligned columns): one 16-B load
// of scores and of arrival ranks, one 4-B load of flags.
__device__ __forceinline__ void soa64_value4(const SrcSoa64& s, uint32_t i, uint64_t (&v)[4]) {
    const float4 sc = *reinterpret_cast<const float4*>(s.score + i);
    const uint4 ar = *reinterpret_cast<const uint4*>(s.arrival_rank + i);
    const uint32_t fl = *reinterpret_cast<const uint32_t*>(s.flags + i);
    const float scv[4] = {sc.x, sc.y, sc.z, sc.w};
    const uint32_t arv[4] = {ar.x, ar.y, ar.z, ar.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t f = (fl >> (8 * k)) & 0xffu;
        const bool scored = f & RS_FLAG_SCORED;
        const bool prio = f & RS_FLAG_PRIORITY;
        const bool running = f & RS_FLAG_RUNNING;
        float x = 0.0f;
        if (scored) {
            x = scv[k];
            if (x != x) atomicOr(s.err, 1);
        }
        const uint32_t pin = s.preemptive ? 0u : (running ? 0u : 1u);
        const uint32_t cls = (pin << 2) | ((scored ? 1u : 0u) << 1) | (prio ? 0u : 1u);
        v[k] = ((uint64_t)cls << 61) | ((uint64_t)orderable_f32(x) << 29) | (uint64_t)(arv[k] & RANK_MASK);
    }
}
// Class bits of the four rows of a packed flag word, one per byte (bit 2: not pinned,
// bit 1: scored, bit 0: not priority) — the RankingPolicy class order of SrcSoa64::value.
__device__ __forceinline__ uint32_t soa64_classes(uint32_t fw, int preemptive) {
    const uint32_t s1 = (fw & 0x01010101u) << 1;
    const uint32_t s0 = (~fw >> 1) & 0x01010101u;
    const uint32_t s2 = preemptive ? 0u : (~fw & 0x04040404u);
    return s2 | s1 | s0;
}
// Order-preserving image of a row's effective score (0 for unscored rows; -0.0 -> +0.0);
// NaN scores are OR-ed into nan.
__device__ __forceinline__ uint32_t soa64_img(float sc, bool scored, bool& nan) {
    const float x = scored ? sc + 0.0f : 0.0f;  // + 0.0f: -0.0 -> +0.0 (as orderable_f32)
    nan |= x != x;
    const uint32_t b = __float_as_uint(x);
    return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}
// The top 32 bits of the SoA key, (class << 29) | (f32 image >> 3), of four consecutive
// rows (aligned, all < n) from one 16-B score load and one 4-B flag load (no arrival
// ranks); lo (optional) gets the key's low word without the rank, img << 29.
__device__ __forceinline__ void soa64_hi4(const SrcSoa64& s, uint32_t i, uint32_t (&hi)[4], uint32_t* lo = nullptr) {
    const float4 sc = *reinterpret_cast<const float4*>(s.score + i);
    const uint32_t fl = *reinterpret_cast<const uint32_t*>(s.flags + i);
    const float scv[4] = {sc.x, sc.y, sc.z, sc.w};
    const uint32_t C = soa64_classes(fl, s.preemptive);
    bool nan = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t img = soa64_img(scv[k], (fl >> (8 * k)) & RS_FLAG_SCORED, nan);
        hi[k] = (((C >> (8 * k)) & 7u) << 29) | (img >> 3);
        if (lo) lo[k] = img << 29;
    }
    if (nan) atomicOr(s.err, 1);
}
// Warp-aggregated add of 1 per lane into bin `digit` of a shared histogram at shared
// address `hbase`, for all 32 lanes (warp-uniform, all lanes active): the lanes holding
// the same digit add once, from the highest such lane, by a predicated red.shared.
__device__ __forceinline__ void hist_add_all(uint32_t hbase, uint32_t digit) {
    const unsigned peers = __match_any_sync(0xffffffffu, digit);
    const uint32_t lead = (threadIdx.x & 31u) == (uint32_t)(31 - __clz(peers));
    asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p red.shared.add.u32 [%0], %1; }"
                 :: "r"(hbase + 4u * digit), "r"((uint32_t)__popc(peers)), "r"(lead) : "memory");
}
// Row loop of the select kernels: 4-row vector steps for SrcSoa64 on aligned columns,
// scalar rows otherwise (and for the tail). Trip counts are warp-uniform (f gets a valid
// flag) so f may use full-warp ballots.
template <typename Src, typename F>
__device__ __forceinline__ void sel_rows(const Src& src, uint32_t n, F&& f) {
    const uint32_t stride = gridDim.x * SEL_THREADS;
    const uint32_t wbase = blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u), lane = threadIdx.x & 31u;
    uint32_t done = 0;
    if constexpr (std::is_same<Src, SrcSoa64>::value) {
        const bool al = ((reinterpret_cast<uintptr_t>(src.score) | reinterpret_cast<uintptr_t>(src.arrival_rank)) & 15u) == 0 &&
                        (reinterpret_cast<uintptr_t>(src.flags) & 3u) == 0;
        if (al) {
            const uint32_t n4 = n & ~3u;
            for (uint32_t i0 = wbase * 4u; i0 < n4; i0 += stride * 4u) {
                const uint32_t i = i0 + lane * 4u;
                const bool ok = i < n4;
                uint64_t v[4] = {0, 0, 0, 0};
                if (ok) soa64_value4(src, i, v);
#pragma unroll
                for (int k = 0; k < 4; ++k) f(i + k, v[k], ok);
            }
            done = n4;
        }
    }
    for (uint32_t i0 = done + wbase; i0 < n; i0 += stride) {
        const uint32_t i = i0 + lane;
        const bool ok = i < n;
        f(i, ok ? src.value(i) : (typename Src::V)0, ok);
    }
}
// sel_rows for sources with a split load / finish (Src::Raw): each warp takes R x 32
// consecutive rows per step and issues all R loads before any value is handed to f, so
// a thread has R rows in flight (the small-grid passes of the fused select are bound by
// load latency, not bandwidth). Warp-uniform trip count.
template <int R, typename Src, typename F>
__device__ __forceinline__ void sel_rows_batch(const Src& src, uint32_t n, F&& f) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t stride = gridDim.x * SEL_THREADS * R;
    for (uint32_t i0 = (blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u)) * R; i0 < n; i0 += stride) {
        typename Src::Raw raw[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t i = i0 + 32u * j + lane;
            if (i < n) raw[j] = src.load(i);
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t i = i0 + 32u * j + lane;
            const bool ok = i < n;
            f(i, ok ? src.finish(raw[j], i) : (typename Src::V)0, ok);
        }
    }
}
template <typename T, typename = void>
struct has_raw : std::false_type {};
template <typename T>
struct has_raw<T, std::void_t<typename T::Raw>> : std::true_type {};
// the fused select's passes: batched where the source splits its loads
template <typename Src, typename F>
__device__ __forceinline__ void sel_rows_fused(const Src& src, uint32_t n, F&& f) {
    if constexpr (has_raw<Src>::value)
        sel_rows_batch<Src::BATCH>(src, n, f);
    else
        sel_rows(src, n, f);
}

// Like sel_rows, but hands f up to four consecutive rows per lane at once (i0, values,
// count); warp-uniform trip counts.
template <typename Src, typename F>
__device__ __forceinline__ void sel_rows4(const Src& src, uint32_t n, F&& f) {
    const uint32_t stride = gridDim.x * SEL_THREADS;
    const uint32_t wbase = blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u), lane = threadIdx.x & 31u;
    uint32_t done = 0;
    if constexpr (std::is_same<Src, SrcSoa64>::value) {
        const bool al = ((reinterpret_cast<uintptr_t>(src.score) | reinterpret_cast<uintptr_t>(src.arrival_rank)) & 15u) == 0 &&
                        (reinterpret_cast<uintptr_t>(src.flags) & 3u) == 0;
        if (al) {
            const uint32_t n4 = n & ~3u;
            for (uint32_t i0 = wbase * 4u; i0 < n4; i0 += stride * 4u) {
                const uint32_t i = i0 + lane * 4u;
                uint64_t v[4] = {0, 0, 0, 0};
                const int nv = i < n4 ? 4 : 0;
                if (nv) soa64_value4(src, i, v);
                f(i, v, nv);
            }
            done = n4;
        }
    }
    for (uint32_t i0 = done + wbase; i0 < n; i0 += stride) {
        const uint32_t i = i0 + lane;
        typename Src::V v[4] = {0, 0, 0, 0};
        const int nv = i < n ? 1 : 0;
        if (nv) v[0] = src.value(i);
        f(i, v, nv);
    }
}
// Rows already filtered by the level-1 pass: (value, row) pairs, one slice of `capc` per
// CTA (the select kernels keep the same grid, so CTA c re-reads the rows it kept).
template <typename V>
struct SrcBuf {
    const V* v;
    const uint32_t* idx;
    const uint32_t* cnt;
    uint32_t capc;
};
template <typename V, typename F>
__device__ __forceinline__ void buf_rows(const SrcBuf<V>& b, F&& f) {
    const uint32_t n = b.cnt[blockIdx.x];
    const size_t off = (size_t)blockIdx.x * b.capc;
    for (uint32_t i0 = threadIdx.x & ~31u; i0 < n; i0 += SEL_THREADS) {
        const uint32_t i = i0 + (threadIdx.x & 31u);
        const bool ok = i < n;
        f(ok ? b.idx[off + i] : 0u, ok ? b.v[off + i] : (V)0, ok);
    }
}
// warp-aggregated append of (v, row) for the lanes with p set
__device__ __forceinline__ void sel_append(bool p, unsigned __int128 v, uint32_t row, uint32_t* counter,
                                           unsigned __int128* ov, uint32_t* oi, uint32_t cap) {
    const unsigned b = __ballot_sync(0xffffffffu, p);
    if (!b) return;
    const int lane = threadIdx.x & 31, leader = __ffs(b) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(b));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (p) {
        const uint32_t pos = base + (uint32_t)__popc(b & ((1u << lane) - 1u));
        if (pos < cap) {
            ov[pos] = v;
            oi[pos] = row;
        }
    }
}

template <typename Src>
__device__ __forceinline__ uint32_t sel_digit(typename Src::V v, uint32_t level) {
    return (uint32_t)vshr<Src>(v, Src::BITS - SEL_BITS * (int)(level + 1)) & (SEL_BINS - 1);
}

template <typename Src>
__device__ void sel_pick_block(SelState* st, unsigned __int128* pfx128, uint32_t* hist, uint32_t k, uint32_t* c,
                               uint32_t dom_cap, uint32_t cap);

// Warp-aggregated shared-memory histogram increment: lanes holding the same digit add once
// (the SoA keys concentrate on few level-0 / level-1 bins: one atomic per lane would
// serialise on them). Warp-uniform call; lanes with !p take no part.
__device__ __forceinline__ void hist_add_warp(uint32_t* h, uint32_t digit, bool p) {
    if (!__any_sync(0xffffffffu, p)) return;
    const uint32_t key = p ? digit : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (p && (threadIdx.x & 31u) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[digit], (uint32_t)__popc(peers));
}

template <typename Src>
__device__ __forceinline__ bool soa64_aligned(const Src& s) {
    if constexpr (std::is_same<Src, SrcSoa64>::value)
        return ((reinterpret_cast<uintptr_t>(s.score) | reinterpret_cast<uintptr_t>(s.arrival_rank)) & 15u) == 0 &&
               (reinterpret_cast<uintptr_t>(s.flags) & 3u) == 0;
    else
        return false;
}
template <typename Src>
__device__ __forceinline__ const SrcSoa64& soa64_of(const Src& s) {
    if constexpr (std::is_same<Src, SrcSoa64>::value) return s;
    else { __trap(); return *reinterpret_cast<const SrcSoa64*>(&s); }
}
// Level 0 of the select on the score and flag columns only (aligned SrcSoa64): every row
// counted into the shared histogram h (+ a scratch bin at SEL_BINS), next chunk prefetched.
__device__ __forceinline__ void sel_l0_soa(const SrcSoa64& so, uint32_t n, uint32_t* h) {
    const uint32_t stride = gridDim.x * SEL_THREADS * 4u, lane = threadIdx.x & 31u;
    const uint32_t n4 = n & ~3u;
    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(h);
    uint32_t i = (blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u)) * 4u + lane * 4u;
    float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t fl = 0;
    if (i < n4) {
        sc = __ldcs(reinterpret_cast<const float4*>(so.score + i));
        fl = __ldcs(reinterpret_cast<const uint32_t*>(so.flags + i));
    }
    bool nan = false;
    for (; i - lane * 4u < n4; i += stride) {  // warp-uniform trip count
        const bool ok = i < n4;
        const float scv[4] = {sc.x, sc.y, sc.z, sc.w};
        const uint32_t fw = fl;
        if (i + stride < n4) {
            sc = __ldcs(reinterpret_cast<const float4*>(so.score + i + stride));
            fl = __ldcs(reinterpret_cast<const uint32_t*>(so.flags + i + stride));
        }
        const uint32_t C = soa64_classes(fw, so.preemptive);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t img = soa64_img(scv[q], (fw >> (8 * q)) & RS_FLAG_SCORED, nan);
            const uint32_t d = __byte_perm(img, C, 0x4443u + 0x0010u * q) & (SEL_BINS - 1);
            hist_add_all(hbase, ok ? d : (uint32_t)SEL_BINS);
        }
    }
    if (nan) atomicOr(so.err, 1);
    for (uint32_t t = n4 + blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u) + lane; t - lane < n;
         t += gridDim.x * SEL_THREADS) {
        const bool ok = t < n;  // tail rows (< 4), warp-uniform trip count
        hist_add_warp(h, ok ? sel_digit<SrcSoa64>(so.value(t), 0) : 0u, ok);
    }
}

// LEVEL: the level this launch histograms (the host launches LEVEL = 0, 1, ... in order;
// st->level == LEVEL unless the select is already done), so every shift is a constant.
template <typename Src, int LEVEL>
__global__ void __launch_bounds__(SEL_THREADS) sel_hist(Src src, uint32_t n, SelState* __restrict__ st,
                                                        unsigned __int128* __restrict__ pfx128,
                                                        uint32_t* __restrict__ hist, uint32_t k,
                                                        unsigned __int128* __restrict__ dom_v,
                                                        uint32_t* __restrict__ dom_i, uint32_t* __restrict__ dom_cnt,
                                                        uint32_t dom_cap, uint32_t cap) {
    if (st->done) return;
    __shared__ uint32_t h[SEL_BINS + 1];  // [SEL_BINS]: scratch for masked-off lanes
    __shared__ uint32_t scnt;
    for (int b = threadIdx.x; b < SEL_BINS; b += SEL_THREADS) h[b] = 0;
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
    const uint32_t capc = dom_cap / gridDim.x;
    using V = typename Src::V;
    constexpr uint32_t level = LEVEL;
    constexpr int shift = Src::BITS - SEL_BITS * LEVEL;
    const V wsh = (V)(*pfx128 >> shift);  // the chosen prefix digits
    V* dv = reinterpret_cast<V*>(dom_v);
    if (st->compacted) {
        buf_rows(SrcBuf<V>{dv, dom_i, dom_cnt, capc}, [&](uint32_t, V v, bool ok) {
            if (ok && vshr<Src>(v, shift) == wsh) atomicAdd(&h[sel_digit<Src>(v, level)], 1u);
        });
    } else if (LEVEL == 1 && st->dom_ok && soa64_aligned(src)) {
        // as below, on the top 32 key bits (scores + flags, 5 B per row): the level-0 digit
        // decides keep / count, the arrival rank is read only for the kept rows
        const SrcSoa64& so = soa64_of(src);
        const size_t off = (size_t)blockIdx.x * capc;
        const uint32_t w0 = (uint32_t)wsh, lane = threadIdx.x & 31u;
        auto rows = [&](uint32_t i0, const uint32_t (&hi)[4], const uint32_t (&lo)[4], int nv) {
            uint32_t keep = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t d0 = hi[q] >> 21;
                if (q < nv && d0 <= w0) keep |= 1u << q;
                hist_add_warp(h, (hi[q] >> 10) & (SEL_BINS - 1), q < nv && d0 == w0);
            }
            if (!__any_sync(0xffffffffu, keep)) return;
            const uint32_t c = __popc(keep);
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            uint32_t base = 0;
            if (lane == 31) base = atomicAdd(&scnt, tot);
            base = __shfl_sync(0xffffffffu, base, 31) + x - c;
            if (!keep) return;
            uint32_t ar[4];
            if (nv == 4) {  // the lane's four arrival ranks in one 16-B load
                const uint4 a4 = *reinterpret_cast<const uint4*>(so.arrival_rank + i0);
                ar[0] = a4.x; ar[1] = a4.y; ar[2] = a4.z; ar[3] = a4.w;
            } else {
                ar[0] = so.arrival_rank[i0];
                ar[1] = ar[2] = ar[3] = 0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (keep >> q & 1u) {
                    if (base < capc) {
                        dv[off + base] = (V)(((uint64_t)hi[q] << 32) | lo[q] | (ar[q] & RANK_MASK));
                        dom_i[off + base] = i0 + q;
                    }
                    ++base;
                }
            }
        };
        const uint32_t stride = gridDim.x * SEL_THREADS;
        const uint32_t n4 = n & ~3u;
        for (uint32_t j0 = (blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u)) * 4u; j0 < n4; j0 += stride * 4u) {
            const uint32_t i = j0 + lane * 4u;
            uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
            const int nv = i < n4 ? 4 : 0;
            if (nv) soa64_hi4(so, i, hi, lo);
            rows(i, hi, lo, nv);
        }
        for (uint32_t i = n4 + blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u) + lane; i - lane < n; i += stride) {
            uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
            const int nv = i < n ? 1 : 0;
            if (nv) {
                const uint64_t v = so.value(i);
                hi[0] = (uint32_t)(v >> 32);
                lo[0] = (uint32_t)v & ~RANK_MASK;
            }
            rows(i, hi, lo, nv);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            dom_cnt[blockIdx.x] = min(scnt, capc);
            if (scnt > capc) atomicOr(&st->dom_overflow, 1u);
        }
    } else if (LEVEL == 1 && st->dom_ok) {
        // level 1 over all rows also keeps every row at or below the level-0 bucket (all
        // candidates: the passes after this one read only them), in this CTA's slice
        const size_t off = (size_t)blockIdx.x * capc;
        sel_rows4(src, n, [&](uint32_t i0, const V (&v)[4], int nv) {
            // the lane's kept rows (<= 4), one warp scan + one shared atomic per warp
            uint32_t keep = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const V t = vshr<Src>(v[k], shift);
                if (k < nv && t <= wsh) keep |= 1u << k;
                hist_add_warp(h, sel_digit<Src>(v[k], level), k < nv && t == wsh);
            }
            if (!__any_sync(0xffffffffu, keep)) return;  // most warps keep nothing
            const uint32_t c = __popc(keep);
            uint32_t x = c;
            const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            if (!tot) return;
            uint32_t base = 0;
            if (lane == 31) base = atomicAdd(&scnt, tot);
            base = __shfl_sync(0xffffffffu, base, 31) + x - c;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (keep >> k & 1u) {
                    if (base < capc) {
                        dv[off + base] = v[k];
                        dom_i[off + base] = i0 + k;
                    }
                    ++base;
                }
            }
        });
        __syncthreads();
        if (threadIdx.x == 0) {
            dom_cnt[blockIdx.x] = min(scnt, capc);
            if (scnt > capc) atomicOr(&st->dom_overflow, 1u);
        }
    } else if (LEVEL == 0 && soa64_aligned(src) && n >= SEL_L0_KEEP_N) {
        // Level 0 on scores + flags only (5 B per row): the digit is (class << 8) | the top
        // byte of the f32 image. Phase A counts every row of the warp's first SEL_PHASE_A
        // chunks; the CTA then knows a bin U holding, with all bins below it, >= k of its
        // own rows, so the k-th key's bin is <= U. Phase B counts only rows at or below U
        // and keeps them (full key + row) in this CTA's slice of the candidate buffer; the
        // phase-A rows at or below U are kept by a second (L2-resident) read at the end.
        // With every slice in capacity the later levels read only the kept rows (no
        // level-1 pass over the columns); otherwise level 1 runs its own keep pass.
        const SrcSoa64& so = soa64_of(src);
        const uint32_t stride = gridDim.x * SEL_THREADS * 4u, lane = threadIdx.x & 31u;
        const uint32_t n4 = n & ~3u;
        const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(h);
        const size_t off = (size_t)blockIdx.x * capc;
        const uint32_t i_first = (blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u)) * 4u + lane * 4u;
        __shared__ uint32_t sU;
        bool nan = false;
        // keep (v, row) of the lane's rows in `keep` (bit q: row i + q), warp-aggregated
        // mark (bit 31 of the stored row index): a phase-A row, already counted. Phase-B rows
        // are counted from the slice at the end (or here, when the slice is full)
        auto append = [&](uint32_t i, uint32_t keep, const uint32_t (&img)[4], uint32_t C, uint32_t mark) {
            if (!__any_sync(0xffffffffu, keep)) return;
            const uint32_t c = __popc(keep);
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            uint32_t base = 0;
            if (lane == 31) base = atomicAdd(&scnt, tot);
            base = __shfl_sync(0xffffffffu, base, 31) + x - c;
            if (!keep) return;
            const uint4 a4 = *reinterpret_cast<const uint4*>(so.arrival_rank + i);
            const uint32_t ar[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (keep >> q & 1u) {
                    const uint64_t v = (((uint64_t)((C >> (8 * q)) & 7u)) << 61) | ((uint64_t)img[q] << 29) |
                                       (uint64_t)(ar[q] & RANK_MASK);
                    if (base < capc) {
                        dv[off + base] = (V)v;
                        dom_i[off + base] = (i + q) | mark;
                    } else if (!mark) {
                        atomicAdd(&h[(uint32_t)(v >> 53)], 1u);  // dropped (slice full): count now
                    }
                    ++base;
                }
            }
        };
        // one chunk of four rows per lane: count (rows <= U), keep (rows <= U when `kp`)
        auto chunk = [&](uint32_t i, float4 sc, uint32_t fw, uint32_t U, bool phase_a) {
            const bool ok = i < n4;
            const float scv[4] = {sc.x, sc.y, sc.z, sc.w};
            const uint32_t C = soa64_classes(fw, so.preemptive);
            uint32_t img[4], keep = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                img[q] = soa64_img(scv[q], (fw >> (8 * q)) & RS_FLAG_SCORED, nan);
                const uint32_t d = __byte_perm(img[q], C, 0x4443u + 0x0010u * q) & (SEL_BINS - 1);
                const bool p = ok && d <= U;
                keep |= (p ? 1u : 0u) << q;
                if (phase_a) hist_add_all(hbase, p ? d : (uint32_t)SEL_BINS);  // every row counted
            }
            if (!phase_a) append(i, keep, img, C, 0u);
        };
        auto load = [&](uint32_t i, float4& sc, uint32_t& fl) {
            sc = make_float4(0.f, 0.f, 0.f, 0.f);
            fl = 0;
            if (i < n4) {
                sc = __ldcs(reinterpret_cast<const float4*>(so.score + i));
                fl = __ldcs(reinterpret_cast<const uint32_t*>(so.flags + i));
            }
        };
        // phase A (block-uniform: SEL_PHASE_A chunks per warp, masked past n4)
        for (int it = 0; it < SEL_PHASE_A; ++it) {
            float4 sc;
            uint32_t fl;
            const uint32_t i = i_first + it * stride;
            load(i, sc, fl);
            chunk(i, sc, fl, SEL_BINS - 1, true);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // U = first bin whose inclusive prefix count reaches k
            uint32_t acc = 0, U = SEL_BINS - 1;
            for (uint32_t b0 = 0; b0 < SEL_BINS; b0 += 32) {
                uint32_t x = h[b0 + lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, acc + x >= k);
                if (hit) {
                    U = b0 + (uint32_t)(__ffs(hit) - 1);
                    break;
                }
                acc += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) sU = U;
        }
        __syncthreads();
        const uint32_t U = sU;
        // phase B, the next chunk's loads issued before this one is processed
        {
            uint32_t i = i_first + SEL_PHASE_A * stride;
            float4 sc;
            uint32_t fl;
            load(i, sc, fl);
            for (; i - lane * 4u < n4; i += stride) {  // warp-uniform trip count
                const float4 cs = sc;
                const uint32_t cf = fl;
                load(i + stride, sc, fl);
                chunk(i, cs, cf, U, false);
            }
        }
        // phase-A rows at or below U (no counting: they are in the histogram already)
        for (int it = 0; it < SEL_PHASE_A; ++it) {
            const uint32_t i = i_first + it * stride;
            if (i - lane * 4u >= n4) break;  // warp-uniform
            float4 sc;
            uint32_t fl;
            load(i, sc, fl);
            const bool ok = i < n4;
            const float scv[4] = {sc.x, sc.y, sc.z, sc.w};
            const uint32_t C = soa64_classes(fl, so.preemptive);
            uint32_t img[4], keep = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                img[q] = soa64_img(scv[q], (fl >> (8 * q)) & RS_FLAG_SCORED, nan);
                const uint32_t d = __byte_perm(img[q], C, 0x4443u + 0x0010u * q) & (SEL_BINS - 1);
                keep |= ((ok && d <= U) ? 1u : 0u) << q;
            }
            append(i, keep, img, C, 0x80000000u);
        }
        if (nan) atomicOr(so.err, 1);
        // tail rows (< 4): counted and kept one per lane, warp-uniform trip count
        for (uint32_t t = n4 + blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u) + lane; t - lane < n;
             t += gridDim.x * SEL_THREADS) {
            const bool ok = t < n;
            const uint64_t v = ok ? so.value(t) : 0ull;
            const uint32_t d = (uint32_t)(v >> 53);
            hist_add_warp(h, d, ok);
            const bool kp = ok && d <= U;
            const unsigned bb = __ballot_sync(0xffffffffu, kp);
            if (bb) {
                uint32_t base = 0;
                if (lane == (uint32_t)(__ffs(bb) - 1)) base = atomicAdd(&scnt, (uint32_t)__popc(bb));
                base = __shfl_sync(0xffffffffu, base, __ffs(bb) - 1) + (uint32_t)__popc(bb & ((1u << lane) - 1u));
                if (kp && base < capc) {
                    dv[off + base] = (V)v;
                    dom_i[off + base] = t | 0x80000000u;  // counted above
                }
            }
        }
        __syncthreads();
        // count the stored phase-B rows; clear the marks
        const uint32_t ns = min(scnt, capc);
        for (uint32_t e = threadIdx.x; e < ns; e += SEL_THREADS) {
            const uint32_t r = dom_i[off + e];
            if (r & 0x80000000u) dom_i[off + e] = r & 0x7fffffffu;
            else atomicAdd(&h[(uint32_t)((uint64_t)dv[off + e] >> 53)], 1u);
        }
        if (threadIdx.x == 0) {
            dom_cnt[blockIdx.x] = ns;
            if (scnt > capc) atomicOr(&st->dom_overflow, 1u);
        }
    } else if (LEVEL == 0 && soa64_aligned(src)) {
        // smaller queues: the same digit from scores + flags, every row counted, no keep
        sel_l0_soa(soa64_of(src), n, h);
    } else {
        sel_rows(src, n, [&](uint32_t, V v, bool ok) {
            hist_add_warp(h, sel_digit<Src>(v, level), ok && (LEVEL == 0 || vshr<Src>(v, shift) == wsh));
        });
    }
    __syncthreads();
    for (int b = threadIdx.x; b < SEL_BINS; b += SEL_THREADS)
        if (h[b]) atomicAdd(&hist[b], h[b]);
    // the last block to finish picks the bucket (no separate launch per level)
    __threadfence();
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->arrived, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
        __threadfence();
        if (threadIdx.x == 0) {
            if (LEVEL == 0 && soa64_aligned(src) && n >= SEL_L0_KEEP_N && !st->dom_overflow) st->compacted = 1;  // kept by level 0
            if (LEVEL == 0) st->dom_overflow = 0;  // level 1's own keep pass (if any) starts clean
            if (LEVEL == 1 && st->dom_ok && !st->dom_overflow) st->compacted = 1;
        }
        sel_pick_block<Src>(st, pfx128, hist, k, h, dom_cap, cap);
    }
}

// The bin holding the need-th key (need >= 1 <= the bins' total), 1024-thread block, thread
// t holding bins (t / 32) * 64 + t % 32 and + 32: each warp sums its 64 bins, warp 0 scans
// the 32 sums, the warp owning the bin scans its own 64. pick / below (the keys in the
// bins before it) returned to every thread.
__device__ __forceinline__ void sel_bin_search(uint32_t c0, uint32_t c1, uint32_t need, uint32_t& pick_out,
                                               uint32_t& below_out) {
    static_assert(SEL_BINS == 64 * (SEL_THREADS / 32), "64 bins per warp");
    __shared__ uint32_t pick, below, wsum[32], wsel, wbefore;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t ws = warp_sum(c0 + c1);
    if (lane == 0) wsum[wid] = ws;
    __syncthreads();
    if (wid == 0) {
        const uint32_t v = wsum[lane];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, x >= need);
        const int f = __ffs(hit) - 1;
        if (lane == f) {
            wsel = (uint32_t)f;
            wbefore = x - v;
        }
    }
    __syncthreads();
    if (wid == (int)wsel) {
        uint32_t acc = wbefore;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const uint32_t v = half ? c1 : c0;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, acc + x >= need);
            if (hit) {
                const int f = __ffs(hit) - 1;
                if (lane == f) {
                    pick = (uint32_t)(wid * 64 + half * 32 + f);
                    below = acc + x - v;
                }
                break;
            }
            acc += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    __syncthreads();
    pick_out = pick;
    below_out = below;
}

// The fused select's per-CTA copy of the pick state (the engine loop: every CTA picks from
// the per-CTA histogram slices itself, no second barrier per level).
struct SelLocal {
    unsigned __int128 pfx;
    uint32_t less, level, done, final_level;
};
template <typename Src>
__device__ __forceinline__ void sel_pick_local(SelLocal& L, const uint32_t* __restrict__ slices, uint32_t nsl,
                                               uint32_t k, uint32_t cap) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t c0 = 0, c1 = 0;
    for (uint32_t s = 0; s < nsl; ++s) {
        c0 += __ldcg(&slices[s * SEL_BINS + wid * 64 + lane]);
        c1 += __ldcg(&slices[s * SEL_BINS + wid * 64 + 32 + lane]);
    }
    uint32_t pick, below;
    sel_bin_search(c0, c1, k - L.less, pick, below);
    const int pl = (int)(pick & 63u);
    if (wid == (int)(pick >> 6) && lane == (pl & 31)) {  // the thread holding the bin
        const uint32_t cnt = pl < 32 ? c0 : c1;
        const uint32_t level = L.level;
        L.pfx |= (unsigned __int128)pick << (Src::BITS - SEL_BITS * (level + 1));
        L.less += below;
        L.level = level + 1;
        if (cnt <= cap || level + 1 == Src::LEVELS) {
            L.done = 1;
            L.final_level = level + 1;
        }
    }
    __syncthreads();
}

// One block: choose the bucket holding the k-th key from the level's global histogram
// (c = shared scratch of SEL_BINS words), clear the histogram for the next level.
template <typename Src>
__device__ void sel_pick_block(SelState* st, unsigned __int128* pfx128, uint32_t* hist, uint32_t k, uint32_t* c,
                               uint32_t dom_cap, uint32_t cap) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t c0 = __ldcg(&hist[wid * 64 + lane]), c1 = __ldcg(&hist[wid * 64 + 32 + lane]);
    c[wid * 64 + lane] = c0;
    c[wid * 64 + 32 + lane] = c1;
    uint32_t pick, below;
    sel_bin_search(c0, c1, k - st->less, pick, below);
    for (int b = threadIdx.x; b < SEL_BINS; b += SEL_THREADS) hist[b] = 0;
    if (threadIdx.x == 0) {
        const uint32_t level = st->level;
        *pfx128 |= (unsigned __int128)pick << (Src::BITS - SEL_BITS * (level + 1));
        st->less += below;
        st->level = level + 1;
        st->arrived = 0;
        if (level == 0) st->dom_ok = (st->less + c[pick] <= dom_cap) ? 1u : 0u;
        if (c[pick] <= cap || level + 1 == Src::LEVELS) {
            st->done = 1;
            st->final_level = level + 1;
        }
    }
}

// every key at or below the chosen bucket (exactly st->less + bucket size of them)
template <typename Src>
__global__ void __launch_bounds__(SEL_THREADS) sel_gather(Src src, uint32_t n, SelState* __restrict__ st,
                                                          const unsigned __int128* __restrict__ pfx128,
                                                          unsigned __int128* __restrict__ ck, uint32_t* __restrict__ ci,
                                                          const unsigned __int128* __restrict__ dom_v,
                                                          const uint32_t* __restrict__ dom_i,
                                                          const uint32_t* __restrict__ dom_cnt, uint32_t dom_cap) {
    using V = typename Src::V;
    const int shift = Src::BITS - SEL_BITS * (int)st->final_level;
    const V lim = (V)(*pfx128 >> shift);
    auto take = [&](uint32_t i, V v, bool ok) {
        sel_append(ok && vshr<Src>(v, shift) <= lim, to128<Src>(v), i, &st->n_cand, ck, ci, SEL_SORT);
    };
    if (st->compacted)
        buf_rows(SrcBuf<V>{reinterpret_cast<const V*>(dom_v), dom_i, dom_cnt, dom_cap / gridDim.x}, take);
    else
        sel_rows(src, n, take);
}

// one block: sort the <= SEL_SORT candidates (bitonic, smem), emit the first k in order
__global__ void __launch_bounds__(SEL_THREADS) sel_sort_emit(const unsigned __int128* __restrict__ ck,
                                                             const uint32_t* __restrict__ ci,
                                                             const SelState* __restrict__ st,
                                                             const int64_t* __restrict__ id, uint32_t k,
                                                             int64_t* __restrict__ run, uint8_t* __restrict__ sched,
                                                             int32_t* __restrict__ counts) {
    extern __shared__ __align__(16) uint8_t sm[];
    unsigned __int128* sk = reinterpret_cast<unsigned __int128*>(sm);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + SEL_SORT);
    const uint32_t m = min(st->n_cand, (uint32_t)SEL_SORT);
    uint32_t P = 1;
    while (P < m) P <<= 1;
    for (uint32_t i = threadIdx.x; i < P; i += SEL_THREADS) {
        if (i < m) {
            sk[i] = ck[i];
            sv[i] = ci[i];
        } else {
            sk[i] = ~(unsigned __int128)0;
            sv[i] = 0xffffffffu;
        }
    }
    __syncthreads();
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            // one compare-exchange per thread slot (pairs enumerated directly, no idle half)
            for (uint32_t t = threadIdx.x; t < (P >> 1); t += SEL_THREADS) {
                const uint32_t i = 2 * stride * (t / stride) + (t % stride), j = i + stride;
                const bool up = (i & size) == 0;
                const unsigned __int128 a = sk[i], b = sk[j];
                const bool swap = up ? (b < a) : (a < b);
                if (swap) {
                    sk[i] = b;
                    sk[j] = a;
                    const uint32_t tv = sv[i];
                    sv[i] = sv[j];
                    sv[j] = tv;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t r = threadIdx.x; r < k; r += SEL_THREADS) {
        const uint32_t idx = sv[r];
        run[r] = id[idx];
        sched[idx] = 1;
    }
    if (threadIdx.x == 0) counts[0] = (int32_t)k;
}

// The same for <= 1024 candidates: one element per thread, the bitonic stages of stride
// < 32 over warp shuffles (no barriers), the wider ones through shared memory. Keys are
// distinct (the arrival rank is in them), so the network's order is the sort order.
__device__ __forceinline__ bool u128_less(const uint4& a, const uint4& b) {  // .w most significant
    if (a.w != b.w) return a.w < b.w;
    if (a.z != b.z) return a.z < b.z;
    if (a.y != b.y) return a.y < b.y;
    return a.x < b.x;
}
// one 1024-thread block; sk / sv: shared scratch of 1024 entries
__device__ __forceinline__ void sel_emit_small_block(const unsigned __int128* __restrict__ ck,
                                                     const uint32_t* __restrict__ ci, uint32_t n_cand,
                                                     const int64_t* __restrict__ id, uint32_t k,
                                                     int64_t* __restrict__ run, uint8_t* __restrict__ sched,
                                                     int32_t* __restrict__ counts, uint4* sk, uint32_t* sv) {
    const uint32_t m = min(n_cand, 1024u);
    uint32_t P = 32;
    while (P < m) P <<= 1;
    const uint32_t t = threadIdx.x;
    uint4 v = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    uint32_t ix = 0xffffffffu;
    if (t < m) {
        v = *reinterpret_cast<const uint4*>(ck + t);
        ix = ci[t];
    }
    for (uint32_t kk = 2; kk <= P; kk <<= 1) {
        const bool up = (t & kk) == 0;
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            uint4 o;
            uint32_t oi;
            if (j >= 32) {  // block-uniform branch
                __syncthreads();
                if (t < P) {
                    sk[t] = v;
                    sv[t] = ix;
                }
                __syncthreads();
                if (t < P) {
                    o = sk[t ^ j];
                    oi = sv[t ^ j];
                }
            } else {
                o.x = __shfl_xor_sync(0xffffffffu, v.x, j);
                o.y = __shfl_xor_sync(0xffffffffu, v.y, j);
                o.z = __shfl_xor_sync(0xffffffffu, v.z, j);
                o.w = __shfl_xor_sync(0xffffffffu, v.w, j);
                oi = __shfl_xor_sync(0xffffffffu, ix, j);
            }
            if (t < P) {
                const bool lower = (t & j) == 0;
                const bool take_o = (lower == up) ? u128_less(o, v) : u128_less(v, o);
                if (take_o) {
                    v = o;
                    ix = oi;
                }
            }
        }
    }
    if (t < k && t < P) {
        run[t] = id[ix];
        sched[ix] = 1;
    }
    if (t == 0) counts[0] = (int32_t)k;
}
// The same emit spread over every CTA of a fused select: each candidate's place in the
// order is the number of candidates with a smaller key (the <= 1024 keys staged in each
// CTA's shared memory; a CTA ranks every gridDim.x-th candidate, S threads per candidate
// over strided slices of the keys). Live keys are distinct; the finished rows the engine
// loop leaves in place share the all-ones key, above every live one, so they never place
// below k. counts[0] = k.
// thr (optional): the key placed at rank `target` is stored there (all ones if there are
// <= target candidates) — the engine loop's next speculative threshold.
__device__ __forceinline__ void sel_emit_rank(const unsigned __int128* __restrict__ ck,
                                              const uint32_t* __restrict__ ci, uint32_t n_cand,
                                              const int64_t* __restrict__ id, uint32_t k, int64_t* __restrict__ run,
                                              uint8_t* __restrict__ sched, int32_t* __restrict__ counts, uint4* sk,
                                              unsigned __int128* thr = nullptr, uint32_t target = 0,
                                              uint32_t* __restrict__ run_row = nullptr) {
    const uint32_t m = min(n_cand, 1024u), t = threadIdx.x;
    for (uint32_t i = t; i < m; i += blockDim.x) sk[i] = __ldcg(reinterpret_cast<const uint4*>(ck + i));
    if (blockIdx.x == 0 && t == 0) {
        counts[0] = (int32_t)k;
        if (thr != nullptr && m <= target) *thr = ~(unsigned __int128)0;
    }
    __syncthreads();
    const uint32_t G = gridDim.x;
    const uint32_t nl = m > blockIdx.x ? (m - blockIdx.x + G - 1) / G : 0u;  // this CTA's candidates
    if (nl == 0) return;
    uint32_t S = 32;
    while (S > 1 && S * nl > blockDim.x) S >>= 1;
    for (uint32_t base = 0; base < nl * S; base += blockDim.x) {  // (one pass unless nl > blockDim.x)
        const uint32_t w = base + t, j = w / S, seg = w % S;
        const bool act = j < nl;
        const uint32_t c = blockIdx.x + j * G;
        uint32_t cnt = 0;
        if (act) {
            const uint4 key = sk[c];
            for (uint32_t x = seg; x < m; x += S) cnt += u128_less(sk[x], key) ? 1u : 0u;
        }
        for (uint32_t o = S >> 1; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (act && seg == 0 && cnt < k) {
            const uint32_t row = __ldcg(ci + c);
            run[cnt] = id[row];
            sched[row] = 1;
            if (run_row != nullptr) run_row[cnt] = row;
        }
        if (thr != nullptr && act && seg == 0 && cnt == target) {
            const uint4 kv = sk[c];
            *reinterpret_cast<uint4*>(thr) = kv;
        }
    }
}
__global__ void __launch_bounds__(1024) sel_sort_emit_small(const unsigned __int128* __restrict__ ck,
                                                            const uint32_t* __restrict__ ci,
                                                            const SelState* __restrict__ st,
                                                            const int64_t* __restrict__ id, uint32_t k,
                                                            int64_t* __restrict__ run, uint8_t* __restrict__ sched,
                                                            int32_t* __restrict__ counts) {
    __shared__ uint4 sk[1024];
    __shared__ uint32_t sv[1024];
    sel_emit_small_block(ck, ci, st->n_cand, id, k, run, sched, counts, sk, sv);
}

constexpr int UPD_THREADS = 1024;
constexpr int UPD_ITEMS = 4;  // rows per thread: element k * UPD_THREADS + tid of the block's chunk
constexpr int UPD_CHUNK = UPD_THREADS * UPD_ITEMS;

// State update (schedulers.py:224-240) + per-block counts of promoted / demoted.
__global__ void __launch_bounds__(UPD_THREADS) starvation_update(rs_queue_soa q, const uint8_t* __restrict__ sched,
                                                                 int32_t threshold, int32_t pquantum,
                                                                 uint8_t* __restrict__ pd, uint32_t* __restrict__ bcnt) {
    __shared__ uint32_t wsum[2][UPD_THREADS / 32];
    uint32_t np = 0, nd = 0;
#pragma unroll
    for (int k = 0; k < UPD_ITEMS; ++k) {
        const uint32_t i = blockIdx.x * UPD_CHUNK + k * UPD_THREADS + threadIdx.x;
        if (i >= (uint32_t)q.n) break;
        uint8_t code = 0;
        uint8_t f = q.flags[i];
        int32_t st = q.starvation[i];
        int32_t qu = q.quantum[i];
        bool prio = f & RS_FLAG_PRIORITY;
        if (sched[i]) {
            st = 0;
            if (prio) qu -= 1;
        } else {
            st += 1;
        }
        if (threshold > 0 && st >= threshold) {
            prio = true;
            qu = pquantum;
            st = 0;
            code = 1;
        } else if (prio && qu <= 0) {
            prio = false;
            code = 2;
        }
        q.flags[i] = prio ? (f | RS_FLAG_PRIORITY) : (f & ~RS_FLAG_PRIORITY);
        q.starvation[i] = st;
        q.quantum[i] = qu;
        pd[i] = code;
        np += code == 1;
        nd += code == 2;
    }
    np = warp_sum(np);
    nd = warp_sum(nd);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        wsum[0][w] = np;
        wsum[1][w] = nd;
    }
    __syncthreads();
    if (w == 0) {
        uint32_t a = wsum[0][lane], b = wsum[1][lane];
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
            bcnt[2 * blockIdx.x] = a;
            bcnt[2 * blockIdx.x + 1] = b;
        }
    }
}

// Exclusive scan of the interleaved (promoted, demoted) block counts by one block
// (per-thread chunk sums, then warp-shuffle scans); writes the totals to counts[1, 2].
// (one 1024-thread block; src == dst allowed: each thread reads its entries before writing them)
__device__ __forceinline__ void scan_pairs_block(const uint32_t* src, uint32_t* dst, uint32_t nblk,
                                                 int32_t* __restrict__ counts) {
    __shared__ uint32_t wp[32], wd[32];
    const uint32_t per = (nblk + 1023) / 1024;
    const uint32_t b0 = threadIdx.x * per, b1 = min(nblk, b0 + per);
    uint32_t sp = 0, sd = 0;
    for (uint32_t b = b0; b < b1; ++b) {
        sp += src[2 * b];
        sd += src[2 * b + 1];
    }
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t ip = sp, id2 = sd;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yp = __shfl_up_sync(0xffffffffu, ip, o), yd = __shfl_up_sync(0xffffffffu, id2, o);
        if (lane >= (uint32_t)o) {
            ip += yp;
            id2 += yd;
        }
    }
    if (lane == 31) {
        wp[w] = ip;
        wd[w] = id2;
    }
    __syncthreads();
    if (w == 0) {
        uint32_t xp = wp[lane], xd = wd[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yp = __shfl_up_sync(0xffffffffu, xp, o), yd = __shfl_up_sync(0xffffffffu, xd, o);
            if (lane >= (uint32_t)o) {
                xp += yp;
                xd += yd;
            }
        }
        wp[lane] = xp;  // inclusive over warps
        wd[lane] = xd;
        if (lane == 31) {
            counts[1] = (int32_t)xp;
            counts[2] = (int32_t)xd;
        }
    }
    __syncthreads();
    uint32_t ap = (w ? wp[w - 1] : 0u) + ip - sp, ad = (w ? wd[w - 1] : 0u) + id2 - sd;
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t vp = src[2 * b], vd = src[2 * b + 1];
        dst[2 * b] = ap;
        dst[2 * b + 1] = ad;
        ap += vp;
        ad += vd;
    }
}
__global__ void __launch_bounds__(1024) scan_pairs(uint32_t* __restrict__ bcnt, uint32_t nblk,
                                                   int32_t* __restrict__ counts) {
    scan_pairs_block(bcnt, bcnt, nblk, counts);
}

// Order-preserving compaction of the promoted / demoted ids: within a block, rows in
// (item k, warp, lane) order = index order; per-(k, warp) counts scanned by one warp.
__global__ void __launch_bounds__(UPD_THREADS) scatter_pd(const uint8_t* __restrict__ pd,
                                                          const int64_t* __restrict__ id, uint32_t n,
                                                          const uint32_t* __restrict__ boff,
                                                          int64_t* __restrict__ prom, int64_t* __restrict__ dem) {
    constexpr int NW = UPD_THREADS / 32;
    __shared__ uint32_t cp[UPD_ITEMS * NW], cd[UPD_ITEMS * NW];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint8_t c[UPD_ITEMS];
    unsigned bp[UPD_ITEMS], bd[UPD_ITEMS];
#pragma unroll
    for (int k = 0; k < UPD_ITEMS; ++k) {
        const uint32_t i = blockIdx.x * UPD_CHUNK + k * UPD_THREADS + threadIdx.x;
        c[k] = i < n ? pd[i] : 0;
        bp[k] = __ballot_sync(0xffffffffu, c[k] == 1);
        bd[k] = __ballot_sync(0xffffffffu, c[k] == 2);
        if (lane == 0) {
            cp[k * NW + w] = __popc(bp[k]);
            cd[k * NW + w] = __popc(bd[k]);
        }
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of UPD_ITEMS * NW = 128 counts, 4 per lane
        uint32_t vp[UPD_ITEMS], vd[UPD_ITEMS], sp = 0, sd = 0;
#pragma unroll
        for (int j = 0; j < UPD_ITEMS; ++j) {
            vp[j] = cp[lane * UPD_ITEMS + j];
            vd[j] = cd[lane * UPD_ITEMS + j];
            sp += vp[j];
            sd += vd[j];
        }
        uint32_t ip = sp, id2 = sd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yp = __shfl_up_sync(0xffffffffu, ip, o), yd = __shfl_up_sync(0xffffffffu, id2, o);
            if (lane >= (uint32_t)o) {
                ip += yp;
                id2 += yd;
            }
        }
        uint32_t ap = ip - sp, ad = id2 - sd;
#pragma unroll
        for (int j = 0; j < UPD_ITEMS; ++j) {
            cp[lane * UPD_ITEMS + j] = ap;
            cd[lane * UPD_ITEMS + j] = ad;
            ap += vp[j];
            ad += vd[j];
        }
    }
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
    const uint32_t bp0 = boff[2 * blockIdx.x], bd0 = boff[2 * blockIdx.x + 1];
#pragma unroll
    for (int k = 0; k < UPD_ITEMS; ++k) {
        const uint32_t i = blockIdx.x * UPD_CHUNK + k * UPD_THREADS + threadIdx.x;
        if (c[k] == 1) prom[bp0 + cp[k * NW + w] + __popc(bp[k] & below)] = id[i];
        if (c[k] == 2) dem[bd0 + cd[k * NW + w] + __popc(bd[k] & below)] = id[i];
    }
}


// ---- vectorised state update + compaction (aligned columns) --------------------------
// Each thread owns 4 consecutive rows per iteration (16-B int4 starvation / quantum, 4-B
// flag / sched / code words); rows of a block are in (iteration, thread, sub-row) order =
// index order, so the compaction stays order-preserving.
constexpr int UPV_T = 1024, UPV_IT = 4, UPV_CHUNK = UPV_T * 4 * UPV_IT;  // 16K rows per block

__device__ __forceinline__ uint8_t upd_row(uint8_t& f, int32_t& st, int32_t& qu, bool sched, int32_t threshold,
                                           int32_t pquantum) {
    bool prio = f & RS_FLAG_PRIORITY;
    uint8_t code = 0;
    if (sched) {
        st = 0;
        if (prio) qu -= 1;
    } else {
        st += 1;
    }
    if (threshold > 0 && st >= threshold) {
        prio = true;
        qu = pquantum;
        st = 0;
        code = 1;
    } else if (prio && qu <= 0) {
        prio = false;
        code = 2;
    }
    f = prio ? (f | RS_FLAG_PRIORITY) : (f & ~RS_FLAG_PRIORITY);
    return code;
}

// Also compacts, order-preserving within the block, the promoted / demoted row indices
// into plist / dlist at the block's slice (the rows are few: the copy kernel then reads
// only them instead of a per-row code array).
// (one 1024-thread block per 16K-row chunk; also run inside sel_fused)
__device__ __forceinline__ void upd_chunk_v(const rs_queue_soa& q, const uint8_t* __restrict__ sched,
                                            int32_t threshold, int32_t pquantum, uint32_t* __restrict__ plist,
                                            uint32_t* __restrict__ dlist, uint32_t* __restrict__ bcnt,
                                            const uint32_t chunk) {
    constexpr int NW = UPV_T / 32;
    __shared__ uint32_t cp[UPV_IT * NW], cd[UPV_IT * NW];
    const uint32_t n = (uint32_t)q.n;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t codes[UPV_IT], ep[UPV_IT], ed[UPV_IT];
#pragma unroll
    for (int it = 0; it < UPV_IT; ++it) {
        const uint32_t i = chunk * UPV_CHUNK + it * (UPV_T * 4) + threadIdx.x * 4;
        if (i + 3 < n) {
            uint32_t fw = *reinterpret_cast<const uint32_t*>(q.flags + i);
            const uint32_t sw = *reinterpret_cast<const uint32_t*>(sched + i);
            int4 st = *reinterpret_cast<const int4*>(q.starvation + i);
            int4 qu = *reinterpret_cast<const int4*>(q.quantum + i);
            int32_t sa[4] = {st.x, st.y, st.z, st.w}, qa[4] = {qu.x, qu.y, qu.z, qu.w};
            uint32_t cw = 0, nf = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint8_t f = (uint8_t)(fw >> (8 * k));
                const uint8_t c = upd_row(f, sa[k], qa[k], (sw >> (8 * k)) & 0xffu, threshold, pquantum);
                nf |= (uint32_t)f << (8 * k);
                cw |= (uint32_t)c << (8 * k);
            }
            *reinterpret_cast<uint32_t*>(q.flags + i) = nf;
            *reinterpret_cast<int4*>(q.starvation + i) = make_int4(sa[0], sa[1], sa[2], sa[3]);
            *reinterpret_cast<int4*>(q.quantum + i) = make_int4(qa[0], qa[1], qa[2], qa[3]);
            codes[it] = cw;
        } else {
            uint32_t cw = 0;
            for (uint32_t r = i; r < min(i + 4, n); ++r) {
                uint8_t f = q.flags[r];
                int32_t st = q.starvation[r], qu = q.quantum[r];
                const uint8_t c = upd_row(f, st, qu, sched[r], threshold, pquantum);
                q.flags[r] = f;
                q.starvation[r] = st;
                q.quantum[r] = qu;
                cw |= (uint32_t)c << (8 * (r - i));
            }
            codes[it] = cw;
        }
        uint32_t a = 0, b = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t ck = (codes[it] >> (8 * k)) & 0xffu;
            a += ck == 1;
            b += ck == 2;
        }
        uint32_t xa = a, xb = b;  // inclusive warp scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= (uint32_t)o) {
                xa += ya;
                xb += yb;
            }
        }
        ep[it] = xa - a;
        ed[it] = xb - b;
        if (lane == 31) {
            cp[it * NW + w] = xa;
            cd[it * NW + w] = xb;
        }
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the UPV_IT * NW (iteration, warp) totals, 4 per lane
        uint32_t vp[UPV_IT], vd[UPV_IT], sp = 0, sd = 0;
#pragma unroll
        for (int j = 0; j < UPV_IT; ++j) {
            vp[j] = cp[lane * UPV_IT + j];
            vd[j] = cd[lane * UPV_IT + j];
            sp += vp[j];
            sd += vd[j];
        }
        uint32_t ip = sp, id2 = sd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yp = __shfl_up_sync(0xffffffffu, ip, o), yd = __shfl_up_sync(0xffffffffu, id2, o);
            if (lane >= (uint32_t)o) {
                ip += yp;
                id2 += yd;
            }
        }
        uint32_t ap = ip - sp, ad = id2 - sd;
#pragma unroll
        for (int j = 0; j < UPV_IT; ++j) {
            cp[lane * UPV_IT + j] = ap;
            cd[lane * UPV_IT + j] = ad;
            ap += vp[j];
            ad += vd[j];
        }
        if (lane == 31) {
            bcnt[2 * chunk] = ip;
            bcnt[2 * chunk + 1] = id2;
        }
    }
    __syncthreads();
    const uint32_t base = chunk * UPV_CHUNK;
#pragma unroll
    for (int it = 0; it < UPV_IT; ++it) {
        if (!codes[it]) continue;
        const uint32_t i = base + it * (UPV_T * 4) + threadIdx.x * 4;
        uint32_t op = cp[it * NW + w] + ep[it], od = cd[it * NW + w] + ed[it];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t ck = (codes[it] >> (8 * k)) & 0xffu;
            if (ck == 1) plist[base + op++] = i + k;
            if (ck == 2) dlist[base + od++] = i + k;
        }
    }
}
__global__ void __launch_bounds__(UPV_T) starvation_update_v(rs_queue_soa q, const uint8_t* __restrict__ sched,
                                                             int32_t threshold, int32_t pquantum,
                                                             uint32_t* __restrict__ plist, uint32_t* __restrict__ dlist,
                                                             uint32_t* __restrict__ bcnt) {
    upd_chunk_v(q, sched, threshold, pquantum, plist, dlist, bcnt, blockIdx.x);
}

// promoted / demoted ids from the per-block lists, at the scanned block offsets
__device__ __forceinline__ void copy_pd_chunk(const uint32_t* __restrict__ plist, const uint32_t* __restrict__ dlist,
                                              const uint32_t* __restrict__ bcnt_raw, const uint32_t* __restrict__ boff,
                                              const int64_t* __restrict__ id, int64_t* __restrict__ prom,
                                              int64_t* __restrict__ dem, const uint32_t b) {
    const uint32_t base = b * UPV_CHUNK;
    const uint32_t np = bcnt_raw[2 * b], nd = bcnt_raw[2 * b + 1];
    for (uint32_t k = threadIdx.x; k < np; k += blockDim.x) prom[boff[2 * b] + k] = id[plist[base + k]];
    for (uint32_t k = threadIdx.x; k < nd; k += blockDim.x) dem[boff[2 * b + 1] + k] = id[dlist[base + k]];
}
__global__ void __launch_bounds__(256) copy_pd_lists(const uint32_t* __restrict__ plist,
                                                     const uint32_t* __restrict__ dlist,
                                                     const uint32_t* __restrict__ bcnt_raw,
                                                     const uint32_t* __restrict__ boff, const int64_t* __restrict__ id,
                                                     int64_t* __restrict__ prom, int64_t* __restrict__ dem) {
    copy_pd_chunk(plist, dlist, bcnt_raw, boff, id, prom, dem, blockIdx.x);
}

// ---- queues of 2^11 .. 2^18 rows: the whole select in one cooperative launch ----------
// The levels' histogram passes, the bucket picks, the gather and the one-block sort of the
// candidates, separated by grid barriers (all CTAs co-resident: cooperative launch), so a
// step costs one launch instead of LEVELS + 2 (most of them no-ops past the decision).
__device__ __forceinline__ void grid_barrier(uint32_t* count, volatile uint32_t* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(const_cast<uint32_t*>(gen), 1u);
        } else {
            while (*gen == g) {}
        }
        __threadfence();
    }
    __syncthreads();
}

// CL: the grid is one thread-block cluster (<= 8 CTAs), so the barriers are the hardware
// cluster barrier (release / acquire at cluster scope) instead of the global-memory one.
template <bool CL>
__device__ __forceinline__ void sel_gsync(uint32_t* bar) {
    if constexpr (CL) {
        __syncthreads();
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        grid_barrier(bar, bar + 1);
    }
}

// The select body (run by every CTA of the grid; h / sk / sv: the CTA's shared scratch).
// plist == nullptr: no state update; prom == nullptr: the update without the ordered
// promoted / demoted id lists (the engine loop does not read them).
struct NoMark {
    __device__ __forceinline__ void operator()(int) const {}
};
template <typename Src, bool CL, typename Mark = NoMark, typename Src0 = Src>
__device__ __forceinline__ void sel_fused_body(const Src& src, uint32_t n, SelState* __restrict__ st,
                                               unsigned __int128* __restrict__ pfx128, uint32_t* __restrict__ hist,
                                               uint32_t k, uint32_t cap, unsigned __int128* __restrict__ ck,
                                               uint32_t* __restrict__ ci, uint32_t* __restrict__ bar,
                                               const int64_t* __restrict__ id, int64_t* __restrict__ run,
                                               uint8_t* __restrict__ sched, int32_t* __restrict__ counts,
                                               const rs_queue_soa& q, int32_t threshold, int32_t pquantum,
                                               uint32_t* __restrict__ plist, uint32_t* __restrict__ dlist,
                                               uint32_t* __restrict__ raw, uint32_t* __restrict__ boff,
                                               int64_t* __restrict__ prom, int64_t* __restrict__ dem, uint32_t* h,
                                               uint4* sk, uint32_t* sv, const Mark& mark = Mark{},
                                               const Src0* src0 = nullptr, uint32_t* slices = nullptr,
                                               uint32_t k_sel = 0, unsigned __int128* thr = nullptr,
                                               uint32_t* run_row = nullptr) {
    // k_sel (>= k, optional): the select keeps every key up to the k_sel-th (the emit still
    // places k); thr: see sel_emit_rank (target k_sel)
    if (k_sel < k) k_sel = k;
    // src0 (optional): level 0's row values, e.g. keys built (and stored for src) on the way.
    // slices (optional, 2 x gridDim.x x SEL_BINS words): each CTA stores its level histogram
    // in its own slice (level parity double-buffered) and every CTA picks the bucket itself
    // from their sum — no global atomics, one barrier per level instead of two (small grids).
    using V = typename Src::V;
    static_assert(std::is_same<typename Src0::V, V>::value && Src0::BITS == Src::BITS, "level-0 source");
    auto gsync = [&]() { sel_gsync<CL>(bar); };
    __shared__ SelLocal L;
    if (slices != nullptr) {
        if (threadIdx.x == 0) L = SelLocal{0, 0u, 0u, 0u, 0u};
        __syncthreads();
    }
    for (uint32_t level = 0; level < (uint32_t)Src::LEVELS; ++level) {
        if (slices != nullptr ? L.done != 0 : *(volatile uint32_t*)&st->done != 0) break;
        mark(20);
        for (int b = threadIdx.x; b < SEL_BINS; b += SEL_THREADS) h[b] = 0;
        __syncthreads();
        const int shift = Src::BITS - SEL_BITS * (int)level;
        const V wsh = level ? (V)((slices != nullptr ? L.pfx : *(volatile unsigned __int128*)pfx128) >> shift) : (V)0;
        if (level == 0 && soa64_aligned(src)) {
            sel_l0_soa(soa64_of(src), n, h);
        } else if (level == 0 && src0 != nullptr) {
            sel_rows_fused(*src0, n, [&](uint32_t, V v, bool ok) { hist_add_warp(h, sel_digit<Src>(v, 0), ok); });
        } else {
            sel_rows_fused(src, n, [&](uint32_t, V v, bool ok) {
                hist_add_warp(h, sel_digit<Src>(v, level), ok && (level == 0 || vshr<Src>(v, shift) == wsh));
            });
        }
        __syncthreads();
        if (slices != nullptr) {
            uint32_t* buf = slices + (size_t)(level & 1u) * gridDim.x * SEL_BINS;
            for (int b = threadIdx.x; b < SEL_BINS; b += SEL_THREADS) buf[blockIdx.x * SEL_BINS + b] = h[b];
            mark(12);
            gsync();
            mark(13);
            sel_pick_local<Src>(L, buf, gridDim.x, k_sel, cap);
            mark(14);
            continue;
        }
        for (int b = threadIdx.x; b < SEL_BINS; b += SEL_THREADS)
            if (h[b]) atomicAdd(&hist[b], h[b]);
        mark(12);
        gsync();
        mark(13);
        if (blockIdx.x == 0) sel_pick_block<Src>(st, pfx128, hist, k_sel, h, 0u, cap);
        mark(14);
        gsync();
        mark(15);
    }
    {  // gather every key at or below the chosen bucket
        const uint32_t fl = slices != nullptr ? L.final_level : *(volatile uint32_t*)&st->final_level;
        const int shift = Src::BITS - SEL_BITS * (int)fl;
        const V lim = (V)((slices != nullptr ? L.pfx : *(volatile unsigned __int128*)pfx128) >> shift);
        sel_rows_fused(src, n, [&](uint32_t i, V v, bool ok) {
            sel_append(ok && vshr<Src>(v, shift) <= lim, to128<Src>(v), i, &st->n_cand, ck, ci, SEL_SORT);
        });
    }
    mark(8);
    gsync();
    mark(9);
    sel_emit_rank(ck, ci, *(volatile uint32_t*)&st->n_cand, id, k, run, sched, counts, sk, thr, k_sel, run_row);
    mark(16);
    if (plist == nullptr) return;  // the state update runs as separate kernels (unaligned columns)
    // the state update (schedulers.py:224-240) and the ordered promoted / demoted lists:
    // starvation_update_v's chunks, scan_pairs and copy_pd_lists, between grid barriers
    gsync();  // the batch's sched flags are set
    mark(10);
    const uint32_t nblk = (n + UPV_CHUNK - 1) / UPV_CHUNK;
    for (uint32_t c = blockIdx.x; c < nblk; c += gridDim.x)
        upd_chunk_v(q, sched, threshold, pquantum, plist, dlist, raw, c);
    gsync();
    mark(11);
    if (prom == nullptr) return;
    if (blockIdx.x == 0) scan_pairs_block(raw, boff, nblk, counts);
    gsync();
    for (uint32_t c = blockIdx.x; c < nblk; c += gridDim.x) copy_pd_chunk(plist, dlist, raw, boff, id, prom, dem, c);
}

template <typename Src, bool CL>
__global__ void __launch_bounds__(SEL_THREADS) sel_fused(Src src, uint32_t n, SelState* __restrict__ st,
                                                         unsigned __int128* __restrict__ pfx128,
                                                         uint32_t* __restrict__ hist, uint32_t k, uint32_t cap,
                                                         unsigned __int128* __restrict__ ck, uint32_t* __restrict__ ci,
                                                         uint32_t* __restrict__ bar, const int64_t* __restrict__ id,
                                                         int64_t* __restrict__ run, uint8_t* __restrict__ sched,
                                                         int32_t* __restrict__ counts, rs_queue_soa q, int32_t threshold,
                                                         int32_t pquantum, uint32_t* __restrict__ plist,
                                                         uint32_t* __restrict__ dlist, uint32_t* __restrict__ raw,
                                                         uint32_t* __restrict__ boff, int64_t* __restrict__ prom,
                                                         int64_t* __restrict__ dem) {
    __shared__ uint32_t h[SEL_BINS + 1];
    __shared__ uint4 sk[1024];
    __shared__ uint32_t sv[1024];
    sel_fused_body<Src, CL>(src, n, st, pfx128, hist, k, cap, ck, ci, bar, id, run, sched, counts, q, threshold,
                            pquantum, plist, dlist, raw, boff, prom, dem, h, sk, sv);
}

__global__ void build_arrival_keys(const double* __restrict__ arr, const int64_t* __restrict__ id, uint32_t n,
                                   Key128* __restrict__ keys) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = Key128{orderable_f64(arr[i]), orderable_i64(id[i])};
}
__global__ void invert_perm(const uint32_t* __restrict__ order, uint32_t n, uint32_t* __restrict__ rank) {
    uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) rank[order[k]] = k;
}

struct RankWs {
    RankKey* ka;
    RankKey* kb;
    uint32_t* va;
    uint32_t* vb;
    uint8_t* sched;
    uint8_t* pd;
    uint32_t* bcnt;
    int* err;
    SelState* sel;
    unsigned __int128* pfx;
    uint32_t* hist;
    unsigned __int128* ck;
    uint32_t* ci;
    unsigned __int128* dv;
    uint32_t* di;
    uint32_t* dcnt;
    uint32_t dcap;
    int* splits;
};
template <typename A>
static void rank_layout(A& a, uint64_t n, RankWs* w) {
    const uint32_t np = ms_padded(n);
    const uint32_t nblk = (uint32_t)((n + UPD_THREADS - 1) / UPD_THREADS) + 1;
    auto ka = a.template take<RankKey>(np);
    auto kb = a.template take<RankKey>(np);
    auto va = a.template take<uint32_t>(np);
    auto vb = a.template take<uint32_t>(np);
    auto sc = a.template take<uint8_t>(n + 1);
    auto pd = a.template take<uint8_t>(n + 1);
    auto bc = a.template take<uint32_t>(2 * nblk);
    auto er = a.template take<int>(4);
    auto sl = a.template take<SelState>(1);
    auto px = a.template take<unsigned __int128>(1);
    auto hi = a.template take<uint32_t>(SEL_BINS);
    auto ck = a.template take<unsigned __int128>(SEL_SORT);
    auto ci = a.template take<uint32_t>(SEL_SORT);
    // rows kept by the select's level-1 pass (at most 4M: beyond, the passes read the columns)
    const uint32_t dcap = (uint32_t)std::min<uint64_t>(n, 1u << 22);
    auto dv = a.template take<unsigned __int128>(n > sel_min_n() ? dcap : 1);
    auto di = a.template take<uint32_t>(n > sel_min_n() ? dcap : 1);
    auto dc = a.template take<uint32_t>(1024);  // per-CTA kept-row counts (grid <= 1024)
    auto sp = a.template take<int>(ms_splits(np));
    if (w) *w = RankWs{ka, kb, va, vb, sc, pd, bc, er, sl, px, hi, ck, ci, dv, di, dc, n > sel_min_n() ? dcap : 0u, sp};
}
// the select's histogram launches, LEVEL = 0 .. Src::LEVELS - 1 in order
template <typename Src, int... L>
static void sel_levels(std::integer_sequence<int, L...>, uint32_t gb, cudaStream_t st, const Src& src, uint32_t n,
                       const RankWs& w, uint32_t k) {
    const uint32_t cap = n <= SEL_SMALL_N ? SEL_CAP_SMALL : SEL_CAP;
    ((sel_hist<Src, L><<<gb, SEL_THREADS, 0, st>>>(src, n, w.sel, w.pfx, w.hist, k, w.dv, w.di, w.dcnt, w.dcap, cap)),
     ...);
}
struct RankSizer {
    ArenaSizer s;
    template <typename T>
    T* take(size_t c) { s.take<T>(c); return nullptr; }
};

// The state update alone (no promoted / demoted lists), grid-stride over 4-row groups
// (flags 4-B, starvation / quantum 16-B aligned: the engine's columns).
// The batch flags are cleared on the way (the engine loop's next key pass needs them zero).
__device__ __forceinline__ void upd_rows_plain(const rs_queue_soa& q, uint8_t* __restrict__ sched, uint32_t n,
                                               int32_t threshold, int32_t pquantum) {
    const uint32_t n4 = n & ~3u, G = gridDim.x * blockDim.x;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) * 4u; i < n4; i += 4u * G) {
        const uint32_t fw = *reinterpret_cast<const uint32_t*>(q.flags + i);
        const uint32_t sw = *reinterpret_cast<const uint32_t*>(sched + i);
        const int4 st = *reinterpret_cast<const int4*>(q.starvation + i);
        const int4 qu = *reinterpret_cast<const int4*>(q.quantum + i);
        int32_t sa[4] = {st.x, st.y, st.z, st.w}, qa[4] = {qu.x, qu.y, qu.z, qu.w};
        uint32_t nf = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint8_t f = (uint8_t)(fw >> (8 * k));
            upd_row(f, sa[k], qa[k], (sw >> (8 * k)) & 0xffu, threshold, pquantum);
            nf |= (uint32_t)f << (8 * k);
        }
        *reinterpret_cast<uint32_t*>(q.flags + i) = nf;
        *reinterpret_cast<int4*>(q.starvation + i) = make_int4(sa[0], sa[1], sa[2], sa[3]);
        *reinterpret_cast<int4*>(q.quantum + i) = make_int4(qa[0], qa[1], qa[2], qa[3]);
        if (sw) *reinterpret_cast<uint32_t*>(sched + i) = 0u;
    }
    const uint32_t r = n4 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) {
        uint8_t f = q.flags[r];
        int32_t st = q.starvation[r], qu = q.quantum[r];
        upd_row(f, st, qu, sched[r], threshold, pquantum);
        q.flags[r] = f;
        q.starvation[r] = st;
        q.quantum[r] = qu;
        sched[r] = 0;
    }
}

// The engine loop's state update on CTAs 1 .. gridDim.x - 1 while CTA 0 executes: the
// priority bit flipped with word atomics (execute sets / clears other bits of the same
// bytes), starvation / quantum stored as before; the batch flags stay (CTA 0 clears them
// at the next step's start).
__device__ __forceinline__ void upd_rows_loop(const rs_queue_soa& q, const uint8_t* __restrict__ sched, uint32_t n,
                                              int32_t threshold, int32_t pquantum) {
    const uint32_t n4 = n & ~3u, parts = gridDim.x - 1, part = blockIdx.x - 1;
    const uint32_t G = parts * blockDim.x;
    for (uint32_t i = (part * blockDim.x + threadIdx.x) * 4u; i < n4; i += 4u * G) {
        const uint32_t fw = *reinterpret_cast<const volatile uint32_t*>(q.flags + i);
        const uint32_t sw = *reinterpret_cast<const uint32_t*>(sched + i);
        const int4 st = *reinterpret_cast<const int4*>(q.starvation + i);
        const int4 qu = *reinterpret_cast<const int4*>(q.quantum + i);
        int32_t sa[4] = {st.x, st.y, st.z, st.w}, qa[4] = {qu.x, qu.y, qu.z, qu.w};
        uint32_t delta = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint8_t f = (uint8_t)(fw >> (8 * k));
            const uint8_t f0 = f;
            upd_row(f, sa[k], qa[k], (sw >> (8 * k)) & 0xffu, threshold, pquantum);
            delta |= (uint32_t)((f ^ f0) & RS_FLAG_PRIORITY) << (8 * k);
        }
        if (delta) atomicXor(reinterpret_cast<unsigned int*>(q.flags + i), delta);
        *reinterpret_cast<int4*>(q.starvation + i) = make_int4(sa[0], sa[1], sa[2], sa[3]);
        *reinterpret_cast<int4*>(q.quantum + i) = make_int4(qa[0], qa[1], qa[2], qa[3]);
    }
    const uint32_t r = n4 + part * blockDim.x + threadIdx.x;
    if (r < n) {
        uint8_t f = *reinterpret_cast<const volatile uint8_t*>(q.flags + r);
        const uint8_t f0 = f;
        int32_t st = q.starvation[r], qu = q.quantum[r];
        upd_row(f, st, qu, sched[r], threshold, pquantum);
        if ((f ^ f0) & RS_FLAG_PRIORITY)
            atomicXor(reinterpret_cast<unsigned int*>(q.flags + (r & ~3u)), (unsigned int)RS_FLAG_PRIORITY << (8 * (r & 3u)));
        q.starvation[r] = st;
        q.quantum[r] = qu;
    }
}

// ---- the whole engine loop as one launch (record-free runs, unlimited KV budget) -------
// engine.py:382-460 step for step, on one thread-block cluster: CTA 0 does the bookkeeping
// the host loop did (idle jump, admission of the arrivals up to `now` in arrival order,
// dropping requests whose full context never fits, the stop tests, the step's clock and
// totals), then every CTA runs the rank step (keys, the fused select, the state update),
// CTA 0 the execute phases — separated by cluster barriers. No launch or host round trip
// per step remains. Finished rows are not compacted out every step (a step retires about
// one row of tens of thousands): they stay in place flagged EX_DONE, rank after every live
// row (all-ones key) and are compacted out, into the other column set, once they are an
// eighth of the rows. Nothing the record-free run reports depends on row positions (the
// sort key carries the arrival rank; only the per-step id lists, not written here, follow
// row order), so the decisions are the per-kernel host loop's — tests/test_gpu_engine.py
// checks both against the reference.
constexpr int ENGINE_LOOP_CTAS = 8;        // one portable cluster
constexpr int ENGINE_LOOP_CTAS_WIDE = 16;  // non-portable, where the device can place it
constexpr uint32_t ENGINE_SPEC_MARGIN = 256;  // speculative threshold: rank k + this
// CTA 0's loop state (shared memory; copied to global memory for the host at the end)
struct EngineLoopState {
    int64_t now, nxt, n_rows, n_alive, step, n_fin, n_drop, tot_prefill, tot_decode, tot_pred, pred;
    int32_t cur, stop, status, acct;
};
// what the other CTAs need of it, published by CTA 0 before a barrier
struct EngineLoopPub {
    int64_t n_rows, n_alive, step, live;
    int32_t stop, compact;
};
struct EngineLoopArgs {
    rs_engine_queue q[2];
    rs_queue_soa soa[2];
    rs_engine_trace tr;
    rs_engine_cost cost;
    const uint8_t* fits;
    int64_t* dropped;
    int64_t n_req;
    int32_t* counts;   // int32[4]
    int64_t *run, *pre, *fin, *prev_run;
    int32_t *prev_n, *block_keep;
    uint32_t* run_row;  // the batch's rows (int32[max_batch])
    SelState* sel;
    unsigned __int128* pfx;
    uint32_t* hist;
    uint32_t* slices;  // 2 x grid x SEL_BINS words
    unsigned __int128* thr;  // speculative select threshold (all ones at the start)
    uint32_t margin;         // ENGINE_SPEC_MARGIN (RS_ENGINE_MARGIN overrides: experiments)
    unsigned __int128* ck;
    uint32_t* ci;
    RankKey* keys;
    uint8_t* sched;
    int32_t max_batch, threshold, pquantum, calibrated, preemptive;
    int64_t pred_per_req, limit_ns, stop_after;
    EngineLoopState* ls;
    EngineLoopPub* pub;
    unsigned long long* prof;  // RS_ENGINE_PROF: per-phase ns totals (CTA 0's view), else null
};
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// CTA 0, between the previous step's last barrier and this step's first: account the
// previous step, stop tests, reset the select state, idle jump + admission (engine.py:
// 404-413: the arrivals up to `now`, in trace order, the ones that can never fit dropped)
__device__ void engine_loop_head(const EngineLoopArgs& a, EngineLoopState& S, int64_t* out, int cur,
                                 int* warp_tot, int* s_first) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        if (S.acct) {
            const int64_t iter = out[1], prefill = out[2];
            S.now = out[0];
            S.n_alive -= out[5];
            S.n_fin += out[5];
            S.tot_prefill += prefill;
            S.tot_pred += S.pred;
            S.tot_decode += iter - prefill - S.pred;
            S.step += 1;
            if ((a.stop_after >= 0 && S.n_fin >= a.stop_after) || (a.limit_ns >= 0 && S.now >= a.limit_ns))
                S.stop = 1;
        }
        if (!S.stop && S.n_alive == 0 && S.nxt < a.n_req) {
            const int64_t t = a.tr.arrival_ns[S.nxt];
            if (t > S.now) S.now = t;  // jump_if_idle
        }
    }
    if (tid < 4) a.counts[tid] = 0;
    if (tid == 32) {
        SelState* st = a.sel;
        st->dom_ok = st->compacted = st->dom_overflow = 0;
        st->level = st->less = st->done = st->final_level = st->n_cand = st->arrived = 0;
        *a.pfx = 0;
    }
    __syncthreads();
    if (S.stop) {
        if (tid == 0) {
            S.cur = cur;
            a.pub->stop = 1;
        }
        return;
    }
    const int64_t now = S.now, n_rows = S.n_rows;
    int64_t nxt = S.nxt, n_drop = S.n_drop;
    int64_t kadm = 0;
    const rs_engine_queue& q = a.q[cur];
    for (;;) {
        if (tid == 0) *s_first = EX_THREADS;
        __syncthreads();
        const int64_t i = nxt + tid;
        if (!(i < a.n_req && a.tr.arrival_ns[i] <= now)) atomicMin(s_first, tid);
        __syncthreads();
        const int first = *(volatile int*)s_first;
        const bool valid = tid < first;  // the arrivals are the prefix up to the first later one
        if (first == 0) break;           // (no scans needed: the common case of no arrival)
        const bool fit = valid && a.fits[i];
        int tf, td;
        const int pf = block_excl_scan(fit ? 1 : 0, warp_tot, tf);
        if (fit) engine_admit_row(q, a.tr, (int)i, n_rows + kadm + pf);
        const int pd = block_excl_scan(valid && !fit ? 1 : 0, warp_tot, td);
        if (valid && !fit) a.dropped[n_drop + pd] = i;
        kadm += tf;
        n_drop += td;
        nxt += first;
        if (first < EX_THREADS) break;
    }
    if (tid == 0) {
        S.nxt = nxt;
        S.n_drop = n_drop;
        S.n_rows = n_rows + kadm;
        S.n_alive += kadm;
        S.pred = kadm * a.pred_per_req;
        EngineLoopPub* pub = a.pub;
        if (S.n_alive == 0 || (a.limit_ns >= 0 && now >= a.limit_ns)) {
            S.stop = 1;
            S.cur = cur;
            pub->stop = 1;
        } else {
            S.acct = 1;
            out[0] = now;  // the execute phase advances the clock from here
            pub->n_rows = S.n_rows;
            pub->n_alive = S.n_alive;
            pub->step = S.step;
            // compaction (this step, before its key pass) once the finished rows are an eighth
            pub->live = S.n_alive;
            pub->compact = (S.n_rows - S.n_alive) * 8 >= S.n_rows ? 1 : 0;
        }
    }
    __syncthreads();  // (s_first / warp_tot reuse)
}

// One row's sort-key value (build_rank_keys, as SrcKeys reads it back) from its columns;
// finished rows (EX_DONE, left in place by the engine loop) get all ones, after every live row.
__device__ __forceinline__ RankKey eng_key(uint8_t f, double score, int32_t gen, uint32_t rank, int calibrated,
                                           int preemptive, int* err) {
    RankKey key;
    key.pad = 0;
    if (f & EX_DONE) {
        key.eff = ~0ull;
        key.cr = ~0u;
        return key;
    }
    const bool scored = f & RS_FLAG_SCORED;
    const bool prio = f & RS_FLAG_PRIORITY;
    const bool running = f & RS_FLAG_RUNNING;
    double eff = 0.0;
    if (scored) {
        eff = calibrated ? score - (double)gen : score;
        if (eff != eff) atomicOr(err, 1);
    }
    const uint32_t pin = preemptive ? 0u : (running ? 0u : 1u);
    const uint32_t cls = (pin << 2) | ((scored ? 1u : 0u) << 1) | (prio ? 0u : 1u);
    key.eff = orderable_f64(eff);
    key.cr = (cls << RANK_BITS) | (rank & RANK_MASK);
    return key;
}
// The keys stored for SrcKeys (the engine loop's full-select fallback).
struct SrcEngBuild {
    using V = unsigned __int128;
    static constexpr int BITS = SrcKeys::BITS, LEVELS = SrcKeys::LEVELS, PAD = 0;
    rs_queue_soa q;
    RankKey* keys;
    int calibrated, preemptive;
    int* err;
    __device__ __forceinline__ unsigned __int128 value(uint32_t i) const {
        const double sc = q.score_dtype == RS_F32 ? (double)static_cast<const float*>(q.score)[i]
                                                  : static_cast<const double*>(q.score)[i];
        const RankKey key = eng_key(q.flags[i], sc, calibrated ? q.generated_tokens[i] : 0, q.arrival_rank[i],
                                    calibrated, preemptive, err);
        keys[i] = key;
        return rank_key_value(key);
    }
};
// The engine loop's speculative pass: every row whose key lies below T appended to (ck, ci)
// (count in *cnt). Four consecutive rows per lane, 16-B column loads (f64 scores, arrival
// ranks, generated tokens) — the engine's columns are 16-B aligned.
__device__ __forceinline__ void eng_spec_pass(const rs_queue_soa& q, uint32_t n, unsigned __int128 T, int calibrated,
                                              int preemptive, int* err, uint32_t* cnt,
                                              unsigned __int128* __restrict__ ck, uint32_t* __restrict__ ci) {
    const uint32_t n4 = n & ~3u, lane = threadIdx.x & 31u, G4 = gridDim.x * SEL_THREADS * 4u;
    const bool f64 = q.score_dtype == RS_F64;
    for (uint32_t base = (blockIdx.x * SEL_THREADS + (threadIdx.x & ~31u)) * 4u; base < n4; base += G4) {
        const uint32_t i = base + lane * 4u;
        const bool ok = i < n4;
        uint32_t fw = 0;
        uint4 rk = make_uint4(0, 0, 0, 0);
        int4 ge = make_int4(0, 0, 0, 0);
        double sc[4] = {0.0, 0.0, 0.0, 0.0};
        if (ok) {
            fw = *reinterpret_cast<const uint32_t*>(q.flags + i);
            rk = *reinterpret_cast<const uint4*>(q.arrival_rank + i);
            if (calibrated) ge = *reinterpret_cast<const int4*>(q.generated_tokens + i);
            if (f64) {
                const double2 a = *reinterpret_cast<const double2*>(static_cast<const double*>(q.score) + i);
                const double2 b = *reinterpret_cast<const double2*>(static_cast<const double*>(q.score) + i + 2);
                sc[0] = a.x;
                sc[1] = a.y;
                sc[2] = b.x;
                sc[3] = b.y;
            } else {
                const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(q.score) + i);
                sc[0] = a.x;
                sc[1] = a.y;
                sc[2] = a.z;
                sc[3] = a.w;
            }
        }
        const uint32_t ra[4] = {rk.x, rk.y, rk.z, rk.w};
        const int32_t ga[4] = {ge.x, ge.y, ge.z, ge.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned __int128 v =
                rank_key_value(eng_key((uint8_t)(fw >> (8 * j)), sc[j], ga[j], ra[j], calibrated, preemptive, err));
            sel_append(ok && v < T, v, i + j, cnt, ck, ci, SEL_SORT);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {  // the last n % 4 rows
        const uint32_t i = n4 + lane;
        const bool ok = i < n;
        unsigned __int128 v = 0;
        if (ok) {
            const double s = f64 ? static_cast<const double*>(q.score)[i] : (double)static_cast<const float*>(q.score)[i];
            v = rank_key_value(eng_key(q.flags[i], s, calibrated ? q.generated_tokens[i] : 0, q.arrival_rank[i],
                                       calibrated, preemptive, err));
        }
        sel_append(ok && v < T, v, i, cnt, ck, ci, SEL_SORT);
    }
}

// Flag bits set / cleared with word atomics: in the engine loop the state update (priority
// bit) runs on the other CTAs while CTA 0 executes (running / done bits), on the same bytes.
__device__ __forceinline__ void flags_or(uint8_t* flags, uint32_t row, uint8_t bits) {
    atomicOr(reinterpret_cast<unsigned int*>(flags + (row & ~3u)), (unsigned int)bits << (8 * (row & 3u)));
}
__device__ __forceinline__ void flags_and_not(uint8_t* flags, uint32_t row, uint8_t bits) {
    atomicAnd(reinterpret_cast<unsigned int*>(flags + (row & ~3u)), ~((unsigned int)bits << (8 * (row & 3u))));
}

// CTA 0 of the engine loop: _Sim.execute (engine.py:247-284) for the step's batch (run ids
// and rows, n_run of them, sched[row] = 1 on them). Preemption (last step's batch rows
// left out: prev_id / prev_row in shared memory, rows re-read through row_of after a
// compaction) and the batch's prefill touch disjoint rows, so they run side by side
// (threads 0..511 / 512..1023), every column the token phase needs loaded up front;
// out: CTA 0's shared {now, iter, prefill, -, -, n_finished}.
__device__ __forceinline__ void engine_execute_loop(const rs_engine_queue& q, const rs_engine_trace& tr,
                                                    const rs_engine_cost& cost, const int64_t* __restrict__ run,
                                                    const uint32_t* __restrict__ run_row, int n_run,
                                                    const uint8_t* __restrict__ sched, int64_t predictor_ns,
                                                    int64_t* out, int64_t* prev_id, uint32_t* prev_row, int& prev_n,
                                                    bool prev_rows_ok, int* s_fin,
                                                    unsigned long long* s_pf) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int pn = prev_n;
    if (tid < pn) {
        const int64_t id = prev_id[tid];
        bool live = true;
        uint32_t row;
        if (prev_rows_ok) {
            row = prev_row[tid];
        } else {
            live = tr.finish_ns[id] < 0;  // finished rows were compacted out
            row = live ? (uint32_t)tr.row_of[id] : 0u;
        }
        if (live) {
            const uint8_t fl = q.flags[row];
            if (!(fl & EX_DONE) && (fl & RS_FLAG_RUNNING) && !sched[row]) {
                flags_and_not(q.flags, row, RS_FLAG_RUNNING);
                tr.n_preempted[id] += 1;
            }
        }
    }
    const int kk = tid - EX_THREADS / 2;
    const bool mine = kk >= 0 && kk < n_run;
    int64_t id = 0, le = 0, mg = 0, ft = 0;
    uint32_t row = 0;
    uint8_t fl = 0;
    int32_t gen = 0, to = 0;
    unsigned long long pf = 0ull;
    if (mine) {
        id = run[kk];
        row = run_row[kk];
        fl = q.flags[row];
        gen = q.generated_tokens[row];
        const int32_t pr = q.prompt_tokens[row];
        le = tr.last_event_ns[id];
        mg = tr.max_gap_ns[id];
        ft = tr.first_token_ns[id];
        to = tr.true_output[id];
        if (!(fl & RS_FLAG_RUNNING)) {  // prefill (engine.py:257-262)
            pf = (unsigned long long)(pr + gen);
            fl |= RS_FLAG_RUNNING;
        }
    }
    pf = warp_sum(pf);
    if (lane == 0 && pf) atomicAdd(s_pf, pf);
    __syncthreads();
    if (tid == 0) {  // the clock
        long long dec;
        if (cost.decode_table_len > 0) {
            const int b = n_run < cost.decode_table_len ? n_run : cost.decode_table_len;
            dec = cost.decode_table[b - 1];
        } else {
            dec = cost.decode_ns;
        }
        const long long pfn = (long long)*s_pf * cost.prefill_ns_per_token;
        out[1] = pfn + dec + predictor_ns;
        out[2] = pfn;
        out[0] += out[1];
    }
    __syncthreads();
    int fin = 0;
    if (mine) {  // one token each (engine.py:270-280)
        const long long now = out[0];
        const int g = gen + 1;
        q.generated_tokens[row] = g;
        if (now - le > mg) tr.max_gap_ns[id] = now - le;
        if (ft < 0) tr.first_token_ns[id] = now;
        tr.last_event_ns[id] = now;
        if (g >= to) {
            tr.finish_ns[id] = now;
            fl |= EX_DONE;
            fin = 1;
        }
        const uint8_t set = fl & (uint8_t)(RS_FLAG_RUNNING | EX_DONE);  // (the priority bit is the update's)
        if (set) flags_or(q.flags, row, set);
        prev_id[kk] = id;
        prev_row[kk] = row;
    }
    const unsigned b = __ballot_sync(0xffffffffu, fin);
    if (lane == 0 && b) atomicAdd(s_fin, __popc(b));
    __syncthreads();
    if (tid == 0) {
        out[5] = *s_fin;
        prev_n = n_run;
        *s_fin = 0;
        *s_pf = 0ull;
    }
}

struct LoopMark {
    unsigned long long* prof;
    unsigned long long* t0;
    __device__ __forceinline__ void operator()(int ph) const {
        if (prof != nullptr && ph >= 20) {
            prof[ph] += 1;  // a count, not a time
        } else if (prof != nullptr) {
            const unsigned long long t = gtimer();
            prof[ph] += t - *t0;
            *t0 = t;
        }
    }
};

template <bool CL>
__global__ void __launch_bounds__(SEL_THREADS) engine_loop_kernel(const __grid_constant__ EngineLoopArgs a) {
    __shared__ uint32_t h[SEL_BINS + 1];
    __shared__ uint4 sk[1024];  // also the execute phase's preempted-row scratch (EX_PRE_CAP ints)
    __shared__ uint32_t sv[1024];
    __shared__ int warp_tot[32];
    __shared__ int s_int;
    __shared__ long long s_base;
    __shared__ EngineLoopState S;  // CTA 0's
    __shared__ int64_t s_out[6];  // CTA 0's execute results (rs_engine_execute's out_dev)
    __shared__ int64_t s_prev_id[EX_THREADS / 2];  // CTA 0: last step's batch
    __shared__ uint32_t s_prev_row[EX_THREADS / 2];
    __shared__ int s_prev_n, s_fin;
    __shared__ unsigned long long s_pf;
    __shared__ bool s_prev_ok;
    static_assert(sizeof(sk) >= EX_PRE_CAP * sizeof(int), "pre_rows scratch");
    uint32_t* bar = &a.sel->bar_count;
    volatile EngineLoopPub* pub = a.pub;
    const uint32_t G = gridDim.x * SEL_THREADS;
    unsigned long long t0 = 0;
    const LoopMark mark{a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0 ? a.prof : nullptr, &t0};
    if (a.prof) t0 = gtimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        S = EngineLoopState{};
        s_out[0] = 0;
        s_prev_n = 0;
        s_fin = 0;
        s_pf = 0ull;
        s_prev_ok = true;
    }
    __syncthreads();
    for (int cur = 0;;) {
        if (blockIdx.x == 0) engine_loop_head(a, S, s_out, cur, warp_tot, &s_int);
        sel_gsync<CL>(bar);
        mark(0);
        if (pub->stop) break;
        uint32_t n = (uint32_t)pub->n_rows;
        const uint32_t n_alive = (uint32_t)pub->n_alive;
        const int32_t step = (int32_t)pub->step;
        // last step's batch flags off (the update on the other CTAs has read them)
        if (blockIdx.x == 0 && threadIdx.x < (uint32_t)s_prev_n) a.sched[s_prev_row[threadIdx.x]] = 0;
        if (pub->compact) {  // finished rows out, into the other column set (stable)
            const uint32_t live = (uint32_t)pub->live;
            const rs_engine_queue qc = [&] { rs_engine_queue t = a.q[cur]; t.n = n; return t; }();
            const uint32_t nb = (n + EX_THREADS - 1) / EX_THREADS;
            for (uint32_t c = blockIdx.x; c < nb; c += gridDim.x) {
                const int t = compact_count_chunk(qc.flags, n, c, warp_tot);
                if (threadIdx.x == 0) a.block_keep[c] = t;
            }
            sel_gsync<CL>(bar);
            for (uint32_t c = blockIdx.x; c < nb; c += gridDim.x) {
                if (threadIdx.x < 32) {
                    long long bsum = 0;
                    for (uint32_t j = threadIdx.x; j < c; j += 32) bsum += __ldcg(a.block_keep + j);
                    bsum = warp_sum(bsum);
                    if (threadIdx.x == 0) s_base = bsum;
                }
                __syncthreads();
                compact_scatter_chunk(qc, a.q[cur ^ 1], a.tr, c, s_base, warp_tot);
            }
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                S.n_rows = live;
                s_prev_ok = false;  // rows moved: the preemption pass finds them through row_of
            }
            cur ^= 1;
            n = live;
            sel_gsync<CL>(bar);
            mark(7);
        }
        rs_queue_soa soa = a.soa[cur];
        soa.n = n;
        rs_engine_queue q = a.q[cur];
        q.n = n;
        // the rank step. One pass builds the keys and keeps every key below the threshold
        // a previous step left (thr: the key then placed at rank k + margin). When that
        // kept between k and 1024 keys they hold the k smallest (>= k keys lie below thr),
        // so they are placed directly; otherwise the full select runs over the built keys,
        // keeping k + margin keys, and resets thr. Exact either way.
        const uint32_t k = min(n_alive, (uint32_t)a.max_batch);
        eng_spec_pass(soa, n, *(volatile unsigned __int128*)a.thr, a.calibrated, a.preemptive, a.counts + 3,
                      &a.sel->arrived, a.ck, a.ci);
        sel_gsync<CL>(bar);
        mark(1);
        if (*(volatile int32_t*)(a.counts + 3)) {  // NaN effective score: every CTA sees it
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                S.status = RS_ERR_NAN;
                S.cur = cur;
            }
            break;
        }
        const uint32_t m = *(volatile uint32_t*)&a.sel->arrived;
        if (m >= k && m <= 1024u) {
            mark(21);
            const bool reset = m > k + 2 * a.margin;  // too many below thr: lower it
            sel_emit_rank(a.ck, a.ci, m, soa.id, k, a.run, a.sched, a.counts, sk, reset ? a.thr : nullptr,
                          k + a.margin, a.run_row);
            mark(16);
        } else {
            const SrcEngBuild kb{soa, a.keys, a.calibrated, a.preemptive, a.counts + 3};
            for (uint32_t i = blockIdx.x * SEL_THREADS + threadIdx.x; i < n; i += G) kb.value(i);
            sel_gsync<CL>(bar);
            // (candidates <= ks + SEL_CAP_SMALL must fit the 1024-key emit)
            const uint32_t ks = min(n_alive, max(k, min(k + a.margin, 1024u - SEL_CAP_SMALL)));
            sel_fused_body<SrcKeys, CL, LoopMark>(SrcKeys{a.keys}, n, a.sel, a.pfx, a.hist, k, (uint32_t)SEL_CAP_SMALL,
                                                  a.ck, a.ci, bar, soa.id, a.run, a.sched, a.counts, soa, a.threshold,
                                                  a.pquantum, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, h,
                                                  sk, sv, mark, (const SrcKeys*)nullptr, a.slices, ks, a.thr,
                                                  a.run_row);
        }
        sel_gsync<CL>(bar);  // the batch (run, run_row, sched) is set
        mark(10);
        // CTA 0 executes while the other CTAs run the state update (schedulers.py:224-240):
        // disjoint state (running / done bits, tokens vs priority bit, starvation, quantum),
        // the shared flag bytes written with word atomics; the next step's first barrier
        // joins them
        if (blockIdx.x == 0) {
            engine_execute_loop(q, a.tr, a.cost, a.run, a.run_row, (int)k, a.sched, S.pred, s_out, s_prev_id,
                                s_prev_row, s_prev_n, s_prev_ok, &s_fin, &s_pf);
            if (threadIdx.x == 0) s_prev_ok = true;
            mark(6);
        } else {
            upd_rows_loop(soa, a.sched, n, a.threshold, a.pquantum);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.ls = S;
}

// RS_ENGINE_LOOP=host keeps the per-kernel host loop (measurement experiments)
static bool engine_loop_device_enabled() {
    static const bool v = [] {
        const char* e = getenv("RS_ENGINE_LOOP");
        return !(e && strcmp(e, "host") == 0);
    }();
    return v;
}

}  // namespace rs

using namespace rs;

extern "C" size_t rs_arrival_rank_workspace_size(int64_t n) {
    const uint32_t np = ms_padded((uint64_t)(n > 0 ? n : 1));
    ArenaSizer s;
    s.take<Key128>(np);
    s.take<Key128>(np);
    s.take<uint32_t>(np);
    s.take<uint32_t>(np);
    s.take<int>(ms_splits(np));
    return s.used + 256;
}

extern "C" int rs_arrival_rank(const double* arr, const int64_t* id, int64_t n, uint32_t* rank, void* ws,
                               size_t ws_bytes, void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(n >= 0 && n <= (int64_t)RANK_MASK, "rs_arrival_rank: n out of range");
    if (n == 0) return RS_OK;
    if (ws_bytes < rs_arrival_rank_workspace_size(n)) {
        set_error("rs_arrival_rank: workspace too small");
        return RS_ERR_WORKSPACE;
    }
    const uint32_t un = (uint32_t)n, np = ms_padded(un);
    Arena ar(ws, ws_bytes);
    Key128* ka = ar.take<Key128>(np);
    Key128* kb = ar.take<Key128>(np);
    uint32_t* va = ar.take<uint32_t>(np);
    uint32_t* vb = ar.take<uint32_t>(np);
    int* splits = ar.take<int>(ms_splits(np));
    const int T = 256;
    build_arrival_keys<<<(un + T - 1) / T, T, 0, st>>>(arr, id, un, kb);
    RS_LAUNCH_CHECK();
    Key128* sk;
    uint32_t* sv;
    RS_TRY((merge_sort<Key128, true, false>(kb, nullptr, un, ka, kb, va, vb, nullptr, st, &sk, &sv, splits)));
    invert_perm<<<(un + T - 1) / T, T, 0, st>>>(sv, un, rank);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" size_t rs_rank_step_workspace_size(int64_t n) {
    RankSizer s;
    rank_layout(s, (uint64_t)(n > 0 ? n : 1), nullptr);
    return s.s.used + 256;
}

extern "C" int rs_rank_step(const rs_queue_soa* q, int32_t max_batch, int64_t kv_budget, int32_t threshold,
                            int32_t pquantum, int32_t calibrated, int32_t preemptive, int64_t* run,
                            int64_t* prom, int64_t* dem, int32_t* counts, void* ws, size_t ws_bytes,
                            void* stream) {
    RS_NVTX();
    cudaStream_t st = as_stream(stream);
    RS_CHECK_ARG(q != nullptr, "rs_rank_step: queue is NULL");
    RS_CHECK_ARG(q->n >= 0 && q->n <= (int64_t)RANK_MASK, "rs_rank_step: n out of range");
    RS_CHECK_ARG(max_batch >= 1, "max_batch must be >= 1");
    RS_CHECK_ARG(threshold >= 0, "starvation_threshold must be >= 0");
    RS_CHECK_ARG(pquantum >= 1, "priority_quantum must be >= 1");
    RS_CHECK_ARG(q->score_dtype == RS_F32 || q->score_dtype == RS_F64, "score dtype must be f32/f64");
    const uint32_t n = (uint32_t)q->n;
    if (n == 0) {
        RS_CUDA(cudaMemsetAsync(counts, 0, 4 * sizeof(int32_t), st));
        return RS_OK;
    }
    if (ws_bytes < rs_rank_step_workspace_size(n)) {
        set_error("rs_rank_step: workspace too small");
        return RS_ERR_WORKSPACE;
    }
    Arena ar(ws, ws_bytes);
    RankWs w;
    rank_layout(ar, n, &w);
    RS_CUDA(cudaMemsetAsync(w.sched, 0, n, st));
    RS_CUDA(cudaMemsetAsync(counts, 0, 4 * sizeof(int32_t), st));
    const int T = 256;
    const uint32_t k = min(n, (uint32_t)max_batch);
    const bool soa64 = q->score_dtype == RS_F32 && !calibrated;
    const bool vec = (reinterpret_cast<uintptr_t>(q->flags) & 3u) == 0 &&
                     ((reinterpret_cast<uintptr_t>(q->starvation) | reinterpret_cast<uintptr_t>(q->quantum)) & 15u) == 0;
    bool fused_update = false;
    if (kv_budget < 0 && n > sel_min_n() && k + SEL_CAP <= (uint32_t)SEL_SORT) {
        // top-k select (see sel_hist): <= LEVELS histogram passes, most no-ops
        const size_t smem = SEL_SORT * (sizeof(unsigned __int128) + sizeof(uint32_t));
        RS_CUDA(ensure_smem((const void*)sel_sort_emit, (int)smem));
        RS_CUDA(cudaMemsetAsync(w.sel, 0, sizeof(SelState), st));
        RS_CUDA(cudaMemsetAsync(w.pfx, 0, sizeof(unsigned __int128), st));
        RS_CUDA(cudaMemsetAsync(w.hist, 0, SEL_BINS * sizeof(uint32_t), st));
        const uint32_t gb = min((n / 4 + SEL_THREADS) / SEL_THREADS, (uint32_t)num_sms() * 2);
        // (measured: at 2^20 rows the multi-launch select below is faster, 68 vs 82 us as a
        // CUDA graph — the grid barriers over 148 CTAs cost more than the launches they save)
        const bool fused = n <= env_u32("RS_SEL_FUSED_N", SEL_FUSED_N) && k + SEL_CAP_SMALL <= 1024;
        fused_update = fused && vec;
        const uint32_t unblk = (n + UPV_CHUNK - 1) / UPV_CHUNK;
        uint32_t* f_plist = fused_update ? reinterpret_cast<uint32_t*>(w.va) : nullptr;
        uint32_t* f_dlist = reinterpret_cast<uint32_t*>(w.vb);
        uint32_t* f_raw = w.bcnt + 2 * unblk;
        if (fused) {
            // one launch: levels, picks, gather, the candidates' sort and the state update;
            // up to SEL_CLUSTER_N rows the grid is one cluster of <= 8 CTAs (hardware
            // barriers), above it a cooperative grid with global-memory barriers
            const bool cl = n <= env_u32("RS_SEL_CLUSTER_N", SEL_CLUSTER_N);
            // cooperative: one 1024-thread CTA per SM at most (register file)
            const uint32_t csz = min(env_u32("RS_SEL_CLUSTER", 8u), 16u);  // (experiments: 16 non-portable)
            const uint32_t grid = cl ? min(gb, csz) : min(gb, (uint32_t)num_sms());
            if (cl && grid > 8) {
                if (soa64)
                    RS_CUDA(cudaFuncSetAttribute(sel_fused<SrcSoa64, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                else
                    RS_CUDA(cudaFuncSetAttribute(sel_fused<SrcKeys, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            }
            cudaLaunchConfig_t lc{};
            cudaLaunchAttribute at[1];
            if (cl) {
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = grid;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
            } else {
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
            }
            lc.gridDim = dim3(grid);
            lc.blockDim = dim3(SEL_THREADS);
            lc.dynamicSmemBytes = 0;
            lc.stream = st;
            lc.attrs = at;
            lc.numAttrs = 1;
            uint32_t* bar = &w.sel->bar_count;
#define RS_SEL_FUSED(SRC, CL)                                                                                   \
    RS_CUDA(cudaLaunchKernelEx(&lc, sel_fused<SRC, CL>, src, n, w.sel, w.pfx, w.hist, k, (uint32_t)SEL_CAP_SMALL, \
                               w.ck, w.ci, bar, q->id, run, w.sched, counts, *q, threshold, pquantum, f_plist,  \
                               f_dlist, f_raw, w.bcnt, prom, dem))
            if (soa64) {
                const SrcSoa64 src{static_cast<const float*>(q->score), q->flags, q->arrival_rank, preemptive, counts + 3};
                if (cl) RS_SEL_FUSED(SrcSoa64, true); else RS_SEL_FUSED(SrcSoa64, false);
            } else {
                build_rank_keys<<<(n + T - 1) / T, T, 0, st>>>(*q, calibrated, preemptive, w.kb, counts + 3);
                RS_LAUNCH_CHECK();
                const SrcKeys src{w.kb};
                if (cl) RS_SEL_FUSED(SrcKeys, true); else RS_SEL_FUSED(SrcKeys, false);
            }
#undef RS_SEL_FUSED
        } else if (soa64) {
            // keys straight from the queue columns: no key pass, 9 B per row per level
            const SrcSoa64 src{static_cast<const float*>(q->score), q->flags, q->arrival_rank, preemptive, counts + 3};
            sel_levels<SrcSoa64>(std::make_integer_sequence<int, SrcSoa64::LEVELS>{}, gb, st, src, n, w, k);
            sel_gather<SrcSoa64><<<gb, SEL_THREADS, 0, st>>>(src, n, w.sel, w.pfx, w.ck, w.ci, w.dv, w.di, w.dcnt, w.dcap);
        } else {
            build_rank_keys<<<(n + T - 1) / T, T, 0, st>>>(*q, calibrated, preemptive, w.kb, counts + 3);
            RS_LAUNCH_CHECK();
            const SrcKeys src{w.kb};
            sel_levels<SrcKeys>(std::make_integer_sequence<int, SrcKeys::LEVELS>{}, gb, st, src, n, w, k);
            sel_gather<SrcKeys><<<gb, SEL_THREADS, 0, st>>>(src, n, w.sel, w.pfx, w.ck, w.ci, w.dv, w.di, w.dcnt, w.dcap);
        }
        RS_LAUNCH_CHECK();
        if (fused) {
            // sorted and emitted inside sel_fused
        } else if (n <= SEL_SMALL_N && k + SEL_CAP_SMALL <= 1024)  // candidates <= k + SEL_CAP_SMALL
            sel_sort_emit_small<<<1, 1024, 0, st>>>(w.ck, w.ci, w.sel, q->id, k, run, w.sched, counts);
        else
            sel_sort_emit<<<1, SEL_THREADS, smem, st>>>(w.ck, w.ci, w.sel, q->id, k, run, w.sched, counts);
    } else {
        build_rank_keys<<<(n + T - 1) / T, T, 0, st>>>(*q, calibrated, preemptive, w.kb, counts + 3);
        RS_LAUNCH_CHECK();
        RankKey* sk;
        uint32_t* order;
        RS_TRY((merge_sort<RankKey, true, false>(w.kb, nullptr, n, w.ka, w.kb, w.va, w.vb, nullptr, st, &sk,
                                                 &order, w.splits)));
        if (kv_budget < 0) {
            fill_unlimited<<<(k + T - 1) / T, T, 0, st>>>(order, q->id, n, max_batch, run, w.sched, counts);
        } else {
            fill_budget<<<1, 32, 0, st>>>(order, q->prompt_tokens, q->generated_tokens, q->id, n, max_batch,
                                          kv_budget, run, w.sched, counts);
        }
    }
    RS_LAUNCH_CHECK();
    if (fused_update) return RS_OK;  // done inside sel_fused
    if (vec) {
        const uint32_t nblk = (n + UPV_CHUNK - 1) / UPV_CHUNK;
        uint32_t* plist = reinterpret_cast<uint32_t*>(w.va);  // the sort buffers are idle here
        uint32_t* dlist = reinterpret_cast<uint32_t*>(w.vb);
        uint32_t* raw = w.bcnt + 2 * nblk;
        starvation_update_v<<<nblk, UPV_T, 0, st>>>(*q, w.sched, threshold, pquantum, plist, dlist, raw);
        RS_LAUNCH_CHECK();
        RS_CUDA(cudaMemcpyAsync(w.bcnt, raw, 2 * nblk * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        scan_pairs<<<1, 1024, 0, st>>>(w.bcnt, nblk, counts);
        RS_LAUNCH_CHECK();
        copy_pd_lists<<<nblk, 256, 0, st>>>(plist, dlist, raw, w.bcnt, q->id, prom, dem);
        RS_LAUNCH_CHECK();
        return RS_OK;
    }
    const uint32_t nblk = (n + UPD_CHUNK - 1) / UPD_CHUNK;
    starvation_update<<<nblk, UPD_THREADS, 0, st>>>(*q, w.sched, threshold, pquantum, w.pd, w.bcnt);
    RS_LAUNCH_CHECK();
    scan_pairs<<<1, 1024, 0, st>>>(w.bcnt, nblk, counts);
    RS_LAUNCH_CHECK();
    scatter_pd<<<nblk, UPD_THREADS, 0, st>>>(w.pd, q->id, n, w.bcnt, prom, dem);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

namespace rs {
// rs_engine_run's one-launch path (engine.cu): taken when the rank step is the fused
// select (unlimited KV budget, max_batch + SEL_CAP_SMALL <= 1024) and the state columns
// are aligned for its vector update; *handled = false leaves the run to the host loop.
int rs_engine_run_device(const rs_engine_queue* q2, const rs_queue_soa* soa2, const rs_engine_trace* tr,
                         const rs_engine_cost* cost, const rs_engine_loop* lp, rs_engine_loop_out* res,
                         cudaStream_t st, bool* handled) {
    *handled = false;
    const int64_t n = lp->n_requests;
    if (!engine_loop_device_enabled() || lp->kv_budget >= 0 || n <= 0 || n > (int64_t)RANK_MASK ||
        lp->max_batch + SEL_CAP_SMALL > 1024 || lp->ws_bytes < rs_rank_step_workspace_size(n))
        return RS_OK;
    for (int c = 0; c < 2; ++c) {  // the vector column accesses (eng_spec_pass, upd_rows_plain)
        const rs_queue_soa& s = soa2[c];
        if ((reinterpret_cast<uintptr_t>(s.flags) & 3u) ||
            ((reinterpret_cast<uintptr_t>(s.starvation) | reinterpret_cast<uintptr_t>(s.quantum) |
              reinterpret_cast<uintptr_t>(s.score) | reinterpret_cast<uintptr_t>(s.arrival_rank) |
              reinterpret_cast<uintptr_t>(s.generated_tokens)) & 15u))
            return RS_OK;
    }
    *handled = true;
    Arena ar(lp->ws, lp->ws_bytes);
    RankWs w;
    rank_layout(ar, (uint64_t)n, &w);
    EngineLoopArgs a{};
    for (int c = 0; c < 2; ++c) {
        a.q[c] = q2[c];
        a.soa[c] = soa2[c];
    }
    a.tr = *tr;
    a.cost = *cost;
    a.n_req = n;
    a.counts = reinterpret_cast<int32_t*>(lp->stat_dev + 6);
    a.run = lp->run_dev;
    a.pre = lp->pre_dev;
    a.fin = lp->fin_dev;
    a.prev_run = lp->prev_run_dev;
    a.prev_n = lp->prev_n_dev;
    a.block_keep = lp->scratch_dev;
    a.sel = w.sel;
    a.pfx = w.pfx;
    a.hist = w.hist;
    a.ck = w.ck;
    a.ci = w.ci;
    a.keys = w.kb;
    a.sched = w.sched;
    a.margin = ENGINE_SPEC_MARGIN;
    if (const char* e = getenv("RS_ENGINE_MARGIN")) a.margin = (uint32_t)std::min(512, std::max(1, atoi(e)));
    a.max_batch = lp->max_batch;
    a.threshold = lp->starvation_threshold;
    a.pquantum = lp->priority_quantum;
    a.calibrated = lp->length_calibrated;
    a.preemptive = lp->preemptive;
    a.pred_per_req = lp->predictor_ns_per_request;
    a.limit_ns = lp->limit_ns;
    a.stop_after = lp->stop_after_finished;
    uint8_t* fits = nullptr;
    int64_t* dropped = nullptr;
    EngineLoopState* ls = nullptr;
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&fits), (size_t)n, st));
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dropped), (size_t)n * sizeof(int64_t), st));
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ls), sizeof(EngineLoopState) + sizeof(EngineLoopPub), st));
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.slices), 2 * 16 * SEL_BINS * sizeof(uint32_t), st));
    a.fits = fits;
    a.dropped = dropped;
    a.ls = ls;
    a.pub = reinterpret_cast<EngineLoopPub*>(ls + 1);
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.thr), sizeof(unsigned __int128), st));
    RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.run_row), 1024 * sizeof(uint32_t), st));
    RS_CUDA(cudaMemsetAsync(a.thr, 0xff, sizeof(unsigned __int128), st));
    RS_CUDA(cudaMemcpyAsync(fits, lp->fits, (size_t)n, cudaMemcpyHostToDevice, st));
    RS_CUDA(cudaMemsetAsync(ls, 0, sizeof(EngineLoopState) + sizeof(EngineLoopPub), st));
    RS_CUDA(cudaMemsetAsync(w.sel, 0, sizeof(SelState), st));
    RS_CUDA(cudaMemsetAsync(w.hist, 0, SEL_BINS * sizeof(uint32_t), st));
    RS_CUDA(cudaMemsetAsync(w.sched, 0, (size_t)n, st));  // kept zero between steps by the update
    cudaLaunchConfig_t lc{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    // 16 CTAs (a non-portable cluster: measured 18.0 vs 20.6 us per cfg5 step with 8) when
    // the device can place one, else the portable 8; RS_ENGINE_CTAS overrides (experiments)
    int ctas = ENGINE_LOOP_CTAS_WIDE;
    if (const char* e = getenv("RS_ENGINE_CTAS")) ctas = std::min(16, std::max(1, atoi(e)));
    RS_CUDA(cudaFuncSetAttribute(engine_loop_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.blockDim = dim3(SEL_THREADS);
    lc.stream = st;
    lc.attrs = at;
    lc.numAttrs = 1;
    for (;;) {
        at[0].val.clusterDim.x = ctas;
        lc.gridDim = dim3(ctas);
        int fit = 0;
        if (ctas <= ENGINE_LOOP_CTAS ||
            (cudaOccupancyMaxActiveClusters(&fit, engine_loop_kernel<true>, &lc) == cudaSuccess && fit >= 1))
            break;
        (void)cudaGetLastError();
        ctas = ENGINE_LOOP_CTAS;
    }
    const bool prof = getenv("RS_ENGINE_PROF") != nullptr;
    if (prof) {
        RS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a.prof), 32 * sizeof(unsigned long long), st));
        RS_CUDA(cudaMemsetAsync(a.prof, 0, 32 * sizeof(unsigned long long), st));
    }
    RS_CUDA(cudaLaunchKernelEx(&lc, engine_loop_kernel<true>, a));
    if (prof) {
        unsigned long long p[32];
        RS_CUDA(cudaMemcpyAsync(p, a.prof, sizeof(p), cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaStreamSynchronize(st));
        RS_CUDA(cudaFreeAsync(a.prof, st));
        static const char* names[] = {"head", "spec_pass", "", "", "", "", "execute", "compact", "gather",
                                      "gather_barrier", "emit_barrier", "update+bar", "level_pass", "level_bar1",
                                      "level_pick", "level_bar2", "emit"};
        for (int i = 0; i < 17; ++i)
            if (names[i][0]) fprintf(stderr, "engine_loop %-16s %10.3f ms\n", names[i], p[i] * 1e-6);
        fprintf(stderr, "engine_loop levels %llu fast steps %llu\n", p[20], p[21]);
    }
    EngineLoopState h{};
    RS_CUDA(cudaMemcpyAsync(&h, ls, sizeof(h), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaStreamSynchronize(st));
    if (h.n_drop > 0)
        RS_CUDA(cudaMemcpyAsync(lp->dropped_host, dropped, (size_t)h.n_drop * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RS_CUDA(cudaFreeAsync(fits, st));
    RS_CUDA(cudaFreeAsync(dropped, st));
    RS_CUDA(cudaFreeAsync(ls, st));
    RS_CUDA(cudaFreeAsync(a.slices, st));
    RS_CUDA(cudaFreeAsync(a.thr, st));
    RS_CUDA(cudaFreeAsync(a.run_row, st));
    RS_CUDA(cudaStreamSynchronize(st));
    res->now_ns = h.now;
    res->steps = h.step;
    res->n_finished = h.n_fin;
    res->next_arrival = h.nxt;
    res->n_dropped = h.n_drop;
    res->total_prefill_ns = h.tot_prefill;
    res->total_decode_ns = h.tot_decode;
    res->total_predictor_ns = h.tot_pred;
    res->final_set = h.cur;
    if (h.status == RS_ERR_NAN) {
        set_error("ranking policy: NaN effective score");
        return RS_ERR_NAN;
    }
    return RS_OK;
}
}  // namespace rs
