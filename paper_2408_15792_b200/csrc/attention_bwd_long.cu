// K7 (attention part) for 128 < S <= 512: causal attention backward over 128-token blocks
// on tcgen05, head dim 64 (the paper's < 2048-token recipe; BASELINE
// configs[2]'s S = 512 secondary run). The S <= 128 case keeps the single-block kernel
// of attention_bwd.cu.
//
// With several query / key blocks, dQ_i sums over key blocks j <= i and dK_j, dV_j over
// query blocks i >= j. Two kernels, each owning one accumulator in TMEM, so nothing is
// accumulated through global memory (no atomics, deterministic):
//   dq kernel, CTA (b, h, i): pass 1 over j <= i: S_ij = Q_i K_j^T -> online row max / sum
//             -> row LSE (base 2) and D_i = rowsum(dO_i * O_i), both written to scratch
//             (given the training forward's LSE, pass 1 is skipped: only D is computed);
//             pass 2 over j <= i: S_ij, dP_ij = dO_i V_j^T -> dS = P (dP - D) / 8 ->
//             dQ_i += dS K_j.
//   dkv kernel, CTA (b, h, j): over i >= j: S_ij, dP_ij (P from the saved LSE) ->
//             dV_j += P^T dO_i, dK_j += dS^T Q_i.
// P and dS are written once in the K-major SW128 layout (read as MN-major for the
// transposed products), as in attention_bwd.cu. Warp 0 issues TMA and MMA (one elected
// thread, each step waits for the previous one: the per-(prompt, head) chains are short
// and many CTAs run at once); warps 1-4 own one query row each per lane.
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "tma.cuh"

namespace rs {
using namespace sm100;

constexpr int AL_T = 128, AL_D = 64;
constexpr int AL_TILE = AL_T * AL_D * 2;   // 16 KB
constexpr int AL_SQ = AL_T * AL_T * 2;     // 32 KB (P or dS)
constexpr int AL_THREADS = 160;
constexpr int AL_MAXB = 4;                 // S <= 512
constexpr float AL_C = 0.125f * 1.4426950408889634f;

struct AlBars {
    uint64_t ld, kv, s_full, s_free, p_full, g_done;
    uint64_t kvb[2];  // double-buffered operand loads of the main loop
    uint32_t tmem;
};

__device__ __forceinline__ float al_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float al_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// element (row, c) of a 128-row x 64-col bf16 tile stored K-major SW128 by TMA
__device__ __forceinline__ float al_tile_elem(const uint8_t* tile, int row, int c) {
    const int off = row * 128 + ((((c >> 3) ^ (row & 7)) << 4)) + (c & 7) * 2;
    return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(tile + off));
}
// 32 columns (cc .. cc + 31) of a 128 x 128 bf16 matrix row r into K-major SW128 (two
// 64-column chunks of 128 rows x 128 B)
__device__ __forceinline__ void al_store_row32(uint8_t* base, int r, int cc, const uint32_t (&pk)[16]) {
    const int off = (cc >> 6) * (AL_T * 128) + r * 128;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        const int ch = ((cc & 63) >> 3) + qq;
        *reinterpret_cast<uint4*>(base + off + ((ch ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
    }
}
__device__ __forceinline__ void al_store_out64(__nv_bfloat16* dst, const uint32_t (&a0)[32], const uint32_t (&a1)[32]) {
    uint4* o4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        o4[qq] = make_uint4(pack_bf16(__uint_as_float(a0[8 * qq]), __uint_as_float(a0[8 * qq + 1])),
                            pack_bf16(__uint_as_float(a0[8 * qq + 2]), __uint_as_float(a0[8 * qq + 3])),
                            pack_bf16(__uint_as_float(a0[8 * qq + 4]), __uint_as_float(a0[8 * qq + 5])),
                            pack_bf16(__uint_as_float(a0[8 * qq + 6]), __uint_as_float(a0[8 * qq + 7])));
        o4[4 + qq] = make_uint4(pack_bf16(__uint_as_float(a1[8 * qq]), __uint_as_float(a1[8 * qq + 1])),
                                pack_bf16(__uint_as_float(a1[8 * qq + 2]), __uint_as_float(a1[8 * qq + 3])),
                                pack_bf16(__uint_as_float(a1[8 * qq + 4]), __uint_as_float(a1[8 * qq + 5])),
                                pack_bf16(__uint_as_float(a1[8 * qq + 6]), __uint_as_float(a1[8 * qq + 7])));
    }
}

__device__ __forceinline__ void al_init(AlBars* bar) {
    mbar_init(&bar->ld, 1);
    mbar_init(&bar->kv, 1);
    mbar_init(&bar->s_full, 1);
    mbar_init(&bar->s_free, 4);
    mbar_init(&bar->p_full, 4);
    mbar_init(&bar->g_done, 1);
    mbar_init(&bar->kvb[0], 1);
    mbar_init(&bar->kvb[1], 1);
    fence_barrier_init();
}

// ---- dQ (+ LSE, D) ----------------------------------------------------------------------
constexpr int ALQ_SMEM = 7 * AL_TILE + AL_SQ + 128;  // Q dO O | K V | dS | K' V' (next block)

__global__ void __launch_bounds__(AL_THREADS, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tatt,
                       const __grid_constant__ CUtensorMap tdo, __nv_bfloat16* __restrict__ dqkv,
                       float* __restrict__ lse_out, float* __restrict__ d_out, const float* __restrict__ lse_in,
                       int B, int S, int H) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint8_t* sQ = smem;
    uint8_t* sdO = sQ + AL_TILE;
    uint8_t* sO = sdO + AL_TILE;
    uint8_t* sK = sO + AL_TILE;
    uint8_t* sV = sK + AL_TILE;
    uint8_t* sdS = sV + AL_TILE;
    uint8_t* sK1 = sdS + AL_SQ;
    uint8_t* sV1 = sK1 + AL_TILE;
    AlBars* bar = reinterpret_cast<AlBars*>(sV1 + AL_TILE);
    const int nq = (S + AL_T - 1) / AL_T;
    const int i = blockIdx.x % nq, bh = blockIdx.x / nq;
    const int b = bh / H, h = bh % H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int dm = H * AL_D;
    const int row0 = b * S;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tqkv);
        al_init(bar);
    }
    if (warp == 0) tmem_alloc<512>(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;
    const uint32_t tS = tmem, tdP = tmem + 128, tdQ = tmem + 256;

    if (warp == 0) {
        if (elect_one()) {
            constexpr uint32_t id_ss = idesc_bf16(AL_T, AL_T);
            constexpr uint32_t id_nn = idesc_bf16(AL_T, AL_D, 0, 1);
            const uint32_t q = smem_u32(sQ), dO = smem_u32(sdO), k = smem_u32(sK), v = smem_u32(sV),
                           ds = smem_u32(sdS);
            mbar_arrive_expect_tx(&bar->ld, 3 * AL_TILE);
            tma_load_2d(sQ, &tqkv, &bar->ld, h * AL_D, row0 + i * AL_T);
            tma_load_2d(sdO, &tdo, &bar->ld, h * AL_D, row0 + i * AL_T);
            tma_load_2d(sO, &tatt, &bar->ld, h * AL_D, row0 + i * AL_T);
            int it = 0;
            // pass 1: S blocks for the row statistics (skipped given the forward's LSE)
            for (int j = 0; lse_in == nullptr && j <= i; ++j, ++it) {
                if (j > 0) mbar_wait(&bar->s_free, (j - 1) & 1);  // S read, K free
                mbar_arrive_expect_tx(&bar->kv, AL_TILE);
                tma_load_2d(sK, &tqkv, &bar->kv, dm + h * AL_D, row0 + j * AL_T);
                mbar_wait(&bar->kv, it & 1);
                if (j == 0) mbar_wait(&bar->ld, 0);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < AL_D / 16; ++s)
                    mma_bf16_ss(tS, desc_kmajor_sw128(q + s * 32), desc_kmajor_sw128(k + s * 32), id_ss, s != 0);
                mma_commit(&bar->s_full);
            }
            if (lse_in == nullptr) mbar_wait(&bar->s_free, i & 1);  // pass 1's last S read: K free
            if (lse_in != nullptr) mbar_wait(&bar->ld, 0);
            // pass 2: dS blocks -> dQ. K, V double-buffered: block j + 1's loads are in
            // flight while block j's softmax and dQ MMA run
            auto load_kv = [&](int jj) {
                const int u = jj & 1;
                mbar_arrive_expect_tx(&bar->kvb[u], 2 * AL_TILE);
                tma_load_2d(u ? sK1 : sK, &tqkv, &bar->kvb[u], dm + h * AL_D, row0 + jj * AL_T);
                tma_load_2d(u ? sV1 : sV, &tqkv, &bar->kvb[u], 2 * dm + h * AL_D, row0 + jj * AL_T);
            };
            load_kv(0);
            for (int j = 0; j <= i; ++j) {
                const int u = j & 1;
                const uint32_t kj = smem_u32(u ? sK1 : sK), vj = smem_u32(u ? sV1 : sV);
                mbar_wait(&bar->kvb[u], (j >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < AL_D / 16; ++s) {
                    mma_bf16_ss(tS, desc_kmajor_sw128(q + s * 32), desc_kmajor_sw128(kj + s * 32), id_ss, s != 0);
                    mma_bf16_ss(tdP, desc_kmajor_sw128(dO + s * 32), desc_kmajor_sw128(vj + s * 32), id_ss, s != 0);
                }
                mma_commit(&bar->s_full);
                if (j < i) {
                    if (j > 0) mbar_wait(&bar->g_done, (j - 1) & 1);  // dQ MMA j - 1 read the other K
                    load_kv(j + 1);
                }
                mbar_wait(&bar->p_full, j & 1);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < AL_T / 16; ++s)
                    mma_bf16_ss(tdQ, desc_kmajor_sw128(ds + (s >> 2) * (AL_T * 128) + (s & 3) * 32),
                                desc_mnmajor_sw128(kj + s * 2048, 8192), id_nn, (j > 0 || s > 0) ? 1u : 0u);
                mma_commit(&bar->g_done);
            }
        }
    } else {
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t la = (uint32_t)(q4 * 32) << 16;
        const int qg = i * AL_T + r;
        const bool row_ok = qg < S;
        mbar_wait(&bar->ld, 0);
        float Dr = 0.f;
#pragma unroll 8
        for (int cc = 0; cc < AL_D; ++cc) Dr += al_tile_elem(sdO, r, cc) * al_tile_elem(sO, r, cc);
        int it = 0;
        float m = -INFINITY, l = 0.f;
        uint32_t v[32];
        for (int j = 0; lse_in == nullptr && j <= i; ++j, ++it) {
            mbar_wait(&bar->s_full, it & 1);
            tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < AL_T; cc += 32) {
                tmem_ld_32x32b_x32(tS + la + cc, v);
                tmem_ld_wait();
                float cm = -INFINITY;
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    if (j * AL_T + cc + e <= qg) cm = fmaxf(cm, __uint_as_float(v[e]));
                const float mn = fmaxf(m, cm);
                if (mn != -INFINITY) {
                    float add = 0.f;
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (j * AL_T + cc + e <= qg) add += al_exp2((__uint_as_float(v[e]) - mn) * AL_C);
                    l = l * al_exp2((m - mn) * AL_C) + add;
                    m = mn;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->s_free);
        }
        // row statistics, [b, h, row] with row stride S (the forward's LSE layout)
        const float lse2 = lse_in != nullptr ? (row_ok ? lse_in[(size_t)bh * S + qg] : 0.f)
                                             : ((row_ok && l > 0.f) ? m * AL_C + al_lg2(l) : 0.f);
        if (row_ok) {
            if (lse_in == nullptr) lse_out[(size_t)bh * S + qg] = lse2;
            d_out[(size_t)bh * S + qg] = Dr;
        }
        for (int j = 0; j <= i; ++j, ++it) {
            mbar_wait(&bar->s_full, it & 1);
            tc_fence_after();
            if (j > 0) mbar_wait(&bar->g_done, (j - 1) & 1);  // previous dQ MMA read sdS
#pragma unroll 1
            for (int cc = 0; cc < AL_T; cc += 32) {
                uint32_t dp[32];
                tmem_ld_32x32b_x32(tS + la + cc, v);
                tmem_ld_32x32b_x32(tdP + la + cc, dp);
                tmem_ld_wait();
                uint32_t dk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    const bool ok0 = row_ok && j * AL_T + cc + e <= qg, ok1 = row_ok && j * AL_T + cc + e + 1 <= qg;
                    const float p0 = ok0 ? al_exp2(__uint_as_float(v[e]) * AL_C - lse2) : 0.f;
                    const float p1 = ok1 ? al_exp2(__uint_as_float(v[e + 1]) * AL_C - lse2) : 0.f;
                    dk[e / 2] = pack_bf16(p0 * (__uint_as_float(dp[e]) - Dr) * 0.125f,
                                          p1 * (__uint_as_float(dp[e + 1]) - Dr) * 0.125f);
                }
                al_store_row32(sdS, r, cc, dk);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->p_full);
        }
        mbar_wait(&bar->g_done, i & 1);
        tc_fence_after();
        uint32_t a0[32], a1[32];
        tmem_ld_32x32b_x32(tdQ + la, a0);
        tmem_ld_32x32b_x32(tdQ + la + 32, a1);
        tmem_ld_wait();
        if (row_ok) al_store_out64(dqkv + (size_t)(row0 + qg) * 3 * dm + h * AL_D, a0, a1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// ---- dK, dV --------------------------------------------------------------------------
constexpr int ALK_SMEM = 6 * AL_TILE + 2 * AL_SQ + 128;  // K V | Q dO | P dS | Q' dO' (next block)

__global__ void __launch_bounds__(AL_THREADS, 1)
    attn_bwd_dkv_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tdo,
                        __nv_bfloat16* __restrict__ dqkv, const float* __restrict__ lse_in,
                        const float* __restrict__ d_in, int B, int S, int H) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint8_t* sK = smem;
    uint8_t* sV = sK + AL_TILE;
    uint8_t* sQ = sV + AL_TILE;
    uint8_t* sdO = sQ + AL_TILE;
    uint8_t* sP = sdO + AL_TILE;
    uint8_t* sdS = sP + AL_SQ;
    uint8_t* sQ1 = sdS + AL_SQ;
    uint8_t* sdO1 = sQ1 + AL_TILE;
    AlBars* bar = reinterpret_cast<AlBars*>(sdO1 + AL_TILE);
    const int nq = (S + AL_T - 1) / AL_T;
    const int j = blockIdx.x % nq, bh = blockIdx.x / nq;
    const int b = bh / H, h = bh % H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int dm = H * AL_D;
    const int row0 = b * S;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tqkv);
        al_init(bar);
    }
    if (warp == 0) tmem_alloc<512>(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;
    const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320;

    if (warp == 0) {
        if (elect_one()) {
            constexpr uint32_t id_ss = idesc_bf16(AL_T, AL_T);
            constexpr uint32_t id_tn = idesc_bf16(AL_T, AL_D, 1, 1);
            const uint32_t q = smem_u32(sQ), dO = smem_u32(sdO), k = smem_u32(sK), v = smem_u32(sV),
                           p = smem_u32(sP), ds = smem_u32(sdS);
            mbar_arrive_expect_tx(&bar->ld, 2 * AL_TILE);
            tma_load_2d(sK, &tqkv, &bar->ld, dm + h * AL_D, row0 + j * AL_T);
            tma_load_2d(sV, &tqkv, &bar->ld, 2 * dm + h * AL_D, row0 + j * AL_T);
            // Q, dO double-buffered: block i + 1's loads are in flight while block i's
            // softmax and dV / dK MMAs run
            auto load_qdo = [&](int tt, int ii) {
                const int u = tt & 1;
                mbar_arrive_expect_tx(&bar->kvb[u], 2 * AL_TILE);
                tma_load_2d(u ? sQ1 : sQ, &tqkv, &bar->kvb[u], h * AL_D, row0 + ii * AL_T);
                tma_load_2d(u ? sdO1 : sdO, &tdo, &bar->kvb[u], h * AL_D, row0 + ii * AL_T);
            };
            load_qdo(0, j);
            for (int i = j, t = 0; i < nq; ++i, ++t) {
                const int u = t & 1;
                const uint32_t qi = smem_u32(u ? sQ1 : sQ), oi = smem_u32(u ? sdO1 : sdO);
                mbar_wait(&bar->kvb[u], (t >> 1) & 1);
                if (t == 0) mbar_wait(&bar->ld, 0);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < AL_D / 16; ++s) {
                    mma_bf16_ss(tS, desc_kmajor_sw128(qi + s * 32), desc_kmajor_sw128(k + s * 32), id_ss, s != 0);
                    mma_bf16_ss(tdP, desc_kmajor_sw128(oi + s * 32), desc_kmajor_sw128(v + s * 32), id_ss, s != 0);
                }
                mma_commit(&bar->s_full);
                if (i + 1 < nq) {
                    if (t > 0) mbar_wait(&bar->g_done, (t - 1) & 1);  // MMAs of t - 1 read the other Q, dO
                    load_qdo(t + 1, i + 1);
                }
                mbar_wait(&bar->p_full, t & 1);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < AL_T / 16; ++s) {
                    const uint32_t acc = (t > 0 || s > 0) ? 1u : 0u;
                    mma_bf16_ss(tdV, desc_mnmajor_sw128(p + s * 2048, AL_T * 128),
                                desc_mnmajor_sw128(oi + s * 2048, 8192), id_tn, acc);
                    mma_bf16_ss(tdK, desc_mnmajor_sw128(ds + s * 2048, AL_T * 128),
                                desc_mnmajor_sw128(qi + s * 2048, 8192), id_tn, acc);
                }
                mma_commit(&bar->g_done);
            }
        }
    } else {
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t la = (uint32_t)(q4 * 32) << 16;
        uint32_t v[32];
        int t = 0;
        for (int i = j; i < nq; ++i, ++t) {
            const int qg = i * AL_T + r;
            const bool row_ok = qg < S;
            const float lse2 = row_ok ? lse_in[(size_t)bh * S + qg] : 0.f;
            const float Dr = row_ok ? d_in[(size_t)bh * S + qg] : 0.f;
            mbar_wait(&bar->s_full, t & 1);
            tc_fence_after();
            if (t > 0) mbar_wait(&bar->g_done, (t - 1) & 1);  // previous dV / dK MMAs read sP, sdS
#pragma unroll 1
            for (int cc = 0; cc < AL_T; cc += 32) {
                uint32_t dp[32];
                tmem_ld_32x32b_x32(tS + la + cc, v);
                tmem_ld_32x32b_x32(tdP + la + cc, dp);
                tmem_ld_wait();
                uint32_t pk[16], dk[16];
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    const bool ok0 = row_ok && j * AL_T + cc + e <= qg, ok1 = row_ok && j * AL_T + cc + e + 1 <= qg;
                    const float p0 = ok0 ? al_exp2(__uint_as_float(v[e]) * AL_C - lse2) : 0.f;
                    const float p1 = ok1 ? al_exp2(__uint_as_float(v[e + 1]) * AL_C - lse2) : 0.f;
                    pk[e / 2] = pack_bf16(p0, p1);
                    dk[e / 2] = pack_bf16(p0 * (__uint_as_float(dp[e]) - Dr) * 0.125f,
                                          p1 * (__uint_as_float(dp[e + 1]) - Dr) * 0.125f);
                }
                al_store_row32(sP, r, cc, pk);
                al_store_row32(sdS, r, cc, dk);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->p_full);
        }
        mbar_wait(&bar->g_done, (t - 1) & 1);
        tc_fence_after();
        // key row r of block j: dK and dV
        const int kg = j * AL_T + r;
        const uint32_t src[2] = {tdK, tdV};
#pragma unroll
        for (int which = 0; which < 2; ++which) {
            uint32_t a0[32], a1[32];
            tmem_ld_32x32b_x32(src[which] + la, a0);
            tmem_ld_32x32b_x32(src[which] + la + 32, a1);
            tmem_ld_wait();
            if (kg < S) al_store_out64(dqkv + (size_t)(row0 + kg) * 3 * dm + (1 + which) * dm + h * AL_D, a0, a1);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

size_t attention_bwd_long_ws(int B, int S, int H) {
    const int nq = (S + AL_T - 1) / AL_T;
    return 2 * (size_t)B * H * nq * AL_T * sizeof(float) + 256;
}

// lse_fwd: the training forward's row LSE (attention_fwd_lse, [b, h, row]) — the dQ
// kernel then skips its statistics pass; nullptr recomputes it into the workspace.
int attention_bwd_long(const void* qkv, const void* att, const void* dout, void* dqkv, int B, int S, int H, void* ws,
                       size_t ws_bytes, cudaStream_t st, const float* lse_fwd) {
    RS_CHECK_ARG(B > 0 && S > AL_T && S <= AL_T * AL_MAXB && H > 0, "attention_bwd_long: need 128 < S <= 512");
    RS_CHECK_ARG(ws_bytes >= attention_bwd_long_ws(B, S, H), "attention_bwd_long: workspace too small");
    RS_CUDA(ensure_smem((const void*)attn_bwd_dq_kernel, ALQ_SMEM));
    RS_CUDA(ensure_smem((const void*)attn_bwd_dkv_kernel, ALK_SMEM));
    const int nq = (S + AL_T - 1) / AL_T;
    float* lse = static_cast<float*>(ws);
    float* dd = lse + (size_t)B * H * nq * AL_T;
    const uint64_t rows = (uint64_t)B * S;
    const uint64_t dmc = (uint64_t)H * AL_D;
    CUtensorMap mq, ma, md;
    RS_TRY(make_tmap_bf16(&mq, qkv, rows, 3 * dmc, 3 * dmc * 2, AL_T, AL_D));
    RS_TRY(make_tmap_bf16(&ma, att, rows, dmc, dmc * 2, AL_T, AL_D));
    RS_TRY(make_tmap_bf16(&md, dout, rows, dmc, dmc * 2, AL_T, AL_D));
    attn_bwd_dq_kernel<<<B * H * nq, AL_THREADS, ALQ_SMEM, st>>>(mq, ma, md, static_cast<__nv_bfloat16*>(dqkv), lse,
                                                                 dd, lse_fwd, B, S, H);
    RS_LAUNCH_CHECK();
    attn_bwd_dkv_kernel<<<B * H * nq, AL_THREADS, ALK_SMEM, st>>>(mq, md, static_cast<__nv_bfloat16*>(dqkv),
                                                                  lse_fwd != nullptr ? lse_fwd : lse, dd,
                                                                  B, S, H);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs

extern "C" size_t rs_attention_bwd_long_workspace_size(int32_t B, int32_t S, int32_t H) {
    return rs::attention_bwd_long_ws(B, S, H);
}

extern "C" int rs_attention_bwd_long(const void* qkv, const void* att, const void* dout, void* dqkv, int32_t B,
                                     int32_t S, int32_t H, void* ws, size_t ws_bytes, void* stream) {
    RS_NVTX();
    return rs::attention_bwd_long(qkv, att, dout, dqkv, B, S, H, ws, ws_bytes, rs::as_stream(stream), nullptr);
}

extern "C" int rs_attention_bwd_long_lse(const void* qkv, const void* att, const void* dout, const float* lse,
                                         void* dqkv, int32_t B, int32_t S, int32_t H, void* ws, size_t ws_bytes,
                                         void* stream) {
    RS_NVTX();
    if (lse == nullptr) {
        rs::set_error("rs_attention_bwd_long_lse: lse is NULL");
        return RS_ERR_INVALID;
    }
    return rs::attention_bwd_long(qkv, att, dout, dqkv, B, S, H, ws, ws_bytes, rs::as_stream(stream), lse);
}
