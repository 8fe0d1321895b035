// K7 (attention part): causal attention backward on tcgen05 for S <= 128 (the training
// configuration, BASELINE.json configs[2]: prompts of 128 tokens), head dim 64.
//
// One CTA per (prompt, head); all of Q, K, V, O, dO fit in smem as 128x64 tiles:
//   S  = Q K^T, dP = dO V^T                       (tcgen05, TMEM)
//   P  = softmax(S / 8 + causal mask)            (one query row per thread; recomputed,
//                                                  so the forward keeps no LSE)
//   D  = rowsum(dO * O), dS = P * (dP - D) / 8   (gradient w.r.t. q.k)
//   dV = P^T dO, dK = dS^T Q, dQ = dS K          (tcgen05; P and dS are written once in
//                                                  the K-major SW128 layout, which read as
//                                                  an MN-major operand is their transpose)
// dQ, dK, dV land in dqkv [B*S, 3*H*64] (bf16) in the same packing as the forward qkv.
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "tma.cuh"

namespace rs {
using namespace sm100;

constexpr int AB_T = 128, AB_D = 64;
constexpr int AB_TILE_BYTES = AB_T * AB_D * 2;  // 16 KB
constexpr int AB_SQ_BYTES = AB_T * AB_T * 2;    // 32 KB (P or dS)
constexpr int AB_THREADS = 192;       // TMA warp, MMA warp, 4 softmax warps (one query row each)
constexpr int AB_THREADS_LSE = 320;   // with the forward's LSE: 8 softmax warps, two per row (64 keys each)
// Two CTAs per SM (each CTA is a serial load -> MMA -> softmax -> MMA -> store chain, so a
// second resident CTA overlaps one's phases with the other's): 112 KB of tiles and 256
// TMEM columns each. V is dead once S / dP are computed and O once D is, so dS reuses V's
// slot (plus one more 16 KB chunk) and P is written over O.
constexpr int AB_SMEM_TILES = 3 * AB_TILE_BYTES + 2 * AB_SQ_BYTES;  // Q K dO | V+dS | O+P
constexpr int AB_SMEM = AB_SMEM_TILES + 128;

struct AbBars {
    uint64_t load_full, s_full, p_full, g_full;
    uint32_t tmem;
};

__device__ __forceinline__ float ab_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// LSE: the forward's row log2-sum-exp is given (lse[(b H + h) S + row]), so P comes from S
// in one pass with no row max / sum, and two warps share each row (key halves): half the
// per-thread softmax work on the CTA's serial chain.
template <bool LSE>
__global__ void __launch_bounds__(LSE ? AB_THREADS_LSE : AB_THREADS, 2)
    attention_bwd_kernel(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tatt,
                         const __grid_constant__ CUtensorMap tdo, __nv_bfloat16* __restrict__ dqkv, int B, int S,
                         int H, const float* __restrict__ lse, float* __restrict__ colsum) {
    // the SW128 tiles need 1024-B alignment; dynamic shared memory of a kernel without
    // static shared memory starts at the window base (checked, not padded: padding would
    // push two CTAs past the SM's 228 KB)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if ((smem_u32(smem) & 1023u) != 0u) __trap();
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + AB_TILE_BYTES;
    uint8_t* sdO = sK + AB_TILE_BYTES;
    uint8_t* sV = sdO + AB_TILE_BYTES;  // dS chunk 0 once S / dP are done
    uint8_t* sdS = sV;                  // 32 KB: V's slot + the next 16 KB
    uint8_t* sP = sdS + AB_SQ_BYTES;    // 32 KB: O in its first 16 KB until D is taken
    uint8_t* sO = sP;
    AbBars* bar = reinterpret_cast<AbBars*>(sP + AB_SQ_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x / H, h = blockIdx.x % H;
    const int dm = H * AB_D;
    const int row0 = b * S;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tqkv);
        mbar_init(&bar->load_full, 1);
        mbar_init(&bar->s_full, 1);
        mbar_init(&bar->p_full, LSE ? 8 : 4);
        mbar_init(&bar->g_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;
    // S, dP first; the gradient accumulators reuse their columns once P / dS are out
    const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem, tdK = tmem + 64, tdQ = tmem + 128;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(&bar->load_full, 5 * AB_TILE_BYTES);
            tma_load_2d(sQ, &tqkv, &bar->load_full, h * AB_D, row0);
            tma_load_2d(sK, &tqkv, &bar->load_full, dm + h * AB_D, row0);
            tma_load_2d(sV, &tqkv, &bar->load_full, 2 * dm + h * AB_D, row0);
            tma_load_2d(sO, &tatt, &bar->load_full, h * AB_D, row0);
            tma_load_2d(sdO, &tdo, &bar->load_full, h * AB_D, row0);
        }
    } else if (warp == 1) {
        if (elect_one()) {
            mbar_wait(&bar->load_full, 0);
            tc_fence_after();
            constexpr uint32_t id_ss = idesc_bf16(AB_T, AB_T);        // S, dP: K-major x K-major
            constexpr uint32_t id_tn = idesc_bf16(AB_T, AB_D, 1, 1);  // dV, dK: A^T (MN-major) x B MN-major
            constexpr uint32_t id_nn = idesc_bf16(AB_T, AB_D, 0, 1);  // dQ: A K-major x B MN-major
            const uint32_t q = smem_u32(sQ), k = smem_u32(sK), v = smem_u32(sV), dO = smem_u32(sdO);
#pragma unroll
            for (int s = 0; s < AB_D / 16; ++s) {
                mma_bf16_ss(tS, desc_kmajor_sw128(q + s * 32), desc_kmajor_sw128(k + s * 32), id_ss, s != 0);
                mma_bf16_ss(tdP, desc_kmajor_sw128(dO + s * 32), desc_kmajor_sw128(v + s * 32), id_ss, s != 0);
            }
            mma_commit(&bar->s_full);
            mbar_wait(&bar->p_full, 0);
            tc_fence_after();
            const uint32_t p = smem_u32(sP), ds = smem_u32(sdS);
#pragma unroll
            for (int s = 0; s < AB_T / 16; ++s) {
                // reduction over queries (K = 16 rows of 128 B per step) for dV, dK
                mma_bf16_ss(tdV, desc_mnmajor_sw128(p + s * 2048, AB_T * 128), desc_mnmajor_sw128(dO + s * 2048, 8192),
                            id_tn, s != 0);
                mma_bf16_ss(tdK, desc_mnmajor_sw128(ds + s * 2048, AB_T * 128), desc_mnmajor_sw128(q + s * 2048, 8192),
                            id_tn, s != 0);
                // reduction over keys for dQ: dS K-major (two 64-key chunks), K MN-major
                mma_bf16_ss(tdQ, desc_kmajor_sw128(ds + (s >> 2) * (AB_T * 128) + (s & 3) * 32),
                            desc_mnmajor_sw128(k + s * 2048, 8192), id_nn, s != 0);
            }
            mma_commit(&bar->g_full);
        }
    } else if (LSE) {
        const int q4 = warp & 3, half = (warp - 2) >> 2;  // TMEM lane quadrant; key half
        const int r = q4 * 32 + lane;
        const uint32_t la = (uint32_t)(q4 * 32) << 16;
        const float c = 0.125f * 1.4426950408889634f;
        const int nvalid = min(S, AB_T);
        const bool row_ok = r < nvalid;
        const int lim = row_ok ? r : -1;
        const float ls = row_ok ? lse[((size_t)b * H + h) * S + r] : 0.f;
        mbar_wait(&bar->load_full, 0);
        float Dr = 0.f;  // D = rowsum(dO * O), both halves (16-B chunks of the SW128 tiles)
#pragma unroll
        for (int ch = 0; ch < AB_D / 8; ++ch) {
            const int off = r * 128 + ((ch ^ (r & 7)) << 4);
            const uint4 a = *reinterpret_cast<const uint4*>(sdO + off);
            const uint4 o = *reinterpret_cast<const uint4*>(sO + off);
            const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 af = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&aw[q]));
                const float2 of = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ow[q]));
                Dr += af.x * of.x;
                Dr += af.y * of.y;
            }
        }
        // P is written over O: both halves of every row have read O first (named barrier
        // over the 8 softmax warps)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        mbar_wait(&bar->s_full, 0);
        tc_fence_after();
        // keys [64 half, 64 half + 64) of the row; a key half entirely past the diagonal
        // of this warp's rows is P = dS = 0 without reading S
#pragma unroll 1
        for (int cc = half * 64; cc < half * 64 + 64; cc += 32) {
            uint32_t v[32], dp[32];
            tmem_ld_32x32b_x32(tS + la + cc, v);
            tmem_ld_32x32b_x32(tdP + la + cc, dp);
            tmem_ld_wait();
            uint32_t pk[16], dk[16];
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
                const float p0 = (cc + e <= lim) ? ab_exp2(__uint_as_float(v[e]) * c - ls) : 0.f;
                const float p1 = (cc + e + 1 <= lim) ? ab_exp2(__uint_as_float(v[e + 1]) * c - ls) : 0.f;
                const float s0 = p0 * (__uint_as_float(dp[e]) - Dr) * 0.125f;
                const float s1 = p1 * (__uint_as_float(dp[e + 1]) - Dr) * 0.125f;
                pk[e / 2] = pack_bf16(p0, p1);
                dk[e / 2] = pack_bf16(s0, s1);
            }
            const int off = (cc >> 6) * (AB_T * 128) + r * 128;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int ch = ((cc & 63) >> 3) + qq;
                *reinterpret_cast<uint4*>(sP + off + ((ch ^ (r & 7)) << 4)) =
                    make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
                *reinterpret_cast<uint4*>(sdS + off + ((ch ^ (r & 7)) << 4)) =
                    make_uint4(dk[4 * qq], dk[4 * qq + 1], dk[4 * qq + 2], dk[4 * qq + 3]);
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar->p_full);
        mbar_wait(&bar->g_full, 0);
        tc_fence_after();
        {  // this half's 32 of the 64 columns of dQ, dK, dV
            __nv_bfloat16* base = dqkv + (size_t)(row0 + r) * 3 * dm + h * AB_D + half * 32;
            const uint32_t src[3] = {tdQ, tdK, tdV};
            // colsum (optional): the prompt's column sums of the bf16 dQ | dK | dV (the
            // q / k / v bias gradients' share of this prompt): each warp's 32 rows summed
            // by a register transpose-reduction, the four row quadrants in fixed order
            // through shared memory (Q's tile: every MMA has completed)
            float* red = reinterpret_cast<float*>(sQ);  // [3][4 quadrants][2 halves][32]
#pragma unroll
            for (int which = 0; which < 3; ++which) {
                uint32_t a0[32];
                tmem_ld_32x32b_x32(src[which] + la + half * 32, a0);
                tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = pack_bf16(__uint_as_float(a0[2 * e]), __uint_as_float(a0[2 * e + 1]));
                if (row_ok) {
                    uint4* o4 = reinterpret_cast<uint4*>(base + which * dm);
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) o4[qq] = make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
                }
                if (colsum != nullptr) {
                    float v[32];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[e]));
                        v[2 * e] = row_ok ? f.x : 0.f;
                        v[2 * e + 1] = row_ok ? f.y : 0.f;
                    }
                    // lane j ends with the sum over the warp's rows of column j
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) {
                        const bool up = (lane & o) != 0;
#pragma unroll
                        for (int i = 0; i < o; ++i) {
                            const float send = up ? v[i] : v[i + o];
                            const float keep = up ? v[i + o] : v[i];
                            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                        }
                    }
                    red[((which * 4 + q4) * 2 + half) * 32 + lane] = v[0];
                }
            }
            if (colsum != nullptr) {
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (q4 == 0) {
#pragma unroll
                    for (int which = 0; which < 3; ++which) {
                        const float* rr = red + (which * 4 * 2 + half) * 32 + lane;
                        colsum[(size_t)b * 3 * dm + which * dm + h * AB_D + half * 32 + lane] =
                            ((rr[0] + rr[64]) + rr[128]) + rr[192];
                    }
                }
            }
        }
    } else {
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;  // query row (S, dP, dQ) / key row (dK, dV) == TMEM lane
        const uint32_t la = (uint32_t)(q4 * 32) << 16;
        const float c = 0.125f * 1.4426950408889634f;
        const int nvalid = min(S, AB_T);
        const bool row_ok = r < nvalid;
        const int lim = row_ok ? r : -1;  // causal: key kk valid iff kk <= lim
        mbar_wait(&bar->load_full, 0);
        // D = rowsum(dO * O): the row's eight 16-B chunks of each tile (SW128: chunk ch of
        // row r at (ch ^ (r & 7)) * 16), same order of products as element by element
        float Dr = 0.f;
#pragma unroll
        for (int ch = 0; ch < AB_D / 8; ++ch) {
            const int off = r * 128 + ((ch ^ (r & 7)) << 4);
            const uint4 a = *reinterpret_cast<const uint4*>(sdO + off);
            const uint4 o = *reinterpret_cast<const uint4*>(sO + off);
            const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 af = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&aw[q]));
                const float2 of = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ow[q]));
                Dr += af.x * of.x;
                Dr += af.y * of.y;
            }
        }
        mbar_wait(&bar->s_full, 0);
        tc_fence_after();
        uint32_t v[32];
        float m = -INFINITY;
#pragma unroll 1
        for (int cc = 0; cc < AB_T; cc += 32) {
            tmem_ld_32x32b_x32(tS + la + cc, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
                if (cc + e <= lim) m = fmaxf(m, __uint_as_float(v[e]));
        }
        float l = 0.f;
#pragma unroll 1
        for (int cc = 0; cc < AB_T; cc += 32) {
            tmem_ld_32x32b_x32(tS + la + cc, v);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
                if (cc + e <= lim) l += ab_exp2((__uint_as_float(v[e]) - m) * c);
        }
        const float inv = row_ok ? 1.f / l : 0.f;
#pragma unroll 1
        for (int cc = 0; cc < AB_T; cc += 32) {
            uint32_t dp[32];
            tmem_ld_32x32b_x32(tS + la + cc, v);
            tmem_ld_32x32b_x32(tdP + la + cc, dp);
            tmem_ld_wait();
            uint32_t pk[16], dk[16];
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
                float p0 = (cc + e <= lim) ? ab_exp2((__uint_as_float(v[e]) - m) * c) * inv : 0.f;
                float p1 = (cc + e + 1 <= lim) ? ab_exp2((__uint_as_float(v[e + 1]) - m) * c) * inv : 0.f;
                const float s0 = p0 * (__uint_as_float(dp[e]) - Dr) * 0.125f;
                const float s1 = p1 * (__uint_as_float(dp[e + 1]) - Dr) * 0.125f;
                pk[e / 2] = pack_bf16(p0, p1);
                dk[e / 2] = pack_bf16(s0, s1);
            }
            const int off = (cc >> 6) * (AB_T * 128) + r * 128;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int ch = ((cc & 63) >> 3) + qq;
                *reinterpret_cast<uint4*>(sP + off + ((ch ^ (r & 7)) << 4)) =
                    make_uint4(pk[4 * qq], pk[4 * qq + 1], pk[4 * qq + 2], pk[4 * qq + 3]);
                *reinterpret_cast<uint4*>(sdS + off + ((ch ^ (r & 7)) << 4)) =
                    make_uint4(dk[4 * qq], dk[4 * qq + 1], dk[4 * qq + 2], dk[4 * qq + 3]);
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar->p_full);
        mbar_wait(&bar->g_full, 0);
        tc_fence_after();
        // tcgen05.ld is .sync.aligned: every lane of the warp issues it, rows past S only
        // skip the store (a partial warp here deadlocks when S % 32 != 0)
        {
            __nv_bfloat16* base = dqkv + (size_t)(row0 + r) * 3 * dm + h * AB_D;
            const uint32_t src[3] = {tdQ, tdK, tdV};
#pragma unroll
            for (int which = 0; which < 3; ++which) {
                uint32_t a0[32], a1[32];
                tmem_ld_32x32b_x32(src[which] + la, a0);
                tmem_ld_32x32b_x32(src[which] + la + 32, a1);
                tmem_ld_wait();
                if (!row_ok) continue;
                uint4* o4 = reinterpret_cast<uint4*>(base + which * dm);
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
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<256>(tmem);
}

int attention_bwd(const void* qkv, const void* att, const void* dout, void* dqkv, int B, int S, int H, cudaStream_t st,
                  const float* lse, float* colsum) {
    RS_CHECK_ARG(B > 0 && S > 0 && H > 0, "attention_bwd: empty shape");
    RS_CHECK_ARG(S <= AB_T, "attention_bwd: S=%d > 128 not supported yet (training uses S <= 128)", S);
    const void* kfn = lse ? (const void*)attention_bwd_kernel<true> : (const void*)attention_bwd_kernel<false>;
    RS_CUDA(ensure_smem(kfn, AB_SMEM));
    RS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    const uint64_t rows = (uint64_t)B * S;
    const uint64_t dmc = (uint64_t)H * AB_D;
    CUtensorMap mq, ma, md;
    RS_TRY(make_tmap_bf16(&mq, qkv, rows, 3 * dmc, 3 * dmc * 2, AB_T, AB_D));
    RS_TRY(make_tmap_bf16(&ma, att, rows, dmc, dmc * 2, AB_T, AB_D));
    RS_TRY(make_tmap_bf16(&md, dout, rows, dmc, dmc * 2, AB_T, AB_D));
    if (lse)
        attention_bwd_kernel<true><<<B * H, AB_THREADS_LSE, AB_SMEM, st>>>(mq, ma, md, static_cast<__nv_bfloat16*>(dqkv),
                                                                           B, S, H, lse, colsum);
    else
        attention_bwd_kernel<false><<<B * H, AB_THREADS, AB_SMEM, st>>>(mq, ma, md, static_cast<__nv_bfloat16*>(dqkv),
                                                                        B, S, H, nullptr, nullptr);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs

extern "C" int rs_attention_bwd(const void* qkv, const void* att, const void* dout, void* dqkv, int32_t B, int32_t S,
                                int32_t H, void* stream) {
    RS_NVTX();
    return rs::attention_bwd(qkv, att, dout, dqkv, B, S, H, rs::as_stream(stream), nullptr, nullptr);
}

extern "C" int rs_attention_bwd_lse(const void* qkv, const void* att, const void* dout, const float* lse, void* dqkv,
                                    int32_t B, int32_t S, int32_t H, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(lse != nullptr, "rs_attention_bwd_lse: lse is NULL");
    return rs::attention_bwd(qkv, att, dout, dqkv, B, S, H, rs::as_stream(stream), lse, nullptr);
}
