// K3: dense bf16 GEMM with fused epilogues on the 5th-generation tensor cores.
//
//   C[M,N] = epi(A[M,K] . W[N,K]^T + bias[N])      A, W bf16 K-major, fp32 accumulate
//
// Persistent, warp-specialised sm_100a kernel (one CTA per SM, 256 threads):
//   warp 0      TMA producer: 128x64 A tile + 256x64 W tile per stage, 4-stage ring
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=256, K=16)
//               into a double-buffered TMEM accumulator (2 x 256 fp32 columns)
//   warp 2      TMEM allocator (512 columns)
//   warps 4-7   epilogue: tcgen05.ld 32 columns at a time, + bias, ReLU / GELU /
//               residual add, bf16 pack, global store; releases the TMEM buffer so
//               the next tile's MMAs overlap this tile's epilogue.
// It replaces the `X @ w + b` of the reference's _Net.forward (predictors.py:190-196)
// with the OPT-125M projections: QKV 768->2304, out 768->768 (+residual),
// FC1 768->3072 (+ReLU), FC2 3072->768 (+residual).
#include <cuda_bf16.h>
#include "common.cuh"
#include "gemm.cuh"
#include "sm100.cuh"
#include "tma.cuh"

namespace rs {

using namespace sm100;

constexpr int G_BM = 128, G_BN = 256, G_BK = 64, G_STAGES = 4;
constexpr int G_A_BYTES = G_BM * G_BK * 2;
constexpr int G_B_BYTES = G_BN * G_BK * 2;
constexpr int G_STAGE_BYTES = G_A_BYTES + G_B_BYTES;
constexpr int G_THREADS = 256;
constexpr int G_SMEM = G_STAGES * G_STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}

template <int EPI>
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                     const __nv_bfloat16* __restrict__ bias, const float* __restrict__ R, void* __restrict__ Cv,
                     int M, int N, int K, int ldc) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + G_STAGES * G_A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + G_STAGES * G_STAGE_BYTES);
    uint64_t* empty = full + G_STAGES;
    uint64_t* tfull = empty + G_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tA);
        tma_prefetch_desc(&tB);
        for (int s = 0; s < G_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_n = N / G_BN;
    const int n_tiles = (M / G_BM) * tiles_n;
    const int kblocks = K / G_BK;

    if (warp == 0) {
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int m0 = (tile / tiles_n) * G_BM, n0 = (tile % tiles_n) * G_BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], G_STAGE_BYTES);
                    tma_load_2d(sA + stage * G_A_BYTES, &tA, &full[stage], kb * G_BK, m0);
                    tma_load_2d(sB + stage * G_B_BYTES, &tB, &full[stage], kb * G_BK, n0);
                    if (++stage == G_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_bf16(G_BM, G_BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * G_BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * G_A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * G_B_BYTES);
#pragma unroll
                    for (int k = 0; k < G_BK / 16; ++k) {
                        mma_bf16_ss(d, desc_kmajor_sw128(a0 + k * 32), desc_kmajor_sw128(b0 + k * 32), idesc,
                                    (kb | k) != 0);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == G_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            const int m0 = (tile / tiles_n) * G_BM, n0 = (tile % tiles_n) * G_BN;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const size_t grow = (size_t)(m0 + row);
            // EPI 2 (residual) keeps the residual stream in fp32: C, R are float.
            __nv_bfloat16* crow = (EPI == 2) ? nullptr : static_cast<__nv_bfloat16*>(Cv) + grow * ldc + n0;
            float* frow = (EPI == 2) ? static_cast<float*>(Cv) + grow * ldc + n0 : nullptr;
            const float* rrow = (EPI == 2) ? R + grow * ldc + n0 : nullptr;
#pragma unroll 1
            for (int c = 0; c < G_BN; c += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * G_BN + c, r);
                tmem_ld_wait();
                float v[32];
                const uint4* bv = reinterpret_cast<const uint4*>(bias + n0 + c);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint4 b4 = __ldg(bv + j);
                    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b4);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        float2 bf = __bfloat1622float2(b2[h]);
                        v[j * 8 + 2 * h] = __uint_as_float(r[j * 8 + 2 * h]) + bf.x;
                        v[j * 8 + 2 * h + 1] = __uint_as_float(r[j * 8 + 2 * h + 1]) + bf.y;
                    }
                }
                if (EPI == 2) {
                    const float4* rv = reinterpret_cast<const float4*>(rrow + c);
                    float4* out = reinterpret_cast<float4*>(frow + c);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4 r4 = rv[j];
                        out[j] = make_float4(v[4 * j] + r4.x, v[4 * j + 1] + r4.y, v[4 * j + 2] + r4.z,
                                             v[4 * j + 3] + r4.w);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (EPI == 1) v[j] = fmaxf(v[j], 0.0f);
                        if (EPI == 3) v[j] = gelu_tanh(v[j]);
                    }
                    uint4* out = reinterpret_cast<uint4*>(crow + c);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint4 o;
                        o.x = pack_bf16(v[j * 8 + 0], v[j * 8 + 1]);
                        o.y = pack_bf16(v[j * 8 + 2], v[j * 8 + 3]);
                        o.z = pack_bf16(v[j * 8 + 4], v[j * 8 + 5]);
                        o.w = pack_bf16(v[j * 8 + 6], v[j * 8 + 7]);
                        out[j] = o;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem_base);
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a 256 x 256 output tile per cluster of 2 CTAs. Each CTA
// TMA-loads its 128-row half of A and its 128-row half of W into the same smem offsets;
// the leader issues tcgen05.mma.cta_group::2 (M=256, N=256, K=16) over both halves, so
// every SM streams only half of the W tile (half the smem operand bandwidth of the
// 1-CTA kernel at the same tile size). Accumulators live in each CTA's TMEM (its 128
// rows x 256 columns, double-buffered); the epilogue stages 32x32 sub-tiles in swizzled
// smem and writes them with TMA stores.
// ---------------------------------------------------------------------------------------
constexpr int G2_BM = 256, G2_BN = 256, G2_BK = 64, G2_STAGES = 6;
constexpr int G2_HALF = 128;
constexpr int G2_A_BYTES = G2_HALF * G2_BK * 2;  // 16 KB per CTA
constexpr int G2_B_BYTES = G2_HALF * G2_BK * 2;  // 16 KB per CTA
constexpr int G2_STAGE_BYTES = G2_A_BYTES + G2_B_BYTES;
constexpr int G2_EPI_BUF = 32 * 32 * 4;          // one 32x32 fp32 (or bf16) staging sub-tile
// The residual epilogue (EPI 2) streams R through the staging buffers with TMA (5 per
// warp, 2 sub-tiles prefetched ahead) and gives up one mainloop stage for them: with
// K = 768 the mainloop is short and the fp32 R read + C write (8 B per output) bound it.
template <int EPI>
struct G2Cfg {
    // EPI 2 (fp32 residual) and 5 (bf16 ReLU mask) stream an input sub-tile per output
    // sub-tile through the staging buffers
    static constexpr bool streams = EPI == 2 || EPI == 5;
    static constexpr int stages = streams ? 5 : G2_STAGES;
    static constexpr int nbuf = streams ? 4 : 2;
    static constexpr int smem = stages * G2_STAGE_BYTES + 4 * nbuf * G2_EPI_BUF + 1024 + 512;
};

// EPI: 0 bf16, 1 ReLU->bf16, 2 +fp32 residual->fp32, 3 GELU->bf16, 4 fp32 (bias optional),
// 5 bf16 * (mask > 0) with the bf16 mask in `aux` (ReLU backward), 6 fp32 split-K partial
// (slice `split` of C), 7 = 0 with the last third of the columns (the V block of a fused
// q|k|v projection) in fp16. A_MN / B_MN: operand stored MN-contiguous ([K, M] / [K, N]).
template <int EPI, bool A_MN = false, bool B_MN = false>
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                         const __grid_constant__ CUtensorMap tC, const __grid_constant__ CUtensorMap tR,
                         const __nv_bfloat16* __restrict__ bias, const void* __restrict__ aux, int M, int N, int K,
                         int ldc, int k_splits, int f16_col0) {
    constexpr int G2_STAGES = G2Cfg<EPI>::stages;
    constexpr int NBUF = G2Cfg<EPI>::nbuf;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + G2_STAGES * G2_A_BYTES;
    uint8_t* sE = smem + G2_STAGES * G2_STAGE_BYTES;  // epilogue staging: 4 warps x NBUF buffers
    uint64_t* full = reinterpret_cast<uint64_t*>(sE + 4 * NBUF * G2_EPI_BUF);
    uint64_t* empty = full + G2_STAGES;
    uint64_t* tfull = empty + G2_STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* rfull = tempty + 2;  // [4 warps][NBUF]: residual sub-tile landed (EPI 2)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 4 * NBUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tA);
        tma_prefetch_desc(&tB);
        tma_prefetch_desc(&tC);
        if (G2Cfg<EPI>::streams) tma_prefetch_desc(&tR);
        for (int s = 0; s < G2_STAGES; ++s) {
            mbar_init(&full[s], 2);  // leader: both CTAs' producers arrive (+ 64 KB of tx)
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);  // leader: 4 epilogue warps x 2 CTAs
        }
        for (int a = 0; a < 4 * NBUF; ++a) mbar_init(&rfull[a], 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_2sm<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_n = N / G2_BN;
    const int n_work = (M / G2_BM) * tiles_n * k_splits;
    const int kblocks_all = K / G2_BK;
    const int kb_per = (kblocks_all + k_splits - 1) / k_splits;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    // work item w -> output tile (w % n_tiles) and K split (w / n_tiles): split-major, so
    // the clusters running at the same time share one K range (the wgrad token slab) and
    // its A / B k-blocks are read from DRAM about once, then served from L2
    const int n_tiles = (M / G2_BM) * tiles_n;
    auto kb_range = [&](int w, int& kb0, int& kb1) {
        const int sp = w / n_tiles;
        kb0 = sp * kb_per;
        kb1 = min(kblocks_all, kb0 + kb_per);
    };

    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol_a = policy_evict_normal(), pol_b = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int w = cid; w < n_work; w += ncl) {
                const int tile = w % n_tiles;
                int kb0, kb1;
                kb_range(w, kb0, kb1);
                const int m0 = (tile / tiles_n) * G2_BM + rank * G2_HALF;
                const int n0 = (tile % tiles_n) * G2_BN + rank * G2_HALF;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader)
                        mbar_arrive_expect_tx(&full[stage], 2 * G2_STAGE_BYTES);
                    else
                        mbar_arrive_cluster(&full[stage], 0);
                    if (A_MN) {  // two 64(M) x 64(K) boxes, 8 KB apart (the MN-major LBO)
                        tma_load_2d_2sm(sA + stage * G2_A_BYTES, &tA, &full[stage], m0, kb * G2_BK, pol_a);
                        tma_load_2d_2sm(sA + stage * G2_A_BYTES + 8192, &tA, &full[stage], m0 + 64, kb * G2_BK,
                                        pol_a);
                    } else {
                        tma_load_2d_2sm(sA + stage * G2_A_BYTES, &tA, &full[stage], kb * G2_BK, m0, pol_a);
                    }
                    if (B_MN) {
                        tma_load_2d_2sm(sB + stage * G2_B_BYTES, &tB, &full[stage], n0, kb * G2_BK, pol_b);
                        tma_load_2d_2sm(sB + stage * G2_B_BYTES + 8192, &tB, &full[stage], n0 + 64, kb * G2_BK,
                                        pol_b);
                    } else {
                        tma_load_2d_2sm(sB + stage * G2_B_BYTES, &tB, &full[stage], kb * G2_BK, n0, pol_b);
                    }
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && elect_one()) {
            constexpr uint32_t idesc = idesc_bf16(G2_BM, G2_BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int w = cid; w < n_work; w += ncl) {
                int kb0, kb1;
                kb_range(w, kb0, kb1);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * G2_BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * G2_A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * G2_B_BYTES);
#pragma unroll
                    for (int k = 0; k < G2_BK / 16; ++k) {
                        // K-major: +32 B per 16-element K step inside the 128-B swizzle row;
                        // MN-major: +16 K rows of 128 B
                        const uint64_t ad = A_MN ? desc_mnmajor_sw128(a0 + k * 2048, 8192) : desc_kmajor_sw128(a0 + k * 32);
                        const uint64_t bd = B_MN ? desc_mnmajor_sw128(b0 + k * 2048, 8192) : desc_kmajor_sw128(b0 + k * 32);
                        mma_bf16_ss_2sm(d, ad, bd, idesc, (kb != kb0) || (k != 0));
                    }
                    mma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_2sm(&tfull[acc], 0x3);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;
        const int row = q * 32 + lane;
        uint8_t* ebuf = sE + q * NBUF * G2_EPI_BUF;
        uint64_t* rf = rfull + q * NBUF;
        int acc = 0;
        uint32_t acc_phase = 0;
        int nst = 0;  // staging sub-tiles issued by this warp (buffer = nst % NBUF)
        // EPI 2: sub-tile n of this warp's sequence is column chunk n % 8 of work item
        // cid + (n / 8) * ncl; its residual is TMA-loaded PD sub-tiles ahead
        constexpr int PD = NBUF - 2;
        auto prefetch_r = [&](int n) {
            const int w = cid + (n >> 3) * ncl;
            if (w >= n_work) return;
            const int tile = w % n_tiles;
            const int rm0 = (tile / tiles_n) * G2_BM + rank * G2_HALF;
            const int rn0 = (tile % tiles_n) * G2_BN;
            const int b = n % NBUF;
            mbar_arrive_expect_tx(&rf[b], EPI == 2 ? G2_EPI_BUF : G2_EPI_BUF / 2);
            tma_load_2d(ebuf + b * G2_EPI_BUF, &tR, &rf[b], rn0 + (n & 7) * 32, rm0 + q * 32);
        };
        if (G2Cfg<EPI>::streams && lane == 0)
            for (int n = 0; n < PD; ++n) prefetch_r(n);
        for (int w = cid; w < n_work; w += ncl) {
            const int tile = w % n_tiles;
            const int m0 = (tile / tiles_n) * G2_BM + rank * G2_HALF;
            const int n0 = (tile % tiles_n) * G2_BN;
            // split-K partials land in slice (w / n_tiles) of a [k_splits * M, N] buffer
            const int mo = (EPI == 6) ? m0 + (w / n_tiles) * M : m0;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < G2_BN; c += 32, ++nst) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * G2_BN + c, r);
                float v[32];
                const uint4* bv = reinterpret_cast<const uint4*>(bias + n0 + c);
                uint8_t* buf = ebuf + (nst % NBUF) * G2_EPI_BUF;
                if (G2Cfg<EPI>::streams) {
                    // reuse of buffer (nst + PD) % NBUF: its last store (sub-tile nst - 2) has
                    // been read; then queue that residual / mask sub-tile
                    if (lane == 0) {
                        tma_store_wait_read<1>();
                        prefetch_r(nst + PD);
                    }
                } else {
                    // the TMA store that last read this buffer (two sub-tiles ago) must be done
                    if (lane == 0 && nst >= 2) tma_store_wait_read<1>();
                }
                tmem_ld_wait();
                if (bias != nullptr) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint4 b4 = __ldg(bv + j);
                        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b4);
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            float2 bf = __bfloat1622float2(b2[h]);
                            v[j * 8 + 2 * h] = __uint_as_float(r[j * 8 + 2 * h]) + bf.x;
                            v[j * 8 + 2 * h + 1] = __uint_as_float(r[j * 8 + 2 * h + 1]) + bf.y;
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                }
                if (G2Cfg<EPI>::streams) mbar_wait(&rf[nst % NBUF], (nst / NBUF) & 1);
                if (EPI == 5) {
                    // the mask sub-tile sits in this buffer in the output's SW64 layout
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint4 m4 =
                            *reinterpret_cast<const uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
                        const __nv_bfloat162* m2 = reinterpret_cast<const __nv_bfloat162*>(&m4);
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            float2 mf = __bfloat1622float2(m2[h]);
                            if (!(mf.x > 0.f)) v[j * 8 + 2 * h] = 0.f;
                            if (!(mf.y > 0.f)) v[j * 8 + 2 * h + 1] = 0.f;
                        }
                    }
                }
                __syncwarp();
                if (EPI == 2 || EPI == 4 || EPI == 6) {
                    // fp32 32x32 sub-tile, 128-B rows, SWIZZLE_128B: chunk j ^ (row % 8)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4* p = reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
                        float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        if (EPI == 2) {
                            const float4 rr = *p;
                            o.x += rr.x;
                            o.y += rr.y;
                            o.z += rr.z;
                            o.w += rr.w;
                        }
                        *p = o;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (EPI == 1) v[j] = fmaxf(v[j], 0.0f);
                        if (EPI == 3) v[j] = gelu_tanh(v[j]);
                    }
                    // bf16 32x32 sub-tile, 64-B rows, SWIZZLE_64B: chunk j ^ ((row / 2) % 4)
                    if (EPI == 7 && n0 >= f16_col0) {  // fp16 columns (the attention V operand)
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
                                make_uint4(pack_f16(v[j * 8 + 0], v[j * 8 + 1]), pack_f16(v[j * 8 + 2], v[j * 8 + 3]),
                                           pack_f16(v[j * 8 + 4], v[j * 8 + 5]), pack_f16(v[j * 8 + 6], v[j * 8 + 7]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
                                make_uint4(pack_bf16(v[j * 8 + 0], v[j * 8 + 1]), pack_bf16(v[j * 8 + 2], v[j * 8 + 3]),
                                           pack_bf16(v[j * 8 + 4], v[j * 8 + 5]), pack_bf16(v[j * 8 + 6], v[j * 8 + 7]));
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tC, buf, n0 + c, mo + q * 32);
                    tma_store_commit();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) tma_store_wait<0>();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 2) tmem_dealloc_2sm<512>(tmem_base);
}

static int g_num_sms = 0;

template <int E, bool AM, bool BM>
static int launch_2sm(cudaLaunchConfig_t& lc, const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tC,
                      const CUtensorMap& tR, const __nv_bfloat16* b, const void* aux, int M, int N, int K,
                      int k_splits) {
    RS_CUDA(ensure_smem((const void*)gemm_bf16_2sm_kernel<E, AM, BM>, G2Cfg<E>::smem));
    lc.dynamicSmemBytes = G2Cfg<E>::smem;
    RS_CUDA(cudaLaunchKernelEx(&lc, gemm_bf16_2sm_kernel<E, AM, BM>, tA, tB, tC, tR, b, aux, M, N, K, N, k_splits,
                               (2 * N) / 3));
    RS_LAUNCH_CHECK();
    return RS_OK;
}

// General CTA-pair GEMM: C = epi(op(A) . op(B)^T [+ bias]) with
//   a_mn = 0: A stored [M, K] (K contiguous)   a_mn = 1: A stored [K, M] (M contiguous)
//   b_mn = 0: W stored [N, K]                   b_mn = 1: W stored [K, N]
// M, N multiples of 256, K a multiple of 64. epi 6 writes k_splits fp32 partial slices.
int gemm_bf16_ex(const void* A, const void* W, const void* bias, const void* aux, void* C, int M, int N, int K,
                 int epi, int a_mn, int b_mn, int k_splits, cudaStream_t st) {
    RS_CHECK_ARG(M > 0 && N > 0 && K > 0 && M % G2_BM == 0 && N % G2_BN == 0 && K % G2_BK == 0,
                 "gemm_ex: need M, N %% 256 == 0 and K %% 64 == 0 (got %d %d %d)", M, N, K);
    RS_CHECK_ARG(epi >= 0 && epi <= 7, "gemm_ex: bad epilogue %d", epi);
    RS_CHECK_ARG(epi != 7 || ((2 * N) / 3) % G2_BN == 0, "gemm_ex: epilogue 7 needs 2N/3 %% 256 == 0");

    RS_CHECK_ARG((epi != 2 && epi != 5) || aux != nullptr, "gemm_ex: epilogue %d needs aux", epi);
    RS_CHECK_ARG(k_splits >= 1 && (epi == 6 || k_splits == 1), "gemm_ex: split-K needs epilogue 6");
    if (g_num_sms == 0) {  // identical on every B200 of a box
        int dev;
        RS_CUDA(cudaGetDevice(&dev));
        RS_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    CUtensorMap tA, tB, tC, tR;
    if (a_mn)
        RS_TRY(make_tmap_bf16(&tA, A, (uint64_t)K, (uint64_t)M, (uint64_t)M * 2, G2_BK, 64));
    else
        RS_TRY(make_tmap_bf16(&tA, A, (uint64_t)M, (uint64_t)K, (uint64_t)K * 2, G2_HALF, G2_BK));
    if (b_mn)
        RS_TRY(make_tmap_bf16(&tB, W, (uint64_t)K, (uint64_t)N, (uint64_t)N * 2, G2_BK, 64));
    else
        RS_TRY(make_tmap_bf16(&tB, W, (uint64_t)N, (uint64_t)K, (uint64_t)K * 2, G2_HALF, G2_BK));
    const bool f32out = epi == 2 || epi == 4 || epi == 6;
    const uint64_t crows = (uint64_t)M * (epi == 6 ? k_splits : 1);
    if (f32out)
        RS_TRY(make_tmap_2d(&tC, C, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, crows, (uint64_t)N, (uint64_t)N * 4, 32, 32,
                            CU_TENSOR_MAP_SWIZZLE_128B));
    else
        RS_TRY(make_tmap_2d(&tC, C, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, crows, (uint64_t)N, (uint64_t)N * 2, 32, 32,
                            CU_TENSOR_MAP_SWIZZLE_64B));
    if (epi == 2)  // the residual R [M, N] fp32, read in the store's sub-tile geometry
        RS_TRY(make_tmap_2d(&tR, aux, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)M, (uint64_t)N, (uint64_t)N * 4, 32,
                            32, CU_TENSOR_MAP_SWIZZLE_128B));
    else if (epi == 5)  // the ReLU mask [M, N] bf16, likewise
        RS_TRY(make_tmap_2d(&tR, aux, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)M, (uint64_t)N, (uint64_t)N * 2, 32,
                            32, CU_TENSOR_MAP_SWIZZLE_64B));
    else
        tR = tC;
    const int n_work = (M / G2_BM) * (N / G2_BN) * k_splits;
    int clusters = g_num_sms / 2;
    if (n_work < clusters) clusters = n_work;
    const __nv_bfloat16* b = static_cast<const __nv_bfloat16*>(bias);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * clusters);
    lc.blockDim = dim3(G_THREADS);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    const int sel = epi * 4 + a_mn * 2 + b_mn;
    switch (sel) {
        case 0 * 4 + 0: return launch_2sm<0, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 1 * 4 + 0: return launch_2sm<1, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 2 * 4 + 0: return launch_2sm<2, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 3 * 4 + 0: return launch_2sm<3, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 7 * 4 + 0: return launch_2sm<7, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        // backward: dgrad (B MN-major) with bf16 / fp32 / ReLU-mask outputs, wgrad (both MN-major)
        case 0 * 4 + 1: return launch_2sm<0, false, true>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 4 * 4 + 1: return launch_2sm<4, false, true>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 5 * 4 + 1: return launch_2sm<5, false, true>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 4 * 4 + 3: return launch_2sm<4, true, true>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 6 * 4 + 3: return launch_2sm<6, true, true>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 4 * 4 + 0: return launch_2sm<4, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        case 6 * 4 + 0: return launch_2sm<6, false, false>(lc, tA, tB, tC, tR, b, aux, M, N, K, k_splits);
        default:
            set_error("gemm_ex: unsupported combination epi=%d a_mn=%d b_mn=%d", epi, a_mn, b_mn);
            return RS_ERR_UNSUPPORTED;
    }
}

int gemm_bf16(const void* A, const void* W, const void* bias, const void* R, void* C, int M, int N, int K, int epi,
              cudaStream_t st) {
    RS_CHECK_ARG(M > 0 && N > 0 && K > 0, "gemm: empty shape");
    RS_CHECK_ARG(M % G_BM == 0 && N % G_BN == 0 && K % G_BK == 0,
                 "gemm: need M %% 128 == 0, N %% 256 == 0, K %% 64 == 0 (got %d %d %d)", M, N, K);
    RS_CHECK_ARG(epi >= 0 && epi <= 3 || epi == 7, "gemm: bad epilogue %d", epi);
    RS_CHECK_ARG(bias != nullptr, "gemm: bias is required");
    RS_CHECK_ARG(epi != 2 || R != nullptr, "gemm: residual epilogue needs R");
    if (g_num_sms == 0) {  // identical on every B200 of a box
        int dev;
        RS_CUDA(cudaGetDevice(&dev));
        RS_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    if (M % G2_BM == 0 && N % G2_BN == 0)  // CTA-pair kernel (the ranker pads M to 256)
        return gemm_bf16_ex(A, W, bias, R, C, M, N, K, epi, 0, 0, 1, st);
    RS_CHECK_ARG(epi != 7, "gemm: epilogue 7 needs M %% 256 == 0");
    CUtensorMap tA, tB;
    RS_TRY(make_tmap_bf16(&tA, A, (uint64_t)M, (uint64_t)K, (uint64_t)K * 2, G_BM, G_BK));
    RS_TRY(make_tmap_bf16(&tB, W, (uint64_t)N, (uint64_t)K, (uint64_t)K * 2, G_BN, G_BK));
    const int n_tiles = (M / G_BM) * (N / G_BN);
    const int grid = n_tiles < g_num_sms ? n_tiles : g_num_sms;
    const __nv_bfloat16* b = static_cast<const __nv_bfloat16*>(bias);
    const float* r = static_cast<const float*>(R);
    void* c = C;
#define RS_GEMM_LAUNCH(E)                                                                                     \
    do {                                                                                                      \
        RS_CUDA(ensure_smem((const void*)gemm_bf16_kernel<E>, G_SMEM));                                      \
        gemm_bf16_kernel<E><<<grid, G_THREADS, G_SMEM, st>>>(tA, tB, b, r, c, M, N, K, N);                    \
    } while (0)
    switch (epi) {
        case 0: RS_GEMM_LAUNCH(0); break;
        case 1: RS_GEMM_LAUNCH(1); break;
        case 2: RS_GEMM_LAUNCH(2); break;
        default: RS_GEMM_LAUNCH(3); break;
    }
#undef RS_GEMM_LAUNCH
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace rs

extern "C" int rs_gemm_bf16_ex(const void* A, const void* W, const void* bias, const void* aux, void* C, int32_t M,
                               int32_t N, int32_t K, int32_t epi, int32_t a_mn, int32_t b_mn, int32_t k_splits,
                               void* stream) {
    RS_NVTX();
    return rs::gemm_bf16_ex(A, W, bias, aux, C, M, N, K, epi, a_mn, b_mn, k_splits, rs::as_stream(stream));
}

extern "C" int rs_gemm_bf16(const void* A, const void* W, const void* bias, const void* R, void* C, int32_t M,
                            int32_t N, int32_t K, int32_t epi, void* stream) {
    RS_NVTX();
    return rs::gemm_bf16(A, W, bias, R, C, M, N, K, epi, rs::as_stream(stream));
}
