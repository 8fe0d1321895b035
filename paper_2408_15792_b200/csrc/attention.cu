// K4: causal multi-head self-attention forward on tcgen05 (head dim 64, S <= 512).
//
// OPT attention (PAPER.md:195-201 backbone; HF OPTAttention semantics): per prompt and
// head, softmax(q k^T / sqrt(64) + causal mask) v over the packed qkv activation
// [B*S, 3*H*64] written by the QKV GEMM. The reference package has no backbone
// (SPEC.md:12), so the oracle is oracle/opt_ranker.py.
//
// Persistent CTA per SM, one (prompt, head, 128-query tile) work item at a time:
//   warp 0      TMA: Q tile (128x64) once per item, K_j / V_j blocks (128x64) in a
//               2-stage ring
//   warp 1      MMA: S_j = Q K_j^T  (M=128, N=128, K=64) into a double-buffered TMEM
//               score tile; O_j = P_j V_j (M=128, N=64, K=128, V as an MN-major
//               operand) into its own TMEM slice O_j (j < 4)
//   warps 4-7   softmax: one query row per thread; block-local max m_j and sum l_j,
//               P_j = exp(s - m_j) as bf16 into swizzled smem (the A operand of the
//               PV MMA); at the end O = sum_j e^(m_j - m) O_j / sum_j e^(m_j - m) l_j.
// Using a per-block max means no TMEM accumulator ever needs rescaling; the combine
// of the <= 4 partial outputs happens once in registers.
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "tma.cuh"

namespace rs {
using namespace sm100;

constexpr int AT_TILE = 128;  // queries per item, keys per block
constexpr int AT_D = 64;
constexpr int AT_MAXKB = 4;  // S <= 512: all K/V blocks of a (prompt, head) stay in smem
constexpr int AT_Q_BYTES = AT_TILE * AT_D * 2;   // 16 KB
constexpr int AT_KV_BYTES = AT_TILE * AT_D * 2;  // 16 KB each of K and V
constexpr int AT_P_BYTES = AT_TILE * AT_TILE * 2;  // 32 KB
constexpr int AT_QST = 2;   // Q buffers: the next item's Q loads while this one computes
constexpr int AT_KVST = AT_MAXKB;  // one resident K/V slot per key block
constexpr int AT_THREADS = 384;  // 4 control warps + 8 softmax warps

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x for x <= 0 on the FMA pipe (offloads the MUFU): round-to-nearest split
// x = j + f, f in [-0.5, 0.5], degree-4 polynomial for 2^f (rel. err ~1e-5, far below
// the bf16 rounding P gets), exponent add for 2^j.
__device__ __forceinline__ float poly_exp2(float x) {
    x = fmaxf(x, -126.0f);
    const float t = x + 12582912.0f;  // 1.5 * 2^23: low mantissa bits = round(x)
    const float j = t - 12582912.0f;
    const float f = x - j;
    float p = fmaf(f, 0.0096181291f, 0.0555041087f);
    p = fmaf(p, f, 0.2402265070f);
    p = fmaf(p, f, 0.6931471806f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ uint32_t f16x2_splat(float x) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(x));
    return r;
}
// (p0, p1) = 2^(s0*c - m*c), 2^(s1*c - m*c): the exponent x <= 0 is formed in fp32 (so the
// dominant terms, x near 0, keep full precision) and exponentiated two at a time by one
// f16x2 MUFU op.
__device__ __forceinline__ void exp2_pair(float s0, float s1, float c, float nmc, float& p0, float& p1) {
    uint32_t xh, ph;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(xh) : "f"(fmaf(s1, c, nmc)), "f"(fmaf(s0, c, nmc)));
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(ph) : "r"(xh));
    asm("{\n\t.reg .f16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\tcvt.f32.f16 %0, lo;\n\tcvt.f32.f16 %1, hi;\n\t}"
        : "=f"(p0), "=f"(p1)
        : "r"(ph));
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int AT_PST = 1;  // one P buffer (smem budget: Q 32 KB + resident K/V 128 KB + P 32 KB)
constexpr int AT_SMEM = AT_QST * AT_Q_BYTES + AT_KVST * 2 * AT_KV_BYTES + AT_PST * AT_P_BYTES + 1024 + 8192;

struct AtBars {
    uint64_t q_full[AT_QST], q_empty[AT_QST], o_full, o_empty;
    uint64_t kv_full[AT_KVST], kv_empty[AT_KVST];
    uint64_t s_full[2], s_empty[2];
    uint64_t p_full[2], p_empty[2];
    uint32_t tmem;
    float redm[2 * 2 * 128];         // row-max exchange between the two column halves
    float redl[2 * AT_MAXKB * 128];  // row-sum exchange at the end of an item
};

__global__ void __launch_bounds__(AT_THREADS, 1)
    attention_fwd_kernel(const __grid_constant__ CUtensorMap tqkv, __nv_bfloat16* __restrict__ out, int B, int S,
                         int H, unsigned long long* __restrict__ trace) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                          // AT_QST buffers
    uint8_t* sK = sQ + AT_QST * AT_Q_BYTES;      // AT_KVST stages
    uint8_t* sV = sK + AT_KVST * AT_KV_BYTES;    // AT_KVST stages
    uint8_t* sP = sV + AT_KVST * AT_KV_BYTES;    // 2 buffers
    AtBars* bar = reinterpret_cast<AtBars*>(sP + AT_PST * AT_P_BYTES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_qt = (S + AT_TILE - 1) / AT_TILE;
    const int dm = H * AT_D;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tqkv);
        for (int i = 0; i < AT_QST; ++i) {
            mbar_init(&bar->q_full[i], 1);
            mbar_init(&bar->q_empty[i], 1);
        }
        for (int i = 0; i < AT_KVST; ++i) {
            mbar_init(&bar->kv_full[i], 1);
            mbar_init(&bar->kv_empty[i], 1);
        }
        mbar_init(&bar->o_full, 1);
        mbar_init(&bar->o_empty, 8);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar->s_full[i], 1);
            mbar_init(&bar->s_empty[i], 8);
            mbar_init(&bar->p_full[i], 8);
            mbar_init(&bar->p_empty[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(&bar->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;

    // work unit = one (prompt, head): its K/V blocks are loaded once and stay resident
    // while its q-tiles run, heaviest (most key blocks) first
    const int n_units = B * H;
    const int my_units = blockIdx.x < n_units ? (n_units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int my_items = my_units * n_qt;

    if (warp == 0) {
        if (elect_one()) {
            int t = 0, u = 0;
            for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x, ++u) {
                const int b = unit / H, h = unit % H;
                const int row0 = b * S;
                for (int qt = n_qt - 1; qt >= 0; --qt, ++t) {
                    const int qb = t % AT_QST;
                    mbar_wait(&bar->q_empty[qb], ((t / AT_QST) & 1) ^ 1);
                    mbar_arrive_expect_tx(&bar->q_full[qb], AT_Q_BYTES);
                    tma_load_2d(sQ + qb * AT_Q_BYTES, &tqkv, &bar->q_full[qb], h * AT_D, row0 + qt * AT_TILE);
                    if (qt == n_qt - 1) {
                        // every K/V block of the unit, diagonal first; slot j is reused by the
                        // next unit once q-tile j (its last user) has consumed it
                        for (int j = n_qt - 1; j >= 0; --j) {
                            mbar_wait(&bar->kv_empty[j], (u & 1) ^ 1);
                            mbar_arrive_expect_tx(&bar->kv_full[j], 2 * AT_KV_BYTES);
                            tma_load_2d(sK + j * AT_KV_BYTES, &tqkv, &bar->kv_full[j], dm + h * AT_D,
                                        row0 + j * AT_TILE);
                            tma_load_2d(sV + j * AT_KV_BYTES, &tqkv, &bar->kv_full[j], 2 * dm + h * AT_D,
                                        row0 + j * AT_TILE);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            constexpr uint32_t id_s = idesc_bf16(AT_TILE, AT_TILE);
            constexpr uint32_t id_o = idesc_bf16(AT_TILE, AT_D, 0, 1);
            int t = 0, u = 0, sc = 0, pc = 0;
            for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x, ++u) {
                for (int qt = n_qt - 1; qt >= 0; --qt, ++t) {
                    const int nkb = qt + 1;
                    const int qb = t % AT_QST;
                    mbar_wait(&bar->q_full[qb], (t / AT_QST) & 1);
                    // block i of this q-tile is key block j = qt - i (diagonal first);
                    // O_i = P_i V_j accumulates into TMEM slice i
                    auto issue_pv = [&](int i) {
                        const int j = qt - i;
                        const int pb = pc % AT_PST;
                        mbar_wait(&bar->p_full[pb], (pc / AT_PST) & 1);
                        if (i == 0) mbar_wait(&bar->o_empty, (t & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t pa = smem_u32(sP + pb * AT_P_BYTES);
                        const uint32_t vb = smem_u32(sV + j * AT_KV_BYTES);
                        const uint32_t d = tmem + 256 + i * AT_D;
#pragma unroll
                        for (int kk = 0; kk < AT_TILE / 16; ++kk)
                            mma_bf16_ss(d, desc_kmajor_sw128(pa + (kk >> 2) * (AT_TILE * 128) + (kk & 3) * 32),
                                        desc_mnmajor_sw128(vb + kk * 2048, 8192), id_o, kk != 0);
                        mma_commit(&bar->p_empty[pb]);
                        if (i == 0) mma_commit(&bar->kv_empty[j]);  // q-tile j is key block j's last user
                        ++pc;
                    };
                    for (int i = 0; i < nkb; ++i, ++sc) {
                        const int j = qt - i;
                        const int sb = sc & 1;
                        mbar_wait(&bar->s_empty[sb], ((sc >> 1) & 1) ^ 1);
                        if (qt == n_qt - 1) mbar_wait(&bar->kv_full[j], u & 1);
                        tc_fence_after();
                        const uint32_t qa = smem_u32(sQ + qb * AT_Q_BYTES);
                        const uint32_t ka = smem_u32(sK + j * AT_KV_BYTES);
#pragma unroll
                        for (int k = 0; k < AT_D / 16; ++k)
                            mma_bf16_ss(tmem + sb * AT_TILE, desc_kmajor_sw128(qa + k * 32),
                                        desc_kmajor_sw128(ka + k * 32), id_s, k != 0);
                        mma_commit(&bar->s_full[sb]);
                        if (i == nkb - 1) mma_commit(&bar->q_empty[qb]);
                        if (i >= 1) issue_pv(i - 1);
                    }
                    issue_pv(nkb - 1);
                    mma_commit(&bar->o_full);
                }
            }
        }
    } else if (warp >= 4) {
        // 8 softmax warps: warp w and w+4 share TMEM lane quarter q4 (rows q4*32..+31)
        // and split the 128 key columns of each block (half 0: keys 0-63, half 1: 64-127).
        const int q4 = warp & 3;
        const int half = (warp - 4) >> 2;
        const int r = q4 * 32 + lane;  // query row within the tile == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const float sl2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
        float* redm = bar->redm;  // [2 parity][2 half][128]
        float* redl = bar->redl;  // [2 half][AT_MAXKB][128]
        int t = 0, sc = 0, pc = 0;
        for (int item = 0; item < my_items; ++item, ++t) {
            const int unit = blockIdx.x + (item / n_qt) * gridDim.x;
            const int b = unit / H, h = unit % H;
            const int qt = n_qt - 1 - item % n_qt;
            const int nkb = qt + 1;
            float mj[AT_MAXKB], lj[AT_MAXKB];
#pragma unroll
            for (int j = 0; j < AT_MAXKB; ++j) {
                mj[j] = 0.f;
                lj[j] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < AT_MAXKB; ++j) {
                if (j >= nkb) break;
                const int sb = sc & 1;
                // diagnostics: per-block phase timestamps of CTA 0 / warp 4 (trace != nullptr)
                const bool tr = trace != nullptr && blockIdx.x == 0 && warp == 4 && lane == 0 && sc < 64;
                if (tr) trace[sc * 8 + 0] = clock64();
                mbar_wait(&bar->s_full[sb], (sc >> 1) & 1);
                if (tr) trace[sc * 8 + 1] = clock64();
                tc_fence_after();
                const uint32_t sa = tmem + lane_addr + sb * AT_TILE + half * 64;
                // causal: key c (within this half) valid iff half*64 + c <= lim
                const int lim = ((j == 0) ? r : AT_TILE - 1) - half * 64;  // block 0 = diagonal
                uint32_t v[64];
                tmem_ld_32x32b_x32(sa, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                tmem_ld_32x32b_x32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                tmem_ld_wait();
                float m = -INFINITY;
                if (lim >= 63) {
#pragma unroll
                    for (int e = 0; e < 64; e += 2) m = fmax3(m, __uint_as_float(v[e]), __uint_as_float(v[e + 1]));
                } else {
#pragma unroll
                    for (int e = 0; e < 64; ++e)
                        if (e <= lim) m = fmaxf(m, __uint_as_float(v[e]));
                }
                // row max across the two halves (smem, double-buffered by block parity)
                redm[(sb * 2 + half) * AT_TILE + r] = m;
                named_bar_sync(1 + q4, 64);
                if (tr) trace[sc * 8 + 2] = clock64();
                m = fmaxf(redm[(sb * 2 + 0) * AT_TILE + r], redm[(sb * 2 + 1) * AT_TILE + r]);
                const int pb = pc % AT_PST;
                mbar_wait(&bar->p_empty[pb], ((pc / AT_PST) & 1) ^ 1);
                if (tr) trace[sc * 8 + 3] = clock64();
                // p = 2^(s*c - m*c), two columns per f16x2 MUFU op (P is rounded to bf16 for
                // the MMA anyway; f16 keeps 10 mantissa bits through the exponential)
                const float c2 = sl2;
                const float nm2 = -m * sl2;
                float l = 0.f;
                uint32_t pk[32];
                if (lim >= 63) {
#pragma unroll
                    for (int e = 0; e < 64; e += 2) {
                        float p0, p1;
                        exp2_pair(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), c2, nm2, p0, p1);
                        pk[e / 2] = pack_bf16(p0, p1);
                        l += p0 + p1;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 64; e += 2) {
                        float p0, p1;
                        exp2_pair(__uint_as_float(v[e]), __uint_as_float(v[e + 1]), c2, nm2, p0, p1);
                        if (e > lim) p0 = 0.f;
                        if (e + 1 > lim) p1 = 0.f;
                        pk[e / 2] = pack_bf16(p0, p1);
                        l += p0 + p1;
                    }
                }
                tc_fence_before();
                // this row's 8 x 16-byte chunks of key block `half`, K-major SW128
                // (chunk index ^= row % 8)
                uint8_t* blk = sP + pb * AT_P_BYTES + half * (AT_TILE * 128) + r * 128;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    *reinterpret_cast<uint4*>(blk + ((q ^ (r & 7)) << 4)) =
                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                fence_proxy_async_smem();
                __syncwarp();
                if (tr) trace[sc * 8 + 4] = clock64();
                if (lane == 0) {
                    mbar_arrive(&bar->s_empty[sb]);
                    mbar_arrive(&bar->p_full[pb]);
                }
                mj[j] = m;
                lj[j] = l;
                ++sc;
                ++pc;
            }
            // combine the partial outputs: exchange the per-half row sums, then each
            // warp of the pair produces 32 of the 64 output columns
#pragma unroll
            for (int j = 0; j < AT_MAXKB; ++j)
                if (j < nkb) redl[(half * AT_MAXKB + j) * AT_TILE + r] = lj[j];
            named_bar_sync(1 + q4, 64);
            float mx = mj[0];
#pragma unroll
            for (int j = 1; j < AT_MAXKB; ++j)
                if (j < nkb) mx = fmaxf(mx, mj[j]);
            float w[AT_MAXKB];
            float den = 0.f;
#pragma unroll
            for (int j = 0; j < AT_MAXKB; ++j) {
                w[j] = 0.f;
                if (j < nkb) {
                    w[j] = exp2f((mj[j] - mx) * sl2);
                    den += w[j] * (redl[(0 * AT_MAXKB + j) * AT_TILE + r] + redl[(1 * AT_MAXKB + j) * AT_TILE + r]);
                }
            }
            named_bar_sync(1 + q4, 64);  // redl may be rewritten by the next item
            const float inv = 1.f / den;
            const bool tr2 = trace != nullptr && blockIdx.x == 0 && warp == 4 && lane == 0 && sc <= 64;
            if (tr2) trace[(sc - 1) * 8 + 5] = clock64();
            mbar_wait(&bar->o_full, t & 1);
            if (tr2) trace[(sc - 1) * 8 + 6] = clock64();
            tc_fence_after();
            const int qi = qt * AT_TILE + r;
            const int c = half * 32;
            float acc[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) acc[e] = 0.f;
#pragma unroll
            for (int j = 0; j < AT_MAXKB; ++j) {
                if (j < nkb) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(tmem + lane_addr + 256 + j * AT_D + c, v);
                    tmem_ld_wait();
                    const float wj = w[j] * inv;
#pragma unroll
                    for (int e = 0; e < 32; ++e) acc[e] = fmaf(wj, __uint_as_float(v[e]), acc[e]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->o_empty);
            if (tr2) trace[(sc - 1) * 8 + 7] = clock64();
            if (qi < S) {
                __nv_bfloat16* orow = out + ((size_t)b * S + qi) * dm + h * AT_D + c;
                uint4* o4 = reinterpret_cast<uint4*>(orow);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    o4[q] = make_uint4(pack_bf16(acc[8 * q], acc[8 * q + 1]), pack_bf16(acc[8 * q + 2], acc[8 * q + 3]),
                                       pack_bf16(acc[8 * q + 4], acc[8 * q + 5]),
                                       pack_bf16(acc[8 * q + 6], acc[8 * q + 7]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

static int g_at_sms = 0;

int attention_fwd_impl(const void* qkv, void* out, int B, int S, int H, unsigned long long* trace, cudaStream_t st) {
    RS_CHECK_ARG(B > 0 && S > 0 && H > 0, "attention: empty shape");
    RS_CHECK_ARG(S <= AT_TILE * AT_MAXKB, "attention: S=%d > %d not supported by the TMEM layout", S,
                 AT_TILE * AT_MAXKB);
    if (g_at_sms == 0) {
        int dev;
        RS_CUDA(cudaGetDevice(&dev));
        RS_CUDA(cudaDeviceGetAttribute(&g_at_sms, cudaDevAttrMultiProcessorCount, dev));
        RS_CUDA(cudaFuncSetAttribute(attention_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM));
    }
    const uint64_t rows = (uint64_t)B * S;
    const uint64_t cols = (uint64_t)3 * H * AT_D;
    CUtensorMap m;
    RS_TRY(make_tmap_bf16(&m, qkv, rows, cols, cols * 2, AT_TILE, AT_D));
    const int n_units = B * H;
    const int grid = n_units < g_at_sms ? n_units : g_at_sms;
    attention_fwd_kernel<<<grid, AT_THREADS, AT_SMEM, st>>>(m, static_cast<__nv_bfloat16*>(out), B, S, H, trace);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

int attention_fwd(const void* qkv, void* out, int B, int S, int H, cudaStream_t st) {
    return attention_fwd_impl(qkv, out, B, S, H, nullptr, st);
}

}  // namespace rs

extern "C" int rs_attention_fwd_trace(const void* qkv, void* out, int32_t B, int32_t S, int32_t H,
                                      unsigned long long* trace, void* stream) {
    return rs::attention_fwd_impl(qkv, out, B, S, H, trace, rs::as_stream(stream));
}

extern "C" int rs_attention_fwd(const void* qkv, void* out, int32_t B, int32_t S, int32_t H, void* stream) {
    return rs::attention_fwd(qkv, out, B, S, H, rs::as_stream(stream));
}
