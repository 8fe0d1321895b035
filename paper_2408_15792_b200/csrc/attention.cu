// K4: causal multi-head self-attention forward on tcgen05 (head dim 64, S <= 512).
//
// OPT attention (PAPER.md:195-201 backbone; HF OPTAttention semantics): per prompt and
// head, softmax(q k^T / sqrt(64) + causal mask) v over the packed qkv activation
// [B*S, 3*H*64] written by the QKV GEMM. The reference package has no backbone
// (SPEC.md:12), so the oracle is oracle/opt_ranker.py.
//
// Work: a unit is one (prompt, head); its q-tiles (128 queries) need key blocks
// 0..t (causal). A group of 4 / n_qt units keeps all its K/V blocks resident in smem
// (4 x 32 KB); the group's q-tiles are split between two softmax "slots" balanced by
// block count, and the two slots ping-pong on the tensor core:
//   warp 8      TMA: K/V blocks through a 5-deep ring (the next group's blocks land
//               while this group works); warps 10, 11: Q tiles of slot 0 / slot 1
//   warp 9      MMA: per slot S = Q K_j^T (M=128, N=128) into the slot's TMEM S region,
//               then O += P V_j (M=128, N=64) with P read from TMEM (tcgen05 A operand
//               in tensor memory) and V as an MN-major smem operand
//   warp 10     also the TMEM allocator (512 columns: slot s uses S at 256 s, O at 256 s + 128)
//   warps 0-3   slot 0 softmax, warps 4-7 slot 1: one query row per thread, the whole
//               128-key block in registers; online softmax with a lazily updated row
//               maximum (O is rescaled in TMEM only when the block max exceeds the running
//               max by more than 2^8); exponentials split between MUFU ex2 and a
//               degree-3 polynomial on the packed-fp32 FMA pipe; P goes back to TMEM as
//               bf16 over the S columns it replaces.
// Key blocks run diagonal first, so every row sees a valid key in its first block.
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "tma.cuh"

namespace rs {
using namespace sm100;

constexpr int AT_TILE = 128;  // queries per tile, keys per block
constexpr int AT_D = 64;
constexpr int AT_MAXKB = 4;  // S <= 512
constexpr int AT_BUF = AT_TILE * AT_D * 2;  // 16 KB: one Q tile or one K / V block
constexpr int AT_THREADS = 384;
// Warp roles. The SM's warp schedulers favour higher warp ids, so the latency-critical
// control warps sit above the 8 softmax warps (else the MMA issuer starves behind them).
constexpr int AT_W_KV = 8, AT_W_MMA = 9, AT_W_Q0 = 10;  // + AT_W_Q0 + 1; softmax: warps 0-7
constexpr int AT_KVB = 4;  // K/V ring depth (one group of <= 4 blocks)
// Q [2 slots][2] + K, V [AT_KVB] + the fp16 "ones" tile (F16V) + barriers
constexpr int AT_SMEM = (4 + 2 * AT_KVB + 1) * AT_BUF + 1024 + 1024;
constexpr float AT_RESCALE = 8.0f;
#ifndef AT_POLL_NS
#define AT_POLL_NS 32
#endif  // lazy-rescale threshold (log2 units)
// which of every 8 exponential pairs go to MUFU (bit set) vs the FMA-pipe polynomial
#ifndef AT_MUFU_MASK
#define AT_MUFU_MASK 0x57u  // 5 of 8 on MUFU (measured best of 0x11, 0x15, 0x55, 0x57, 0x77)
#endif

struct AtBars {
    uint64_t q_full[2][2], q_empty[2][2];
    uint64_t kv_full[AT_KVB], kv_empty[AT_KVB];
    uint64_t s_full[2], p_full[2], o_full[2];
    uint32_t tmem;
};

// i-th q-tile (heaviest first) of `slot` in a group of U units with n_qt tiles each:
// tiles sorted by block count (t + 1) descending, then unit; each goes to the slot with
// the smaller accumulated block count (ties to slot 0). Every role derives the same list.
__device__ __forceinline__ bool at_slot_tile(int n_qt, int U, int slot, int i, int& k, int& t) {
    int load0 = 0, load1 = 0;
    int seen = 0;
    for (int tt = n_qt - 1; tt >= 0; --tt)
        for (int kk = 0; kk < U; ++kk) {
            const int s = load1 < load0 ? 1 : 0;
            if (s) load1 += tt + 1; else load0 += tt + 1;
            if (s == slot) {
                if (seen == i) {
                    k = kk;
                    t = tt;
                    return true;
                }
                ++seen;
            }
        }
    return false;
}

// 2^x for x <= 0 on the FMA pipe, two lanes per packed-fp32 op: x = j + f with
// j = round(x), f in [-0.5, 0.5]; 2^f by a degree-3 minimax polynomial (max rel. error
// 1.0e-4, far below the bf16 rounding P gets); 2^j by an exponent-field add.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& p0, float& p1) {
    const uint64_t magic = f2pack(12582912.0f, 12582912.0f);  // 1.5 * 2^23
    const uint64_t X = f2pack(fmaxf(x0, -127.0f), fmaxf(x1, -127.0f));
    const uint64_t T = fadd2(X, magic);  // low mantissa bits = round(x)
    const uint64_t F = fsub2(X, fsub2(T, magic));
    uint64_t P = ffma2(F, f2pack(0.0550082f, 0.0550082f), f2pack(0.24220941f, 0.24220941f));
    P = ffma2(P, F, f2pack(0.69328284f, 0.69328284f));
    P = ffma2(P, F, f2pack(1.0f, 1.0f));
    float t0, t1, q0, q1;
    f2unpack(T, t0, t1);
    f2unpack(P, q0, q1);
    p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
    p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}
__device__ __forceinline__ float exp2_mufu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// D[tmem] (+)= A[tmem] * B[smem]: A (M x K, bf16 packed two per 32-bit column) read from
// tensor memory.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns from 16 registers per thread.
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

template <bool F16V>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attention_fwd_kernel(const __grid_constant__ CUtensorMap tqkv, __nv_bfloat16* __restrict__ out, int B, int S,
                         int H, float* __restrict__ lse) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                  // [slot][2]
    uint8_t* sK = sQ + 4 * AT_BUF;       // [AT_KVB]
    uint8_t* sV = sK + AT_KVB * AT_BUF;  // [AT_KVB]
    uint8_t* sOnes = sV + AT_KVB * AT_BUF;  // F16V: 128 keys x 64 fp16, column 0 = 1
    AtBars* bar = reinterpret_cast<AtBars*>(sOnes + AT_BUF);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_qt = (S + AT_TILE - 1) / AT_TILE;
    const int dm = H * AT_D;
    const int n_units = B * H;
    const int gU = AT_MAXKB / n_qt;  // units per group
    const int n_groups = (n_units + gU - 1) / gU;

    if (warp == AT_W_KV && lane == 0) {
        tma_prefetch_desc(&tqkv);
        for (int s = 0; s < 2; ++s) {
            for (int q = 0; q < 2; ++q) {
                mbar_init(&bar->q_full[s][q], 1);
                mbar_init(&bar->q_empty[s][q], 1);
            }
            mbar_init(&bar->s_full[s], 1);
            mbar_init(&bar->p_full[s], 4);
            mbar_init(&bar->o_full[s], 1);
        }
        for (int i = 0; i < AT_KVB; ++i) {
            mbar_init(&bar->kv_full[i], 1);
            mbar_init(&bar->kv_empty[i], 1);  // committed by the buffer's last PV
        }
        fence_barrier_init();
    }
    if (warp == AT_W_Q0) tmem_alloc<512>(&bar->tmem);
    if (F16V) {
        // The PV MMA runs with N = 80: V (64 columns) plus this tile as the next 64-wide
        // MN chunk, whose first column is all ones, so O column 64 accumulates the row sum
        // of the fp16 P the MMA actually used (no ALU sums). MN-major SW128 layout: key
        // row k at k * 128 B, 16-B chunk c stored at position c ^ (k % 8).
        for (int i = threadIdx.x; i < AT_BUF / 16; i += AT_THREADS) {
            const int k = i >> 3, cpos = i & 7;
            const uint32_t one = (cpos == (k & 7)) ? 0x3C00u : 0u;  // chunk 0 holds column 0
            reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(one, 0u, 0u, 0u);
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem;

    // K/V blocks stream through a ring of AT_KVB buffers in load order: load n of this CTA
    // (group gi, block j from n_qt - 1 down to 0, unit k) goes to buffer n % AT_KVB, so the
    // next group's first blocks land while this group still works (the ring holds one
    // group plus a spare). Q is single-buffered per slot; its next tile loads as soon as
    // the current tile's last S retires (a softmax + PV ahead of its use).
    auto kv_seq = [&](int gi, int U, int k, int j) { return gi * gU * n_qt + (n_qt - 1 - j) * U + k; };
    if (warp == AT_W_KV) {
        if (elect_one()) {
            int gi = 0;
            for (int g = blockIdx.x; g < n_groups; g += gridDim.x, ++gi) {
                const int U = min(gU, n_units - g * gU);
                for (int j = n_qt - 1; j >= 0; --j)
                    for (int kk = 0; kk < U; ++kk) {
                        const int n = kv_seq(gi, U, kk, j);
                        const int buf = n % AT_KVB;
                        const int unit = g * gU + kk;
                        const int b = unit / H, h = unit % H;
                        mbar_wait(&bar->kv_empty[buf], ((n / AT_KVB) & 1) ^ 1);
                        mbar_arrive_expect_tx(&bar->kv_full[buf], 2 * AT_BUF);
                        tma_load_2d(sK + buf * AT_BUF, &tqkv, &bar->kv_full[buf], dm + h * AT_D, b * S + j * AT_TILE);
                        tma_load_2d(sV + buf * AT_BUF, &tqkv, &bar->kv_full[buf], 2 * dm + h * AT_D,
                                    b * S + j * AT_TILE);
                    }
            }
        }
    } else if (warp == AT_W_Q0 || warp == AT_W_Q0 + 1) {
        // Q producer for slot warp - AT_W_Q0
        const int s = warp - AT_W_Q0;
        if (elect_one()) {
            int tq = 0;
            for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
                const int U = min(gU, n_units - g * gU);
                int k, t;
                for (int i = 0; at_slot_tile(n_qt, U, s, i, k, t); ++i, ++tq) {
                    const int unit = g * gU + k;
                    const int b = unit / H, h = unit % H;
                    const int qb = tq & 1;
                    mbar_wait(&bar->q_empty[s][qb], ((tq >> 1) & 1) ^ 1);
                    mbar_arrive_expect_tx(&bar->q_full[s][qb], AT_BUF);
                    tma_load_2d(sQ + (s * 2 + qb) * AT_BUF, &tqkv, &bar->q_full[s][qb], h * AT_D, b * S + t * AT_TILE);
                }
            }
        }
    } else if (warp == AT_W_MMA) {
        if (elect_one()) {
            constexpr uint32_t id_s = idesc_bf16(AT_TILE, AT_TILE);
            // PV: bf16 P x bf16 V (N = 64), or fp16 P x [fp16 V | ones] (N = 80)
            constexpr uint32_t id_o = F16V ? (idesc_bf16(AT_TILE, AT_D + 16, 0, 1) & ~((7u << 7) | (7u << 10)))
                                           : idesc_bf16(AT_TILE, AT_D, 0, 1);
            // All MMA-issuer state stays in registers: with ~225 KB of shared memory the L1
            // left for local memory is tiny, and a spilled / dynamically indexed array costs
            // an L2 round trip per access on this latency-critical path.
            struct Slot {
                int tseq, bseq;  // tiles / blocks issued so far
                int i, k, t, j;  // tile index in the group's list, its unit, q-tile, block
                bool live;
            };
            Slot s0{0, 0, 0, 0, 0, 0, false}, s1{0, 0, 0, 0, 0, 0, false};
            uint32_t uses = 0;  // PVs still to read each K/V buffer, 4 bits per ring slot
            int gi = 0;
            for (int g = blockIdx.x; g < n_groups; g += gridDim.x, ++gi) {
                const int U = min(gU, n_units - g * gU);
                for (int j = 0; j < n_qt; ++j)
                    for (int kk = 0; kk < U; ++kk) {
                        const int b4 = 4 * (kv_seq(gi, U, kk, j) % AT_KVB);
                        uses = (uses & ~(15u << b4)) | ((uint32_t)(n_qt - j) << b4);
                    }
                auto start = [&](Slot& c, int slot) {
                    c.i = 0;
                    c.live = at_slot_tile(n_qt, U, slot, 0, c.k, c.t);
                    c.j = c.t;
                };
                auto issue_s = [&](Slot& c, int slot) {
                    const int n = kv_seq(gi, U, c.k, c.j);
                    const int buf = n % AT_KVB;
                    const int qb = c.tseq & 1;
                    if (c.j == c.t) mbar_wait(&bar->q_full[slot][qb], (c.tseq >> 1) & 1);
                    mbar_wait(&bar->kv_full[buf], (n / AT_KVB) & 1);
                    tc_fence_after();
                    const uint32_t qa = smem_u32(sQ + (slot * 2 + qb) * AT_BUF);
                    const uint32_t ka = smem_u32(sK + buf * AT_BUF);
#pragma unroll
                    for (int kk = 0; kk < AT_D / 16; ++kk)
                        mma_bf16_ss(tmem + slot * 256, desc_kmajor_sw128(qa + kk * 32),
                                    desc_kmajor_sw128(ka + kk * 32), id_s, kk != 0);
                    mma_commit(&bar->s_full[slot]);
                    if (c.j == 0) mma_commit(&bar->q_empty[slot][qb]);  // last S of the tile
                };
                auto issue_pv = [&](Slot& c, int slot) {
                    const int buf = kv_seq(gi, U, c.k, c.j) % AT_KVB;
                    ++c.bseq;
                    tc_fence_after();
                    const uint32_t vb = smem_u32(sV + buf * AT_BUF);
                    const uint32_t lbo = F16V ? (uint32_t)(sOnes - (sV + buf * AT_BUF)) : 8192u;  // V -> ones
#pragma unroll
                    for (int kk = 0; kk < AT_TILE / 16; ++kk)
                        mma_bf16_ts(tmem + slot * 256 + 128, tmem + slot * 256 + kk * 8,
                                    desc_mnmajor_sw128(vb + kk * 2048, lbo), id_o, (c.j != c.t) || kk != 0);
                    uses -= 1u << (4 * buf);
                    if (((uses >> (4 * buf)) & 15u) == 0) mma_commit(&bar->kv_empty[buf]);
                    if (c.j == 0) {  // tile done: O is final once this PV retires
                        mma_commit(&bar->o_full[slot]);
                        ++c.tseq;
                        ++c.i;
                        c.live = at_slot_tile(n_qt, U, slot, c.i, c.k, c.t);
                        c.j = c.t;
                    } else {
                        --c.j;
                    }
                    if (c.live) issue_s(c, slot);
                };
                start(s0, 0);
                start(s1, 1);
                if (s0.live) issue_s(s0, 0);
                if (s1.live) issue_s(s1, 1);
                while (s0.live || s1.live) {
                    // issue for whichever slot's P is ready first (no head-of-line blocking)
                    // (test_wait: try_wait may park the thread on one barrier while the other
                    // slot is ready)
                    if (s0.live && mbar_test_wait(&bar->p_full[0], s0.bseq & 1))
                        issue_pv(s0, 0);
                    else if (s1.live && mbar_test_wait(&bar->p_full[1], s1.bseq & 1))
                        issue_pv(s1, 1);
                    else
                        __nanosleep(AT_POLL_NS);  // back off: this warp shares its SM sub-partition
                                                  // with two softmax warps and would steal their issue slots
                }
            }
        }
    } else if (warp < 8) {
        const int s = warp >> 2;         // slot
        const int q4 = warp & 3;         // TMEM lane quarter
        const int r = q4 * 32 + lane;    // query row within the tile == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const uint32_t tS = tmem + s * 256 + lane_addr, tO = tS + 128;
        const float c = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)
        const uint64_t c2 = f2pack(c, c);
        int tseq = 0, bseq = 0;
        for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
            const int U = min(gU, n_units - g * gU);
            int k, t;
            for (int i = 0; at_slot_tile(n_qt, U, s, i, k, t); ++i, ++tseq) {
                const int unit = g * gU + k;
                const int b = unit / H, h = unit % H;
                float m_run = 0.f, l = 0.f;
                for (int j = t; j >= 0; --j, ++bseq) {
                    mbar_wait(&bar->s_full[s], bseq & 1);
                    tc_fence_after();
                    // pass 1: row max over the block, 32 columns at a time (a whole row in
                    // registers would leave ptxas no room for ILP; TMEM loads are cheap)
                    const bool diag = j == t;  // diagonal block: key e valid iff e <= r
                    float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        // diagonal block: chunks past this warp's 32 rows are fully masked, the
                        // chunk on its rows is masked per lane (key e valid iff e <= lane)
                        if (diag && cc > q4) break;
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(tS + cc * 32, v);
                        tmem_ld_wait();
                        if (diag && cc == q4) {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e > lane) v[e] = __float_as_uint(-INFINITY);
                        }
#pragma unroll
                        for (int e = 0; e < 32; e += 8)
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                mq[u] = fmax3(mq[u], __uint_as_float(v[e + 2 * u]), __uint_as_float(v[e + 2 * u + 1]));
                    }
                    const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
                    const float mb = mx * c;
                    float alpha = 1.f;
                    if (j == t) {
                        m_run = mb;
                    } else if (mb > m_run + AT_RESCALE) {
                        alpha = exp2_mufu(m_run - mb);
                        m_run = mb;
                    }
                    // pass 2: P = 2^(s c - m_run), bf16 pairs over the first 64 S columns (the
                    // PV MMA's A operand; chunk cc's 16 P columns lie in S columns already read)
                    const uint64_t nm2 = f2pack(-m_run, -m_run);
                    uint64_t lsum[4] = {f2pack(0.f, 0.f), f2pack(0.f, 0.f), f2pack(0.f, 0.f), f2pack(0.f, 0.f)};
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        uint32_t pk[16];
                        if (diag && cc > q4) {  // fully masked: P = 0
#pragma unroll
                            for (int e = 0; e < 16; ++e) pk[e] = 0u;
                            tmem_st_32x32b_x16(tS + cc * 16, pk);
                            continue;
                        }
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(tS + cc * 32, v);
                        tmem_ld_wait();
                        if (diag && cc == q4) {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (e > lane) v[e] = __float_as_uint(-INFINITY);
                        }
#pragma unroll
                        for (int e = 0; e < 32; e += 2) {
                            float x0, x1;
                            f2unpack(ffma2(f2pack(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), c2, nm2), x0, x1);
                            float p0, p1;
                            if (((AT_MUFU_MASK >> ((e >> 1) & 7)) & 1) != 0) {  // MUFU, else the FMA pipe
                                p0 = exp2_mufu(x0);
                                p1 = exp2_mufu(x1);
                            } else {
                                exp2_poly2(x0, x1, p0, p1);
                            }
                            if (F16V) {
                                pk[e / 2] = pack_f16(p0, p1);  // row sum: O column 64 (ones column)
                            } else {
                                lsum[(e >> 1) & 3] = fadd2(lsum[(e >> 1) & 3], f2pack(p0, p1));
                                pk[e / 2] = pack_bf16(p0, p1);
                            }
                        }
                        tmem_st_32x32b_x16(tS + cc * 16, pk);
                    }
                    if (!F16V) {
                        float l0, l1;
                        f2unpack(fadd2(fadd2(lsum[0], lsum[1]), fadd2(lsum[2], lsum[3])), l0, l1);
                        l = l * alpha + l0 + l1;
                    }
                    if (__any_sync(0xffffffffu, alpha != 1.f)) {
                        // O holds PV of the earlier blocks,
                        // retired: the S commit covers them
#pragma unroll
                        for (int hh = 0; hh < (F16V ? 3 : 2); ++hh) {  // F16V: + the row-sum column
                            uint32_t o[32];
                            tmem_ld_32x32b_x32(tO + hh * 32, o);
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                            tmem_st_32x32b_x32(tO + hh * 32, o);
                        }
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bar->p_full[s]);
                }
                // epilogue: O / l -> bf16 rows of `out`
                mbar_wait(&bar->o_full[s], tseq & 1);
                tc_fence_after();
                uint32_t o[64];
                tmem_ld_32x32b_x32(tO, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                tmem_ld_32x32b_x32(tO + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
                if (F16V) {
                    uint32_t ls;
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(ls) : "r"(tO + 64));
                    tmem_ld_wait();
                    l = __uint_as_float(ls);
                } else {
                    tmem_ld_wait();
                }
                tc_fence_before();
                const float inv = 1.f / l;
                const int qi = t * AT_TILE + r;
                // the row's log2-sum-exp (scaled scores): P = 2^(s c - lse) for the backward
                if (lse != nullptr && qi < S) lse[((size_t)b * H + h) * S + qi] = m_run + __log2f(l);
                if (qi < S) {
                    uint4* o4 = reinterpret_cast<uint4*>(out + ((size_t)b * S + qi) * dm + h * AT_D);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        o4[q] = make_uint4(pack_bf16(__uint_as_float(o[8 * q]) * inv, __uint_as_float(o[8 * q + 1]) * inv),
                                           pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv),
                                           pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv),
                                           pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == AT_W_Q0) tmem_dealloc<512>(tmem);
}

template <bool F16V>
static int launch_attention(const void* qkv, void* out, int B, int S, int H, cudaStream_t st, float* lse) {
    const int sms = num_sms();
    RS_CUDA(ensure_smem((const void*)attention_fwd_kernel<F16V>, AT_SMEM));
    const uint64_t rows = (uint64_t)B * S;
    const uint64_t cols = (uint64_t)3 * H * AT_D;
    CUtensorMap m;
    RS_TRY(make_tmap_bf16(&m, qkv, rows, cols, cols * 2, AT_TILE, AT_D));  // 16-bit elements; V may be fp16
    const int n_qt = (S + AT_TILE - 1) / AT_TILE;
    const int gU = AT_MAXKB / n_qt;
    const int n_groups = (B * H + gU - 1) / gU;
    const int grid = n_groups < sms ? n_groups : sms;
    attention_fwd_kernel<F16V><<<grid, AT_THREADS, AT_SMEM, st>>>(m, static_cast<__nv_bfloat16*>(out), B, S, H, lse);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

int attention_fwd_impl(const void* qkv, void* out, int B, int S, int H, int v_f16, cudaStream_t st,
                       float* lse = nullptr) {
    RS_CHECK_ARG(B > 0 && S > 0 && H > 0, "attention: empty shape");
    RS_CHECK_ARG(S <= AT_TILE * AT_MAXKB, "attention: S=%d > %d not supported", S, AT_TILE * AT_MAXKB);
    return v_f16 ? launch_attention<true>(qkv, out, B, S, H, st, lse)
                 : launch_attention<false>(qkv, out, B, S, H, st, lse);
}
// the training forward: also the rows' log2-sum-exp, lse[(b H + h) S + row] (fp32)
int attention_fwd_lse(const void* qkv, void* out, float* lse, int B, int S, int H, cudaStream_t st) {
    return attention_fwd_impl(qkv, out, B, S, H, 0, st, lse);
}

int attention_fwd(const void* qkv, void* out, int B, int S, int H, cudaStream_t st) {
    return attention_fwd_impl(qkv, out, B, S, H, 0, st);
}
int attention_fwd_f16v(const void* qkv, void* out, int B, int S, int H, cudaStream_t st) {
    return attention_fwd_impl(qkv, out, B, S, H, 1, st);
}

}  // namespace rs

extern "C" int rs_attention_fwd(const void* qkv, void* out, int32_t B, int32_t S, int32_t H, void* stream) {
    RS_NVTX();
    return rs::attention_fwd(qkv, out, B, S, H, rs::as_stream(stream));
}

extern "C" int rs_attention_fwd_f16v(const void* qkv, void* out, int32_t B, int32_t S, int32_t H, void* stream) {
    RS_NVTX();
    return rs::attention_fwd_f16v(qkv, out, B, S, H, rs::as_stream(stream));
}

extern "C" int rs_attention_fwd_lse(const void* qkv, void* out, float* lse, int32_t B, int32_t S, int32_t H,
                                    void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(lse != nullptr, "rs_attention_fwd_lse: lse is NULL");
    return rs::attention_fwd_lse(qkv, out, lse, B, S, H, rs::as_stream(stream));
}
