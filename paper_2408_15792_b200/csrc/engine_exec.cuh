// Block-level pieces of the device engine step (engine.cu's kernels and the one-launch
// engine loop in rankstep.cu): admission of one request into a queue row, the reference's
// `_Sim.execute` (engine.py:247-284) on one CTA, and the chunks of the stable out-of-place
// compaction of the surviving rows.
#pragma once
#include "common.cuh"

namespace rs {

constexpr int EX_THREADS = 1024;
constexpr uint8_t EX_DONE = 8;     // row finished this step (dropped by the compaction)
constexpr uint8_t EX_PRE = 16;     // row preempted this step (cleared before the step ends)
constexpr int EX_PRE_CAP = 4096;   // preempted rows ordered in shared memory up to this many

__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    total = warp_tot[(blockDim.x >> 5) - 1];
    const int before = wid ? warp_tot[wid - 1] : 0;
    __syncthreads();
    return before + x - v;
}

// request r of the trace enters the queue at `row` (engine.py:404-412's alive insert)
__device__ __forceinline__ void engine_admit_row(const rs_engine_queue& q, const rs_engine_trace& tr, int r,
                                                 int64_t row) {
    if (q.score_dtype == RS_F64)
        static_cast<double*>(q.score)[row] = static_cast<const double*>(tr.score)[r];
    else
        static_cast<float*>(q.score)[row] = static_cast<const float*>(tr.score)[r];
    q.flags[row] = RS_FLAG_SCORED;
    q.prompt_tokens[row] = tr.prompt_tokens[r];
    q.generated_tokens[row] = 0;
    q.arrival_rank[row] = tr.arrival_rank[r];
    q.id[row] = r;
    q.starvation[row] = 0;
    q.quantum[row] = 0;
    tr.row_of[r] = (int32_t)row;
    tr.last_event_ns[r] = tr.arrival_ns[r];
}

// Phases 1-3 of _Sim.execute on one CTA of EX_THREADS threads (µs of work: every phase
// needs the previous one complete). Preemption only concerns rows that were RUNNING (<=
// last step's batch) and prefill only rows in this step's run, so neither phase walks the
// queue with ordered scans: preempted rows are collected unordered and put back in alive
// (row) order by a shared-memory bitonic sort. Compaction is either in place (InPlace, one
// CTA, ordered block scans) or left to the compaction chunks below (out of place, many
// CTAs). pre_rows: shared scratch of EX_PRE_CAP ints; warp_tot: shared int[32].
// Lists = false (the record-free engine loop): the preempted / finished id lists are not
// written, so neither is ordered (only counted).
template <bool InPlace, bool Lists = true>
__device__ __forceinline__ void engine_execute_block(const rs_engine_queue& q, const rs_engine_trace& tr,
                                                     const rs_engine_cost& cost, const int64_t* __restrict__ run,
                                                     const int32_t* __restrict__ counts, int32_t step,
                                                     int64_t predictor_ns, int64_t* __restrict__ out,
                                                     int64_t* __restrict__ preempted, int64_t* __restrict__ finished,
                                                     int64_t* __restrict__ prev_run, int32_t* __restrict__ prev_n,
                                                     int* pre_rows, int* warp_tot) {
    __shared__ unsigned long long prefill_tokens;
    __shared__ int n_pre;
    __shared__ long long now_s;
    __shared__ int n_fin_s;
    const int tid = threadIdx.x;
    const int n_run = *(volatile const int32_t*)counts;
    const int64_t n = q.n;
    if (tid == 0) {
        prefill_tokens = 0ull;
        n_pre = 0;
        n_fin_s = 0;
    }
    for (int k = tid; k < n_run; k += EX_THREADS) tr.run_stamp[run[k]] = step;
    __syncthreads();
    // 1a. preemption (engine.py:248-256): RUNNING rows left out of the batch. RUNNING is
    // set only on the rows of a step's batch and cleared when they are left out, so with
    // the previous batch at hand (prev_run) only those rows need looking at; else scan.
    auto preempt_row = [&](int64_t row, int64_t id) {
        const uint8_t fl = q.flags[row];
        if ((fl & RS_FLAG_RUNNING) && tr.run_stamp[id] != step) {
            q.flags[row] = (uint8_t)((fl & ~RS_FLAG_RUNNING) | (Lists ? EX_PRE : 0));
            tr.n_preempted[id] += 1;
            const int slot = atomicAdd(&n_pre, 1);
            if (Lists && slot < EX_PRE_CAP) pre_rows[slot] = (int)row;
        }
    };
    if (prev_run) {
        const int pn = *prev_n;
        for (int i = tid; i < pn; i += EX_THREADS) {
            const int64_t id = prev_run[i];
            if (tr.finish_ns[id] >= 0) continue;  // finished last step: already retired
            preempt_row(tr.row_of[id], id);
        }
    } else {
        for (int64_t row = tid; row < n; row += EX_THREADS)
            if (q.flags[row] & RS_FLAG_RUNNING) preempt_row(row, q.id[row]);
    }
    __syncthreads();
    const int total_pre = n_pre;
    if constexpr (!Lists) {
    } else if (total_pre <= EX_PRE_CAP) {
        int np2 = 1;
        while (np2 < total_pre) np2 <<= 1;
        for (int i = total_pre + tid; i < np2; i += EX_THREADS) pre_rows[i] = 0x7fffffff;
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = tid; t < (np2 >> 1); t += EX_THREADS) {
                    const int i = 2 * j * (t / j) + (t % j), p = i + j;
                    const int a = pre_rows[i], b = pre_rows[p];
                    if ((b < a) == ((i & k) == 0)) {
                        pre_rows[i] = b;
                        pre_rows[p] = a;
                    }
                }
                __syncthreads();
            }
        }
        for (int i = tid; i < total_pre; i += EX_THREADS) {
            const int row = pre_rows[i];
            preempted[i] = q.id[row];
            q.flags[row] &= (uint8_t)~EX_PRE;
        }
    } else {
        // more than EX_PRE_CAP preemptions (max_batch > EX_PRE_CAP): ordered block scans
        int base_out = 0;
        for (int64_t base = 0; base < n; base += EX_THREADS) {
            const int64_t row = base + tid;
            int pre = 0;
            if (row < n && (q.flags[row] & EX_PRE)) {
                pre = 1;
                q.flags[row] &= (uint8_t)~EX_PRE;
            }
            int total;
            const int pos = block_excl_scan(pre, warp_tot, total);
            if (pre) preempted[base_out + pos] = q.id[row];
            base_out += total;
        }
    }
    // 1b. prefill (engine.py:257-262): scheduled rows that were not running
    unsigned long long pf = 0ull;
    for (int k = tid; k < n_run; k += EX_THREADS) {
        const int row = tr.row_of[run[k]];
        const uint8_t fl = q.flags[row];
        if (!(fl & RS_FLAG_RUNNING)) {
            pf += (unsigned long long)(q.prompt_tokens[row] + q.generated_tokens[row]);
            q.flags[row] = (uint8_t)(fl | RS_FLAG_RUNNING);
        }
    }
    pf = warp_sum(pf);
    if ((tid & 31) == 0 && pf) atomicAdd(&prefill_tokens, pf);
    __syncthreads();
    // 2. clock
    if (tid == 0) {
        long long dec;
        if (cost.decode_table_len > 0) {
            const int b = n_run < cost.decode_table_len ? n_run : cost.decode_table_len;
            dec = cost.decode_table[b - 1];
        } else {
            dec = cost.decode_ns;
        }
        const long long iter = (long long)prefill_tokens * cost.prefill_ns_per_token + dec + predictor_ns;
        now_s = out[0] + iter;
        out[0] = now_s;
        out[1] = iter;
        out[2] = (long long)prefill_tokens * cost.prefill_ns_per_token;
        out[4] = total_pre;
    }
    __syncthreads();
    const long long now = now_s;
    // 3. one token per scheduled request, in fill order (engine.py:270-280)
    int done_before = 0;
    for (int base = 0; base < n_run; base += EX_THREADS) {
        const int k = base + tid;
        int fin = 0;
        int64_t id = 0;
        if (k < n_run) {
            id = run[k];
            const int row = tr.row_of[id];
            const int g = q.generated_tokens[row] + 1;
            q.generated_tokens[row] = g;
            const long long gap = now - tr.last_event_ns[id];
            if (gap > tr.max_gap_ns[id]) tr.max_gap_ns[id] = gap;
            if (tr.first_token_ns[id] < 0) tr.first_token_ns[id] = now;
            tr.last_event_ns[id] = now;
            if (g >= tr.true_output[id]) {
                tr.finish_ns[id] = now;
                q.flags[row] |= EX_DONE;
                fin = 1;
            }
        }
        if constexpr (Lists) {
            int total;
            const int pos = block_excl_scan(fin, warp_tot, total);
            if (fin) finished[done_before + pos] = id;
            done_before += total;
        } else {
            const unsigned b = __ballot_sync(0xffffffffu, fin);
            if ((tid & 31) == 0 && b) atomicAdd(&n_fin_s, __popc(b));
        }
    }
    if constexpr (!Lists) {
        __syncthreads();
        done_before = n_fin_s;
    }
    __syncthreads();
    if (tid == 0) out[5] = done_before;
    if (prev_run) {  // this batch is the next step's RUNNING set
        for (int k = tid; k < n_run; k += EX_THREADS) prev_run[k] = run[k];
        if (tid == 0) *prev_n = n_run;
    }
    if constexpr (!InPlace) return;
    // 4. stable in-place compaction of the rows still alive
    int64_t kept = 0;
    for (int64_t base = 0; base < n; base += EX_THREADS) {
        const int64_t row = base + tid;
        const bool valid = row < n;
        double sc = 0.0;
        uint8_t fl = 0;
        int32_t pr = 0, ge = 0, st = 0, qu = 0;
        uint32_t ar = 0;
        int64_t id = 0;
        if (valid) {
            sc = q.score_dtype == RS_F64 ? static_cast<const double*>(q.score)[row]
                                         : (double)static_cast<const float*>(q.score)[row];
            fl = q.flags[row];
            pr = q.prompt_tokens[row];
            ge = q.generated_tokens[row];
            ar = q.arrival_rank[row];
            id = q.id[row];
            st = q.starvation[row];
            qu = q.quantum[row];
        }
        const int keep = valid && !(fl & EX_DONE);
        int total;
        const int pos = block_excl_scan(keep, warp_tot, total);  // (its barriers order reads before writes)
        if (keep) {
            const int64_t dst = kept + pos;
            if (q.score_dtype == RS_F64)
                static_cast<double*>(q.score)[dst] = sc;
            else
                static_cast<float*>(q.score)[dst] = (float)sc;
            q.flags[dst] = fl;
            q.prompt_tokens[dst] = pr;
            q.generated_tokens[dst] = ge;
            q.arrival_rank[dst] = ar;
            q.id[dst] = id;
            q.starvation[dst] = st;
            q.quantum[dst] = qu;
            tr.row_of[id] = (int32_t)dst;
        }
        kept += total;
        __syncthreads();
    }
    if (tid == 0) out[3] = kept;
}

// Out-of-place stable compaction (queue q -> q_out), chunk c = rows [c * EX_THREADS, ...):
// the chunk's survivor count, then (once every chunk's count is known) its scatter at
// `base` = the survivors of the chunks before it. Both return the chunk's survivor count.
__device__ __forceinline__ int compact_count_chunk(const uint8_t* __restrict__ flags, int64_t n, int64_t c,
                                                   int* warp_tot) {
    const int64_t row = c * EX_THREADS + threadIdx.x;
    const int keep = row < n && !(flags[row] & EX_DONE);
    int total;
    block_excl_scan(keep, warp_tot, total);
    return total;
}
__device__ __forceinline__ int compact_scatter_chunk(const rs_engine_queue& q, const rs_engine_queue& qo,
                                                     const rs_engine_trace& tr, int64_t c, int64_t base,
                                                     int* warp_tot) {
    const int64_t row = c * EX_THREADS + threadIdx.x;
    const bool valid = row < q.n;
    const uint8_t fl = valid ? q.flags[row] : (uint8_t)EX_DONE;
    const int keep = !(fl & EX_DONE);
    int total;
    const int pos = block_excl_scan(keep, warp_tot, total);
    if (keep) {
        const int64_t dst = base + pos;
        if (q.score_dtype == RS_F64)
            static_cast<double*>(qo.score)[dst] = static_cast<const double*>(q.score)[row];
        else
            static_cast<float*>(qo.score)[dst] = static_cast<const float*>(q.score)[row];
        const int64_t id = q.id[row];
        qo.flags[dst] = fl;
        qo.prompt_tokens[dst] = q.prompt_tokens[row];
        qo.generated_tokens[dst] = q.generated_tokens[row];
        qo.arrival_rank[dst] = q.arrival_rank[row];
        qo.id[dst] = id;
        qo.starvation[dst] = q.starvation[row];
        qo.quantum[dst] = q.quantum[row];
        tr.row_of[id] = (int32_t)dst;
    }
    return total;
}

}  // namespace rs
