// Device-resident engine step (the caller of the hot path):
// admission into the resident queue and the reference's `_Sim.execute`
// (engine.py:247-284) — preempt running requests left out of the batch, charge prefill
// for the ones (re)starting, advance the clock by prefill + decode + predictor time,
// emit one token per scheduled request (`_ReqTrack.on_token`, engine.py:108-125), retire
// finished requests and compact the queue in place (stable, so row order stays the
// `alive` dict's insertion order the ranking policy's promoted / demoted lists follow).
// One CTA: a step touches each alive row a few times (µs of work) and every phase needs
// the previous one complete, so grid-wide synchronisation would cost more than it saves.
#include "common.cuh"

namespace rs {

constexpr int EX_THREADS = 1024;
constexpr uint8_t EX_DONE = 8;  // row finished this step (dropped by the compaction)

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

__global__ void __launch_bounds__(EX_THREADS) engine_admit_kernel(rs_engine_queue q, rs_engine_trace tr,
                                                                  const int32_t* __restrict__ req, int32_t k,
                                                                  int64_t n_alive) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const int r = req[i];
    const int64_t row = n_alive + i;
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

constexpr uint8_t EX_PRE = 16;     // row preempted this step (cleared before the kernel ends)
constexpr int EX_PRE_CAP = 4096;   // preempted rows ordered in shared memory up to this many

// Phases 1-3 of _Sim.execute on one CTA (µs of work: every phase needs the previous one
// complete). Preemption only concerns rows that were RUNNING (<= last step's batch) and
// prefill only rows in this step's run, so neither phase walks the queue with ordered
// scans: preempted rows are collected unordered and put back in alive (row) order by a
// shared-memory bitonic sort. Compaction is either in place (InPlace, one CTA, ordered
// block scans) or left to engine_compact_* (out of place, many CTAs).
template <bool InPlace>
__global__ void __launch_bounds__(EX_THREADS) engine_execute_kernel(rs_engine_queue q, rs_engine_trace tr,
                                                                    rs_engine_cost cost, const int64_t* __restrict__ run,
                                                                    const int32_t* __restrict__ counts, int32_t step,
                                                                    int64_t predictor_ns, int64_t* __restrict__ out,
                                                                    int64_t* __restrict__ preempted,
                                                                    int64_t* __restrict__ finished,
                                                                    int64_t* __restrict__ prev_run,
                                                                    int32_t* __restrict__ prev_n) {
    __shared__ int warp_tot[32];
    __shared__ unsigned long long prefill_tokens;
    __shared__ int n_pre;
    __shared__ int pre_rows[EX_PRE_CAP];
    const int tid = threadIdx.x;
    const int n_run = counts[0];
    const int64_t n = q.n;
    if (tid == 0) {
        prefill_tokens = 0ull;
        n_pre = 0;
    }
    for (int k = tid; k < n_run; k += EX_THREADS) tr.run_stamp[run[k]] = step;
    __syncthreads();
    // 1a. preemption (engine.py:248-256): RUNNING rows left out of the batch. RUNNING is
    // set only on the rows of a step's batch and cleared when they are left out, so with
    // the previous batch at hand (prev_run) only those rows need looking at; else scan.
    auto preempt_row = [&](int64_t row, int64_t id) {
        const uint8_t fl = q.flags[row];
        if ((fl & RS_FLAG_RUNNING) && tr.run_stamp[id] != step) {
            q.flags[row] = (uint8_t)((fl & ~RS_FLAG_RUNNING) | EX_PRE);
            tr.n_preempted[id] += 1;
            const int slot = atomicAdd(&n_pre, 1);
            if (slot < EX_PRE_CAP) pre_rows[slot] = (int)row;
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
    if (total_pre <= EX_PRE_CAP) {
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
    __shared__ long long now_s;
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
        int total;
        const int pos = block_excl_scan(fin, warp_tot, total);
        if (fin) finished[done_before + pos] = id;
        done_before += total;
    }
    __syncthreads();
    if (tid == 0) out[5] = done_before;
    if (prev_run) {  // this batch is the next step's RUNNING set
        for (int k = tid; k < n_run; k += EX_THREADS) prev_run[k] = run[k];
        if (tid == 0) *prev_n = n_run;
    }
    if (!InPlace) return;
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

// Out-of-place stable compaction (queue q -> q_out) over many CTAs: per-CTA survivor
// counts, then each CTA sums the counts before it (<= n / 1024 of them) and scatters.
__global__ void __launch_bounds__(EX_THREADS) engine_compact_count(const uint8_t* __restrict__ flags, int64_t n,
                                                                   int32_t* __restrict__ block_keep) {
    __shared__ int warp_tot[32];
    const int64_t row = (int64_t)blockIdx.x * EX_THREADS + threadIdx.x;
    const int keep = row < n && !(flags[row] & EX_DONE);
    int total;
    block_excl_scan(keep, warp_tot, total);
    if (threadIdx.x == 0) block_keep[blockIdx.x] = total;
}

__global__ void __launch_bounds__(EX_THREADS) engine_compact_scatter(rs_engine_queue q, rs_engine_queue qo,
                                                                     rs_engine_trace tr,
                                                                     const int32_t* __restrict__ block_keep,
                                                                     int64_t* __restrict__ out) {
    __shared__ int warp_tot[32];
    __shared__ long long base_s;
    const int tid = threadIdx.x;
    if (tid < 32) {
        long long b = 0;
        for (int k = tid; k < (int)blockIdx.x; k += 32) b += block_keep[k];
        b = warp_sum(b);
        if (tid == 0) base_s = b;
    }
    const int64_t row = (int64_t)blockIdx.x * EX_THREADS + tid;
    const bool valid = row < q.n;
    const uint8_t fl = valid ? q.flags[row] : (uint8_t)EX_DONE;
    const int keep = !(fl & EX_DONE);
    int total;
    const int pos = block_excl_scan(keep, warp_tot, total);  // its barriers publish base_s
    if (keep) {
        const int64_t dst = base_s + pos;
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
    if (blockIdx.x == gridDim.x - 1 && tid == 0) out[3] = base_s + total;
}

}  // namespace rs

using namespace rs;

extern "C" int rs_engine_admit(const rs_engine_queue* q, const rs_engine_trace* tr, const int32_t* req_dev,
                               int32_t k, int64_t n_alive, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(q && tr && (k == 0 || req_dev), "rs_engine_admit: NULL argument");
    RS_CHECK_ARG(k >= 0 && n_alive >= 0, "rs_engine_admit: negative count");
    if (k == 0) return RS_OK;
    engine_admit_kernel<<<(k + EX_THREADS - 1) / EX_THREADS, EX_THREADS, 0, as_stream(stream)>>>(*q, *tr, req_dev, k,
                                                                                              n_alive);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" int rs_engine_execute_ex(const rs_engine_queue* q, const rs_engine_queue* q_out,
                                    const rs_engine_trace* tr, const rs_engine_cost* cost, const int64_t* run_dev,
                                    const int32_t* counts_dev, int32_t step, int64_t predictor_ns, int64_t* out_dev,
                                    int64_t* preempted_dev, int64_t* finished_dev, int32_t* scratch_dev,
                                    int64_t* prev_run_dev, int32_t* prev_n_dev, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(q && tr && cost && run_dev && counts_dev && out_dev && preempted_dev && finished_dev,
                 "rs_engine_execute: NULL argument");
    RS_CHECK_ARG(cost->decode_table_len == 0 || cost->decode_table != nullptr, "rs_engine_execute: decode table");
    RS_CHECK_ARG(q_out == nullptr || (scratch_dev != nullptr && q_out->score_dtype == q->score_dtype),
                 "rs_engine_execute_ex: out-of-place compaction needs scratch and a matching q_out");
    RS_CHECK_ARG((prev_run_dev == nullptr) == (prev_n_dev == nullptr), "rs_engine_execute_ex: prev_run / prev_n");
    cudaStream_t st = as_stream(stream);
    if (q_out == nullptr) {
        engine_execute_kernel<true><<<1, EX_THREADS, 0, st>>>(*q, *tr, *cost, run_dev, counts_dev, step, predictor_ns,
                                                               out_dev, preempted_dev, finished_dev, prev_run_dev,
                                                               prev_n_dev);
        RS_LAUNCH_CHECK();
        return RS_OK;
    }
    engine_execute_kernel<false><<<1, EX_THREADS, 0, st>>>(*q, *tr, *cost, run_dev, counts_dev, step, predictor_ns,
                                                            out_dev, preempted_dev, finished_dev, prev_run_dev,
                                                            prev_n_dev);
    RS_LAUNCH_CHECK();
    const int64_t nb64 = (q->n + EX_THREADS - 1) / EX_THREADS;
    const unsigned nb = nb64 > 0 ? (unsigned)nb64 : 1u;
    engine_compact_count<<<nb, EX_THREADS, 0, st>>>(q->flags, q->n, scratch_dev);
    RS_LAUNCH_CHECK();
    engine_compact_scatter<<<nb, EX_THREADS, 0, st>>>(*q, *q_out, *tr, scratch_dev, out_dev);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" int rs_engine_execute(const rs_engine_queue* q, const rs_engine_trace* tr, const rs_engine_cost* cost,
                                 const int64_t* run_dev, const int32_t* counts_dev, int32_t step,
                                 int64_t predictor_ns, int64_t* out_dev, int64_t* preempted_dev,
                                 int64_t* finished_dev, void* stream) {
    RS_NVTX();
    return rs_engine_execute_ex(q, nullptr, tr, cost, run_dev, counts_dev, step, predictor_ns, out_dev, preempted_dev,
                                finished_dev, nullptr, nullptr, nullptr, stream);
}

// ---- the engine loop itself, natively (record-free runs) ------------------------------
// engine.py:382-460 as DeviceEngine.run drives it from Python, step for step: idle jump,
// admission of the arrivals up to `now` (dropping requests whose full context can never
// fit the KV budget), rank step, execute with out-of-place compaction into the other
// column set, one 64-byte status read-back per step. The C++ loop saves the Python
// interpreter's share of every step; the decisions are identical by construction (same
// kernels, same order), which tests/test_gpu_engine.py checks against the reference.
extern "C" int rs_engine_run(const rs_engine_queue* q2, const rs_queue_soa* soa2, const rs_engine_trace* tr,
                             const rs_engine_cost* cost, const rs_engine_loop* lp, rs_engine_loop_out* res,
                             void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(q2 && soa2 && tr && cost && lp && res, "rs_engine_run: NULL argument");
    RS_CHECK_ARG(lp->arrival_ns && lp->fits && lp->adm_host && lp->adm_dev && lp->stat_dev && lp->stat_host &&
                     lp->run_dev && lp->prom_dev && lp->dem_dev && lp->pre_dev && lp->fin_dev && lp->scratch_dev &&
                     lp->dropped_host,
                 "rs_engine_run: NULL buffer");
    cudaStream_t st = as_stream(stream);
    rs_engine_queue q[2] = {q2[0], q2[1]};
    rs_queue_soa soa[2] = {soa2[0], soa2[1]};
    int64_t* out = lp->stat_dev;                                    // int64[6]
    int32_t* counts = reinterpret_cast<int32_t*>(lp->stat_dev + 6);  // int32[4]
    const int64_t* hout = lp->stat_host;
    const int32_t* hcnt = reinterpret_cast<const int32_t*>(lp->stat_host + 6);
    const int64_t n = lp->n_requests;
    int64_t now = 0, nxt = 0, n_alive = 0, step = 0, n_fin = 0, n_drop = 0, dev_now = -1;
    int64_t tot_prefill = 0, tot_decode = 0, tot_pred = 0;
    bool have_dev_now = false;
    int cur = 0;
    int status = RS_OK;
    while (true) {
        if (n_alive == 0 && nxt < n && lp->arrival_ns[nxt] > now) now = lp->arrival_ns[nxt];  // jump_if_idle
        int64_t end = nxt;
        while (end < n && lp->arrival_ns[end] <= now) ++end;
        int32_t k = 0;
        for (int64_t i = nxt; i < end; ++i) {
            if (lp->fits[i])
                lp->adm_host[k++] = (int32_t)i;
            else
                lp->dropped_host[n_drop++] = i;
        }
        nxt = end;
        if (k) {
            RS_CUDA(cudaMemcpyAsync(lp->adm_dev, lp->adm_host, (size_t)k * sizeof(int32_t), cudaMemcpyHostToDevice, st));
            q[cur].n = n_alive;
            RS_TRY(rs_engine_admit(&q[cur], tr, lp->adm_dev, k, n_alive, st));
            n_alive += k;
        }
        if (n_alive == 0) break;
        if (lp->limit_ns >= 0 && now >= lp->limit_ns) break;
        const int64_t pred = (int64_t)k * lp->predictor_ns_per_request;
        soa[cur].n = n_alive;
        RS_TRY(rs_rank_step(&soa[cur], lp->max_batch, lp->kv_budget, lp->starvation_threshold, lp->priority_quantum,
                            lp->length_calibrated, lp->preemptive, lp->run_dev, lp->prom_dev, lp->dem_dev, counts,
                            lp->ws, lp->ws_bytes, st));
        if (!have_dev_now || now != dev_now) {  // the clock moved on the host (idle jump / first step)
            lp->stat_host[0] = now;
            RS_CUDA(cudaMemcpyAsync(out, lp->stat_host, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        }
        q[cur].n = n_alive;
        RS_TRY(rs_engine_execute_ex(&q[cur], &q[1 - cur], tr, cost, lp->run_dev, counts, (int32_t)step, pred, out,
                                    lp->pre_dev, lp->fin_dev, lp->scratch_dev, lp->prev_run_dev, lp->prev_n_dev, st));
        cur = 1 - cur;
        RS_CUDA(cudaMemcpyAsync(lp->stat_host, lp->stat_dev, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        RS_CUDA(cudaStreamSynchronize(st));
        if (hcnt[3]) {
            set_error("ranking policy: NaN effective score");
            status = RS_ERR_NAN;
            break;
        }
        const int64_t iter = hout[1], prefill = hout[2];
        now = hout[0];
        n_alive = hout[3];
        dev_now = now;
        have_dev_now = true;
        n_fin += hout[5];
        tot_prefill += prefill;
        tot_pred += pred;
        tot_decode += iter - prefill - pred;
        ++step;
        if (lp->stop_after_finished >= 0 && n_fin >= lp->stop_after_finished) break;
        if (lp->limit_ns >= 0 && now >= lp->limit_ns) break;
    }
    res->now_ns = now;
    res->steps = step;
    res->n_finished = n_fin;
    res->next_arrival = nxt;
    res->n_dropped = n_drop;
    res->total_prefill_ns = tot_prefill;
    res->total_decode_ns = tot_decode;
    res->total_predictor_ns = tot_pred;
    res->final_set = cur;
    return status;
}
