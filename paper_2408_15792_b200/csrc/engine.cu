// Device-resident engine step (the caller of the hot path):
// admission into the resident queue and the reference's `_Sim.execute`
// (engine.py:247-284) — preempt running requests left out of the batch, charge prefill
// for the ones (re)starting, advance the clock by prefill + decode + predictor time,
// emit one token per scheduled request (`_ReqTrack.on_token`, engine.py:108-125), retire
// finished requests and compact the queue in place (stable, so row order stays the
// `alive` dict's insertion order the ranking policy's promoted / demoted lists follow).
// One CTA: a step touches each alive row a few times (µs of work) and every phase needs
// the previous one complete, so grid-wide synchronisation would cost more than it saves.
#include "engine_exec.cuh"

namespace rs {

__global__ void __launch_bounds__(EX_THREADS) engine_admit_kernel(rs_engine_queue q, rs_engine_trace tr,
                                                                  const int32_t* __restrict__ req, int32_t k,
                                                                  int64_t n_alive) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    engine_admit_row(q, tr, req[i], n_alive + i);
}

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
    __shared__ int pre_rows[EX_PRE_CAP];
    engine_execute_block<InPlace>(q, tr, cost, run, counts, step, predictor_ns, out, preempted, finished, prev_run,
                                  prev_n, pre_rows, warp_tot);
}

// Out-of-place stable compaction (queue q -> q_out) over many CTAs: per-CTA survivor
// counts, then each CTA sums the counts before it (<= n / 1024 of them) and scatters.
__global__ void __launch_bounds__(EX_THREADS) engine_compact_count(const uint8_t* __restrict__ flags, int64_t n,
                                                                   int32_t* __restrict__ block_keep) {
    __shared__ int warp_tot[32];
    const int total = compact_count_chunk(flags, n, blockIdx.x, warp_tot);
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
    __syncthreads();
    const int total = compact_scatter_chunk(q, qo, tr, blockIdx.x, base_s, warp_tot);
    if (blockIdx.x == gridDim.x - 1 && tid == 0) out[3] = base_s + total;
}

}  // namespace rs

namespace rs {
int rs_engine_run_device(const rs_engine_queue* q2, const rs_queue_soa* soa2, const rs_engine_trace* tr,
                         const rs_engine_cost* cost, const rs_engine_loop* lp, rs_engine_loop_out* res,
                         cudaStream_t st, bool* handled);  // rankstep.cu
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
    bool handled = false;
    {
        const int rc = rs_engine_run_device(q2, soa2, tr, cost, lp, res, st, &handled);
        if (handled || rc != RS_OK) return rc;
    }
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
