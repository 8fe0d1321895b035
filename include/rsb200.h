/*
 * rsb200.h — C ABI of the B200-native learning-to-rank scheduler hot path.
 *
 * One shared library (librsb200.so, built for sm_100a) exports these entry points.
 * Every pointer argument named *_dev is a device pointer owned by the caller; every
 * call is stream-ordered on `stream` (a cudaStream_t passed as void*, NULL = legacy
 * default stream) and returns RS_OK or a negative status. rs_last_error() returns a
 * thread-local message for the last failing call. No torch / C++ types cross this
 * boundary.
 *
 * The reference (`ranksched` 0.1.0, pure Python + numpy) has no FFI; the functions
 * below replace the bodies of its Python entry points, which the host package
 * `paper_2408_15792_b200` re-exposes with the reference signatures:
 *
 *   rs_tau_counts          <- ranking.kendall_tau_b          ranking.py:24-63
 *   rs_listmle_order       <- ranking.list_mle_loss/gradient ranking.py:71-120
 *   rs_listmle_lengths     <- train_ranking inner step       predictors.py:379-384
 *                             (bucket_lengths ranking.py:123-132 + stable argsort +
 *                              loss/n + grad/n)
 *   rs_arrival_rank        <- the (arrival_time, id) tail of RankingPolicy.sort_key
 *                             schedulers.py:211-218
 *   rs_rank_step           <- RankingPolicy.schedule + Policy.schedule/_fill
 *                             schedulers.py:86-109, 203-240
 *   rs_ranker_forward      <- RankingModelScorer.raw_outputs predictors.py:245-247
 *                             (the OPT-125M-shape backbone of PAPER.md:195-201 that
 *                              replaces _Net.forward predictors.py:190-196)
 *   rs_ranker_* (training) <- _Net.backward / _Adam.step     predictors.py:198-225
 *   rs_linear_* / rs_standard* <- the reference's own linear / MLP ranker
 *                             (_Standardizer, _Net, train_ranking step, _Adam)
 *                             predictors.py:159-225, 374-386 (cfg1 parity bridge)
 */
#ifndef RSB200_H
#define RSB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---- status codes ------------------------------------------------------------ */
#define RS_OK 0
#define RS_ERR_INVALID (-1)          /* bad argument (shape, dtype, size)  -> ValueError  */
#define RS_ERR_CUDA (-2)             /* CUDA runtime / launch failure       -> RuntimeError */
#define RS_ERR_NAN (-3)              /* NaN in an ordering key              -> ValueError  */
#define RS_ERR_NOT_PERMUTATION (-4)  /* true_order is not a permutation     -> ValueError  */
#define RS_ERR_WORKSPACE (-5)        /* workspace too small                 -> ValueError  */
#define RS_ERR_UNSUPPORTED (-6)      /* feature not built / device mismatch -> RuntimeError */

/* ---- dtypes ------------------------------------------------------------------ */
#define RS_F32 0
#define RS_F64 1
#define RS_I32 2
#define RS_I64 3
#define RS_BF16 4

const char* rs_last_error(void);
int rs_version(void);
/* Number of SMs / compute capability of `device`; also resolves the driver entry
 * point used to encode TMA descriptors. Must be called once per device before the
 * ranker entry points (the Python wrapper does this). */
int rs_device_init(int device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---- K10: exact Kendall tau-b pair counts (ranking.py:24-63) -----------------
 * x, y: n values each of dtype RS_F32/RS_F64/RS_I32/RS_I64 (compared as float64,
 * exactly like `np.asarray(x, dtype=np.float64)`, -0.0 == +0.0). NaN -> RS_ERR_NAN.
 * counts_dev: int64[6] on device = {concordant, discordant, n1 (x-tied pairs),
 * n2 (y-tied pairs), n3 (pairs tied in both), status (1 if any NaN was seen; the
 * counts are then meaningless)}. tau is finished on the host with the reference
 * expression (ranking.py:60-63).
 * rs_tau_counts runs the bucket fast path (y images spanning < 4096 values) and reads
 * its status back once (one stream synchronisation; none while the stream is being
 * captured), running the general merge-sort path when the fast one does not apply.
 * rs_tau_counts_fast runs the fast path only and never synchronises (graph
 * capturable): status 2 = these inputs need rs_tau_counts. */
size_t rs_tau_workspace_size(int64_t n, int x_dtype, int y_dtype);
int rs_tau_counts(const void* x_dev, int x_dtype, const void* y_dev, int y_dtype, int64_t n,
                  int64_t* counts_dev, void* ws_dev, size_t ws_bytes, void* stream);
int rs_tau_counts_fast(const void* x_dev, int x_dtype, const void* y_dev, int y_dtype, int64_t n,
                       int64_t* counts_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* ---- K6: ListMLE ------------------------------------------------------------
 * rs_listmle_order: n_lists independent lists of length list_len, scores (RS_F32 or
 * RS_F64) and an int64 permutation `order` per list (best first, ranking.py:86-120).
 * loss_dev[n_lists] and grad_dev[n_lists*list_len] are written in the scores dtype.
 * bad_dev (int32, device) is set to 1 if any `order` row is not a permutation; the
 * call itself still returns RS_OK (the wrapper checks the flag and raises). */
int rs_listmle_order(const void* scores_dev, int dtype, const int64_t* order_dev,
                     int32_t n_lists, int32_t list_len, void* loss_dev, void* grad_dev,
                     int32_t* bad_dev, void* stream);
/* rs_listmle_lengths: the training form (predictors.py:379-384). g = net outputs
 * (higher = shorter) f32 [n_lists*list_len]; lengths int32 true output lengths;
 * the target order is argsort(lengths // bucket_width, stable) per list. Writes
 * loss_dev[n_lists] = list_mle_loss/list_len and dg_dev = list_mle_gradient/list_len. */
int rs_listmle_lengths(const float* g_dev, const int32_t* lengths_dev, int32_t n_lists,
                       int32_t list_len, int32_t bucket_width, float* loss_dev, float* dg_dev,
                       void* stream);

/* ---- K9: one ranking-policy scheduling step ----------------------------------
 * The queue is an SoA of the Request runtime fields the policy reads and writes
 * (workload.py:40-61). Row order = candidate order (the order the reference's
 * `candidates` list has; promoted/demoted come out in this order). */
#define RS_FLAG_SCORED 1u
#define RS_FLAG_PRIORITY 2u
#define RS_FLAG_RUNNING 4u
typedef struct rs_queue_soa {
    int64_t n;
    int32_t score_dtype;          /* RS_F32 or RS_F64 */
    const void* score;            /* valid where flags & RS_FLAG_SCORED */
    const int32_t* prompt_tokens;
    const int32_t* generated_tokens;
    const uint32_t* arrival_rank; /* position in (arrival_time, id) order; see rs_arrival_rank */
    const int64_t* id;
    uint8_t* flags;               /* in/out (priority bit is written) */
    int32_t* starvation;          /* in/out */
    int32_t* quantum;             /* in/out */
} rs_queue_soa;

/* arrival_rank[i] = rank of (arrival_time[i], id[i]) in ascending tuple order. */
size_t rs_arrival_rank_workspace_size(int64_t n);
int rs_arrival_rank(const double* arrival_dev, const int64_t* id_dev, int64_t n,
                    uint32_t* rank_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* Writes run ids in fill order, promoted / demoted ids in candidate order, and
 * counts_dev int32[4] = {n_run, n_promoted, n_demoted, nan} (nan = 1 if an effective
 * score was NaN; the wrapper raises ValueError and the state must be discarded). run_dev needs max_batch
 * slots, promoted_dev / demoted_dev need n slots. kv_budget < 0 means unlimited.
 * preemptive = policy.preemptive && config.preemption (schedulers.py:100). */
size_t rs_rank_step_workspace_size(int64_t n);
int rs_rank_step(const rs_queue_soa* q, int32_t max_batch, int64_t kv_budget,
                 int32_t starvation_threshold, int32_t priority_quantum, int32_t length_calibrated,
                 int32_t preemptive, int64_t* run_dev, int64_t* promoted_dev, int64_t* demoted_dev,
                 int32_t* counts_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* ---- §8f #1: device-resident engine step (the caller of the hot path) ------------
 * The reference loop (engine.run, engine.py:382-460) with its queue resident in HBM:
 * rs_engine_admit appends newly arrived requests to the queue (engine.py:218-243),
 * rs_rank_step schedules, rs_engine_execute runs _Sim.execute (engine.py:247-284):
 * preemption, prefill / decode / predictor time, one token per scheduled request with
 * the _ReqTrack bookkeeping (engine.py:108-125), retirement and a stable compaction of
 * the queue. Requests are referred to by their index r in the trace (queue id = r). */
typedef struct rs_engine_queue {   /* all columns writable; n = alive rows */
    int64_t n;
    int32_t score_dtype;           /* RS_F32 or RS_F64 */
    void* score;
    int32_t* prompt_tokens;
    int32_t* generated_tokens;
    uint32_t* arrival_rank;
    int64_t* id;
    uint8_t* flags;
    int32_t* starvation;
    int32_t* quantum;
} rs_engine_queue;
typedef struct rs_engine_trace {   /* per request r of the trace */
    const void* score;             /* the score cache (same dtype as the queue's) */
    const int32_t* prompt_tokens;
    const int32_t* true_output;
    const uint32_t* arrival_rank;  /* position in (arrival_time, id) order */
    const int64_t* arrival_ns;
    int32_t* row_of;               /* queue row while alive */
    int32_t* run_stamp;            /* init -1 */
    int64_t* first_token_ns;       /* init -1 */
    int64_t* last_event_ns;
    int64_t* max_gap_ns;           /* init 0 */
    int64_t* finish_ns;            /* init -1 */
    int32_t* n_preempted;          /* init 0 */
} rs_engine_trace;
typedef struct rs_engine_cost {    /* CostModel (engine.py:42-78) */
    int64_t decode_ns;
    int64_t prefill_ns_per_token;
    const int64_t* decode_table;   /* device, may be NULL */
    int32_t decode_table_len;
} rs_engine_cost;
int rs_engine_admit(const rs_engine_queue* q, const rs_engine_trace* tr, const int32_t* req_dev, int32_t k,
                    int64_t n_alive, void* stream);
/* out_dev int64[6] = {now_ns (in/out), iter_ns, prefill_ns, n_alive after, n_preempted, n_finished};
 * preempted_dev (alive order, >= n slots), finished_dev (fill order, >= max_batch slots).
 * run_dev / counts_dev are rs_rank_step's run ids and counts; step must differ per call. */
int rs_engine_execute(const rs_engine_queue* q, const rs_engine_trace* tr, const rs_engine_cost* cost,
                      const int64_t* run_dev, const int32_t* counts_dev, int32_t step, int64_t predictor_ns,
                      int64_t* out_dev, int64_t* preempted_dev, int64_t* finished_dev, void* stream);
/* Same step with the surviving rows compacted out of place into q_out's columns (same
 * capacity and score dtype; q_out->n is ignored) by many CTAs instead of in place by one —
 * the caller swaps the two column sets every step. scratch_dev: int32[ceil(n / 1024)].
 * prev_run_dev (int64[>= max_batch]) / prev_n_dev (int32[1], 0 before the first step), both
 * or neither: the previous step's batch, kept by the call, so preemption only looks at
 * those rows instead of scanning the queue. q_out == NULL is in-place compaction. */
int rs_engine_execute_ex(const rs_engine_queue* q, const rs_engine_queue* q_out, const rs_engine_trace* tr,
                         const rs_engine_cost* cost, const int64_t* run_dev, const int32_t* counts_dev, int32_t step,
                         int64_t predictor_ns, int64_t* out_dev, int64_t* preempted_dev, int64_t* finished_dev,
                         int32_t* scratch_dev, int64_t* prev_run_dev, int32_t* prev_n_dev, void* stream);
/* The whole engine loop natively (engine.py:382-460; records are not produced — use the
 * per-step calls for that): q2 / soa2 = the two column sets (views of the same columns),
 * starting in set 0 with no alive rows. Host arrays: arrival_ns[n] (sorted), fits[n]
 * (uint8: prompt + true output <= KV budget), adm_host int32[n] (pinned), dropped_host
 * int64[n] (receives the dropped request indices). Device: adm_dev int32[n], stat_dev
 * int64[8] (out[6] | counts int32[4]) with its pinned host mirror stat_host, the
 * rank-step / execute outputs and workspace sized for n rows. limit_ns / stop_after <
 * 0: none. Returns RS_ERR_NAN on a NaN effective score.
 * With an unlimited KV budget, max_batch <= 512 and 16-B aligned columns the whole loop
 * is ONE launch (a thread-block cluster stepping the queue on the device; finished rows
 * are compacted out lazily, so final_set / the queue columns at return hold the alive
 * rows among finished ones, and the last step's state update is applied); otherwise the
 * host steps the per-kernel calls. RS_ENGINE_LOOP=host forces the latter. Both give the
 * same per-request results. */
typedef struct rs_engine_loop {
    int64_t n_requests;
    const int64_t* arrival_ns;
    const uint8_t* fits;
    int32_t* adm_host;
    int32_t* adm_dev;
    int64_t* dropped_host;
    int64_t* stat_dev;
    int64_t* stat_host;
    int64_t* run_dev;
    int64_t* prom_dev;
    int64_t* dem_dev;
    int64_t* pre_dev;
    int64_t* fin_dev;
    int32_t* scratch_dev;
    int64_t* prev_run_dev;  /* int64[max_batch], prev_n_dev int32[1] = 0: see rs_engine_execute_ex */
    int32_t* prev_n_dev;
    void* ws;
    size_t ws_bytes;
    int32_t max_batch, starvation_threshold, priority_quantum, length_calibrated, preemptive;
    int64_t kv_budget;                 /* < 0: unlimited */
    int64_t predictor_ns_per_request;  /* 0 when the scorer is not charged */
    int64_t limit_ns;
    int64_t stop_after_finished;
} rs_engine_loop;
typedef struct rs_engine_loop_out {
    int64_t now_ns, steps, n_finished, next_arrival, n_dropped;
    int64_t total_prefill_ns, total_decode_ns, total_predictor_ns;
    int32_t final_set;
} rs_engine_loop_out;
int rs_engine_run(const rs_engine_queue* q2, const rs_queue_soa* soa2, const rs_engine_trace* tr,
                  const rs_engine_cost* cost, const rs_engine_loop* loop, rs_engine_loop_out* out, void* stream);

/* ---- §8f #2: prompt strings -> token ids on the device ---------------------------
 * The scorer's id map (workload.prompt_token_ids; the reference's salted crc32 token
 * hash, workload.py:125-126): whitespace tokens, the first min(seq_len, 2048), lower-cased,
 * id = 4 + crc32(salt + token) % (vocab - 4), padded with pad_id; empty prompt -> {2}.
 * text_dev: the prompts' UTF-8 bytes back to back; offsets_dev int64[n + 1]; salt_crc =
 * crc32(salt). ids_dev int32[n, seq_len], last_dev int32[n] (last token index), bad_dev
 * int32[n] = 1 for a prompt whose result depends on non-ASCII bytes (str.split / lower
 * are Unicode-aware): the caller must reject it. */
int rs_tokenize(const uint8_t* text_dev, const int64_t* offsets_dev, int32_t n, int32_t seq_len, int32_t vocab,
                int32_t pad_id, uint32_t salt_crc, int32_t* ids_dev, int32_t* last_dev, int32_t* bad_dev,
                void* stream);

/* ---- A5/K1-K5: OPT-shape ranker ------------------------------------------------
 * Parameters live in ONE contiguous bf16 buffer laid out by rs_ranker_layout():
 *   tok_emb[V,d] pos_emb[P+2,d] { ln1_w[d] ln1_b[d] qkv_w[3d,d] qkv_b[3d] out_w[d,d]
 *   out_b[d] ln2_w[d] ln2_b[d] fc1_w[F,d] fc1_b[F] fc2_w[d,F] fc2_b[d] } x L
 *   lnf_w[d] lnf_b[d] head_w[d] head_b[1]
 * every tensor starting on a 64-element (128-byte) boundary. Weights are [out, in]
 * row-major (torch nn.Linear layout). */
typedef struct rs_ranker_config {
    int32_t vocab;      /* 50272 */
    int32_t max_pos;    /* 2048 (the table has max_pos + 2 rows, OPT offset 2) */
    int32_t d_model;    /* 768 */
    int32_t n_layers;   /* 12 */
    int32_t n_heads;    /* 12 (head dim must be 64) */
    int32_t d_ffn;      /* 3072 */
    int32_t activation; /* 0 = ReLU (OPT), 1 = GELU(tanh) */
} rs_ranker_config;

#define RS_RANKER_N_GLOBAL 6  /* tok_emb pos_emb lnf_w lnf_b head_w head_b */
#define RS_RANKER_N_PER_LAYER 12
/* offsets (in bf16 elements) of every tensor in the order listed above (global ones
 * first: tok, pos, lnf_w, lnf_b, head_w, head_b; then per layer in the order above);
 * returns the total element count (padded). offsets may be NULL. */
int64_t rs_ranker_layout(const rs_ranker_config* cfg, int64_t* offsets);

/* Scores B prompts of S token ids (int32 [B,S], row-major). last_pos_dev (int32[B],
 * may be NULL = S-1) is the index of each prompt's last real token. g_dev f32[B] =
 * head(LN_f(h[last_pos])) — the net output; score_dev (f32[B], may be NULL) receives
 * -g, the scheduler score (predictors.py:249-250). The residual stream is fp32, the
 * GEMM operands bf16. */
size_t rs_ranker_workspace_size(const rs_ranker_config* cfg, int32_t B, int32_t S);
int rs_ranker_forward(const rs_ranker_config* cfg, const void* params_dev, const int32_t* ids_dev,
                      const int32_t* last_pos_dev, int32_t B, int32_t S, float* g_dev, float* score_dev,
                      void* ws_dev, size_t ws_bytes, void* stream);
/* Same forward, also writing feat_dev f32[B, d] = LN_f(h[last_pos]) (may be NULL): the
 * input of the classification head (§8f #4). */
int rs_ranker_forward_ex(const rs_ranker_config* cfg, const void* params_dev, const int32_t* ids_dev,
                         const int32_t* last_pos_dev, int32_t B, int32_t S, float* g_dev, float* score_dev,
                         float* feat_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* ---- §8f #4: bucketed-classification baseline on the same backbone ------------------
 * The reference's ClassifierScorer / train_classifier (predictors.py:262-300, :409-479):
 * logits = feat W^T + b over C length buckets, softmax cross-entropy. Here the features
 * are the OPT backbone's LN_f(h_last) instead of the 24 hashed prompt features.
 * rs_cls_logits: feat f32[B,d], W f32[C,d], b f32[C] -> logits f32[B,C].
 * rs_cls_ce: per-prompt nll f32[B] and dlogits = softmax - onehot(label) f32[B,C]
 *   (labels int32[B] in [0, C); out of range -> RS_ERR_INVALID via bad_dev != 0).
 * rs_ranker_grad_cls: like rs_ranker_grad, with the CE stage in place of ListMLE:
 *   accumulates d(sum of nll)/d params into grad (the backbone, rs_ranker_layout; the
 *   score head gets none) and into cls_grad f32[C*d + C] (dW then db); loss_out f32[n]
 *   per-prompt nll; prompts_per_micro prompts per micro-batch. Scale by 1/n in Adam. */
int rs_cls_logits(const float* feat_dev, const float* w_dev, const float* b_dev, int32_t B, int32_t d, int32_t C,
                  float* logits_dev, void* stream);
int rs_cls_ce(const float* logits_dev, const int32_t* labels_dev, int32_t B, int32_t C, float* loss_dev,
              float* dlogits_dev, int32_t* bad_dev, void* stream);
size_t rs_ranker_grad_cls_workspace_size(const rs_ranker_config* cfg, int32_t prompts_per_micro, int32_t S,
                                         int32_t n_classes);
int rs_ranker_grad_cls(const rs_ranker_config* cfg, const void* params_dev, float* grad_dev, const int32_t* ids_dev,
                       const int32_t* last_pos_dev, const int32_t* labels_dev, int32_t n_prompts, int32_t S,
                       int32_t n_classes, const float* cls_w_dev, const float* cls_b_dev, float* cls_grad_dev,
                       int32_t prompts_per_micro, float* loss_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* ---- A10/K7/K8: training (ListMLE over whole lists, predictors.py:347-406) ----------
 * Accumulates into grad_dev (fp32, rs_ranker_layout order and length) the gradient of
 * sum over lists of list_mle_loss(g_list, order_list) / list_len, where g = the ranker's
 * net output for the list's prompts (read at last_pos, like rs_ranker_forward; NULL =
 * S-1) and order_list = stable argsort of lengths // bucket_width (predictors.py:379-384).
 * ids: int32 [n_lists * list_len, S] (S <= 128); lengths: int32 [n_lists * list_len];
 * loss_dev[n_lists] = per-list loss / n. Processes lists_per_micro lists at a time.
 * Deterministic (no float atomics). */
size_t rs_ranker_grad_workspace_size(const rs_ranker_config* cfg, int32_t lists_per_micro, int32_t list_len, int32_t S);
int rs_ranker_grad(const rs_ranker_config* cfg, const void* params_dev, float* grad_dev, const int32_t* ids_dev,
                   const int32_t* last_pos_dev, const int32_t* lengths_dev, int32_t n_lists, int32_t list_len,
                   int32_t S, int32_t bucket_width, int32_t lists_per_micro, float* loss_dev, void* ws_dev,
                   size_t ws_bytes, void* stream);
/* Adam (predictors.py:218-225) over the flat buffer: g = grad * grad_scale; m, v, fp32
 * master updated with bias correction at step t (>= 1); the bf16 working copy is
 * rewritten and grad is zeroed for the next accumulation. */
int rs_adam_step(float* master_dev, float* m_dev, float* v_dev, float* grad_dev, void* params_bf16_dev, int64_t n,
                 float lr, float beta1, float beta2, float eps, int64_t t, float grad_scale, void* stream);

/* ---- building blocks exported for parity tests ---------------------------------
 * C[M,N] (row-major) = epi(A[M,K] . W[N,K]^T + bias[N]) with A/W bf16 K-major.
 * epi: 0 = none, 1 = ReLU, 3 = GELU(tanh) -> C bf16; 2 = + residual R[M,N] -> C, R
 * fp32 (C may alias R: the residual stream is updated in place); 7 = as 0 with the last
 * third of the columns (v of a fused q|k|v projection) written as fp16 (M % 256 == 0).
 * M % 128 == 0, N % 64 == 0, K % 64 == 0 (the ranker's shapes). tcgen05 + TMA. */
int rs_gemm_bf16(const void* A_dev, const void* W_dev, const void* bias_dev, const void* R_dev,
                 void* C_dev, int32_t M, int32_t N, int32_t K, int32_t epi, void* stream);
/* Causal multi-head attention over packed qkv [B*S, 3*H*64] bf16 -> out [B*S, H*64] bf16.
 * rs_attention_fwd_f16v: the same with the v block of qkv in fp16 (the layout the
 * ranker forward's QKV GEMM writes); P is then fp16 as well. */
int rs_attention_fwd(const void* qkv_dev, void* out_dev, int32_t B, int32_t S, int32_t H,
                     void* stream);
int rs_attention_fwd_f16v(const void* qkv_dev, void* out_dev, int32_t B, int32_t S, int32_t H,
                          void* stream);
/* rs_attention_fwd that also writes each row's log2-sum-exp of the scaled scores,
 * lse_dev[(b * H + h) * S + row] (fp32; P = 2^(s / 8 * log2 e - lse)) for
 * rs_attention_bwd_lse (the ranker's training forward). */
int rs_attention_fwd_lse(const void* qkv_dev, void* out_dev, float* lse_dev, int32_t B, int32_t S, int32_t H,
                         void* stream);
/* General CTA-pair GEMM used by the backward pass: a_mn / b_mn = operand stored
 * MN-contiguous ([K, M] / [K, N]); epi 4 = fp32 out, 5 = bf16 out * (aux > 0) (ReLU
 * backward, aux bf16 [M, N]), 6 = fp32 split-K partials (C holds k_splits x [M, N]).
 * M, N multiples of 256, K of 64. bias may be NULL for epi >= 4. */
int rs_gemm_bf16_ex(const void* A_dev, const void* W_dev, const void* bias_dev, const void* aux_dev, void* C_dev,
                    int32_t M, int32_t N, int32_t K, int32_t epi, int32_t a_mn, int32_t b_mn, int32_t k_splits,
                    void* stream);
/* Causal attention backward for S <= 128: dqkv [B*S, 3*H*64] bf16 from the forward's
 * qkv, its output att [B*S, H*64] and dout = d loss / d att. */
int rs_attention_bwd(const void* qkv_dev, const void* att_dev, const void* dout_dev, void* dqkv_dev, int32_t B,
                     int32_t S, int32_t H, void* stream);
/* The same given the forward's lse (rs_attention_fwd_lse): P in one pass, no row max /
 * sum recompute (S <= 128). */
int rs_attention_bwd_lse(const void* qkv_dev, const void* att_dev, const void* dout_dev, const float* lse_dev,
                         void* dqkv_dev, int32_t B, int32_t S, int32_t H, void* stream);
/* Causal attention backward for 128 < S <= 512 (128-token blocks: a dQ kernel that also
 * writes each row's log-sum-exp and rowsum(dO * O) into the workspace, then a dK / dV
 * kernel); same layouts as rs_attention_bwd. */
size_t rs_attention_bwd_long_workspace_size(int32_t B, int32_t S, int32_t H);
int rs_attention_bwd_long(const void* qkv_dev, const void* att_dev, const void* dout_dev, void* dqkv_dev,
                          int32_t B, int32_t S, int32_t H, void* ws_dev, size_t ws_bytes, void* stream);
/* The same given the forward's lse (rs_attention_fwd_lse, [b, h, row]): the dQ kernel
 * skips its row-statistics pass (the ranker's training backward for S > 128). */
int rs_attention_bwd_long_lse(const void* qkv_dev, const void* att_dev, const void* dout_dev, const float* lse_dev,
                              void* dqkv_dev, int32_t B, int32_t S, int32_t H, void* ws_dev, size_t ws_bytes,
                              void* stream);
/* Number of kernels this library has launched in the process (all entry points). */
uint64_t rs_launch_count(void);

/* ---- linear / MLP ranker over the 24 prompt features (the cfg1 parity bridge) ------
 * Replaces _Standardizer.fit / __call__ (predictors.py:159-172), _Net.forward / backward
 * (predictors.py:175-206), one train_ranking minibatch step (predictors.py:374-386) and
 * _Adam.step (predictors.py:209-225). float64 throughout. params = the reference's
 * params list flattened: hidden == 0 -> [w (D), b]; hidden > 0 -> [W1 (D x H row-major),
 * b1 (H), w2 (H), b2]. */
int64_t rs_linear_n_params(int32_t n_features, int32_t hidden);
int rs_standardizer_fit(const double* X_dev, int64_t n_rows, int32_t n_features, double* mean_dev,
                        double* std_dev, void* stream);
int rs_standardize(const double* X_dev, int64_t n_rows, int32_t n_features, const double* mean_dev,
                   const double* std_dev, double* out_dev, void* stream);
/* out[r] = net((X[r] - mean) / std) */
int rs_linear_forward(const double* X_dev, int64_t n_rows, int32_t n_features, const double* mean_dev,
                      const double* std_dev, int32_t hidden, const double* params_dev, double* out_dev,
                      void* stream);
/* One list: Xb = Xs[batch] (Xs already standardised), order = stable argsort(lengths[batch]
 * // width), loss = ListMLE / n -> loss_dev[0], grads of (ListMLE / n) -> grad_dev
 * (optional), Adam step t on params / m / v in place. n >= 2. */
int rs_linear_train_step(const double* Xs_dev, const int64_t* batch_dev, const int64_t* lengths_dev, int32_t n,
                         int32_t n_features, int32_t hidden, int32_t bucket_width, double* params_dev,
                         double* adam_m_dev, double* adam_v_dev, double lr, double beta1, double beta2, double eps,
                         int64_t t, double* loss_dev, double* grad_dev, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RSB200_H */
