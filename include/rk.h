/* rk.h — C-ABI of librk.so: B200-native batched ensemble-subset scoring.
 *
 * The data-parallel hot path of Rafiki's online ensemble inference service (Wang et al.,
 * arXiv 1804.06087, §5.2; PAPER.md line numbers cited below):
 *   A1 rk_score            K synthetic dense classifier heads: logit = 2^s * X.W^T + bias
 *                          (stand-in for the ConvNets' classifier layer).
 *   A2                     per-model top-1 and softmax normaliser.
 *   A3 rk_subset_*         majority vote of every model subset v, the action
 *                          space (2^|M|-1)*|B| with v = 0 excluded.
 *   A4                     averaged softmax probabilities of every subset.
 *   A5                     per-subset / per-(subset, batch size) correct counts and batch
 *                          overdue moments.
 *   A6                     sum of the integer table across GPUs (one NCCL all-reduce).
 *   A7                     the reward of eq. `multi_acc_reward`.
 *
 * Conventions (all entry points):
 *  - Every call returns rk_status; RK_OK = 0. On error, rk_last_error(ctx) holds a message.
 *  - The caller owns every input and output buffer. The context owns its copy of the
 *    weights and its device workspaces; rk_destroy frees them.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). Calls are
 *    stream-ordered; rk_subset_finalize / rk_subset_stats synchronise `stream` and return
 *    host results.
 *  - Pointers documented "host or device" are classified with cudaPointerGetAttributes; host
 *    inputs are copied with cudaMemcpyAsync on the call's stream(s), so -- as with cudaMemcpyAsync --
 *    a HOST INPUT MUST STAY VALID AND UNMODIFIED UNTIL `stream` HAS COMPLETED THE CALL'S WORK (e.g. the
 *    next rk_subset_finalize / rk_subset_stats, which synchronise, or a cudaStreamSynchronize).
 *    Page-locked buffers are then read by DMA asynchronously; pageable ones are staged by the driver.
 *  - Subset mask v in [1, 2^K): bit m selects model m. Tables are indexed v-1 (v fastest),
 *    then batch-size index, then rate index: T[r][b][v-1]. RL action index of (v, B[b]) is
 *    (v-1)*nB + b (index 0 <-> (v = 0b001, B[0])).
 *  - Not thread-safe per context; one context per process / GPU rank.
 */
#ifndef RK_H
#define RK_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct rk_ctx rk_ctx;

typedef enum {
  RK_OK = 0,
  RK_EINVAL = 1,      /* bad argument (sizes, NULLs, v == 0, misaligned shard/chunk)      */
  RK_ESTATE = 2,      /* call out of order (e.g. accumulate before score)                  */
  RK_ENOMEM = 3,      /* device or pinned allocation failed                                */
  RK_ECUDA = 4,       /* CUDA runtime/driver error (message in rk_last_error)              */
  RK_ENCCL = 5,       /* NCCL error                                                        */
  RK_ELABEL = 6,      /* a label outside [0, C)                                            */
  RK_ENONFINITE = 7,  /* a NaN or +inf logit, or a row that is entirely -inf               */
  RK_EUNSUPPORTED = 8 /* feature not available in this build (e.g. NCCL for world > 1)     */
} rk_status;

typedef enum {
  RK_TIE_BEST_MEMBER = 0, /* paper: "when there is a tie, the prediction from the
                             model with the best accuracy is selected" -- the best-ranked member
                             among the tied voters (reading Q2)                          */
  RK_TIE_LOWEST_CLASS = 1 /* north_star: lowest class index among the tied classes              */
} rk_tie_mode;

/* Create a context on `cuda_device`. world > 1: every rank passes the same 128-byte
 * ncclUniqueId (from rk_nccl_unique_id on rank 0, broadcast by the caller, e.g. through
 * torch.distributed) and its rank; the table all-reduce (A6) then runs over NCCL (NVLink /
 * NVSwitch). world == 1: nccl_unique_id may be NULL (no communicator); a non-NULL id creates a
 * one-rank communicator and runs the same all-reduce code path (used by the tests). */
rk_status rk_create(rk_ctx** out, int cuda_device, const void* nccl_unique_id, int rank, int world);
/* Fill `out128` with a fresh ncclUniqueId (rank 0 only). */
rk_status rk_nccl_unique_id(void* out128);

/* Load the ensemble M (PAPER.md:337 Table tb:notation "M: model list").
 *  K in [1,12] models (S = 2^K-1 <= 4095 subsets), C in [2,65535] classes (rows wider than 1024
 *  classes are averaged by a slower fp64 kernel, rk_vote_large.cu; no bench config needs it).
 *  W_bf16: [K][C][D] bfloat16 bit patterns, row-major (D contiguous), host or device; NULL
 *          loads a logits-only ensemble (rk_score then returns RK_ESTATE). D % 64 == 0, D <= 16384.
 *  bias:   [K][C] fp32 or NULL (= 0). logit = 2^logit_scale_log2 * sum_d x*w + bias.
 *  member_rank: [K] permutation, 0 = most accurate model (used by RK_TIE_BEST_MEMBER);
 *          NULL = index order (model 0 best). Never estimated inside the library (Q3).
 *  The context copies everything it needs; the caller may free its buffers on return. */
rk_status rk_load_ensemble(rk_ctx* ctx, int K, int C, int D, const void* W_bf16, const float* bias,
                           int logit_scale_log2, const int* member_rank, rk_tie_mode tie);

/* A1+A2: run the K heads on N feature rows. X_bf16: [N][D] bfloat16 bits, host or device.
 * global_offset = index of row 0 in the global request stream (fixes batch ids and arrival
 * times). Produces the context's logits workspace [N][K][ldc] fp32 (ldc = C rounded up to 4),
 * per-(row, model) top-1 and log-sum-exp, fused in the GEMM epilogue. N < 2^31 per call
 * (larger streams go in chunks; RK_EINVAL otherwise). */
rk_status rk_score(rk_ctx* ctx, const void* X_bf16, int64_t N, int64_t global_offset, void* stream);

/* NEXT-3, fused forward + vote: A1+A2 with the labels known at scoring time. Same X / N / offset contract
 * as rk_score; labels: [N] int32 host or device, the values rk_subset_accumulate would receive (it must then
 * be called with the same pointer or NULL). For K <= 8 and more than 128 classes (the GEMM's per-model
 * column tiles), the epilogue does NOT store the fp32 logits: per (row, model) it keeps the row statistics,
 * the label's logit and the 16 largest logits with their classes, from which the vote stage decides every
 * subset's average exactly where the bounds allow; the remaining samples' rows are recomputed with logits
 * (inside rk_subset_accumulate) and averaged by the logits path, so the table is identical to
 * rk_score + rk_subset_accumulate. Other shapes run exactly that path. rk_predict after this call is
 * RK_ESTATE, and rk_outputs returns no logits. Device X must stay valid until rk_subset_accumulate, which
 * for such a batch synchronises `stream` once (it reads the number of recomputed rows to size their GEMM). */
rk_status rk_score_labelled(rk_ctx* ctx, const void* X_bf16, const int32_t* labels, int64_t N, int64_t global_offset,
                            void* stream);

/* Vote-stage entry on caller-provided logits: [N][K][ldc] fp32 DEVICE memory, ldc % 4 == 0,
 * ldc >= C, 16-byte aligned. The pointer is borrowed until the next rk_score* call. */
rk_status rk_score_logits(rk_ctx* ctx, const float* logits, int ldc, int64_t N, int64_t global_offset,
                          void* stream);

/* Reward configuration for A5/A7 (eq. `multi_acc_reward`). */
typedef struct {
  int nB;                  /* 0..8 candidate batch sizes; 0 = counts only  */
  const int* B;            /* [nB] host; lcm(B) <= 4096                                         */
  double beta;             /* balancing factor beta                               */
  int64_t tau_ns;          /* SLO tau in integer ns (strict l(s) > tau) */
  const int64_t* lat_ns;   /* [K][nB] host: c(m, b) in ns                     */
  int nR;                  /* 0..8 arrival rates                                                 */
  const double* rates;     /* [nR] host, req/s: t_s = floor(s * 1e9 / r) ns, s global (Q9)      */
  const int64_t* arrival_ns; /* [N] host or device, non-decreasing, for the last rk_score* call;
                                if non-NULL, nR must be 1 and rates is ignored                   */
  int want_exceed;         /* also accumulate E = sum max(0, l(s) - tau) (eq. `eq:single`)      */
  int want_labelled;       /* also accumulate Q = sum_j corr_j * o_j (labelled reward variant)  */
  int queue;               /* 0: batch j is dispatched when full, l(s) = t_last(j) - t_s + c(v,b)
                              (reading Q8). 1: one ensemble server runs the batches of (v,b) in FIFO
                              order, "the next batch has to wait" (reading Q15):
                              finish_j = max(t_last(j), finish_{j-1}) + c(v,b), l(s) = finish_j - t_s.
                              Chunks must then arrive in global order; a rank whose first chunk
                              starts after sample 0 derives the backlog from `rates` (arrival_ns
                              with a non-zero first offset -> RK_EUNSUPPORTED).                     */
} rk_reward_cfg;

/* Result table (host arrays, caller-allocated; any pointer may be NULL to skip it). */
typedef struct {
  int64_t N;               /* samples accumulated over all chunks and ranks                      */
  uint64_t* cnt_vote;      /* [S] majority-vote correct counts; a(M[v]) = cnt_vote/N */
  uint64_t* cnt_avg;       /* [S] averaged-probability correct counts                            */
  uint64_t* n_recheck;     /* [S] (sample, v) pairs whose fp32 relative top-2 gap was within the band
                              (2e-5) and were decided from the definition in fp64. This is the
                              library's counterpart of SURVEY.md §8(b)'s n_ambiguous_avg, but not
                              the same count: n_ambiguous_avg (the oracle's, any two classes) flags
                              pairs whose fp64 top-2 gap is <= 1e-12, where fp64 itself cannot
                              decide. Here every pair whose decision about the label could flip
                              under fp32 rounding is redone in fp64, so cnt_avg can differ from the
                              exact-arithmetic count only on rechecked pairs:
                              |cnt_avg[v] - exact| <= n_recheck[v], a bound callers get from library
                              output alone (singletons are exact: top-1, invariant I1). The tests
                              hold cnt_avg to the tighter oracle bound n_ambiguous_avg.        */
  uint64_t* corr;          /* [nB][S] vote-correct samples inside complete batches of size B[b]   */
  uint64_t* O;             /* [nR][nB][S] overdue requests sum_j o_j(v,b,r)                      */
  uint64_t* Q;             /* [nR][nB][S] sum_j corr_j(v) * o_j(v,b,r)   (want_labelled)         */
  uint64_t* E;             /* [nR][nB][S] exceed time in ns            (want_exceed)             */
  double* reward_sur;      /* [nR][nB][S] sum over batches of a(v) * (b - beta*o_j)              */
  double* reward_lab;      /* [nR][nB][S] sum over batches of corr_j/b * (b - beta*o_j)          */
} rk_table;

/* Streaming form: reset (zero the table, set cfg; cfg NULL = counts only), then one
 * rk_score* + rk_subset_accumulate per chunk, then finalize. Chunk (and shard) boundaries
 * must be multiples of lcm(B); only the globally last chunk may be ragged. */
rk_status rk_subset_reset(rk_ctx* ctx, const rk_reward_cfg* cfg);
/* A2-A5 on the last rk_score* batch. labels: [N] int32, host or device. */
rk_status rk_subset_accumulate(rk_ctx* ctx, const int32_t* labels, void* stream);
/* A6 (all-reduce when world > 1) + A7 (reward fold) + copy to `out`. Blocks on `stream`. The table and
 * rewards come back through a page-locked host buffer the context allocates on first use (grow-only,
 * freed by rk_destroy; 3.5 MB at K = 12 with 5 batch sizes and 4 rates), then are copied into `out`.
 * Returns RK_ENONFINITE / RK_ELABEL if any accumulated chunk had bad input (table zeroed).
 * The all-reduce runs once per reset: a repeated finalize returns the same global table, and
 * rk_subset_accumulate after a finalize is RK_ESTATE until the next rk_subset_reset. The wait for the
 * all-reduce is bounded: it polls ncclCommGetAsyncError and gives up after RK_NCCL_TIMEOUT_S seconds
 * (environment, read at rk_create; default 600); either failure aborts the communicator and returns
 * RK_ENCCL (the context can no longer all-reduce). */
rk_status rk_subset_finalize(rk_ctx* ctx, rk_table* out, void* stream);
/* One-shot: reset + accumulate + finalize on the last rk_score* batch. */
rk_status rk_subset_stats(rk_ctx* ctx, const int32_t* labels, const rk_reward_cfg* cfg, rk_table* out,
                          void* stream);

/* NEXT-1 serving policy: Algorithm 3 greedy batching of EVERY subset v run as a
 * synchronous ensemble (c(v,b) = max over members of c(m,b)) on N requests whose
 * arrivals are those of cfg (rates, or arrival_ns [N] host/device with nR = 1), per rate and subset
 * (reading S1): when the server is idle at t, infer max B if that many requests wait,
 * else the largest b in B not above the queue length once c(v,b) + w(q0) + delta >= tau; a batch
 * inferred at t completes at t + c(v,b). Uses cfg->B, lat_ns, tau_ns, beta and the arrivals
 * (queue, want_* ignored). acc: [S] host a(v) (e.g. cnt_vote / N from rk_subset_stats) or NULL;
 * reward = a(v) * (served - beta * overdue), eq. `multi_acc_reward` summed over the greedy batches.
 * Output arrays are host [nR][S], each may be NULL. Blocks on `stream`. Needs rk_load_ensemble. */
typedef struct {
  uint64_t* served;        /* requests inferred                                               */
  uint64_t* overdue;       /* requests with l(s) > tau                                        */
  uint64_t* exceed_ns;     /* sum of max(0, l(s) - tau) (eq. `eq:single`)                     */
  uint64_t* batches;       /* batches inferred                                                */
  uint64_t* unserved;      /* requests left in the queue (< min B) after the last arrival     */
  double* reward;          /* a(v) * (served - beta * overdue)          (needs acc)           */
} rk_serve_out;
rk_status rk_greedy_serve(rk_ctx* ctx, const rk_reward_cfg* cfg, int64_t N, int64_t delta_ns, const double* acc,
                          rk_serve_out* out, void* stream);

/* NEXT-1 baseline: "runs all models asynchronously, one model per batch of requests" (r_u
 * is the sum of the models' throughputs in this mode). Reading S2: K servers
 * (one per model) share one FIFO queue; whenever a model is idle at t, the lowest-index idle model m
 * applies Algorithm 3's rule with its own c(m, b) (len(q) >= max B -> the oldest max B; else the largest
 * b <= len(q) once c(m,b) + w(q0) + delta >= tau); the batch occupies m until t + c(m, b) and another idle
 * model may dispatch at the same t. Same cfg fields as rk_greedy_serve. acc: [K] host single-model
 * accuracies a({m}) or NULL; reward = sum over batches of a(m) * (b - beta * overdue). Output arrays are
 * host [nR] (out fields; each may be NULL), model_batches host [nR][K] or NULL. Blocks on `stream`. */
rk_status rk_async_serve(rk_ctx* ctx, const rk_reward_cfg* cfg, int64_t N, int64_t delta_ns, const double* acc,
                         rk_serve_out* out, uint64_t* model_batches, void* stream);

/* NEXT-1 serving loop: serve N requests with features X ([N][D] bf16, DEVICE, request order = arrival
 * order) under action v with Algorithm 3 batching (rk_greedy_serve's rule for subset v on the single
 * arrival stream of cfg, nR == 1): every dispatched batch runs the K heads (A1+A2, tcgen05 GEMM) on its
 * rows and the per-request prediction of v (rk_predict's kernel), one batch at a time, in dispatch order.
 * pred_vote / pred_avg: [N] int32 DEVICE or NULL; requests never served (fewer than min B left at the end)
 * get -1. out: host, one element per field (may be NULL); *n_batches = batches served (may be NULL).
 * Needs heads (rk_load_ensemble with W). The context's rk_score workspaces are reused: call rk_score again
 * before rk_subset_accumulate / rk_predict. Blocks on `stream`. */
rk_status rk_serve_stream(rk_ctx* ctx, const void* X_bf16, int64_t N, const rk_reward_cfg* cfg, int64_t delta_ns,
                          uint32_t v, int32_t* pred_vote, int32_t* pred_avg, rk_serve_out* out, int64_t* n_batches,
                          void* stream);

/* NEXT-2: the actor-critic scheduler (§2.4 eqs. `eq:J`, `eq:dJ`, `eq:hatJ` with the
 * baseline V(s_t); §5.2: state, action space (2^|M|-1)*|B|, reward eq. `multi_acc_reward`;
 * reading S3). Environment: the loaded ensemble's K models as K servers, one FIFO request queue
 * (arrival times `arrival` [Narr], device, non-decreasing -- e.g. rk_sine_arrivals), B / c(m,b) / tau /
 * beta from cfg (rates ignored), a(v) = acc [S] (host; e.g. cnt_vote / N of rk_subset_stats: the
 * surrogate accuracy). At decision time t the state (F = L + K*nB + K floats) is the waits
 * (t - t_s)/tau of the oldest L queued requests (0-padded), c(m,b)/tau, and max(0, free_m - t)/tau; the
 * action a = (v-1)*nB + b_index; the batch (next b requests) starts at max(t, its last arrival, free_m for
 * m in v), runs c(v,b) = max_{m in v} c(m,b) on every member; R = a(v) (b - beta * overdue); the next
 * decision is at max(start, min_m free_m). Policy pi = softmax(W2 tanh(W1 x + b1) + b2) over A = S*nB
 * actions, value V = v2 . tanh(V1 x + c1) + c2; params: flat fp32 [W1 H*F | b1 H | W2 A*H | b2 A |
 * V1 H*F | c1 H | v2 H | c2 1] (row-major), n_params = rk_ac_dims. Limits: H in [1,64], A <= 2048,
 * F <= 1024, L in [0,256]. */
typedef struct {
  int L;                   /* queue waits in the state                                        */
  int H;                   /* hidden units of both networks                                   */
  int n_steps;             /* decisions per episode (n of eq. eq:J)                           */
  double gamma;            /* discount                                                        */
  double reward_scale;     /* returns are formed from R * reward_scale                        */
  double entropy;          /* entropy bonus c: the policy loss adds -c * mean_t H(pi(.|s_t)) (the
                              entropy term of the PPO objective the paper cites, X4); 0 = plain
                              actor-critic                                                     */
} rk_ac_cfg;
/* Trajectories of E episodes x n_steps, DEVICE buffers (caller-owned): states [E][n][F] fp32,
 * actions [E][n] int32, rewards [E][n] fp64 (unscaled R), overdue / t_dec / t_start / t_done [E][n]
 * (int32 / int64 ns; each may be NULL). */
typedef struct {
  float* states; int32_t* actions; double* rewards; int32_t* overdue; int64_t* t_dec; int64_t* t_start; int64_t* t_done;
} rk_ac_traj;
/* F, A and the parameter count for the loaded ensemble with nB batch sizes. */
rk_status rk_ac_dims(rk_ctx* ctx, int nB, const rk_ac_cfg* ac, int* F, int* A, int64_t* n_params);
/* Roll out E episodes in parallel (one warp each): episode e starts at request h0[e] (device [E]) with every
 * model idle at its arrival. forced: [E][n] device actions, or NULL to sample from the policy with a
 * counter-based uniform of (seed, e, step). RK_EINVAL if an episode would run past Narr. */
rk_status rk_ac_rollout(rk_ctx* ctx, const rk_reward_cfg* cfg, const double* acc, const int64_t* arrival, int64_t Narr,
                        const rk_ac_cfg* ac, const float* params, int E, const int64_t* h0, const int32_t* forced,
                        uint64_t seed, rk_ac_traj* traj, void* stream);
/* Actor-critic gradient of the trajectories (states, actions, rewards): G_t = sum_{k>=t} gamma^(k-t) R_k
 * reward_scale, A_t = G_t - V(s_t); policy loss -(1/(E n)) sum_t [A_t log pi(a_t|s_t) + entropy * H(pi(.|s_t))]
 * (A_t held fixed, eq. eq:hatJ), value loss (1/(E n)) sum_t (V(s_t) - G_t)^2. grad: device [n_params] (policy then value
 * parts, the params layout); losses: host [2] (policy, value) or NULL. Deterministic (fixed-order sums). */
rk_status rk_ac_grad(rk_ctx* ctx, const rk_reward_cfg* cfg, const rk_ac_cfg* ac, const float* params,
                     const rk_ac_traj* traj, int E, float* grad, double* losses, void* stream);
/* One SGD step: params -= lr_pi * grad on the policy part and lr_v * grad on the value part (device). */
rk_status rk_ac_apply(rk_ctx* ctx, const rk_reward_cfg* cfg, const rk_ac_cfg* ac, float* params, const float* grad,
                      float lr_pi, float lr_v, void* stream);

/* NEXT-4: the paper's request-arrival process (§7.2, eqs. `eq:r1`/`eq:r2`; reading Q16):
 * rate(t) = k sin(2 pi t / T) + b with k = 0.1 ref / (1 - s0), b = 1.1 ref - k, s0 = sin(0.3 pi) =
 * (1 + sqrt 5)/4 (the rate exceeds ref for 20 % of each period T and peaks at 1.1 ref).
 * The simulator is invoked every delta_ns; invocation j adds n_j = floor(max(0, delta * rate(j delta) *
 * (1 + phi_j)) + 0.5) requests ("delta x (gamma sin(t) + b) x (1 + phi), phi ~ N(0, 0.1)"), phi_j =
 * noise_std * z_j, z_j the Irwin-Hall(4) unit normal sum of the four 16-bit fields of
 * h = mix(mix(mix(seed ^ 0x51AE0A77) ^ j) + 0x2545F4914F6CDD1D) minus 131070, times 7 / 2^18 (mix = the
 * SplitMix64 finalizer), and the n_j requests arrive evenly spaced inside the invocation:
 * t = j delta + floor(i delta / n_j), i < n_j. Writes the arrival times (ns, non-decreasing) of global
 * requests [n0, n0 + N) to out_ns ([N] int64, DEVICE memory; earlier requests are generated and skipped,
 * so shards of one stream agree). Feeds rk_reward_cfg.arrival_ns and rk_greedy_serve. Blocks on `stream`
 * (the chunk loop reads each chunk's request total). Errors: ref <= 0, period_ns <= 0, delta_ns <= 0,
 * noise_std < 0 or non-finite, n0 < 0, N < 0 -> RK_EINVAL. */
typedef struct {
  double ref_rate;         /* r_u or r_l in req/s                                   */
  int64_t period_ns;       /* T; the paper uses 500 * tau                           */
  int64_t delta_ns;        /* invocation interval delta                                              */
  double noise_std;        /* 0.1 in the paper ("phi ~ N(0, 0.1)", read as the standard deviation) */
  uint64_t seed;
} rk_sine_cfg;
rk_status rk_sine_arrivals(rk_ctx* ctx, const rk_sine_cfg* cfg, int64_t n0, int64_t N, int64_t* out_ns, void* stream);

/* Serving of one action (NEXT-1) and parity hook: per-sample predictions of subset v on the
 * last rk_score* batch. pred_vote, pred_avg: [N] int32; avgprob: [N][C] fp32 averaged
 * probabilities. Device pointers; each may be NULL. v == 0 -> RK_EINVAL. */
rk_status rk_predict(rk_ctx* ctx, uint32_t v, int32_t* pred_vote, int32_t* pred_avg, float* avgprob,
                     void* stream);

/* Device pointers of the last rk_score* outputs: logits [N][K][ldc] fp32, top1 [N][K] int32 (A2),
 * rmax [N][K] fp32 = max_c logit, lsum [N][K] fp32 = log sum_c exp(logit - rmax) -- the softmax
 * normaliser RELATIVE to the row max, so p[n][m][c] = exp((logit - rmax) - lsum) and the log-sum-exp is
 * rmax + lsum (kept apart: their fp32 sum would round at the magnitude of the logits). top1/rmax/lsum
 * are NULL after rk_score_logits. Any pointer argument may be NULL. Valid until the next rk_score*. */
rk_status rk_outputs(rk_ctx* ctx, const float** logits, int* ldc, const int32_t** top1, const float** rmax,
                     const float** lsum, int64_t* N);
/* The GEMM epilogue's second-largest logit per (row, model) of the last rk_score batch, [N][K] fp32 device
 * memory (the row maximum over all classes but one occurrence of rmax, so equal to rmax on a tied maximum;
 * the averaging kernel's row-skip proof), or NULL when that batch did not produce it
 * (rk_score_logits, rk_score_labelled, C <= 128). Valid until the next rk_score*. */
rk_status rk_outputs_s2(rk_ctx* ctx, const float** s2);

/* Parity hook for the labelled moments (A5): the per-(group, subset) majority-vote correct counts of the
 * LAST rk_subset_accumulate chunk, out[g][v-1] = #{n in group g : vote of v correct} (uint8), groups of
 * *gs consecutive samples (gs = the largest power of two <= 16 dividing gcd(B); the last group may be
 * partial), *groups = ceil(N_chunk / gs). They exist only when cfg had want_labelled, nB > 0 and nR > 0
 * (otherwise *gs = *groups = 0). out: host or device, cap >= groups * S bytes, may be NULL to query
 * the sizes. Blocks on `stream`. RK_ESTATE before the first accumulate after a reset. */
rk_status rk_group_counts(rk_ctx* ctx, uint8_t* out, int64_t cap, int* gs, int64_t* groups, void* stream);

/* Diagnostics of the LAST rk_subset_accumulate chunk (K <= 8 path): *worklist = samples whose label is an
 * averaging candidate of some subset and that are not unanimous (the samples the averaging kernels visit),
 * *fallback = of those, the samples a fused batch (rk_score_labelled) recomputed with logits (0 otherwise),
 * *rows_skipped = (worklist sample, model) rows the averaging kernel did not stream because the GEMM's
 * second-largest logit proves they add only the label to the candidate set (rk_score batches with more
 * than 128 classes; 0 otherwise; a 32-bit diagnostic counter).
 * Synchronises the device. Any pointer may be NULL. */
rk_status rk_vote_diag(rk_ctx* ctx, int64_t* worklist, int64_t* fallback, int64_t* rows_skipped);

/* Per-kernel device time, measured with CUDA events on the launch stream when profiling is on. */
typedef struct {
  const char* name;        /* static string                                                     */
  int64_t launches;
  double total_ms;
  double bytes;            /* algorithmic bytes moved (HBM roofline), summed over launches      */
  double flops;            /* algorithmic flops (tensor roofline), summed over launches         */
} rk_kernel_stat;
rk_status rk_set_profiling(rk_ctx* ctx, int on);   /* on=1 resets the counters                  */
/* Writes up to max entries; *n = number of kernel kinds. Synchronises the context's events. */
rk_status rk_kernel_stats(rk_ctx* ctx, rk_kernel_stat* out, int max, int* n);

const char* rk_last_error(const rk_ctx* ctx);
const char* rk_status_string(rk_status s);
void rk_destroy(rk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
