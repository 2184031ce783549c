/* oracle.h — plain, slow CPU oracle for the Rafiki ensemble-subset hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_1804_06087_b200/, librk.so) never links, imports or calls it, and shares no
 * code with it (the seeded input generators in gen/ are the only shared module).
 *
 * Every function follows a definition in PAPER.md (arXiv 1804.06087) written out
 * directly: loops over samples, then subsets v = 1..2^K-1, then members/classes.
 * No pruning, no fast paths, fp64/int64 arithmetic. Readings of silent/ambiguous
 * passages are the SURVEY.md §8(c) Q-readings, listed in DESIGN.md.
 *
 * Pins (tests/test_oracle_*.py, tests/golden/): hand-computed examples W1-W4,
 * invariants I1-I8, reward examples R1-R5, R6 (queue-aware latency,
 * reading Q15) and S1 (Algorithm 3 greedy batching, reading S1) worked by hand, brute force
 * against an independently written pairwise formulation, library pins (numpy
 * argmax/bincount, torch.softmax). Parity unpinned: the paper's Fig. `fig:ensemble` values
 * (images only).
 */
#ifndef RK_ORACLE_H
#define RK_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OR_TIE_BEST_MEMBER = 0, OR_TIE_LOWEST_CLASS = 1 };
enum { OR_OK = 0, OR_EINVAL = 1, OR_ELABEL = 6, OR_ENONFINITE = 7, OR_ENOMEM = 3 };

/* Batch/latency configuration for the eq. `multi_acc_reward` moments. */
typedef struct {
  int nB;                 /* number of candidate batch sizes (0 = counts only)          */
  const int* B;           /* [nB] batch sizes                         */
  double beta;            /* balancing factor (PAPER.md:345 Table tb:notation)            */
  int64_t tau_ns;         /* SLO tau in ns                                 */
  const int64_t* lat_ns;  /* [K][nB] c(m,b) in ns                      */
  int nR;                 /* number of arrival rates                                      */
  const double* rates;    /* [nR] req/s; t_s = floor(s*1e9/r) (reading Q9)                */
  const int64_t* arrival_ns; /* [N] or NULL: caller arrivals (then nR must be 1)          */
  int want_exceed;        /* also compute E (eq. `eq:single`)           */
  int queue;              /* 0: batch j dispatched when full (reading Q8); 1: one ensemble
                             server, FIFO: start_j = max(t_last(j), finish_{j-1}), "the next
                             batch has to wait" (reading Q15)                */
} or_cfg;

/* Output table (host, caller-allocated). S = 2^K-1, index v-1. */
typedef struct {
  uint64_t* cnt_vote;  /* [S]   majority-vote correct counts                     */
  uint64_t* cnt_avg;   /* [S]   averaged-probability correct counts              */
  uint64_t* n_amb;     /* [S]   (n,v) pairs whose fp64 avg top-2 gap <= 1e-12 rel */
  uint64_t* corr;      /* [nB][S]                                                */
  uint64_t* O;         /* [nR][nB][S]                                            */
  uint64_t* Q;         /* [nR][nB][S]                                            */
  uint64_t* E;         /* [nR][nB][S] or NULL                                    */
  double* reward_sur;  /* [nR][nB][S]                                            */
  double* reward_lab;  /* [nR][nB][S]                                            */
  uint8_t* vote_ok;    /* [N][S] or NULL: per-sample majority-vote correctness (parity of the
                          per-(group, subset) counts behind the labelled moments)  */
  uint8_t* avg_ok;     /* [N][S] or NULL: per-sample averaged-probability correctness */
} or_table;

/* Per-model top-1: smallest class index attaining the max (reading Q4). */
int or_top1_f32(const float* row, int C);
int or_top1_f64(const double* row, int C);
/* Softmax with max subtraction in fp64 (reading Q5, "average the results"). */
void or_softmax(const double* l, int C, double* p);
/* log-sum-exp in fp64. */
double or_lse(const double* l, int C);
/* Majority vote over members of v (§5.2). tie: OR_TIE_BEST_MEMBER (paper:
 * prediction of the best-ranked member among the tied voters, reading Q2) or
 * OR_TIE_LOWEST_CLASS (north_star). rank: [K] 0 = best, NULL = index order. */
int or_vote(const int* top1, int K, int C, uint32_t v, const int* rank, int tie);
/* Averaged-probability prediction: argmax_c (sum_{i in v asc} p[i][c])/|v|,
 * smallest index on ties; *amb = 1 if (a1-a2)/a1 <= 1e-12 (reading Q6). p is [K][C]. */
int or_avg(const double* p, int K, int C, uint32_t v, int* amb, double* avg_out /*[C] or NULL*/);

/* Step A1: logits of K synthetic dense heads, fp64: out[n][m][c] = 2^s * sum_d x*w + bias.
 * X [N][D] bf16 bits, W [K][C][D] bf16 bits, bias [K][C] or NULL. Exact for small-int inputs. */
void or_logits_gemm(const uint16_t* X, const uint16_t* W, const float* bias, int64_t N, int K, int C,
                    int D, int scale_log2, double* out, int threads);

/* Steps A2-A7 over the whole dataset. Exactly one of logits_f32 ([N][K][ldc]) or
 * logits_f64 ([N][K][C]) is non-NULL. top1 ties use the given precision. */
int or_table_build(const float* logits_f32, int ldc, const double* logits_f64, int64_t N, int K, int C,
                   const int32_t* labels, const int* rank, int tie, const or_cfg* cfg, or_table* out,
                   int threads);

/* Per-sample outputs for one action v (serving step, NEXT-1; parity hook for I4):
 * pred_vote/pred_avg [N] and avgprob [N][C] (each may be NULL), top1 [N][K], lse [N][K] (NULL ok). */
int or_predict(const float* logits_f32, int ldc, const double* logits_f64, int64_t N, int K, int C,
               uint32_t v, const int* rank, int tie, int32_t* pred_vote, int32_t* pred_avg, double* avgprob,
               int32_t* top1, double* lse, int threads);

/* Arrival time of global request s at rate r (reading Q9): floor((double)s*1e9/r) ns. */
int64_t or_arrival_ns(int64_t s, double rate);

/* NEXT-4: sine-plus-noise arrivals (eqs. eq:r1/eq:r2, reading Q16):
 * k, b of rate(t) = k sin(2 pi t / T) + b for ref = r_u or r_l; the request count of simulator invocation j;
 * the arrival times of global requests [n0, n0 + N) (invocation j's n_j requests evenly spaced inside it). */
void or_sine_params(double ref, double* k, double* b);
int64_t or_sine_count(double ref, int64_t period_ns, int64_t delta_ns, double sigma, uint64_t seed, int64_t j);
int or_sine_arrivals(double ref, int64_t period_ns, int64_t delta_ns, double sigma, uint64_t seed, int64_t n0,
                     int64_t N, int64_t* out);

/* NEXT-1: Algorithm 3, Inference(Queue q, Model m), greedy batching of one
 * synchronous ensemble v (c(v,b) = max over members of c(m,b)) on a request stream,
 * single server, inference blocks the loop (reading S1): whenever the server is idle at time t,
 * with q the arrived, unserved requests (oldest first):
 *   len(q) >= max B                                   -> infer the oldest max B at t;
 *   b = max{b in B : b <= len(q)} exists and
 *     c(v,b) + (t - t_q0) + delta >= tau              -> infer the oldest b at t;
 *   otherwise wait until the next arrival or until that condition becomes true.
 * A batch inferred at t completes at t + c(v,b); l(s) = completion - t_s; overdue iff l(s) > tau.
 * Requests still queued (fewer than min B) after the last arrival are unserved.
 * Output per (rate r, subset v): out[r*S + v-1]. */
typedef struct { uint64_t served, overdue, exceed_ns, batches, unserved; } or_serve;
int or_greedy_serve(const or_cfg* cfg, int K, int64_t N, int64_t delta_ns, or_serve* out);

/* NEXT-1 baseline: all models asynchronously, one model per batch (reading S2): K
 * servers, one FIFO queue, Algorithm 3's rule evaluated by the lowest-index idle model with its own
 * c(m, b). acc: [K] single-model accuracies a(m) or NULL; per rate r: out[r], reward[r] (sum over batches
 * of a(m) * (b - beta * overdue)) and model_batches[r][K] (each may be NULL except out). */
int or_async_serve(const or_cfg* cfg, int K, int64_t N, int64_t delta_ns, const double* acc, or_serve* out,
                   double* reward, uint64_t* model_batches);

/* NEXT-2: the RL scheduler's environment and actor-critic estimator (§2.4 eqs. eq:J /
 * eq:dJ / eq:hatJ and the baseline V(s_t); §5.2 state, action, reward; reading S3).
 * Environment: K model servers, one FIFO request queue with the given arrival times. At decision time t
 * the state is x = [waits of the oldest L queued requests (t - t_s)/tau, 0-padded | c(m,b)/tau for m, b |
 * max(0, free_m - t)/tau for m], each (float)((double)ns / (double)tau). Action a = (v-1)*nB + b_index
 * (SPEC.md:603-611). The batch is the next b requests; it starts at max(t, arrival of its last request,
 * free_m for m in v), takes c(v,b) = max_{m in v} c(m,b), occupies every m in v until done; reward
 * R = a(v) * (b - beta * #{s : done - t_s > tau}) (eq. multi_acc_reward); the next decision is at
 * max(start, min_m free_m). */
typedef struct {
  int K, nB, L;
  const int* B;            /* [nB] */
  const int64_t* lat_ns;   /* [K][nB] */
  int64_t tau_ns;
  double beta;
  const double* acc;       /* [S] a(v) */
  const int64_t* arrival;  /* [Narr] non-decreasing */
  int64_t Narr;
} or_env;
/* One episode of n decisions from request h0 (all models idle at t = arrival[h0]) under the given actions.
 * states [n][F] (F = L + K*nB + K), rewards [n], overdue [n], t_dec / t_start / t_done [n] (each may be NULL
 * except actions). Returns OR_EINVAL if a batch would run past Narr. */
int or_env_rollout(const or_env* env, const int32_t* actions, int n, int64_t h0, float* states, double* rewards,
                   int32_t* overdue, int64_t* t_dec, int64_t* t_start, int64_t* t_done);
/* Actor-critic gradients (fp64) for E episodes of n steps: G_t = sum_{k>=t} gamma^(k-t) R_k * scale,
 * A_t = G_t - V(s_t); policy loss -(1/(E n)) sum A_t log pi(a_t|s_t) (A_t constant), value loss
 * (1/(E n)) sum (V(s_t) - G_t)^2; with ent > 0 the policy loss also has -(ent/(E n)) sum_t H(pi(.|s_t)).
 * Networks: pi = softmax(W2 tanh(W1 x + b1) + b2) over A actions,
 * V = v2 . tanh(V1 x + c1) + c2, hidden H. params / grad: the flat layout
 * [W1 H*F | b1 H | W2 A*H | b2 A | V1 H*F | c1 H | v2 H | c2 1] (row-major). Also returns the mean
 * unscaled episode return sum_t R_t and the two losses (each pointer may be NULL). */
int or_ac_grad(int F, int H, int A, const double* params, const float* states, const int32_t* actions,
               const double* rewards, int E, int n, double gamma, double scale, double ent, double* grad,
               double* loss_pi, double* loss_v);

#ifdef __cplusplus
}
#endif
#endif
