/* oracle.c — plain CPU oracle. TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Written from PAPER.md (arXiv 1804.06087). Each function cites the passage it follows.
 * Loops are in the order the definitions are stated; no pruning, no fast paths.
 */
#include "oracle.h"
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---- A2: per-model top-1 ("top-1"; reading Q4: lowest index on ties) ---- */
int or_top1_f32(const float* row, int C) {
  int best = 0;
  for (int c = 1; c < C; ++c)
    if (row[c] > row[best]) best = c;
  return best;
}
int or_top1_f64(const double* row, int C) {
  int best = 0;
  for (int c = 1; c < C; ++c)
    if (row[c] > row[best]) best = c;
  return best;
}

/* ---- A2: softmax probabilities, fp64, max-subtracted (reading Q5) ---------------------- */
void or_softmax(const double* l, int C, double* p) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) { p[c] = exp(l[c] - mx); s += p[c]; }
  for (int c = 0; c < C; ++c) p[c] = p[c] / s;
}
double or_lse(const double* l, int C) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += exp(l[c] - mx);
  return mx + log(s);
}

/* ---- A3: majority vote of the members' top-1 predictions (§5.2:
 * "Majority voting is applied to aggregate the predictions ... when there is a tie, the
 * prediction from the model with the best accuracy is selected as the final prediction").
 * cnt[c] = #members predicting c; M = max cnt.
 *   BEST_MEMBER : top1[i*], i* = argmin rank[i] over members i with cnt[top1[i]] == M  (Q2)
 *   LOWEST_CLASS: min { c : cnt[c] == M }                                             (north_star)
 * cnt is a full class histogram (thread-local, re-zeroed after each call). */
int or_vote(const int* top1, int K, int C, uint32_t v, const int* rank, int tie) {
  static _Thread_local int* cnt = NULL; /* class histogram, all zero between calls */
  static _Thread_local int cap = 0;
  if (cap < C) { free(cnt); cnt = (int*)calloc((size_t)C, sizeof(int)); cap = C; }
  int M = 0;
  for (int i = 0; i < K; ++i)
    if ((v >> i) & 1u) cnt[top1[i]]++;
  for (int i = 0; i < K; ++i)
    if (((v >> i) & 1u) && cnt[top1[i]] > M) M = cnt[top1[i]];
  int winner = -1;
  if (tie == OR_TIE_BEST_MEMBER) {
    int best_i = -1;
    for (int i = 0; i < K; ++i) {
      if (!((v >> i) & 1u) || cnt[top1[i]] != M) continue;
      if (best_i < 0 || (rank ? rank[i] < rank[best_i] : i < best_i)) best_i = i;
    }
    winner = top1[best_i];
  } else {
    for (int c = 0; c < C && winner < 0; ++c)
      if (cnt[c] == M) winner = c;
  }
  for (int i = 0; i < K; ++i)
    if ((v >> i) & 1u) cnt[top1[i]] = 0;
  return winner;
}

/* ---- A4: averaged softmax probabilities ("ensemble multiple models and average
 * the results"): avg[c] = (sum_{i in v, ascending i} p[i][c]) / |v|; prediction = smallest c
 * attaining the max (reading Q6). a1 >= a2 are the two largest avg values over distinct
 * classes; the pair is ambiguous if (a1 - a2)/a1 <= 1e-12 (includes exact ties). */
int or_avg(const double* p, int K, int C, uint32_t v, int* amb, double* avg_out) {
  int nv = 0;
  for (int i = 0; i < K; ++i) nv += (int)((v >> i) & 1u);
  int pred = 0;
  double a1 = -1.0, a2 = -1.0;
  for (int c = 0; c < C; ++c) {
    double s = 0.0;
    for (int i = 0; i < K; ++i)
      if ((v >> i) & 1u) s += p[(int64_t)i * C + c];
    double a = s / (double)nv;
    if (avg_out) avg_out[c] = a;
    if (a > a1) { a2 = a1; a1 = a; pred = c; }
    else if (a > a2) a2 = a;
  }
  if (amb) *amb = (a1 - a2) / a1 <= 1e-12;
  return pred;
}

/* ---- A1: synthetic dense heads (stand-in for the ConvNets' classifier layer, PAPER.md:152-154;
 * "inference time which depends on the model complexity"). fp64 sums of exact
 * bf16 products. ---------------------------------------------------------------------------- */
static double bf16_val(uint16_t b) {
  union { uint32_t u; float f; } v;
  v.u = (uint32_t)b << 16;
  return (double)v.f;
}

typedef struct {
  const uint16_t *X, *W;
  const float* bias;
  int64_t n0, n1;
  int K, C, D, s;
  double* out;
} gemm_job;

static void* gemm_thr(void* a) {
  gemm_job* j = (gemm_job*)a;
  double* xr = (double*)malloc(sizeof(double) * j->D);
  double scale = ldexp(1.0, j->s);
  for (int64_t n = j->n0; n < j->n1; ++n) {
    for (int d = 0; d < j->D; ++d) xr[d] = bf16_val(j->X[n * j->D + d]);
    for (int m = 0; m < j->K; ++m)
      for (int c = 0; c < j->C; ++c) {
        const uint16_t* w = j->W + ((int64_t)m * j->C + c) * j->D;
        double acc = 0.0;
        for (int d = 0; d < j->D; ++d) acc += xr[d] * bf16_val(w[d]);
        double b = j->bias ? (double)j->bias[(int64_t)m * j->C + c] : 0.0;
        j->out[(n * j->K + m) * j->C + c] = acc * scale + b;
      }
  }
  free(xr);
  return NULL;
}

void or_logits_gemm(const uint16_t* X, const uint16_t* W, const float* bias, int64_t N, int K, int C, int D,
                    int scale_log2, double* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  gemm_job jobs[256];
  int64_t per = (N + threads - 1) / threads;
  int nt = 0;
  for (int t = 0; t < threads; ++t) {
    int64_t a = t * per, b = a + per < N ? a + per : N;
    if (a >= b) break;
    gemm_job g = {X, W, bias, a, b, K, C, D, scale_log2, out};
    jobs[t] = g;
    pthread_create(&th[t], NULL, gemm_thr, &jobs[t]);
    nt++;
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* ---- arrivals (reading Q9) --------------------------------------------------------------- */
int64_t or_arrival_ns(int64_t s, double rate) {
  volatile double num = (double)s * 1e9; /* two IEEE roundings, in this order */
  return (int64_t)floor(num / rate);
}

/* ---- NEXT-4: the sine-plus-noise arrival process (eqs. eq:r1/eq:r2; reading Q16) ----
 * rate(t) = k sin(2 pi t / T) + b. Eq. eq:r1: the rate exceeds ref for 20 % of each period -> the
 * threshold phase 0.3 pi, s0 = sin(0.3 pi); eq. eq:r2: peak k + b = 1.1 ref. Hence k (1 - s0) = 0.1 ref
 * (SPEC.md:705). The simulator, invoked every delta, adds delta * rate * (1 + phi) requests (rounded
 * half up, never negative), phi = sigma * z with z the counter-based Irwin-Hall(4) normal of invocation j;
 * they arrive evenly spaced inside the invocation. */
static uint64_t or_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void or_sine_params(double ref, double* k, double* b) {
  const double s0 = sin(0.3 * M_PI);
  *k = 0.1 * ref / (1.0 - s0);
  *b = 1.1 * ref - *k;
}

int64_t or_sine_count(double ref, int64_t period_ns, int64_t delta_ns, double sigma, uint64_t seed, int64_t j) {
  double k, b;
  or_sine_params(ref, &k, &b);
  const double t = (double)((j * delta_ns) % period_ns) / (double)period_ns; /* phase of t = j delta in [0, 1) */
  const double rate = k * sin(2.0 * M_PI * t) + b;
  const uint64_t h = or_mix64(or_mix64(or_mix64(seed ^ 0x51AE0A77ull) ^ (uint64_t)j) + 0x2545F4914F6CDD1Dull);
  const int64_t ih = (int64_t)(h & 0xffff) + (int64_t)((h >> 16) & 0xffff) + (int64_t)((h >> 32) & 0xffff) +
                     (int64_t)(h >> 48) - 131070;
  const double z = (double)ih * 7.0 / 262144.0;
  const double phi = sigma * z;
  double y = ((double)delta_ns / 1e9) * rate * (1.0 + phi);
  if (!(y > 0.0)) y = 0.0;
  return (int64_t)floor(y + 0.5);
}

int or_sine_arrivals(double ref, int64_t period_ns, int64_t delta_ns, double sigma, uint64_t seed, int64_t n0,
                     int64_t N, int64_t* out) {
  if (!(ref > 0) || period_ns <= 0 || delta_ns <= 0 || !(sigma >= 0) || n0 < 0 || N < 0) return OR_EINVAL;
  int64_t s = 0; /* global index of the next request */
  for (int64_t j = 0; s < n0 + N; ++j) {
    const int64_t n = or_sine_count(ref, period_ns, delta_ns, sigma, seed, j);
    for (int64_t i = 0; i < n; ++i, ++s)
      if (s >= n0 && s < n0 + N) out[s - n0] = j * delta_ns + (i * delta_ns) / n;
  }
  return OR_OK;
}

/* ---- A5-A7: table ------------------------------------------------------------------------- */
typedef struct {
  const float* lf;
  int ldc;
  const double* ld;
  int64_t N, a, b;
  int K, C;
  const int32_t* labels;
  const int* rank;
  int tie;
  const or_cfg* cfg;
  const int64_t* fin;  /* queue mode: finish time of every complete batch [nR][nB][S][nbmax] */
  int64_t nbmax;
  int status;
  uint8_t *vote_bits, *avg_bits;  /* [N][S] per-sample outputs or NULL (shared, disjoint rows) */
  /* thread-local accumulators */
  uint64_t *cnt_vote, *cnt_avg, *n_amb, *corr, *O, *Q, *E;
} table_job;

static int64_t gcd64(int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; }

/* Row access: returns 0 on non-finite (NaN, +inf, or all -inf). */
static int load_row(const table_job* j, int64_t n, int m, double* l, int* top1) {
  double mx = -INFINITY;
  for (int c = 0; c < j->C; ++c) {
    double x = j->lf ? (double)j->lf[(n * j->K + m) * (int64_t)j->ldc + c] : j->ld[(n * j->K + m) * (int64_t)j->C + c];
    if (isnan(x) || x == INFINITY) return 0;
    l[c] = x;
    if (x > mx) mx = x;
  }
  if (mx == -INFINITY) return 0;
  *top1 = j->lf ? or_top1_f32(j->lf + (n * j->K + m) * (int64_t)j->ldc, j->C)
                : or_top1_f64(j->ld + (n * j->K + m) * (int64_t)j->C, j->C);
  return 1;
}

static int64_t arrival(const or_cfg* cfg, int r, int64_t s) {
  return cfg->arrival_ns ? cfg->arrival_ns[s] : or_arrival_ns(s, cfg->rates[r]);
}

static void* table_thr(void* arg) {
  table_job* j = (table_job*)arg;
  const int K = j->K, C = j->C, S = (1 << K) - 1;
  const or_cfg* cfg = j->cfg;
  const int nB = cfg ? cfg->nB : 0, nR = cfg ? cfg->nR : 0;
  double* l = (double*)malloc(sizeof(double) * C);
  double* p = (double*)malloc(sizeof(double) * (size_t)K * C);
  int top1[32];
  uint8_t* vote_ok = (uint8_t*)malloc((size_t)S);
  uint64_t* corr_cur = (uint64_t*)calloc((size_t)(nB > 0 ? nB : 1) * S, sizeof(uint64_t));
  for (int64_t n = j->a; n < j->b; ++n) {
    int y = j->labels[n];
    if (y < 0 || y >= C) { j->status = OR_ELABEL; break; }
    for (int m = 0; m < K; ++m) {
      if (!load_row(j, n, m, l, &top1[m])) { j->status = OR_ENONFINITE; goto done; }
      or_softmax(l, C, p + (int64_t)m * C);
    }
    for (uint32_t v = 1; v <= (uint32_t)S; ++v) {
      int wv = or_vote(top1, K, C, v, j->rank, j->tie);
      int amb = 0;
      int wa = or_avg(p, K, C, v, &amb, NULL);
      vote_ok[v - 1] = (uint8_t)(wv == y);
      if (j->vote_bits) j->vote_bits[n * S + (v - 1)] = (uint8_t)(wv == y);
      if (j->avg_bits) j->avg_bits[n * S + (v - 1)] = (uint8_t)(wa == y);
      j->cnt_vote[v - 1] += (uint64_t)(wv == y);
      j->cnt_avg[v - 1] += (uint64_t)(wa == y);
      j->n_amb[v - 1] += (uint64_t)amb;
    }
    /* per-(v,b) batch moments over complete global batches j = [jb*b, (jb+1)*b) (reading Q8, Q13) */
    for (int bi = 0; bi < nB; ++bi) {
      const int64_t b = cfg->B[bi];
      const int64_t nb = j->N / b;
      const int64_t jb = n / b;
      if (jb >= nb) continue; /* trailing partial batch excluded */
      for (int v = 0; v < S; ++v) corr_cur[(int64_t)bi * S + v] += vote_ok[v];
      if (n % b != b - 1) continue;
      /* batch complete: latency of each request l(s) = wait + c(v,b),
       * wait = t_last - t_s (dispatch when the batch is full), c(v,b) = max over members
       * (straggler); overdue <=> l(s) > tau, strict (reading Q10) */
      /* queue mode (reading Q15): l(s) = finish_j - t_s, finish_j from the FIFO recurrence */
      const int64_t s0 = jb * b, s1 = s0 + b;
      for (int r = 0; r < nR; ++r) {
        const int64_t tlast = arrival(cfg, r, s1 - 1);
        for (uint32_t v = 1; v <= (uint32_t)S; ++v) {
          int64_t c = 0;
          for (int m = 0; m < K; ++m)
            if (((v >> m) & 1u) && cfg->lat_ns[m * nB + bi] > c) c = cfg->lat_ns[m * nB + bi];
          const int64_t done = cfg->queue ? j->fin[(((int64_t)r * nB + bi) * S + (v - 1)) * j->nbmax + jb]
                                          : tlast + c;
          uint64_t o = 0, e = 0;
          for (int64_t s = s0; s < s1; ++s) {
            int64_t lat = done - arrival(cfg, r, s);
            if (lat > cfg->tau_ns) { o++; e += (uint64_t)(lat - cfg->tau_ns); }
          }
          const int64_t idx = ((int64_t)r * nB + bi) * S + (v - 1);
          j->O[idx] += o;
          j->Q[idx] += corr_cur[(int64_t)bi * S + (v - 1)] * o;
          if (j->E) j->E[idx] += e;
        }
      }
      for (int v = 0; v < S; ++v) {
        j->corr[(int64_t)bi * S + v] += corr_cur[(int64_t)bi * S + v];
        corr_cur[(int64_t)bi * S + v] = 0;
      }
    }
  }
done:
  free(l); free(p); free(vote_ok); free(corr_cur);
  return NULL;
}

int or_table_build(const float* logits_f32, int ldc, const double* logits_f64, int64_t N, int K, int C,
                   const int32_t* labels, const int* rank, int tie, const or_cfg* cfg, or_table* out,
                   int threads) {
  if (K < 1 || K > 12 || C < 2 || N < 0 || (!logits_f32 == !logits_f64)) return OR_EINVAL;
  if (cfg && cfg->nB > 0 && (!cfg->B || !cfg->lat_ns)) return OR_EINVAL;
  if (cfg && cfg->nR > 0 && !cfg->rates && !cfg->arrival_ns) return OR_EINVAL;
  if (cfg && cfg->arrival_ns && cfg->nR != 1) return OR_EINVAL;
  const int S = (1 << K) - 1;
  const int nB = cfg ? cfg->nB : 0, nR = cfg ? cfg->nR : 0;
  const int64_t nT = (int64_t)nR * nB * S;
  /* threads split at multiples of lcm(B) so no batch straddles two threads */
  int64_t L = 1;
  for (int bi = 0; bi < nB; ++bi) L = L / gcd64(L, cfg->B[bi]) * cfg->B[bi];
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  int64_t units = (N + L - 1) / L;
  if (threads > units) threads = (int)(units > 0 ? units : 1);
  int64_t per = (units + threads - 1) / threads;
  /* queue mode: the FIFO recurrence over the whole stream, in batch order, for every (r, b, v):
   * start_j = max(t_last(j), finish_{j-1}), finish_j = start_j + c(v,b) (Q15) */
  int64_t* fin = NULL;
  int64_t nbmax = 0;
  if (cfg && cfg->queue && nB > 0 && nR > 0) {
    for (int bi = 0; bi < nB; ++bi) if (N / cfg->B[bi] > nbmax) nbmax = N / cfg->B[bi];
    fin = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nT ? nT : 1) * (size_t)(nbmax ? nbmax : 1));
    if (!fin) return OR_EINVAL;
    for (int r = 0; r < nR; ++r)
      for (int bi = 0; bi < nB; ++bi) {
        const int64_t b = cfg->B[bi];
        for (uint32_t v = 1; v <= (uint32_t)S; ++v) {
          int64_t c = 0;
          for (int m = 0; m < K; ++m)
            if (((v >> m) & 1u) && cfg->lat_ns[m * nB + bi] > c) c = cfg->lat_ns[m * nB + bi];
          int64_t prev = INT64_MIN;
          for (int64_t jb = 0; jb < N / b; ++jb) {
            const int64_t ready = arrival(cfg, r, (jb + 1) * b - 1);
            const int64_t start = (prev == INT64_MIN || ready > prev) ? ready : prev;
            prev = start + c;
            fin[(((int64_t)r * nB + bi) * S + (v - 1)) * nbmax + jb] = prev;
          }
        }
      }
  }
  pthread_t th[256];
  table_job* jobs = (table_job*)calloc((size_t)threads, sizeof(table_job));
  int nt = 0;
  for (int t = 0; t < threads; ++t) {
    int64_t a = t * per * L, b = (t + 1) * per * L;
    if (b > N) b = N;
    if (a >= b) break;
    table_job* j = &jobs[t];
    j->lf = logits_f32; j->ldc = ldc; j->ld = logits_f64; j->N = N; j->a = a; j->b = b;
    j->K = K; j->C = C; j->labels = labels; j->rank = rank; j->tie = tie; j->cfg = cfg;
    j->fin = fin; j->nbmax = nbmax;
    j->vote_bits = out->vote_ok; j->avg_bits = out->avg_ok;
    j->cnt_vote = (uint64_t*)calloc((size_t)S, 8);
    j->cnt_avg = (uint64_t*)calloc((size_t)S, 8);
    j->n_amb = (uint64_t*)calloc((size_t)S, 8);
    j->corr = (uint64_t*)calloc((size_t)(nB ? nB : 1) * S, 8);
    j->O = (uint64_t*)calloc((size_t)(nT ? nT : 1), 8);
    j->Q = (uint64_t*)calloc((size_t)(nT ? nT : 1), 8);
    j->E = (cfg && cfg->want_exceed) ? (uint64_t*)calloc((size_t)(nT ? nT : 1), 8) : NULL;
    pthread_create(&th[t], NULL, table_thr, j);
    nt++;
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  int status = OR_OK;
  memset(out->cnt_vote, 0, (size_t)S * 8);
  memset(out->cnt_avg, 0, (size_t)S * 8);
  if (out->n_amb) memset(out->n_amb, 0, (size_t)S * 8);
  if (nB && out->corr) memset(out->corr, 0, (size_t)nB * S * 8);
  if (nT) {
    if (out->O) memset(out->O, 0, (size_t)nT * 8);
    if (out->Q) memset(out->Q, 0, (size_t)nT * 8);
    if (out->E) memset(out->E, 0, (size_t)nT * 8);
  }
  for (int t = 0; t < nt; ++t) {
    table_job* j = &jobs[t];
    if (j->status != OR_OK && status == OR_OK) status = j->status;
    for (int v = 0; v < S; ++v) {
      out->cnt_vote[v] += j->cnt_vote[v];
      out->cnt_avg[v] += j->cnt_avg[v];
      if (out->n_amb) out->n_amb[v] += j->n_amb[v];
    }
    for (int64_t i = 0; i < (int64_t)nB * S; ++i) if (out->corr) out->corr[i] += j->corr[i];
    for (int64_t i = 0; i < nT; ++i) {
      if (out->O) out->O[i] += j->O[i];
      if (out->Q) out->Q[i] += j->Q[i];
      if (out->E && j->E) out->E[i] += j->E[i];
    }
    free(j->cnt_vote); free(j->cnt_avg); free(j->n_amb); free(j->corr); free(j->O); free(j->Q); free(j->E);
  }
  free(jobs);
  free(fin);
  if (status != OR_OK) return status;
  /* A7: eq. `multi_acc_reward` a(M[v]) * (b - beta*|{s in batch : l(s) > tau}|),
   * summed over the n_b complete batches. Surrogate a(v) = validation accuracy of the vote
   * (reading Q7/Q11); labelled variant uses the batch's own correct fraction. */
  for (int r = 0; r < nR; ++r)
    for (int bi = 0; bi < nB; ++bi) {
      const double b = (double)cfg->B[bi];
      const double nb = (double)(N / cfg->B[bi]);
      for (int v = 0; v < S; ++v) {
        const int64_t idx = ((int64_t)r * nB + bi) * S + v;
        const double a = N > 0 ? (double)out->cnt_vote[v] / (double)N : 0.0;
        if (out->reward_sur) out->reward_sur[idx] = a * (nb * b - cfg->beta * (double)out->O[idx]);
        if (out->reward_lab)
          out->reward_lab[idx] = (double)out->corr[(int64_t)bi * S + v] - (cfg->beta / b) * (double)out->Q[idx];
      }
    }
  return OR_OK;
}

/* ---- per-sample outputs for one action v --------------------------------------------------- */
int or_predict(const float* logits_f32, int ldc, const double* logits_f64, int64_t N, int K, int C, uint32_t v,
               const int* rank, int tie, int32_t* pred_vote, int32_t* pred_avg, double* avgprob, int32_t* top1_out,
               double* lse_out, int threads) {
  (void)threads;
  if (K < 1 || K > 12 || C < 2 || v == 0 || v >= (1u << K) || (!logits_f32 == !logits_f64)) return OR_EINVAL;
  table_job j;
  memset(&j, 0, sizeof j);
  j.lf = logits_f32; j.ldc = ldc; j.ld = logits_f64; j.K = K; j.C = C;
  double* l = (double*)malloc(sizeof(double) * C);
  double* p = (double*)malloc(sizeof(double) * (size_t)K * C);
  int top1[32];
  int status = OR_OK;
  for (int64_t n = 0; n < N; ++n) {
    for (int m = 0; m < K; ++m) {
      if (!load_row(&j, n, m, l, &top1[m])) { status = OR_ENONFINITE; goto out; }
      if (top1_out) top1_out[n * K + m] = top1[m];
      if (lse_out) lse_out[n * K + m] = or_lse(l, C);
      or_softmax(l, C, p + (int64_t)m * C);
    }
    if (pred_vote) pred_vote[n] = or_vote(top1, K, C, v, rank, tie);
    if (pred_avg || avgprob) {
      int amb;
      int a = or_avg(p, K, C, v, &amb, avgprob ? avgprob + n * (int64_t)C : NULL);
      if (pred_avg) pred_avg[n] = a;
    }
  }
out:
  free(l); free(p);
  return status;
}

/* ---- NEXT-1: Algorithm 3 greedy batching (reading S1) ------------------------ */
int or_greedy_serve(const or_cfg* cfg, int K, int64_t N, int64_t delta_ns, or_serve* out) {
  if (!cfg || K < 1 || K > 12 || N < 0 || cfg->nB < 1 || !cfg->B || !cfg->lat_ns || cfg->nR < 1) return OR_EINVAL;
  if (!cfg->rates && !cfg->arrival_ns) return OR_EINVAL;
  const int S = (1 << K) - 1, nB = cfg->nB;
  int bmax = 0, bmin = 1 << 30;
  for (int bi = 0; bi < nB; ++bi) {
    if (cfg->B[bi] > bmax) bmax = cfg->B[bi];
    if (cfg->B[bi] < bmin) bmin = cfg->B[bi];
  }
  for (int r = 0; r < cfg->nR; ++r)
    for (uint32_t v = 1; v <= (uint32_t)S; ++v) {
      or_serve o = {0, 0, 0, 0, 0};
      int64_t t = 0, head = 0, tail = 0;
      while (head < N) {
        while (tail < N && arrival(cfg, r, tail) <= t) ++tail;
        const int64_t qlen = tail - head;
        int b = 0;  /* the batch size to infer now, 0 = wait */
        int bsel = 0;
        for (int bi = 0; bi < nB; ++bi)
          if (cfg->B[bi] <= qlen && cfg->B[bi] > bsel) bsel = cfg->B[bi];
        int64_t c = 0;
        if (bsel > 0) {
          int bi_sel = 0;
          for (int bi = 0; bi < nB; ++bi) if (cfg->B[bi] == bsel) bi_sel = bi;
          for (int m = 0; m < K; ++m)
            if (((v >> m) & 1u) && cfg->lat_ns[m * nB + bi_sel] > c) c = cfg->lat_ns[m * nB + bi_sel];
        }
        if (qlen >= bmax) {
          b = bmax;  /* bsel == bmax */
        } else if (bsel > 0 && c + (t - arrival(cfg, r, head)) + delta_ns >= cfg->tau_ns) {
          b = bsel;
        }
        if (b > 0) {
          const int64_t done = t + c;
          for (int64_t s = head; s < head + b; ++s) {
            const int64_t l = done - arrival(cfg, r, s);
            o.served++;
            if (l > cfg->tau_ns) { o.overdue++; o.exceed_ns += (uint64_t)(l - cfg->tau_ns); }
          }
          o.batches++;
          head += b;
          t = done;
        } else if (tail == N) {
          if (bsel == 0) { o.unserved = (uint64_t)qlen; break; }
          t = arrival(cfg, r, head) + cfg->tau_ns - delta_ns - c; /* the condition becomes true */
        } else {
          int64_t tn = arrival(cfg, r, tail);
          if (bsel > 0) {
            const int64_t tthr = arrival(cfg, r, head) + cfg->tau_ns - delta_ns - c;
            if (tthr < tn) tn = tthr;
          }
          t = tn;
        }
      }
      out[(int64_t)r * S + (v - 1)] = o;
    }
  return OR_OK;
}

/* ---- NEXT-1: the asynchronous baseline, one model per batch (reading S2) ----------
 * K servers (one per model) share one FIFO queue; no ensemble. Whenever some model is idle at time t, the
 * lowest-index idle model m evaluates Algorithm 3's rule with its own c(m, b): len(q) >= max B -> infer
 * the oldest max B on m; else b = max{b in B : b <= len(q)} and c(m,b) + w(q0) + delta >= tau -> infer the
 * oldest b on m; a dispatched batch occupies m until t + c(m,b) and the loop re-evaluates at the same t
 * (another idle model may take the next batch). Otherwise time advances to the next arrival, the instant
 * the rule becomes true for m, or the instant a lower-index model becomes idle -- the only events that
 * can change the decision; with every model busy, to the earliest completion. Requests still queued
 * (fewer than min B) after the last arrival are unserved. reward = sum over batches of
 * a(m) * (b - beta * overdue) (eq. multi_acc_reward with v = {m}). Output per rate r. */
int or_async_serve(const or_cfg* cfg, int K, int64_t N, int64_t delta_ns, const double* acc, or_serve* out,
                   double* reward, uint64_t* model_batches) {
  if (!cfg || K < 1 || K > 12 || N < 0 || cfg->nB < 1 || !cfg->B || !cfg->lat_ns || cfg->nR < 1) return OR_EINVAL;
  if (!cfg->rates && !cfg->arrival_ns) return OR_EINVAL;
  const int nB = cfg->nB;
  int bmax = 0;
  for (int bi = 0; bi < nB; ++bi) if (cfg->B[bi] > bmax) bmax = cfg->B[bi];
  for (int r = 0; r < cfg->nR; ++r) {
    or_serve o = {0, 0, 0, 0, 0};
    double rew = 0.0;
    int64_t free_at[12];
    for (int m = 0; m < K; ++m) { free_at[m] = 0; if (model_batches) model_batches[(int64_t)r * K + m] = 0; }
    int64_t t = 0, head = 0, tail = 0;
    while (head < N) {
      while (tail < N && arrival(cfg, r, tail) <= t) ++tail;
      int m = -1;
      for (int i = 0; i < K && m < 0; ++i) if (free_at[i] <= t) m = i;
      if (m < 0) { /* every model busy: the next completion */
        int64_t tn = free_at[0];
        for (int i = 1; i < K; ++i) if (free_at[i] < tn) tn = free_at[i];
        t = tn;
        continue;
      }
      const int64_t qlen = tail - head;
      int bsel = 0, bi_sel = -1;
      for (int bi = 0; bi < nB; ++bi)
        if (cfg->B[bi] <= qlen && cfg->B[bi] > bsel) { bsel = cfg->B[bi]; bi_sel = bi; }
      const int64_t c = bi_sel >= 0 ? cfg->lat_ns[m * nB + bi_sel] : 0;
      int b = 0;
      if (qlen >= bmax) b = bmax;
      else if (bsel > 0 && c + (t - arrival(cfg, r, head)) + delta_ns >= cfg->tau_ns) b = bsel;
      if (b > 0) {
        const int64_t done = t + c;
        uint64_t od = 0;
        for (int64_t s = head; s < head + b; ++s) {
          const int64_t l = done - arrival(cfg, r, s);
          o.served++;
          if (l > cfg->tau_ns) { od++; o.exceed_ns += (uint64_t)(l - cfg->tau_ns); }
        }
        o.overdue += od;
        o.batches++;
        if (model_batches) model_batches[(int64_t)r * K + m]++;
        if (acc) rew += acc[m] * ((double)b - cfg->beta * (double)od);
        free_at[m] = done;
        head += b;
        continue; /* same t: the next idle model may dispatch too */
      }
      int64_t tn = INT64_MAX;
      if (tail < N) tn = arrival(cfg, r, tail);
      if (bsel > 0) {
        const int64_t tthr = arrival(cfg, r, head) + cfg->tau_ns - delta_ns - c;
        if (tthr < tn) tn = tthr;
      }
      for (int i = 0; i < m; ++i) if (free_at[i] > t && free_at[i] < tn) tn = free_at[i];
      if (tn == INT64_MAX) { o.unserved = (uint64_t)qlen; break; }
      t = tn;
    }
    out[r] = o;
    if (reward) reward[r] = rew;
  }
  return OR_OK;
}

/* ---- NEXT-2: RL environment and actor-critic gradients (reading S3) ------- */
static void env_features(const or_env* e, int64_t t, int64_t head, const int64_t* free_at, float* x) {
  const int L = e->L, K = e->K, nB = e->nB;
  int64_t tail = head;
  while (tail < e->Narr && e->arrival[tail] <= t) ++tail;
  for (int i = 0; i < L; ++i)
    x[i] = (head + i < tail) ? (float)((double)(t - e->arrival[head + i]) / (double)e->tau_ns) : 0.0f;
  for (int m = 0; m < K; ++m)
    for (int bi = 0; bi < nB; ++bi) x[L + m * nB + bi] = (float)((double)e->lat_ns[m * nB + bi] / (double)e->tau_ns);
  for (int m = 0; m < K; ++m) {
    const int64_t left = free_at[m] > t ? free_at[m] - t : 0;
    x[L + K * nB + m] = (float)((double)left / (double)e->tau_ns);
  }
}

int or_env_rollout(const or_env* e, const int32_t* actions, int n, int64_t h0, float* states, double* rewards,
                   int32_t* overdue, int64_t* t_dec, int64_t* t_start, int64_t* t_done) {
  if (!e || !actions || e->K < 1 || e->K > 12 || h0 < 0 || h0 >= e->Narr) return OR_EINVAL;
  const int K = e->K, nB = e->nB, S = (1 << K) - 1, F = e->L + K * nB + K;
  int64_t free_at[12];
  int64_t t = e->arrival[h0], head = h0;
  for (int m = 0; m < K; ++m) free_at[m] = t;
  for (int st = 0; st < n; ++st) {
    if (states) env_features(e, t, head, free_at, states + (int64_t)st * F);
    const int a = actions[st];
    if (a < 0 || a >= S * nB) return OR_EINVAL;
    const uint32_t v = (uint32_t)(a / nB) + 1u;
    const int bi = a % nB, b = e->B[bi];
    if (head + b > e->Narr) return OR_EINVAL;
    int64_t start = t, c = 0;
    if (e->arrival[head + b - 1] > start) start = e->arrival[head + b - 1];
    for (int m = 0; m < K; ++m)
      if ((v >> m) & 1u) {
        if (free_at[m] > start) start = free_at[m];
        if (e->lat_ns[m * nB + bi] > c) c = e->lat_ns[m * nB + bi];
      }
    const int64_t done = start + c;
    int32_t o = 0;
    for (int64_t s = head; s < head + b; ++s) if (done - e->arrival[s] > e->tau_ns) ++o;
    const double R = e->acc[v - 1] * ((double)b - e->beta * (double)o);
    for (int m = 0; m < K; ++m) if ((v >> m) & 1u) free_at[m] = done;
    if (rewards) rewards[st] = R;
    if (overdue) overdue[st] = o;
    if (t_dec) t_dec[st] = t;
    if (t_start) t_start[st] = start;
    if (t_done) t_done[st] = done;
    head += b;
    int64_t fmin = free_at[0];
    for (int m = 1; m < K; ++m) if (free_at[m] < fmin) fmin = free_at[m];
    t = fmin > start ? fmin : start;
  }
  return OR_OK;
}

int or_ac_grad(int F, int H, int A, const double* P, const float* states, const int32_t* actions,
               const double* rewards, int E, int n, double gamma, double scale, double ent, double* grad,
               double* loss_pi, double* loss_v) {
  if (F < 1 || H < 1 || A < 1 || E < 1 || n < 1 || !P || !states || !actions || !rewards || !grad) return OR_EINVAL;
  const double *W1 = P, *b1 = W1 + (int64_t)H * F, *W2 = b1 + H, *b2 = W2 + (int64_t)A * H;
  const double *V1 = b2 + A, *c1 = V1 + (int64_t)H * F, *v2 = c1 + H, *c2 = v2 + H;
  const int64_t np = (int64_t)H * F + H + (int64_t)A * H + A + (int64_t)H * F + H + H + 1;
  double *gW1 = grad, *gb1 = gW1 + (int64_t)H * F, *gW2 = gb1 + H, *gb2 = gW2 + (int64_t)A * H;
  double *gV1 = gb2 + A, *gc1 = gV1 + (int64_t)H * F, *gv2 = gc1 + H, *gc2 = gv2 + H;
  for (int64_t i = 0; i < np; ++i) grad[i] = 0.0;
  double* x = (double*)malloc(sizeof(double) * F);
  double* h = (double*)malloc(sizeof(double) * H);
  double* hv = (double*)malloc(sizeof(double) * H);
  double* z = (double*)malloc(sizeof(double) * A);
  double* G = (double*)malloc(sizeof(double) * n);
  double* dh = (double*)malloc(sizeof(double) * H);
  const double inv = 1.0 / ((double)E * (double)n);
  double lp = 0.0, lv = 0.0;
  for (int e = 0; e < E; ++e) {
    /* discounted return from each step (eq. eq:J), rewards scaled */
    double g = 0.0;
    for (int t = n - 1; t >= 0; --t) { g = rewards[(int64_t)e * n + t] * scale + gamma * g; G[t] = g; }
    for (int t = 0; t < n; ++t) {
      const float* xs = states + ((int64_t)e * n + t) * F;
      for (int f = 0; f < F; ++f) x[f] = (double)xs[f];
      /* policy forward */
      for (int j = 0; j < H; ++j) {
        double a = b1[j];
        for (int f = 0; f < F; ++f) a += W1[(int64_t)j * F + f] * x[f];
        h[j] = tanh(a);
      }
      double zmax = -INFINITY;
      for (int k = 0; k < A; ++k) {
        double a = b2[k];
        for (int j = 0; j < H; ++j) a += W2[(int64_t)k * H + j] * h[j];
        z[k] = a;
        if (a > zmax) zmax = a;
      }
      double zs = 0.0;
      for (int k = 0; k < A; ++k) zs += exp(z[k] - zmax);
      const double lse = zmax + log(zs);
      /* value forward */
      for (int j = 0; j < H; ++j) {
        double a = c1[j];
        for (int f = 0; f < F; ++f) a += V1[(int64_t)j * F + f] * x[f];
        hv[j] = tanh(a);
      }
      double V = c2[0];
      for (int j = 0; j < H; ++j) V += v2[j] * hv[j];
      const double adv = G[t] - V;  /* actor-critic: R_t - V(s_t) with the return */
      const int at = actions[(int64_t)e * n + t];
      /* policy entropy Hs = -sum_k pi_k log pi_k (the entropy bonus of the PPO objective, X4) */
      double hs = 0.0;
      for (int k = 0; k < A; ++k) hs -= exp(z[k] - lse) * (z[k] - lse);
      lp += (-adv * (z[at] - lse) - ent * hs) * inv;
      lv += (V - G[t]) * (V - G[t]) * inv;
      /* d(-A log pi(a|s))/dz_k = -A (1[k = a] - pi_k); d(-c H)/dz_k = c pi_k (log pi_k + H) */
      for (int j = 0; j < H; ++j) dh[j] = 0.0;
      for (int k = 0; k < A; ++k) {
        const double pk = exp(z[k] - lse);
        const double dz = (-adv * ((k == at ? 1.0 : 0.0) - pk) + ent * pk * ((z[k] - lse) + hs)) * inv;
        gb2[k] += dz;
        for (int j = 0; j < H; ++j) {
          gW2[(int64_t)k * H + j] += dz * h[j];
          dh[j] += dz * W2[(int64_t)k * H + j];
        }
      }
      for (int j = 0; j < H; ++j) {
        const double dp = dh[j] * (1.0 - h[j] * h[j]);
        gb1[j] += dp;
        for (int f = 0; f < F; ++f) gW1[(int64_t)j * F + f] += dp * x[f];
      }
      /* d (V - G)^2 / dV = 2 (V - G) */
      const double dV = 2.0 * (V - G[t]) * inv;
      gc2[0] += dV;
      for (int j = 0; j < H; ++j) {
        gv2[j] += dV * hv[j];
        const double dp = dV * v2[j] * (1.0 - hv[j] * hv[j]);
        gc1[j] += dp;
        for (int f = 0; f < F; ++f) gV1[(int64_t)j * F + f] += dp * x[f];
      }
    }
  }
  if (loss_pi) *loss_pi = lp;
  if (loss_v) *loss_v = lv;
  free(x); free(h); free(hv); free(z); free(G); free(dh);
  return OR_OK;
}
