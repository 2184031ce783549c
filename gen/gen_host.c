/* gen_host.c — bulk host-side fill of the synthetic inputs defined in rk_gen.h.
 * Multi-threaded over samples (pthreads). Holds no method arithmetic. */
#include "rk_gen.h"
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int kind;
  uint64_t seed;
  int64_t n0, i0, i1;
  int K, C, ldc, D, real;
  uint32_t a, b;
  int64_t p0, p1;
  const int32_t* labels;
  void* out;
} job_t;

enum { J_LABELS, J_LOGITS, J_X, J_W };

static void run_range(const job_t* j) {
  for (int64_t i = j->i0; i < j->i1; ++i) {
    switch (j->kind) {
      case J_LABELS:
        ((int32_t*)j->out)[i] = rkg_label(j->seed, j->n0 + i, j->C);
        break;
      case J_LOGITS: {
        int64_t n = j->n0 + i;
        int y = j->labels ? j->labels[i] : rkg_label(j->seed, n, j->C);
        rkg_logit_params prm = {j->p0, j->p1};
        float* row = (float*)j->out + i * (int64_t)j->K * j->ldc;
        for (int m = 0; m < j->K; ++m) {
          for (int c = 0; c < j->C; ++c) row[(int64_t)m * j->ldc + c] = rkg_logit(j->seed, n, m, c, j->K, y, prm);
          for (int c = j->C; c < j->ldc; ++c) row[(int64_t)m * j->ldc + c] = NAN; /* never read by the method */
        }
        break;
      }
      case J_X: {
        int64_t n = j->n0 + i;
        int y = j->labels ? j->labels[i] : rkg_label(j->seed, n, j->C);
        uint16_t* row = (uint16_t*)j->out + i * (int64_t)j->D;
        for (int d = 0; d < j->D; ++d)
          row[d] = j->real ? rkg_x_real(j->seed, n, d, y, j->a) : rkg_int_to_bf16(rkg_x_int(j->seed, n, d, y, j->a));
        break;
      }
      case J_W: { /* i indexes (m, c) rows of W[K][C][D] */
        int m = (int)(i / j->C), c = (int)(i % j->C);
        uint32_t fq = rkg_flip_q16(m, j->a, j->b);
        uint16_t* row = (uint16_t*)j->out + i * (int64_t)j->D;
        for (int d = 0; d < j->D; ++d)
          row[d] = j->real ? rkg_w_real(j->seed, m, c, d, fq) : rkg_int_to_bf16(rkg_w_int(j->seed, m, c, d, fq));
        break;
      }
    }
  }
}

static void* thr_main(void* p) { run_range((const job_t*)p); return NULL; }

static void run_parallel(job_t base, int64_t count, int threads) {
  if (threads <= 1 || count < 64) { base.i0 = 0; base.i1 = count; run_range(&base); return; }
  if (threads > 256) threads = 256;
  pthread_t th[256];
  job_t jobs[256];
  int64_t per = (count + threads - 1) / threads;
  int started = 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t] = base;
    jobs[t].i0 = t * per;
    jobs[t].i1 = (t + 1) * per < count ? (t + 1) * per : count;
    if (jobs[t].i0 >= jobs[t].i1) break;
    if (pthread_create(&th[t], NULL, thr_main, &jobs[t]) != 0) { run_range(&jobs[t]); continue; }
    started = t + 1;
  }
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

void rkg_fill_labels(uint64_t seed, int64_t n0, int64_t n, int C, int32_t* out, int threads) {
  job_t j; memset(&j, 0, sizeof j);
  j.kind = J_LABELS; j.seed = seed; j.n0 = n0; j.C = C; j.out = out;
  run_parallel(j, n, threads);
}

void rkg_fill_logits(uint64_t seed, int64_t n0, int64_t n, int K, int C, int ldc, int64_t mu0_q24,
                     int64_t dmu_q24, const int32_t* labels, float* out, int threads) {
  job_t j; memset(&j, 0, sizeof j);
  j.kind = J_LOGITS; j.seed = seed; j.n0 = n0; j.K = K; j.C = C; j.ldc = ldc;
  j.p0 = mu0_q24; j.p1 = dmu_q24; j.labels = labels; j.out = out;
  run_parallel(j, n, threads);
}

void rkg_fill_x(uint64_t seed, int64_t n0, int64_t n, int D, int C, uint32_t psig_q16, int real,
                const int32_t* labels, uint16_t* out, int threads) {
  job_t j; memset(&j, 0, sizeof j);
  j.kind = J_X; j.seed = seed; j.n0 = n0; j.D = D; j.C = C; j.a = psig_q16; j.real = real;
  j.labels = labels; j.out = out;
  run_parallel(j, n, threads);
}

void rkg_fill_w(uint64_t seed, int K, int C, int D, uint32_t flip0_q16, uint32_t dflip_q16, int real,
                uint16_t* out, int threads) {
  job_t j; memset(&j, 0, sizeof j);
  j.kind = J_W; j.seed = seed; j.K = K; j.C = C; j.D = D; j.a = flip0_q16; j.b = dflip_q16; j.real = real;
  j.out = out;
  run_parallel(j, (int64_t)K * C, threads);
}

void rkg_fill_bias(uint64_t seed, int K, int C, int real, float* out) {
  for (int m = 0; m < K; ++m)
    for (int c = 0; c < C; ++c) out[(int64_t)m * C + c] = rkg_bias(seed, m, c, real);
}
