// rk_internal.h — structures shared between the host orchestration (rk_api.cpp) and the
// CUDA kernels of librk.so. Not part of the public ABI (include/rk.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rk {

constexpr int kMaxK = 12;
constexpr int kMaxB = 8;
constexpr int kMaxR = 8;
constexpr int kVoteThreads = 256;   // vote kernel block size (8 warps)
constexpr int kMaxCFast = 1024;     // register/shared-resident rows up to ldc <= 1024; wider rows: rk_vote_large.cu

#ifdef __CUDACC__
// θ pruning threshold of model `lane`, from the row statistics
// mx = max_c l[m][c] and ls = log sum_c exp(l[m][c] - mx): p[m][c] = exp((l - mx) - ls), so
// p[m][top_m] = exp(-ls) and theta = min_j exp(-ls_j) / K. Returns the logit threshold
// mx + ls + log(theta) of lane m minus a slack that can only ENLARGE the candidate set (fp32 rounding
// of ls, of the sum with mx, and of the comparison). Lanes >= K return garbage and must not use it.
__device__ __forceinline__ float theta_threshold(float mx, float ls, int K, int lane) {
  float th = lane < K ? __expf(-ls) : INFINITY;
  for (int off = 16; off; off >>= 1) th = fminf(th, __shfl_xor_sync(0xffffffffu, th, off));
  const float lth = logf(th / (float)K);
  return mx + (ls + lth) - (1e-3f + 2e-6f * fabsf(mx) + 1e-6f * (fabsf(ls) + fabsf(lth)));
}
#endif

// ---- vote / average / subset-count kernel (steps A2-A5) --------------------------------------
struct VoteParams {
  const float* logits;       // [N][K][ldc]
  int64_t ldc;
  const float* lsum_in;      // [N][K] log sum_c exp(l[c] - rmax), relative to the row max, or null
                             // (then computed here); p[m][c] = exp((l - rmax_m) - lsum_m)
  const int32_t* top1_in;    // [N][K] or null
  const float* rmax_in;      // [N][K] or null (row max, from the GEMM epilogue)
  const float* ly_in;        // [N][K] label logits l[m][y] or null (fused mode: no logits rows exist)
  const float* s2_in;        // [N][K] second-largest logit per row (GEMM epilogue) or null: rows whose top-1 is
                             // y and whose other classes all lie below the theta threshold add only y to the
                             // averaging candidate set, so the averaging kernel skips streaming them
  unsigned int* n_skip;      // with s2_in: number of such rows over the worklist (diagnostic) or null
  unsigned int* dyn_ctr;     // with wrec: zeroed counter from which the averaging kernel's warps grab entries
  uint32_t* wrec;            // K <= 8 logits path: [worklist][kRecWords] records written by the classify kernel
                             // (l[m][y], rmax, lsum, top-1 as u16, n, y) so the averaging kernel's per-sample
                             // inputs arrive in one coalesced load issued a sample ahead; null = read them by n
  int sm_count;
  const int32_t* labels;     // [N] device
  int64_t N;                 // samples in this chunk
  int K, C, S, tie;
  int G;                     // samples per tile (1)
  int gs;                    // samples per count group (power of 2 dividing gcd(B)); 0 = no groups
  int U;                     // samples per unit
  int nW32;                  // ceil(C / 32) candidate-bitmap words
  int CAP;                   // candidate capacity (P matrix in smem)
  int TCAP;                  // candidate capacity of the subset-sum tables in smem
  int K1;                    // low half of the models for the subset-sum tables
  float band;                // relative fp32 near-tie band -> fp64 recheck
  int cta_cols;              // K >= 9: most table columns (y + competitors) of the CTA averaging kernel
  const uint8_t* best_of;    // [2^K] best-ranked model in a mask (device)
  int nB;
  int64_t tail_start[kMaxB]; // local sample index from which a sample is in the tail of B[b]
  // outputs (device)
  unsigned long long* cnt_vote;   // [S]
  unsigned long long* cnt_avg;    // [S]
  unsigned long long* n_recheck;  // [S]
  unsigned long long* tail;       // [nB][S]
  uint8_t* grp;                   // [ceil(N/gs)][S] or null
  float* scratch;                 // per-CTA overflow P [gridDim][G][C][K]
  int32_t* scratch_cls;           // per-CTA overflow class list [gridDim][G][C]
  unsigned int* err;              // [0] non-finite logits, [1] bad label
  int32_t* ovf_work;              // K >= 9: worklist samples whose columns exceed cta_cols (rk_vote_cta_avg.cu) [N]
  unsigned int* ovf_count;
  int32_t* cta_work;              // K >= 9, ldc <= 128: samples the warp kernel hands to the CTA kernel [N]
  unsigned int* cta_count;
  uint64_t* pairs;                // K >= 9, ldc <= 128: near-tie pairs (n << 16 | v) for the fp64 recheck kernel
  unsigned int* pair_count;
  int64_t pair_cap;
};

// warp-per-sample variant for K <= 8, C <= 1024 (rk_vote_warp.cu); uses CAP, TCAP, K1, gs, scratch
size_t vote_warp_smem_per_warp(const VoteParams& p);
int vote_warp_threads();
int vote_warp_min_blocks();
// averaging kernel of the warp path (rk_vote_avg.cu)
size_t vote_avg_smem_per_warp(const VoteParams& p);
cudaError_t launch_vote_avg(const VoteParams& q, int grid, cudaStream_t st, const int32_t* work,
                            const unsigned int* work_count);

// K = 9..12 (rk_vote_batch.cu): the same two-kernel split with a batch-transposed layout (threads
// own subsets, sweep a batch of per-sample records in shared memory).
size_t vote_batch_smem_per_sample(const VoteParams& p);
int vote_batch_avg_ctas_samples();
cudaError_t launch_vote_batch(const VoteParams& p, int sm_count, cudaStream_t st, int32_t* work,
                              unsigned int* work_count, int32_t* st_top, float* st_lsum, float* st_max);
cudaError_t launch_vote_batch_avg(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                                  const unsigned int* work_count);  // rk_vote_batch_avg.cu
// CTA-per-sample averaging with exact tables over every competitor (rk_vote_cta_avg.cu); samples with
// more than 32 competitors are appended to ovf_work for launch_vote_batch_avg.
size_t vote_cta_avg_smem(const VoteParams& q);
cudaError_t launch_vote_cta_avg(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                                const unsigned int* work_count, int32_t* ovf_work, unsigned int* ovf_count);

// Warp-per-sample averaging for K = 9..12 with ldc <= 128 (rk_vote_wsample_avg.cu): samples with more
// than 7 competitors, a near-subnormal label probability or a near-tie go, untouched, to cta_work.
// Near-tie subsets of its samples are appended as (sample, subset) pairs to q.pairs and decided by
// launch_vote_pair_recheck (fp64, one warp per pair, from the definition).
bool vote_wsample_avg_supported(const VoteParams& q);
cudaError_t launch_vote_pair_recheck(const VoteParams& q, int sm_count, cudaStream_t st);
// The samples left for the CTA kernel are returned in (*rest, *rest_count): cta_work, or (K = 12, after
// a second wide pass that consumes cta_work) the reused worklist buffer.
cudaError_t launch_vote_wsample_avg(const VoteParams& q, int sm_count, cudaStream_t st, int32_t* work,
                                    unsigned int* work_count, int32_t* cta_work, unsigned int* cta_count,
                                    const int32_t** rest, const unsigned int** rest_count);

// A4 for rows wider than 1024 classes (any K; rk_vote_large.cu): one CTA per worklist sample, fp64
// from the definition over the candidate set; used instead of the kernels above when ldc > kMaxCFast.
bool vote_large_needed(const VoteParams& q);
cudaError_t launch_vote_large_avg(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                                  const unsigned int* work_count);

// Two kernels: classify+votes over all samples, then averages over the worklist of samples whose
// label is an averaging candidate. work: [N] int32, work_count: 1 uint; st_*: [N][K] statistics
// scratch (written by kernel A when the logits came without statistics).
cudaError_t launch_vote_warp(const VoteParams& p, int grid, cudaStream_t st, int32_t* work, unsigned int* work_count,
                             int32_t* st_top, float* st_lsum, float* st_max, int sm_count);

// NEXT-3 (rk_vote_sparse.cu): averages of the classify kernel's worklist from the fused GEMM's top-kFuseT
// lists (K <= 8); samples whose bounds leave a subset undecided are appended to fb / fb_count.
cudaError_t launch_vote_sparse(const VoteParams& p, const float* ly, const float* tv, const uint16_t* ti,
                               const int32_t* work, const unsigned int* work_count, int32_t* fb,
                               unsigned int* fb_count, int sm_count, cudaStream_t st);
// compact copies of the fallback rows' features and labels (+ the identity worklist 0..M-1)
cudaError_t launch_gather_rows(const uint16_t* X, int D, const int32_t* labels, const int32_t* idx,
                               const unsigned int* count, int64_t M, uint16_t* Xc, int32_t* yc, int32_t* iota,
                               cudaStream_t st);
// kernel A of launch_vote_warp alone (classify + votes + worklist)
cudaError_t launch_vote_classify(const VoteParams& p, cudaStream_t st, int32_t* work, unsigned int* work_count,
                                 int sm_count);

// ---- per-sample predictions for one action v (rk_predict) ---------------------------------------
struct PredictParams {
  const float* logits; int64_t ldc;
  int64_t N; int K, C, tie; uint32_t v;
  const uint8_t* best_of;
  int32_t* pred_vote; int32_t* pred_avg; float* avgprob;
  unsigned int* err;
};
cudaError_t launch_predict(const PredictParams& p, cudaStream_t st);

// ---- batch moments, merge and reward fold (A5 tail, A7) ----------------------------------------
struct MomentParams {
  int K, S, nB, nR;
  int B[kMaxB];
  int64_t lat[kMaxK * kMaxB];     // [K][nB]
  double rates[kMaxR];
  const int64_t* arrival;         // [N] device or null
  int64_t tau, goff, N;           // chunk
  int want_exceed;
  unsigned long long* osum;       // [nR][nB][K] overdue counts per slowest model
  unsigned long long* esum;       // [nR][nB][K]
  const int64_t* fin;             // queue mode: finish time of local batch j: fin[fin_off[bi] + (r*K + m)*nb + j]
  int64_t fin_off[kMaxB];
  uint16_t* ovd;                  // per-batch overdue counts: ovd[ovd_off[bi] + (j*K + m)*ovd_nrp + r], or null
  int64_t ovd_off[kMaxB];
  int ovd_nrp;                    // rates padded to 4 or 8 (ovd_nrp(nR))
};
// elements of the per-batch overdue table for N samples
int ovd_nrp(int nR);
int64_t ovd_elems(int nB, const int* B, int nR, int K, int64_t N, int64_t* off /*[kMaxB] or null*/);
cudaError_t launch_overdue(const MomentParams& p, cudaStream_t st);  // err flags follow esum
// queue mode (reading Q15): finish times of this chunk's complete batches per (b, r, slowest model m)
// by a prefix-max scan, finish_j = (J+1) c + max(carry, max_{i<=j} (t_last(i) - i c)), J global;
// carry [nB][nR][K] holds the running max over earlier chunks (derived from rates when seed_rates).
int64_t fin_elems(int nB, const int* B, int nR, int K, int64_t N, int64_t* off /*[kMaxB] or null*/);
cudaError_t launch_queue_scan(const MomentParams& p, int64_t* fin, int64_t* carry, int seed_rates, cudaStream_t st);

struct QParams {
  int K, S, nB, nR, gs;
  int B[kMaxB];
  int64_t N, L;                   // L = lcm(B)
  const uint8_t* grp;             // [ceil(N/gs)][S] correct votes per group of gs samples
  const uint8_t* slow;            // [nB][S] slowest member of v at batch size b
  const uint16_t* ovd;            // per-batch overdue counts (MomentParams::ovd)
  int64_t ovd_off[kMaxB];
  unsigned long long* Q;          // [nR][nB][S] (table section)
  unsigned long long* cnt_vote;   // [S] or null: also add sum_g grp[g][v] (K >= 9: the vote kernel leaves
                                  // the per-subset totals to this pass when it writes group counts)
};
cudaError_t launch_q(const QParams& p, int sm_count, cudaStream_t st);

struct MergeParams {
  int S, nB, nR;
  const unsigned long long* chunk;  // chunk counters: vote[S], avg[S], rc[S], tail[nB][S], osum, esum
  const uint8_t* slow;              // [nB][S]
  int K;
  unsigned long long* table;        // table sections
  int64_t off_vote, off_avg, off_rc, off_corr, off_O, off_E;
  int want_exceed;
  const unsigned int* err;          // chunk error flags [3] -> table words off_err..off_err+2
  int64_t off_err;
};
cudaError_t launch_merge(const MergeParams& p, int64_t N, int64_t off_N, cudaStream_t st);

struct FoldParams {
  int S, nB, nR;
  int B[kMaxB];
  double beta;
  const unsigned long long* table;
  int64_t off_vote, off_corr, off_O, off_Q, off_N;
  int has_Q;
  double* reward_sur;  // [nR][nB][S]
  double* reward_lab;
};
cudaError_t launch_fold(const FoldParams& p, cudaStream_t st);

// ---- NEXT-1: Algorithm 3 greedy batching per (rate, subset) (rk_serve.cu) -----------------------
struct ServeParams {
  int K, S, nB, nR;
  int B[kMaxB];
  int64_t lat[kMaxK * kMaxB];
  double rates[kMaxR];
  const int64_t* arrival;          // [nR][N] device arrival times (launch_arrival_fill for rates)
  int64_t N, tau, delta;
  double beta;
  const double* acc;               // [S] device a(v) or null
  unsigned long long* out;         // [5][nR][S]: served, overdue, exceed_ns, batches, unserved
  double* reward;                  // [nR][S] or null
  uint32_t v_only;                 // != 0: one scenario (rate 0, subset v_only), results at index 0
  int64_t* sched;                  // v_only: the dispatched batches as (first request, size) pairs, or null
};
cudaError_t launch_greedy_serve(const ServeParams& p, cudaStream_t st);
cudaError_t launch_arrival_fill(const ServeParams& p, int64_t* out /*[nR][N]*/, cudaStream_t st);
// the asynchronous one-model-per-batch baseline (reading S2): one thread per rate; out [5][nR],
// reward [nR] (acc_single [K] device or null), model_batches [nR][K] or null
cudaError_t launch_async_serve(const ServeParams& p, const double* acc_single, unsigned long long* model_batches,
                               cudaStream_t st);

// ---- NEXT-4: the sine-plus-noise arrival process (rk_arrivals.cu, reading Q16) ------
struct SineParams {
  double k, b;          // rate(t) = k sin(2 pi t / T) + b, req/s (eqs. eq:r1 / eq:r2)
  int64_t period;       // T in ns
  int64_t delta;        // simulator invocation interval in ns
  double delta_s;       // delta in seconds (delta / 1e9, one rounding on the host)
  double sigma;         // noise std: phi = sigma * z
  uint64_t seed;
};
int64_t sine_chunk_blocks(int64_t J);
// counts of invocations [j0, j0 + J) into cnt [J], exclusive block offsets into bsum [blocks + 1]
// (bsum[blocks] = the chunk's total)
cudaError_t launch_sine_counts(const SineParams& p, int64_t j0, int64_t J, int64_t* cnt, int64_t* bsum,
                               cudaStream_t st);
cudaError_t launch_sine_scatter(const SineParams& p, int64_t j0, int64_t J, const int64_t* cnt, const int64_t* bsum,
                                int64_t base, int64_t n0, int64_t N, int64_t* out, cudaStream_t st);

// ---- NEXT-2: actor-critic scheduler (rk_rl.cu, reading S3) ----------------
constexpr int kRlMaxH = 64;     // hidden units (register tiles of the gradient kernel)
constexpr int kRlMaxA = 2048;   // actions (2^K - 1) * nB held per warp in shared memory
struct RLParams {
  int K, nB, L, F, H, A, E, n;
  int B[kMaxB];
  int64_t lat[kMaxK * kMaxB];    // [K][nB] ns
  int64_t tau;
  double beta;
  const double* acc;             // [S] a(v), device
  const int64_t* arrival;        // [Narr] device, non-decreasing
  int64_t Narr;
  const float* params;           // flat [W1 | b1 | W2 | b2 | V1 | c1 | v2 | c2]
  const int64_t* h0;             // [E] first request of each episode
  const int32_t* forced;         // [E][n] actions or null (sample from the policy)
  uint64_t seed;
  float* states;                 // [E][n][F]
  int32_t* actions;              // [E][n]
  double* rewards;               // [E][n]
  int32_t* overdue;              // [E][n] or null
  int64_t *t_dec, *t_start, *t_done;  // [E][n] or null
  unsigned int* err;
  double gamma, scale, ent;
};
int64_t ac_param_count(int F, int H, int A);
cudaError_t launch_ac_rollout(const RLParams& p, cudaStream_t st);
size_t ac_grad_scratch_bytes(const RLParams& p);
cudaError_t launch_ac_grad(const RLParams& p, float* grad, float* loss2 /*device [2] or null*/, void* scratch,
                           cudaStream_t st);
cudaError_t launch_ac_apply(float* P, const float* g, int64_t npol, int64_t np, float lr_pi, float lr_v,
                            cudaStream_t st);

constexpr int kRecWords = 32;  // worklist record: [0,8) l[m][y], [8,16) rmax, [16,24) lsum, [24,28) top-1 u16,
                               // 28 n, 29 y, 30 mask of the rows the averaging kernel need not stream (K <= 8)
constexpr int kFuseT = 16;  // NEXT-3: logits kept per (row, model) by the fused GEMM epilogue
constexpr int kFuseNone = 0xFFFF;  // class of a bound-only top-T entry: its value bounds every unlisted class
// ---- GEMM (A1) -----------------------------------------------------------------------------------
struct GemmParams {
  const void* tmap_x;    // CUtensorMap* (host copy passed by value via __grid_constant__)
  const void* tmap_w;
  const void* tmap_out;
  const void* tmap_out16;  // 16-column store boxes (packed mode, Cp <= 128)
  int64_t N;             // rows
  int K, C, Cp, D, ldc;  // Cp = per-model padded columns (multiple of 16)
  int scale_log2;
  const float* bias;     // [K][Cp] (-inf on padding columns)
  int32_t* top1;         // [N][K]
  float* lsum;           // [N][K] log sum_c exp(l - rmax) (relative to the row max)
  float* rmax;           // [N][K] row max (theta of the candidate pruning)
  float* rs2;            // [N][K] second-largest logit (max without one occurrence of rmax), or null;
                         // written by the per-model (Cp > 128) logits epilogue only
  float* logits;         // [N][K][ldc]
  unsigned int* err;
  int cluster;           // 1 = one CTA per 128-row tile; 2 = CTA pair, tcgen05.mma.cta_group::2 on 256-row tiles
  // NEXT-3 fused forward + vote (labels != null; Cp > 128): no logits stored; instead the label's logit
  // ly [N][K] and the kFuseT largest logits per (row, model): tv [N][K][kFuseT] fp32 descending (equal
  // values: lower class first), ti [N][K][kFuseT] classes
  const int32_t* labels;
  float* ly;
  float* tv;
  uint16_t* ti;
};
cudaError_t launch_gemm(const GemmParams& p, int sm_count, cudaStream_t st);
int gemm_build_tmaps(GemmParams& p, const void* X, const void* W, float* logits, void* storage /*4*128B*/);

}  // namespace rk
