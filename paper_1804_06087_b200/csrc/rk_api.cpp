// rk_api.cpp — host orchestration behind the C-ABI in include/rk.h.
//
// Owns the per-rank context: the ensemble copy in HBM, workspaces sized to the largest chunk seen,
// the integer result table, the NCCL communicator for the cross-GPU sum (A6), and the per-kernel
// CUDA-event profiler used by bench.py. Every compute step runs in the CUDA kernels of
// rk_gemm.cu / rk_vote.cu / rk_moments.cu; this file only validates, allocates and launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <thread>
#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a profiler is attached

#include "../../include/rk.h"
#include "rk_internal.h"

namespace {
struct NvtxRange {  // names each C-ABI entry point's host span on the profiler timeline (nsys / ncu --nvtx)
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace rk;

namespace {

enum KernelKind { KK_GEMM = 0, KK_VOTE, KK_OVERDUE, KK_MERGE, KK_Q, KK_FOLD, KK_PREDICT, KK_ALLREDUCE, KK_SERVE,
                  KK_FALLBACK, KK_COUNT };
const char* kKernelNames[KK_COUNT] = {"gemm_heads_tcgen05", "vote_subsets", "overdue_moments", "merge_table",
                                      "labelled_moments", "reward_fold", "predict", "nccl_allreduce", "greedy_serve",
                                      "fused_fallback"};

struct Prof {
  bool on = false;
  struct Ev { cudaEvent_t a, b; int kind; double bytes, flops; };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> pool;
  int64_t launches[KK_COUNT] = {};
  double ms[KK_COUNT] = {}, bytes[KK_COUNT] = {}, flops[KK_COUNT] = {};
};

int64_t gcd64(int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; }

}  // namespace

struct rk_ctx {
  int dev = 0, rank = 0, world = 1, sm_count = 148;
  ncclComm_t comm = nullptr;
  std::string err;
  // ensemble
  bool loaded = false, has_heads = false;
  int K = 0, C = 0, D = 0, S = 0, Cp = 0, ldc = 0, scale_log2 = 0, tie = 0;
  int member_rank[kMaxK] = {};
  uint8_t* d_best_of = nullptr;
  uint16_t* d_W = nullptr;
  float* d_bias = nullptr;
  // last rk_score* batch
  bool have_batch = false, batch_stats = false;
  bool batch_fused = false;            // NEXT-3: rk_score_labelled kept top-T lists instead of logits
  const uint16_t* cur_X = nullptr;     // fused: the batch's features (device), for fallback rows
  const int32_t* cur_labels = nullptr; // fused: device labels of the batch
  const int32_t* cur_labels_arg = nullptr;
  float* d_ly = nullptr; float* d_tv = nullptr; uint16_t* d_ti = nullptr;
  int64_t ly_cap = 0, tv_cap = 0, ti_cap = 0;
  int32_t* d_fb = nullptr; int64_t fb_cap = 0;          // fallback list [N] + count, identity list [N]
  uint16_t* d_xc = nullptr; int64_t xc_cap = 0;         // fallback rows: compact X
  float* d_lc = nullptr; int64_t lc_cap = 0;            // fallback rows: logits
  int32_t* d_tc = nullptr; int64_t tc_cap = 0;          // fallback rows: top1 | labels
  float* d_sc = nullptr; int64_t sc_cap = 0;            // fallback rows: lsum | rmax
  int64_t last_fallback = 0, last_worklist = 0;
  const float* cur_logits = nullptr;
  int64_t cur_ldc = 0, cur_N = 0, cur_off = 0;
  // GEMM workspaces
  float* ws_logits = nullptr;
  int32_t* ws_top1 = nullptr;
  float* ws_lsum = nullptr;
  float* ws_max = nullptr;
  int64_t ws_cap = 0, ws_top1_cap = 0, ws_lsum_cap = 0, ws_max_cap = 0;
  float* ws_s2 = nullptr;      // [N][K] second-largest logit per row (per-model epilogue, Cp > 128)
  int64_t ws_s2_cap = 0;
  bool cur_s2 = false;         // the last rk_score wrote ws_s2
  bool last_skip_valid = false;  // the last accumulate counted skipped rows (K <= 8 logits path, ldc <= 1024)
  uint16_t* ws_x = nullptr;
  int64_t ws_x_cap = 0;
  alignas(64) uint8_t tmaps[4 * 128];
  int cta_cols = 52;                   // K >= 9 CTA averaging: column capacity (env RK_CTA_AVG_COLS, tests)
  int64_t pair_cap_test = 0;           // K >= 9: near-tie pair list capacity override (env RK_PAIR_CAP, tests)
  int gemm_cluster = 2;                // head GEMM: 2 = CTA pair (tcgen05 cta_group::2, M = 256), 1 = single CTA (env RK_GEMM_CLUSTER)
  cudaStream_t copy_stream = nullptr;  // H2D of host X, overlapped with the GEMM
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> ev_chunks;
  // accumulation state
  bool reset_done = false, final_seen = false;
  // rk_subset_reset has no stream: its device work (table zeroing, the slowest-member and backlog-carry
  // uploads) is deferred to the next accumulate / finalize and issued on that call's stream, so a reset
  // never synchronises the device (a previous chunk's GEMM may still be running on another stream)
  bool reset_pending = false;
  std::vector<uint8_t> h_slow;
  std::vector<int64_t> h_qcarry;
  size_t slow_cap = 0, qcarry_cap = 0;
  bool finalized = false;      // the table holds the global sum (A6 done): no more accumulate / all-reduce
  double nccl_timeout_s = 600; // bounded wait on the all-reduce (env RK_NCCL_TIMEOUT_S)
  bool has_cfg = false;
  int nB = 0, nR = 0, want_exceed = 0, want_labelled = 0;
  int B[kMaxB] = {};
  int64_t lat[kMaxK * kMaxB] = {};
  double rates[kMaxR] = {};
  double beta = 0;
  int64_t tau = 0;
  const int64_t* arrival_user = nullptr;
  int64_t L = 1;       // lcm(B)
  int gs = 0;          // group size for labelled moments
  unsigned long long* d_table = nullptr;
  size_t table_words = 0;
  int64_t off_N = 0, off_err = 1, off_vote = 0, off_avg = 0, off_rc = 0, off_corr = 0, off_O = 0, off_Q = 0, off_E = 0;
  unsigned long long* d_chunk = nullptr;
  size_t chunk_words = 0;
  uint8_t* d_slow = nullptr;
  uint8_t* d_grp = nullptr;
  size_t grp_cap = 0;
  uint16_t* d_ovd = nullptr;  // per-batch overdue counts (labelled moments)
  size_t ovd_cap = 0;
  int queue = 0;               // reading Q15 (FIFO ensemble server)
  int64_t* d_fin = nullptr;    // queue mode: finish times of the chunk's batches
  size_t fin_cap = 0;
  int64_t* d_qcarry = nullptr; // queue mode: running max of t_last(i) - i c per (b, r, m)
  uint64_t* d_serve = nullptr; // greedy serving outputs
  int64_t serve_cap = 0;
  bool q_started = false;
  int64_t q_next_off = 0;
  int32_t* d_labels = nullptr;
  int64_t labels_cap = 0;
  int32_t* d_work = nullptr;  // vote worklist [N] + count
  int64_t work_cap = 0;
  uint32_t* d_wrec = nullptr;  // K <= 8 logits path: worklist records [N][kRecWords]
  int64_t wrec_cap = 0;
  void* h_stage = nullptr;     // page-locked host staging of the finalized table and rewards (grow-only)
  size_t h_stage_bytes = 0;
  uint64_t* d_pairs = nullptr;  // K >= 9: near-tie (sample, subset) pairs for the fp64 recheck kernel
  int64_t pairs_cap = 0;
  int64_t* d_arr = nullptr;
  int64_t arr_cap = 0;
  float* d_scratch = nullptr;
  int32_t* d_scratch_cls = nullptr;
  size_t scratch_floats = 0, scratch_ints = 0;
  double* d_rew = nullptr;
  size_t rew_cap = 0;
  int64_t chunks = 0;
  int64_t grp_groups = 0;      // group counts of the last accumulated chunk: ceil(N/gs) rows of S bytes
  int grp_gs = 0;
  Prof prof;
};

namespace {

rk_status fail(rk_ctx* c, rk_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}
#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess) return fail(ctx, RK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
rk_status ensure(rk_ctx* ctx, T** p, int64_t* cap, int64_t need) {
  if (*cap >= need && *p) return RK_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  if (cudaMalloc((void**)p, sizeof(T) * std::max<int64_t>(need, 1)) != cudaSuccess)
    return fail(ctx, RK_ENOMEM, "cudaMalloc failed (" + std::to_string(sizeof(T) * need) + " bytes)");
  *cap = need;
  return RK_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Begin / end a profiled launch on stream st.
struct ProfScope {
  rk_ctx* c; int kind; cudaStream_t st; double bytes, flops; cudaEvent_t a = nullptr;
  ProfScope(rk_ctx* c_, int k, cudaStream_t s, double by, double fl) : c(c_), kind(k), st(s), bytes(by), flops(fl) {
    c->prof.launches[kind]++;
    if (!c->prof.on) return;
    a = take();
    cudaEventRecord(a, st);
  }
  cudaEvent_t take() {
    if (!c->prof.pool.empty()) { cudaEvent_t e = c->prof.pool.back(); c->prof.pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
  }
  ~ProfScope() {
    if (!c->prof.on || !a) return;
    cudaEvent_t b = take();
    cudaEventRecord(b, st);
    c->prof.pending.push_back({a, b, kind, bytes, flops});
  }
};

void prof_collect(rk_ctx* c) {
  for (auto& e : c->prof.pending) {
    cudaEventSynchronize(e.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    c->prof.ms[e.kind] += ms;
    c->prof.bytes[e.kind] += e.bytes;
    c->prof.flops[e.kind] += e.flops;
    c->prof.pool.push_back(e.a);
    c->prof.pool.push_back(e.b);
  }
  c->prof.pending.clear();
}

// Wait for `st` (which holds the table all-reduce) while polling the communicator: a peer failure
// (ncclCommGetAsyncError) or a wait longer than nccl_timeout_s aborts the communicator -> RK_ENCCL.
rk_status wait_nccl(rk_ctx* ctx, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return RK_OK;
    if (q != cudaErrorNotReady) return fail(ctx, RK_ECUDA, std::string("stream: ") + cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(ctx->comm, &ar) != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
      ncclCommAbort(ctx->comm);
      ctx->comm = nullptr;
      return fail(ctx, RK_ENCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > ctx->nccl_timeout_s) {
      ncclCommAbort(ctx->comm);
      ctx->comm = nullptr;
      return fail(ctx, RK_ENCCL, "all-reduce did not complete within RK_NCCL_TIMEOUT_S (peer lost?)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(el < 0.01 ? 5 : 200));
  }
}

}  // namespace

extern "C" {

const char* rk_status_string(rk_status s) {
  switch (s) {
    case RK_OK: return "RK_OK";
    case RK_EINVAL: return "RK_EINVAL";
    case RK_ESTATE: return "RK_ESTATE";
    case RK_ENOMEM: return "RK_ENOMEM";
    case RK_ECUDA: return "RK_ECUDA";
    case RK_ENCCL: return "RK_ENCCL";
    case RK_ELABEL: return "RK_ELABEL";
    case RK_ENONFINITE: return "RK_ENONFINITE";
    case RK_EUNSUPPORTED: return "RK_EUNSUPPORTED";
  }
  return "RK_?";
}

const char* rk_last_error(const rk_ctx* c) { return c ? c->err.c_str() : "null context"; }

rk_status rk_nccl_unique_id(void* out128) {
  if (!out128) return RK_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RK_ENCCL;
  memcpy(out128, &id, sizeof(id));
  return RK_OK;
}

rk_status rk_create(rk_ctx** out, int cuda_device, const void* nccl_unique_id, int rank, int world) {
  if (!out || world < 1 || rank < 0 || rank >= world) return RK_EINVAL;
  if (world > 1 && !nccl_unique_id) return RK_EINVAL;
  *out = nullptr;
  rk_ctx* ctx = new rk_ctx();
  ctx->dev = cuda_device;
  ctx->rank = rank;
  ctx->world = world;
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) { delete ctx; return RK_ECUDA; }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
  if (const char* gc = getenv("RK_GEMM_CLUSTER")) ctx->gemm_cluster = atoi(gc) == 1 ? 1 : 2;
  // tests only: a smaller column capacity of the K >= 9 CTA averaging kernel routes more samples through
  // the overflow kernel (rk_vote_batch_avg.cu), so both paths stay covered
  if (const char* cc = getenv("RK_CTA_AVG_COLS")) ctx->cta_cols = std::max(4, std::min(52, atoi(cc) / 4 * 4));
  // tests only: a tiny near-tie pair list makes the warp averaging kernel hand whole samples to the CTA kernel
  if (const char* pc = getenv("RK_PAIR_CAP")) ctx->pair_cap_test = std::max(1, atoi(pc));
  if (const char* to = getenv("RK_NCCL_TIMEOUT_S")) ctx->nccl_timeout_s = std::max(0.001, atof(to));
  if (nccl_unique_id) {  // world ranks (world may be 1: a one-rank communicator, same code path)
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    if (ncclCommInitRank(&ctx->comm, world, id, rank) != ncclSuccess) { delete ctx; return RK_ENCCL; }
  }
  *out = ctx;
  return RK_OK;
}

void rk_destroy(rk_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->dev);
  cudaDeviceSynchronize();
  void* ptrs[] = {ctx->d_ly, ctx->d_tv, ctx->d_ti, ctx->d_fb, ctx->d_xc, ctx->d_lc, ctx->d_tc, ctx->d_sc,
                  ctx->d_best_of, ctx->d_W, ctx->d_bias, ctx->ws_logits, ctx->ws_top1, ctx->ws_lsum, ctx->ws_max, ctx->ws_s2, ctx->ws_x,
                  ctx->d_table, ctx->d_chunk, ctx->d_slow, ctx->d_grp, ctx->d_ovd, ctx->d_fin, ctx->d_qcarry, ctx->d_serve, ctx->d_labels, ctx->d_work, ctx->d_wrec, ctx->d_pairs, ctx->d_arr, ctx->d_scratch,
                  ctx->d_scratch_cls, ctx->d_rew};
  for (void* p : ptrs) if (p) cudaFree(p);
  for (auto& e : ctx->prof.pending) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  for (auto e : ctx->prof.pool) cudaEventDestroy(e);
  for (auto e : ctx->ev_chunks) cudaEventDestroy(e);
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  delete ctx;
}

rk_status rk_load_ensemble(rk_ctx* ctx, int K, int C, int D, const void* W_bf16, const float* bias,
                           int logit_scale_log2, const int* member_rank, rk_tie_mode tie) {
  NvtxRange nvtx_("rk_load_ensemble");
  if (!ctx) return RK_EINVAL;
  if (K < 1 || K > kMaxK) return fail(ctx, RK_EINVAL, "K must be in [1,12]");
  if (C < 2 || C > 65535) return fail(ctx, RK_EINVAL, "C must be in [2,65535]");
  if (tie != RK_TIE_BEST_MEMBER && tie != RK_TIE_LOWEST_CLASS) return fail(ctx, RK_EINVAL, "bad tie mode");
  if (W_bf16 && (D <= 0 || D % 64 != 0 || D > 16384)) return fail(ctx, RK_EINVAL, "D must be a positive multiple of 64 (<= 16384)");
  if (logit_scale_log2 < -60 || logit_scale_log2 > 60) return fail(ctx, RK_EINVAL, "scale out of range");
  int rk_[kMaxK];
  bool seen[kMaxK] = {};
  for (int m = 0; m < K; ++m) {
    rk_[m] = member_rank ? member_rank[m] : m;
    if (rk_[m] < 0 || rk_[m] >= K || seen[rk_[m]]) return fail(ctx, RK_EINVAL, "member_rank must be a permutation of 0..K-1");
    seen[rk_[m]] = true;
  }
  CK(cudaSetDevice(ctx->dev));
  const int Cp = (C + 15) / 16 * 16;
  const size_t wrows = (size_t)K * Cp;
  // Validate and stage everything BEFORE touching the context: on any failure the previously loaded
  // ensemble (and the state built on it) stays intact.
  std::vector<float> hb;
  if (W_bf16) {
    hb.assign(wrows, -INFINITY);  // padding columns: -inf never wins the max, exp -> 0
    std::vector<float> ub;
    if (bias) {
      ub.resize((size_t)K * C);
      CK(cudaMemcpy(ub.data(), bias, ub.size() * 4, is_device_ptr(bias) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    }
    for (int m = 0; m < K; ++m)
      for (int c = 0; c < C; ++c) {
        const float b = bias ? ub[(size_t)m * C + c] : 0.f;
        if (!(b == b) || b == INFINITY || b == -INFINITY) return fail(ctx, RK_ENONFINITE, "bias must be finite");
        hb[(size_t)m * Cp + c] = b;
      }
  }
  // best_of[mask] = member of `mask` with the smallest rank ("the model with the best accuracy")
  std::vector<uint8_t> best(size_t(1) << K, 0);
  for (uint32_t msk = 1; msk < (1u << K); ++msk) {
    int b = -1;
    for (int m = 0; m < K; ++m)
      if (((msk >> m) & 1u) && (b < 0 || rk_[m] < rk_[b])) b = m;
    best[msk] = (uint8_t)b;
  }
  uint8_t* n_best = nullptr;
  uint16_t* n_W = nullptr;
  float* n_bias = nullptr;
  auto undo = [&](rk_status st, const std::string& msg) {
    if (n_best) cudaFree(n_best);
    if (n_W) cudaFree(n_W);
    if (n_bias) cudaFree(n_bias);
    return fail(ctx, st, msg);
  };
#define CKU(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return undo(RK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
  CKU(cudaMalloc(&n_best, best.size()));
  CKU(cudaMemcpy(n_best, best.data(), best.size(), cudaMemcpyHostToDevice));
  if (W_bf16) {
    // pad each model's C rows to Cp (zero rows) and its bias to -inf, so tiles never mix models
    CKU(cudaMalloc(&n_W, wrows * D * 2));
    CKU(cudaMemset(n_W, 0, wrows * D * 2));
    const bool wdev = is_device_ptr(W_bf16);
    CKU(cudaMemcpy2D(n_W, (size_t)Cp * D * 2, W_bf16, (size_t)C * D * 2, (size_t)C * D * 2, K,
                     wdev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    CKU(cudaMalloc(&n_bias, wrows * 4));
    CKU(cudaMemcpy(n_bias, hb.data(), wrows * 4, cudaMemcpyHostToDevice));
  }
#undef CKU
  // commit
  if (ctx->d_best_of) cudaFree(ctx->d_best_of);
  if (ctx->d_W) cudaFree(ctx->d_W);
  if (ctx->d_bias) cudaFree(ctx->d_bias);
  ctx->d_best_of = n_best; ctx->d_W = n_W; ctx->d_bias = n_bias;
  ctx->K = K; ctx->C = C; ctx->D = W_bf16 ? D : 0; ctx->S = (1 << K) - 1; ctx->tie = tie;
  ctx->ldc = (C + 3) / 4 * 4;
  ctx->Cp = Cp;
  ctx->scale_log2 = logit_scale_log2;
  memcpy(ctx->member_rank, rk_, sizeof(rk_));
  ctx->has_heads = W_bf16 != nullptr;
  ctx->loaded = true;
  ctx->have_batch = false;   // workspaces and tables were sized for the old ensemble:
  ctx->reset_done = false;   // rk_score* and rk_subset_reset must run again
  ctx->finalized = false;
  return RK_OK;
}

// A1+A2 over N rows; dlabels (device) != null -> the fused epilogue (NEXT-3): no logits, top-T lists.
static rk_status score_impl(rk_ctx* ctx, const void* X, int64_t N, int64_t goff, cudaStream_t st,
                            const int32_t* dlabels) {
  CK(cudaSetDevice(ctx->dev));
  rk_status s;
  const bool fused = dlabels != nullptr;
  if (!fused && (s = ensure(ctx, &ctx->ws_logits, &ctx->ws_cap, std::max<int64_t>(N, 1) * ctx->K * ctx->ldc)) != RK_OK) return s;
  if ((s = ensure(ctx, &ctx->ws_top1, &ctx->ws_top1_cap, std::max<int64_t>(N, 1) * ctx->K)) != RK_OK) return s;
  if ((s = ensure(ctx, &ctx->ws_lsum, &ctx->ws_lsum_cap, std::max<int64_t>(N, 1) * ctx->K)) != RK_OK) return s;
  if ((s = ensure(ctx, &ctx->ws_max, &ctx->ws_max_cap, std::max<int64_t>(N, 1) * ctx->K)) != RK_OK) return s;
  const bool want_s2 = !fused && ctx->Cp > 128;  // per-model epilogue: the averaging kernel's row skipping
  if (want_s2 && (s = ensure(ctx, &ctx->ws_s2, &ctx->ws_s2_cap, std::max<int64_t>(N, 1) * ctx->K)) != RK_OK) return s;
  if (fused) {
    if ((s = ensure(ctx, &ctx->d_ly, &ctx->ly_cap, std::max<int64_t>(N, 1) * ctx->K)) != RK_OK) return s;
    if ((s = ensure(ctx, &ctx->d_tv, &ctx->tv_cap, std::max<int64_t>(N, 1) * ctx->K * kFuseT)) != RK_OK) return s;
    if ((s = ensure(ctx, &ctx->d_ti, &ctx->ti_cap, std::max<int64_t>(N, 1) * ctx->K * kFuseT)) != RK_OK) return s;
  }
  ctx->cur_logits = fused ? nullptr : ctx->ws_logits;
  ctx->cur_s2 = want_s2;
  ctx->cur_ldc = ctx->ldc;
  ctx->cur_N = N;
  ctx->cur_off = goff;
  ctx->batch_stats = true;
  ctx->batch_fused = fused;
  ctx->have_batch = true;
  if (N == 0) return RK_OK;
  // Host X: the H2D copy of chunk i+1 (copy stream) overlaps the GEMM of chunk i (caller stream).
  // Device X: one launch over all rows.
  const bool host = !is_device_ptr(X);
  const int64_t chunk = host ? std::max<int64_t>(65536, ((N + 7) / 8 + 127) / 128 * 128) : N;
  if (host) {
    if ((s = ensure(ctx, &ctx->ws_x, &ctx->ws_x_cap, N * ctx->D)) != RK_OK) return s;
    if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    if (!ctx->ev_start) CK(cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->ev_start, st));  // copies must not overwrite ws_x still read by earlier work
    CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_start, 0));
  }
  // Host X: the last chunk's GEMM runs after its copy, exposed; the final `chunk` rows therefore go in
  // quarter-size pieces (at least 16,384 rows) so that only a short GEMM trails the last copy
  const int64_t tail0 = host ? std::max<int64_t>(0, N - chunk) : N;
  const int64_t piece = host ? std::max<int64_t>(16384, (chunk / 4 + 127) / 128 * 128) : N;
  for (int64_t r0 = 0, ci = 0, n = 0; r0 < N; r0 += n, ++ci) {
    n = std::min(r0 >= tail0 ? piece : std::min(chunk, tail0 - r0), N - r0);
    const void* Xd = X;
    if (host) {
      uint16_t* dst = ctx->ws_x + r0 * ctx->D;
      CK(cudaMemcpyAsync(dst, static_cast<const uint16_t*>(X) + r0 * ctx->D, (size_t)n * ctx->D * 2,
                         cudaMemcpyHostToDevice, ctx->copy_stream));
      if ((int64_t)ctx->ev_chunks.size() <= ci) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->ev_chunks.push_back(e);
      }
      CK(cudaEventRecord(ctx->ev_chunks[ci], ctx->copy_stream));
      CK(cudaStreamWaitEvent(st, ctx->ev_chunks[ci], 0));
      Xd = dst;
    } else {
      Xd = static_cast<const uint16_t*>(X) + r0 * ctx->D;
    }
    GemmParams gp{};
    gp.N = n; gp.K = ctx->K; gp.C = ctx->C; gp.Cp = ctx->Cp; gp.D = ctx->D; gp.ldc = ctx->ldc;
    gp.scale_log2 = ctx->scale_log2; gp.bias = ctx->d_bias;
    gp.cluster = ctx->gemm_cluster;
    gp.top1 = ctx->ws_top1 + r0 * ctx->K; gp.lsum = ctx->ws_lsum + r0 * ctx->K; gp.rmax = ctx->ws_max + r0 * ctx->K;
    gp.rs2 = want_s2 ? ctx->ws_s2 + r0 * ctx->K : nullptr;
    if (fused) {
      gp.labels = dlabels + r0;
      gp.ly = ctx->d_ly + r0 * ctx->K;
      gp.tv = ctx->d_tv + r0 * ctx->K * kFuseT;
      gp.ti = ctx->d_ti + r0 * ctx->K * kFuseT;
      gp.logits = gp.tv;  // the logits tensor map is encoded but never used by the fused epilogue
    } else {
      gp.logits = ctx->ws_logits + r0 * ctx->K * ctx->ldc;
    }
    int rc = gemm_build_tmaps(gp, Xd, ctx->d_W, gp.logits, ctx->tmaps);  // maps are passed by value
    if (rc != 0) return fail(ctx, RK_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(rc) + ")");
    const double flops = 2.0 * n * ctx->D * (double)ctx->K * ctx->C;
    const double bytes = (double)n * ctx->D * 2 + (fused ? (double)n * ctx->K * (kFuseT * 6 + 16) : (double)n * ctx->K * ctx->C * 4);
    ProfScope ps(ctx, KK_GEMM, st, bytes, flops);
    CK(launch_gemm(gp, ctx->sm_count, st));
  }
  ctx->cur_X = host ? ctx->ws_x : static_cast<const uint16_t*>(X);
  return RK_OK;
}

static bool fused_supported(const rk_ctx* ctx) {
  return ctx->K <= 8 && ctx->Cp > 128 && ctx->ldc <= kMaxCFast && ctx->C <= 65535;
}

rk_status rk_score(rk_ctx* ctx, const void* X, int64_t N, int64_t goff, void* stream) {
  NvtxRange nvtx_("rk_score");
  if (!ctx) return RK_EINVAL;
  if (!ctx->loaded || !ctx->has_heads) return fail(ctx, RK_ESTATE, "no heads loaded (rk_load_ensemble with W)");
  if (N < 0 || goff < 0 || (N > 0 && !X)) return fail(ctx, RK_EINVAL, "bad X / N / offset");
  if (N > INT32_MAX) return fail(ctx, RK_EINVAL, "N per call must be < 2^31 (stream larger sets in chunks)");
  ctx->cur_labels_arg = nullptr;
  return score_impl(ctx, X, N, goff, (cudaStream_t)stream, nullptr);
}

rk_status rk_score_labelled(rk_ctx* ctx, const void* X, const int32_t* labels, int64_t N, int64_t goff, void* stream) {
  NvtxRange nvtx_("rk_score_labelled");
  if (!ctx) return RK_EINVAL;
  if (!ctx->loaded || !ctx->has_heads) return fail(ctx, RK_ESTATE, "no heads loaded (rk_load_ensemble with W)");
  if (N < 0 || goff < 0 || (N > 0 && (!X || !labels))) return fail(ctx, RK_EINVAL, "bad X / labels / N / offset");
  if (N > INT32_MAX) return fail(ctx, RK_EINVAL, "N per call must be < 2^31 (stream larger sets in chunks)");
  cudaStream_t st = (cudaStream_t)stream;
  if (!fused_supported(ctx)) {  // K > 8 or <= 128 classes: the logits path (same results)
    rk_status s = score_impl(ctx, X, N, goff, st, nullptr);
    ctx->cur_labels_arg = labels;
    return s;
  }
  CK(cudaSetDevice(ctx->dev));
  const int32_t* dl = labels;
  if (N > 0 && !is_device_ptr(labels)) {
    rk_status s;
    if ((s = ensure(ctx, &ctx->d_labels, &ctx->labels_cap, N)) != RK_OK) return s;
    CK(cudaMemcpyAsync(ctx->d_labels, labels, N * 4, cudaMemcpyHostToDevice, st));
    dl = ctx->d_labels;
  }
  rk_status s = N > 0 ? score_impl(ctx, X, N, goff, st, dl) : score_impl(ctx, X, N, goff, st, nullptr);
  ctx->cur_labels = dl;
  ctx->cur_labels_arg = labels;
  return s;
}

rk_status rk_score_logits(rk_ctx* ctx, const float* logits, int ldc, int64_t N, int64_t goff, void* stream) {
  NvtxRange nvtx_("rk_score_logits");
  (void)stream;
  if (!ctx) return RK_EINVAL;
  if (!ctx->loaded) return fail(ctx, RK_ESTATE, "rk_load_ensemble first");
  if (N < 0 || goff < 0 || ldc < ctx->C || ldc % 4 != 0) return fail(ctx, RK_EINVAL, "bad ldc / N / offset (ldc % 4 == 0, ldc >= C)");
  if (N > INT32_MAX) return fail(ctx, RK_EINVAL, "N per call must be < 2^31 (stream larger sets in chunks)");
  if (N > 0 && (!logits || (reinterpret_cast<uintptr_t>(logits) & 15))) return fail(ctx, RK_EINVAL, "logits must be 16-byte aligned");
  if (N > 0 && !is_device_ptr(logits)) return fail(ctx, RK_EINVAL, "logits must be device memory");
  ctx->cur_logits = logits;
  ctx->cur_ldc = ldc;
  ctx->cur_N = N;
  ctx->cur_off = goff;
  ctx->cur_s2 = false;
  ctx->batch_stats = false;
  ctx->batch_fused = false;
  ctx->cur_labels_arg = nullptr;
  ctx->have_batch = true;
  return RK_OK;
}

rk_status rk_subset_reset(rk_ctx* ctx, const rk_reward_cfg* cfg) {
  NvtxRange nvtx_("rk_subset_reset");
  if (!ctx) return RK_EINVAL;
  if (!ctx->loaded) return fail(ctx, RK_ESTATE, "rk_load_ensemble first");
  CK(cudaSetDevice(ctx->dev));
  const int K = ctx->K, S = ctx->S;
  ctx->has_cfg = cfg != nullptr;
  ctx->nB = ctx->nR = ctx->want_exceed = ctx->want_labelled = 0;
  ctx->L = 1;
  ctx->gs = 0;
  ctx->arrival_user = nullptr;
  ctx->beta = 0; ctx->tau = 0;
  ctx->queue = 0;
  ctx->q_started = false;
  ctx->q_next_off = 0;
  if (cfg) {
    if (cfg->nB < 0 || cfg->nB > kMaxB || (cfg->nB > 0 && (!cfg->B || !cfg->lat_ns))) return fail(ctx, RK_EINVAL, "nB in [0,8] with B and lat_ns");
    if (cfg->arrival_ns && cfg->nR != 1) return fail(ctx, RK_EINVAL, "arrival_ns requires nR == 1");
    if (cfg->nR < 0 || cfg->nR > kMaxR || (cfg->nR > 0 && !cfg->rates && !cfg->arrival_ns)) return fail(ctx, RK_EINVAL, "nR in [0,8] with rates");
    if (cfg->tau_ns < 0 || !(cfg->beta == cfg->beta)) return fail(ctx, RK_EINVAL, "tau >= 0, finite beta");
    ctx->nB = cfg->nB;
    ctx->nR = cfg->nB > 0 ? cfg->nR : 0;
    ctx->beta = cfg->beta;
    ctx->tau = cfg->tau_ns;
    ctx->want_exceed = cfg->want_exceed ? 1 : 0;
    ctx->want_labelled = cfg->want_labelled ? 1 : 0;
    ctx->arrival_user = cfg->arrival_ns;
    ctx->queue = cfg->queue ? 1 : 0;
    int64_t g = 0;
    for (int i = 0; i < cfg->nB; ++i) {
      if (cfg->B[i] < 1 || cfg->B[i] > 4096) return fail(ctx, RK_EINVAL, "batch sizes in [1,4096]");
      ctx->B[i] = cfg->B[i];
      ctx->L = ctx->L / gcd64(ctx->L, cfg->B[i]) * cfg->B[i];
      g = gcd64(g, cfg->B[i]);
      if (ctx->L > 4096) return fail(ctx, RK_EINVAL, "lcm(B) must be <= 4096");
      for (int m = 0; m < K; ++m) {
        if (cfg->lat_ns[m * cfg->nB + i] < 0) return fail(ctx, RK_EINVAL, "latencies must be >= 0");
        ctx->lat[m * cfg->nB + i] = cfg->lat_ns[m * cfg->nB + i];
      }
    }
    for (int r = 0; r < ctx->nR; ++r) {
      const double rt = cfg->arrival_ns ? 1.0 : cfg->rates[r];
      if (!(rt > 0) || rt > 1e12) return fail(ctx, RK_EINVAL, "rates must be > 0");
      ctx->rates[r] = rt;
    }
    if (g > 0) {
      int gs = 1;
      while (gs < 16 && g % (gs * 2) == 0) gs *= 2;
      ctx->gs = gs;
    }
  }
  const int nB = ctx->nB, nR = ctx->nR;
  // table layout (u64 words): N, err[3], vote[S], avg[S], rc[S], corr[nB][S], O, Q, E [nR][nB][S]
  ctx->off_N = 0; ctx->off_err = 1;
  ctx->off_vote = 4;
  ctx->off_avg = ctx->off_vote + S;
  ctx->off_rc = ctx->off_avg + S;
  ctx->off_corr = ctx->off_rc + S;
  ctx->off_O = ctx->off_corr + (int64_t)nB * S;
  ctx->off_Q = ctx->off_O + (int64_t)nR * nB * S;
  ctx->off_E = ctx->off_Q + (int64_t)nR * nB * S;
  const size_t words = (size_t)(ctx->off_E + (int64_t)nR * nB * S);
  if (ctx->table_words < words) {
    if (ctx->d_table) cudaFree(ctx->d_table);
    ctx->d_table = nullptr;
    CK(cudaMalloc(&ctx->d_table, words * 8));
    ctx->table_words = words;
  }
  // chunk counters: vote, avg, rc [S], tail [nB][S], osum, esum [nR][nB][K], err (4 x u32 = 2 words)
  const size_t cw = 3 * (size_t)S + (size_t)nB * S + 2 * (size_t)nR * nB * K + 2;
  if (ctx->chunk_words < cw) {
    if (ctx->d_chunk) cudaFree(ctx->d_chunk);
    ctx->d_chunk = nullptr;
    CK(cudaMalloc(&ctx->d_chunk, cw * 8));
    ctx->chunk_words = cw;
  }
  // slowest member of each subset at each batch size (PAPER.md:410 stragglers)
  ctx->h_slow.clear();
  if (nB > 0) {
    ctx->h_slow.resize((size_t)nB * S);
    for (int bi = 0; bi < nB; ++bi)
      for (uint32_t v = 1; v <= (uint32_t)S; ++v) {
        int sm = -1;
        for (int m = 0; m < K; ++m)
          if (((v >> m) & 1u) && (sm < 0 || ctx->lat[m * nB + bi] > ctx->lat[sm * nB + bi])) sm = m;
        ctx->h_slow[(size_t)bi * S + v - 1] = (uint8_t)sm;
      }
    if (ctx->slow_cap < ctx->h_slow.size()) {  // grow-only allocations (a cudaFree would synchronise)
      if (ctx->d_slow) cudaFree(ctx->d_slow);
      ctx->d_slow = nullptr;
      CK(cudaMalloc(&ctx->d_slow, ctx->h_slow.size()));
      ctx->slow_cap = ctx->h_slow.size();
    }
  }
  ctx->h_qcarry.clear();
  if (ctx->queue && nB > 0 && nR > 0) {  // backlog carry per (b, r, m): empty server
    ctx->h_qcarry.assign((size_t)nB * nR * K, INT64_MIN / 4);
    if (ctx->qcarry_cap < ctx->h_qcarry.size()) {
      if (ctx->d_qcarry) cudaFree(ctx->d_qcarry);
      ctx->d_qcarry = nullptr;
      CK(cudaMalloc(&ctx->d_qcarry, ctx->h_qcarry.size() * 8));
      ctx->qcarry_cap = ctx->h_qcarry.size();
    }
  }
  ctx->reset_pending = true;
  ctx->reset_done = true;
  ctx->finalized = false;
  ctx->final_seen = false;
  ctx->chunks = 0;
  return RK_OK;
}

// the device half of rk_subset_reset, on the first accumulate / finalize stream after it
static rk_status flush_reset(rk_ctx* ctx, cudaStream_t st) {
  if (!ctx->reset_pending) return RK_OK;
  CK(cudaMemsetAsync(ctx->d_table, 0, ctx->table_words * 8, st));
  if (!ctx->h_slow.empty())
    CK(cudaMemcpyAsync(ctx->d_slow, ctx->h_slow.data(), ctx->h_slow.size(), cudaMemcpyHostToDevice, st));
  if (!ctx->h_qcarry.empty())
    CK(cudaMemcpyAsync(ctx->d_qcarry, ctx->h_qcarry.data(), ctx->h_qcarry.size() * 8, cudaMemcpyHostToDevice, st));
  ctx->reset_pending = false;
  return RK_OK;
}

rk_status rk_subset_accumulate(rk_ctx* ctx, const int32_t* labels, void* stream) {
  NvtxRange nvtx_("rk_subset_accumulate");
  if (!ctx) return RK_EINVAL;
  if (!ctx->reset_done) return fail(ctx, RK_ESTATE, "rk_subset_reset first");
  if (ctx->finalized) return fail(ctx, RK_ESTATE, "table already finalized (all-reduced): rk_subset_reset first");
  if (!ctx->have_batch) return fail(ctx, RK_ESTATE, "rk_score / rk_score_logits first");
  const int64_t N = ctx->cur_N;
  if (ctx->batch_fused) {  // NEXT-3: the labels were given to rk_score_labelled
    if (labels && labels != ctx->cur_labels_arg)
      return fail(ctx, RK_EINVAL, "after rk_score_labelled, pass the same labels (or NULL)");
    labels = ctx->cur_labels;
  } else if (!labels && ctx->cur_labels_arg) {
    labels = ctx->cur_labels_arg;
  }
  if (N > 0 && !labels) return fail(ctx, RK_EINVAL, "labels required");
  if (ctx->final_seen && N > 0) return fail(ctx, RK_EINVAL, "a ragged chunk must be the last one (chunks are multiples of lcm(B))");
  if (ctx->cur_off % ctx->L != 0) return fail(ctx, RK_EINVAL, "chunk offset must be a multiple of lcm(B)");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  const int K = ctx->K, S = ctx->S, nB = ctx->nB, nR = ctx->nR, C = ctx->C;
  rk_status s;
  if ((s = flush_reset(ctx, st)) != RK_OK) return s;
  CK(cudaMemsetAsync(ctx->d_chunk, 0, ctx->chunk_words * 8, st));
  if (N > 0) {
    const int32_t* dl = labels;
    if (!is_device_ptr(labels)) {
      if ((s = ensure(ctx, &ctx->d_labels, &ctx->labels_cap, N)) != RK_OK) return s;
      CK(cudaMemcpyAsync(ctx->d_labels, labels, N * 4, cudaMemcpyHostToDevice, st));
      dl = ctx->d_labels;
    }
    unsigned long long* ch = ctx->d_chunk;
    unsigned int* errp = reinterpret_cast<unsigned int*>(ch + 3 * (size_t)S + (size_t)nB * S + 2 * (size_t)nR * nB * K);
    // ---- A2-A5: vote / average / counts ----
    VoteParams vp{};
    vp.logits = ctx->cur_logits; vp.ldc = ctx->cur_ldc;
    vp.lsum_in = ctx->batch_stats ? ctx->ws_lsum : nullptr;
    vp.top1_in = ctx->batch_stats ? ctx->ws_top1 : nullptr;
    vp.labels = dl; vp.N = N; vp.K = K; vp.C = C; vp.S = S; vp.tie = ctx->tie;
    const int gs = (ctx->want_labelled && nB > 0 && nR > 0) ? ctx->gs : 0;
    vp.rmax_in = ctx->batch_stats ? ctx->ws_max : nullptr;
    // K <= 8: warp-per-sample kernels (rk_vote_warp.cu); K = 9..12: batch-transposed (rk_vote_batch.cu)
    const bool warp_path = K <= 8;
    vp.G = 1;
    vp.gs = gs;
    vp.U = std::max(1, gs);
    vp.nW32 = (C + 31) / 32;
    vp.K1 = K / 2;
    const int TT = (1 << vp.K1) + (1 << (K - vp.K1));
    vp.CAP = warp_path ? 96 : 64;
    vp.TCAP = warp_path ? std::min(vp.CAP, (int)(6272 / (4 * TT))) : std::min(vp.CAP, (int)(16384 / (4 * TT)) - 1);
    vp.band = 2e-5f;
    vp.cta_cols = ctx->cta_cols;
    vp.best_of = ctx->d_best_of;
    vp.nB = nB;
    for (int bi = 0; bi < nB; ++bi) vp.tail_start[bi] = (N / ctx->B[bi]) * ctx->B[bi];
    vp.cnt_vote = ch; vp.cnt_avg = ch + S; vp.n_recheck = ch + 2 * S; vp.tail = ch + 3 * S;
    vp.err = errp;
    ctx->grp_gs = gs;
    ctx->grp_groups = gs > 0 ? (N + gs - 1) / gs : 0;
    if (gs > 0) {
      const size_t need = (size_t)((N + gs - 1) / gs) * S;
      if (ctx->grp_cap < need) {
        if (ctx->d_grp) cudaFree(ctx->d_grp);
        ctx->d_grp = nullptr;
        CK(cudaMalloc(&ctx->d_grp, need));
        ctx->grp_cap = need;
      }
      vp.grp = ctx->d_grp;
    }
    int grid = 0;
    if (warp_path) {
      const int wt = vote_warp_threads();
      const size_t smem = vote_warp_smem_per_warp(vp) * (wt / 32);
      const int per_sm = (int)std::max<size_t>(
          1, std::min<size_t>((size_t)vote_warp_min_blocks(), (227 * 1024) / (smem + 1024)));
      const int64_t units = (N + (gs > 0 ? gs : 16) - 1) / (gs > 0 ? gs : 16);
      grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + wt / 32 - 1) / (wt / 32), (int64_t)ctx->sm_count * per_sm));
    } else if (vote_batch_smem_per_sample(vp) * vote_batch_avg_ctas_samples() > 220 * 1024) {
      return fail(ctx, RK_EUNSUPPORTED, "vote kernel: per-sample tables do not fit in shared memory");
    }
    // overflow scratch (candidate sets larger than CAP): one region per warp
    const size_t owners = warp_path ? (size_t)grid * (vote_warp_threads() / 32)
                                    : (size_t)ctx->sm_count * vote_batch_avg_ctas_samples();
    // (rows wider than kMaxCFast go to rk_vote_large.cu, which needs no global scratch)
    const bool wide = ctx->cur_ldc > kMaxCFast;
    const size_t sf = wide ? 0 : owners * C * K, si = wide ? 0 : owners * C;
    if (ctx->scratch_floats < sf) {
      if (ctx->d_scratch) cudaFree(ctx->d_scratch);
      ctx->d_scratch = nullptr;
      CK(cudaMalloc(&ctx->d_scratch, sf * 4));
      ctx->scratch_floats = sf;
    }
    if (ctx->scratch_ints < si) {
      if (ctx->d_scratch_cls) cudaFree(ctx->d_scratch_cls);
      ctx->d_scratch_cls = nullptr;
      CK(cudaMalloc(&ctx->d_scratch_cls, si * 4));
      ctx->scratch_ints = si;
    }
    vp.scratch = ctx->d_scratch;
    vp.scratch_cls = ctx->d_scratch_cls;
    vp.sm_count = ctx->sm_count;

    {
      // worklist [N] + count, then (K >= 9) the overflow and the CTA-kernel worklists, [N] + count each,
      // and the near-tie pair count
      if ((s = ensure(ctx, &ctx->d_work, &ctx->work_cap, 3 * N + 6)) != RK_OK) return s;
      if (!warp_path) {  // near-tie pairs of the warp averaging kernel (a full list sends samples to the CTA kernel)
        if ((s = ensure(ctx, &ctx->d_pairs, &ctx->pairs_cap, N / 2 + 65536)) != RK_OK) return s;
        vp.pairs = ctx->d_pairs;
        vp.dyn_ctr = reinterpret_cast<unsigned int*>(ctx->d_work + 3 * N + 5);  // warp averaging kernel's grabs
        vp.pair_cap = ctx->pair_cap_test > 0 ? std::min<int64_t>(ctx->pair_cap_test, ctx->pairs_cap) : ctx->pairs_cap;
        vp.pair_count = reinterpret_cast<unsigned int*>(ctx->d_work + 3 * N + 3);
      }
      int32_t* st_top = nullptr;
      float *st_lsum = nullptr, *st_max = nullptr;
      if (!ctx->batch_stats) {  // the classify kernel writes row statistics for the averaging kernel
        if ((s = ensure(ctx, &ctx->ws_top1, &ctx->ws_top1_cap, N * K)) != RK_OK) return s;
        if ((s = ensure(ctx, &ctx->ws_lsum, &ctx->ws_lsum_cap, N * K)) != RK_OK) return s;
        if ((s = ensure(ctx, &ctx->ws_max, &ctx->ws_max_cap, N * K)) != RK_OK) return s;
        st_top = ctx->ws_top1; st_lsum = ctx->ws_lsum; st_max = ctx->ws_max;
      }
      unsigned int* wc = reinterpret_cast<unsigned int*>(ctx->d_work + N);
      vp.ovf_work = ctx->d_work + N + 1;
      vp.ovf_count = reinterpret_cast<unsigned int*>(ctx->d_work + 2 * N + 1);
      vp.cta_work = ctx->d_work + 2 * N + 2;  // K >= 9: warp averaging kernel -> CTA kernel
      vp.cta_count = reinterpret_cast<unsigned int*>(ctx->d_work + 3 * N + 2);
      const double bytes = (double)N * ((double)K * C * 4 + 4);
      if (ctx->batch_fused) {
        // NEXT-3: classify from the statistics and l_y, averages from the top-T lists; undecided samples
        // are recomputed below with logits (fallback)
        vp.ly_in = ctx->d_ly;
        vp.logits = nullptr;
        vp.dyn_ctr = reinterpret_cast<unsigned int*>(ctx->d_work + 3 * N + 5);  // sparse kernel's grabs
        if ((s = ensure(ctx, &ctx->d_fb, &ctx->fb_cap, 2 * N + 2)) != RK_OK) return s;
        unsigned int* fbc = reinterpret_cast<unsigned int*>(ctx->d_fb + 2 * N);
        {
          ProfScope ps(ctx, KK_VOTE, st, (double)N * K * (kFuseT * 6 + 16 + 4) + 4.0 * N, 0);
          CK(cudaMemsetAsync(fbc, 0, 4, st));
          CK(launch_vote_classify(vp, st, ctx->d_work, wc, ctx->sm_count));
          CK(launch_vote_sparse(vp, ctx->d_ly, ctx->d_tv, ctx->d_ti, ctx->d_work, wc, ctx->d_fb, fbc, ctx->sm_count, st));
        }
        unsigned int hc[2] = {0, 0};
        CK(cudaMemcpyAsync(&hc[0], fbc, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&hc[1], wc, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const int64_t M = hc[0];
        ctx->last_fallback = M;
        ctx->last_worklist = hc[1];
        if (M > 0) {
          ProfScope ps(ctx, KK_FALLBACK, st, (double)M * ((double)K * C * 8 + ctx->D * 4), 2.0 * M * ctx->D * (double)K * C);
          if ((s = ensure(ctx, &ctx->d_xc, &ctx->xc_cap, M * ctx->D)) != RK_OK) return s;
          if ((s = ensure(ctx, &ctx->d_lc, &ctx->lc_cap, M * K * ctx->ldc)) != RK_OK) return s;
          if ((s = ensure(ctx, &ctx->d_tc, &ctx->tc_cap, M * K + M)) != RK_OK) return s;
          if ((s = ensure(ctx, &ctx->d_sc, &ctx->sc_cap, 2 * M * K)) != RK_OK) return s;
          int32_t* iota = ctx->d_fb + N;
          int32_t* yc = ctx->d_tc + M * K;
          CK(launch_gather_rows(ctx->cur_X, ctx->D, ctx->cur_labels, ctx->d_fb, fbc, M, ctx->d_xc, yc, iota, st));
          GemmParams gp{};
          gp.N = M; gp.K = K; gp.C = C; gp.Cp = ctx->Cp; gp.D = ctx->D; gp.ldc = ctx->ldc;
          gp.scale_log2 = ctx->scale_log2; gp.bias = ctx->d_bias; gp.cluster = ctx->gemm_cluster;
          gp.top1 = ctx->d_tc; gp.lsum = ctx->d_sc; gp.rmax = ctx->d_sc + M * K; gp.logits = ctx->d_lc;
          int rc = gemm_build_tmaps(gp, ctx->d_xc, ctx->d_W, gp.logits, ctx->tmaps);
          if (rc != 0) return fail(ctx, RK_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(rc) + ")");
          CK(launch_gemm(gp, ctx->sm_count, st));
          VoteParams q = vp;
          q.logits = ctx->d_lc; q.ldc = ctx->ldc; q.N = M;
          q.top1_in = ctx->d_tc; q.lsum_in = ctx->d_sc; q.rmax_in = ctx->d_sc + M * K; q.ly_in = nullptr;
          q.labels = yc;
          CK(launch_vote_avg(q, grid, st, iota, fbc));
        }
      } else {
      if (warp_path && !wide) {  // records for the averaging kernel (its inputs in one load per sample)
        if ((s = ensure(ctx, &ctx->d_wrec, &ctx->wrec_cap, N * kRecWords)) != RK_OK) return s;
        vp.wrec = ctx->d_wrec;
        static const bool no_skip = getenv("RK_NO_ROW_SKIP") != nullptr;  // development knob (A/B timing)
        vp.s2_in = (ctx->batch_stats && ctx->cur_s2 && !no_skip) ? ctx->ws_s2 : nullptr;
        vp.n_skip = reinterpret_cast<unsigned int*>(ctx->d_work + 3 * N + 4);
        vp.dyn_ctr = reinterpret_cast<unsigned int*>(ctx->d_work + 3 * N + 5);
        CK(cudaMemsetAsync(vp.n_skip, 0, 8, st));  // n_skip and dyn_ctr
      }
      ctx->last_skip_valid = warp_path && !wide;
      ProfScope ps(ctx, KK_VOTE, st, bytes, 0);
      if (warp_path) CK(launch_vote_warp(vp, grid, st, ctx->d_work, wc, st_top, st_lsum, st_max, ctx->sm_count));
      else CK(launch_vote_batch(vp, ctx->sm_count, st, ctx->d_work, wc, st_top, st_lsum, st_max));
      }
    }
    // ---- A5: batch latency moments (label independent) ----
    const int64_t* arr = nullptr;
    if (nB > 0 && nR > 0) {
      if (ctx->arrival_user) {
        if (is_device_ptr(ctx->arrival_user)) arr = ctx->arrival_user;
        else {
          if ((s = ensure(ctx, &ctx->d_arr, &ctx->arr_cap, N)) != RK_OK) return s;
          CK(cudaMemcpyAsync(ctx->d_arr, ctx->arrival_user, N * 8, cudaMemcpyHostToDevice, st));
          arr = ctx->d_arr;
        }
      }
      MomentParams mp{};
      mp.K = K; mp.S = S; mp.nB = nB; mp.nR = nR;
      for (int bi = 0; bi < nB; ++bi) mp.B[bi] = ctx->B[bi];
      memcpy(mp.lat, ctx->lat, sizeof(mp.lat));
      memcpy(mp.rates, ctx->rates, sizeof(mp.rates));
      mp.arrival = arr; mp.tau = ctx->tau; mp.goff = ctx->cur_off; mp.N = N; mp.want_exceed = ctx->want_exceed;
      mp.osum = ch + 3 * (size_t)S + (size_t)nB * S;
      mp.esum = mp.osum + (size_t)nR * nB * K;
      if (gs > 0) {  // per-batch counts for the labelled moments
        const size_t need = (size_t)ovd_elems(nB, ctx->B, nR, K, N, mp.ovd_off) * sizeof(uint16_t);
        if (ctx->ovd_cap < need) {
          if (ctx->d_ovd) cudaFree(ctx->d_ovd);
          ctx->d_ovd = nullptr;
          CK(cudaMalloc(&ctx->d_ovd, need));
          ctx->ovd_cap = need;
        }
        mp.ovd = ctx->d_ovd;
        mp.ovd_nrp = ovd_nrp(nR);
      }
      ProfScope ps(ctx, KK_OVERDUE, st, 0, 0);
      if (ctx->queue) {  // reading Q15: FIFO finish times, carried across chunks in global order
        int seed = 0;
        if (!ctx->q_started) {
          if (ctx->cur_off > 0) {
            if (ctx->arrival_user)
              return fail(ctx, RK_EUNSUPPORTED, "queue mode with arrival_ns needs the stream to start at sample 0");
            seed = 1;
          }
          ctx->q_started = true;
        } else if (ctx->cur_off != ctx->q_next_off) {
          return fail(ctx, RK_EINVAL, "queue mode: chunks must be contiguous and in global order");
        }
        ctx->q_next_off = ctx->cur_off + N;
        const size_t need = (size_t)fin_elems(nB, ctx->B, nR, K, N, mp.fin_off) * sizeof(int64_t);
        if (ctx->fin_cap < need) {
          if (ctx->d_fin) cudaFree(ctx->d_fin);
          ctx->d_fin = nullptr;
          CK(cudaMalloc(&ctx->d_fin, need ? need : 8));
          ctx->fin_cap = need;
        }
        mp.fin = ctx->d_fin;
        CK(launch_queue_scan(mp, ctx->d_fin, ctx->d_qcarry, seed, st));
      }
      CK(launch_overdue(mp, st));
    }
    // ---- labelled moments (before the merge: for K >= 9 this pass also adds the vote totals) ----
    if (gs > 0) {
      QParams qp{};
      qp.K = K; qp.S = S; qp.nB = nB; qp.nR = nR; qp.gs = gs;
      for (int bi = 0; bi < nB; ++bi) qp.B[bi] = ctx->B[bi];
      qp.N = N; qp.L = ctx->L;
      qp.grp = ctx->d_grp; qp.slow = ctx->d_slow; qp.Q = ctx->d_table + ctx->off_Q;
      qp.ovd = ctx->d_ovd;
      qp.cnt_vote = warp_path ? nullptr : ch;  // K >= 9: per-subset vote totals from the group counts
      ovd_elems(nB, ctx->B, nR, K, N, qp.ovd_off);
      ProfScope ps(ctx, KK_Q, st, 0, 0);
      CK(launch_q(qp, ctx->sm_count, st));
    }
    // ---- merge chunk counters into the table ----
    MergeParams gp{};
    gp.S = S; gp.nB = nB; gp.nR = nR; gp.K = K; gp.chunk = ch; gp.slow = ctx->d_slow; gp.table = ctx->d_table;
    gp.off_vote = ctx->off_vote; gp.off_avg = ctx->off_avg; gp.off_rc = ctx->off_rc; gp.off_corr = ctx->off_corr;
    gp.off_O = ctx->off_O; gp.off_E = ctx->off_E; gp.want_exceed = ctx->want_exceed;
    gp.err = errp; gp.off_err = ctx->off_err;
    {
      ProfScope ps(ctx, KK_MERGE, st, 0, 0);
      CK(launch_merge(gp, N, ctx->off_N, st));
    }
  }
  if (N % ctx->L != 0) ctx->final_seen = true;
  ctx->chunks++;
  return RK_OK;
}

rk_status rk_subset_finalize(rk_ctx* ctx, rk_table* out, void* stream) {
  NvtxRange nvtx_("rk_subset_finalize");
  if (!ctx) return RK_EINVAL;
  if (!ctx->reset_done) return fail(ctx, RK_ESTATE, "rk_subset_reset first");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  const int S = ctx->S, nB = ctx->nB, nR = ctx->nR;
  {
    const rk_status fr = flush_reset(ctx, st);
    if (fr != RK_OK) return fr;
  }
  // A6: one all-reduce of the whole integer table (order-free, bit-exact), at most once per reset: a
  // repeated finalize returns the same global table instead of summing it again
  if (ctx->comm && !ctx->finalized) {
    ProfScope ps(ctx, KK_ALLREDUCE, st, (double)ctx->table_words * 8, 0);
    if (ncclAllReduce(ctx->d_table, ctx->d_table, ctx->table_words, ncclUint64, ncclSum, ctx->comm, st) != ncclSuccess)
      return fail(ctx, RK_ENCCL, "ncclAllReduce failed");
    // bounded wait before any blocking copy: a dead peer must not hang the caller (NCCL async error poll)
    rk_status w = wait_nccl(ctx, st);
    if (w != RK_OK) return w;
  }
  ctx->finalized = true;
  // A7: reward fold on the device
  const size_t nrew = (size_t)nR * nB * S;
  if (nrew > 0) {
    if (ctx->rew_cap < 2 * nrew) {
      if (ctx->d_rew) cudaFree(ctx->d_rew);
      ctx->d_rew = nullptr;
      CK(cudaMalloc(&ctx->d_rew, 2 * nrew * 8));
      ctx->rew_cap = 2 * nrew;
    }
    FoldParams fp{};
    fp.S = S; fp.nB = nB; fp.nR = nR;
    for (int bi = 0; bi < nB; ++bi) fp.B[bi] = ctx->B[bi];
    fp.beta = ctx->beta; fp.table = ctx->d_table;
    fp.off_vote = ctx->off_vote; fp.off_corr = ctx->off_corr; fp.off_O = ctx->off_O; fp.off_Q = ctx->off_Q;
    fp.off_N = ctx->off_N; fp.has_Q = ctx->want_labelled;
    fp.reward_sur = ctx->d_rew; fp.reward_lab = ctx->d_rew + nrew;
    ProfScope ps(ctx, KK_FOLD, st, 0, 0);
    CK(launch_fold(fp, st));
  }
  // the table and rewards come back by DMA into a context-owned page-locked buffer (grow-only): a pageable
  // destination made the driver stage the copy, and a fresh vector per call paid zeroing and page faults
  const size_t need = (ctx->table_words + 2 * nrew) * 8;
  if (ctx->h_stage_bytes < need) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_bytes = 0;
    CK(cudaMallocHost(&ctx->h_stage, need));
    ctx->h_stage_bytes = need;
  }
  unsigned long long* h = static_cast<unsigned long long*>(ctx->h_stage);
  double* rew = reinterpret_cast<double*>(h + ctx->table_words);
  CK(cudaMemcpyAsync(h, ctx->d_table, ctx->table_words * 8, cudaMemcpyDeviceToHost, st));
  if (nrew) CK(cudaMemcpyAsync(rew, ctx->d_rew, 2 * nrew * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  rk_status status = RK_OK;
  if (h[ctx->off_err + 0]) status = fail(ctx, RK_ENONFINITE, "non-finite logits (NaN, +inf or an all -inf row)");
  else if (h[ctx->off_err + 1]) status = fail(ctx, RK_ELABEL, "label outside [0, C)");
  else if (h[ctx->off_err + 2]) status = fail(ctx, RK_EINVAL, "arrival_ns not non-decreasing inside a batch");
  if (status != RK_OK) {
    std::fill(h, h + ctx->table_words, 0ull);
    std::fill(rew, rew + 2 * nrew, 0.0);
  }
  if (out) {
    out->N = (int64_t)h[ctx->off_N];
    auto cp = [&](uint64_t* dst, int64_t off, size_t n) { if (dst && n) memcpy(dst, h + off, n * 8); };
    cp(out->cnt_vote, ctx->off_vote, S);
    cp(out->cnt_avg, ctx->off_avg, S);
    cp(out->n_recheck, ctx->off_rc, S);
    cp(out->corr, ctx->off_corr, (size_t)nB * S);
    cp(out->O, ctx->off_O, nrew);
    cp(out->Q, ctx->off_Q, ctx->want_labelled ? nrew : 0);
    cp(out->E, ctx->off_E, ctx->want_exceed ? nrew : 0);
    if (out->reward_sur && nrew) memcpy(out->reward_sur, rew, nrew * 8);
    if (out->reward_lab && nrew) memcpy(out->reward_lab, rew + nrew, nrew * 8);
  }
  return status;
}

rk_status rk_subset_stats(rk_ctx* ctx, const int32_t* labels, const rk_reward_cfg* cfg, rk_table* out, void* stream) {
  rk_status s = rk_subset_reset(ctx, cfg);
  if (s != RK_OK) return s;
  if ((s = rk_subset_accumulate(ctx, labels, stream)) != RK_OK) return s;
  return rk_subset_finalize(ctx, out, stream);
}

rk_status rk_predict(rk_ctx* ctx, uint32_t v, int32_t* pred_vote, int32_t* pred_avg, float* avgprob, void* stream) {
  NvtxRange nvtx_("rk_predict");
  if (!ctx) return RK_EINVAL;
  if (!ctx->have_batch) return fail(ctx, RK_ESTATE, "rk_score / rk_score_logits first");
  if (v == 0 || v >= (1u << ctx->K)) return fail(ctx, RK_EINVAL, "v must be in [1, 2^K) (PAPER.md:429 excludes v = 0)");
  if (ctx->batch_fused) return fail(ctx, RK_ESTATE, "rk_score_labelled keeps no logits: rk_score the batch for rk_predict");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  PredictParams pp{};
  pp.logits = ctx->cur_logits; pp.ldc = ctx->cur_ldc;
  pp.N = ctx->cur_N; pp.K = ctx->K; pp.C = ctx->C; pp.tie = ctx->tie; pp.v = v; pp.best_of = ctx->d_best_of;
  pp.pred_vote = pred_vote; pp.pred_avg = pred_avg; pp.avgprob = avgprob;
  ProfScope ps(ctx, KK_PREDICT, st, 0, 0);
  CK(launch_predict(pp, st));
  return RK_OK;
}

// Validate a serving configuration and fill ServeParams (+ the [nR][N] arrival times on the device).
static rk_status serve_setup(rk_ctx* ctx, const rk_reward_cfg* cfg, int64_t N, int64_t delta_ns, ServeParams& sp,
                      cudaStream_t st) {
  if (!ctx->loaded) return fail(ctx, RK_ESTATE, "rk_load_ensemble first");
  if (N < 0) return fail(ctx, RK_EINVAL, "N >= 0");
  if (cfg->nB < 1 || cfg->nB > kMaxB || !cfg->B || !cfg->lat_ns) return fail(ctx, RK_EINVAL, "nB in [1,8] with B and lat_ns");
  if (cfg->arrival_ns ? cfg->nR != 1 : (cfg->nR < 1 || cfg->nR > kMaxR || !cfg->rates))
    return fail(ctx, RK_EINVAL, "rates (nR in [1,8]) or arrival_ns with nR == 1");
  if (cfg->tau_ns < 0 || !(cfg->beta == cfg->beta)) return fail(ctx, RK_EINVAL, "tau >= 0, finite beta");
  CK(cudaSetDevice(ctx->dev));
  const int K = ctx->K;
  sp = ServeParams{};
  sp.K = K; sp.S = ctx->S; sp.nB = cfg->nB; sp.nR = cfg->nR; sp.N = N; sp.tau = cfg->tau_ns; sp.delta = delta_ns;
  sp.beta = cfg->beta;
  for (int bi = 0; bi < cfg->nB; ++bi) {
    if (cfg->B[bi] < 1) return fail(ctx, RK_EINVAL, "batch sizes >= 1");
    sp.B[bi] = cfg->B[bi];
    for (int m = 0; m < K; ++m) {
      if (cfg->lat_ns[m * cfg->nB + bi] < 0) return fail(ctx, RK_EINVAL, "latencies must be >= 0");
      sp.lat[m * cfg->nB + bi] = cfg->lat_ns[m * cfg->nB + bi];
    }
  }
  for (int r = 0; r < sp.nR; ++r) {
    sp.rates[r] = cfg->arrival_ns ? 1.0 : cfg->rates[r];
    if (!(sp.rates[r] > 0) || sp.rates[r] > 1e12) return fail(ctx, RK_EINVAL, "rates must be > 0");
  }
  rk_status s;
  if (cfg->arrival_ns && is_device_ptr(cfg->arrival_ns)) {
    sp.arrival = cfg->arrival_ns;
  } else {  // [nR][N] arrival times on the device: the caller's, or filled from the rates
    if ((s = ensure(ctx, &ctx->d_arr, &ctx->arr_cap, std::max<int64_t>(N * sp.nR, 1))) != RK_OK) return s;
    if (cfg->arrival_ns) CK(cudaMemcpyAsync(ctx->d_arr, cfg->arrival_ns, N * 8, cudaMemcpyHostToDevice, st));
    else CK(launch_arrival_fill(sp, ctx->d_arr, st));
    sp.arrival = ctx->d_arr;
  }
  return RK_OK;
}

rk_status rk_greedy_serve(rk_ctx* ctx, const rk_reward_cfg* cfg, int64_t N, int64_t delta_ns, const double* acc,
                          rk_serve_out* out, void* stream) {
  NvtxRange nvtx_("rk_greedy_serve");
  if (!ctx || !cfg || !out) return RK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  ServeParams sp;
  rk_status s = serve_setup(ctx, cfg, N, delta_ns, sp, st);
  if (s != RK_OK) return s;
  const int S = ctx->S;
  const int64_t n = (int64_t)sp.nR * S;
  // device scratch: 5 counter arrays + reward + acc
  const size_t words = 5 * (size_t)n + (size_t)n + (size_t)S;
  if ((s = ensure(ctx, &ctx->d_serve, &ctx->serve_cap, (int64_t)words)) != RK_OK) return s;
  sp.out = reinterpret_cast<unsigned long long*>(ctx->d_serve);
  if (acc) {
    sp.reward = reinterpret_cast<double*>(ctx->d_serve + 5 * n);
    sp.acc = reinterpret_cast<const double*>(ctx->d_serve + 6 * n);
    CK(cudaMemcpyAsync(ctx->d_serve + 6 * n, acc, (size_t)S * 8, cudaMemcpyHostToDevice, st));
  }
  {
    ProfScope ps(ctx, KK_SERVE, st, 0, 0);
    CK(launch_greedy_serve(sp, st));
  }
  uint64_t* dst[5] = {out->served, out->overdue, out->exceed_ns, out->batches, out->unserved};
  for (int k = 0; k < 5; ++k)
    if (dst[k]) CK(cudaMemcpyAsync(dst[k], ctx->d_serve + k * n, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  if (out->reward && acc) CK(cudaMemcpyAsync(out->reward, ctx->d_serve + 5 * n, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return RK_OK;
}

rk_status rk_async_serve(rk_ctx* ctx, const rk_reward_cfg* cfg, int64_t N, int64_t delta_ns, const double* acc,
                         rk_serve_out* out, uint64_t* model_batches, void* stream) {
  NvtxRange nvtx_("rk_async_serve");
  if (!ctx || !cfg || !out) return RK_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  ServeParams sp;
  rk_status s = serve_setup(ctx, cfg, N, delta_ns, sp, st);
  if (s != RK_OK) return s;
  const int K = ctx->K, nR = sp.nR;
  // device scratch: 5 x [nR] counters, [nR] reward, [nR][K] batches per model, [K] accuracies
  const size_t words = 6 * (size_t)nR + (size_t)nR * K + (size_t)K;
  if ((s = ensure(ctx, &ctx->d_serve, &ctx->serve_cap, (int64_t)words)) != RK_OK) return s;
  sp.out = reinterpret_cast<unsigned long long*>(ctx->d_serve);
  sp.reward = reinterpret_cast<double*>(ctx->d_serve + 5 * nR);
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(ctx->d_serve + 6 * nR);
  const double* dacc = nullptr;
  if (acc) {
    CK(cudaMemcpyAsync(ctx->d_serve + 6 * nR + nR * K, acc, (size_t)K * 8, cudaMemcpyHostToDevice, st));
    dacc = reinterpret_cast<const double*>(ctx->d_serve + 6 * nR + nR * K);
  }
  {
    ProfScope ps(ctx, KK_SERVE, st, 0, 0);
    CK(launch_async_serve(sp, dacc, mb, st));
  }
  uint64_t* dst[5] = {out->served, out->overdue, out->exceed_ns, out->batches, out->unserved};
  for (int k = 0; k < 5; ++k)
    if (dst[k]) CK(cudaMemcpyAsync(dst[k], ctx->d_serve + k * nR, (size_t)nR * 8, cudaMemcpyDeviceToHost, st));
  if (out->reward && acc) CK(cudaMemcpyAsync(out->reward, ctx->d_serve + 5 * nR, (size_t)nR * 8, cudaMemcpyDeviceToHost, st));
  if (model_batches) CK(cudaMemcpyAsync(model_batches, mb, (size_t)nR * K * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return RK_OK;
}

rk_status rk_serve_stream(rk_ctx* ctx, const void* X, int64_t N, const rk_reward_cfg* cfg, int64_t delta_ns,
                          uint32_t v, int32_t* pred_vote, int32_t* pred_avg, rk_serve_out* out, int64_t* n_batches,
                          void* stream) {
  NvtxRange nvtx_("rk_serve_stream");
  if (!ctx || !cfg) return RK_EINVAL;
  if (!ctx->loaded || !ctx->has_heads) return fail(ctx, RK_ESTATE, "no heads loaded (rk_load_ensemble with W)");
  if (v == 0 || v >= (1u << ctx->K)) return fail(ctx, RK_EINVAL, "v must be in [1, 2^K) (PAPER.md:429 excludes v = 0)");
  if (cfg->nR != 1) return fail(ctx, RK_EINVAL, "rk_serve_stream serves one arrival stream (nR == 1)");
  if (N > 0 && (!X || !is_device_ptr(X))) return fail(ctx, RK_EINVAL, "X must be device memory");
  if ((pred_vote && !is_device_ptr(pred_vote)) || (pred_avg && !is_device_ptr(pred_avg)))
    return fail(ctx, RK_EINVAL, "predictions must be device memory");
  if (N > INT32_MAX) return fail(ctx, RK_EINVAL, "N < 2^31");
  cudaStream_t st = (cudaStream_t)stream;
  ServeParams sp;
  rk_status s = serve_setup(ctx, cfg, N, delta_ns, sp, st);
  if (s != RK_OK) return s;
  // 1. Algorithm 3 for this one action: counters + the batch schedule
  const int64_t n = (int64_t)sp.nR * ctx->S;  // counters [5][n], this scenario at index 0
  if ((s = ensure(ctx, &ctx->d_serve, &ctx->serve_cap, 5 * n)) != RK_OK) return s;
  int64_t* d_sched = nullptr;
  CK(cudaMallocAsync((void**)&d_sched, (size_t)std::max<int64_t>(N, 1) * 16, st));
  sp.out = reinterpret_cast<unsigned long long*>(ctx->d_serve);
  sp.v_only = v;
  sp.sched = d_sched;
  {
    ProfScope ps(ctx, KK_SERVE, st, 0, 0);
    CK(launch_greedy_serve(sp, st));
  }
  uint64_t cnt[5];
  for (int k = 0; k < 5; ++k) CK(cudaMemcpyAsync(&cnt[k], ctx->d_serve + k * n, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int64_t> sched(2 * cnt[3]);
  if (cnt[3]) CK(cudaMemcpyAsync(sched.data(), d_sched, sched.size() * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaFreeAsync(d_sched, st);
  if (out) {
    uint64_t* dst[5] = {out->served, out->overdue, out->exceed_ns, out->batches, out->unserved};
    for (int k = 0; k < 5; ++k) if (dst[k]) *dst[k] = cnt[k];
  }
  if (n_batches) *n_batches = (int64_t)cnt[3];
  // 2. serve every batch through the heads (A1+A2) and the per-request prediction of v
  if (pred_vote && N) CK(cudaMemsetAsync(pred_vote, 0xff, N * 4, st));  // unserved requests: -1
  if (pred_avg && N) CK(cudaMemsetAsync(pred_avg, 0xff, N * 4, st));
  int64_t bmax = 0;
  for (size_t i = 0; i < cnt[3]; ++i) bmax = std::max(bmax, sched[2 * i + 1]);
  if ((s = ensure(ctx, &ctx->ws_logits, &ctx->ws_cap, std::max<int64_t>(bmax, 1) * ctx->K * ctx->ldc)) != RK_OK) return s;
  if ((s = ensure(ctx, &ctx->ws_top1, &ctx->ws_top1_cap, std::max<int64_t>(bmax, 1) * ctx->K)) != RK_OK) return s;
  if ((s = ensure(ctx, &ctx->ws_lsum, &ctx->ws_lsum_cap, std::max<int64_t>(bmax, 1) * ctx->K)) != RK_OK) return s;
  if ((s = ensure(ctx, &ctx->ws_max, &ctx->ws_max_cap, std::max<int64_t>(bmax, 1) * ctx->K)) != RK_OK) return s;
  for (size_t i = 0; i < cnt[3]; ++i) {
    const int64_t h = sched[2 * i], b = sched[2 * i + 1];
    GemmParams gp{};
    gp.N = b; gp.K = ctx->K; gp.C = ctx->C; gp.Cp = ctx->Cp; gp.D = ctx->D; gp.ldc = ctx->ldc;
    gp.scale_log2 = ctx->scale_log2; gp.bias = ctx->d_bias; gp.cluster = ctx->gemm_cluster;
    gp.top1 = ctx->ws_top1; gp.lsum = ctx->ws_lsum; gp.rmax = ctx->ws_max; gp.logits = ctx->ws_logits;
    int rc = gemm_build_tmaps(gp, static_cast<const uint16_t*>(X) + h * ctx->D, ctx->d_W, gp.logits, ctx->tmaps);
    if (rc != 0) return fail(ctx, RK_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(rc) + ")");
    {
      ProfScope ps(ctx, KK_GEMM, st, (double)b * ctx->D * 2 + (double)b * ctx->K * ctx->C * 4,
                   2.0 * b * ctx->D * (double)ctx->K * ctx->C);
      CK(launch_gemm(gp, ctx->sm_count, st));
    }
    PredictParams pp{};
    pp.logits = ctx->ws_logits; pp.ldc = ctx->ldc; pp.N = b; pp.K = ctx->K; pp.C = ctx->C; pp.tie = ctx->tie; pp.v = v;
    pp.best_of = ctx->d_best_of;
    pp.pred_vote = pred_vote ? pred_vote + h : nullptr;
    pp.pred_avg = pred_avg ? pred_avg + h : nullptr;
    ProfScope ps(ctx, KK_PREDICT, st, 0, 0);
    CK(launch_predict(pp, st));
  }
  ctx->have_batch = false;  // the workspaces hold the last served batch only
  CK(cudaStreamSynchronize(st));
  return RK_OK;
}

rk_status rk_sine_arrivals(rk_ctx* ctx, const rk_sine_cfg* cfg, int64_t n0, int64_t N, int64_t* out, void* stream) {
  NvtxRange nvtx_("rk_sine_arrivals");
  if (!ctx || !cfg) return RK_EINVAL;
  if (!(cfg->ref_rate > 0) || cfg->ref_rate > 1e12 || cfg->period_ns <= 0 || cfg->delta_ns <= 0 ||
      !(cfg->noise_std >= 0) || cfg->noise_std > 1e3 || n0 < 0 || N < 0 || (N > 0 && !out))
    return fail(ctx, RK_EINVAL, "sine arrivals: ref > 0, period > 0, delta > 0, noise_std >= 0, n0, N >= 0");
  if (N > 0 && !is_device_ptr(out)) return fail(ctx, RK_EINVAL, "out_ns must be device memory");
  if (N == 0) return RK_OK;
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  SineParams sp{};
  const double s0 = (1.0 + std::sqrt(5.0)) / 4.0;  // sin(0.3 pi)
  sp.k = 0.1 * cfg->ref_rate / (1.0 - s0);
  sp.b = 1.1 * cfg->ref_rate - sp.k;
  sp.period = cfg->period_ns; sp.delta = cfg->delta_ns; sp.delta_s = (double)cfg->delta_ns / 1e9;
  sp.sigma = cfg->noise_std; sp.seed = cfg->seed;
  // chunks of invocations: about twice the expected count at the mean rate b, at least 64k
  const double per = std::max(1e-9, sp.delta_s * sp.b);
  const int64_t J = std::min<int64_t>(int64_t(1) << 26, std::max<int64_t>(65536, (int64_t)(2.0 * (n0 + N) / per) + 1024));
  const int64_t nb = sine_chunk_blocks(J);
  int64_t *d_cnt = nullptr, *d_bs = nullptr;
  CK(cudaMallocAsync((void**)&d_cnt, (size_t)J * 8, st));
  CK(cudaMallocAsync((void**)&d_bs, (size_t)(nb + 1) * 8, st));
  rk_status status = RK_OK;
  int64_t base = 0, j0 = 0;
  for (int iter = 0; base < n0 + N; ++iter, j0 += J) {
    if (iter > 4096) { status = fail(ctx, RK_EINVAL, "sine arrivals: the rate is (almost) zero"); break; }
    cudaError_t e = launch_sine_counts(sp, j0, J, d_cnt, d_bs, st);
    int64_t tot = 0;
    if (e == cudaSuccess) e = launch_sine_scatter(sp, j0, J, d_cnt, d_bs, base, n0, N, out, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&tot, d_bs + nb, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { status = fail(ctx, RK_ECUDA, std::string("sine arrivals: ") + cudaGetErrorString(e)); break; }
    base += tot;
  }
  cudaFreeAsync(d_cnt, st);
  cudaFreeAsync(d_bs, st);
  if (status == RK_OK) CK(cudaStreamSynchronize(st));
  return status;
}

// ---- NEXT-2: actor-critic scheduler ---------------------------------------------------------------------
static rk_status ac_setup(rk_ctx* ctx, const rk_reward_cfg* cfg, const rk_ac_cfg* ac, RLParams& rp) {
  if (!ctx->loaded) return fail(ctx, RK_ESTATE, "rk_load_ensemble first");
  if (!cfg || !ac) return fail(ctx, RK_EINVAL, "cfg and ac required");
  if (cfg->nB < 1 || cfg->nB > kMaxB || !cfg->B || !cfg->lat_ns) return fail(ctx, RK_EINVAL, "nB in [1,8] with B and lat_ns");
  if (cfg->tau_ns <= 0 || !(cfg->beta == cfg->beta)) return fail(ctx, RK_EINVAL, "tau > 0, finite beta");
  if (ac->L < 0 || ac->L > 256 || ac->H < 1 || ac->H > kRlMaxH || ac->n_steps < 1 ||
      !(ac->gamma >= 0 && ac->gamma <= 1) || !(ac->reward_scale == ac->reward_scale) ||
      !(ac->entropy >= 0 && ac->entropy < 1e6))
    return fail(ctx, RK_EINVAL, "ac: L in [0,256], H in [1,64], n_steps >= 1, gamma in [0,1], entropy >= 0");
  rp = RLParams{};
  rp.K = ctx->K; rp.nB = cfg->nB; rp.L = ac->L; rp.H = ac->H; rp.n = ac->n_steps;
  rp.F = ac->L + ctx->K * cfg->nB + ctx->K;
  rp.A = ctx->S * cfg->nB;
  if (rp.A > kRlMaxA || rp.F > 1024) return fail(ctx, RK_EINVAL, "ac: (2^K - 1) * nB <= 2048 actions, F <= 1024");
  for (int bi = 0; bi < cfg->nB; ++bi) {
    if (cfg->B[bi] < 1) return fail(ctx, RK_EINVAL, "batch sizes >= 1");
    rp.B[bi] = cfg->B[bi];
    for (int m = 0; m < ctx->K; ++m) {
      if (cfg->lat_ns[m * cfg->nB + bi] < 0) return fail(ctx, RK_EINVAL, "latencies must be >= 0");
      rp.lat[m * cfg->nB + bi] = cfg->lat_ns[m * cfg->nB + bi];
    }
  }
  rp.tau = cfg->tau_ns; rp.beta = cfg->beta; rp.gamma = ac->gamma; rp.scale = ac->reward_scale; rp.ent = ac->entropy;
  return RK_OK;
}

rk_status rk_ac_dims(rk_ctx* ctx, int nB, const rk_ac_cfg* ac, int* F, int* A, int64_t* n_params) {
  if (!ctx || !ac) return RK_EINVAL;
  if (!ctx->loaded) return fail(ctx, RK_ESTATE, "rk_load_ensemble first");
  if (nB < 1 || nB > kMaxB || ac->L < 0 || ac->H < 1) return fail(ctx, RK_EINVAL, "nB in [1,8], L >= 0, H >= 1");
  const int f = ac->L + ctx->K * nB + ctx->K, a = ctx->S * nB;
  if (F) *F = f;
  if (A) *A = a;
  if (n_params) *n_params = ac_param_count(f, ac->H, a);
  return RK_OK;
}

rk_status rk_ac_rollout(rk_ctx* ctx, const rk_reward_cfg* cfg, const double* acc, const int64_t* arrival, int64_t Narr,
                        const rk_ac_cfg* ac, const float* params, int E, const int64_t* h0, const int32_t* forced,
                        uint64_t seed, rk_ac_traj* traj, void* stream) {
  NvtxRange nvtx_("rk_ac_rollout");
  if (!ctx) return RK_EINVAL;
  RLParams rp;
  rk_status s = ac_setup(ctx, cfg, ac, rp);
  if (s != RK_OK) return s;
  if (!acc || !traj || !traj->actions || !traj->rewards || E < 1 || Narr < 1)
    return fail(ctx, RK_EINVAL, "acc, traj.actions, traj.rewards, E >= 1, Narr >= 1 required");
  if (!is_device_ptr(arrival) || !is_device_ptr(h0) || (!forced && !is_device_ptr(params)) ||
      (forced && !is_device_ptr(forced)) || !is_device_ptr(traj->actions) || !is_device_ptr(traj->rewards))
    return fail(ctx, RK_EINVAL, "arrival, h0, params, forced and trajectory buffers must be device memory");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  // a(v) and the error flag in the serving scratch: [S] doubles + 1 word
  if ((s = ensure(ctx, &ctx->d_serve, &ctx->serve_cap, (int64_t)ctx->S + 1)) != RK_OK) return s;
  CK(cudaMemcpyAsync(ctx->d_serve, acc, (size_t)ctx->S * 8, cudaMemcpyHostToDevice, st));
  unsigned int* err = reinterpret_cast<unsigned int*>(ctx->d_serve + ctx->S);
  CK(cudaMemsetAsync(err, 0, 8, st));
  rp.acc = reinterpret_cast<const double*>(ctx->d_serve);
  rp.arrival = arrival; rp.Narr = Narr; rp.params = params; rp.h0 = h0; rp.forced = forced; rp.seed = seed;
  rp.E = E; rp.err = err;
  rp.states = traj->states; rp.actions = traj->actions; rp.rewards = traj->rewards; rp.overdue = traj->overdue;
  rp.t_dec = traj->t_dec; rp.t_start = traj->t_start; rp.t_done = traj->t_done;
  {
    ProfScope ps(ctx, KK_SERVE, st, 0, 0);
    CK(launch_ac_rollout(rp, st));
  }
  unsigned int herr = 0;
  CK(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (herr & 4u) return fail(ctx, RK_ENONFINITE, "the policy's probabilities are not finite (diverged parameters)");
  if (herr & 2u) return fail(ctx, RK_EINVAL, "a forced action is outside [0, (2^K - 1) * nB)");
  if (herr & 1u) return fail(ctx, RK_EINVAL, "an episode starts outside or runs past the end of the arrival array (Narr)");
  return RK_OK;
}

rk_status rk_ac_grad(rk_ctx* ctx, const rk_reward_cfg* cfg, const rk_ac_cfg* ac, const float* params,
                     const rk_ac_traj* traj, int E, float* grad, double* losses, void* stream) {
  NvtxRange nvtx_("rk_ac_grad");
  if (!ctx) return RK_EINVAL;
  RLParams rp;
  rk_status s = ac_setup(ctx, cfg, ac, rp);
  if (s != RK_OK) return s;
  if (!traj || !traj->states || !traj->actions || !traj->rewards || !grad || !params || E < 1)
    return fail(ctx, RK_EINVAL, "traj (states, actions, rewards), params, grad, E >= 1 required");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  rp.E = E; rp.params = params;
  rp.states = traj->states; rp.actions = traj->actions; rp.rewards = traj->rewards;
  void* scratch = nullptr;
  float* dl = nullptr;
  CK(cudaMallocAsync(&scratch, ac_grad_scratch_bytes(rp), st));
  CK(cudaMallocAsync((void**)&dl, 8, st));
  cudaError_t e = launch_ac_grad(rp, grad, dl, scratch, st);
  float hl[2] = {0.f, 0.f};
  if (e == cudaSuccess && losses) e = cudaMemcpyAsync(hl, dl, 8, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(scratch, st);
  cudaFreeAsync(dl, st);
  if (e != cudaSuccess) return fail(ctx, RK_ECUDA, std::string("ac grad: ") + cudaGetErrorString(e));
  if (losses) {
    CK(cudaStreamSynchronize(st));
    losses[0] = hl[0];
    losses[1] = hl[1];
  }
  return RK_OK;
}

rk_status rk_ac_apply(rk_ctx* ctx, const rk_reward_cfg* cfg, const rk_ac_cfg* ac, float* params, const float* grad,
                      float lr_pi, float lr_v, void* stream) {
  NvtxRange nvtx_("rk_ac_apply");
  if (!ctx) return RK_EINVAL;
  RLParams rp;
  rk_status s = ac_setup(ctx, cfg, ac, rp);
  if (s != RK_OK) return s;
  if (!params || !grad) return fail(ctx, RK_EINVAL, "params and grad required");
  CK(cudaSetDevice(ctx->dev));
  const int64_t npol = (int64_t)rp.H * rp.F + rp.H + (int64_t)rp.A * rp.H + rp.A;
  CK(launch_ac_apply(params, grad, npol, ac_param_count(rp.F, rp.H, rp.A), lr_pi, lr_v, (cudaStream_t)stream));
  return RK_OK;
}

rk_status rk_group_counts(rk_ctx* ctx, uint8_t* out, int64_t cap, int* gs, int64_t* groups, void* stream) {
  if (!ctx) return RK_EINVAL;
  if (!ctx->reset_done || ctx->chunks == 0) return fail(ctx, RK_ESTATE, "no chunk accumulated since rk_subset_reset");
  if (gs) *gs = ctx->grp_gs;
  if (groups) *groups = ctx->grp_groups;
  const int64_t bytes = ctx->grp_groups * ctx->S;
  if (!out || bytes == 0) return RK_OK;
  if (cap < bytes) return fail(ctx, RK_EINVAL, "out holds fewer than groups * S bytes");
  CK(cudaSetDevice(ctx->dev));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(out, ctx->d_grp, (size_t)bytes, cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
  return RK_OK;
}

rk_status rk_vote_diag(rk_ctx* ctx, int64_t* worklist, int64_t* fallback, int64_t* rows_skipped) {
  if (!ctx) return RK_EINVAL;
  if (!ctx->reset_done || ctx->chunks == 0) return fail(ctx, RK_ESTATE, "no chunk accumulated since rk_subset_reset");
  CK(cudaSetDevice(ctx->dev));
  CK(cudaDeviceSynchronize());  // the counts of the last accumulate, whatever stream it ran on
  unsigned int w = 0;
  if (ctx->d_work && ctx->cur_N > 0) CK(cudaMemcpy(&w, reinterpret_cast<unsigned int*>(ctx->d_work + ctx->cur_N), 4,
                                                   cudaMemcpyDeviceToHost));
  unsigned int k = 0;
  if (ctx->d_work && ctx->cur_N > 0 && ctx->last_skip_valid && !ctx->batch_fused)
    CK(cudaMemcpy(&k, reinterpret_cast<unsigned int*>(ctx->d_work + 3 * ctx->cur_N + 4), 4, cudaMemcpyDeviceToHost));
  if (worklist) *worklist = w;
  if (fallback) *fallback = ctx->batch_fused ? ctx->last_fallback : 0;
  if (rows_skipped) *rows_skipped = k;
  return RK_OK;
}

rk_status rk_outputs_s2(rk_ctx* ctx, const float** s2) {
  if (!ctx) return RK_EINVAL;
  if (!ctx->have_batch) return fail(ctx, RK_ESTATE, "no batch scored yet");
  if (s2) *s2 = ctx->cur_s2 ? ctx->ws_s2 : nullptr;
  return RK_OK;
}

rk_status rk_outputs(rk_ctx* ctx, const float** logits, int* ldc, const int32_t** top1, const float** rmax,
                     const float** lsum, int64_t* N) {
  if (!ctx) return RK_EINVAL;
  if (!ctx->have_batch) return fail(ctx, RK_ESTATE, "no batch scored yet");
  if (logits) *logits = ctx->cur_logits;  // NULL after rk_score_labelled (fused: no logits rows)
  if (ldc) *ldc = (int)ctx->cur_ldc;
  if (top1) *top1 = ctx->batch_stats ? ctx->ws_top1 : nullptr;
  if (rmax) *rmax = ctx->batch_stats ? ctx->ws_max : nullptr;
  if (lsum) *lsum = ctx->batch_stats ? ctx->ws_lsum : nullptr;
  if (N) *N = ctx->cur_N;
  return RK_OK;
}

rk_status rk_set_profiling(rk_ctx* ctx, int on) {
  if (!ctx) return RK_EINVAL;
  prof_collect(ctx);
  ctx->prof.on = on != 0;
  if (on) {
    for (int k = 0; k < KK_COUNT; ++k) { ctx->prof.launches[k] = 0; ctx->prof.ms[k] = 0; ctx->prof.bytes[k] = 0; ctx->prof.flops[k] = 0; }
  }
  return RK_OK;
}

rk_status rk_kernel_stats(rk_ctx* ctx, rk_kernel_stat* out, int max, int* n) {
  if (!ctx) return RK_EINVAL;
  prof_collect(ctx);
  if (n) *n = KK_COUNT;
  for (int k = 0; k < KK_COUNT && k < max; ++k) {
    out[k].name = kKernelNames[k];
    out[k].launches = ctx->prof.launches[k];
    out[k].total_ms = ctx->prof.ms[k];
    out[k].bytes = ctx->prof.bytes[k];
    out[k].flops = ctx->prof.flops[k];
  }
  return RK_OK;
}

}  // extern "C"
