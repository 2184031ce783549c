// rk_vote_sparse.cu — NEXT-3: step A4 (subset softmax average; readings Q5, Q6) for the
// worklist samples of a FUSED forward + vote (rk_score_labelled): the GEMM epilogue kept, per (sample,
// model), only the row statistics (rmax, lsum, top1), the label's logit l_y and the T = kFuseT largest
// logits with their classes -- the fp32 logits never reach HBM. One WARP per worklist sample.
//
// For a subset v, with p[m][c] = exp((l - rmax_m) - lsum_m) and sums over the members of v:
//   A_v(y) = sum p[m][y]                                   exact (l_y is kept),
//   c listed by model m (one of its T largest):            p[m][c] exact,
//   c not listed by m:                                     0 <= p[m][c] <= pT_m (m's T-th largest value,
//                                                          or the bound-only entry the epilogue leaves there),
// so every competitor c has  LB_v(c) = sum_{m listed} p[m][c]  <=  A_v(c)  <=  UB_v(c) = LB_v(c) +
// sum_{m not listed} pT_m, and every class listed by no model has A_v(c) <= sum_m pT_m. Hence
//   y wrong for v  if some c has LB_v(c) > A_v(y) (1 + band);
//   y right for v  if every c has UB_v(c) (1 + band) < A_v(y)   (ties fall inside the band);
// a class with ub_m(c) (1 + band) < p[m][y] in EVERY model can never beat y and is dropped first (the
// R pruning of the streaming kernel). Singletons are decided by the top-1 (invariant I1). A sample with
// any subset left undecided (bounds too loose, or a near-tie inside the band) is handed WHOLE to the
// fallback list: its rows are recomputed by the GEMM with logits stored and averaged by the streaming
// kernel (rk_vote_avg.cu) with the fp64 recheck, so the table stays exact.
//
// Classes are merged across the K lists with a 256-slot open-addressing table per warp in shared memory.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SW = 4;      // warps per CTA
constexpr int HS = 256;    // hash slots per warp (>= 2 x kMaxFuseK x kFuseT)
constexpr int kMaxFuseK = 8;
constexpr int JM = 8;      // subsets per lane (S <= 255)
constexpr int kSpChunk = 2;  // worklist entries per dynamic grab

struct SparseSmem {
  int key[HS];                  // class or -1
  unsigned int mask[HS];        // models listing the class
  float P[HS][kMaxFuseK];       // p[m][class] where listed
  int list[HS];                 // threat slots
  float tab[64];                // one threat's half-mask sums: LB lo [16] | LB hi [16] | UB lo [16] | UB hi [16]
};

// max over subsets v with |v| >= 2 of sum_{m in v} d_m = d_(1) + d_(2) + sum_{k >= 3} max(0, d_(k))
__device__ __forceinline__ float best_pair_sum(const float* d, int K) {
  float m1 = -INFINITY, m2 = -INFINITY, pos = 0.f;
#pragma unroll
  for (int m = 0; m < kMaxFuseK; ++m) {
    if (m >= K) break;
    const float x = d[m];
    pos += fmaxf(x, 0.f);
    if (x > m1) { m2 = m1; m1 = x; } else if (x > m2) { m2 = x; }
  }
  return m1 + m2 + (pos - fmaxf(m1, 0.f) - fmaxf(m2, 0.f));
}

__global__ void __launch_bounds__(32 * SW) vote_sparse_average_kernel(const VoteParams p, const float* ly,
                                                                     const float* tv, const uint16_t* ti,
                                                                     const int32_t* work, const unsigned int* work_count,
                                                                     int32_t* fb, unsigned int* fb_count) {
  __shared__ SparseSmem smem_all[SW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SparseSmem& sh = smem_all[warp];
  const int K = p.K, S = p.S;
  constexpr int T = kFuseT;
  const float band1 = 1.f + p.band;
  for (int i = lane; i < HS; i += 32) { sh.key[i] = -1; sh.mask[i] = 0u; }
  __syncwarp();
  uint32_t cnt[JM];
#pragma unroll
  for (int j = 0; j < JM; ++j) cnt[j] = 0;
  const int64_t W = *work_count;
  const int64_t gw = (int64_t)blockIdx.x * SW + warp, nw = (int64_t)gridDim.x * SW;
  // worklist entries handed out dynamically in chunks of kSpChunk when p.dyn_ctr is set (see rk_vote_avg.cu)
  const bool dyng = p.dyn_ctr != nullptr;
  auto grab = [&]() -> int64_t {
    unsigned int b = 0;
    if (lane == 0) b = atomicAdd(p.dyn_ctr, (unsigned int)kSpChunk);
    return (int64_t)__shfl_sync(FULL, b, 0);
  };
  for (int64_t cb = dyng ? grab() : gw; cb < W; cb = dyng ? grab() : cb + nw)
  for (int64_t e = cb, ce = dyng ? (cb + kSpChunk < W ? cb + kSpChunk : W) : cb + 1; e < ce; ++e) {
    const int64_t n = work[e];
    const int y = p.labels[n];
    float rmx = 0.f, lsm = 0.f, pyl = 0.f, ptl = 0.f;
    int t1 = -1;
    if (lane < K) {
      const size_t o = (size_t)n * K + lane;
      rmx = p.rmax_in[o];
      lsm = p.lsum_in[o];
      t1 = p.top1_in[o];
      pyl = __expf((ly[o] - rmx) - lsm);
      ptl = __expf((tv[o * T + (T - 1)] - rmx) - lsm);
    }
    float py[kMaxFuseK], pt[kMaxFuseK];
    int top[kMaxFuseK];
#pragma unroll
    for (int m = 0; m < kMaxFuseK; ++m) {
      py[m] = __shfl_sync(FULL, pyl, m);
      pt[m] = __shfl_sync(FULL, ptl, m);
      top[m] = __shfl_sync(FULL, t1, m);
    }
    // 1. merge the K lists by class (y itself is exact and skipped)
    int myslot[(kMaxFuseK * kFuseT) / 32];
#pragma unroll
    for (int r = 0; r < (kMaxFuseK * kFuseT) / 32; ++r) {
      myslot[r] = -1;
      const int ent = lane + 32 * r, m = ent / T;
      const float rm = __shfl_sync(FULL, rmx, m < K ? m : 0), lm = __shfl_sync(FULL, lsm, m < K ? m : 0);
      if (m < K) {
        const size_t o = ((size_t)n * K + m) * T + (ent % T);
        const int c = ti[o];
        if (c != y && c != kFuseNone) {  // (a bound-only entry lists no class; its value is pT_m)
          const float pv = __expf((tv[o] - rm) - lm);
          int h = (int)(((uint32_t)c * 2654435761u) >> 24);
          for (;;) {
            const int old = atomicCAS(&sh.key[h], -1, c);
            if (old == -1 || old == c) break;
            h = (h + 1) & (HS - 1);
          }
          sh.P[h][m] = pv;
          atomicOr(&sh.mask[h], 1u << m);
          myslot[r] = h;
        }
      }
    }
    __syncwarp();
    // 2. threats: classes whose upper bound can reach y's average in some subset with |v| >= 2 (singletons
    // are decided by the top-1); and the same test for the classes no model lists (bound pT_m each)
    float d[kMaxFuseK];
#pragma unroll
    for (int m = 0; m < kMaxFuseK; ++m) d[m] = pt[m] * band1 - py[m];
    const bool oth = K >= 2 && best_pair_sum(d, K) >= 0.f;
    int nthr = 0;
#pragma unroll
    for (int i = 0; i < HS / 32; ++i) {
      const int s = lane + 32 * i;
      bool thr = false;
      if (sh.key[s] != -1) {
        const unsigned int mk = sh.mask[s];
#pragma unroll
        for (int m = 0; m < kMaxFuseK; ++m) d[m] = (((mk >> m) & 1u) ? sh.P[s][m] : pt[m]) * band1 - py[m];
        thr = K >= 2 && best_pair_sum(d, K) >= 0.f;
      }
      const unsigned int b = __ballot_sync(FULL, thr);
      if (thr) sh.list[nthr + __popc(b & ((1u << lane) - 1u))] = s;
      nthr += __popc(b);
    }
    __syncwarp();
    // 3. every subset of this lane: A_v(y) and the unlisted bound, then each threat's LB / UB from its
    // half-mask tables (low models 0-3 index v & 15, high models 4-7 index v >> 4)
    float A[JM], Ab[JM];
    uint32_t lose = 0, und = 0, multi = 0;
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      const uint32_t v = (uint32_t)(lane + 32 * j + 1);
      float a = 0.f, u = 0.f;
#pragma unroll
      for (int m = 0; m < kMaxFuseK; ++m)
        if ((v >> m) & 1u) { a += py[m]; u += pt[m]; }
      A[j] = a;
      Ab[j] = a * band1;
      if (v <= (uint32_t)S && __popc(v) > 1) {
        multi |= 1u << j;
        if (oth && u * band1 >= a) und |= 1u << j;
      }
    }
    for (int t = 0; t < nthr; ++t) {
      const int s = sh.list[t];
      {  // lane l builds entry l & 15 of table (l >> 4): 0 = low models, 1 = high models; LB and UB
        const unsigned int mk = sh.mask[s];
        const int e = lane & 15, hi = lane >> 4;
        float lb = 0.f, ub = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = 4 * hi + i;
          if (m < K && ((e >> i) & 1)) {
            const bool lst = (mk >> m) & 1u;
            const float pm = lst ? sh.P[s][m] : 0.f;
            lb += pm;
            ub += lst ? pm : pt[m];
          }
        }
        sh.tab[lane] = lb;
        sh.tab[32 + lane] = ub;
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < JM; ++j) {
        const uint32_t v = (uint32_t)(lane + 32 * j + 1);
        const int lo = (int)(v & 15u), hi = (int)((v >> 4) & 15u);
        const float LB = sh.tab[lo] + sh.tab[16 + hi];
        const float UB = sh.tab[32 + lo] + sh.tab[48 + hi];
        lose |= (LB > Ab[j]) ? (1u << j) : 0u;
        und |= (UB * band1 >= A[j]) ? (1u << j) : 0u;
      }
      __syncwarp();
    }
    uint32_t okm = 0;
#pragma unroll
    for (int j = 0; j < JM; ++j) {
      const uint32_t v = (uint32_t)(lane + 32 * j + 1);
      if (v > (uint32_t)S) break;
      if (!((multi >> j) & 1u)) okm |= (top[__ffs(v) - 1] == y) ? (1u << j) : 0u;  // singleton: top-1 (I1)
      else if (!((lose >> j) & 1u) && !((und >> j) & 1u)) okm |= 1u << j;
    }
    const bool undecided = (und & ~lose & multi) != 0u;
    if (__any_sync(FULL, undecided)) {
      if (lane == 0) fb[atomicAdd(fb_count, 1u)] = (int32_t)n;
    } else {
#pragma unroll
      for (int j = 0; j < JM; ++j) cnt[j] += (okm >> j) & 1u;
    }
    // 4. clear this sample's hash slots
    __syncwarp();
#pragma unroll
    for (int r = 0; r < (kMaxFuseK * kFuseT) / 32; ++r)
      if (myslot[r] >= 0) { sh.key[myslot[r]] = -1; sh.mask[myslot[r]] = 0u; }
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < JM; ++j) {
    const int v1 = lane + 32 * j;
    if (v1 < S && cnt[j]) atomicAdd(p.cnt_avg + v1, (unsigned long long)cnt[j]);
  }
}

// fallback rows: compact copies of their features (bf16 [D]) and labels
__global__ void gather_rows_kernel(const uint16_t* X, int D, const int32_t* labels, const int32_t* idx,
                                   const unsigned int* count, uint16_t* Xc, int32_t* yc, int32_t* iota) {
  const int64_t M = *count;
  const int per = D / 8;  // uint4 = 8 bf16
  for (int64_t i = blockIdx.x; i < M; i += gridDim.x) {
    const int64_t n = idx[i];
    const uint4* src = reinterpret_cast<const uint4*>(X + (size_t)n * D);
    uint4* dst = reinterpret_cast<uint4*>(Xc + (size_t)i * D);
    for (int k = threadIdx.x; k < per; k += blockDim.x) dst[k] = src[k];
    if (threadIdx.x == 0) { yc[i] = labels[n]; iota[i] = (int32_t)i; }
  }
}

}  // namespace

cudaError_t launch_vote_sparse(const VoteParams& p, const float* ly, const float* tv, const uint16_t* ti,
                               const int32_t* work, const unsigned int* work_count, int32_t* fb,
                               unsigned int* fb_count, int sm_count, cudaStream_t st) {
  if (p.K > kMaxFuseK) return cudaErrorInvalidValue;
  if (p.dyn_ctr) {
    const cudaError_t e = cudaMemsetAsync(p.dyn_ctr, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return e;
  }
  vote_sparse_average_kernel<<<sm_count * 8, 32 * SW, 0, st>>>(p, ly, tv, ti, work, work_count, fb, fb_count);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const uint16_t* X, int D, const int32_t* labels, const int32_t* idx,
                               const unsigned int* count, int64_t M, uint16_t* Xc, int32_t* yc, int32_t* iota,
                               cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  const int64_t g = M < 148 * 16 ? M : 148 * 16;
  gather_rows_kernel<<<(unsigned)g, 256, 0, st>>>(X, D, labels, idx, count, Xc, yc, iota);
  return cudaGetLastError();
}

}  // namespace rk
