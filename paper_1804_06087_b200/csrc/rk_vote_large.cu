// rk_vote_large.cu — step A4 for rows wider than the register/shared-memory kernels hold (ldc > 1024,
// up to C = 65535, any K <= 12): averaged-probability decision of every subset for the worklist samples,
// one CTA per sample, decided from the definition in fp64.
//
// PAPER.md:72 "ensemble multiple models and average the results" (softmax average, reading Q5; lowest
// class on ties, Q6); :429 every non-empty subset is an action. SURVEY.md §8(b) fixes C in [2, 65535].
//
// Per sample (the classify kernel has already decided votes, unanimity and that y is a candidate):
//   1. one coalesced pass over the K rows: the fp64 softmax denominators s_m = sum_c exp(l - mx_m) and
//      the candidate set R = S_c ∩ {c : exists m, l[m][c] >= l[m][y]} minus y (θ pruning, SURVEY.md §8(d):
//      if y is not the averaged argmax of v, the argmax lies in R and beats y; if it is, nothing in R does);
//   2. p[m][j] = exp(l[m][c_j] - mx_m) / s_m in fp64 for y and the members of R (shared memory);
//   3. thread t owns subsets v = t + 1 + 256 k: y is correct iff no c in R has avg_v[c] > avg_v[y], or an
//      equal average with c < y (avg = (sum_{m in v, ascending} p[m][c]) / |v|, the definition's order).
//      Singletons use the top-1 (softmax is monotone, invariant I1). Pairs whose relative gap is within
//      `band` are counted in n_recheck (they are the pairs an fp32 path would have rechecked).
// When R exceeds the shared-memory capacity (e.g. flat rows) the sweep reads the logits again and tests
// every class: slower, same result. Throughput is not a goal here (no bench config has C > 1000).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LT = 256;      // threads per CTA
constexpr int LW = LT / 32;
constexpr int LCAP = 384;    // candidates held in shared memory (y is slot LCAP)

struct LargeSmem {
  double P[kMaxK][LCAP + 1];  // p[m][j], j = LCAP -> y
  double s[kMaxK];            // sum_c exp(l - mx_m)
  double part[LW][kMaxK];
  int32_t cls[LCAP];
  float mx[kMaxK], thr[kMaxK], ly[kMaxK];
  int32_t top[kMaxK];
  int32_t y, nc;
  uint32_t cnt[4096], rc[4096];  // per-subset counters of this CTA (v - 1), thread-owned
};

__global__ void __launch_bounds__(LT, 1) vote_large_average_kernel(const VoteParams p, const int32_t* work,
                                                                    const unsigned int* work_count) {
  extern __shared__ __align__(16) char smem_raw[];
  LargeSmem& sh = *reinterpret_cast<LargeSmem*>(smem_raw);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, C = p.C, S = p.S;
  for (int i = t; i < S; i += LT) { sh.cnt[i] = 0u; sh.rc[i] = 0u; }
  const int64_t W = *work_count;
  for (int64_t e = blockIdx.x; e < W; e += gridDim.x) {
    const int64_t n = work[e];
    const float* rowbase = p.logits + n * K * p.ldc;
    if (warp == 0) {
      float mx = 0.f, ls = 0.f;
      int tp = 0;
      if (lane < K) { tp = p.top1_in[n * K + lane]; ls = p.lsum_in[n * K + lane]; mx = p.rmax_in[n * K + lane]; }
      const float thr = theta_threshold(mx, ls, K, lane);
      const int y = p.labels[n];
      if (lane < K) {
        sh.top[lane] = tp; sh.mx[lane] = mx; sh.thr[lane] = thr;
        sh.ly[lane] = rowbase[(size_t)lane * p.ldc + y];
      }
      if (lane == 0) { sh.y = y; sh.nc = 0; }
    }
    __syncthreads();
    const int y = sh.y;
    // ---- 1. denominators and candidates: one pass, threads stride the classes ----------------------
    double sp[kMaxK];
#pragma unroll
    for (int m = 0; m < kMaxK; ++m) sp[m] = 0.0;
    for (int c = t; c < C; c += LT) {
      bool ins = false, nb = false;
#pragma unroll
      for (int m = 0; m < kMaxK; ++m) {
        if (m < K) {
          const float x = rowbase[(size_t)m * p.ldc + c];
          sp[m] += exp((double)x - (double)sh.mx[m]);
          ins |= x >= sh.thr[m];
          nb |= x >= sh.ly[m];
        }
      }
      if (ins && nb && c != y) {
        const int slot = atomicAdd(&sh.nc, 1);
        if (slot < LCAP) sh.cls[slot] = c;
      }
    }
#pragma unroll
    for (int m = 0; m < kMaxK; ++m) {
      if (m < K) {
        double v = sp[m];
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
        if (lane == 0) sh.part[warp][m] = v;
      }
    }
    __syncthreads();
    if (t < K) {
      double v = 0.0;
      for (int w = 0; w < LW; ++w) v += sh.part[w][t];
      sh.s[t] = v;
    }
    __syncthreads();
    const int nc = sh.nc;
    const bool fits = nc <= LCAP;
    // ---- 2. fp64 probabilities of the candidates (and of y, slot LCAP) -------------------------------
    if (fits) {
      for (int i = t; i < K * (nc + 1); i += LT) {
        const int m = i / (nc + 1), j = i - m * (nc + 1);
        const int c = j < nc ? sh.cls[j] : y;
        sh.P[m][j < nc ? j : LCAP] = exp((double)rowbase[(size_t)m * p.ldc + c] - (double)sh.mx[m]) / sh.s[m];
      }
    }
    __syncthreads();
    // ---- 3. every subset --------------------------------------------------------------------------
    for (int v1 = t; v1 < S; v1 += LT) {
      const uint32_t v = (uint32_t)v1 + 1u;
      if (__popc(v) == 1) {
        sh.cnt[v1] += (uint32_t)(sh.top[__ffs(v) - 1] == y);
        continue;
      }
      const double nv = (double)__popc(v);
      double sy = 0.0;
      for (uint32_t a = v; a; a &= a - 1) {
        const int m = __ffs(a) - 1;
        sy += fits ? sh.P[m][LCAP] : exp((double)rowbase[(size_t)m * p.ldc + y] - (double)sh.mx[m]) / sh.s[m];
      }
      const double ay = sy / nv;
      bool beat = false, near = false;
      const int nj = fits ? nc : C;
      for (int j = 0; j < nj && !beat; ++j) {
        const int c = fits ? sh.cls[j] : j;
        if (c == y) continue;
        double s = 0.0;
        for (uint32_t a = v; a; a &= a - 1) {
          const int m = __ffs(a) - 1;
          s += fits ? sh.P[m][j] : exp((double)rowbase[(size_t)m * p.ldc + c] - (double)sh.mx[m]) / sh.s[m];
        }
        const double ac = s / nv;
        beat = ac > ay || (ac == ay && c < y);
        near |= ac >= ay * (1.0 - (double)p.band);
      }
      sh.cnt[v1] += (uint32_t)!beat;
      sh.rc[v1] += (uint32_t)near;
    }
    __syncthreads();  // shared state of this sample is reused by the next
  }
  for (int i = t; i < S; i += LT) {
    if (sh.cnt[i]) atomicAdd(p.cnt_avg + i, (unsigned long long)sh.cnt[i]);
    if (sh.rc[i]) atomicAdd(p.n_recheck + i, (unsigned long long)sh.rc[i]);
  }
}

}  // namespace

bool vote_large_needed(const VoteParams& q) { return q.ldc > kMaxCFast; }

cudaError_t launch_vote_large_avg(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                                  const unsigned int* work_count) {
  const size_t smem = sizeof(LargeSmem);
  cudaError_t e = cudaFuncSetAttribute(vote_large_average_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  vote_large_average_kernel<<<sm_count, LT, smem, st>>>(q, work, work_count);
  return cudaGetLastError();
}

}  // namespace rk
