// rk_predict.cu — per-sample outputs of ONE action v on the last scored batch (serving step NEXT-1,
// and the parity hook for invariant I4): majority-vote prediction, averaged-probability
// prediction and the averaged probability vector. One warp per sample.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {
constexpr unsigned FULL = 0xffffffffu;
}  // namespace

// ---- rk_predict: per-sample outputs of one action v (plain, one warp per sample) -------------------
__global__ void predict_kernel(const PredictParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int K = p.K, C = p.C;
  for (int64_t n = warp; n < p.N; n += nwarps) {
    int top[kMaxK];
    float mxs[kMaxK], lsum[kMaxK];
    for (int m = 0; m < K; ++m) {
      const float* row = p.logits + (n * K + m) * p.ldc;
      float mx = -INFINITY;
      int arg = 0x7fffffff;
      for (int c = lane; c < C; c += 32) {
        const float x = row[c];
        if (x > mx) { mx = x; arg = c; }
      }
      for (int off = 16; off; off >>= 1) {
        const float om = __shfl_xor_sync(FULL, mx, off);
        const int oa = __shfl_xor_sync(FULL, arg, off);
        if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
      }
      float s = 0.f;
      for (int c = lane; c < C; c += 32) s += __expf(row[c] - mx);
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
      top[m] = arg;
      mxs[m] = mx;
      lsum[m] = logf(s);  // relative to the row max: p = exp((l - mx) - lsum) is exact for any offset
    }
    // vote
    if (p.pred_vote && lane == 0) {
      int bestc = -1, bestcnt = 0;
      uint32_t tied = 0;
      for (int m = 0; m < K; ++m) {
        if (!((p.v >> m) & 1u)) continue;
        uint32_t mk = 0;
        for (int q = 0; q < K; ++q)
          if (((p.v >> q) & 1u) && top[q] == top[m]) mk |= 1u << q;
        const int cnt = __popc(mk);
        if (cnt > bestcnt || (cnt == bestcnt && top[m] < bestc)) { bestcnt = cnt; bestc = top[m]; }
      }
      for (int m = 0; m < K; ++m) {
        if (!((p.v >> m) & 1u)) continue;
        uint32_t mk = 0;
        for (int q = 0; q < K; ++q)
          if (((p.v >> q) & 1u) && top[q] == top[m]) mk |= 1u << q;
        if (__popc(mk) == bestcnt) tied |= 1u << m;
      }
      p.pred_vote[n] = p.tie == 0 ? top[p.best_of[tied]] : bestc;
    }
    // average (fp32 probabilities; lowest class on ties)
    if (p.pred_avg || p.avgprob) {
      const float inv = 1.f / (float)__popc(p.v);
      float bm = -1.f;
      int bc = 0x7fffffff;
      for (int c = lane; c < C; c += 32) {
        float s = 0.f;
        for (int m = 0; m < K; ++m)
          if ((p.v >> m) & 1u) s += expf((p.logits[(n * K + m) * p.ldc + c] - mxs[m]) - lsum[m]);
        const float a = s * inv;
        if (p.avgprob) p.avgprob[n * C + c] = a;
        if (a > bm) { bm = a; bc = c; }
      }
      for (int off = 16; off; off >>= 1) {
        const float om = __shfl_xor_sync(FULL, bm, off);
        const int oc = __shfl_xor_sync(FULL, bc, off);
        if (om > bm || (om == bm && oc < bc)) { bm = om; bc = oc; }
      }
      if (p.pred_avg && lane == 0) p.pred_avg[n] = bc;
    }
  }
}

cudaError_t launch_predict(const PredictParams& p, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  int64_t blocks = (p.N + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  predict_kernel<<<(int)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rk
