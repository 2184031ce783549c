// rk_vote_batch_avg.cu — step A4 for K = 9..12 (511..4095 subsets): averaged-probability decision
// of every subset for the worklist samples, batch-transposed.
//
// PAPER.md:72 (softmax average, readings Q5/Q6), :429 (action space). Exactness arguments as in
// rk_vote_avg.cu: R = S_c ∩ {c : exists m, l[m][c] >= l[m][y]}; exact half-mask tables for y and the
// members' distinct top-1 classes (D); a bound on every other candidate; scan R when the bound is
// not conclusive; fp64 recheck inside the relative band.
//
// Layout: a CTA takes SBW worklist samples (one per warp). Phase 1: each warp builds its sample's
// record (candidate set, gathered probabilities, tables) in shared memory. Phase 2: every thread owns
// subsets v = t + 1 + 256k and sweeps the SBW records (uniform control flow, broadcast reads,
// register counters). Phase 3 (rare): fp64 log-sum-exp of flagged samples, then pending pairs.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int BT = 256;
constexpr int SBW = BT / 32;   // worklist samples per batch: one per warp
constexpr int KM = 12;
constexpr int DSTR = 13;       // exact columns: y + up to 12 distinct top-1 classes (odd stride)

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float f4c(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }


struct SmpB {   // per-sample arrays in the CTA's dynamic smem
  float* P;     // [K][CAP+1]
  float* T;     // [TT][DSTR] exact-column half-mask sums (col 0 = y)
  float* QB;    // [TT] bound half-mask sums
  int32_t* cls; // [CAP]
  uint32_t* bm; // [32]
  uint32_t* bmB;// [32]
};

__host__ __device__ inline size_t smp_bytes(const VoteParams& p, char* base, SmpB* s) {
  const int TT = (1 << p.K1) + (1 << (p.K - p.K1));
  size_t o = 0;
  auto take = [&](size_t b) -> char* { char* r = base ? base + o : nullptr; o = a16(o + b); return r; };
  char* P = take(4ull * p.K * (p.CAP + 1));
  char* T = take(4ull * TT * DSTR);
  char* QB = take(4ull * TT);
  char* cl = take(4ull * p.CAP);
  char* bm = take(4 * 32);
  char* bmB = take(4 * 32);
  if (s) { s->P = (float*)P; s->T = (float*)T; s->QB = (float*)QB; s->cls = (int32_t*)cl; s->bm = (uint32_t*)bm; s->bmB = (uint32_t*)bmB; }
  return o;
}

struct HdrB {  // per-sample scalars
  int64_t n;
  int32_t y, nc, ys, nd, valid, ovf, need64;
  int32_t top[KM];
  int32_t dslot[KM];
  float mx[KM];
  float q[KM];
  double sum64[KM];
};

template <int NK>
__global__ void __launch_bounds__(BT, 2) vote_batch_average_kernel(const VoteParams p, const int32_t* work,
                                                                   const unsigned int* work_count) {
  extern __shared__ __align__(16) char smem_raw[];
  __shared__ HdrB hd[SBW];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, S = p.S, C = p.C;
  const int F = (int)(p.ldc >> 2);
  const int TA = 1 << p.K1, TT = TA + (1 << (K - p.K1));
  const int CAPS = p.CAP + 1;
  const size_t sbytes = smp_bytes(p, nullptr, nullptr);
  const int64_t W = *work_count;
  const int64_t nbatch = (W + SBW - 1) / SBW;
  uint32_t ca[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) ca[k] = 0;

  for (int64_t batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
    __syncthreads();
    // ---- phase 1: warp `warp` prepares worklist sample e ---------------------------------------
    {
      const int64_t e = batch * SBW + warp;
      SmpB sm;
      smp_bytes(p, smem_raw + warp * sbytes, &sm);
      if (e < W) {
        const int64_t n = work[e];
        const int y = p.labels[n];
        const float* rowbase = p.logits + n * K * p.ldc;
        int tp = 0;
        float mx = 0.f, ls = 0.f;
        if (lane < K) { tp = p.top1_in[n * K + lane]; ls = p.lsum_in[n * K + lane]; mx = p.rmax_in[n * K + lane]; }
        const float thr = theta_threshold(mx, ls, K, lane);
        const float ly = lane < K ? rowbase[(size_t)lane * p.ldc + y] : INFINITY;
        sm.bm[lane] = 0u;
        sm.bmB[lane] = 0u;
        __syncwarp();
#pragma unroll 1
        for (int m = 0; m < K; ++m) {  // R: one streaming pass
          const float* row = rowbase + (size_t)m * p.ldc;
          const float t_m = __shfl_sync(FULL, thr, m), y_m = __shfl_sync(FULL, ly, m);
          const float lo = fminf(t_m, y_m);
#pragma unroll 1
          for (int c4 = lane; c4 < F; c4 += 32) {
            if (c4 * 4 >= C) continue;
            const float4 x4 = ldg_stream(row + c4 * 4);
            if (fmaxf(fmaxf(x4.x, x4.y), fmaxf(x4.z, x4.w)) >= lo) {
              const int cb = c4 * 4;
              uint32_t bits = 0, bitsB = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float x = f4c(x4, q);
                bits |= (x >= t_m && cb + q < C) ? (1u << q) : 0u;
                bitsB |= (x >= y_m && cb + q < C) ? (1u << q) : 0u;
              }
              if (bits) atomicOr(&sm.bm[cb >> 5], bits << (cb & 31));
              if (bitsB) atomicOr(&sm.bmB[cb >> 5], bitsB << (cb & 31));
            }
          }
        }
        __syncwarp();
        const uint32_t word = sm.bm[lane] & sm.bmB[lane];
        const int cnt = __popc(word);
        int incl = cnt;
        for (int off = 1; off < 32; off <<= 1) {
          const int o = __shfl_up_sync(FULL, incl, off);
          if (lane >= off) incl += o;
        }
        const int pre = incl - cnt;
        const int nc = __shfl_sync(FULL, incl, 31);
        auto slot_of = [&](int c) -> int {
          return __shfl_sync(FULL, pre, c >> 5) + __popc(__shfl_sync(FULL, word, c >> 5) & ((1u << (c & 31)) - 1u));
        };
        const int ys = slot_of(y);
        const bool ovf = nc > p.CAP;
        float* P = ovf ? p.scratch + ((size_t)blockIdx.x * SBW + warp) * (size_t)K * C : sm.P;
        int32_t* cls = ovf ? p.scratch_cls + ((size_t)blockIdx.x * SBW + warp) * (size_t)C : sm.cls;
        const int ps = ovf ? C : CAPS;
        {
          uint32_t w = word;
          int k = pre;
          while (w) { cls[k++] = lane * 32 + (__ffs(w) - 1); w &= w - 1; }
        }
        int nd = 0;
        for (int m = 0; m < K; ++m) {  // distinct top-1 classes other than y (all in R)
          const int cm = __shfl_sync(FULL, tp, m);
          bool dup = cm == y;
          for (int q = 0; q < m; ++q) dup |= (__shfl_sync(FULL, tp, q) == cm);
          if (!dup) {
            const int sl = slot_of(cm);
            if (lane == 0) hd[warp].dslot[nd] = sl;
            ++nd;
          }
        }
        __syncwarp();
        for (int m = 0; m < K; ++m) {
          const float ls_m = __shfl_sync(FULL, ls, m), mx_m = __shfl_sync(FULL, mx, m);
          for (int sl = lane; sl < nc; sl += 32)
            P[(size_t)m * ps + sl] = expf((__ldg(rowbase + (size_t)m * p.ldc + cls[sl]) - mx_m) - ls_m);
        }
        __syncwarp();
        for (int m = 0; m < K; ++m) {  // bound for candidates outside {y} ∪ D
          float q = 0.f;
          for (int sl = lane; sl < nc; sl += 32) {
            bool ex = sl == ys;
            for (int d = 0; d < nd; ++d) ex |= sl == hd[warp].dslot[d];
            if (!ex) q = fmaxf(q, P[(size_t)m * ps + sl]);
          }
          for (int off = 16; off; off >>= 1) q = fmaxf(q, __shfl_xor_sync(FULL, q, off));
          if (lane == 0) hd[warp].q[m] = q;
        }
        __syncwarp();
        for (int h = lane; h < TT; h += 32) {  // half-mask rows: bound and exact columns
          const uint32_t hm = h < TA ? (uint32_t)h : (uint32_t)(h - TA);
          const int mo = h < TA ? 0 : p.K1;
          float s = 0.f;
          for (uint32_t a = hm; a; a &= a - 1) s += hd[warp].q[mo + __ffs(a) - 1];
          sm.QB[h] = s * (1.f + 1e-6f);
          for (int d = 0; d <= nd; ++d) {
            const int sl = d == 0 ? ys : hd[warp].dslot[d - 1];
            float x = 0.f;
            for (uint32_t a = hm; a; a &= a - 1) x += P[(size_t)(mo + __ffs(a) - 1) * ps + sl];
            sm.T[(size_t)h * DSTR + d] = x;
          }
        }
        if (lane < K) { hd[warp].top[lane] = tp; hd[warp].mx[lane] = mx; }
        if (lane == 0) {
          hd[warp].n = n; hd[warp].y = y; hd[warp].nc = nc; hd[warp].ys = ys; hd[warp].nd = nd;
          hd[warp].valid = 1; hd[warp].ovf = ovf; hd[warp].need64 = 0;
        }
      } else if (lane == 0) {
        hd[warp].valid = 0;
      }
    }
    __syncthreads();
    // ---- phase 2: thread t owns subsets v = t + 1 + 256k ---------------------------------------
    uint32_t pending[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) pending[k] = 0;
#pragma unroll 1
    for (int s = 0; s < SBW; ++s) {
      if (!hd[s].valid) continue;
      SmpB sm;
      smp_bytes(p, smem_raw + s * sbytes, &sm);
      const int y = hd[s].y, nc = hd[s].nc, ys = hd[s].ys, nd = hd[s].nd;
      const bool ovf = hd[s].ovf;
      const float* P = ovf ? p.scratch + ((size_t)blockIdx.x * SBW + s) * (size_t)K * C : sm.P;
      const int ps = ovf ? C : CAPS;
#pragma unroll
      for (int k = 0; k < NK; ++k) {  // A4
        const uint32_t v = (uint32_t)(t + 1 + BT * k);
        if (v > (uint32_t)S) break;
        uint32_t oka = 0;
        if (__popc(v) == 1) {
          oka = hd[s].top[__ffs(v) - 1] == y;  // softmax is monotone (invariant I1)
        } else {
          const uint32_t a = v & (TA - 1), bb = TA + (v >> p.K1);
          const float* A = sm.T + (size_t)a * DSTR;
          const float* B = sm.T + (size_t)bb * DSTR;
          const float sy = A[0] + B[0];
          const float hiT = sy * (1.f + p.band), loT = sy * (1.f - p.band);
          bool beat = false, near = false;
#pragma unroll 1
          for (int d = 1; d <= nd; ++d) {
            const float sd = A[d] + B[d];
            beat |= sd > hiT;
            near |= sd >= loT;
          }
          if (beat) {
            oka = 0;
          } else if (sm.QB[a] + sm.QB[bb] < loT) {
            if (near) { pending[k] |= 1u << s; hd[s].need64 = 1; }
            else oka = 1;
          } else {
            float m2 = -1.f;
            for (int q = 0; q < nc; ++q) {
              if (q == ys) continue;
              float x = 0.f;
              for (uint32_t m = v; m; m &= m - 1) x += P[(size_t)(__ffs(m) - 1) * ps + q];
              m2 = fmaxf(m2, x);
            }
            if (m2 > hiT) oka = 0;
            else if (m2 < loT) oka = 1;
            else { pending[k] |= 1u << s; hd[s].need64 = 1; }
          }
        }
        ca[k] += oka;
      }
    }
    __syncthreads();
    // ---- phase 3 (rare): fp64 log-sum-exp of flagged samples (warp each), then pending pairs ----
    if (hd[warp].valid && hd[warp].need64) {
      const float* rowbase = p.logits + hd[warp].n * K * p.ldc;
      for (int m = 0; m < K; ++m) {
        const double m64 = (double)hd[warp].mx[m];
        double s = 0.0;
        for (int c = lane; c < C; c += 32) s += exp((double)rowbase[(size_t)m * p.ldc + c] - m64);
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
        if (lane == 0) hd[warp].sum64[m] = s;  // sum_c exp(l - hd.mx[m])
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      uint32_t pm = pending[k];
      while (pm) {
        const int s = __ffs(pm) - 1;
        pm &= pm - 1;
        const uint32_t v = (uint32_t)(t + 1 + BT * k);
        atomicAdd(p.n_recheck + (v - 1), 1ull);
        SmpB sm;
        smp_bytes(p, smem_raw + s * sbytes, &sm);
        const int y = hd[s].y, nc = hd[s].nc, ys = hd[s].ys;
        const bool ovf = hd[s].ovf;
        const float* P = ovf ? p.scratch + ((size_t)blockIdx.x * SBW + s) * (size_t)K * C : sm.P;
        const int32_t* cls = ovf ? p.scratch_cls + ((size_t)blockIdx.x * SBW + s) * (size_t)C : sm.cls;
        const int ps = ovf ? C : CAPS;
        const float* rowbase = p.logits + hd[s].n * K * p.ldc;
        float sy = 0.f;
        for (uint32_t m = v; m; m &= m - 1) sy += P[(size_t)(__ffs(m) - 1) * ps + ys];
        const float lo = sy * (1.f - p.band);
        double best = -1.0;
        int bestc = 0x7fffffff;
        for (int q = 0; q < nc; ++q) {
          float s32 = 0.f;
          for (uint32_t m = v; m; m &= m - 1) s32 += P[(size_t)(__ffs(m) - 1) * ps + q];
          if (q != ys && s32 < lo) continue;
          const int cq = cls[q];
          double acc = 0.0;
          for (uint32_t m = v; m; m &= m - 1) {
            const int mi = __ffs(m) - 1;
            acc += exp((double)rowbase[(size_t)mi * p.ldc + cq] - (double)hd[s].mx[mi]) / hd[s].sum64[mi];
          }
          const double a64 = acc / (double)__popc(v);
          if (a64 > best || (a64 == best && cq < bestc)) { best = a64; bestc = cq; }
        }
        ca[k] += (bestc == y);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int v1 = t + BT * k;
    if (v1 < S && ca[k]) atomicAdd(p.cnt_avg + v1, (unsigned long long)ca[k]);
  }
}

template <int NK>
cudaError_t launch_avg_nk(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                          const unsigned int* work_count) {
  const size_t smem = smp_bytes(q, nullptr, nullptr) * SBW;
  cudaError_t e = cudaFuncSetAttribute(vote_batch_average_kernel<NK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int per_sm = smem <= 100 * 1024 ? 2 : 1;
  vote_batch_average_kernel<NK><<<sm_count * per_sm, BT, smem, st>>>(q, work, work_count);
  return cudaGetLastError();
}

}  // namespace

size_t vote_batch_smem_per_sample(const VoteParams& p) { return smp_bytes(p, nullptr, nullptr); }
int vote_batch_avg_ctas_samples() { return 2 * SBW; }  // overflow-scratch owners per SM

cudaError_t launch_vote_batch_avg(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                                  const unsigned int* work_count) {
  const int nk = (q.S + BT - 1) / BT;
  if (nk <= 2) return launch_avg_nk<2>(q, sm_count, st, work, work_count);
  if (nk <= 4) return launch_avg_nk<4>(q, sm_count, st, work, work_count);
  if (nk <= 8) return launch_avg_nk<8>(q, sm_count, st, work, work_count);
  return launch_avg_nk<16>(q, sm_count, st, work, work_count);
}

}  // namespace rk
