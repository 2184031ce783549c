// rk_vote_avg.cu — step A4 for K <= 8: averaged-probability decision of every subset for the
// worklist samples (label y is an averaging candidate), one WARP per sample.
//
// PAPER.md:72 "ensemble multiple models and average the results" (softmax average, reading Q5;
// lowest class on ties, Q6); :429 every non-empty subset is an action.
//
// Per sample:
//   1. one coalesced streaming pass over the K*ldc logits marks
//        R = S_c ∩ {c : exists m, l[m][c] >= l[m][y]}
//      S_c = {c : exists m, p[m][c] >= theta}, theta = min_j p[j][top_j] / K (the averaged argmax of
//      every subset lies in S_c); a class below y in EVERY model has
//      avg_v[c] < avg_v[y] for all v and can never decide whether y wins;
//   2. p[m][c] = exp((l - mx_m) - lsum_m) is gathered for c in R (slots in class order, warp scan);
//   3. the members' distinct top-1 classes other than y (D, at most K) are the natural competitors:
//      their subset sums, and y's, come from half-mask tables (one add per subset and column);
//      every other candidate is bounded by Q[v] = sum_{m in v} max_{c in R \ ({y} ∪ D)} p[m][c];
//   4. per subset: a D-class clearly above y -> wrong; D and the bound clearly below -> right;
//      bound not conclusive -> scan R; decisions inside the relative band `band` are redone in fp64
//      (warp-cooperative fp64 log-sum-exp, then eq. (2) of PAPER.md:72 in fp64) -- rare.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WT = 128;  // threads per CTA (4 warps)
constexpr int WPC = WT / 32;
constexpr int kAvgChunk = 2;  // worklist entries per dynamic grab (REC path)
constexpr int JMAX = 8;  // subsets per lane (S <= 255)
constexpr int DSTR = 9;  // exact columns: y + up to 8 distinct top-1 classes (odd stride)

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }


struct WS {  // per-warp shared memory
  double* sum64;    // [16]: [0,8) sum_c exp(l - mx) in fp64, [8,16) the row max mx
  int32_t* stop;    // [8] top-1 per model
  uint32_t* bitmap; // [32] R = S_c (theta test) ∩ classes not below y in some model
  int32_t* ccls;    // [CAP] candidate classes in ascending order
  float* P;         // [K][CAP+1]
  float* T;         // [32][DSTR] half-mask sums of the exact columns (col 0 = y, 1.. = D)
  float* QB;        // [32] half-mask sums of the competitor bound
  float* Q;         // [8]
  uint32_t* cnt;    // [JMAX][32] lane-owned avg counters
};

__host__ __device__ inline size_t warp_smem(const VoteParams& p, char* base, WS* w) {
  size_t o = 0;
  auto take = [&](size_t b) -> char* { char* r = base ? base + o : nullptr; o = a16(o + b); return r; };
  char* l64 = take(16 * 8);
  char* st = take(4 * 8);
  char* bm = take(4 * 32);
  char* cc = take(4ull * p.CAP);
  char* P = take(4ull * p.K * (p.CAP + 1));
  char* T = take(4ull * 32 * DSTR);
  char* QB = take(4 * 32);
  char* Q = take(4 * 8);
  char* CN = take(4 * JMAX * 32);
  if (w) {
    w->sum64 = (double*)l64; w->stop = (int32_t*)st; w->bitmap = (uint32_t*)bm;
    w->ccls = (int32_t*)cc; w->P = (float*)P; w->T = (float*)T; w->QB = (float*)QB; w->Q = (float*)Q;
    w->cnt = (uint32_t*)CN;
  }
  return o;
}

// Near-ties (rare, out of line). First the exact ties: when every candidate inside the band has the
// same logit as y in every member of v, its average equals y's in any precision (same terms, same
// order), so the lowest class wins (reading Q6) without fp64 -- 86 % of the pending subsets of the
// integer-grid bench workload. The rest: warp-cooperative fp64 log-sum-exp of every row, then each lane
// decides its remaining subsets in fp64 per readings Q5-Q6 (avg = (sum_{m in v, asc} exp(l - mx_m) /
// sum_c exp(l - mx_m)) / |v|, lowest class on ties; softmax with max subtraction, reading Q5) over the
// candidates inside the band.
__device__ __noinline__ void recheck_fp64(const VoteParams& p, WS& ws, uint32_t pending, const float* rowbase,
                                          float mx, const float* Pm, int ps, const int32_t* cls, int nc, int ys,
                                          int y, int lane) {
  const int K = p.K, C = p.C;
  uint32_t left = 0;
  for (int j = 0; j < JMAX; ++j) {
    if (!((pending >> j) & 1u)) continue;
    const uint32_t v = (uint32_t)(lane + 32 * j + 1);
    atomicAdd(p.n_recheck + (v - 1), 1ull);
    float sy = 0.f;
    for (uint32_t a = v; a; a &= a - 1) sy += Pm[(size_t)(__ffs(a) - 1) * ps + ys];
    const float lo = sy * (1.f - p.band);
    bool tie = true, ywins = true;
    for (int q = 0; q < nc && tie; ++q) {
      if (q == ys) continue;
      float s32 = 0.f;
      for (uint32_t a = v; a; a &= a - 1) s32 += Pm[(size_t)(__ffs(a) - 1) * ps + q];
      if (s32 < lo) continue;
      const int cq = cls[q];
      for (uint32_t a = v; a && tie; a &= a - 1) {
        const float* r = rowbase + (size_t)(__ffs(a) - 1) * p.ldc;
        tie = r[cq] == r[y];
      }
      ywins &= y < cq;
    }
    if (tie) ws.cnt[j * 32 + lane] += ywins;
    else left |= 1u << j;
  }
  if (!__any_sync(FULL, left != 0)) return;
  pending = left;
  for (int m = 0; m < K; ++m) {
    const float* row = rowbase + (size_t)m * p.ldc;
    const double m64 = (double)__shfl_sync(FULL, mx, m);
    double s = 0.0;
    for (int cc = lane; cc < C; cc += 32) s += exp((double)row[cc] - m64);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
    if (lane == 0) { ws.sum64[m] = s; ws.sum64[8 + m] = m64; }
  }
  __syncwarp();
  for (int j = 0; j < JMAX; ++j) {
    if (!((pending >> j) & 1u)) continue;
    const uint32_t v = (uint32_t)(lane + 32 * j + 1);
    float sy = 0.f;  // fp32 sums select the band; fp64 decides
    for (uint32_t a = v; a; a &= a - 1) sy += Pm[(size_t)(__ffs(a) - 1) * ps + ys];
    const float lo = sy * (1.f - p.band);
    const int nv = __popc(v);
    double best = -1.0;
    int bestc = 0x7fffffff;
    for (int q = 0; q < nc; ++q) {
      float s32 = 0.f;
      for (uint32_t a = v; a; a &= a - 1) s32 += Pm[(size_t)(__ffs(a) - 1) * ps + q];
      if (q != ys && s32 < lo) continue;
      const int cq = cls[q];
      double s = 0.0;
      for (uint32_t a = v; a; a &= a - 1) {
        const int m = __ffs(a) - 1;
        s += exp((double)rowbase[(size_t)m * p.ldc + cq] - ws.sum64[8 + m]) / ws.sum64[m];
      }
      const double a64 = s / (double)nv;
      if (a64 > best || (a64 == best && cq < bestc)) { best = a64; bestc = cq; }
    }
    ws.cnt[j * 32 + lane] += (bestc == y);
  }
  __syncwarp();
}

#ifndef RK_AVG_MINB
#define RK_AVG_MINB 7
#endif
template <bool REC>
__global__ void __launch_bounds__(WT, RK_AVG_MINB) vote_average_kernel(const VoteParams p, const int32_t* work,
                                                              const unsigned int* work_count) {
  extern __shared__ __align__(16) char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WS ws;
  warp_smem(p, smem_raw + warp * warp_smem(p, nullptr, nullptr), &ws);
  const int K = p.K, S = p.S, C = p.C;
  const int TA = 1 << p.K1, TT = TA + (1 << (K - p.K1));
  const int CAPS = p.CAP + 1;
  const int64_t gw = (int64_t)blockIdx.x * WPC + warp;
  const int64_t nw = (int64_t)gridDim.x * WPC;
  float* ovP = p.scratch + gw * (size_t)K * C;  // overflow candidate matrix [K][C]
  int32_t* ovC = p.scratch_cls + gw * (size_t)C;
  for (int i = lane; i < JMAX * 32; i += 32) ws.cnt[i] = 0u;
  const int64_t W = *work_count;
  // REC: the classify kernel's record of worklist entry e (lane i holds word i); the next entry's record is
  // loaded one sample ahead, so the per-sample dependent chain (entry -> label -> l[m][y], statistics) is gone
  // REC with p.dyn_ctr: entries are handed out dynamically in chunks of kAvgChunk (one atomic per chunk,
  // grabbed a chunk ahead) instead of a fixed stride, so warps that drew hard samples do not leave the
  // others idle at the end of the kernel
  const bool dyn = REC && p.dyn_ctr != nullptr;
  auto grab = [&]() -> int64_t {
    unsigned int b = 0;
    if (lane == 0) b = atomicAdd(p.dyn_ctr, (unsigned int)kAvgChunk);
    return (int64_t)__shfl_sync(FULL, b, 0);
  };
  int64_t cbase = 0, cnext = 0;
  if (dyn) { cbase = grab(); cnext = grab(); }
  const int64_t e0 = dyn ? cbase : gw;
  uint32_t rvn = (REC && e0 < W) ? __ldcs(p.wrec + (size_t)e0 * kRecWords + lane) : 0u;

  for (int64_t e = e0, en = 0; e < W; e = en) {
    if (dyn && e == cnext) { cbase = cnext; cnext = grab(); }  // entered the chunk grabbed ahead
    en = dyn ? (e + 1 < cbase + kAvgChunk ? e + 1 : cnext) : e + nw;
    const uint32_t rv = rvn;
    if (REC && en < W) rvn = __ldcs(p.wrec + (size_t)en * kRecWords + lane);
    const int64_t n = REC ? (int64_t)__shfl_sync(FULL, rv, 28) : (int64_t)work[e];
    const int y = REC ? (int)__shfl_sync(FULL, rv, 29) : p.labels[n];
    const float* rowbase = p.logits + n * K * p.ldc;
    int tp = 0;
    float mx = 0.f, ls = 0.f, ly = INFINITY;  // ly = l[m][y]
    if (REC) {
      const uint32_t wmx = __shfl_sync(FULL, rv, 8 + (lane & 7)), wls = __shfl_sync(FULL, rv, 16 + (lane & 7));
      const uint32_t wtp = __shfl_sync(FULL, rv, 24 + ((lane & 7) >> 1));
      if (lane < K) {
        tp = (int)((wtp >> (16 * (lane & 1))) & 0xffffu);
        mx = __uint_as_float(wmx);
        ls = __uint_as_float(wls);
        ly = __uint_as_float(rv);
      }
    } else if (lane < K) {
      tp = p.top1_in[n * K + lane];
      ls = p.lsum_in[n * K + lane];
      mx = p.rmax_in[n * K + lane];
    }
    __syncwarp();
    if (lane < K) ws.stop[lane] = tp;
    __syncwarp();
    const float thr = theta_threshold(mx, ls, K, lane);
    if (!REC) ly = lane < K ? rowbase[(size_t)lane * p.ldc + y] : INFINITY;
    // ---- 1. candidate set R: one streaming pass over the sample's K rows ----------------------
    const int64_t nnext = REC ? -1 : (e + nw < W ? (int64_t)work[e + nw] : -1);
    // candidate bits of the lane's classes (lane + 32 i) * 4 + q kept as nibble i of two registers:
    // S_c (>= θ threshold) and "not below y" (>= l[m][y]), OR-ed over the models, no shared atomics
    uint32_t B1 = 0, B2 = 0;
    // rows to stream: REC drops the rows the classify kernel proved add only y to R (record word 30)
    const uint32_t live = ((1u << K) - 1u) & ~(REC ? __shfl_sync(FULL, rv, 30) : 0u);
#pragma unroll 1
    for (uint32_t lm = live; lm; lm &= lm - 1) {
      const int m = __ffs(lm) - 1;
      const float* row = rowbase + (size_t)m * p.ldc;
      {  // one-row-ahead L2 prefetch (the next live row, else the next sample's first one): 128 B per lane
        const uint32_t rest = lm & (lm - 1);
        const float* nrow = nullptr;
        if (rest) {
          nrow = rowbase + (size_t)(__ffs(rest) - 1) * p.ldc;
        } else if (REC) {
          if (en < W) {  // late in the sample: the next record has arrived
            const int64_t n2 = (int64_t)__shfl_sync(FULL, rvn, 28);
            const uint32_t l2 = ((1u << K) - 1u) & ~__shfl_sync(FULL, rvn, 30);
            if (l2) nrow = p.logits + (n2 * K + (__ffs(l2) - 1)) * p.ldc;
          }
        } else if (nnext >= 0) {
          nrow = p.logits + nnext * K * p.ldc;
        }
        if (nrow && lane * 32 < p.ldc) asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + lane * 32));
      }
      float4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c4 = lane + 32 * i;
        v[i] = c4 * 4 < C ? ldg_stream(row + c4 * 4) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
      if (C & 3) {  // the padding components (c >= C, never written) of the last float4 -> -inf, once per row
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (lane + 32 * i == ((C - 1) >> 2)) {
            if ((C & 3) < 2) v[i].y = -INFINITY;
            if ((C & 3) < 3) v[i].z = -INFINITY;
            v[i].w = -INFINITY;
          }
      }
      const float t_m = __shfl_sync(FULL, thr, m);
      const float y_m = __shfl_sync(FULL, ly, m);
      const float lo = fminf(t_m, y_m);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 x4 = v[i];
        if (fmaxf(fmaxf(x4.x, x4.y), fmaxf(x4.z, x4.w)) >= lo) {  // fast reject
          const uint32_t bits = (x4.x >= t_m ? 1u : 0u) | (x4.y >= t_m ? 2u : 0u) | (x4.z >= t_m ? 4u : 0u) |
                                (x4.w >= t_m ? 8u : 0u);
          const uint32_t bitsB = (x4.x >= y_m ? 1u : 0u) | (x4.y >= y_m ? 2u : 0u) | (x4.z >= y_m ? 4u : 0u) |
                                 (x4.w >= y_m ? 8u : 0u);
          B1 |= bits << (4 * i);
          B2 |= bitsB << (4 * i);
        }
      }
    }
    // y is in R on every worklist sample (y >= l[m][y] in each model; the classify kernel put the sample
    // on the worklist because l[m][y] >= theta threshold in some model). With skipped rows that model's
    // row may not have been streamed, so y's bits are set here explicitly (a no-op otherwise).
    if (lane == ((y >> 2) & 31)) {
      const uint32_t yb = 1u << (4 * (y >> 7) + (y & 3));
      B1 |= yb;
      B2 |= yb;
    }
    {  // R nibbles -> 32-class words: nibble i of lanes 8k..8k+7 forms word 4i + k
      const uint32_t Rn = B1 & B2;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t wv = ((Rn >> (4 * i)) & 0xfu) << (4 * (lane & 7));
        wv |= __shfl_xor_sync(FULL, wv, 1);
        wv |= __shfl_xor_sync(FULL, wv, 2);
        wv |= __shfl_xor_sync(FULL, wv, 4);
        if ((lane & 7) == 0) ws.bitmap[(lane >> 3) + 4 * i] = wv;
      }
    }
    __syncwarp();
    const uint32_t word = ws.bitmap[lane];
    const int cnt = __popc(word);
    int incl = cnt;
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += o;
    }
    const int pre = incl - cnt;
    const int nc = __shfl_sync(FULL, incl, 31);
    const bool ovf = nc > p.CAP;
    int32_t* cls = ovf ? ovC : ws.ccls;
    {
      uint32_t w = word;
      int k = pre;
      while (w) {
        cls[k++] = lane * 32 + (__ffs(w) - 1);
        w &= w - 1;
      }
    }
    auto slot_of = [&](int c) -> int {  // warp-uniform c in R
      return __shfl_sync(FULL, pre, c >> 5) + __popc(__shfl_sync(FULL, word, c >> 5) & ((1u << (c & 31)) - 1u));
    };
    const int ys = slot_of(y);
    // exact columns: y, then the members' distinct top-1 classes other than y (all lie in R)
    int dslot[8];
    int nd = 0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      dslot[m] = ys;
      if (m < K) {
        const int cm = __shfl_sync(FULL, tp, m);
        bool dup = cm == y;
        for (int q = 0; q < m; ++q) dup |= (__shfl_sync(FULL, tp, q) == cm);
        if (!dup) dslot[nd++] = slot_of(cm);
      }
    }
    __syncwarp();
    // ---- 2. gather p[m][c] = exp((l - mx_m) - lsum_m) for c in R ------------------------------------------
    float* P = ovf ? ovP : ws.P;
    const int ps = ovf ? C : CAPS;
    {  // lane = 4 m + part gathers model m's columns sl = part, part + 4, ... (L2 hits: the rows were just
       // streamed; skipped rows come from DRAM), all loads of a lane issued before their exponentials
      const int m = lane >> 2, part = lane & 3;
      const float mxl = __shfl_sync(FULL, mx, m), lsl = __shfl_sync(FULL, ls, m);
      if (m < K) {
        const float* row = rowbase + (size_t)m * p.ldc;
        float* Pm = P + (size_t)m * ps;
        int sl = part;
        for (; sl + 4 < nc; sl += 8) {
          const float l0 = __ldg(row + cls[sl]), l1 = __ldg(row + cls[sl + 4]);
          Pm[sl] = expf((l0 - mxl) - lsl);  // exact l - mx near the max
          Pm[sl + 4] = expf((l1 - mxl) - lsl);
        }
        if (sl < nc) Pm[sl] = expf((__ldg(row + cls[sl]) - mxl) - lsl);
      }
    }
    __syncwarp();
    // ---- 3. bound for candidates outside {y} ∪ D, and the exact-column half tables ------------
    {  // lane = 4 m + part: model m's competitors sl = part, part + 4, ... (K <= 8 -> all models at once)
      const int m = lane >> 2, part = lane & 3;
      float q = 0.f;
      if (m < K)
        for (int sl = part; sl < nc; sl += 4) {
          bool ex = sl == ys;
#pragma unroll
          for (int d = 0; d < 8; ++d) ex |= (d < nd && sl == dslot[d]);
          if (!ex) q = fmaxf(q, P[(size_t)m * ps + sl]);
        }
      q = fmaxf(q, __shfl_xor_sync(FULL, q, 1));
      q = fmaxf(q, __shfl_xor_sync(FULL, q, 2));
      if (part == 0 && m < K) ws.Q[m] = q;
    }
    __syncwarp();
    if (lane < TT) {  // lane h builds half-mask row h
      const uint32_t hm = lane < TA ? (uint32_t)lane : (uint32_t)(lane - TA);
      const int mo = lane < TA ? 0 : p.K1;
      float s = 0.f;
      for (uint32_t a = hm; a; a &= a - 1) s += ws.Q[mo + __ffs(a) - 1];
      ws.QB[lane] = s * (1.f + 1e-6f);  // round the bound up past fp32 summation error
      float sy0 = 0.f;
      for (uint32_t a = hm; a; a &= a - 1) sy0 += P[(size_t)(mo + __ffs(a) - 1) * ps + ys];
      ws.T[lane * DSTR] = sy0;
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        if (d < nd) {
          float sd = 0.f;
          for (uint32_t a = hm; a; a &= a - 1) sd += P[(size_t)(mo + __ffs(a) - 1) * ps + dslot[d]];
          ws.T[lane * DSTR + 1 + d] = sd;
        }
      }
    }
    __syncwarp();
    // ---- 4. A4 decision of every subset ------------------------------------------
    uint32_t pending = 0;
#pragma unroll 1
    for (int j = 0; j < JMAX; ++j) {
      const uint32_t v = (uint32_t)(lane + 32 * j + 1);
      if (v > (uint32_t)S) break;
      uint32_t oka = 0;
      if (__popc(v) == 1) {
        oka = (ws.stop[__ffs(v) - 1] == y);  // softmax is monotone (invariant I1)
      } else {
        const float* A = ws.T + (v & (TA - 1)) * DSTR;
        const float* B = ws.T + (TA + (v >> p.K1)) * DSTR;
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
        } else if (ws.QB[v & (TA - 1)] + ws.QB[TA + (v >> p.K1)] < loT) {
          if (near) pending |= 1u << j;
          else oka = 1;  // every competitor provably below y: decided in O(1)
        } else {  // bound not conclusive: scan R
          float m2 = -1.f;
          for (int q = 0; q < nc; ++q) {
            if (q == ys) continue;
            float s = 0.f;
            for (uint32_t a = v; a; a &= a - 1) s += P[(size_t)(__ffs(a) - 1) * ps + q];
            m2 = fmaxf(m2, s);
          }
          if (m2 > hiT) oka = 0;
          else if (m2 < loT) oka = 1;
          else pending |= 1u << j;
        }
      }
      ws.cnt[j * 32 + lane] += oka;
    }
    if (__any_sync(FULL, pending != 0)) recheck_fp64(p, ws, pending, rowbase, mx, P, ps, cls, nc, ys, y, lane);
    __syncwarp();
  }
#pragma unroll 1
  for (int j = 0; j < JMAX; ++j) {
    const int v1 = lane + 32 * j;
    const uint32_t c = ws.cnt[j * 32 + lane];
    if (v1 < S && c) atomicAdd(p.cnt_avg + v1, (unsigned long long)c);
  }
}

}  // namespace

size_t vote_avg_smem_per_warp(const VoteParams& p) { return warp_smem(p, nullptr, nullptr); }

cudaError_t launch_vote_avg(const VoteParams& q, int grid, cudaStream_t st, const int32_t* work,
                            const unsigned int* work_count) {
  const size_t smem = warp_smem(q, nullptr, nullptr) * WPC;
  cudaError_t e;
  if (q.wrec) {
    e = cudaFuncSetAttribute(vote_average_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) vote_average_kernel<true><<<grid, WT, smem, st>>>(q, work, work_count);
  } else {
    e = cudaFuncSetAttribute(vote_average_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) vote_average_kernel<false><<<grid, WT, smem, st>>>(q, work, work_count);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace rk
