// rk_vote_warp.cu — steps A2-A5 for K <= 8 models, C <= 1024 classes: one WARP per sample, no
// block-level barriers. (rk_vote.cu holds the CTA-tile kernel used for K > 8.)
//
// PAPER.md passages: :153 top-1 (reading Q4), :407 majority vote with best-accuracy tie-break
// (RK_TIE_BEST_MEMBER; RK_TIE_LOWEST_CLASS = north_star), :72 averaged softmax (readings Q5, Q6),
// :429 every non-empty subset v is an action; a(M[v]) = validation accuracy.
//
// Per sample (warp; lane m < K owns model m's row statistics):
//   1. row statistics: from the GEMM epilogue (top1, lse, max) or, for caller logits, one pass
//      over the K rows (lanes stride the row; xor-shuffle reductions).
//   2. decided from statistics alone, before touching the logits again:
//        * unanimous members -> (t == y) for every subset (invariant I6)           no logit reads
//        * theta = min_j p[j][top_j] / K; label y is an averaging candidate iff some model has
//          l[m][y] >= lse_m + log(theta) (K scattered loads). If not, the averaged argmax of every
//          subset differs from y (pruning proof) and only votes are evaluated.
//   3. otherwise: one coalesced streaming pass over the K*ldc logits marks the candidate set S_c in
//      a warp-private bitmap; a warp scan assigns slots in class order; p[m][c] = exp(l - lse_m) is
//      gathered for c in S_c; two half-tables (low / high models) give every subset's sums with
//      one add per candidate.
//   4. lanes own subsets v = lane + 32j + 1 (j < 8): vote via the distinct-class masks
//      (__match_any_sync), average via the half-tables; fp32 decisions inside the relative band
//      are redone in fp64 with warp-cooperative fp64 log-sum-exp (rare).
//   5. counts live in registers (exclusive ownership), per-group counts for the labelled moments
//      are written once per unit, totals are flushed with one 64-bit atomic per (warp, subset).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WT = 256;  // threads per CTA
constexpr int WPC = WT / 32;
constexpr int JMAX = 8;  // subsets per lane (S <= 255)

struct WS {  // per-warp shared memory
  int32_t* scls;    // [8] distinct predicted classes
  uint32_t* smsk;   // [8] models voting for each
  int32_t* stop;    // [8] top-1 per model
  double* lse64;    // [8]
  uint32_t* bitmap; // [32] S_c (theta test)
  uint32_t* bitmapB;// [32] classes not below y in some model
  int32_t* ccls;    // [CAP] candidate classes in ascending order
  float* P;         // [K][CAP+1]
  float* T;         // [TT][TCAP|1]
};

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t warp_smem(const VoteParams& p, char* base, WS* w) {
  const int TT = (1 << p.K1) + (1 << (p.K - p.K1));
  size_t o = 0;
  auto take = [&](size_t b) -> char* { char* r = base ? base + o : nullptr; o = a16(o + b); return r; };
  char* l64 = take(8 * 8);
  char* sc = take(4 * 8);
  char* sm = take(4 * 8);
  char* st = take(4 * 8);
  char* bm = take(4 * 32);
  char* bmB = take(4 * 32);
  char* cc = take(4ull * p.CAP);
  char* P = take(4ull * p.K * (p.CAP + 1));
  char* T = take(4ull * TT * (p.TCAP | 1));
  if (w) {
    w->lse64 = (double*)l64; w->scls = (int32_t*)sc; w->smsk = (uint32_t*)sm; w->stop = (int32_t*)st;
    w->bitmap = (uint32_t*)bm; w->bitmapB = (uint32_t*)bmB; w->ccls = (int32_t*)cc; w->P = (float*)P; w->T = (float*)T;
  }
  return o;
}

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float f4c(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }

template <bool STATS>
__global__ void __launch_bounds__(WT, 2) vote_warp_kernel(const VoteParams p) {
  extern __shared__ __align__(16) char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t wbytes = warp_smem(p, nullptr, nullptr);
  WS ws;
  warp_smem(p, smem_raw + warp * wbytes, &ws);
  const int K = p.K, S = p.S, C = p.C;
  const int F = (int)(p.ldc >> 2);
  const uint32_t kmask = (1u << K) - 1u;
  const int TA = 1 << p.K1, TT = TA + (1 << (K - p.K1));
  const int TSTR = p.TCAP | 1, CAPS = p.CAP + 1;
  const int U = p.gs > 0 ? p.gs : 16;
  const int64_t N = p.N;
  const int64_t nunits = (N + U - 1) / U;
  const int64_t gw = (int64_t)blockIdx.x * WPC + warp;
  const int64_t nw = (int64_t)gridDim.x * WPC;
  float* ovP = p.scratch + gw * (size_t)K * C;       // overflow candidate matrix [K][C]
  int32_t* ovC = p.scratch_cls + gw * (size_t)C;

  uint32_t cv[JMAX], ca[JMAX], gv[JMAX];
#pragma unroll
  for (int j = 0; j < JMAX; ++j) { cv[j] = 0; ca[j] = 0; gv[j] = 0; }

  for (int64_t unit = gw; unit < nunits; unit += nw) {
    uint32_t uni = 0;
    const int64_t s1 = (unit + 1) * U < N ? (unit + 1) * U : N;
    for (int64_t n = unit * U; n < s1; ++n) {
      const int y = p.labels[n];
      if (y < 0 || y >= C) {
        if (lane == 0) atomicOr(p.err + 1, 1u);
        continue;
      }
      const float* rowbase = p.logits + n * K * p.ldc;
      // ---- 1. row statistics (lane m < K holds model m) --------------------------------------
      int tp = 0;
      float mx = 0.f, ls = 0.f;
      bool bad = false;
      if (STATS) {
        if (lane < K) {
          tp = p.top1_in[n * K + lane];
          ls = p.lse_in[n * K + lane];
          mx = p.rmax_in[n * K + lane];
          bad = !(ls > -INFINITY && ls < INFINITY) || !(mx > -INFINITY);
        }
      } else {
        for (int m = 0; m < K; ++m) {
          const float* row = rowbase + (size_t)m * p.ldc;
          float4 v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c4 = lane + 32 * i;
            v[i] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            if (c4 < F && c4 * 4 < C) {
              v[i] = ldg_stream(row + c4 * 4);
              if (c4 * 4 + 4 > C) {  // padding components of the last partial float4
                const int valid = C - c4 * 4;
                if (valid < 4) v[i].w = -INFINITY;
                if (valid < 3) v[i].z = -INFINITY;
                if (valid < 2) v[i].y = -INFINITY;
              }
            }
          }
          float bm = -INFINITY;
          int ba = 0x7fffffff;
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float x = f4c(v[i], e);
              if (x > bm) { bm = x; ba = (lane + 32 * i) * 4 + e; }
            }
          for (int off = 16; off; off >>= 1) {
            const float om = __shfl_xor_sync(FULL, bm, off);
            const int oa = __shfl_xor_sync(FULL, ba, off);
            if (om > bm || (om == bm && oa < ba)) { bm = om; ba = oa; }
          }
          float sum = 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) sum += __expf(f4c(v[i], e) - bm);
          for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(FULL, sum, off);
          if (lane == m) {
            tp = ba; mx = bm; ls = bm + logf(sum);
            bad = !(sum == sum) || !(bm > -INFINITY) || bm == INFINITY;
          }
        }
      }
      if (__any_sync(FULL, bad)) {
        if (lane == 0) atomicOr(p.err, 1u);
        continue;
      }
      // ---- 2. vote structure and exact shortcuts ---------------------------------------------
      const int c = lane < K ? tp : -1 - lane;
      const uint32_t mm = __match_any_sync(FULL, c);
      const bool leader = lane < K && (__ffs(mm) - 1) == lane;
      const uint32_t lb = __ballot_sync(FULL, leader);
      const int nd = __popc(lb);
      uint32_t tm = 0;
      for (int bi = 0; bi < p.nB; ++bi)
        if (n >= p.tail_start[bi]) tm |= 1u << bi;
      if (__shfl_sync(FULL, mm, 0) == kmask) {  // unanimous (invariant I6)
        if (__shfl_sync(FULL, c, 0) == y) {
          ++uni;
          if (tm)  // rare: unanimous-correct sample in the ragged tail of this chunk
            for (int bi = 0; bi < p.nB; ++bi)
              if ((tm >> bi) & 1u)
                for (int v1 = lane; v1 < S; v1 += 32) atomicAdd(p.tail + (size_t)bi * S + v1, 1ull);
        }
        continue;
      }
      const bool vote_poss = __any_sync(FULL, lane < K && c == y);
      // theta = min_j p[j][top_j] / K ; candidate <=> l[m][c] >= lse_m + log(theta) (- slack)
      float th = lane < K ? __expf(mx - ls) : INFINITY;
      for (int off = 16; off; off >>= 1) th = fminf(th, __shfl_xor_sync(FULL, th, off));
      const float lth = logf(th / (float)K);
      const float thr = (ls + lth) - (1e-3f + 1e-6f * fabsf(ls) + 1e-6f * fabsf(lth));
      const float ly = lane < K ? rowbase[(size_t)lane * p.ldc + y] : INFINITY;  // l[m][y]
      const bool ycand = __any_sync(FULL, lane < K && ly >= thr);
      if (!vote_poss && !ycand) continue;  // no subset can be correct
      __syncwarp();
      if (leader) {
        const int pos = __popc(lb & ((1u << lane) - 1u));
        ws.scls[pos] = c;
        ws.smsk[pos] = mm;
      }
      if (lane < K) ws.stop[lane] = tp;
      int nc = 0, ys = -1;
      bool ovf = false, tables = false;
      if (ycand) {
        // ---- 3. candidate set: one streaming pass, warp-private bitmaps --------------------
        // R = S_c  ∩  {c : exists m, l[m][c] >= l[m][y]}: a class below y in EVERY model has
        // avg_v[c] < avg_v[y] for every subset v, so it can never decide "y is the argmax".
        ws.bitmap[lane] = 0u;
        ws.bitmapB[lane] = 0u;
        __syncwarp();
        for (int m0 = 0; m0 < K; m0 += 2) {  // two rows per step: 16 x 16-byte loads in flight per lane
          float4 v[2][8];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const float* row = rowbase + (size_t)(m0 + r) * p.ldc;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int c4 = lane + 32 * i;
              v[r][i] = (m0 + r < K && c4 < F && c4 * 4 < C)
                            ? ldg_stream(row + c4 * 4)
                            : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
          }
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const float t_m = __shfl_sync(FULL, thr, (m0 + r) < K ? m0 + r : 0);
            const float y_m = __shfl_sync(FULL, ly, (m0 + r) < K ? m0 + r : 0);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int cb = (lane + 32 * i) * 4;
              uint32_t bits = 0, bitsB = 0;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float x = f4c(v[r][i], e);
                bits |= (x >= t_m && cb + e < C) ? (1u << e) : 0u;
                bitsB |= (x >= y_m && cb + e < C) ? (1u << e) : 0u;
              }
              if (bits) atomicOr(&ws.bitmap[cb >> 5], bits << (cb & 31));
              if (bitsB) atomicOr(&ws.bitmapB[cb >> 5], bitsB << (cb & 31));
            }
          }
        }
        __syncwarp();
        const uint32_t word = ws.bitmap[lane] & ws.bitmapB[lane];
        const int cnt = __popc(word);
        int incl = cnt;
        for (int off = 1; off < 32; off <<= 1) {
          const int o = __shfl_up_sync(FULL, incl, off);
          if (lane >= off) incl += o;
        }
        const int pre = incl - cnt;
        nc = __shfl_sync(FULL, incl, 31);
        ovf = nc > p.CAP;
        tables = !ovf && nc <= p.TCAP;
        int32_t* cls = ovf ? ovC : ws.ccls;
        {
          uint32_t w = word;
          int k = pre;
          while (w) {
            const int b = __ffs(w) - 1;
            cls[k++] = lane * 32 + b;
            w &= w - 1;
          }
        }
        {
          const uint32_t wy = __shfl_sync(FULL, word, y >> 5);
          const int py = __shfl_sync(FULL, pre, y >> 5);
          ys = py + __popc(wy & ((1u << (y & 31)) - 1u));
        }
        __syncwarp();
        // gather p[m][c] = exp(l - lse_m) for c in S_c
        float* P = ovf ? ovP : ws.P;
        const int ps = ovf ? C : CAPS;
        float lsm[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) lsm[m] = __shfl_sync(FULL, ls, m < K ? m : 0);
        for (int sl = lane; sl < nc; sl += 32) {
          const int cq = cls[sl];
          float l[8];
#pragma unroll
          for (int m = 0; m < 8; ++m)  // K independent loads in flight (L2 hits: the rows were just streamed)
            l[m] = m < K ? __ldg(rowbase + (size_t)m * p.ldc + cq) : 0.f;
#pragma unroll
          for (int m = 0; m < 8; ++m)
            if (m < K) P[(size_t)m * ps + sl] = expf(l[m] - lsm[m]);
        }
        __syncwarp();
        if (tables) {
          for (int h = 0; h < TT; ++h)
            for (int sl = lane; sl < nc; sl += 32) {
              float s = 0.f;
              if (h < TA) {
                for (uint32_t a = (uint32_t)h; a; a &= a - 1) s += ws.P[(size_t)(__ffs(a) - 1) * CAPS + sl];
              } else {
                for (uint32_t b = (uint32_t)(h - TA); b; b &= b - 1) s += ws.P[(size_t)(p.K1 + __ffs(b) - 1) * CAPS + sl];
              }
              ws.T[(size_t)h * TSTR + sl] = s;
            }
          __syncwarp();
        }
      } else {
        __syncwarp();
      }
      // ---- 4. subsets owned by this lane ---------------------------------------------------
      uint32_t pending = 0;  // subsets whose averaged decision needs the fp64 recheck
      const float* Pm = ovf ? ovP : ws.P;
      const int ps = ovf ? C : CAPS;
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        const uint32_t v = (uint32_t)(lane + 32 * j + 1);
        if (v > (uint32_t)S) break;
        uint32_t okv = 0, oka = 0;
        if (vote_poss) {  // A3
          int bc = 0, bcls = 0x7fffffff;
          uint32_t tied = 0;
          for (int q = 0; q < nd; ++q) {
            const uint32_t mv = v & ws.smsk[q];
            const int cnt = __popc(mv);
            const int cq = ws.scls[q];
            if (cnt > bc) { bc = cnt; bcls = cq; tied = mv; }
            else if (cnt == bc && cnt > 0) { tied |= mv; bcls = min(bcls, cq); }
          }
          const int winner = (p.tie == 0) ? ws.stop[p.best_of[tied]] : bcls;
          okv = (winner == y);
        }
        if (ycand) {  // A4
          if (__popc(v) == 1) {
            oka = (ws.stop[__ffs(v) - 1] == y);  // softmax is monotone (invariant I1)
          } else {
            float sy = 0.f, m2 = -1.f;
            if (tables) {
              const float* A = ws.T + (size_t)(v & (TA - 1)) * TSTR;
              const float* B = ws.T + (size_t)(TA + (v >> p.K1)) * TSTR;
              sy = A[ys] + B[ys];
              for (int q = 0; q < nc; ++q) {
                const float s = A[q] + B[q];
                if (q != ys) m2 = fmaxf(m2, s);
              }
            } else {
              for (int q = 0; q < nc; ++q) {
                float s = 0.f;
                for (uint32_t a = v; a; a &= a - 1) s += Pm[(size_t)(__ffs(a) - 1) * ps + q];
                if (q == ys) sy = s; else m2 = fmaxf(m2, s);
              }
            }
            if (m2 > sy * (1.f + p.band)) oka = 0;
            else if (m2 < sy * (1.f - p.band)) oka = 1;
            else pending |= 1u << j;
          }
        }
        gv[j] += okv;
        ca[j] += oka;
        if (okv && tm)
          for (int bi = 0; bi < p.nB; ++bi)
            if ((tm >> bi) & 1u) atomicAdd(p.tail + (size_t)bi * S + (v - 1), 1ull);
      }
      // ---- fp64 recheck of near-ties (rare): warp-cooperative log-sum-exp, then per lane ----
      if (__any_sync(FULL, pending != 0)) {
        for (int m = 0; m < K; ++m) {
          const float* row = rowbase + (size_t)m * p.ldc;
          const double m64 = (double)__shfl_sync(FULL, mx, m);
          double s = 0.0;
          for (int cc = lane; cc < C; cc += 32) s += exp((double)row[cc] - m64);
          for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
          if (lane == 0) ws.lse64[m] = m64 + log(s);
        }
        __syncwarp();
        const int32_t* cls = ovf ? ovC : ws.ccls;
#pragma unroll
        for (int j = 0; j < JMAX; ++j) {
          if (!((pending >> j) & 1u)) continue;
          const uint32_t v = (uint32_t)(lane + 32 * j + 1);
          atomicAdd(p.n_recheck + (v - 1), 1ull);
          // fp32 sums again to select the band, fp64 decides
          float sy = 0.f;
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
              s += exp((double)rowbase[(size_t)m * p.ldc + cq] - ws.lse64[m]);
            }
            const double a64 = s / (double)nv;
            if (a64 > best || (a64 == best && cq < bestc)) { best = a64; bestc = cq; }
          }
          ca[j] += (bestc == y);
        }
      }
      __syncwarp();
    }  // samples of the unit
    // ---- unit end: group counts (labelled moments) and totals ---------------------------------
#pragma unroll
    for (int j = 0; j < JMAX; ++j) {
      const int v1 = lane + 32 * j;
      if (v1 < S) {
        const uint32_t tot = gv[j] + uni;
        if (p.grp) p.grp[unit * (size_t)S + v1] = (uint8_t)tot;
        cv[j] += tot;
        ca[j] += uni;
      }
      gv[j] = 0;
    }
  }
#pragma unroll
  for (int j = 0; j < JMAX; ++j) {
    const int v1 = lane + 32 * j;
    if (v1 < S) {
      if (cv[j]) atomicAdd(p.cnt_vote + v1, (unsigned long long)cv[j]);
      if (ca[j]) atomicAdd(p.cnt_avg + v1, (unsigned long long)ca[j]);
    }
  }
}

}  // namespace

size_t vote_warp_smem_per_warp(const VoteParams& p) { return warp_smem(p, nullptr, nullptr); }
int vote_warp_threads() { return WT; }

cudaError_t launch_vote_warp(const VoteParams& p, int grid, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  const size_t smem = warp_smem(p, nullptr, nullptr) * WPC;
  auto k = p.lse_in ? vote_warp_kernel<true> : vote_warp_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, WT, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rk
