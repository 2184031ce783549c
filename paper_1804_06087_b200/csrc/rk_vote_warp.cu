// rk_vote_warp.cu — steps A2-A5 for K <= 8 models (caller rows are read in blocks of 1024 classes). One WARP per sample, no
// block-level barriers, two kernels (rk_vote.cu holds the CTA-tile kernel used for K > 8).
//
// PAPER.md passages: :153 top-1 (reading Q4), :407 majority vote with best-accuracy tie-break
// (RK_TIE_BEST_MEMBER; RK_TIE_LOWEST_CLASS = north_star), :72 averaged softmax (readings Q5, Q6),
// :429 every non-empty subset v is an action; a(M[v]) = validation accuracy.
//
// Kernel A, vote_classify (every sample; reads per-row statistics, not the logits):
//   * row statistics (top1, lse, max) from the GEMM epilogue, or one pass over the rows for caller
//     logits (then written out for kernel B);
//   * unanimous members -> (t == y) for every subset, vote AND average (invariant I6);
//   * majority vote of every subset (lanes own subsets v = lane + 32j + 1; distinct-class masks
//     from __match_any_sync);
//   * theta = min_j p[j][top_j] / K; the label y can be the averaged argmax of some subset only if
//     some model has l[m][y] >= lse_m + log(theta) (K scattered loads; pruning proof, SURVEY.md
//     §8(d)). If not, every subset's average is wrong; otherwise the sample joins a worklist.
// Kernel B, vote_average (worklist samples only; all warps run the same phases):
//   * one coalesced streaming pass over the K*ldc logits marks
//       R = S_c ∩ {c : exists m, l[m][c] >= l[m][y]}
//     (S_c: theta candidates; a class below y in EVERY model has avg_v[c] < avg_v[y] for all v);
//   * warp scan assigns slots in class order; p[m][c] = exp(l - lse_m) is gathered for c in R;
//   * per subset: sum_y from two half-tables (low / high models), an upper bound on every
//     competitor (half-table sums of q_m = max_{c != y} p[m][c]) decides most subsets in O(1),
//     the rest scan R; fp32 decisions inside the relative band are redone in fp64 (rare).
// Counts are lane-owned (no atomics in the loops), flushed with one 64-bit atomic per (warp, v).
#include <cuda_runtime.h>
#include <stdlib.h>

#include <algorithm>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WT = 128;  // threads per CTA (4 warps)
constexpr int WPC = WT / 32;
constexpr int JMAX = 8;  // subsets per lane (S <= 255)

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float f4c(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }



// rare: a vote-correct sample in the ragged tail of the chunk (outside complete batches of B[b])
__device__ __noinline__ void tail_add(const VoteParams& p, uint32_t tm, uint32_t v) {
  for (int bi = 0; bi < p.nB; ++bi)
    if ((tm >> bi) & 1u) atomicAdd(p.tail + (size_t)bi * p.S + (v - 1), 1ull);
}

// =============================== kernel A: classify + votes ====================================
template <bool STATS>
__global__ void __launch_bounds__(WT, 6) vote_classify_kernel(const VoteParams p, int32_t* work,
                                                              unsigned int* work_count, int32_t* st_top,
                                                              float* st_lsum, float* st_max) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.K, S = p.S, C = p.C;
  const int F = (int)(p.ldc >> 2);
  const uint32_t kmask = (1u << K) - 1u;
  const int U = p.gs > 0 ? p.gs : 16;
  const int64_t N = p.N;
  const int64_t nunits = (N + U - 1) / U;
  const int64_t gw = (int64_t)blockIdx.x * WPC + warp;
  const int64_t nw = (int64_t)gridDim.x * WPC;
  int64_t tail0 = N;
  for (int bi = 0; bi < p.nB; ++bi) tail0 = p.tail_start[bi] < tail0 ? p.tail_start[bi] : tail0;

  uint32_t cv[JMAX], ca[JMAX], gv[JMAX];
#pragma unroll
  for (int j = 0; j < JMAX; ++j) { cv[j] = 0; ca[j] = 0; gv[j] = 0; }
  __shared__ uint32_t srec[WPC][16][kRecWords];  // worklist records of the warp's current unit (U <= 16)
  uint32_t nskip = 0;

  for (int64_t unit = gw; unit < nunits; unit += nw) {
    uint32_t uni = 0, wmask = 0;
    const int64_t u0 = unit * U;
    const int64_t s1 = u0 + U < N ? u0 + U : N;
    // the unit's labels in one load (lane i: sample u0 + i); with STATS the next sample's statistics and
    // l[m][y] are loaded one sample ahead, off the per-sample dependent load chain
    const int ylane = (lane < U && u0 + lane < s1) ? p.labels[u0 + lane] : 0;
    int ntp = 0;
    float nls = 0.f, nmx = 0.f, nly = 0.f, ns2 = INFINITY;
    auto prefetch = [&](int64_t nn) {
      const int yy = __shfl_sync(FULL, ylane, (int)(nn - u0) & 31);
      if (STATS && nn < s1 && lane < K) {
        ntp = p.top1_in[nn * K + lane];
        nls = p.lsum_in[nn * K + lane];
        nmx = p.rmax_in[nn * K + lane];
        if (p.s2_in) ns2 = p.s2_in[nn * K + lane];
        nly = (yy >= 0 && yy < C) ? (p.ly_in ? p.ly_in[nn * K + lane] : p.logits[(nn * K + lane) * p.ldc + yy]) : 0.f;
      }
    };
    prefetch(u0);
#pragma unroll 1
    for (int64_t n = u0; n < s1; ++n) {
      int tp = ntp;
      float mx = nmx, ls = nls;
      const float lyv = nly, s2v = ns2;
      prefetch(n + 1);
      const int y = __shfl_sync(FULL, ylane, (int)(n - u0));
      if (y < 0 || y >= C) {
        if (lane == 0) atomicOr(p.err + 1, 1u);
        continue;
      }
      const float* rowbase = p.logits + n * K * p.ldc;
      bool bad = false;
      if (STATS) {
        if (lane < K) bad = !(ls > -INFINITY && ls < INFINITY) || !(mx > -INFINITY);
      } else {
#pragma unroll 1
        for (int m = 0; m < K; ++m) {  // one pass over the row: max, lowest argmax, sum exp
          const float* row = rowbase + (size_t)m * p.ldc;
          float bm = -INFINITY, sum = 0.f;
          int ba = 0x7fffffff;
#pragma unroll 1
          for (int f0 = 0; f0 < F; f0 += 256) {  // blocks of 1024 classes (one block when ldc <= 1024)
            float4 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int c4 = f0 + lane + 32 * i;
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
            float km = -INFINITY;
            int ka = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float x = f4c(v[i], e);
                if (x > km) { km = x; ka = (f0 + lane + 32 * i) * 4 + e; }
              }
            for (int off = 16; off; off >>= 1) {
              const float om = __shfl_xor_sync(FULL, km, off);
              const int oa = __shfl_xor_sync(FULL, ka, off);
              if (om > km || (om == km && oa < ka)) { km = om; ka = oa; }
            }
            // running max / lowest argmax (earlier blocks hold lower classes) / rescaled sum
            const float nm = fmaxf(bm, km);
            if (km > bm) ba = ka;
            float ks = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
              for (int e = 0; e < 4; ++e) ks += __expf(f4c(v[i], e) - nm);
            for (int off = 16; off; off >>= 1) ks += __shfl_xor_sync(FULL, ks, off);
            sum = (bm == -INFINITY ? 0.f : sum * __expf(bm - nm)) + ks;
            bm = nm;
          }
          if (lane == m) {
            tp = ba; mx = bm; ls = logf(sum);  // log-sum relative to the row max
            bad = !(sum == sum) || !(bm > -INFINITY) || bm == INFINITY;
          }
        }
        if (lane < K) {  // statistics for kernel B
          st_top[n * K + lane] = tp;
          st_lsum[n * K + lane] = ls;
          st_max[n * K + lane] = mx;
        }
      }
      if (__any_sync(FULL, bad)) {
        if (lane == 0) atomicOr(p.err, 1u);
        continue;
      }
      // vote structure
      const int c = lane < K ? tp : -1 - lane;
      const uint32_t mm = __match_any_sync(FULL, c);
      uint32_t tm = 0;
      if (n >= tail0)
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
      // averaging candidate test (theta pruning) for the label
      const float thr = theta_threshold(mx, ls, K, lane);
      const float lym = STATS ? lyv : (lane < K ? rowbase[(size_t)lane * p.ldc + y] : 0.f);
      const bool ycand = __any_sync(FULL, lane < K && lym >= thr);
      if (ycand) {
        wmask |= 1u << (int)(n - u0);
        if (p.wrec) {  // the averaging kernel's per-sample inputs, staged for one coalesced record store
          uint32_t* r = srec[warp][n - u0];
          if (lane < K) {
            r[lane] = __float_as_uint(lym);
            r[8 + lane] = __float_as_uint(mx);
            r[16 + lane] = __float_as_uint(ls);
            reinterpret_cast<uint16_t*>(r + 24)[lane] = (uint16_t)tp;
          }
          // rows that add only y to the candidate set R of the averaging kernel: y is the top-1 and every
          // other class (<= the second-largest logit) lies below the theta threshold, i.e. outside S_c
          // (y itself is in R on every worklist sample), so that kernel need not stream them; the margin
          // absorbs any rounding difference between the two kernels' evaluations of the same threshold
          const uint32_t skip = __ballot_sync(FULL, STATS && lane < K && tp == y && s2v < thr - (1e-4f + 1e-5f * fabsf(thr)));
          if (lane == 0) { r[28] = (uint32_t)n; r[29] = (uint32_t)y; r[30] = skip; }
          nskip += __popc(skip);
        }
      }
      // A3: majority vote, decided relative to y: with c_j = |v ∩ M_j|, y wins iff
      // c_y > 0, no class has more votes, and the tie (if any) goes to y: LOWEST_CLASS -> no tied
      // class below y; BEST_MEMBER -> the best-ranked member among all tied voters votes y (Q2).
      const uint32_t my = __ballot_sync(FULL, lane < K && c == y);  // members voting y
      if (!my) continue;                                              // every vote wrong
      const uint32_t ob = __ballot_sync(FULL, lane < K && (__ffs(mm) - 1) == lane && c != y);
      uint32_t cy[JMAX], tied[JMAX], lose = 0;
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        const uint32_t v = (uint32_t)(lane + 32 * j + 1);
        tied[j] = v & my;
        cy[j] = __popc(tied[j]);
        lose |= (cy[j] == 0u) ? (1u << j) : 0u;
      }
      for (uint32_t w = ob; w; w &= w - 1) {  // other predicted classes (warp-uniform loop)
        const int l = __ffs(w) - 1;
        const uint32_t mj = __shfl_sync(FULL, mm, l);
        const bool ltj = __shfl_sync(FULL, c, l) < y;
#pragma unroll
        for (int j = 0; j < JMAX; ++j) {
          const uint32_t vm = (uint32_t)(lane + 32 * j + 1) & mj;
          const uint32_t cj = __popc(vm);
          lose |= (cj > cy[j] || (p.tie != 0 && cj == cy[j] && ltj)) ? (1u << j) : 0u;
          tied[j] |= (cj == cy[j]) ? vm : 0u;
        }
      }
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        const uint32_t v = (uint32_t)(lane + 32 * j + 1);
        if (v > (uint32_t)S) break;
        uint32_t okv = !((lose >> j) & 1u);
        if (p.tie == 0 && okv) okv = (my >> p.best_of[tied[j]]) & 1u;
        gv[j] += okv;
        if (okv && tm) tail_add(p, tm, v);
      }
    }
    // unit end: worklist append (one atomic per unit), group counts, totals
    if (wmask) {
      unsigned int base = 0;
      if (lane == 0) base = atomicAdd(work_count, (unsigned int)__popc(wmask));
      base = __shfl_sync(FULL, base, 0);
      if ((wmask >> lane) & 1u) work[base + __popc(wmask & ((1u << lane) - 1u))] = (int32_t)(u0 + lane);
      if (p.wrec) {  // records in worklist order: one 128-byte store per worklist sample
        __syncwarp();
        int k = 0;
        for (uint32_t wm = wmask; wm; wm &= wm - 1, ++k)
          p.wrec[(size_t)(base + k) * kRecWords + lane] = srec[warp][__ffs(wm) - 1][lane];
        __syncwarp();  // every lane has read the staged records before the next unit overwrites them
      }
    }
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
  if (p.n_skip && lane == 0 && nskip) atomicAdd(p.n_skip, nskip);
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

// Grid of the classify kernel: its warps stride over the units, so the grid is one full wave (the CTAs that
// fit on the SMs at once, from the occupancy API) or fewer; a grid with a partial second wave leaves most
// SMs idle while the last CTAs finish (sm_count * 8 CTAs had been 1.33 waves at 6 resident per SM).
template <bool STATS>
static int64_t classify_grid(int64_t units, int sm_count) {
  static int per_sm = -1;
  if (per_sm < 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, vote_classify_kernel<STATS>, WT, 0) != cudaSuccess || b < 1)
      b = 6;
    per_sm = b;
  }
  const int64_t ga = (units + WPC - 1) / WPC, cap = (int64_t)sm_count * per_sm;
  return ga < cap ? ga : cap;
}

cudaError_t launch_vote_classify(const VoteParams& p, cudaStream_t st, int32_t* work, unsigned int* work_count,
                                 int sm_count) {
  if (p.N <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(work_count, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  if (!p.lsum_in) return cudaErrorInvalidValue;  // statistics come from the GEMM
  const int U = p.gs > 0 ? p.gs : 16;
  const int64_t units = (p.N + U - 1) / U;
  const int64_t ga = classify_grid<true>(units, sm_count);
  vote_classify_kernel<true><<<(int)ga, WT, 0, st>>>(p, work, work_count, nullptr, nullptr, nullptr);
  return cudaGetLastError();
}

size_t vote_warp_smem_per_warp(const VoteParams& p) { return vote_avg_smem_per_warp(p); }
int vote_warp_threads() { return WT; }
#ifndef RK_AVG_MINB
#define RK_AVG_MINB 7
#endif
int vote_warp_min_blocks() {
  static const int v = [] {
    const char* e = getenv("RK_VOTE_PER_SM");  // development knob: averaging CTAs per SM
    return e ? std::max(1, atoi(e)) : RK_AVG_MINB;
  }();
  return v;
}

cudaError_t launch_vote_warp(const VoteParams& p, int grid, cudaStream_t st, int32_t* work, unsigned int* work_count,
                             int32_t* st_top, float* st_lsum, float* st_max, int sm_count) {
  if (p.N <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(work_count, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  // kernel A: classify + votes
  {
    const int U = p.gs > 0 ? p.gs : 16;
    const int64_t units = (p.N + U - 1) / U;
    const int64_t ga = p.lsum_in ? classify_grid<true>(units, sm_count) : classify_grid<false>(units, sm_count);
#ifdef RK_CARVEOUT
    cudaFuncSetAttribute(vote_classify_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, RK_CARVEOUT);
    cudaFuncSetAttribute(vote_classify_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, RK_CARVEOUT);
#endif
    if (p.lsum_in) vote_classify_kernel<true><<<(int)ga, WT, 0, st>>>(p, work, work_count, st_top, st_lsum, st_max);
    else vote_classify_kernel<false><<<(int)ga, WT, 0, st>>>(p, work, work_count, st_top, st_lsum, st_max);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // kernel B: averages on the worklist (always from statistics: the GEMM's or kernel A's)
  {
    VoteParams q = p;
    if (!p.lsum_in) { q.top1_in = st_top; q.lsum_in = st_lsum; q.rmax_in = st_max; }
    if (vote_large_needed(q)) e = launch_vote_large_avg(q, sm_count, st, work, work_count);  // ldc > 1024
    else e = launch_vote_avg(q, grid, st, work, work_count);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rk
