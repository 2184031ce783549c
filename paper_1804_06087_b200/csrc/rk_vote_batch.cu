// rk_vote_batch.cu — steps A2-A5 for K = 9..12 models (511..4095 subsets), C <= 1024 classes.
//
// PAPER.md passages: :153 top-1 (reading Q4), :407 majority vote with best-accuracy tie-break
// (RK_TIE_BEST_MEMBER; RK_TIE_LOWEST_CLASS = north_star), :72 averaged softmax (readings Q5, Q6),
// :429 every non-empty subset v of the model list is an action (2^|M| - 1 of them).
//
// With thousands of subsets per sample the work is the (sample, subset) sweep, so the layout is
// transposed relative to rk_vote_warp.cu:
//   phase 1  warps build a compact record per sample of a batch (row statistics, distinct-class
//            vote masks, flags; for the averaging kernel: the candidate set R, gathered
//            probabilities, half-tables and the competitor bound) in shared memory;
//   phase 2  every thread owns the fixed subsets v = t + 1 + 256k and sweeps the batch: all threads
//            read the same record at the same time (smem broadcast, uniform control flow), counters
//            live in registers, per-group counts are written once per group.
// Exactness arguments are those of rk_vote_warp.cu (unanimity I6, theta pruning, the y-dominance
// filter, the competitor bound, fp64 recheck of near-ties).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int BT = 256;          // threads per CTA
constexpr int NWB = BT / 32;
constexpr int SB = 128;          // samples per batch (kernel A)
constexpr int SBW = NWB;         // worklist samples per batch (kernel B): one per warp
constexpr int KM = 12;

constexpr uint32_t R_EVAL = 1u, R_UNAN = 2u;

struct Rec {  // per-sample vote record (kernel A)
  int32_t y;
  uint32_t flags;
  int32_t nd;
  uint32_t tm;
  int32_t cls[KM];
  uint32_t msk[KM];
  int32_t top[KM];
};

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float f4c(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

__device__ __forceinline__ float theta_threshold(float mx, float ls, int K, int lane) {
  float th = lane < K ? __expf(mx - ls) : INFINITY;
  for (int off = 16; off; off >>= 1) th = fminf(th, __shfl_xor_sync(FULL, th, off));
  const float lth = logf(th / (float)K);
  return (ls + lth) - (1e-3f + 1e-6f * fabsf(ls) + 1e-6f * fabsf(lth));
}

__device__ __noinline__ void tail_add_b(const VoteParams& p, uint32_t tm, uint32_t v) {
  for (int bi = 0; bi < p.nB; ++bi)
    if ((tm >> bi) & 1u) atomicAdd(p.tail + (size_t)bi * p.S + (v - 1), 1ull);
}

// Row statistics of model `lane` for caller logits: one pass over every row (lanes stride a row).
__device__ void row_stats(const VoteParams& p, const float* rowbase, int lane, int& tp, float& mx, float& ls,
                          bool& bad) {
  const int K = p.K, C = p.C;
#pragma unroll 1
  for (int m = 0; m < K; ++m) {
    const float* row = rowbase + (size_t)m * p.ldc;
    float bm = -INFINITY, sum = 0.f;
    int ba = 0x7fffffff;
    for (int c = lane; c < C; c += 32) {  // C <= 1024: at most 32 values per lane
      const float x = row[c];
      if (x > bm) { bm = x; ba = c; }
    }
    for (int off = 16; off; off >>= 1) {
      const float om = __shfl_xor_sync(FULL, bm, off);
      const int oa = __shfl_xor_sync(FULL, ba, off);
      if (om > bm || (om == bm && oa < ba)) { bm = om; ba = oa; }
    }
    for (int c = lane; c < C; c += 32) sum += __expf(row[c] - bm);
    for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(FULL, sum, off);
    if (lane == m) {
      tp = ba; mx = bm; ls = bm + logf(sum);
      bad = !(sum == sum) || !(bm > -INFINITY) || bm == INFINITY;
    }
  }
}

// =============================== kernel A: classify + votes (batched) ==========================
template <int NK, bool STATS>
__global__ void __launch_bounds__(BT, 2) vote_batch_classify_kernel(const VoteParams p, int32_t* work,
                                                                    unsigned int* work_count, int32_t* st_top,
                                                                    float* st_lse, float* st_max) {
  __shared__ Rec rec[SB];
  __shared__ uint32_t uni[SB];
  __shared__ uint8_t best_of[1 << KM];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, S = p.S, C = p.C;
  const uint32_t kmask = (1u << K) - 1u;
  const int gsz = p.gs > 0 ? p.gs : 16;
  const int64_t N = p.N;
  const int64_t nbatch = (N + SB - 1) / SB;
  int64_t tail0 = N;
  for (int bi = 0; bi < p.nB; ++bi) tail0 = p.tail_start[bi] < tail0 ? p.tail_start[bi] : tail0;
  if (p.tie == 0)
    for (int i = t; i < (1 << K); i += BT) best_of[i] = p.best_of[i];

  uint32_t cv[NK], ca[NK], gv[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) { cv[k] = 0; ca[k] = 0; gv[k] = 0; }

  for (int64_t batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
    const int64_t b0 = batch * SB;
    __syncthreads();
    for (int i = t; i < SB; i += BT) uni[i] = 0;
    __syncthreads();
    // ---- phase 1: per-sample records (warp per sample) --------------------------------------
    uint32_t wl = 0;  // this warp's worklist samples (bit i <-> b = warp + NWB * i)
#pragma unroll 1
    for (int i = 0; i < SB / NWB; ++i) {
      const int b = warp + NWB * i;
      const int64_t n = b0 + b;
      uint32_t fl = 0;
      if (n < N) {
        const int y = p.labels[n];
        if (y < 0 || y >= C) {
          if (lane == 0) atomicOr(p.err + 1, 1u);
        } else {
          const float* rowbase = p.logits + n * K * p.ldc;
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
            row_stats(p, rowbase, lane, tp, mx, ls, bad);
            if (lane < K) { st_top[n * K + lane] = tp; st_lse[n * K + lane] = ls; st_max[n * K + lane] = mx; }
          }
          if (__any_sync(FULL, bad)) {
            if (lane == 0) atomicOr(p.err, 1u);
          } else {
            const int c = lane < K ? tp : -1 - lane;
            const uint32_t mm = __match_any_sync(FULL, c);
            uint32_t tm = 0;
            if (n >= tail0)
              for (int bi = 0; bi < p.nB; ++bi)
                if (n >= p.tail_start[bi]) tm |= 1u << bi;
            if (__shfl_sync(FULL, mm, 0) == kmask) {  // unanimous (invariant I6)
              fl = R_UNAN;
              if (__shfl_sync(FULL, c, 0) == y) {
                if (lane == 0) atomicAdd(&uni[b / gsz], 1u);
                if (tm)
                  for (int bi = 0; bi < p.nB; ++bi)
                    if ((tm >> bi) & 1u)
                      for (int v1 = lane; v1 < S; v1 += 32) atomicAdd(p.tail + (size_t)bi * S + v1, 1ull);
              }
            } else {
              const float thr = theta_threshold(mx, ls, K, lane);
              if (__any_sync(FULL, lane < K && rowbase[(size_t)lane * p.ldc + y] >= thr)) wl |= 1u << i;
              if (__any_sync(FULL, lane < K && c == y)) {
                fl = R_EVAL;
                const bool leader = lane < K && (__ffs(mm) - 1) == lane;
                const uint32_t lb = __ballot_sync(FULL, leader);
                if (leader) {
                  const int pos = __popc(lb & ((1u << lane) - 1u));
                  rec[b].cls[pos] = c;
                  rec[b].msk[pos] = mm;
                }
                if (lane < K) rec[b].top[lane] = tp;
                if (lane == 0) { rec[b].nd = __popc(lb); rec[b].y = y; rec[b].tm = tm; }
              }
            }
          }
        }
      }
      if (lane == 0) rec[b].flags = fl;
    }
    if (wl) {  // worklist append: one atomic per warp per batch
      unsigned int base = 0;
      if (lane == 0) base = atomicAdd(work_count, (unsigned int)__popc(wl));
      base = __shfl_sync(FULL, base, 0);
      if (lane < SB / NWB && ((wl >> lane) & 1u))
        work[base + __popc(wl & ((1u << lane) - 1u))] = (int32_t)(b0 + warp + NWB * lane);
    }
    __syncthreads();
    // ---- phase 2: thread t owns subsets v = t + 1 + 256k and sweeps the batch ----------------
    const int ngroups = SB / gsz;
#pragma unroll 1
    for (int g = 0; g < ngroups; ++g) {
#pragma unroll 1
      for (int b = g * gsz; b < (g + 1) * gsz; ++b) {
        if (!(rec[b].flags & R_EVAL)) continue;  // uniform across the CTA
        const int nd = rec[b].nd, y = rec[b].y;
        const uint32_t tm = rec[b].tm;
#pragma unroll
        for (int k = 0; k < NK; ++k) {  // A3: majority vote
          const uint32_t v = (uint32_t)(t + 1 + BT * k);
          if (v > (uint32_t)S) break;
          int bc = 0, bcls = 0x7fffffff;
          uint32_t tied = 0;
#pragma unroll 1
          for (int q = 0; q < nd; ++q) {
            const uint32_t mv = v & rec[b].msk[q];
            const int cnt = __popc(mv);
            const int cq = rec[b].cls[q];
            if (cnt > bc) { bc = cnt; bcls = cq; tied = mv; }
            else if (cnt == bc && cnt > 0) { tied |= mv; bcls = min(bcls, cq); }
          }
          const int winner = (p.tie == 0) ? rec[b].top[best_of[tied]] : bcls;
          const uint32_t ok = winner == y;
          gv[k] += ok;
          if (ok && tm) tail_add_b(p, tm, v);
        }
      }
      // group end: labelled-moment group counts and totals
      const int64_t gi = (b0 + (int64_t)g * gsz) / gsz;
      const uint32_t u = uni[g * gsz / gsz];
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int v1 = t + BT * k;
        if (v1 < S && b0 + (int64_t)g * gsz < N) {
          const uint32_t tot = gv[k] + u;
          if (p.grp) p.grp[gi * S + v1] = (uint8_t)tot;
          cv[k] += tot;
          ca[k] += u;
        }
        gv[k] = 0;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int v1 = t + BT * k;
    if (v1 < S) {
      if (cv[k]) atomicAdd(p.cnt_vote + v1, (unsigned long long)cv[k]);
      if (ca[k]) atomicAdd(p.cnt_avg + v1, (unsigned long long)ca[k]);
    }
  }
}

// =============================== kernel B: averages on the worklist (batched) ====================
struct SmpB {  // per-sample record (kernel B), pointers into the CTA's dynamic smem
  float* P;      // [K][CAP+1]
  float* T;      // [TT][TCAP|1]
  float* QB;     // [TT]
  int32_t* cls;  // [CAP]
  uint32_t* bm;  // [32]
  uint32_t* bmB; // [32]
};

__host__ __device__ inline size_t smp_bytes(const VoteParams& p, char* base, SmpB* s) {
  const int TT = (1 << p.K1) + (1 << (p.K - p.K1));
  size_t o = 0;
  auto take = [&](size_t b) -> char* { char* r = base ? base + o : nullptr; o = a16(o + b); return r; };
  char* P = take(4ull * p.K * (p.CAP + 1));
  char* T = take(4ull * TT * (p.TCAP | 1));
  char* QB = take(4ull * TT);
  char* cl = take(4ull * p.CAP);
  char* bm = take(4 * 32);
  char* bmB = take(4 * 32);
  if (s) { s->P = (float*)P; s->T = (float*)T; s->QB = (float*)QB; s->cls = (int32_t*)cl; s->bm = (uint32_t*)bm; s->bmB = (uint32_t*)bmB; }
  return o;
}

struct HdrB {  // per-sample scalars
  int64_t n;
  int32_t y, nc, ys, valid, ovf, tables, need64;
  int32_t top[KM];
  float mx[KM];
  float q[KM];
  double lse64[KM];
};

template <int NK>
__global__ void __launch_bounds__(BT, 1) vote_batch_average_kernel(const VoteParams p, const int32_t* work,
                                                                   const unsigned int* work_count) {
  extern __shared__ __align__(16) char smem_raw[];
  __shared__ HdrB hd[SBW];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, S = p.S, C = p.C;
  const int F = (int)(p.ldc >> 2);
  const int TA = 1 << p.K1, TT = TA + (1 << (K - p.K1));
  const int TSTR = p.TCAP | 1, CAPS = p.CAP + 1;
  const size_t sbytes = smp_bytes(p, nullptr, nullptr);
  const int64_t W = *work_count;
  const int64_t nbatch = (W + SBW - 1) / SBW;
  uint32_t ca[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) ca[k] = 0;

  for (int64_t batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
    __syncthreads();
    // ---- phase 1: warp `warp` prepares worklist sample e ----------------------------------------
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
        if (lane < K) { tp = p.top1_in[n * K + lane]; ls = p.lse_in[n * K + lane]; mx = p.rmax_in[n * K + lane]; }
        const float thr = theta_threshold(mx, ls, K, lane);
        const float ly = lane < K ? rowbase[(size_t)lane * p.ldc + y] : INFINITY;
        sm.bm[lane] = 0u;
        sm.bmB[lane] = 0u;
        __syncwarp();
        // candidate set R = S_c ∩ {c : exists m, l[m][c] >= l[m][y]}, one streaming pass
#pragma unroll 1
        for (int m = 0; m < K; ++m) {
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
        const int ys = __shfl_sync(FULL, pre, y >> 5) +
                       __popc(__shfl_sync(FULL, word, y >> 5) & ((1u << (y & 31)) - 1u));
        const bool ovf = nc > p.CAP;
        float* P = ovf ? p.scratch + ((size_t)blockIdx.x * SBW + warp) * (size_t)K * C : sm.P;
        int32_t* cls = ovf ? p.scratch_cls + ((size_t)blockIdx.x * SBW + warp) * (size_t)C : sm.cls;
        const int ps = ovf ? C : CAPS;
        {
          uint32_t w = word;
          int k = pre;
          while (w) { cls[k++] = lane * 32 + (__ffs(w) - 1); w &= w - 1; }
        }
        __syncwarp();
        for (int m = 0; m < K; ++m) {
          const float ls_m = __shfl_sync(FULL, ls, m);
          for (int sl = lane; sl < nc; sl += 32) P[(size_t)m * ps + sl] = expf(__ldg(rowbase + (size_t)m * p.ldc + cls[sl]) - ls_m);
        }
        __syncwarp();
        // competitor bound q_m and its half-mask sums
        for (int m = 0; m < K; ++m) {
          float q = 0.f;
          for (int sl = lane; sl < nc; sl += 32)
            if (sl != ys) q = fmaxf(q, P[(size_t)m * ps + sl]);
          for (int off = 16; off; off >>= 1) q = fmaxf(q, __shfl_xor_sync(FULL, q, off));
          if (lane == 0) hd[warp].q[m] = q;
        }
        __syncwarp();
        for (int h = lane; h < TT; h += 32) {
          float s = 0.f;
          if (h < TA) { for (uint32_t a = (uint32_t)h; a; a &= a - 1) s += hd[warp].q[__ffs(a) - 1]; }
          else { for (uint32_t b = (uint32_t)(h - TA); b; b &= b - 1) s += hd[warp].q[p.K1 + __ffs(b) - 1]; }
          sm.QB[h] = s * (1.f + 1e-6f);
        }
        const bool tables = !ovf && nc <= p.TCAP;
        if (tables) {
          for (int h = 0; h < TT; ++h)
            for (int sl = lane; sl < nc; sl += 32) {
              float s = 0.f;
              if (h < TA) { for (uint32_t a = (uint32_t)h; a; a &= a - 1) s += sm.P[(size_t)(__ffs(a) - 1) * CAPS + sl]; }
              else { for (uint32_t b = (uint32_t)(h - TA); b; b &= b - 1) s += sm.P[(size_t)(p.K1 + __ffs(b) - 1) * CAPS + sl]; }
              sm.T[(size_t)h * TSTR + sl] = s;
            }
        }
        if (lane < K) { hd[warp].top[lane] = tp; hd[warp].mx[lane] = mx; }
        if (lane == 0) {
          hd[warp].n = n; hd[warp].y = y; hd[warp].nc = nc; hd[warp].ys = ys; hd[warp].valid = 1;
          hd[warp].ovf = ovf; hd[warp].tables = tables; hd[warp].need64 = 0;
        }
      } else if (lane == 0) {
        hd[warp].valid = 0;
      }
    }
    __syncthreads();
    // ---- phase 2: thread t owns subsets v = t + 1 + 256k ----------------------------------------
    uint32_t pending[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) pending[k] = 0;
#pragma unroll 1
    for (int s = 0; s < SBW; ++s) {
      if (!hd[s].valid) continue;
      SmpB sm;
      smp_bytes(p, smem_raw + s * sbytes, &sm);
      const int y = hd[s].y, nc = hd[s].nc, ys = hd[s].ys;
      const bool tables = hd[s].tables, ovf = hd[s].ovf;
      const float* P = ovf ? p.scratch + ((size_t)blockIdx.x * SBW + s) * (size_t)K * C : sm.P;
      const int ps = ovf ? C : CAPS;
#pragma unroll
      for (int k = 0; k < NK; ++k) {  // A4: averaged probabilities
        const uint32_t v = (uint32_t)(t + 1 + BT * k);
        if (v > (uint32_t)S) break;
        uint32_t oka = 0;
        if (__popc(v) == 1) {
          oka = hd[s].top[__ffs(v) - 1] == y;  // softmax is monotone (invariant I1)
        } else {
          const uint32_t a = v & (TA - 1), bb = v >> p.K1;
          float sy = 0.f;
          if (tables) sy = sm.T[(size_t)a * TSTR + ys] + sm.T[(size_t)(TA + bb) * TSTR + ys];
          else for (uint32_t m = v; m; m &= m - 1) sy += P[(size_t)(__ffs(m) - 1) * ps + ys];
          const float bnd = sm.QB[a] + sm.QB[TA + bb];
          if (bnd < sy * (1.f - 2.f * p.band)) {
            oka = 1;
          } else {
            float m2 = -1.f;
            if (tables) {
              const float* A = sm.T + (size_t)a * TSTR;
              const float* B = sm.T + (size_t)(TA + bb) * TSTR;
              for (int q = 0; q < nc; ++q) if (q != ys) m2 = fmaxf(m2, A[q] + B[q]);
            } else {
              for (int q = 0; q < nc; ++q) {
                if (q == ys) continue;
                float x = 0.f;
                for (uint32_t m = v; m; m &= m - 1) x += P[(size_t)(__ffs(m) - 1) * ps + q];
                m2 = fmaxf(m2, x);
              }
            }
            if (m2 > sy * (1.f + p.band)) oka = 0;
            else if (m2 < sy * (1.f - p.band)) oka = 1;
            else { pending[k] |= 1u << s; hd[s].need64 = 1; }
          }
        }
        ca[k] += oka;
      }
    }
    __syncthreads();
    // ---- phase 3 (rare): fp64 log-sum-exp of flagged samples (warp each), then pending pairs ----
    if (hd[warp].valid && hd[warp].need64) {
      const int64_t n = hd[warp].n;
      const float* rowbase = p.logits + n * K * p.ldc;
      for (int m = 0; m < K; ++m) {
        const double m64 = (double)hd[warp].mx[m];
        double s = 0.0;
        for (int c = lane; c < C; c += 32) s += exp((double)rowbase[(size_t)m * p.ldc + c] - m64);
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
        if (lane == 0) hd[warp].lse64[m] = m64 + log(s);
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
            acc += exp((double)rowbase[(size_t)mi * p.ldc + cq] - hd[s].lse64[mi]);
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
cudaError_t launch_nk(const VoteParams& p, int sm_count, cudaStream_t st, int32_t* work, unsigned int* work_count,
                      int32_t* st_top, float* st_lse, float* st_max) {
  cudaError_t e;
  {
    const int64_t nb = (p.N + SB - 1) / SB;
    const int grid = (int)(nb < (int64_t)sm_count * 2 ? nb : (int64_t)sm_count * 2);
    if (p.lse_in) vote_batch_classify_kernel<NK, true><<<grid, BT, 0, st>>>(p, work, work_count, st_top, st_lse, st_max);
    else vote_batch_classify_kernel<NK, false><<<grid, BT, 0, st>>>(p, work, work_count, st_top, st_lse, st_max);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  {
    VoteParams q = p;
    if (!p.lse_in) { q.top1_in = st_top; q.lse_in = st_lse; q.rmax_in = st_max; }
    const size_t smem = smp_bytes(q, nullptr, nullptr) * SBW;
    if ((e = cudaFuncSetAttribute(vote_batch_average_kernel<NK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem)) != cudaSuccess)
      return e;
    vote_batch_average_kernel<NK><<<sm_count, BT, smem, st>>>(q, work, work_count);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

size_t vote_batch_smem_per_sample(const VoteParams& p) { return smp_bytes(p, nullptr, nullptr); }
int vote_batch_avg_ctas_samples() { return SBW; }

cudaError_t launch_vote_batch(const VoteParams& p, int sm_count, cudaStream_t st, int32_t* work,
                              unsigned int* work_count, int32_t* st_top, float* st_lse, float* st_max) {
  if (p.N <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(work_count, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  const int nk = (p.S + BT - 1) / BT;
  if (nk <= 2) return launch_nk<2>(p, sm_count, st, work, work_count, st_top, st_lse, st_max);
  if (nk <= 4) return launch_nk<4>(p, sm_count, st, work, work_count, st_top, st_lse, st_max);
  if (nk <= 8) return launch_nk<8>(p, sm_count, st, work, work_count, st_top, st_lse, st_max);
  return launch_nk<16>(p, sm_count, st, work, work_count, st_top, st_lse, st_max);
}

}  // namespace rk
