// rk_vote_batch.cu — steps A2-A5 for K = 9..12 models (511..4095 subsets).
//
// PAPER.md passages: :153 top-1 (reading Q4), :407 majority vote with best-accuracy tie-break
// (RK_TIE_BEST_MEMBER; RK_TIE_LOWEST_CLASS = north_star), :72 averaged softmax (readings Q5, Q6),
// :429 every non-empty subset v of the model list is an action (2^|M| - 1 of them).
//
// With thousands of subsets per sample the work is the (sample, subset) sweep, evaluated bit-sliced:
// 32 subsets per word, vote counts per class from a constant "popcount >= c" table and per-class
// difference masks, the tie race on whole words, per-subset counts in vertical bit counters (kernel A
// below, one warp per 16-sample chunk). The averages go to the kernels of rk_vote_wsample_avg.cu,
// rk_vote_cta_avg.cu and rk_vote_batch_avg.cu over the worklist kernel A builds.
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
constexpr int SB = 128;          // samples per grid-sizing unit (kernel A)
constexpr int KM = 12;




// ragged-tail counts for the correct subsets of one word (samples past the last complete batch; rare)
__device__ __noinline__ void tail_add_word(const VoteParams& p, uint32_t tm, uint32_t w, uint32_t ok) {
  for (uint32_t o = ok; o; o &= o - 1) {
    const uint32_t v = (w << 5) | (uint32_t)(__ffs(o) - 1);
    for (int bi = 0; bi < p.nB; ++bi)
      if ((tm >> bi) & 1u) atomicAdd(p.tail + (size_t)bi * p.S + (v - 1), 1ull);
  }
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
    for (int c = lane; c < C; c += 32) {
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
      tp = ba; mx = bm; ls = logf(sum);  // log-sum relative to the row max
      bad = !(sum == sum) || !(bm > -INFINITY) || bm == INFINITY;
    }
  }
}

// ======================= kernel A: classify + votes, one warp per 16-sample chunk ==================
// A warp owns 16 consecutive samples (whole count groups, gs | 16): it builds each sample's vote record
// (row statistics, distinct-class voter masks) and lane l evaluates the 32-subset words w = l + 32 i
// (subsets v = 32w + lo: the low 5 models <-> bits of lo, the high models <-> bits of w) of every one
// of them -- no block barrier. Per-subset correct counts accumulate in vertical bit counters and leave
// them at each group end through a multiply-spread bit->byte transposition into the warp's staging
// row, which is copied out coalesced (grp, labelled moments) and added to the CTA's per-subset totals.
// (An earlier batch-transposed layout -- threads owning a word across a 128-sample batch in shared
// memory, two block barriers per 16 samples -- measured 5 ms per 1M samples at K = 12 against 2.5.)
constexpr int CH = 16;  // samples per warp chunk
struct WRec {  // one sample's vote record (warp-private)
  uint32_t my, lt, tm;
  int32_t no;
  uint32_t mo[KM];
};
#ifndef RK_GC_MINB
#define RK_GC_MINB 2
#endif
template <int NWL, bool STATS>
__global__ void __launch_bounds__(BT, RK_GC_MINB) vote_group_classify_kernel(const VoteParams p, int32_t* work,
                                                                    unsigned int* work_count, int32_t* st_top,
                                                                    float* st_lsum, float* st_max) {
  __shared__ uint32_t GE[32 * 8];        // GE[L][c] = {lo in [0,32) : popc(lo & L) >= c}
  __shared__ uint32_t LW[32 * 32];       // LW[A][B] = {lo : best-ranked member of lo ∩ (A ∪ B) is in A}
  __shared__ uint8_t LR[KM + 1];         // LR[r] = low models (m < 5) ranked better than r
  __shared__ int8_t rnk[KM];             // rank of each model (0 = best), BEST_MEMBER tie rule
  __shared__ uint16_t RS[2][64];         // model mask -> rank-order mask, 6 models per half
  __shared__ uint32_t cnt[1 << KM];      // per-subset correct votes of this CTA (index v)
  __shared__ uint32_t utot;              // unanimous-correct samples of this CTA
  __shared__ WRec wrec[NWB];
  extern __shared__ __align__(16) uint8_t stage_dyn[];  // [NWB][2^K] per-warp group counts, index v
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, S = p.S, C = p.C;
  const uint32_t kmask = (1u << K) - 1u;
  const int gsz = p.gs > 0 ? p.gs : CH;
  const int64_t N = p.N;
  int64_t tail0 = N;
  for (int bi = 0; bi < p.nB; ++bi) tail0 = p.tail_start[bi] < tail0 ? p.tail_start[bi] : tail0;
  for (int i = t; i < 32 * 8; i += BT) {
    const uint32_t L = (uint32_t)(i >> 3), c = (uint32_t)(i & 7);
    uint32_t wd = 0;
    for (uint32_t lo = 0; lo < 32; ++lo) wd |= ((uint32_t)__popc(lo & L) >= c ? 1u : 0u) << lo;
    GE[i] = wd;
  }
  for (int i = t; i < (1 << K); i += BT) cnt[i] = 0;
  if (t == 0) utot = 0;
  if (p.tie == 0) {
    if (t == 0) {
      uint32_t rem = kmask;
      for (int r = 0; r < K; ++r) {
        const int m = p.best_of[rem];
        rnk[m] = (int8_t)r;
        rem &= ~(1u << m);
      }
    }
    __syncthreads();
    if (t < 128) {
      const int hf = t >> 6, x = t & 63;
      uint32_t r = 0;
      for (int b = 0; b < 6; ++b)
        if (((x >> b) & 1) && 6 * hf + b < K) r |= 1u << rnk[6 * hf + b];
      RS[hf][x] = (uint16_t)r;
    }
    if (t <= K) {
      uint32_t lr = 0;
      for (int m = 0; m < 5; ++m) lr |= (rnk[m] < t ? 1u : 0u) << m;
      LR[t] = (uint8_t)lr;
    }
    for (int i = t; i < 32 * 32; i += BT) {
      const uint32_t A = (uint32_t)i >> 5, B = (uint32_t)i & 31u;
      uint32_t wd = 0;
      for (uint32_t lo = 1; lo < 32; ++lo) {
        const uint32_t s2 = lo & (A | B);
        int best = -1, br = 1 << 30;
        for (int m = 0; m < 5; ++m)
          if (((s2 >> m) & 1u) && rnk[m] < br) { br = rnk[m]; best = m; }
        if (best >= 0 && ((A >> best) & 1u)) wd |= 1u << lo;
      }
      LW[i] = wd;
    }
  }
  __syncthreads();
  const int nwd = 1 << (K - 5);
  uint32_t hwr[NWL];  // each owned word's high models, in rank order
#pragma unroll
  for (int i = 0; i < NWL; ++i) {
    const uint32_t w = (uint32_t)(lane + 32 * i);
    hwr[i] = 0;
    if (p.tie == 0)
      for (int m = 5; m < K; ++m)
        if ((w >> (m - 5)) & 1u) hwr[i] |= 1u << rnk[m];
  }
  WRec& rc = wrec[warp];
  uint8_t* stg = stage_dyn + (size_t)warp * (1 << K);
  uint32_t uw = 0;  // this warp's unanimous-correct samples (lane 0's count is authoritative)
  const int64_t nch = (N + CH - 1) / CH;
  // 16-sample chunks handed out dynamically (one atomic per chunk) when p.dyn_ctr is set, so the warps that
  // draw vote-heavy chunks do not leave the rest idle at the end
  const bool dyng = p.dyn_ctr != nullptr;
  auto grab = [&]() -> int64_t {
    unsigned int b = 0;
    if (lane == 0) b = atomicAdd(p.dyn_ctr, 1u);
    return (int64_t)__shfl_sync(FULL, b, 0);
  };
  for (int64_t ch = dyng ? grab() : (int64_t)blockIdx.x * NWB + warp; ch < nch;
       ch = dyng ? grab() : ch + (int64_t)gridDim.x * NWB) {
    const int64_t n0 = ch * CH;
    uint32_t k0[NWL], k1[NWL], k2[NWL], k3[NWL], k4[NWL];
#pragma unroll
    for (int i = 0; i < NWL; ++i) k0[i] = k1[i] = k2[i] = k3[i] = k4[i] = 0;
    uint32_t u = 0, wl = 0;
    // the chunk's labels (lane i: sample n0 + i), and the next sample's statistics and l[m][y] loaded one
    // sample ahead (STATS): the per-sample dependent load chain leaves the critical path
    const int ylane = (lane < CH && n0 + lane < N) ? p.labels[n0 + lane] : 0;
    int ntp = 0;
    float nls = 0.f, nmx = 0.f, nly = 0.f;
    auto prefetch = [&](int i) {
      const int64_t n = n0 + i;
      const int yy = __shfl_sync(FULL, ylane, i & (CH - 1));
      if (STATS && i < CH && n < N && lane < K) {
        ntp = p.top1_in[n * K + lane];
        nls = p.lsum_in[n * K + lane];
        nmx = p.rmax_in[n * K + lane];
        nly = (yy >= 0 && yy < C) ? p.logits[(n * K + lane) * p.ldc + yy] : 0.f;
      }
    };
    prefetch(0);
#pragma unroll 1
    for (int i = 0; i < CH; ++i) {
      const int64_t n = n0 + i;
      int tp = ntp;
      float mx = nmx, ls = nls;
      const float lyv = nly;
      prefetch(i + 1);
      if (n < N) {
        // ---- phase 1: the sample's record ----------------------------------------------------------
        bool eval = false;
        const int y = __shfl_sync(FULL, ylane, i);
        if (y < 0 || y >= C) {
          if (lane == 0) atomicOr(p.err + 1, 1u);
        } else {
          const float* rowbase = p.logits + n * K * p.ldc;
          bool bad = false;
          if (STATS) {
            if (lane < K) bad = !(ls > -INFINITY && ls < INFINITY) || !(mx > -INFINITY);
          } else {
            row_stats(p, rowbase, lane, tp, mx, ls, bad);
            if (lane < K) { st_top[n * K + lane] = tp; st_lsum[n * K + lane] = ls; st_max[n * K + lane] = mx; }
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
              if (__shfl_sync(FULL, c, 0) == y) {
                ++u;
                if (tm)
                  for (int bi = 0; bi < p.nB; ++bi)
                    if ((tm >> bi) & 1u)
                      for (int v1 = lane; v1 < S; v1 += 32) atomicAdd(p.tail + (size_t)bi * S + v1, 1ull);
              }
            } else {
              const float thr = theta_threshold(mx, ls, K, lane);
              const float lym = STATS ? lyv : (lane < K ? rowbase[(size_t)lane * p.ldc + y] : 0.f);
              if (__any_sync(FULL, lane < K && lym >= thr)) wl |= 1u << i;
              if (__any_sync(FULL, lane < K && c == y)) {
                eval = true;
                const bool other = lane < K && (__ffs(mm) - 1) == lane && c != y;  // one lane per other class
                const uint32_t ob = __ballot_sync(FULL, other);
                const uint32_t ltb = __ballot_sync(FULL, other && c < y);
                __syncwarp();  // the previous sample's readers of rc are done
                if (other) rc.mo[__popc(ob & ((1u << lane) - 1u))] = mm;
                if (lane < K && c == y && (__ffs(mm) - 1) == lane) rc.my = mm;
                if (lane == 0) {
                  rc.no = __popc(ob);
                  rc.tm = tm;
                  uint32_t lt = 0;  // lt bit j refers to the j-th other class in lane order
                  for (uint32_t w = ob, j = 0; w; w &= w - 1, ++j)
                    if ((ltb >> (__ffs(w) - 1)) & 1u) lt |= 1u << j;
                  rc.lt = lt;
                }
                __syncwarp();
              }
            }
          }
        }
        // ---- phase 2: the lane's words of this sample (bit-sliced A3) -----------------
        // For class j, with x(lo) = low-model votes and h = high-model votes of word w: j beats y iff
        // x_y - x_j < h_j - h_y =: -d, ties iff equal. The 32-lane ballots of (x_y - x_j >= t) for
        // t = -7..8 (lane = lo) give DG_j[t]; lane t + 7 keeps it and each lane fetches DG_j[-d] and
        // DG_j[-d + 1] for its words by shuffle: no per-word loop over vote counts.
        if (eval) {
          const uint32_t my = rc.my, lt = rc.lt, Ly = my & 31u, tmr = rc.tm;
          const int no = rc.no;
          const uint32_t gy1 = GE[Ly * 8 + 1];  // lo with x_y >= 1
          uint32_t lose[NWL];
          int hy[NWL];
#pragma unroll
          for (int wi = 0; wi < NWL; ++wi) {
            const uint32_t w = (uint32_t)(lane + 32 * wi);
            hy[wi] = __popc(w & (my >> 5));
            lose[wi] = hy[wi] == 0 ? ~gy1 : 0u;  // c_y == 0
          }
          const int xy = __popc((uint32_t)lane & Ly);
#pragma unroll 1
          for (int j = 0; j < no; ++j) {
            const uint32_t Mj = rc.mo[j];
            const int dif = xy - __popc((uint32_t)lane & Mj & 31u);  // x_y - x_j at lo = lane
            uint32_t dg = lane <= 2 ? ~0u : 0u;                   // t <= -5: always; t >= 6: never
#pragma unroll
            for (int tt = 3; tt <= 12; ++tt) {
              const uint32_t bb = __ballot_sync(FULL, dif >= tt - 7);
              if (lane == tt) dg = bb;
            }
#pragma unroll
            for (int wi = 0; wi < NWL; ++wi) {
              const uint32_t w = (uint32_t)(lane + 32 * wi);
              const int d = hy[wi] - __popc(w & (Mj >> 5));  // in [-7, 7]
              const uint32_t g = __shfl_sync(FULL, dg, 7 - d);      // x_y - x_j >= -d
              const uint32_t g1 = __shfl_sync(FULL, dg, 8 - d);     // x_y - x_j >= -d + 1
              const uint32_t eq = g & ~g1;
              lose[wi] |= ~g;
              if (p.tie != 0) {
                if ((lt >> j) & 1u) lose[wi] |= eq;
              } else if (eq & ~lose[wi]) {
                // tie race (reading Q2): is the best-ranked member of v ∩ (M_y ∪ M_j) a y voter? The high
                // members are fixed by w: the best of them (rank rh) wins unless a better low member is in lo
                const uint32_t myr = RS[0][my & 63u] | RS[1][my >> 6];
                const uint32_t hr = (myr | RS[0][Mj & 63u] | RS[1][Mj >> 6]) & hwr[wi];
                const int rh = hr ? __ffs(hr) - 1 : K;
                const bool hiy = hr && ((myr >> rh) & 1u);
                const uint32_t lr = LR[rh];
                const uint32_t A = Ly & lr, Bm = Mj & 31u & lr;
                const uint32_t ywin = LW[(A << 5) | Bm] | (hiy ? ~GE[(A | Bm) * 8 + 1] : 0u);
                lose[wi] |= eq & ~ywin;
              }
            }
          }
#pragma unroll
          for (int wi = 0; wi < NWL; ++wi) {
            const uint32_t w = (uint32_t)(lane + 32 * wi);
            if ((int)w >= nwd) break;
            const uint32_t ok = ~lose[wi] & (w == 0 ? ~1u : ~0u);  // v = 0 is not a subset
            uint32_t cc = ok, x;  // vertical counter += ok
            x = k0[wi] & cc; k0[wi] ^= cc; cc = x;
            x = k1[wi] & cc; k1[wi] ^= cc; cc = x;
            x = k2[wi] & cc; k2[wi] ^= cc; cc = x;
            x = k3[wi] & cc; k3[wi] ^= cc; cc = x;
            k4[wi] ^= cc;
            if (ok && tmr) tail_add_word(p, tmr, w, ok);
          }
        }
      }
      // ---- group end: per-subset counts (+ unanimous) -> staging row -> grp and the CTA totals -----
      if ((i + 1) % gsz == 0) {
        const int64_t gstart = n0 + i + 1 - gsz;
        if (gstart < N) {
          const uint32_t ub = u * 0x01010101u;
#pragma unroll
          for (int wi = 0; wi < NWL; ++wi) {
            const int w = lane + 32 * wi;
            if (w >= nwd) break;
            uint32_t* dst = reinterpret_cast<uint32_t*>(stg + 32 * w);
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // subsets 4q..4q+3 of the word: bit b of each count -> byte
              uint32_t o = ub;
              o += (((k0[wi] >> (4 * q)) & 0xfu) * 0x00204081u & 0x01010101u);
              o += (((k1[wi] >> (4 * q)) & 0xfu) * 0x00204081u & 0x01010101u) << 1;
              o += (((k2[wi] >> (4 * q)) & 0xfu) * 0x00204081u & 0x01010101u) << 2;
              o += (((k3[wi] >> (4 * q)) & 0xfu) * 0x00204081u & 0x01010101u) << 3;
              o += (((k4[wi] >> (4 * q)) & 0xfu) * 0x00204081u & 0x01010101u) << 4;
              dst[q] = o;
            }
            k0[wi] = k1[wi] = k2[wi] = k3[wi] = k4[wi] = 0;
          }
          __syncwarp();
          const int64_t gi = gstart / gsz;
          if (p.grp) {  // group counts: 4-byte stores on the aligned interior of the row (bytes v1 = v - 1)
            uint8_t* g = p.grp + gi * S;
            const int head = (int)((4 - ((uintptr_t)g & 3)) & 3);
            const int nword = (S - head) >> 2, tail0 = head + 4 * nword;
            if (lane < head) g[lane] = stg[lane + 1];
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(stg);
            const int sh = 8 * ((head + 1) & 3);  // stg byte offset of v1 = head + 4j is head + 4j + 1
            for (int j = lane; j < nword; j += 32) {
              const int o = (head + 4 * j + 1) >> 2;
              const uint32_t lo = sw[o], hi = sw[o + 1];
              reinterpret_cast<uint32_t*>(g + head)[j] = sh ? __funnelshift_r(lo, hi, sh) : lo;
            }
            if (tail0 + lane < S) g[tail0 + lane] = stg[tail0 + lane + 1];
          } else {  // no group counts: per-subset totals here (otherwise the q pass sums the groups)
            for (int v1 = lane; v1 < S; v1 += 32) {
              const uint32_t tot = stg[v1 + 1];
              if (tot) atomicAdd(&cnt[v1 + 1], tot);
            }
          }
          __syncwarp();
          uw += u;
        }
        u = 0;
      }
    }
    if (wl) {  // worklist append: one atomic per warp per chunk
      unsigned int base = 0;
      if (lane == 0) base = atomicAdd(work_count, (unsigned int)__popc(wl));
      base = __shfl_sync(FULL, base, 0);
      if (lane < CH && ((wl >> lane) & 1u)) work[base + __popc(wl & ((1u << lane) - 1u))] = (int32_t)(n0 + lane);
    }
  }
  if (lane == 0 && uw) atomicAdd(&utot, uw);
  __syncthreads();
  const uint32_t ua = utot;
  for (int v1 = t; v1 < S; v1 += BT) {
    if (cnt[v1 + 1]) atomicAdd(p.cnt_vote + v1, (unsigned long long)cnt[v1 + 1]);
    if (ua) atomicAdd(p.cnt_avg + v1, (unsigned long long)ua);
  }
}

template <int NK>
cudaError_t launch_nk(const VoteParams& p, int sm_count, cudaStream_t st, int32_t* work, unsigned int* work_count,
                      int32_t* st_top, float* st_lsum, float* st_max) {
  cudaError_t e;
  {
    const int64_t nb = (p.N + SB - 1) / SB;
    const int grid = (int)(nb < (int64_t)sm_count * RK_GC_MINB ? nb : (int64_t)sm_count * RK_GC_MINB);
    if (p.dyn_ctr && (e = cudaMemsetAsync(p.dyn_ctr, 0, sizeof(unsigned int), st)) != cudaSuccess) return e;
    constexpr int NWL = NK / 4 > 0 ? NK / 4 : 1;  // words per lane: 2^(K-5) / 32 (K = 9: half the lanes idle)
    const int dsm = (NWB << p.K) + 16;  // + padding: the copy-out reads one word past a row
    if (p.lsum_in) {
      if ((e = cudaFuncSetAttribute(vote_group_classify_kernel<NWL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    dsm)) != cudaSuccess)
        return e;
      vote_group_classify_kernel<NWL, true><<<grid, BT, dsm, st>>>(p, work, work_count, st_top, st_lsum, st_max);
    } else {
      if ((e = cudaFuncSetAttribute(vote_group_classify_kernel<NWL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    dsm)) != cudaSuccess)
        return e;
      vote_group_classify_kernel<NWL, false><<<grid, BT, dsm, st>>>(p, work, work_count, st_top, st_lsum, st_max);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  {  // averages on the worklist, from statistics (the GEMM's or the classify kernel's)
    VoteParams q = p;
    if (!p.lsum_in) { q.top1_in = st_top; q.lsum_in = st_lsum; q.rmax_in = st_max; }
    if (vote_large_needed(q)) return launch_vote_large_avg(q, sm_count, st, work, work_count);  // ldc > 1024
    if (vote_wsample_avg_supported(q)) {  // few competitors: warp per sample; the rest -> CTA kernel
      const int32_t* rest = nullptr;
      const unsigned int* rest_count = nullptr;
      if ((e = launch_vote_wsample_avg(q, sm_count, st, work, work_count, p.cta_work, p.cta_count, &rest,
                                       &rest_count)) != cudaSuccess)
        return e;
      if ((e = launch_vote_pair_recheck(q, sm_count, st)) != cudaSuccess) return e;
      if ((e = launch_vote_cta_avg(q, sm_count, st, rest, rest_count, p.ovf_work, p.ovf_count)) != cudaSuccess) return e;
    } else if ((e = launch_vote_cta_avg(q, sm_count, st, work, work_count, p.ovf_work, p.ovf_count)) != cudaSuccess) {
      return e;
    }
    if ((e = launch_vote_batch_avg(q, sm_count, st, p.ovf_work, p.ovf_count)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace


cudaError_t launch_vote_batch(const VoteParams& p, int sm_count, cudaStream_t st, int32_t* work,
                              unsigned int* work_count, int32_t* st_top, float* st_lsum, float* st_max) {
  if (p.N <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(work_count, 0, sizeof(unsigned int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.ovf_count, 0, sizeof(unsigned int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.cta_count, 0, sizeof(unsigned int), st);
  if (e == cudaSuccess && p.pair_count) e = cudaMemsetAsync(p.pair_count, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  const int nk = (p.S + BT - 1) / BT;
  if (nk <= 2) return launch_nk<2>(p, sm_count, st, work, work_count, st_top, st_lsum, st_max);
  if (nk <= 4) return launch_nk<4>(p, sm_count, st, work, work_count, st_top, st_lsum, st_max);
  if (nk <= 8) return launch_nk<8>(p, sm_count, st, work, work_count, st_top, st_lsum, st_max);
  return launch_nk<16>(p, sm_count, st, work, work_count, st_top, st_lsum, st_max);
}

}  // namespace rk
