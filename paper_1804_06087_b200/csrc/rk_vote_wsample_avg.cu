// rk_vote_wsample_avg.cu — step A4 (argmax of the averaged softmax, readings Q5/Q6) of
// every subset for the K = 9..12 worklist samples with few competitors, one WARP per sample.
//
// Same exact decision as rk_vote_cta_avg.cu: R = S_c ∩ {c : l[m][c] >= l[m][y] for some m} minus y
// (θ pruning and y-dominance); with the models split into a low half (K1 = K/2) and a
// high half, sum_{m in v} p[m][c] = TA[a][c] + TB[b][c] for v = a | b << K1, and y is the averaged
// argmax of v iff its sum beats every competitor's (ties: lowest class). fp32 decisions outside the
// relative band are exact (positive sums, relative error << band).
//
// Why a warp per sample: at K = 12, C = 100 the typical worklist sample has 1-7 competitors, so the
// 4096-subset sweep is ~1k warp instructions; the CTA kernel's five barriers and single-warp phases
// per sample cost more than the sweep. Here the whole sample lives in one warp with no block barrier:
//   * the K logit rows are read once into registers (lane l holds classes 4l..4l+3 of every row,
//     ldc <= 128), candidate bits are per-lane nibbles, the column list is a warp prefix sum;
//   * the lane owning a column computes its K probabilities; TB rows go to the warp's shared slice,
//     the lane's TA row(s) stay in registers;
//   * lane l sweeps b for its a-slot(s): per subset two packed FADD2, one FMNMX3, two FFMA whose sign
//     bits are shifted into decision words (win / near-tie), accumulated in vertical bit counters.
// Near-ties (fp32 relative gap inside the band) become (sample, subset) pairs decided in fp64 by
// vote_pair_recheck_kernel below. Samples this kernel does not take — more than WC - 1 competitors or a
// near-subnormal label probability — are appended, untouched, to the CTA kernel's worklist
// (rk_vote_cta_avg.cu); their counts come only from there.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WT = 256;      // threads per CTA
constexpr int WWARPS = WT / 32;
constexpr int kWsChunk = 4;  // worklist entries per dynamic grab
// Column groups (float4 each): y + up to 4*NG - 1 competitors; the first NR groups of the lane's TA
// rows stay in registers, the rest are read from the warp's TAX slice. Instantiations: K <= 11 <5, 3>;
// K = 12 (two a-slots per lane) <3, 3>, then a second pass <5, 0> over the samples it handed on (a
// 4th/5th register group measured slower at K = 12: register pressure).
constexpr int KM = 12;

__device__ __forceinline__ float f4c(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
__device__ __forceinline__ float max3f(float a, float b, float c) {  // FMNMX3 (sm_100)
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float4 add4(const float4& a, const float4& b) {
  const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

template <int K>
struct Geo {
  static constexpr int K1 = K / 2, KH = K - K1;
  static constexpr int TAn = 1 << K1, TBn = 1 << KH;
  static constexpr int NA = TAn >= 32 ? TAn / 32 : 1;   // a-slots per lane
  static constexpr int LPA = TAn < 32 ? 32 / TAn : 1;   // lanes sharing an a (they split b)
  static constexpr int NB = TBn / LPA;                  // b values per lane
  static constexpr int NBW = NB < 32 ? NB : 32;         // bits per decision word
  static constexpr int NWS = NB / NBW;                  // words per a-slot
  static constexpr int NW = NA * NWS;                   // decision words per lane
  static constexpr int S = (1 << K) - 1;
};

template <int NG, int NR>
struct WarpSmem {
  static constexpr int WC = 4 * NG;
  float4 TAX[NG > NR ? 64 * (NG - NR) : 1];  // TA rows' column groups NR.. (a < 2^K1 <= 64)
  float P[KM * WC];    // p[m][j] of the sample's columns (j = 0: y), zero-padded
  int32_t cols[WC];    // c_j (j = 0: y, then R ascending)
  float ls[KM];        // log sum_c exp(l - mx) per model
  float mx[KM];        // row max per model
};

template <int K>
__device__ __forceinline__ uint32_t subset_of(int lane, int s, int bi) {
  using G = Geo<K>;
  const uint32_t a = G::TAn >= 32 ? (uint32_t)(lane + 32 * s) : (uint32_t)(lane & (G::TAn - 1));
  const uint32_t b = (uint32_t)((G::TAn < 32 ? lane / G::TAn : 0) + G::LPA * bi);
  return a | (b << G::K1);
}

// the lane's decision sweep over b for one column-group count NQ (1..NG)
template <int K, int NG, int NR, int NQ>
__device__ __forceinline__ void sweep(const float4 (&ar)[Geo<K>::NA][NR > 0 ? NR : 1], const float4* TAX, const float* TB,
                                      int lane, float bl, float bh, uint32_t (&win)[Geo<K>::NW],
                                      uint32_t (&pen)[Geo<K>::NW]) {
  using G = Geo<K>;
  constexpr int WC = 4 * NG, NX = NG - NR;
  const int b0 = G::TAn < 32 ? lane / G::TAn : 0;
#pragma unroll
  for (int ws = 0; ws < G::NWS; ++ws) {
    uint32_t w[G::NA], n[G::NA];
#pragma unroll
    for (int s = 0; s < G::NA; ++s) w[s] = n[s] = 0;
#pragma unroll 4
    for (int j = 0; j < G::NBW; ++j) {
      const int b = b0 + G::LPA * (ws * G::NBW + j);
      const float4* B = reinterpret_cast<const float4*>(TB + b * WC);
      float4 bv[NQ];
#pragma unroll
      for (int g = 0; g < NQ; ++g) bv[g] = B[g];
#pragma unroll
      for (int s = 0; s < G::NA; ++s) {
        const uint32_t a = G::TAn >= 32 ? (uint32_t)(lane + 32 * s) : (uint32_t)(lane & (G::TAn - 1));
        float sy = 0.f, mc = 0.f;
#pragma unroll
        for (int g = 0; g < NQ; ++g) {
          const float4 av = g < NR ? ar[s][g < NR ? g : 0] : TAX[a * NX + (g - NR)];
          const float4 sg = add4(av, bv[g]);
          if (g == 0) {
            sy = sg.x;
            mc = max3f(sg.y, sg.z, sg.w);
          } else {
            mc = max3f(mc, sg.x, sg.y);
            mc = max3f(mc, sg.z, sg.w);
          }
        }
        // r < 0: clear win; r >= 0 > r2: near-tie; r2 >= 0: clear loss (sums are >= 1e-30 here)
        const float r = fmaf(-sy, bl, mc), r2 = fmaf(-sy, bh, mc);
        w[s] = __funnelshift_l(__float_as_uint(r), w[s], 1);
        n[s] = __funnelshift_l(~__float_as_uint(r) & __float_as_uint(r2), n[s], 1);
      }
    }
#pragma unroll
    for (int s = 0; s < G::NA; ++s) {  // bit NBW-1-j <-> b index j of this word
      win[s * G::NWS + ws] = w[s];
      pen[s * G::NWS + ws] = n[s];
    }
  }
}

template <int K, int NG, int NR>
__global__ void __launch_bounds__(WT, 2) vote_wsample_average_kernel(const VoteParams p, const int32_t* work,
                                                                     const unsigned int* work_count,
                                                                     int32_t* cta_work, unsigned int* cta_count) {
  using G = Geo<K>;
  constexpr int WC = 4 * NG;
  using WarpSmem = rk::WarpSmem<NG, NR>;
  extern __shared__ __align__(16) char dyn[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(dyn);                       // [2^K] per-CTA counts
  float* TBall = reinterpret_cast<float*>(dyn + (size_t)(G::S + 1) * 4);  // [warps][TBn][WC]
  WarpSmem* wsm = reinterpret_cast<WarpSmem*>(TBall + (size_t)WWARPS * G::TBn * WC);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int C = p.C;
  const int64_t ldc = p.ldc;
  float* TB = TBall + (size_t)warp * G::TBn * WC;
  float* P = wsm[warp].P;
  float4* TAX = wsm[warp].TAX;
  const float bh = 1.f + p.band, bl = 1.f - p.band;
  for (int i = t; i <= G::S; i += WT) cnt[i] = 0;
  __syncthreads();

  // positions (word, bit) holding v = 0 or a singleton (decided apart) -> masks per word
  uint32_t valid[G::NW], sing[G::NW];
#pragma unroll
  for (int s = 0; s < G::NA; ++s)
#pragma unroll
    for (int ws = 0; ws < G::NWS; ++ws) {
      uint32_t vm = 0, sm = 0;
      for (int j = 0; j < G::NBW; ++j) {
        const uint32_t v = subset_of<K>(lane, s, ws * G::NBW + j);
        const uint32_t bit = 1u << (G::NBW - 1 - j);
        if (v != 0 && __popc(v) > 1) vm |= bit;
        if (__popc(v) == 1) sm |= bit;
      }
      valid[s * G::NWS + ws] = vm;
      sing[s * G::NWS + ws] = sm;
    }
  uint32_t c0[G::NW], c1[G::NW], c2[G::NW], c3[G::NW], c4[G::NW];  // vertical counters (<= 31)
#pragma unroll
  for (int i = 0; i < G::NW; ++i) c0[i] = c1[i] = c2[i] = c3[i] = c4[i] = 0;
  int nadd = 0;
  auto flush = [&]() {
#pragma unroll
    for (int s = 0; s < G::NA; ++s)
#pragma unroll
      for (int ws = 0; ws < G::NWS; ++ws) {
        const int i = s * G::NWS + ws;
        const uint32_t any = c0[i] | c1[i] | c2[i] | c3[i] | c4[i];
        for (uint32_t q = any; q; q &= q - 1) {
          const int bit = __ffs(q) - 1;
          const uint32_t c = ((c0[i] >> bit) & 1u) | (((c1[i] >> bit) & 1u) << 1) | (((c2[i] >> bit) & 1u) << 2) |
                             (((c3[i] >> bit) & 1u) << 3) | (((c4[i] >> bit) & 1u) << 4);
          atomicAdd(&cnt[subset_of<K>(lane, s, ws * G::NBW + (G::NBW - 1 - bit))], c);
        }
        c0[i] = c1[i] = c2[i] = c3[i] = c4[i] = 0;
      }
    nadd = 0;
  };

  const int64_t W = *work_count;
  const int64_t gw = (int64_t)blockIdx.x * WWARPS + warp, nwarps = (int64_t)gridDim.x * WWARPS;
  const bool lane_ok = 4 * lane < ldc;
  // worklist entries handed out dynamically in chunks of kWsChunk (one atomic per chunk) when q.dyn_ctr is
  // set, instead of a fixed stride: warps that draw wide samples do not leave the others idle at the end
  const bool dyng = p.dyn_ctr != nullptr;
  auto grab = [&]() -> int64_t {
    unsigned int b = 0;
    if (lane == 0) b = atomicAdd(p.dyn_ctr, (unsigned int)kWsChunk);
    return (int64_t)__shfl_sync(FULL, b, 0);
  };
#pragma unroll 1
  for (int64_t cb = dyng ? grab() : gw; cb < W; cb = dyng ? grab() : cb + nwarps)
#pragma unroll 1
  for (int64_t e = cb, ce = dyng ? (cb + kWsChunk < W ? cb + kWsChunk : W) : cb + 1; e < ce; ++e) {
    const int64_t n = work[e];
    const int y = p.labels[n];
    // ---- statistics and θ threshold, lane m < K holds model m ----------------------
    int tp = 0;
    float ls = 0.f, mx = 0.f;
    if (lane < K) { tp = p.top1_in[n * K + lane]; ls = p.lsum_in[n * K + lane]; mx = p.rmax_in[n * K + lane]; }
    const float thr = theta_threshold(mx, ls, K, lane);
    const uint32_t ymask = __ballot_sync(FULL, lane < K && tp == y);  // models whose top-1 is y
    // ---- the K rows in registers (L1-allocating: the column pass re-reads a few values) -----------
    //      lane holds classes 4*lane .. 4*lane+3
    const float* rb = p.logits + n * K * ldc;
    float4 x[K];
#pragma unroll
    for (int m = 0; m < K; ++m)
      x[m] = lane_ok ? __ldg(reinterpret_cast<const float4*>(rb + m * ldc + 4 * lane))
                     : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    // ---- R: S_c (x >= θ threshold of some model) ∩ {x >= l[m][y] for some model}, minus y -------
    uint32_t b1 = 0, b2 = 0;
    float myly = 0.f;
    const int yl = y >> 2, yq = y & 3;
#pragma unroll
    for (int m = 0; m < K; ++m) {
      const float tm = __shfl_sync(FULL, thr, m);
      const float ym = __shfl_sync(FULL, f4c(x[m], yq), yl);
      if (lane == m) myly = ym;
      b1 |= (x[m].x >= tm ? 1u : 0u) | (x[m].y >= tm ? 2u : 0u) | (x[m].z >= tm ? 4u : 0u) | (x[m].w >= tm ? 8u : 0u);
      b2 |= (x[m].x >= ym ? 1u : 0u) | (x[m].y >= ym ? 2u : 0u) | (x[m].z >= ym ? 4u : 0u) | (x[m].w >= ym ? 8u : 0u);
    }
    const int cls0 = 4 * lane;
    uint32_t nib = b1 & b2;
    nib &= cls0 + 4 <= C ? 0xfu : (cls0 >= C ? 0u : (1u << (C - cls0)) - 1u);
    if (lane == yl) nib &= ~(1u << yq);
    const int cnt_l = __popc(nib);
    int incl = cnt_l;
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(FULL, incl, off);
      if (lane >= off) incl += o;
    }
    const int nr = __shfl_sync(FULL, incl, 31);
    // p[m][y] < e^-68 for some model: y's sums may be (nearly) subnormal -> CTA kernel (guarded)
    const bool tiny = __any_sync(FULL, lane < K && (myly - mx) - ls < -68.f);
    if (nr + 1 > WC || tiny) {
      if (lane == 0) cta_work[atomicAdd(cta_count, 1u)] = (int32_t)n;
      continue;
    }
    const int nq = (nr + 1 + 3) >> 2;  // 1..NG float4 column groups
    // ---- probabilities of the columns: lane i handles (m, j) = (i mod K, i div K), re-reading l[m][c_j]
    //      (an L1 hit: the rows were just loaded) -> p[m][j] = exp((l[m][c_j] - mx_m) - lsum_m) -------------------
    __syncwarp();  // the previous sample's readers of P / TB / cols are done
    for (int i = lane; i < K * WC / 4; i += 32) reinterpret_cast<float4*>(P)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    {
      int j = 1 + incl - cnt_l;
      for (uint32_t q = nib; q; q &= q - 1) wsm[warp].cols[j++] = cls0 + __ffs(q) - 1;
      if (lane == 0) wsm[warp].cols[0] = y;
      if (lane < K) { wsm[warp].ls[lane] = ls; wsm[warp].mx[lane] = mx; }
    }
    __syncwarp();
    for (int i = lane; i < K * (nr + 1); i += 32) {
      const int j = i / K, m = i - j * K;
      P[m * WC + j] = expf((__ldg(rb + m * ldc + wsm[warp].cols[j]) - wsm[warp].mx[m]) - wsm[warp].ls[m]);
    }
    __syncwarp();
    // ---- tables: TB rows b = lane + 32r in shared memory, the lane's TA row(s) in registers -------
    const float4* P4 = reinterpret_cast<const float4*>(P);
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      if (g >= nq) break;
#pragma unroll
      for (int r = 0; r < G::TBn / 32; ++r) {
        const uint32_t b = (uint32_t)(lane + 32 * r);
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < G::KH; ++i)
          if ((b >> i) & 1u) s = add4(s, P4[(G::K1 + i) * NG + g]);
        reinterpret_cast<float4*>(TB + b * WC)[g] = s;
      }
    }
    float4 ar[G::NA][NR > 0 ? NR : 1];
#pragma unroll
    for (int s = 0; s < G::NA; ++s) {
      const uint32_t a = G::TAn >= 32 ? (uint32_t)(lane + 32 * s) : (uint32_t)(lane & (G::TAn - 1));
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g < nq) {
#pragma unroll
          for (int i = 0; i < G::K1; ++i)
            if ((a >> i) & 1u) acc = add4(acc, P4[i * NG + g]);
        }
        if (g < NR) ar[s][g < NR ? g : 0] = acc;
        else if (g < nq && (G::TAn >= 32 || lane < G::TAn)) TAX[a * (NG - NR) + (g - NR)] = acc;
      }
    }
    __syncwarp();
    // ---- S6: every subset of the lane ------------------------------------------------------------
    uint32_t win[G::NW], pen[G::NW];
    switch (nq) {
      case 1: sweep<K, NG, NR, 1>(ar, TAX, TB, lane, bl, bh, win, pen); break;
      case 2: sweep<K, NG, NR, NG >= 2 ? 2 : NG>(ar, TAX, TB, lane, bl, bh, win, pen); break;
      case 3: sweep<K, NG, NR, NG >= 3 ? 3 : NG>(ar, TAX, TB, lane, bl, bh, win, pen); break;
      case 4: sweep<K, NG, NR, NG >= 4 ? 4 : NG>(ar, TAX, TB, lane, bl, bh, win, pen); break;
      default: sweep<K, NG, NR, NG>(ar, TAX, TB, lane, bl, bh, win, pen); break;
    }
    uint32_t pq[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < G::NW; ++i) pq[i] = pen[i] & valid[i];
    if (__any_sync(FULL, (pq[0] | pq[1] | pq[2] | pq[3]) != 0)) {
      // near-ties: (sample, subset) pairs for the fp64 recheck kernel; if the pair list is full, the whole
      // sample goes to the CTA kernel instead (slots it reserved below the capacity get a skip sentinel)
      const int np = __popc(pq[0]) + __popc(pq[1]) + __popc(pq[2]) + __popc(pq[3]);
      int incl_p = np;
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(FULL, incl_p, off);
        if (lane >= off) incl_p += o;
      }
      const int tot = __shfl_sync(FULL, incl_p, 31);
      unsigned int base = 0;
      if (lane == 0) base = atomicAdd(p.pair_count, (unsigned int)tot);
      base = __shfl_sync(FULL, base, 0);
      if ((int64_t)base + tot <= p.pair_cap) {
        int64_t slot = (int64_t)base + incl_p - np;
#pragma unroll
        for (int s = 0; s < G::NA; ++s)
#pragma unroll
          for (int wsi = 0; wsi < G::NWS; ++wsi)
            for (uint32_t q = pq[s * G::NWS + wsi]; q; q &= q - 1) {
              const uint32_t v = subset_of<K>(lane, s, wsi * G::NBW + (G::NBW - 1 - (__ffs(q) - 1)));
              p.pairs[slot++] = ((uint64_t)n << 16) | v;
            }
      } else {
        for (int64_t i = (int64_t)base + lane; i < p.pair_cap && i < (int64_t)base + tot; i += 32) p.pairs[i] = ~0ull;
        if (lane == 0) cta_work[atomicAdd(cta_count, 1u)] = (int32_t)n;
        continue;
      }
    }
#pragma unroll
    for (int s = 0; s < G::NA; ++s)
#pragma unroll
      for (int ws = 0; ws < G::NWS; ++ws) {
        const int i = s * G::NWS + ws;
        uint32_t ok = win[i] & valid[i];
        for (uint32_t q = sing[i]; q; q &= q - 1) {  // singletons: softmax is monotone (invariant I1)
          const int bit = __ffs(q) - 1;
          const uint32_t v = subset_of<K>(lane, s, ws * G::NBW + (G::NBW - 1 - bit));
          ok |= ((ymask >> (__ffs(v) - 1)) & 1u) << bit;
        }
        uint32_t c = ok, xx;
        xx = c0[i] & c; c0[i] ^= c; c = xx;
        xx = c1[i] & c; c1[i] ^= c; c = xx;
        xx = c2[i] & c; c2[i] ^= c; c = xx;
        xx = c3[i] & c; c3[i] ^= c; c = xx;
        c4[i] ^= c;
      }
    if (++nadd == 31) flush();
  }
  flush();
  __syncthreads();
  for (int i = t + 1; i <= G::S; i += WT)
    if (cnt[i]) atomicAdd(p.cnt_avg + (i - 1), (unsigned long long)cnt[i]);
}

// fp64 recheck of one near-tie (sample, subset) pair per warp, from the definition (reading
// Q6): p[m][c] = exp(l[m][c] - mx_m) / sum_c exp(l[m][c] - mx_m) in fp64 (mx_m the exact fp32 row max: the
// max-subtracted softmax of reading Q5), avg[c] = sum_{m in v} p[m][c] / |v| over every class, argmax with the lowest
// class on ties; correct iff it is y. Lane l holds classes 4l..4l+3 (ldc <= 128).
__global__ void __launch_bounds__(WT) vote_pair_recheck_kernel(const VoteParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t np = (int64_t)min((unsigned long long)*p.pair_count, (unsigned long long)p.pair_cap);
  const int64_t gw = ((int64_t)blockIdx.x * WT + threadIdx.x) >> 5, nwarps = ((int64_t)gridDim.x * WT) >> 5;
  const int K = p.K, C = p.C;
  const bool lane_ok = 4 * lane < p.ldc;
  for (int64_t e = gw; e < np; e += nwarps) {
    const uint64_t pr = p.pairs[e];
    if (pr == ~0ull) continue;
    const int64_t n = (int64_t)(pr >> 16);
    const uint32_t v = (uint32_t)(pr & 0xffffu);
    const int y = p.labels[n];
    const float* rb = p.logits + n * K * p.ldc;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t mm = v; mm; mm &= mm - 1) {  // ascending member order
      const int m = __ffs(mm) - 1;
      const float4 x = lane_ok ? *reinterpret_cast<const float4*>(rb + m * p.ldc + 4 * lane)
                               : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      const double m64 = (double)p.rmax_in[n * K + m];
      double e4[4], s = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        e4[q] = 4 * lane + q < C ? exp((double)f4c(x, q) - m64) : 0.0;
        s += e4[q];
      }
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * lane + q < C) acc[q] += e4[q] / s;
    }
    const double inv = (double)__popc(v);
    double best = -1.0;
    int bc = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double a = acc[q] / inv;
      if (4 * lane + q < C && a > best) { best = a; bc = 4 * lane + q; }
    }
    for (int off = 16; off; off >>= 1) {
      const double ob = __shfl_xor_sync(FULL, best, off);
      const int oc = __shfl_xor_sync(FULL, bc, off);
      if (ob > best || (ob == best && oc < bc)) { best = ob; bc = oc; }
    }
    if (lane == 0) {
      atomicAdd(p.n_recheck + (v - 1), 1ull);
      if (bc == y) atomicAdd(p.cnt_avg + (v - 1), 1ull);
    }
  }
}

template <int K, int NG, int NR>
cudaError_t launch_k(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                     const unsigned int* work_count, int32_t* cta_work, unsigned int* cta_count) {
  using G = Geo<K>;
  const size_t smem =
      (size_t)(G::S + 1) * 4 + (size_t)WWARPS * G::TBn * 4 * NG * 4 + (size_t)WWARPS * sizeof(WarpSmem<NG, NR>);
  cudaError_t e = cudaFuncSetAttribute(vote_wsample_average_kernel<K, NG, NR>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vote_wsample_average_kernel<K, NG, NR>, WT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  if (q.dyn_ctr && (e = cudaMemsetAsync(q.dyn_ctr, 0, sizeof(unsigned int), st)) != cudaSuccess) return e;
  vote_wsample_average_kernel<K, NG, NR><<<sm_count * per_sm, WT, smem, st>>>(q, work, work_count, cta_work, cta_count);
  return cudaGetLastError();
}

}  // namespace

bool vote_wsample_avg_supported(const VoteParams& q) {
  return q.K >= 9 && q.K <= 12 && q.ldc <= 128 && q.pairs != nullptr;
}

cudaError_t launch_vote_pair_recheck(const VoteParams& q, int sm_count, cudaStream_t st) {
  vote_pair_recheck_kernel<<<sm_count * 4, WT, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_vote_wsample_avg(const VoteParams& q, int sm_count, cudaStream_t st, int32_t* work,
                                    unsigned int* work_count, int32_t* cta_work, unsigned int* cta_count,
                                    const int32_t** rest, const unsigned int** rest_count) {
  *rest = cta_work;
  *rest_count = cta_count;
  switch (q.K) {
    case 9: return launch_k<9, 5, 3>(q, sm_count, st, work, work_count, cta_work, cta_count);
    case 10: return launch_k<10, 5, 3>(q, sm_count, st, work, work_count, cta_work, cta_count);
    case 11: return launch_k<11, 5, 3>(q, sm_count, st, work, work_count, cta_work, cta_count);
    case 12: {  // 3 register groups, then the samples with 12..19 columns from shared-memory TA rows
      cudaError_t e = launch_k<12, 3, 3>(q, sm_count, st, work, work_count, cta_work, cta_count);
      if (e == cudaSuccess) e = cudaMemsetAsync(work_count, 0, sizeof(unsigned int), st);  // work is consumed
      if (e == cudaSuccess) e = launch_k<12, 5, 0>(q, sm_count, st, cta_work, cta_count, work, work_count);
      *rest = work;
      *rest_count = work_count;
      return e;
    }
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rk
