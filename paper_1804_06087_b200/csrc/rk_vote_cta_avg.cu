// rk_vote_cta_avg.cu — step A4 (argmax of the averaged softmax, readings Q5/Q6) of every
// subset for the worklist samples, one sample per CTA at a time, exact half-mask tables over every
// competitor.
//
// For a worklist sample (label y is a candidate, models not unanimous), a class c can be the argmax
// of some subset's average only if c ∈ S_c (θ pruning) and l[m][c] >= l[m][y] for some
// model m (otherwise p[m][c] < p[m][y] in every member). R = that set minus y. With the models split
// into a low half (K1) and a high half, every subset v = a | b<<K1 has
//     sum_{m in v} p[m][c] = TA[a][c] + TB[b][c]
// so y is the subset's averaged argmax iff TA[a][y] + TB[b][y] beats every c ∈ R (ties: lowest class).
// The decision per (v, c) is one add and two compares in fp32 with a relative band: clear wins and
// losses are exact (positive sums, relative error << band); the band (and tiny sums) goes to an fp64
// recheck computed from the sample's rows, which are in shared memory.
//
// sm_100a layout: the K logit rows of a sample are contiguous ([N][K][ldc]); the CTA fetches them with
// one cp.async.bulk (TMA, mbarrier complete_tx), prefetching the next sample while it decides the
// current one (double buffer when two copies fit). 256 threads: thread t decides subsets t + 256k.
// Samples whose columns do not fit p.cta_cols (<= JS) slots are appended to an overflow worklist for rk_vote_batch_avg.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int CT = 256;            // threads per CTA
constexpr int CW = CT / 32;
constexpr int JS = 52;             // table columns: y + up to 51 competitors, padded to float4; 208 B rows
                                   // (13 x 16 B, odd): 128-bit loads from 8 distinct rows hit distinct bank groups
constexpr int KM = 12;

__host__ __device__ inline size_t a128(size_t x) { return (x + 127) & ~size_t(127); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Lay {  // dynamic shared memory layout
  size_t rows, tab, pm, pend, cnt, total;
  int nbuf;
};
__host__ __device__ inline Lay layout(const VoteParams& p) {
  Lay L;
  const size_t rowbytes = a128((size_t)p.K * p.ldc * 4);
  L.nbuf = 2 * rowbytes <= 64 * 1024 ? 2 : 1;
  const int TT = (1 << p.K1) + (1 << (p.K - p.K1));
  L.rows = 0;
  L.tab = L.rows + L.nbuf * rowbytes;
  L.pm = L.tab + a128((size_t)TT * JS * 4);
  L.pend = L.pm + a128((size_t)p.K * JS * 4);
  L.cnt = L.pend + a128((size_t)(p.S + 1) * 2);
  L.total = L.cnt + a128((size_t)((p.S + CT) / CT) * CT * 4);
  return L;
}

struct Stat {  // per-sample statistics, loaded one sample ahead (double-buffered)
  int64_t n;
  int32_t y;
  int32_t top[KM];
  float ls[KM], thr[KM], mx[KM];
};
struct Shared {  // static shared state
  uint64_t bar[2];
  uint32_t bm[32];
  int32_t cols[JS];  // 0 = y, 1..nr = R ascending, -1 = unused
  Stat st[2];
  double sum64[KM];
  int32_t nq, npend, skip, tiny;
};

// warp 0: labels, top-1, log-sum-exp, row max of worklist entry e; θ threshold per model
__device__ __forceinline__ void load_stat(const VoteParams& p, const int32_t* work, int64_t e, Stat& st, int lane) {
  const int K = p.K;
  const int64_t n = work[e];
  float mx = 0.f, ls = 0.f;
  int tp = 0;
  if (lane < K) { tp = p.top1_in[n * K + lane]; ls = p.lsum_in[n * K + lane]; mx = p.rmax_in[n * K + lane]; }
  const float thr = theta_threshold(mx, ls, K, lane);
  if (lane < K) { st.top[lane] = tp; st.ls[lane] = ls; st.mx[lane] = mx; st.thr[lane] = thr; }
  if (lane == 0) { st.n = n; st.y = p.labels[n]; }
}

// S6 for the subsets v = t + 256k of this thread. Because 2^K1 divides 256, the low half a = v mod 2^K1
// is the same for all k: its table row stays in registers (NQ float4 column groups; NQ = 0: runtime
// count, row re-read). The high half b = v >> K1 is uniform across a warp (K1 <= 5) or shared by
// groups of lanes, so its row is a broadcast read. Branch-free: bit k of okm = subset t + 256k clearly
// won by y, bit k of pm = near-tie (fp64 recheck); singletons and invalid slots are fixed by the caller.
__device__ __forceinline__ float max3f(float a, float b, float c) {  // FMNMX3 (sm_100)
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// one float4 column group of the row pair: y's sum (group 0 only) and the running competitor max; the
// four sums as two packed FADD2 (sm_100 add.rn.f32x2), the max as FMNMX3
__device__ __forceinline__ void group_sum(const float4& a, const float4& b, float& sy, float& mc, bool first) {
  const float2 s01 = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  const float2 s23 = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
  if (first) {
    sy = s01.x;
    mc = max3f(s01.y, s23.x, s23.y);
  } else {
    mc = max3f(mc, s01.x, s01.y);
    mc = max3f(mc, s23.x, s23.y);
  }
}

template <int NSUB, int NQ>
__device__ __forceinline__ void decide_subsets(const VoteParams& p, const float* TA, const float* TB, uint32_t& okm,
                                               uint32_t& pm, int nq_rt = 0, bool tiny = false) {
  const int t = threadIdx.x;
  const int K1 = p.K1, TAn = 1 << K1;
  const uint32_t a = (uint32_t)t & (uint32_t)(TAn - 1);
  const float4* A = reinterpret_cast<const float4*>(TA + a * JS);
  const float bh = 1.f + p.band, bl = 1.f - p.band;
  float4 ar[NQ > 0 ? NQ : 1];
#pragma unroll
  for (int q = 0; q < (NQ > 0 ? NQ : 1); ++q) ar[q] = A[q];
  const float4* B0 = reinterpret_cast<const float4*>(TB + (t >> K1) * JS);
  const int bstep = (CT >> K1) * (JS / 4);  // float4 stride of b between k and k + 1
  uint32_t w = 0, n = 0;
#pragma unroll
  for (int k = 0; k < NSUB; ++k) {
    const float4* B = B0 + k * bstep;
    float sy, mc;
    group_sum(ar[0], B[0], sy, mc, true);
    if (NQ > 0) {
#pragma unroll
      for (int q = 1; q < NQ; ++q) group_sum(ar[q], B[q], sy, mc, false);
    } else {
      for (int q = 1; q < nq_rt; ++q) group_sum(A[q], B[q], sy, mc, false);
    }
    // r < 0: every competitor below y by more than the band (clear win); r >= 0 and r2 < 0: near-tie
    // (fp64 recheck); r2 >= 0: clear loss. Positive sums: relative error << band. A sample with a
    // (nearly) subnormal y probability (tiny, runtime-count variant only) decides only clear losses.
    float r = fmaf(-sy, bl, mc), r2 = fmaf(-sy, bh, mc);
    if (NQ == 0 && tiny && !(sy >= 1e-30f)) {
      r = 1.f;
      r2 = mc > 2e-30f ? 1.f : -1.f;
    }
    w = __funnelshift_l(__float_as_uint(r), w, 1);  // w = w << 1 | sign(r)
    n = __funnelshift_l(~__float_as_uint(r) & __float_as_uint(r2), n, 1);
  }
  okm = __brev(w) >> (32 - NSUB);  // bit k <-> subset t + 256k
  pm = __brev(n) >> (32 - NSUB);
}

template <int NSUB>
__global__ void __launch_bounds__(CT, 3) vote_cta_average_kernel(const VoteParams p, const int32_t* work,
                                                                 const unsigned int* work_count, int32_t* ovf_work,
                                                                 unsigned int* ovf_count) {
  extern __shared__ __align__(128) char dyn[];
  __shared__ Shared sh;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, C = p.C, S = p.S, K1 = p.K1;
  const int TAn = 1 << K1;
  const Lay L = layout(p);
  const size_t rowbytes = a128((size_t)K * p.ldc * 4);
  const uint32_t ldbytes = (uint32_t)((size_t)K * p.ldc * 4);
  float* TA = reinterpret_cast<float*>(dyn + L.tab);
  float* TB = TA + (size_t)TAn * JS;
  float* Pm = reinterpret_cast<float*>(dyn + L.pm);
  uint16_t* pend = reinterpret_cast<uint16_t*>(dyn + L.pend);
  const int64_t W = *work_count;

  if (t == 0) {
    mbar_init(&sh.bar[0], 1);
    mbar_init(&sh.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t == 0) sh.npend = 0;
  __syncthreads();
  auto issue = [&](int64_t e, int buf) {
    const int64_t n = work[e];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the buffer first
    mbar_expect_tx(&sh.bar[buf], ldbytes);
    bulk_load(dyn + L.rows + buf * rowbytes, p.logits + n * K * p.ldc, ldbytes, &sh.bar[buf]);
  };
  if (t == 0 && (int64_t)blockIdx.x < W) issue(blockIdx.x, 0);
  if (warp == 0 && (int64_t)blockIdx.x < W) load_stat(p, work, blockIdx.x, sh.st[0], lane);
  __syncthreads();  // the first sample's statistics

  uint32_t* ca = reinterpret_cast<uint32_t*>(dyn + L.cnt);  // ca[t + CT*k]: this thread's subsets only
#pragma unroll
  for (int k = 0; k < NSUB; ++k) ca[t + CT * k] = 0;
  // per-sample decision words (bit k <-> subset t + 256k) accumulate in a 6-plane vertical counter,
  // folded into ca every 63 samples
  uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
  int nadd = 0;
  uint32_t validm = 0, singm = 0;  // slots k holding a subset 1..S; singleton subsets (handled apart)
#pragma unroll
  for (int k = 0; k < NSUB; ++k) {
    const uint32_t v = (uint32_t)(t + CT * k);
    const bool valid = v >= 1 && v <= (uint32_t)S;
    validm |= (uint32_t)valid << k;
    singm |= (uint32_t)(valid && __popc(v) == 1) << k;
  }
  validm &= ~singm;
  auto fold = [&]() {
#pragma unroll
    for (int k = 0; k < NSUB; ++k)
      ca[t + CT * k] += ((c0 >> k) & 1u) | (((c1 >> k) & 1u) << 1) | (((c2 >> k) & 1u) << 2) | (((c3 >> k) & 1u) << 3) |
               (((c4 >> k) & 1u) << 4) | (((c5 >> k) & 1u) << 5);
    c0 = c1 = c2 = c3 = c4 = c5 = 0;
    nadd = 0;
  };

  int64_t it = 0;
  for (int64_t e = blockIdx.x; e < W; e += gridDim.x, ++it) {
    const int buf = L.nbuf == 2 ? (int)(it & 1) : 0;
    const uint32_t par = L.nbuf == 2 ? (uint32_t)((it >> 1) & 1) : (uint32_t)(it & 1);
    if (t == 0 && L.nbuf == 2 && e + gridDim.x < W) issue(e + gridDim.x, buf ^ 1);  // prefetch
    const float* rows = reinterpret_cast<const float*>(dyn + L.rows + buf * rowbytes);
    const int sb = (int)(it & 1);
    const Stat& st = sh.st[sb];
    mbar_wait(&sh.bar[buf], par);  // every thread: the sample's rows have landed (the statistics were
    const int y = st.y;            // loaded last iteration, before its final barrier)
    // ---- S2: R ∪ {y} as a bitmap: warp w owns 32-class words, ORs ballots over the K rows of
    //      S_c (l >= θ-threshold) and of {c : l[m][c] >= l[m][y]}, then stores their AND -------------
    {
      const int nw = (C + 31) >> 5;
      for (int w = warp; w < nw; w += CW) {
        const int c = w * 32 + lane;
        uint32_t b1 = 0, b2 = 0;
        for (int m = 0; m < K; ++m) {
          const float* row = rows + m * (int)p.ldc;
          const float x = c < C ? row[c] : -INFINITY;
          b1 |= __ballot_sync(FULL, x >= st.thr[m]);
          b2 |= __ballot_sync(FULL, x >= row[y]);
        }
        if (lane == 0) sh.bm[w] = b1 & b2;
      }
    }
    __syncthreads();
    // ---- S3: columns (warp 0): 0 = y, 1..nr = R ascending; unused slots up to a float4 boundary hold
    //      -1 (zero probability). Samples whose columns do not fit go to the overflow worklist.
    if (warp == 0) {
      uint32_t word = lane < ((C + 31) >> 5) ? sh.bm[lane] : 0u;
      if (lane == (y >> 5)) word &= ~(1u << (y & 31));
      const int cnt = __popc(word);
      int incl = cnt;
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += o;
      }
      const int nr = __shfl_sync(FULL, incl, 31);
      const int nq = (nr + 1 + 3) >> 2;
      const bool fits = 4 * nq <= p.cta_cols;
      // p[m][y] < e^-68 (~3e-30) for some model: y's subset sums may be (nearly) subnormal
      const bool tiny = __any_sync(FULL, lane < K && (rows[(size_t)lane * p.ldc + y] - st.mx[lane]) - st.ls[lane] < -68.f);
      if (fits) {
        if (lane < 4) sh.cols[4 * nq - 4 + lane] = -1;
        __syncwarp();
        int k = 1 + incl - cnt;
        for (uint32_t w = word; w; w &= w - 1) sh.cols[k++] = lane * 32 + (__ffs(w) - 1);
      }
      if (lane == 0) {
        sh.cols[0] = y;
        sh.nq = nq;
        sh.skip = !fits;
        sh.tiny = tiny;
        if (!fits) ovf_work[atomicAdd(ovf_count, 1u)] = (int32_t)st.n;  // rk_vote_batch_avg.cu
      }
    }
    __syncthreads();
    if (warp == CW - 1 && e + gridDim.x < W) load_stat(p, work, e + gridDim.x, sh.st[sb ^ 1], lane);
    if (!sh.skip) {
      const int nq = sh.nq, nj4 = 4 * nq;
      // ---- S4: p[m][c] = exp((l - mx) - lsum) for every column ------------------------------------------
      for (int i = t; i < K * nj4; i += CT) {
        const int m = i / nj4, j = i - m * nj4;
        const int c = sh.cols[j];
        Pm[m * JS + j] = c >= 0 ? expf((rows[(size_t)m * p.ldc + c] - st.mx[m]) - st.ls[m]) : 0.f;
      }
      __syncthreads();
      // ---- S5: half-mask tables TA[h][j] = sum_{m in h} p[m][j] (ascending m), TB rows after TA:
      //      thread t owns row h = t mod 128 and every other column ---------------------------------
      {
        const int TT = TAn + (1 << (K - K1));
        const int h = t & 127;
        if (h < TT) {
          const bool lo = h < TAn;
          const uint32_t hm = lo ? (uint32_t)h : (uint32_t)(h - TAn);
          const int mo = lo ? 0 : K1;
          const float* pc = Pm + mo * JS;
          for (int j = t >> 7; j < nj4; j += CT / 128) {
            float s = 0.f;
#pragma unroll
            for (int b = 0; b < 6; ++b)
              if ((hm >> b) & 1u) s += pc[b * JS + j];
            TA[h * JS + j] = s;
          }
        }
      }
      __syncthreads();
      // ---- S6: every subset: sum of y's column and the largest competitor, branch-free ----------
      uint32_t okm, pm;
      switch (sh.tiny ? 0 : nq) {
        case 1: decide_subsets<NSUB, 1>(p, TA, TB, okm, pm); break;
        case 2: decide_subsets<NSUB, 2>(p, TA, TB, okm, pm); break;
        case 3: decide_subsets<NSUB, 3>(p, TA, TB, okm, pm); break;
        case 4: decide_subsets<NSUB, 4>(p, TA, TB, okm, pm); break;
        default: decide_subsets<NSUB, 0>(p, TA, TB, okm, pm, nq, sh.tiny); break;
      }
      okm &= validm;
      pm &= validm;
      for (uint32_t sm = singm; sm; sm &= sm - 1) {  // singletons: softmax is monotone (invariant I1)
        const int k = __ffs(sm) - 1;
        const uint32_t v = (uint32_t)(t + CT * k);
        okm |= (uint32_t)(st.top[__ffs(v) - 1] == y) << k;
      }
      for (uint32_t q = pm; q; q &= q - 1)  // rare: near-ties to the fp64 recheck
        pend[atomicAdd(&sh.npend, 1)] = (uint16_t)(t + CT * (__ffs(q) - 1));
      {
        uint32_t c = okm, x;
        x = c0 & c; c0 ^= c; c = x;
        x = c1 & c; c1 ^= c; c = x;
        x = c2 & c; c2 ^= c; c = x;
        x = c3 & c; c3 ^= c; c = x;
        x = c4 & c; c4 ^= c; c = x;
        c5 ^= c;
        if (++nadd == 63) fold();
      }
      __syncthreads();
      // ---- S7 (rare): fp64 recheck of the pending subsets from the rows in shared memory --------
      const int np = sh.npend;
      if (np) {
        for (int m = warp; m < K; m += CW) {
          const double m64 = (double)st.mx[m];
          double s = 0.0;
          for (int c = lane; c < C; c += 32) s += exp((double)rows[(size_t)m * p.ldc + c] - m64);
          for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
          if (lane == 0) sh.sum64[m] = s;  // sum_c exp(l - st.mx[m])
        }
        __syncthreads();
        for (int i = warp; i < np; i += CW) {
          const uint32_t v = pend[i];
          double best = -1.0;
          int bestc = 0x7fffffff;
          for (int j = lane; j < nj4; j += 32) {
            const int c = sh.cols[j];
            if (c < 0) continue;
            double acc = 0.0;
            for (uint32_t mm = v; mm; mm &= mm - 1) {
              const int m = __ffs(mm) - 1;
              acc += exp((double)rows[(size_t)m * p.ldc + c] - (double)st.mx[m]) / sh.sum64[m];
            }
            const double a64 = acc / (double)__popc(v);
            if (a64 > best || (a64 == best && c < bestc)) { best = a64; bestc = c; }
          }
          for (int off = 16; off; off >>= 1) {
            const double ob = __shfl_xor_sync(FULL, best, off);
            const int oc = __shfl_xor_sync(FULL, bestc, off);
            if (ob > best || (ob == best && oc < bestc)) { best = ob; bestc = oc; }
          }
          if (lane == 0) {
            atomicAdd(p.n_recheck + (v - 1), 1ull);
            if (bestc == y) atomicAdd(p.cnt_avg + (v - 1), 1ull);
          }
        }
      }
    }
    __syncthreads();  // rows, tables and the pending list are free again
    if (t == 0) {
      sh.npend = 0;
      if (L.nbuf == 1 && e + gridDim.x < W) issue(e + gridDim.x, 0);
    }
  }
  fold();
#pragma unroll
  for (int k = 0; k < NSUB; ++k) {
    const int v1 = t + CT * k - 1;
    if (v1 >= 0 && v1 < S && ca[t + CT * k]) atomicAdd(p.cnt_avg + v1, (unsigned long long)ca[t + CT * k]);
  }
}

template <int NSUB>
cudaError_t launch_nsub(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                        const unsigned int* work_count, int32_t* ovf_work, unsigned int* ovf_count) {
  const Lay L = layout(q);
  cudaError_t e = cudaFuncSetAttribute(vote_cta_average_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L.total);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vote_cta_average_kernel<NSUB>, CT, L.total);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  vote_cta_average_kernel<NSUB><<<sm_count * per_sm, CT, L.total, st>>>(q, work, work_count, ovf_work, ovf_count);
  return cudaGetLastError();
}

}  // namespace

size_t vote_cta_avg_smem(const VoteParams& q) { return layout(q).total; }

cudaError_t launch_vote_cta_avg(const VoteParams& q, int sm_count, cudaStream_t st, const int32_t* work,
                                const unsigned int* work_count, int32_t* ovf_work, unsigned int* ovf_count) {
  const int nsub = (q.S + 1 + CT - 1) / CT;  // subsets 1..S over thread slots t + 256k
  if (nsub <= 1) return launch_nsub<1>(q, sm_count, st, work, work_count, ovf_work, ovf_count);
  if (nsub <= 2) return launch_nsub<2>(q, sm_count, st, work, work_count, ovf_work, ovf_count);
  if (nsub <= 4) return launch_nsub<4>(q, sm_count, st, work, work_count, ovf_work, ovf_count);
  if (nsub <= 8) return launch_nsub<8>(q, sm_count, st, work, work_count, ovf_work, ovf_count);
  return launch_nsub<16>(q, sm_count, st, work, work_count, ovf_work, ovf_count);
}

}  // namespace rk
