// rk_moments.cu — batch latency moments (A5), chunk -> table merge, labelled moments, and the
// reward fold of eq. `multi_acc_reward` (A7).
//
// PAPER.md passages:
//   PAPER.md:345-346  l(s) = waiting + inference time; overdue <=> l(s) > tau (strict).
//   PAPER.md:410      synchronous ensemble finishes with its slowest member (stragglers):
//                     c(v,b) = max_{m in v} c(m,b).
//   PAPER.md:431-433  reward a(M[v]) * (b - beta * |{s in batch : l(s) > tau}|).
//   PAPER.md:357-359  eq. `eq:single`: exceeding time max(0, l(s) - tau).
// Readings: Q8 wait = t_last(j) - t_s (dispatch when the batch is full, no backlog);
// Q9 t_s = floor(s*1e9/r) in IEEE double, s global; Q13 trailing partial batch excluded.
//
// The overdue count of a batch depends on v only through c(v,b), i.e. through the slowest member,
// so it is computed per (rate, batch size, slowest model) -- K values instead of 2^K-1 -- by a
// binary search over the batch's non-decreasing arrival times, and scattered to subsets by the
// merge kernel.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "rk_internal.h"

namespace rk {
namespace {

__device__ __forceinline__ int64_t arrival_at(const int64_t* arr, int64_t local, int64_t global, double rate) {
  if (arr) return arr[local];
  const double num = __dmul_rn((double)global, 1e9);
  return (int64_t)floor(__ddiv_rn(num, rate));
}
// The same value as arrival_at(nullptr, ., global, rate) (reading Q9: floor of the correctly rounded
// quotient), with the fp64 division replaced by a multiplication by inv = 1/rate whenever the product
// is farther than its error bound (< 4e-16 relative, both roundings and inv's included) from an
// integer: then both floors agree; otherwise (probability ~1e-5) the exact division decides.
__device__ __forceinline__ int64_t arrival_uniform(int64_t global, double rate, double inv) {
  const double num = __dmul_rn((double)global, 1e9);
  const double x = __dmul_rn(num, inv);
  const double q = floor(x), fr = x - q, d = 4e-16 * x + 1e-300;
  if (fr > d && fr < 1.0 - d) return (int64_t)q;
  return (int64_t)floor(__ddiv_rn(num, rate));
}

// ---- overdue / exceed sums per (r, b, slowest model) ------------------------------------------
__global__ void overdue_kernel(const MomentParams p, unsigned int* err) {
  __shared__ unsigned long long so[kMaxR * kMaxB * kMaxK];
  __shared__ unsigned long long se[kMaxR * kMaxB * kMaxK];
  const int nT = p.nR * p.nB * p.K;
  for (int i = threadIdx.x; i < nT; i += blockDim.x) { so[i] = 0; se[i] = 0; }
  __syncthreads();
  // flattened work: (bi, r, jl) with jl < floor(N / B[bi])
  int64_t tot = 0;
  int64_t start[kMaxB];
  for (int bi = 0; bi < p.nB; ++bi) { start[bi] = tot; tot += (p.N / p.B[bi]) * p.nR; }
  // warp-uniform loop: consecutive work items of a warp share (b, r) almost always, so the per-(r, b, m)
  // sums are reduced across the warp first and added with one shared atomic (the per-lane shared
  // atomics on one address were 70 % of this kernel's stall samples at the c5 shape)
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < tot;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = base + lane;
    const bool act = w < tot;
    int bi = 0;
    while (bi + 1 < p.nB && w >= start[bi + 1]) ++bi;
    const int64_t rem = act ? w - start[bi] : 0;
    const int64_t nb = p.N / p.B[bi];
    const int r = (int)(rem / nb);
    const int64_t jl = rem - (int64_t)r * nb;
    const int b = p.B[bi];
    int cnt[kMaxK];
    unsigned long long ex[kMaxK];
#pragma unroll
    for (int m = 0; m < kMaxK; ++m) { cnt[m] = 0; ex[m] = 0; }
    if (act) {
      const int64_t s0 = jl * b;  // local index of the batch's first request
      const double rate = p.rates[r];
      const double inv = __drcp_rn(rate);
      const int64_t tl = arrival_at(p.arrival, s0 + b - 1, p.goff + s0 + b - 1, rate);
      if (p.arrival && r == 0) {  // arrivals must be non-decreasing inside a batch (FIFO)
        for (int i = 1; i < b; ++i)
          if (p.arrival[s0 + i] < p.arrival[s0 + i - 1]) { atomicOr(err + 2, 1u); break; }
      }
      int64_t fm[kMaxK];  // completion time of the batch when m is the slowest member
      for (int m = 0; m < p.K; ++m)
        fm[m] = p.fin ? p.fin[p.fin_off[bi] + ((int64_t)r * p.K + m) * nb + jl] : tl + p.lat[m * p.nB + bi];
      for (int m = 0; m < p.K; ++m) {
        // overdue <=> l(s) = F - t_s > tau <=> t_s < F - tau ; t_s non-decreasing in s. F = t_last + c
        // (reading Q8) or the FIFO finish time (queue mode, reading Q15)
        const int64_t thr = fm[m] - p.tau;
        int lo = 0;  // first i with t_i >= thr
        if (p.arrival) {  // caller arrivals: binary search
          int hi = b;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const int64_t tm = arrival_at(p.arrival, s0 + mid, p.goff + s0 + mid, rate);
            if (tm < thr) lo = mid + 1; else hi = mid;
          }
        } else {  // uniform arrivals (reading Q9): closed-form guess, then exact local correction, so the
                  // result is the same first index the search finds (t non-decreasing in s)
          const double est = ceil((double)thr * rate * 1e-9) - (double)(p.goff + s0);
          lo = est <= 0.0 ? 0 : (est >= (double)b ? b : (int)est);
          while (lo > 0 && arrival_uniform(p.goff + s0 + lo - 1, rate, inv) >= thr) --lo;
          while (lo < b && arrival_uniform(p.goff + s0 + lo, rate, inv) < thr) ++lo;
        }
        cnt[m] = lo;
        if (p.ovd) p.ovd[p.ovd_off[bi] + (jl * p.K + m) * p.ovd_nrp + r] = (uint16_t)lo;
      }
      if (p.want_exceed) {
        // E = sum_{i < cnt} (tl - t_i + c - tau): one sweep with prefix sums of t_i
        int maxc = 0;
        for (int m = 0; m < p.K; ++m) maxc = cnt[m] > maxc ? cnt[m] : maxc;
        int ord[kMaxK];  // models in increasing overdue count (insertion sort; K <= 12)
        for (int m = 0; m < p.K; ++m) {
          int k = m;
          while (k > 0 && cnt[ord[k - 1]] > cnt[m]) { ord[k] = ord[k - 1]; --k; }
          ord[k] = m;
        }
        int64_t pre = 0;
        int k = 0;
        for (int i = 0; i <= maxc; ++i) {
          for (; k < p.K && cnt[ord[k]] == i; ++k) {
            const int m = ord[k];
            ex[m] = (unsigned long long)((int64_t)i * (fm[m] - p.tau) - pre);
          }
          if (i < maxc) pre += p.arrival ? p.arrival[s0 + i] : arrival_uniform(p.goff + s0 + i, rate, inv);
        }
      }
    }
    const int key = act ? r * p.nB + bi : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (grp == 0xffffffffu) {  // the whole warp on one (r, b): warp sums, one atomic per model
#pragma unroll
      for (int m = 0; m < kMaxK; ++m) {
        if (m >= p.K) break;
        const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)cnt[m]);
        unsigned long long e = ex[m];
        if (p.want_exceed)
          for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
        if (lane == 0) {
          atomicAdd(&so[key * p.K + m], (unsigned long long)c);
          if (p.want_exceed) atomicAdd(&se[key * p.K + m], e);
        }
      }
    } else if (act) {
      for (int m = 0; m < p.K; ++m) {
        atomicAdd(&so[key * p.K + m], (unsigned long long)cnt[m]);
        if (p.want_exceed) atomicAdd(&se[key * p.K + m], ex[m]);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nT; i += blockDim.x) {
    if (so[i]) atomicAdd(p.osum + i, so[i]);
    if (p.want_exceed && se[i]) atomicAdd(p.esum + i, se[i]);
  }
}

// ---- queue mode (reading Q15): FIFO finish times by a prefix-max scan --------------------------
// finish_j = max(t_last(j), finish_{j-1}) + c unrolls to finish_j = (j+1) c + max_{i<=j} (t_last(i) - i c)
// (global batch indices). One CTA per (b, r, m); tiles of QS batches, block-wide inclusive max-scan.
constexpr int QS = 256;
constexpr int64_t kNegInf = INT64_MIN / 4;
__device__ __forceinline__ int64_t block_max_i64(int64_t x, int64_t* sm) {
  for (int off = 16; off; off >>= 1) x = max(x, (int64_t)__shfl_xor_sync(0xffffffffu, x, off));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = x;
  __syncthreads();
  int64_t r = kNegInf;
  for (int i = 0; i < QS / 32; ++i) r = max(r, sm[i]);
  return r;
}
__global__ void __launch_bounds__(QS) queue_scan_kernel(const MomentParams p, int64_t* fin, int64_t* carry,
                                                        int seed_rates) {
  __shared__ int64_t sm[QS / 32];
  __shared__ int64_t wsum[QS / 32];
  const int tri = blockIdx.x;  // (bi, r, m)
  const int m = tri % p.K, r = (tri / p.K) % p.nR, bi = tri / (p.K * p.nR);
  const int64_t b = p.B[bi], c = p.lat[m * p.nB + bi];
  const int64_t nb = p.N / b, J0 = p.goff / b;
  const double rate = p.rates[r];
  int64_t* cy = carry + ((int64_t)bi * p.nR + r) * p.K + m;
  int64_t M = *cy;
  if (seed_rates) {  // backlog from the global batches before this rank's first chunk (rates only)
    int64_t x = kNegInf;
    for (int64_t i = threadIdx.x; i < J0; i += QS) x = max(x, arrival_at(nullptr, 0, (i + 1) * b - 1, rate) - i * c);
    M = max(M, block_max_i64(x, sm));
  }
  int64_t* out = fin + p.fin_off[bi] + ((int64_t)r * p.K + m) * nb;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int64_t t0 = 0; t0 < nb; t0 += QS) {
    const int64_t jl = t0 + threadIdx.x;
    int64_t u = kNegInf;
    if (jl < nb) {
      const int64_t s = (jl + 1) * b - 1;
      u = arrival_at(p.arrival, s, p.goff + s, rate) - (J0 + jl) * c;
    }
    for (int off = 1; off < 32; off <<= 1) {  // warp inclusive max-scan
      const int64_t o = __shfl_up_sync(0xffffffffu, u, off);
      if (l >= off) u = max(u, o);
    }
    __syncthreads();
    if (l == 31) wsum[w] = u;
    __syncthreads();
    int64_t pre = M;
    for (int i = 0; i < w; ++i) pre = max(pre, wsum[i]);
    const int64_t incl = max(pre, u);
    if (jl < nb) out[jl] = (J0 + jl + 1) * c + incl;
    int64_t tile = M;
    for (int i = 0; i < QS / 32; ++i) tile = max(tile, wsum[i]);
    M = tile;
  }
  if (threadIdx.x == 0) *cy = M;
}

// ---- chunk counters -> table ------------------------------------------------------------------
__global__ void merge_kernel(const MergeParams p, int64_t N, int64_t off_N) {
  const int S = p.S;
  const unsigned long long* vote = p.chunk;
  const unsigned long long* avg = p.chunk + S;
  const unsigned long long* rc = p.chunk + 2 * S;
  const unsigned long long* tail = p.chunk + 3 * S;
  const unsigned long long* osum = tail + (size_t)p.nB * S;
  const unsigned long long* esum = osum + (size_t)p.nR * p.nB * p.K;
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    if (threadIdx.x == 0) p.table[off_N] += (unsigned long long)N;
    p.table[p.off_err + threadIdx.x] += p.err[threadIdx.x] ? 1ull : 0ull;
  }
  for (int v1 = blockIdx.x * blockDim.x + threadIdx.x; v1 < S; v1 += gridDim.x * blockDim.x) {
    p.table[p.off_vote + v1] += vote[v1];
    p.table[p.off_avg + v1] += avg[v1];
    p.table[p.off_rc + v1] += rc[v1];
    for (int bi = 0; bi < p.nB; ++bi) {
      p.table[p.off_corr + (size_t)bi * S + v1] += vote[v1] - tail[(size_t)bi * S + v1];
      const int m = p.slow[(size_t)bi * S + v1];
      for (int r = 0; r < p.nR; ++r) {
        const size_t idx = ((size_t)r * p.nB + bi) * S + v1;
        p.table[p.off_O + idx] += osum[((size_t)r * p.nB + bi) * p.K + m];
        if (p.want_exceed) p.table[p.off_E + idx] += esum[((size_t)r * p.nB + bi) * p.K + m];
      }
    }
  }
}

// ---- labelled moments Q[r][b][v] = sum_j corr_j(v) * o_j(v,b,r) --------------------------------
// o_j(v,b,r) = overdue count of batch j of size b at rate r when v's slowest member is m (written
// per batch by overdue_kernel into `ovd`, layout [j][m][r] with r padded to NRP so one vector load
// fetches every rate). Grid = (slice of QT subsets) x (range of L-chunks); a thread owns one subset,
// reads each group count of its subset once (coalesced across the warp: grp is [group][S]), keeps
// a running correct-count per batch size and, at each batch end, multiply-adds it into u32 register
// accumulators [NRP][b], spilled to u64 shared accumulators every `flush` chunks (no u32 overflow:
// a chunk adds at most L * max(B)); one atomic per (v, r, b) per block.
constexpr int QT = 128;
#ifndef RK_QG
#define RK_QG 8
#endif
constexpr int QG = RK_QG;  // group counts loaded ahead per thread
constexpr int kQStageBytes = 32 * 1024;
constexpr int kQBlocksPerSM = 6;  // STAGED: the chunk's o values staged in shared memory
template <int NRP>
struct OVec;
template <>
struct OVec<4> { using T = uint2; };
template <>
struct OVec<8> { using T = uint4; };

// Host-computed per-batch-size constants (kernel parameter space: constant-bank operands, no registers).
struct QConst {
  int bg[kMaxB];      // groups per batch
  int nbc[kMaxB];     // batches per chunk (L / B)
  int soff[kMaxB];    // first staged batch of each size
  int64_t nbat[kMaxB];  // complete batches in this accumulate call (reading Q13)
  uint32_t packed;      // q_nested: bit bi set when L * B[bi] < 2^16 (two rates per 32-bit multiply-add)
};

// NB = nB exactly (1..8; 0 = generic loop bound p.nB for the unstaged fallback).
template <int NRP, int NB, bool STAGED>
__global__ void __launch_bounds__(QT, kQBlocksPerSM)
    q_kernel(const QParams p, const QConst qc, int64_t chunks_per_block, int tot, int flush) {
  constexpr int NBX = NB > 0 ? NB : kMaxB;
  extern __shared__ unsigned long long qacc[];  // [nR * nB][QT], then (STAGED) u16 [tot][K][NRP]
  uint16_t* so = reinterpret_cast<uint16_t*>(qacc + (size_t)p.nR * p.nB * QT);
  using V = typename OVec<NRP>::T;
  const int nB = NB > 0 ? NB : p.nB;
  const int v1 = blockIdx.x * QT + threadIdx.x;
  const bool own = v1 < p.S;
  const int KR = p.K * NRP;  // u16 per batch
  for (int i = 0; i < p.nR * nB; ++i) qacc[i * QT + threadIdx.x] = 0;
  const int64_t gpc = p.L / p.gs;  // groups per chunk
  const int64_t ngroups = (p.N + p.gs - 1) / p.gs;
  const int64_t nch = (p.N + p.L - 1) / p.L;
  const int64_t q0 = blockIdx.y * chunks_per_block;
  const int64_t q1 = min(nch, q0 + chunks_per_block);
  // slowest member of v per batch size, 4 bits each
  uint32_t mpack = 0;
  for (int bi = 0; bi < nB; ++bi) mpack |= (uint32_t)(own ? p.slow[(size_t)bi * p.S + v1] : 0) << (4 * bi);
  unsigned int acc[NRP][NBX];
#pragma unroll
  for (int bi = 0; bi < NBX; ++bi)
#pragma unroll
    for (int r = 0; r < NRP; ++r) acc[r][bi] = 0;
  const uint8_t* gp = p.grp + (own ? v1 : 0);
  int since = 0;
  unsigned long long csum = 0;  // sum of the subset's group counts (p.cnt_vote)
  for (int64_t q = q0; q < q1; ++q) {
    if (STAGED) {
      __syncthreads();
#pragma unroll
      for (int bi = 0; bi < NBX; ++bi) {
        if (bi >= nB) break;
        const int64_t jbase = q * qc.nbc[bi];
        const int nvalid = (int)max((int64_t)0, min((int64_t)qc.nbc[bi], qc.nbat[bi] - jbase)) * p.K;
        const V* src = reinterpret_cast<const V*>(p.ovd + p.ovd_off[bi] + jbase * KR);
        V* dst = reinterpret_cast<V*>(so + qc.soff[bi] * KR);
        for (int w = threadIdx.x; w < qc.nbc[bi] * p.K; w += QT) {
          V z{};
          dst[w] = w < nvalid ? src[w] : z;  // incomplete batches contribute 0
        }
      }
      __syncthreads();
    }
    if (!own) continue;
    // per size: (batch index in chunk) << 16 | groups left in the current batch
    int lj[NBX];
    unsigned int part[NBX];
#pragma unroll
    for (int bi = 0; bi < NBX; ++bi) { lj[bi] = qc.bg[bi]; part[bi] = 0; }
    const int64_t ga = q * gpc, gb = min(ngroups, ga + gpc);
    for (int64_t g0 = ga; g0 < gb; g0 += QG) {
      unsigned int cc[QG];  // QG independent loads in flight before the dependent batch bookkeeping
#pragma unroll
      for (int i = 0; i < QG; ++i) cc[i] = g0 + i < gb ? gp[(g0 + i) * p.S] : 0u;
#pragma unroll
      for (int i = 0; i < QG; ++i) {
        if (g0 + i >= gb) break;
        const unsigned int c = cc[i];
        csum += c;
#pragma unroll
        for (int bi = 0; bi < NBX; ++bi) {
          if (NB == 0 && bi >= nB) break;
          part[bi] += c;
          if (((--lj[bi]) & 0xFFFF) == 0) {  // end of batch (lj >> 16) of size B[bi] in this chunk
            const int jj = lj[bi] >> 16;
            const int m = (mpack >> (4 * bi)) & 15;
            if (part[bi] && (STAGED || q * qc.nbc[bi] + jj < qc.nbat[bi])) {
              const uint16_t* ob = STAGED ? so + (qc.soff[bi] + jj) * KR
                                          : p.ovd + p.ovd_off[bi] + (q * qc.nbc[bi] + jj) * KR;
              union { V v; uint16_t h[NRP]; } o;
              o.v = *reinterpret_cast<const V*>(ob + m * NRP);
#pragma unroll
              for (int r = 0; r < NRP; ++r) acc[r][bi] += part[bi] * o.h[r];
            }
            part[bi] = 0;
            lj[bi] += (1 << 16) + qc.bg[bi];
          }
        }
      }
    }
    if (++since == flush || q + 1 == q1) {  // spill the u32 accumulators
      since = 0;
#pragma unroll
      for (int bi = 0; bi < NBX; ++bi) {
        if (bi >= nB) break;
#pragma unroll
        for (int r = 0; r < NRP; ++r) {
          if (r < p.nR) qacc[(r * nB + bi) * QT + threadIdx.x] += acc[r][bi];
          acc[r][bi] = 0;
        }
      }
    }
  }
  if (!own) return;
  if (p.cnt_vote && csum) atomicAdd(p.cnt_vote + v1, csum);
  for (int r = 0; r < p.nR; ++r)
    for (int bi = 0; bi < nB; ++bi) {
      const unsigned long long x = qacc[(r * nB + bi) * QT + threadIdx.x];
      if (x) atomicAdd(p.Q + ((size_t)r * nB + bi) * p.S + v1, x);
    }
}

// ---- A7: reward fold -----------------------------------------------------------------------
__global__ void fold_kernel(const FoldParams p) {
  const unsigned long long Ntot = p.table[p.off_N];
  const int total = p.nR * p.nB * p.S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int v1 = i % p.S;
    const int bi = (i / p.S) % p.nB;
    const double b = (double)p.B[bi];
    const double nb = (double)(Ntot / (unsigned long long)p.B[bi]);
    const double a = Ntot > 0 ? __ddiv_rn((double)p.table[p.off_vote + v1], (double)Ntot) : 0.0;
    const double O = (double)p.table[p.off_O + i];
    // a * (nb*b - beta*O), rounded step by step like the definition (no FMA contraction)
    p.reward_sur[i] = __dmul_rn(a, __dsub_rn(__dmul_rn(nb, b), __dmul_rn(p.beta, O)));
    const double corr = (double)p.table[p.off_corr + (size_t)bi * p.S + v1];
    const double Q = p.has_Q ? (double)p.table[p.off_Q + i] : 0.0;
    p.reward_lab[i] = __dsub_rn(corr, __dmul_rn(__ddiv_rn(p.beta, b), Q));
  }
}

}  // namespace

cudaError_t launch_overdue(const MomentParams& p, cudaStream_t st) {
  if (p.nB == 0 || p.nR == 0 || p.N <= 0) return cudaSuccess;
  int64_t work = 0;
  for (int bi = 0; bi < p.nB; ++bi) work += (p.N / p.B[bi]) * p.nR;
  if (work == 0) return cudaSuccess;
  int64_t blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  // err flags live right after the sums (see rk_api.cpp chunk layout)
  overdue_kernel<<<(int)blocks, 256, 0, st>>>(p, reinterpret_cast<unsigned int*>(p.esum + (size_t)p.nR * p.nB * p.K));
  return cudaGetLastError();
}

int64_t fin_elems(int nB, const int* B, int nR, int K, int64_t N, int64_t* off) {
  int64_t tot = 0;
  for (int bi = 0; bi < nB; ++bi) {
    if (off) off[bi] = tot;
    tot += (N / B[bi]) * nR * K;
  }
  return tot;
}

cudaError_t launch_queue_scan(const MomentParams& p, int64_t* fin, int64_t* carry, int seed_rates, cudaStream_t st) {
  if (p.nB == 0 || p.nR == 0) return cudaSuccess;
  queue_scan_kernel<<<p.nB * p.nR * p.K, QS, 0, st>>>(p, fin, carry, seed_rates);
  return cudaGetLastError();
}

cudaError_t launch_merge(const MergeParams& p, int64_t N, int64_t off_N, cudaStream_t st) {
  merge_kernel<<<(p.S + 255) / 256, 256, 0, st>>>(p, N, off_N);
  return cudaGetLastError();
}

int ovd_nrp(int nR) { return nR <= 4 ? 4 : 8; }

int64_t ovd_elems(int nB, const int* B, int nR, int K, int64_t N, int64_t* off) {
  int64_t tot = 0;
  for (int bi = 0; bi < nB; ++bi) {
    if (off) off[bi] = tot;
    tot += (N / B[bi]) * K * ovd_nrp(nR);
  }
  return tot;
}

// Fast path for doubling batch sizes B = {gs, 2gs, ..., 2^(NB-1) gs} (the configs' {16, ..., 256}): a
// chunk (L = B[NB-1] samples) holds G0 = 2^(NB-1) groups, so a thread loads its subset's G0 group counts
// into registers once and forms every batch size's correct counts as a pairwise-sum tree, each batch
// end costing one 128-bit shared load of the staged overdue counts (u32 per rate) and NRP multiply-adds.
// QC chunks are staged per round; the overdue counts of round i+1 are copied to shared memory with
// cp.async (8-byte pieces, u16 as stored) while round i is computed, so the staging latency is hidden.
constexpr int QC = 4;
constexpr int kQNestedBlocksPerSM = 4;
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// stage chunks qq .. qq+QC-1: level bi's region is [QC][nb][K][NRP] u16, contiguous in ovd for
// consecutive chunks; entries past the last complete batch (reading Q13) or past q1 are zero-filled
template <int NRP, int NB>
__device__ __forceinline__ void q_stage(const QParams& p, const QConst& qc, uint16_t* buf, int64_t qq, int64_t q1) {
  constexpr int G0 = 1 << (NB - 1);
  const int K = p.K;
  int soff = 0;  // u16 offset of level bi in the buffer
#pragma unroll
  for (int bi = 0; bi < NB; ++bi) {
    const int nb = G0 >> bi;
    const int64_t per = (int64_t)nb * K * NRP;              // u16 per chunk and level
    const int64_t lim = min(qc.nbat[bi] * (int64_t)K * NRP,  // valid u16 of this level (complete batches,
                            q1 * per);                       // chunks < q1)
    const int64_t g0 = qq * per;
    const int n8 = (int)(QC * per / 4);                      // 8-byte pieces (4 u16)
    const uint16_t* src = p.ovd + p.ovd_off[bi];
    for (int k = threadIdx.x; k < n8; k += QT) {
      const int64_t g = g0 + 4 * (int64_t)k;
      uint16_t* d = buf + soff + 4 * k;
      if (g + 4 <= lim) cp_async8(d, src + g);
      else *reinterpret_cast<uint2*>(d) = make_uint2(0u, 0u);  // (per and lim are multiples of 4)
    }
    soff += (int)(QC * per);
  }
}

template <int NRP, int NB>
__global__ void __launch_bounds__(QT, kQNestedBlocksPerSM)
    q_nested_kernel(const QParams p, const QConst qc, int64_t chunks_per_block, int flush) {
  constexpr int G0 = 1 << (NB - 1);   // groups (= smallest batches) per chunk
  constexpr int TOT = 2 * G0 - 1;     // batches of every size per chunk
  extern __shared__ unsigned long long qacc[];  // [nR * NB][QT], then u16 [2][QC * TOT * K * NRP]
  const int K = p.K;
  const int BUF = QC * TOT * K * NRP;  // u16 per staging buffer
  uint16_t* sbuf = reinterpret_cast<uint16_t*>(qacc + (size_t)p.nR * NB * QT);
  const int v1 = blockIdx.x * QT + threadIdx.x;
  const bool own = v1 < p.S;
  for (int i = 0; i < p.nR * NB; ++i) qacc[i * QT + threadIdx.x] = 0;
  const int64_t ngroups = (p.N + p.gs - 1) / p.gs;
  const int64_t nch = (p.N + p.L - 1) / p.L;
  const int64_t q0 = blockIdx.y * chunks_per_block;
  const int64_t q1 = min(nch, q0 + chunks_per_block);
  int mo[NB];  // slowest member of v per batch size -> offset of its rates in a staged batch
#pragma unroll
  for (int bi = 0; bi < NB; ++bi) mo[bi] = (own ? p.slow[(size_t)bi * p.S + v1] : 0) * NRP;
  unsigned int acc[NRP][NB];
#pragma unroll
  for (int bi = 0; bi < NB; ++bi)
#pragma unroll
    for (int r = 0; r < NRP; ++r) acc[r][bi] = 0;
  const uint8_t* gp = p.grp + (own ? v1 : 0);
  int since = 0;
  unsigned long long csum = 0;  // sum of the subset's group counts (p.cnt_vote)
  if (q0 < q1) q_stage<NRP, NB>(p, qc, sbuf, q0, q1);
  cp_async_commit();
  int cur = 0;
  for (int64_t qq = q0; qq < q1; qq += QC, cur ^= 1) {
    if (qq + QC < q1) q_stage<NRP, NB>(p, qc, sbuf + (cur ^ 1) * BUF, qq + QC, q1);
    cp_async_commit();
    cp_async_wait1();  // this round's copies have landed (the next round's stay in flight)
    __syncthreads();
    if (own) {
      const uint16_t* sb = sbuf + cur * BUF;
      unsigned int nx[G0];  // group counts of the next chunk, loaded one chunk ahead
#pragma unroll
      for (int i = 0; i < G0; ++i) {
        const int64_t g = qq * G0 + i;
        nx[i] = g < ngroups ? gp[g * p.S] : 0u;
      }
#pragma unroll 1
      for (int c = 0; c < QC; ++c) {
        const int64_t q = qq + c;
        if (q >= q1) break;
        unsigned int sv[G0];
#pragma unroll
        for (int i = 0; i < G0; ++i) {
          sv[i] = nx[i];
          const int64_t g = (q + 1) * G0 + i;
          nx[i] = (c + 1 < QC && g < ngroups) ? gp[g * p.S] : 0u;
        }
        int soff = 0;
#pragma unroll
        for (int bi = 0; bi < NB; ++bi) {
          const int nb = G0 >> bi;
          const uint16_t* lv = sb + soff + ((size_t)c * nb) * K * NRP + mo[bi];
          if (NRP == 4 && (qc.packed >> bi) & 1) {
            // two rates per 32-bit multiply-add: the staged (o_r0 | o_r1 << 16) times the batch's correct
            // count adds sv*o_r0 to the low half and sv*o_r1 to the high half; over the level's batches of
            // one chunk the low half sums to at most L * B[bi] < 2^16 (qc.packed), so it never carries
            uint32_t p01 = 0, p23 = 0;
#pragma unroll
            for (int j = 0; j < nb; ++j) {
              const uint2 o = *reinterpret_cast<const uint2*>(lv + (size_t)j * K * NRP);
              p01 += sv[j] * o.x;
              p23 += sv[j] * o.y;
            }
            acc[0][bi] += p01 & 0xffffu; acc[1][bi] += p01 >> 16;
            acc[2][bi] += p23 & 0xffffu; acc[3][bi] += p23 >> 16;
          } else
#pragma unroll
          for (int j = 0; j < nb; ++j) {
            if (NRP == 4) {
              const uint2 o = *reinterpret_cast<const uint2*>(lv + (size_t)j * K * NRP);
              acc[0][bi] += sv[j] * (o.x & 0xffffu); acc[1][bi] += sv[j] * (o.x >> 16);
              acc[2][bi] += sv[j] * (o.y & 0xffffu); acc[3][bi] += sv[j] * (o.y >> 16);
            } else {
#pragma unroll
              for (int r = 0; r < NRP; ++r) acc[r][bi] += sv[j] * (unsigned int)lv[(size_t)j * K * NRP + r];
            }
          }
          soff += QC * nb * K * NRP;
#pragma unroll
          for (int j = 0; j < nb / 2; ++j) sv[j] = sv[2 * j] + sv[2 * j + 1];  // next batch size
        }
        csum += sv[0];  // the last level is the whole chunk
        if (++since == flush || q + 1 == q1) {  // spill the u32 accumulators
          since = 0;
#pragma unroll
          for (int bi = 0; bi < NB; ++bi)
#pragma unroll
            for (int r = 0; r < NRP; ++r) {
              if (r < p.nR) qacc[(r * NB + bi) * QT + threadIdx.x] += acc[r][bi];
              acc[r][bi] = 0;
            }
        }
      }
    }
    __syncthreads();  // every thread is done with this buffer before the next round's copies land in it
  }
  if (!own) return;
  if (p.cnt_vote && csum) atomicAdd(p.cnt_vote + v1, csum);
  for (int r = 0; r < p.nR; ++r)
    for (int bi = 0; bi < NB; ++bi) {
      const unsigned long long x = qacc[(r * NB + bi) * QT + threadIdx.x];
      if (x) atomicAdd(p.Q + ((size_t)r * NB + bi) * p.S + v1, x);
    }
}

template <int NRP, int NB, bool STAGED>
static cudaError_t launch_q_t(const QParams& p, const QConst& qc, dim3 grid, size_t smem, int64_t cpb, int tot,
                              int flush, cudaStream_t st) {
  cudaError_t e =
      cudaFuncSetAttribute(q_kernel<NRP, NB, STAGED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  q_kernel<NRP, NB, STAGED><<<grid, QT, smem, st>>>(p, qc, cpb, tot, flush);
  return cudaGetLastError();
}
template <int NRP>
static cudaError_t launch_q_nb(const QParams& p, const QConst& qc, bool staged, dim3 grid, size_t smem, int64_t cpb,
                               int tot, int flush, cudaStream_t st) {
  if (!staged) return launch_q_t<NRP, 0, false>(p, qc, grid, smem, cpb, tot, flush, st);
  switch (p.nB) {
    case 1: return launch_q_t<NRP, 1, true>(p, qc, grid, smem, cpb, tot, flush, st);
    case 2: return launch_q_t<NRP, 2, true>(p, qc, grid, smem, cpb, tot, flush, st);
    case 3: return launch_q_t<NRP, 3, true>(p, qc, grid, smem, cpb, tot, flush, st);
    case 4: return launch_q_t<NRP, 4, true>(p, qc, grid, smem, cpb, tot, flush, st);
    case 5: return launch_q_t<NRP, 5, true>(p, qc, grid, smem, cpb, tot, flush, st);
    case 6: return launch_q_t<NRP, 6, true>(p, qc, grid, smem, cpb, tot, flush, st);
    case 7: return launch_q_t<NRP, 7, true>(p, qc, grid, smem, cpb, tot, flush, st);
    default: return launch_q_t<NRP, 8, true>(p, qc, grid, smem, cpb, tot, flush, st);
  }
}

cudaError_t launch_q(const QParams& p, int sm_count, cudaStream_t st) {
  if (p.nB == 0 || p.nR == 0 || p.N <= 0) return cudaSuccess;
  const int64_t nch = (p.N + p.L - 1) / p.L;
  const int slices = (p.S + QT - 1) / QT;
  QConst qc{};
  int tot = 0, bmax = 1;
  for (int bi = 0; bi < p.nB; ++bi) {
    qc.bg[bi] = p.B[bi] / p.gs;
    qc.nbc[bi] = (int)(p.L / p.B[bi]);
    qc.soff[bi] = tot;
    qc.nbat[bi] = p.N / p.B[bi];
    if ((int64_t)p.L * p.B[bi] < 65536 && !getenv("RK_Q_UNPACKED")) qc.packed |= 1u << bi;
    tot += qc.nbc[bi];
    bmax = p.B[bi] > bmax ? p.B[bi] : bmax;
  }
  const int nrp = ovd_nrp(p.nR);
  const size_t acc = sizeof(unsigned long long) * (size_t)p.nR * p.nB * QT;
  const size_t stage = sizeof(uint16_t) * (size_t)tot * p.K * nrp;
  const bool staged = stage <= (size_t)kQStageBytes;
  // one wave: resident blocks per SM limited by the launch bound and shared memory
  const size_t smem = acc + (staged ? stage : 0);
  int per_sm = (int)((200 * 1024) / (smem + 1024));
  per_sm = per_sm < 1 ? 1 : (per_sm > kQBlocksPerSM ? kQBlocksPerSM : per_sm);
  int64_t ranges = ((int64_t)sm_count * per_sm) / slices;
  if (ranges < 1) ranges = 1;
  if (ranges > nch) ranges = nch;
  if (ranges > 65535) ranges = 65535;
  const int64_t cpb = (nch + ranges - 1) / ranges;
  ranges = (nch + cpb - 1) / cpb;
  // u32 register accumulators: one chunk adds at most L * max(B) <= 2^24 per (r, b)
  const unsigned long long fl = 0xFFFFFFFFull / ((unsigned long long)p.L * bmax);
  const int flush = (int)(fl < 1024 ? fl : 1024);
  const dim3 grid((unsigned)slices, (unsigned)ranges);
  // doubling batch sizes starting at the group size, at most 16 groups per chunk: the tree kernel
  bool nested = p.B[0] == p.gs && p.nB <= 5 && p.L == p.B[p.nB - 1];
  for (int bi = 1; bi < p.nB; ++bi) nested = nested && p.B[bi] == 2 * p.B[bi - 1];
  if (nested && !getenv("RK_Q_GENERIC")) {  // env: tests compare against the generic kernel
    const int G0 = 1 << (p.nB - 1);
    const size_t nsmem = acc + 2 * sizeof(uint16_t) * (size_t)QC * (2 * G0 - 1) * p.K * nrp;
    int nper = (int)((200 * 1024) / (nsmem + 1024));
    nper = nper < 1 ? 1 : (nper > kQNestedBlocksPerSM ? kQNestedBlocksPerSM : nper);
    int64_t nr_ = ((int64_t)sm_count * nper) / slices;
    nr_ = nr_ < 1 ? 1 : (nr_ > nch ? nch : (nr_ > 65535 ? 65535 : nr_));
    int64_t ncpb = (nch + nr_ - 1) / nr_;
    ncpb = (ncpb + QC - 1) / QC * QC;  // whole staging rounds per block
    nr_ = (nch + ncpb - 1) / ncpb;
    const dim3 ngrid((unsigned)slices, (unsigned)nr_);
    switch (p.nB * 16 + nrp) {
#define RK_QN(NBV, NRV)                                                                                      \
  case NBV * 16 + NRV: {                                                                                    \
    cudaError_t e = cudaFuncSetAttribute(q_nested_kernel<NRV, NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)nsmem);                                                       \
    if (e != cudaSuccess) return e;                                                                         \
    q_nested_kernel<NRV, NBV><<<ngrid, QT, nsmem, st>>>(p, qc, ncpb, flush);                                \
    return cudaGetLastError();                                                                              \
  }
      RK_QN(1, 4) RK_QN(2, 4) RK_QN(3, 4) RK_QN(4, 4) RK_QN(5, 4)
      RK_QN(1, 8) RK_QN(2, 8) RK_QN(3, 8) RK_QN(4, 8) RK_QN(5, 8)
#undef RK_QN
      default: break;
    }
  }
  return nrp == 4 ? launch_q_nb<4>(p, qc, staged, grid, smem, cpb, tot, flush, st)
                  : launch_q_nb<8>(p, qc, staged, grid, smem, cpb, tot, flush, st);
}

cudaError_t launch_fold(const FoldParams& p, cudaStream_t st) {
  const int total = p.nR * p.nB * p.S;
  if (total == 0) return cudaSuccess;
  fold_kernel<<<(total + 255) / 256, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rk
