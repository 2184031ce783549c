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

#include "rk_internal.h"

namespace rk {
namespace {

__device__ __forceinline__ int64_t arrival_at(const int64_t* arr, int64_t local, int64_t global, double rate) {
  if (arr) return arr[local];
  const double num = __dmul_rn((double)global, 1e9);
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
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < tot; w += (int64_t)gridDim.x * blockDim.x) {
    int bi = 0;
    while (bi + 1 < p.nB && w >= start[bi + 1]) ++bi;
    const int64_t rem = w - start[bi];
    const int64_t nb = p.N / p.B[bi];
    const int r = (int)(rem / nb);
    const int64_t jl = rem - (int64_t)r * nb;
    const int b = p.B[bi];
    const int64_t s0 = jl * b;  // local index of the batch's first request
    const double rate = p.rates[r];
    const int64_t tl = arrival_at(p.arrival, s0 + b - 1, p.goff + s0 + b - 1, rate);
    if (p.arrival && r == 0) {  // arrivals must be non-decreasing inside a batch (FIFO)
      for (int i = 1; i < b; ++i)
        if (p.arrival[s0 + i] < p.arrival[s0 + i - 1]) { atomicOr(err + 2, 1u); break; }
    }
    int cnt[kMaxK];
    for (int m = 0; m < p.K; ++m) {
      // overdue <=> (tl - t_s) + c > tau <=> t_s < tl + c - tau ; t_s non-decreasing in s
      const int64_t thr = tl + p.lat[m * p.nB + bi] - p.tau;
      int lo = 0, hi = b;  // first i with t_i >= thr
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int64_t tm = arrival_at(p.arrival, s0 + mid, p.goff + s0 + mid, rate);
        if (tm < thr) lo = mid + 1; else hi = mid;
      }
      cnt[m] = lo;
      atomicAdd(&so[(r * p.nB + bi) * p.K + m], (unsigned long long)lo);
    }
    if (p.want_exceed) {
      // E = sum_{i < cnt} (tl - t_i + c - tau): one sweep with prefix sums of t_i
      int maxc = 0;
      for (int m = 0; m < p.K; ++m) maxc = cnt[m] > maxc ? cnt[m] : maxc;
      int64_t pre = 0;
      for (int i = 0; i <= maxc; ++i) {
        for (int m = 0; m < p.K; ++m)
          if (cnt[m] == i) {
            const int64_t c = p.lat[m * p.nB + bi];
            const unsigned long long e = (unsigned long long)((int64_t)i * (tl + c - p.tau) - pre);
            atomicAdd(&se[(r * p.nB + bi) * p.K + m], e);
          }
        if (i < maxc) pre += arrival_at(p.arrival, s0 + i, p.goff + s0 + i, rate);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nT; i += blockDim.x) {
    if (so[i]) atomicAdd(p.osum + i, so[i]);
    if (p.want_exceed && se[i]) atomicAdd(p.esum + i, se[i]);
  }
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
// One CTA per L-chunk (L = lcm(B) samples, L/gs groups). o_j per (b, r, batch, slowest model) is
// computed into shared memory, then each thread owns subsets v and sums group counts per batch.
__global__ void q_kernel(const QParams p) {
  extern __shared__ unsigned short so_q[];  // [sum_b L/b][nR][K]
  const int64_t nch = (p.N + p.L - 1) / p.L;
  int off[kMaxB];
  int tot = 0;
  for (int bi = 0; bi < p.nB; ++bi) { off[bi] = tot; tot += (int)(p.L / p.B[bi]); }
  for (int64_t q = blockIdx.x; q < nch; q += gridDim.x) {
    __syncthreads();
    // phase 1: overdue counts of every complete batch in this chunk
    for (int w = threadIdx.x; w < tot * p.nR * p.K; w += blockDim.x) {
      const int m = w % p.K;
      const int r = (w / p.K) % p.nR;
      const int jj = w / (p.K * p.nR);
      int bi = 0;
      while (bi + 1 < p.nB && jj >= off[bi + 1]) ++bi;
      const int b = p.B[bi];
      const int64_t s0 = q * p.L + (int64_t)(jj - off[bi]) * b;
      unsigned short o = 0;
      if (s0 + b <= (p.N / b) * b) {
        const double rate = p.rates[r];
        const int64_t tl = arrival_at(p.arrival, s0 + b - 1, p.goff + s0 + b - 1, rate);
        const int64_t thr = tl + p.lat[m * p.nB + bi] - p.tau;
        int lo = 0, hi = b;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (arrival_at(p.arrival, s0 + mid, p.goff + s0 + mid, rate) < thr) lo = mid + 1; else hi = mid;
        }
        o = (unsigned short)lo;
      }
      so_q[w] = o;
    }
    __syncthreads();
    // phase 2: per subset
    const int64_t g0 = q * p.L / p.gs;
    const int64_t ngroups = (p.N + p.gs - 1) / p.gs;
    for (int v1 = threadIdx.x; v1 < p.S; v1 += blockDim.x) {
      unsigned long long acc[kMaxR * kMaxB];
      for (int i = 0; i < p.nR * p.nB; ++i) acc[i] = 0;
      for (int bi = 0; bi < p.nB; ++bi) {
        const int b = p.B[bi];
        const int m = p.slow[(size_t)bi * p.S + v1];
        const int nbat = (int)(p.L / b);
        for (int jj = 0; jj < nbat; ++jj) {
          const int64_t s0 = q * p.L + (int64_t)jj * b;
          if (s0 + b > (p.N / b) * b) break;
          unsigned int corr = 0;
          const int64_t gg = g0 + (int64_t)jj * (b / p.gs);
          for (int k = 0; k < b / p.gs; ++k)
            if (gg + k < ngroups) corr += p.grp[(gg + k) * p.S + v1];
          if (!corr) continue;
          for (int r = 0; r < p.nR; ++r)
            acc[r * p.nB + bi] += (unsigned long long)corr * so_q[((off[bi] + jj) * p.nR + r) * p.K + m];
        }
      }
      for (int r = 0; r < p.nR; ++r)
        for (int bi = 0; bi < p.nB; ++bi)
          if (acc[r * p.nB + bi]) atomicAdd(p.Q + ((size_t)r * p.nB + bi) * p.S + v1, acc[r * p.nB + bi]);
    }
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

cudaError_t launch_merge(const MergeParams& p, int64_t N, int64_t off_N, cudaStream_t st) {
  merge_kernel<<<(p.S + 255) / 256, 256, 0, st>>>(p, N, off_N);
  return cudaGetLastError();
}

cudaError_t launch_q(const QParams& p, cudaStream_t st) {
  if (p.nB == 0 || p.nR == 0 || p.N <= 0) return cudaSuccess;
  int tot = 0;
  for (int bi = 0; bi < p.nB; ++bi) tot += (int)(p.L / p.B[bi]);
  const size_t smem = sizeof(unsigned short) * (size_t)tot * p.nR * p.K;
  if (smem > 48 * 1024) return cudaErrorInvalidValue;
  int64_t nch = (p.N + p.L - 1) / p.L;
  int blocks = (int)(nch < 148 * 8 ? nch : 148 * 8);
  q_kernel<<<blocks, 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fold(const FoldParams& p, cudaStream_t st) {
  const int total = p.nR * p.nB * p.S;
  if (total == 0) return cudaSuccess;
  fold_kernel<<<(total + 255) / 256, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rk
