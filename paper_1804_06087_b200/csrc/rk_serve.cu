// rk_serve.cu — NEXT-1: Algorithm 3, Inference(Queue q, Model m), greedy batching
// of every subset v run as a synchronous ensemble (c(v,b) = max over members of c(m,b), stragglers
// PAPER.md:410), on one request stream per arrival rate. Reading S1: single server,
// inference blocks the loop; whenever the server is idle at time t, with q the arrived, unserved
// requests (oldest first):
//   len(q) >= max B                                     -> infer the oldest max B at t;
//   b = max{b in B : b <= len(q)} exists and
//     c(v,b) + (t - t_q0) + delta >= tau                -> infer the oldest b at t;
//   otherwise wait for the next arrival or for the instant the condition becomes true.
// A batch inferred at t completes at t + c(v,b); l(s) = completion - t_s; overdue iff l(s) > tau.
// Requests still queued (fewer than min B) after the last arrival are unserved.
//
// The policy is sequential in time but independent across (rate, subset), so one thread simulates
// one scenario (thousands of scenarios per launch) over arrival arrays computed once per rate by a
// parallel fill (the fp64 division of reading Q9 is off the sequential path); integer nanoseconds
// throughout (exact).
// The reward of eq. `multi_acc_reward` summed over the greedy batches,
// a(v) * (served - beta * overdue), is folded in fp64 in the same thread.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

// arrival times of every rate, computed once (reading Q9: t_s = floor(s * 1e9 / r), two roundings)
__global__ void arrival_fill_kernel(int64_t* out, int64_t N, int nR, const ServeParams p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * nR) return;
  const int r = (int)(i / N);
  const int64_t s = i - (int64_t)r * N;
  out[i] = (int64_t)floor(__ddiv_rn(__dmul_rn((double)s, 1e9), p.rates[r]));
}

__global__ void greedy_serve_kernel(const ServeParams p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (p.v_only ? 1 : p.nR * p.S)) return;
  const int r = p.v_only ? 0 : i / p.S;
  const uint32_t v = p.v_only ? p.v_only : (uint32_t)(i % p.S) + 1u;
  const int64_t* arr = p.arrival + (int64_t)r * p.N;  // this rate's arrival times
  int64_t cb[kMaxB];
  int bmax = 0, bmin = 1 << 30;
  for (int bi = 0; bi < p.nB; ++bi) {
    int64_t c = 0;
    for (int m = 0; m < p.K; ++m)
      if (((v >> m) & 1u) && p.lat[m * p.nB + bi] > c) c = p.lat[m * p.nB + bi];
    cb[bi] = c;
    bmax = max(bmax, p.B[bi]);
    bmin = min(bmin, p.B[bi]);
  }
  unsigned long long served = 0, overdue = 0, exceed = 0, batches = 0, unserved = 0;
  int64_t t = 0, head = 0, tail = 0;
  const int64_t N = p.N;
  while (head < N) {
    while (tail < N) {  // arrivals up to t: 8 independent loads per step (sorted, so the count is the advance)
      int adv = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) adv += (tail + i < N && arr[tail + i] <= t) ? 1 : 0;
      tail += adv;
      if (adv < 8) break;
    }
    const int64_t qlen = tail - head;
    int bsel = 0;
    int64_t c = 0;
    for (int bi = 0; bi < p.nB; ++bi)
      if (p.B[bi] <= qlen && p.B[bi] > bsel) { bsel = p.B[bi]; c = cb[bi]; }
    int b = 0;
    const int64_t t0 = head < N ? arr[head] : 0;
    if (qlen >= bmax) b = bmax;
    else if (bsel > 0 && c + (t - t0) + p.delta >= p.tau) b = bsel;
    if (b > 0) {
      const int64_t done = t + c;
#pragma unroll 8
      for (int64_t s = head; s < head + b; ++s) {
        const int64_t l = done - arr[s];
        ++served;
        if (l > p.tau) { ++overdue; exceed += (unsigned long long)(l - p.tau); }
      }
      if (p.sched) { p.sched[2 * batches] = head; p.sched[2 * batches + 1] = b; }
      ++batches;
      head += b;
      t = done;
    } else {
      // wait: the decision can only change when the queue reaches the next batch size above len(q)
      // or when c(v,b) + w(q0) + delta reaches tau for the current b -- jump to the earlier of the two
      // (equivalent to re-evaluating the rule at every arrival, reading S1)
      int bnext = 0x7fffffff;
      for (int bi = 0; bi < p.nB; ++bi)
        if (p.B[bi] > qlen && p.B[bi] < bnext) bnext = p.B[bi];
      int64_t tn = INT64_MAX;
      if (bnext != 0x7fffffff && head + bnext - 1 < N) tn = arr[head + bnext - 1];
      if (bsel > 0) tn = min(tn, t0 + p.tau - p.delta - c);
      if (tn == INT64_MAX) { unserved = (unsigned long long)(N - head); break; }  // never reaches min B
      t = tn;
    }
  }
  const int64_t n = (int64_t)p.nR * p.S;
  p.out[i] = served;
  p.out[n + i] = overdue;
  p.out[2 * n + i] = exceed;
  p.out[3 * n + i] = batches;
  p.out[4 * n + i] = unserved;
  if (p.acc && p.reward)
    p.reward[i] = __dmul_rn(p.acc[v - 1], __dsub_rn((double)served, __dmul_rn(p.beta, (double)overdue)));
}

// NEXT-1 baseline ("runs all models asynchronously, one model per batch"; reading S2):
// K servers share one FIFO queue; whenever a model is idle at t, the lowest-index idle model m evaluates
// Algorithm 3's rule with its own c(m, b); a dispatched batch occupies m until t + c(m, b) and the rule
// is re-evaluated at the same t; otherwise time advances to the next event that can change the decision
// (an arrival, the rule's threshold instant for m, a lower-index model becoming idle; all busy: the
// earliest completion). One thread per rate (sequential by definition), integer ns.
__global__ void async_serve_kernel(const ServeParams p, const double* acc_single, unsigned long long* mb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p.nR) return;
  const int64_t* arr = p.arrival + (int64_t)r * p.N;
  const int K = p.K;
  int bmax = 0;
  for (int bi = 0; bi < p.nB; ++bi) bmax = max(bmax, p.B[bi]);
  int64_t free_at[kMaxK];
  unsigned long long nbat[kMaxK];
  for (int m = 0; m < K; ++m) { free_at[m] = 0; nbat[m] = 0; }
  unsigned long long served = 0, overdue = 0, exceed = 0, batches = 0, unserved = 0;
  double rew = 0.0;
  int64_t t = 0, head = 0, tail = 0;
  const int64_t N = p.N;
  while (head < N) {
    while (tail < N && arr[tail] <= t) ++tail;
    int m = -1;
    for (int i = K - 1; i >= 0; --i) if (free_at[i] <= t) m = i;
    if (m < 0) {
      int64_t tn = free_at[0];
      for (int i = 1; i < K; ++i) tn = min(tn, free_at[i]);
      t = tn;
      continue;
    }
    const int64_t qlen = tail - head;
    int bsel = 0;
    int64_t c = 0;
    for (int bi = 0; bi < p.nB; ++bi)
      if (p.B[bi] <= qlen && p.B[bi] > bsel) { bsel = p.B[bi]; c = p.lat[m * p.nB + bi]; }
    int b = 0;
    if (qlen >= bmax) b = bmax;
    else if (bsel > 0 && c + (t - arr[head]) + p.delta >= p.tau) b = bsel;
    if (b > 0) {
      const int64_t done = t + c;
      unsigned long long od = 0;
      for (int64_t s = head; s < head + b; ++s) {
        const int64_t l = done - arr[s];
        ++served;
        if (l > p.tau) { ++od; exceed += (unsigned long long)(l - p.tau); }
      }
      overdue += od;
      ++batches;
      ++nbat[m];
      if (acc_single) rew = __dadd_rn(rew, __dmul_rn(acc_single[m], __dsub_rn((double)b, __dmul_rn(p.beta, (double)od))));
      free_at[m] = done;
      head += b;
      continue;
    }
    int64_t tn = INT64_MAX;
    if (tail < N) tn = arr[tail];
    if (bsel > 0) tn = min(tn, arr[head] + p.tau - p.delta - c);
    for (int i = 0; i < m; ++i) if (free_at[i] > t && free_at[i] < tn) tn = free_at[i];
    if (tn == INT64_MAX) { unserved = (unsigned long long)(N - head); break; }
    t = tn;
  }
  const int n = p.nR;
  p.out[r] = served;
  p.out[n + r] = overdue;
  p.out[2 * n + r] = exceed;
  p.out[3 * n + r] = batches;
  p.out[4 * n + r] = unserved;
  if (p.reward) p.reward[r] = rew;
  if (mb) for (int m = 0; m < K; ++m) mb[(int64_t)r * K + m] = nbat[m];
}

}  // namespace

cudaError_t launch_arrival_fill(const ServeParams& p, int64_t* out, cudaStream_t st) {
  const int64_t n = p.N * p.nR;
  if (n <= 0) return cudaSuccess;
  arrival_fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, p.N, p.nR, p);
  return cudaGetLastError();
}

cudaError_t launch_greedy_serve(const ServeParams& p, cudaStream_t st) {
  const int n = p.nR * p.S;
  if (n <= 0) return cudaSuccess;
  greedy_serve_kernel<<<(n + 127) / 128, 128, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_async_serve(const ServeParams& p, const double* acc_single, unsigned long long* model_batches,
                               cudaStream_t st) {
  if (p.nR <= 0) return cudaSuccess;
  async_serve_kernel<<<1, 32, 0, st>>>(p, acc_single, model_batches);
  return cudaGetLastError();
}

}  // namespace rk
