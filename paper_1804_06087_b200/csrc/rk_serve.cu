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
// one scenario (thousands of scenarios per launch); integer nanoseconds throughout (exact).
// The reward of eq. `multi_acc_reward` summed over the greedy batches,
// a(v) * (served - beta * overdue), is folded in fp64 in the same thread.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

__device__ __forceinline__ int64_t arrival_ns(const int64_t* arr, int64_t s, double rate) {
  if (arr) return arr[s];
  return (int64_t)floor(__ddiv_rn(__dmul_rn((double)s, 1e9), rate));  // reading Q9, two roundings
}

__global__ void greedy_serve_kernel(const ServeParams p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.nR * p.S) return;
  const int r = i / p.S;
  const uint32_t v = (uint32_t)(i % p.S) + 1u;
  const double rate = p.rates[r];
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
    while (tail < N && arrival_ns(p.arrival, tail, rate) <= t) ++tail;
    const int64_t qlen = tail - head;
    int bsel = 0;
    int64_t c = 0;
    for (int bi = 0; bi < p.nB; ++bi)
      if (p.B[bi] <= qlen && p.B[bi] > bsel) { bsel = p.B[bi]; c = cb[bi]; }
    int b = 0;
    const int64_t t0 = head < N ? arrival_ns(p.arrival, head, rate) : 0;
    if (qlen >= bmax) b = bmax;
    else if (bsel > 0 && c + (t - t0) + p.delta >= p.tau) b = bsel;
    if (b > 0) {
      const int64_t done = t + c;
      for (int64_t s = head; s < head + b; ++s) {
        const int64_t l = done - arrival_ns(p.arrival, s, rate);
        ++served;
        if (l > p.tau) { ++overdue; exceed += (unsigned long long)(l - p.tau); }
      }
      ++batches;
      head += b;
      t = done;
    } else if (tail == N) {
      if (bsel == 0) { unserved = (unsigned long long)qlen; break; }
      t = t0 + p.tau - p.delta - c;
    } else {
      int64_t tn = arrival_ns(p.arrival, tail, rate);
      if (bsel > 0) tn = min(tn, t0 + p.tau - p.delta - c);
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

}  // namespace

cudaError_t launch_greedy_serve(const ServeParams& p, cudaStream_t st) {
  const int n = p.nR * p.S;
  if (n <= 0) return cudaSuccess;
  greedy_serve_kernel<<<(n + 127) / 128, 128, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rk
