// rk_arrivals.cu — NEXT-4: the paper's request-arrival process on the device (§7.2,
// eqs. `eq:r1`/`eq:r2`; SPEC.md:702-710 closed form), reading Q16:
//
//   rate(t) = k sin(2 pi t / T) + b  with  s0 = sin(0.3 pi) = (1 + sqrt 5) / 4,  k = 0.1 ref / (1 - s0),
//   b = 1.1 ref - k  (ref = r_u or r_l: the rate exceeds ref for 20 % of each period, peak 1.1 ref);
//   the simulator is invoked every delta ns; invocation j (covering [j delta, (j+1) delta)) adds
//   n_j = floor(max(0, delta_s * rate(j delta) * (1 + phi_j)) + 0.5) requests, phi_j = sigma * z_j
//   ("a small random noise ... phi ~ N(0, 0.1)"), z_j an Irwin-Hall(4) unit normal from a SplitMix64
//   counter hash of (seed, j) -- a counter-based generator both sides implement independently;
//   the n_j requests of invocation j arrive evenly spaced inside it: t = j delta + floor(i delta / n_j).
//
// Three kernels per chunk of invocations: per-invocation counts with per-block sums, a one-block scan of
// the block sums, and a per-block scan that scatters the arrival times of the requests with global
// index in [n0, n0 + N). The host loops over chunks until n0 + N requests exist (normally one chunk).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr int AT = 1024;  // invocations per block

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// requests added by invocation j (fp64 throughout, explicit roundings: no FMA contraction)
__device__ __forceinline__ int64_t invocation_count(const SineParams& p, int64_t j) {
  const int64_t u = (int64_t)(((unsigned long long)j * (unsigned long long)p.delta) % (unsigned long long)p.period);
  const double f = __ddiv_rn((double)u, (double)p.period);  // phase in [0, 1)
  const double s = sinpi(__dmul_rn(2.0, f));
  const double rate = __dadd_rn(__dmul_rn(p.k, s), p.b);
  const uint64_t h = mix64(mix64(mix64(p.seed ^ 0x51AE0A77ull) ^ (uint64_t)j) + 0x2545F4914F6CDD1Dull);
  const int64_t ih = (int64_t)(h & 0xffff) + (int64_t)((h >> 16) & 0xffff) + (int64_t)((h >> 32) & 0xffff) +
                     (int64_t)(h >> 48) - 131070;
  const double z = __dmul_rn((double)(ih * 7), 3.814697265625e-06);  // * 2^-18, exact
  const double phi = __dmul_rn(p.sigma, z);
  double y = __dmul_rn(__dmul_rn(p.delta_s, rate), __dadd_rn(1.0, phi));
  if (!(y > 0.0)) y = 0.0;
  return (int64_t)floor(__dadd_rn(y, 0.5));
}

__global__ void __launch_bounds__(AT) sine_count_kernel(const SineParams p, int64_t j0, int64_t J, int64_t* cnt,
                                                        int64_t* bsum) {
  __shared__ int64_t red[AT / 32];
  const int64_t j = j0 + (int64_t)blockIdx.x * AT + threadIdx.x;
  const int64_t c = (j - j0) < J ? invocation_count(p, j) : 0;
  if ((j - j0) < J) cnt[j - j0] = c;
  int64_t s = c;
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t t = red[threadIdx.x];
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
  }
}

// exclusive scan of nb block sums (one block, sequential chunks per thread), total to bsum[nb]
__global__ void __launch_bounds__(AT) sine_bscan_kernel(int64_t* bsum, int64_t nb) {
  __shared__ int64_t part[AT];
  const int t = threadIdx.x;
  const int64_t per = (nb + AT - 1) / AT, lo = t * per, hi = min(nb, lo + per);
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += bsum[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t run = 0;
    for (int i = 0; i < AT; ++i) { const int64_t v = part[i]; part[i] = run; run += v; }
    bsum[nb] = run;
  }
  __syncthreads();
  int64_t run = part[t];
  for (int64_t i = lo; i < hi; ++i) { const int64_t v = bsum[i]; bsum[i] = run; run += v; }
}

// base = requests before invocation j0; writes t of every request with global index in [n0, n0 + N)
__global__ void __launch_bounds__(AT) sine_scatter_kernel(const SineParams p, int64_t j0, int64_t J,
                                                          const int64_t* cnt, const int64_t* bsum, int64_t base,
                                                          int64_t n0, int64_t N, int64_t* out) {
  __shared__ int64_t ws[AT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * AT + threadIdx.x;
  const int64_t c = i < J ? cnt[i] : 0;
  int64_t x = c;  // inclusive warp scan
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t v = ws[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    ws[lane] = v - ws[lane];  // exclusive
  }
  __syncthreads();
  const int64_t first = base + bsum[blockIdx.x] + ws[w] + x - c;  // global index of this invocation's first request
  if (c == 0 || first >= n0 + N || first + c <= n0) return;
  const int64_t j = j0 + i;
  const int64_t t0 = j * p.delta;
  const int64_t a = n0 > first ? n0 - first : 0, e = (n0 + N - first) < c ? (n0 + N - first) : c;
  for (int64_t q = a; q < e; ++q) out[first + q - n0] = t0 + (q * p.delta) / c;
}

}  // namespace

int64_t sine_chunk_blocks(int64_t J) { return (J + AT - 1) / AT; }

cudaError_t launch_sine_counts(const SineParams& p, int64_t j0, int64_t J, int64_t* cnt, int64_t* bsum,
                               cudaStream_t st) {
  const int64_t nb = sine_chunk_blocks(J);
  sine_count_kernel<<<(unsigned)nb, AT, 0, st>>>(p, j0, J, cnt, bsum);
  sine_bscan_kernel<<<1, AT, 0, st>>>(bsum, nb);
  return cudaGetLastError();
}

cudaError_t launch_sine_scatter(const SineParams& p, int64_t j0, int64_t J, const int64_t* cnt, const int64_t* bsum,
                                int64_t base, int64_t n0, int64_t N, int64_t* out, cudaStream_t st) {
  sine_scatter_kernel<<<(unsigned)sine_chunk_blocks(J), AT, 0, st>>>(p, j0, J, cnt, bsum, base, n0, N, out);
  return cudaGetLastError();
}

}  // namespace rk
