// rk_rl.cu — NEXT-2: the actor-critic scheduler trained on the reward of eq. `multi_acc_reward`
// (§2.4: eqs. eq:J / eq:dJ / eq:hatJ, actor-critic baseline V(s_t)
// §5.2: state, action space (2^|M|-1)*|B|, reward a(M[v]) * (b - beta * overdue)); reading S3.
//
// Environment (one WARP per episode, many episodes per launch): K model servers, one FIFO request queue
// with device arrival times (rk_sine_arrivals or uniform). At decision time t the state is
//   x = [ (t - t_s)/tau of the oldest L queued requests, 0-padded | c(m,b)/tau | max(0, free_m - t)/tau ],
// each (float)((double)ns / (double)tau); the policy pi = softmax(W2 tanh(W1 x + b1) + b2) picks the action
// a = (v-1)*nB + b_index by inverse-CDF sampling of a counter-based uniform (or the caller forces it);
// the batch = the next b requests starts at max(t, arrival of its last request, free_m for m in v), runs
// c(v,b) = max_{m in v} c(m,b) and occupies the members of v; R = a(v) (b - beta * overdue) in fp64;
// the next decision is at max(start, min_m free_m). Integer ns throughout (exact).
//
// Gradients (deterministic, fp32): returns G_t = sum_{k>=t} gamma^(k-t) R_k scale in fp64 per episode;
// one warp per sample re-runs both networks and forms dz_a = -(A_t / Ns)(1[a = a_t] - pi_a), the hidden
// deltas dp = (W2^T dz) * (1 - h^2) and the value deltas; the weight gradients are sums over samples
// (outer products) done by fixed-order block reductions: gW2/gb2 per 32-action tile, gW1/gb1 and
// gV1/gc1 per hidden unit, gv2/gc2 per hidden unit.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int RW = 4;  // warps (episodes / samples) per block

__device__ __forceinline__ uint64_t rl_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Net {  // views into the flat parameter vector [W1 | b1 | W2 | b2 | V1 | c1 | v2 | c2]
  const float *W1, *b1, *W2, *b2, *V1, *c1, *v2, *c2;
  __device__ Net(const float* P, int F, int H, int A) {
    W1 = P; b1 = W1 + H * F; W2 = b1 + H; b2 = W2 + A * H;
    V1 = b2 + A; c1 = V1 + H * F; v2 = c1 + H; c2 = v2 + H;
  }
};

// hidden layer tanh(Wx + b) for a warp: lanes own units j = lane + 32 k; x and out in shared memory
__device__ __forceinline__ void hidden(const float* W, const float* bvec, const float* x, int F, int H, float* out,
                                       int lane) {
  for (int j = lane; j < H; j += 32) {
    float a = __ldg(bvec + j);
    const float* w = W + (size_t)j * F;
    for (int f = 0; f < F; ++f) a = fmaf(__ldg(w + f), x[f], a);
    out[j] = tanhf(a);
  }
  __syncwarp();
}

// logits z_a = b2[a] + W2[a] . h for the lane's contiguous chunk [a0, a1); returns the warp max
__device__ __forceinline__ float logits(const Net& net, const float* h, int H, float* z, int a0, int a1) {
  float mx = -INFINITY;
  for (int a = a0; a < a1; ++a) {
    float s = __ldg(net.b2 + a);
    const float* w = net.W2 + (size_t)a * H;
    for (int j = 0; j < H; ++j) s = fmaf(__ldg(w + j), h[j], s);
    z[a] = s;
    mx = fmaxf(mx, s);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
  return mx;
}

__global__ void __launch_bounds__(32 * RW) ac_rollout_kernel(const RLParams p) {
  extern __shared__ __align__(16) float rl_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * RW + warp;
  const int F = p.F, H = p.H, A = p.A, K = p.K, nB = p.nB;
  float* x = rl_smem + warp * (p.F + p.H + p.A);
  float* h = x + F;
  float* z = h + H;
  if (e >= p.E) return;
  const Net net(p.params, F, H, A);
  const int per = (A + 31) / 32, a0 = min(A, lane * per), a1 = min(A, a0 + per);
  int64_t head = p.h0[e];
  if (head < 0 || head >= p.Narr) {  // an episode start outside the arrival array
    if (lane == 0) atomicOr(p.err, 1u);
    return;
  }
  int64_t t = p.arrival[head];
  int64_t free_at[kMaxK];
  for (int m = 0; m < K; ++m) free_at[m] = t;
  int64_t tail = head;
  const double tau = (double)p.tau;
  for (int st = 0; st < p.n; ++st) {
    const size_t sidx = (size_t)e * p.n + st;
    // ---- state ----
    for (;;) {  // tail = #{s : arrival[s] <= t}, sorted arrivals
      const int64_t s = tail + lane;
      const bool in = s < p.Narr && p.arrival[s] <= t;
      const unsigned bal = __ballot_sync(FULL, in);
      tail += __popc(bal);
      if (bal != FULL) break;
    }
    for (int i = lane; i < p.L; i += 32)
      x[i] = (head + i < tail) ? (float)__ddiv_rn((double)(t - p.arrival[head + i]), tau) : 0.f;
    for (int i = lane; i < K * nB; i += 32) x[p.L + i] = (float)__ddiv_rn((double)p.lat[i], tau);
    if (lane < K) {
      int64_t fm = free_at[0];
      for (int m = 1; m < K; ++m) fm = (m == lane) ? free_at[m] : fm;
      x[p.L + K * nB + lane] = (float)__ddiv_rn((double)(fm > t ? fm - t : 0), tau);
    }
    __syncwarp();
    if (p.states)
      for (int f = lane; f < F; f += 32) p.states[sidx * F + f] = x[f];
    // ---- action ----
    int act;
    if (p.forced) {
      act = p.forced[sidx];
    } else {
      hidden(net.W1, net.b1, x, F, H, h, lane);
      const float mx = logits(net, h, H, z, a0, a1);
      float cs = 0.f;
      for (int a = a0; a < a1; ++a) cs += __expf(z[a] - mx);
      float incl = cs;  // inclusive scan of the lanes' chunk sums (action order)
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const float total = __shfl_sync(FULL, incl, 31);
      if (!(total > 0.f) || isinf(total)) {  // non-finite parameters (a diverged update)
        if (lane == 0) atomicOr(p.err, 4u);
        return;
      }
      const uint64_t hr = rl_mix(rl_mix(rl_mix(p.seed ^ 0xAC7013ull) ^ (uint64_t)e) + (uint64_t)st);
      const float target = (float)((double)(hr >> 11) * 0x1.0p-53) * total;
      // the first action whose cumulative mass exceeds the target (the last positive one if rounding
      // leaves the target at the total)
      int pick = -1;
      float run = incl - cs;
      for (int a = a0; a < a1; ++a) {
        run += __expf(z[a] - mx);
        if (pick < 0 && run > target) pick = a;
      }
      const unsigned has = __ballot_sync(FULL, pick >= 0);
      if (has) {
        act = __shfl_sync(FULL, pick, __ffs(has) - 1);
      } else {
        int last = -1;
        for (int a = a0; a < a1; ++a) if (z[a] > -INFINITY) last = a;
        const unsigned hl = __ballot_sync(FULL, last >= 0);
        act = __shfl_sync(FULL, last, 31 - __clz(hl));
      }
    }
    // ---- transition ----
    if (act < 0 || act >= A) {  // a forced action outside the action space
      if (lane == 0) atomicOr(p.err, 2u);
      return;
    }
    const uint32_t v = (uint32_t)(act / nB) + 1u;
    const int bi = act % nB, b = p.B[bi];
    if (head + b > p.Narr) {  // the caller's arrival array is too short for this episode
      if (lane == 0) atomicOr(p.err, 1u);
      return;
    }
    int64_t start = max(t, p.arrival[head + b - 1]), c = 0;
    for (int m = 0; m < K; ++m)
      if ((v >> m) & 1u) {
        start = max(start, free_at[m]);
        c = max(c, p.lat[m * nB + bi]);
      }
    const int64_t done = start + c;
    int o = 0;
    for (int s = lane; s < b; s += 32) o += (done - p.arrival[head + s] > p.tau) ? 1 : 0;
    for (int q = 16; q; q >>= 1) o += __shfl_xor_sync(FULL, o, q);
    if (lane == 0) {
      p.actions[sidx] = act;
      p.rewards[sidx] = __dmul_rn(p.acc[v - 1], __dsub_rn((double)b, __dmul_rn(p.beta, (double)o)));
      if (p.overdue) p.overdue[sidx] = o;
      if (p.t_dec) p.t_dec[sidx] = t;
      if (p.t_start) p.t_start[sidx] = start;
      if (p.t_done) p.t_done[sidx] = done;
    }
    int64_t fmin = INT64_MAX;
    for (int m = 0; m < K; ++m) {
      if ((v >> m) & 1u) free_at[m] = done;
      fmin = min(fmin, free_at[m]);
    }
    head += b;
    t = max(start, fmin);
    __syncwarp();
  }
}

// ---- gradients -------------------------------------------------------------------------------------------
__global__ void ac_returns_kernel(const RLParams p, double* G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p.E) return;
  double g = 0.0;
  for (int t = p.n - 1; t >= 0; --t) {
    const size_t i = (size_t)e * p.n + t;
    g = __dadd_rn(__dmul_rn(p.rewards[i], p.scale), __dmul_rn(p.gamma, g));
    G[i] = g;
  }
}

// one warp per sample: both forward passes, the output / value deltas and the hidden deltas
__global__ void __launch_bounds__(32 * RW) ac_sample_kernel(const RLParams p, const double* G, float* Hs, float* HV,
                                                            float* DP, float* DPV, float* coef, float* lse_out,
                                                            float* dV, float* lossv, float* ent_out) {
  extern __shared__ __align__(16) float rl_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = p.F, H = p.H, A = p.A;
  const int64_t Ns = (int64_t)p.E * p.n;
  const int64_t s = (int64_t)blockIdx.x * RW + warp;
  float* x = rl_smem + warp * (F + 2 * H + A);
  float* h = x + F;
  float* hv = h + H;
  float* z = hv + H;
  if (s >= Ns) return;
  const Net net(p.params, F, H, A);
  const float inv = (float)(1.0 / (double)Ns);
  for (int f = lane; f < F; f += 32) x[f] = p.states[s * F + f];
  __syncwarp();
  hidden(net.W1, net.b1, x, F, H, h, lane);
  hidden(net.V1, net.c1, x, F, H, hv, lane);
  const int per = (A + 31) / 32, a0 = min(A, lane * per), a1 = min(A, a0 + per);
  const float mx = logits(net, h, H, z, a0, a1);
  float cs = 0.f;
  for (int a = a0; a < a1; ++a) cs += __expf(z[a] - mx);
  for (int o = 16; o; o >>= 1) cs += __shfl_xor_sync(FULL, cs, o);
  const float lse = mx + logf(cs);
  float V = 0.f;
  for (int j = lane; j < H; j += 32) V = fmaf(__ldg(net.v2 + j), hv[j], V);
  for (int o = 16; o; o >>= 1) V += __shfl_xor_sync(FULL, V, o);
  V += __ldg(net.c2);
  const float g = (float)G[s];
  const float adv = g - V;
  const int at = p.actions[s];
  const float cpi = -adv * inv;  // dz_a = cpi * (1[a = at] - pi_a) + ce * pi_a * (log pi_a + Hs)
  const float ce = (float)p.ent * inv;
  // policy entropy Hs = -sum_a pi_a log pi_a (the entropy bonus of the loss, X4 / PPO)
  float hs = 0.f;
  if (ce != 0.f) {
    for (int a = a0; a < a1; ++a) {
      const float lp = z[a] - lse;
      hs -= __expf(lp) * lp;
    }
    for (int o = 16; o; o >>= 1) hs += __shfl_xor_sync(FULL, hs, o);
  }
  __syncwarp();  // every lane's logits are in shared memory
  const float zat = z[at];
  __syncwarp();
  // dz into shared memory, then hidden deltas dh_j = sum_a dz_a W2[a][j] with lanes owning j
  for (int a = a0; a < a1; ++a) {
    const float lp = z[a] - lse, pa = __expf(lp);
    z[a] = cpi * ((a == at ? 1.f : 0.f) - pa) + (ce != 0.f ? ce * pa * (lp + hs) : 0.f);
  }
  __syncwarp();
  for (int j = lane; j < H; j += 32) {
    float d = 0.f;
    for (int a = 0; a < A; ++a) d = fmaf(z[a], __ldg(net.W2 + (size_t)a * H + j), d);
    DP[s * H + j] = d * (1.f - h[j] * h[j]);
    Hs[s * H + j] = h[j];
    HV[s * H + j] = hv[j];
  }
  const float dv = 2.f * (V - g) * inv;
  for (int j = lane; j < H; j += 32) DPV[s * H + j] = dv * __ldg(net.v2 + j) * (1.f - hv[j] * hv[j]);
  // losses: -(A log pi(a_t) + c H) / Ns and (V - G)^2 / Ns
  if (lane == 0) {
    coef[s] = cpi;
    lse_out[s] = lse;
    dV[s] = dv;
    ent_out[s] = hs;
    lossv[2 * s] = -adv * (zat - lse) * inv - ce * hs;
    lossv[2 * s + 1] = (V - g) * (V - g) * inv;
  }
}

// gW2 / gb2 for a tile of 32 actions (lane = action): sum over samples of dz_s(a) h_s, fixed order
__global__ void __launch_bounds__(256) ac_grad_w2_kernel(const RLParams p, const float* Hs, const float* coef,
                                                         const float* lse, const float* ent, float* grad) {
  extern __shared__ __align__(16) float rl_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int F = p.F, H = p.H, A = p.A;
  const int64_t Ns = (int64_t)p.E * p.n;
  const int a = blockIdx.x * 32 + lane;
  const Net net(p.params, F, H, A);
  float* hrow = rl_smem + warp * H;                 // [nw][H]
  float* red = rl_smem + nw * H;                    // [nw][32][H + 1]
  float acc[kRlMaxH];
  float accb = 0.f;
#pragma unroll
  for (int j = 0; j < kRlMaxH; ++j) acc[j] = 0.f;
  float w[kRlMaxH];
#pragma unroll
  for (int j = 0; j < kRlMaxH; ++j) w[j] = (a < A && j < H) ? __ldg(net.W2 + (size_t)a * H + j) : 0.f;
  const float bb = a < A ? __ldg(net.b2 + a) : 0.f;
  const float ce = (float)p.ent * (float)(1.0 / (double)Ns);
  for (int64_t s = warp; s < Ns; s += nw) {
    for (int j = lane; j < H; j += 32) hrow[j] = Hs[s * H + j];
    __syncwarp();
    float zz = bb;
#pragma unroll
    for (int j = 0; j < kRlMaxH; ++j) if (j < H) zz = fmaf(w[j], hrow[j], zz);
    const float lp = zz - lse[s], pa = __expf(lp);
    const float dz = coef[s] * ((a == p.actions[s] ? 1.f : 0.f) - pa) + (ce != 0.f ? ce * pa * (lp + ent[s]) : 0.f);
#pragma unroll
    for (int j = 0; j < kRlMaxH; ++j) if (j < H) acc[j] = fmaf(dz, hrow[j], acc[j]);
    accb += dz;
    __syncwarp();
  }
  float* mine = red + ((size_t)warp * 32 + lane) * (H + 1);
#pragma unroll
  for (int j = 0; j < kRlMaxH; ++j) if (j < H) mine[j] = acc[j];
  mine[H] = accb;
  __syncthreads();
  if (warp == 0 && a < A) {
    float* gW2 = grad + (size_t)H * F + H;
    float* gb2 = gW2 + (size_t)A * H;
    for (int j = 0; j <= H; ++j) {
      float t = 0.f;
      for (int q = 0; q < nw; ++q) t += red[((size_t)q * 32 + lane) * (H + 1) + j];
      if (j < H) gW2[(size_t)a * H + j] = t;
      else gb2[a] = t;
    }
  }
}

// gW1/gb1 (which = 0, deltas DP) or gV1/gc1 (which = 1, deltas DPV) for hidden unit j = blockIdx.x;
// threads own inputs f. Also gv2[j] / gc2 (which = 1).
__global__ void __launch_bounds__(256) ac_grad_w1_kernel(const RLParams p, const float* D, const float* HV,
                                                         const float* dV, float* grad, int which) {
  const int F = p.F, H = p.H, A = p.A;
  const int64_t Ns = (int64_t)p.E * p.n;
  const int j = blockIdx.x;
  float* gW = grad + (which ? ((size_t)H * F + H + (size_t)A * H + A) : 0);
  float* gb = gW + (size_t)H * F;
  __shared__ float part[256];
  for (int f0 = 0; f0 < F + 1; f0 += blockDim.x) {
    const int f = f0 + threadIdx.x;
    float acc = 0.f;
    if (f < F)
      for (int64_t s = 0; s < Ns; ++s) acc = fmaf(D[s * H + j], p.states[s * F + f], acc);
    else if (f == F)
      for (int64_t s = 0; s < Ns; ++s) acc += D[s * H + j];
    if (f < F) gW[(size_t)j * F + f] = acc;
    else if (f == F) gb[j] = acc;
  }
  if (which) {  // gv2[j] = sum_s dV_s hv_s[j]; block 0 also gc2 = sum_s dV_s (fixed-order tree per block)
    float* gv2 = gb + H;
    float a = 0.f, c = 0.f;
    for (int64_t s = threadIdx.x; s < Ns; s += blockDim.x) {
      a = fmaf(dV[s], HV[s * H + j], a);
      c += dV[s];
    }
    part[threadIdx.x] = a;
    __syncthreads();
    for (int w = blockDim.x / 2; w; w >>= 1) {
      if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) gv2[j] = part[0];
    __syncthreads();
    if (j == 0) {
      part[threadIdx.x] = c;
      __syncthreads();
      for (int w = blockDim.x / 2; w; w >>= 1) {
        if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
      }
      if (threadIdx.x == 0) gv2[H] = part[0];
    }
  }
}

__global__ void ac_loss_kernel(const float* lossv, int64_t Ns, float* out) {
  __shared__ float part[2][256];
  float a = 0.f, b = 0.f;
  for (int64_t s = threadIdx.x; s < Ns; s += blockDim.x) { a += lossv[2 * s]; b += lossv[2 * s + 1]; }
  part[0][threadIdx.x] = a;
  part[1][threadIdx.x] = b;
  __syncthreads();
  for (int w = blockDim.x / 2; w; w >>= 1) {
    if (threadIdx.x < w) { part[0][threadIdx.x] += part[0][threadIdx.x + w]; part[1][threadIdx.x] += part[1][threadIdx.x + w]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = part[0][0]; out[1] = part[1][0]; }
}

__global__ void ac_apply_kernel(float* P, const float* g, int64_t npol, int64_t np, float lr_pi, float lr_v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < np) P[i] -= (i < npol ? lr_pi : lr_v) * g[i];
}

}  // namespace

int64_t ac_param_count(int F, int H, int A) {
  return (int64_t)H * F + H + (int64_t)A * H + A + (int64_t)H * F + H + H + 1;
}

cudaError_t launch_ac_rollout(const RLParams& p, cudaStream_t st) {
  if (p.E <= 0 || p.n <= 0) return cudaSuccess;
  const size_t smem = (size_t)RW * (p.F + p.H + p.A) * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ac_rollout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  ac_rollout_kernel<<<(p.E + RW - 1) / RW, 32 * RW, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ac_grad(const RLParams& p, float* grad, float* loss2, void* scratch, cudaStream_t st) {
  const int64_t Ns = (int64_t)p.E * p.n;
  if (Ns <= 0) return cudaSuccess;
  const int H = p.H;
  char* w = static_cast<char*>(scratch);
  double* G = reinterpret_cast<double*>(w); w += Ns * 8;
  float* Hs = reinterpret_cast<float*>(w); w += Ns * H * 4;
  float* HV = reinterpret_cast<float*>(w); w += Ns * H * 4;
  float* DP = reinterpret_cast<float*>(w); w += Ns * H * 4;
  float* DPV = reinterpret_cast<float*>(w); w += Ns * H * 4;
  float* coef = reinterpret_cast<float*>(w); w += Ns * 4;
  float* lse = reinterpret_cast<float*>(w); w += Ns * 4;
  float* dV = reinterpret_cast<float*>(w); w += Ns * 4;
  float* ent = reinterpret_cast<float*>(w); w += Ns * 4;
  float* lossv = reinterpret_cast<float*>(w);
  ac_returns_kernel<<<(p.E + 127) / 128, 128, 0, st>>>(p, G);
  const size_t smem = (size_t)RW * (p.F + 2 * p.H + p.A) * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ac_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  ac_sample_kernel<<<(unsigned)((Ns + RW - 1) / RW), 32 * RW, smem, st>>>(p, G, Hs, HV, DP, DPV, coef, lse, dV, lossv,
                                                                           ent);
  const size_t smem2 = (size_t)8 * H * 4 + (size_t)8 * 32 * (H + 1) * 4;
  cudaError_t e = cudaFuncSetAttribute(ac_grad_w2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  if (e != cudaSuccess) return e;
  ac_grad_w2_kernel<<<(p.A + 31) / 32, 256, smem2, st>>>(p, Hs, coef, lse, ent, grad);
  ac_grad_w1_kernel<<<H, 256, 0, st>>>(p, DP, HV, dV, grad, 0);
  ac_grad_w1_kernel<<<H, 256, 0, st>>>(p, DPV, HV, dV, grad, 1);
  if (loss2) ac_loss_kernel<<<1, 256, 0, st>>>(lossv, Ns, loss2);
  return cudaGetLastError();
}

size_t ac_grad_scratch_bytes(const RLParams& p) {
  const int64_t Ns = (int64_t)p.E * p.n;
  return (size_t)Ns * (8 + 4 * 4 * p.H + 4 * 4 + 8);
}

cudaError_t launch_ac_apply(float* P, const float* g, int64_t npol, int64_t np, float lr_pi, float lr_v,
                            cudaStream_t st) {
  if (np <= 0) return cudaSuccess;
  ac_apply_kernel<<<(unsigned)((np + 255) / 256), 256, 0, st>>>(P, g, npol, np, lr_pi, lr_v);
  return cudaGetLastError();
}

}  // namespace rk
