// rk_vote.cu — steps A2-A5 of the hot path: per-model top-1 / softmax normaliser, majority vote
// and softmax average of every model subset, and the per-subset / per-group correct counts.
//
// PAPER.md (arXiv 1804.06087) passages implemented here:
//   PAPER.md:153  top-1 prediction of each model; reading Q4: lowest class index on ties.
//   PAPER.md:407  "Majority voting is applied to aggregate the predictions ... when there is a tie,
//                 the prediction from the model with the best accuracy is selected"
//                 (RK_TIE_BEST_MEMBER; RK_TIE_LOWEST_CLASS is the north_star rule).
//   PAPER.md:72   "ensemble multiple models and average the results" (softmax-probability average,
//                 reading Q5; argmax lowest class on ties, reading Q6).
//   PAPER.md:429  action space: every non-empty subset v of M (v = 0 excluded); a(M[v]) is the
//                 accuracy of the subset on a labelled validation set.
//
// Design (B200, HBM-bound):
//   * Persistent CTAs of 256 threads; a CTA processes a tile of G contiguous samples (G*K rows of
//     ldc fp32 logits = one contiguous block). Tiles stream HBM -> shared memory through a ring of
//     NSTAGE slots filled by 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx) issued
//     NSTAGE-1 tiles ahead, so DRAM latency is off the critical path and logits are read once.
//   * Each (sample, model) row is then held in registers by LPR lanes (VPL float4 each): row max /
//     lowest-index argmax / sum-exp by lane loops + xor-shuffle reductions.
//   * Per-sample setup is warp-parallel (lanes = models; __match_any_sync builds the distinct-class
//     vote masks; warp reductions give theta).
//   * Exact candidate pruning: class c can be the averaged argmax of SOME subset only if
//     p[m][c] >= theta = min_j p[j][top_j] / K for some m (SURVEY.md §8(d) proof). Candidates are
//     marked in a per-sample smem bitmap (warp scan -> slots); their probabilities are gathered.
//   * Per-subset sums come from two half-tables (low / high models): one add per (subset,
//     candidate). fp32 decisions whose top-2 relative gap is inside `band` are redone in fp64
//     from the logits (rare), so results equal the fp64 definition.
//   * Unanimous samples, "label not predicted by any member" and "label not a candidate" are
//     exact shortcuts (invariant I6 and the pruning proof) -- no per-subset work.
//   * Counts: per-unit shared-memory histograms (exclusive ownership or register slot counters),
//     flushed once per CTA with 64-bit atomics. Per-group (gs samples) counts feed the labelled
//     batch moments (want_labelled).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NW = kVoteThreads / 32;

// sample flags
constexpr uint32_t F_VALID = 1u, F_UNAN = 2u, F_UNI_OK = 4u, F_VOTE_POSS = 8u, F_AVG_POSS = 16u,
                   F_OVF = 32u, F_TABLES = 64u, F_SKIP = 128u;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
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
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float comp(const float4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

struct Smem {
  float* ring;           // [NSTAGE][tile_floats]
  uint64_t* full;        // [NSTAGE]
  uint8_t* best_of;      // [2^K]
  uint32_t* cta_vote;    // [S]
  uint32_t* cta_avg;     // [S]
  uint32_t* grpcnt;      // [NGU][S]
  uint32_t* uni;         // [NGU]
  float* rmax;           // [G*K]
  float* rlse;
  int32_t* rtop;
  float* rthr;
  int32_t* sy;           // [G]
  uint32_t* sflag;
  int32_t* snd;
  int32_t* sncand;
  int32_t* sys;
  uint32_t* stail;
  int32_t* scls;         // [G][K]
  uint32_t* smsk;        // [G][K]
  double* lse64;         // [G][K]
  uint32_t* bitmap;      // [G][nW32]
  uint32_t* prefix;      // [G][nW32]
  float* P;              // [G][K][CAP+1]
  int32_t* ccls;         // [G][CAP]
  float* T;              // [G][TA+TB][TCAP|1]
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline size_t al128(size_t x) { return (x + 127) & ~size_t(127); }

__host__ __device__ inline int ngu_of(const VoteParams& p) { return p.gs > 0 ? p.U / p.gs : 1; }
__host__ __device__ inline size_t tile_floats(const VoteParams& p) { return (size_t)p.G * p.K * p.ldc; }

// Carve the dynamic shared memory. Host and device use the same function.
__host__ __device__ inline size_t carve(const VoteParams& p, char* base, Smem* s) {
  const int K = p.K, S = p.S, G = p.G, R = G * K, NGU = ngu_of(p);
  const int TA = 1 << p.K1, TB = 1 << (K - p.K1);
  size_t o = 0;
  auto take = [&](size_t bytes) -> char* { char* r = base ? base + o : nullptr; o = al16(o + bytes); return r; };
  char* ring = take(al128(4 * tile_floats(p)) * p.NSTAGE);
  char* full = take(8 * p.NSTAGE);
  char* lse64 = take(sizeof(double) * G * K);
  char* best = take(size_t(1) << K);
  char* cv = take(4ull * S);
  char* ca = take(4ull * S);
  char* gc = take(4ull * NGU * S);
  char* un = take(4ull * NGU);
  char* rmax = take(4ull * R);
  char* rlse = take(4ull * R);
  char* rtop = take(4ull * R);
  char* rthr = take(4ull * R);
  char* sy = take(4ull * G);
  char* sf = take(4ull * G);
  char* snd = take(4ull * G);
  char* snc = take(4ull * G);
  char* sys = take(4ull * G);
  char* stl = take(4ull * G);
  char* scls = take(4ull * G * K);
  char* smsk = take(4ull * G * K);
  char* bm = take(4ull * G * p.nW32);
  char* pf = take(4ull * G * p.nW32);
  char* P = take(4ull * G * (p.CAP + 1) * K);  // [G][K][CAP+1]: odd stride, conflict-free
  char* cc = take(4ull * G * p.CAP);
  char* T = take(4ull * G * (TA + TB) * (p.TCAP | 1));  // odd row stride: conflict-free
  if (s) {
    s->ring = (float*)ring; s->full = (uint64_t*)full;
    s->lse64 = (double*)lse64; s->best_of = (uint8_t*)best; s->cta_vote = (uint32_t*)cv; s->cta_avg = (uint32_t*)ca;
    s->grpcnt = (uint32_t*)gc; s->uni = (uint32_t*)un; s->rmax = (float*)rmax; s->rlse = (float*)rlse;
    s->rtop = (int32_t*)rtop; s->rthr = (float*)rthr; s->sy = (int32_t*)sy; s->sflag = (uint32_t*)sf;
    s->snd = (int32_t*)snd; s->sncand = (int32_t*)snc; s->sys = (int32_t*)sys; s->stail = (uint32_t*)stl;
    s->scls = (int32_t*)scls; s->smsk = (uint32_t*)smsk; s->bitmap = (uint32_t*)bm; s->prefix = (uint32_t*)pf;
    s->P = (float*)P; s->ccls = (int32_t*)cc; s->T = (float*)T;
  }
  return o;
}

// fp64 log-sum-exp of one row (rare recheck path; plain loop over global memory).
__device__ double row_lse64(const float* row, int C) {
  float mx = row[0];
  for (int c = 1; c < C; ++c) mx = fmaxf(mx, row[c]);
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += exp((double)row[c] - (double)mx);
  return (double)mx + log(s);
}

// Start of the CTA's k-th tile (k counts valid tiles only), or -1.
__device__ __forceinline__ int64_t tile_start(const VoteParams& p, int64_t k, int tpu, int64_t nunits) {
  const int64_t unit = blockIdx.x + (k / tpu) * gridDim.x;
  if (unit >= nunits) return -1;
  const int64_t n0 = unit * p.U + (k % tpu) * p.G;
  return n0 < p.N ? n0 : -1;
}

__device__ __forceinline__ void issue_tile(const VoteParams& p, Smem& sm, int64_t k, int tpu, int64_t nunits) {
  const int64_t n0 = tile_start(p, k, tpu, nunits);
  if (n0 < 0) return;
  const int s = (int)(k % p.NSTAGE);
  const int64_t ns = (p.N - n0) < p.G ? (p.N - n0) : p.G;
  const uint32_t bytes = (uint32_t)(ns * p.K * p.ldc * 4);
  float* dst = reinterpret_cast<float*>(reinterpret_cast<char*>(sm.ring) + (size_t)s * al128(4 * tile_floats(p)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  bulk_load(dst, p.logits + n0 * p.K * p.ldc, bytes, &sm.full[s]);
}

template <int VPL, int RP, bool STATS>
__global__ void __launch_bounds__(kVoteThreads, 2) vote_kernel(const VoteParams p) {
  extern __shared__ __align__(128) char smem_raw[];
  Smem sm;
  carve(p, smem_raw, &sm);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int K = p.K, S = p.S, G = p.G, C = p.C;
  const int R = G * K;
  const int NGU = ngu_of(p);
  const int TA = 1 << p.K1;
  const int TB = 1 << (K - p.K1);
  const int TT = TA + TB;
  const int64_t N = p.N;
  const int F = (int)(p.ldc >> 2);
  const int lane_in_row = t % p.LPR;
  const int row0 = t / p.LPR;
  const uint32_t kmask = (1u << K) - 1u;
  const size_t slot_bytes = al128(4 * tile_floats(p));
  const int tpu = p.U / G;
  const int64_t nunits = (N + p.U - 1) / p.U;
  const int CAPS = p.CAP + 1;   // P stride (odd)
  const int TSTR = p.TCAP | 1;  // half-table row stride (odd)
  // candidate probability matrix of sample g: element (slot, model m) at base[m * stride + slot]
  auto Pbase = [&](int g, uint32_t fl) -> float* {
    return (fl & F_OVF) ? p.scratch + ((size_t)blockIdx.x * G + g) * (size_t)C * K : sm.P + (size_t)g * K * CAPS;
  };
  auto Pstride = [&](uint32_t fl) -> int { return (fl & F_OVF) ? C : CAPS; };

  // ---- CTA init ----------------------------------------------------------------------------
  if (p.tie == 0)
    for (int i = t; i < (1 << K); i += kVoteThreads) sm.best_of[i] = p.best_of[i];
  for (int i = t; i < S; i += kVoteThreads) { sm.cta_vote[i] = 0; sm.cta_avg[i] = 0; }
  for (int i = t; i < NGU * S; i += kVoteThreads) sm.grpcnt[i] = 0;
  for (int i = t; i < NGU; i += kVoteThreads) sm.uni[i] = 0;
  if (t == 0) {
    for (int s = 0; s < p.NSTAGE; ++s) mbar_init(&sm.full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < p.NSTAGE - 1; ++k) issue_tile(p, sm, k, tpu, nunits);  // prologue
  }

  constexpr int NIMAX = 4;  // register slot counters when G > 1 (host guarantees G*S <= NIMAX*256)
  uint32_t slot_vote[NIMAX], slot_avg[NIMAX];
#pragma unroll
  for (int i = 0; i < NIMAX; ++i) { slot_vote[i] = 0; slot_avg[i] = 0; }

  int64_t k = 0;
  for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
    for (int tile = 0; tile < tpu; ++tile, ++k) {
      const int64_t n0 = unit * p.U + (int64_t)tile * G;
      if (n0 >= N) break;
      __syncthreads();  // previous tile fully consumed: its ring slot and all per-tile smem are free
      if (t == 0) issue_tile(p, sm, k + p.NSTAGE - 1, tpu, nunits);
      const int slot = (int)(k % p.NSTAGE);
      mbar_wait(&sm.full[slot], (uint32_t)((k / p.NSTAGE) & 1));
      const float* tileb = reinterpret_cast<const float*>(reinterpret_cast<const char*>(sm.ring) + slot * slot_bytes);

      // ---- 1. row pass: smem -> registers; max / argmax / (sum exp) per row -------------------
      float4 val[RP][VPL];
      int rrow[RP];
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int r = j * p.RS + row0;
        rrow[j] = r;
        const int g = r / K;
        const bool rv = (r < R) && (n0 + g < N);
        const float4* base = reinterpret_cast<const float4*>(tileb + (size_t)r * p.ldc);
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int c4 = lane_in_row + i * p.LPR;
          float4 x = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
          if (rv && c4 < F) {
            x = base[c4];
            if ((C & 3) && c4 == (C >> 2)) {  // padding components of the last partial float4
              const int valid = C & 3;
              if (valid < 4) x.w = -INFINITY;
              if (valid < 3) x.z = -INFINITY;
              if (valid < 2) x.y = -INFINITY;
            } else if (c4 * 4 >= C) {
              x = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
          }
          val[j][i] = x;
        }
      }
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int r = rrow[j];
        const int g = r / K;
        const bool rv = (r < R) && (n0 + g < N);
        float mx = -INFINITY;
        int arg = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int cbase = (lane_in_row + i * p.LPR) * 4;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x = comp(val[j][i], e);
            if (x > mx) { mx = x; arg = cbase + e; }
          }
        }
        for (int off = p.LPR >> 1; off > 0; off >>= 1) {
          const float om = __shfl_xor_sync(FULL, mx, off);
          const int oa = __shfl_xor_sync(FULL, arg, off);
          if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
        }
        float lse;
        bool bad;
        if (!STATS) {
          // NaN anywhere makes the sum NaN; +inf makes max +inf -> inf - inf = NaN.
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < VPL; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) s += __expf(comp(val[j][i], e) - mx);
          for (int off = p.LPR >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
          lse = mx + logf(s);
          bad = !(s == s) || !(mx > -INFINITY) || mx == INFINITY;
        } else {
          lse = rv ? p.lse_in[(n0 + g) * K + (r - g * K)] : 0.f;
          bad = !(lse > -INFINITY && lse < INFINITY) || !(mx > -INFINITY);
        }
        if (rv && lane_in_row == 0) {
          sm.rmax[r] = mx;
          sm.rtop[r] = arg;
          sm.rlse[r] = lse;
          if (bad) atomicOr(p.err, 1u);
        }
      }
      __syncthreads();

      // ---- 2. per-sample setup, warp-parallel (lane = model) ---------------------------------
      for (int g = warp; g < G; g += NW) {
        const int64_t n = n0 + g;
        uint32_t fl = 0;
        if (n < N) {
          const int y = p.labels[n];
          if (y < 0 || y >= C) {
            if (lane == 0) { atomicOr(p.err + 1, 1u); sm.sy[g] = -1; }
          } else {
            fl |= F_VALID;
            const int c = lane < K ? sm.rtop[g * K + lane] : -1 - lane;
            const uint32_t mm = __match_any_sync(FULL, c);  // models predicting the same class
            const bool leader = lane < K && (__ffs(mm) - 1) == lane;
            const uint32_t lb = __ballot_sync(FULL, leader);
            const int pos = __popc(lb & ((1u << lane) - 1u));
            if (leader) { sm.scls[g * K + pos] = c; sm.smsk[g * K + pos] = mm; }
            const int nd = __popc(lb);
            const bool unan = __shfl_sync(FULL, mm, 0) == kmask;
            if (__any_sync(FULL, lane < K && c == y)) fl |= F_VOTE_POSS;
            uint32_t tm = 0;
            for (int bi = 0; bi < p.nB; ++bi)
              if (n >= p.tail_start[bi]) tm |= 1u << bi;
            if (unan) {
              fl |= F_UNAN;
              if (c == y) fl |= F_UNI_OK;  // lane 0's class (all equal)
              fl = __shfl_sync(FULL, fl, 0);
              if ((fl & F_UNI_OK) && lane == 0) {
                const int grp = (p.gs > 0 && G > p.gs) ? g / p.gs : 0;
                atomicAdd(&sm.uni[grp], 1u);
              }
              if ((fl & F_UNI_OK) && tm)  // rare: unanimous-correct sample in the ragged tail
                for (int bi = 0; bi < p.nB; ++bi)
                  if ((tm >> bi) & 1u)
                    for (int v = lane; v < S; v += 32) atomicAdd(p.tail + (size_t)bi * S + v, 1ull);
            } else {
              // theta = min_j p[j][top_j] / K ; candidate <=> l[m][c] - lse_m >= log(theta)
              float th = lane < K ? __expf(sm.rmax[g * K + lane] - sm.rlse[g * K + lane]) : INFINITY;
              for (int off = 16; off > 0; off >>= 1) th = fminf(th, __shfl_xor_sync(FULL, th, off));
              const float lth = logf(th / (float)K);
              if (lane < K) {
                const float l = sm.rlse[g * K + lane];
                sm.rthr[g * K + lane] = (l + lth) - (1e-3f + 1e-6f * fabsf(l) + 1e-6f * fabsf(lth));
                sm.lse64[g * K + lane] = __longlong_as_double(0x7ff8000000000000ll);
              }
              for (int w = lane; w < p.nW32; w += 32) sm.bitmap[g * p.nW32 + w] = 0;
            }
            if (lane == 0) { sm.sy[g] = y; sm.snd[g] = nd; sm.stail[g] = tm; }
          }
        }
        if (lane == 0) sm.sflag[g] = fl;
      }
      __syncthreads();

      // ---- 3. mark candidates ----------------------------------------------------------------
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int r = rrow[j];
        const int g = r / K;
        if (r < R && n0 + g < N) {
          const uint32_t fl = sm.sflag[g];
          if ((fl & F_VALID) && !(fl & F_UNAN)) {
            const float thr = sm.rthr[r];
#pragma unroll
            for (int i = 0; i < VPL; ++i)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                if (comp(val[j][i], e) >= thr) {
                  const int c = (lane_in_row + i * p.LPR) * 4 + e;
                  atomicOr(&sm.bitmap[g * p.nW32 + (c >> 5)], 1u << (c & 31));
                }
              }
          }
        }
      }
      __syncthreads();

      // ---- 4. candidate slots: warp scan over bitmap words --------------------------------------
      for (int g = warp; g < G; g += NW) {
        uint32_t fl = sm.sflag[g];
        if ((fl & F_VALID) && !(fl & F_UNAN)) {
          const uint32_t wv = lane < p.nW32 ? sm.bitmap[g * p.nW32 + lane] : 0u;
          const int cnt = __popc(wv);
          int incl = cnt;
          for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(FULL, incl, off);
            if (lane >= off) incl += o;
          }
          if (lane < p.nW32) sm.prefix[g * p.nW32 + lane] = (uint32_t)(incl - cnt);
          const int run = __shfl_sync(FULL, incl, 31);
          const int y = sm.sy[g];
          const int wy = y >> 5;
          const uint32_t word_y = __shfl_sync(FULL, wv, wy);
          const int pre_y = __shfl_sync(FULL, incl - cnt, wy);
          if (lane == 0) {
            sm.sncand[g] = run;
            if ((word_y >> (y & 31)) & 1u) {
              fl |= F_AVG_POSS;
              sm.sys[g] = pre_y + __popc(word_y & ((1u << (y & 31)) - 1u));
            } else {
              sm.sys[g] = -1;
            }
            if (run > p.CAP) fl |= F_OVF;
            else if (run <= p.TCAP) fl |= F_TABLES;
            if (!(fl & (F_VOTE_POSS | F_AVG_POSS))) fl |= F_SKIP;
            sm.sflag[g] = fl;
          }
        }
      }
      __syncthreads();

      // ---- 5. gather candidate probabilities p[m][c] = exp(l - lse_m) -------------------------
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        const int r = rrow[j];
        const int g = r / K, m = r - g * K;
        if (r < R && n0 + g < N) {
          const uint32_t fl = sm.sflag[g];
          if ((fl & F_VALID) && (fl & F_AVG_POSS) && !(fl & (F_UNAN | F_SKIP))) {
            const float lse = sm.rlse[r];
            float* Pg = Pbase(g, fl);
            const int ps = Pstride(fl);
            int32_t* Cg = (fl & F_OVF) ? p.scratch_cls + ((size_t)blockIdx.x * G + g) * (size_t)C
                                       : sm.ccls + (size_t)g * p.CAP;
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
              const int cb = (lane_in_row + i * p.LPR) * 4;
              if (cb < C) {
                const uint32_t w = sm.bitmap[g * p.nW32 + (cb >> 5)];
                const uint32_t bits4 = (w >> (cb & 31)) & 0xFu;  // 4 consecutive classes share a word
                if (bits4) {
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    if ((bits4 >> e) & 1u) {
                      const int c = cb + e;
                      const int slot = (int)(sm.prefix[g * p.nW32 + (c >> 5)] + __popc(w & ((1u << (c & 31)) - 1u)));
                      Pg[(size_t)m * ps + slot] = expf(comp(val[j][i], e) - lse);
                      if (m == 0) Cg[slot] = c;
                    }
                }
              }
            }
          }
        }
      }
      __syncthreads();

      // ---- 6. half tables: A[a][c] = sum_{i in a, asc} p[i][c] (low models), B likewise (high) -
      for (int g = 0; g < G; ++g) {
        const uint32_t fl = sm.sflag[g];
        if (!(fl & F_TABLES) || (fl & (F_UNAN | F_SKIP)) || !(fl & F_VALID) || !(fl & F_AVG_POSS)) continue;
        const int nc = sm.sncand[g];
        for (int h = warp; h < TT; h += NW)
          for (int slot = lane; slot < nc; slot += 32) {
            const float* Pr = sm.P + (size_t)g * K * CAPS + slot;
            float s = 0.f;
            if (h < TA) {
              for (uint32_t a = (uint32_t)h; a; a &= a - 1) s += Pr[(size_t)(__ffs(a) - 1) * CAPS];
            } else {
              for (uint32_t b = (uint32_t)(h - TA); b; b &= b - 1) s += Pr[(size_t)(p.K1 + __ffs(b) - 1) * CAPS];
            }
            sm.T[((size_t)g * TT + h) * TSTR + slot] = s;
          }
      }
      __syncthreads();
      // ---- 7. subsets -------------------------------------------------------------------------
      const int GS = G * S;
      for (int i = 0; i < (GS + kVoteThreads - 1) / kVoteThreads; ++i) {
        const int pidx = t + i * kVoteThreads;
        if (pidx >= GS) break;
        const int g = pidx / S;
        const uint32_t v = (uint32_t)(pidx - g * S) + 1u;
        const uint32_t fl = sm.sflag[g];
        if (!(fl & F_VALID) || (fl & (F_UNAN | F_SKIP))) continue;
        const int y = sm.sy[g];
        uint32_t okv = 0, oka = 0;
        // A3: majority vote
        if (fl & F_VOTE_POSS) {
          const int nd = sm.snd[g];
          int bc = 0, bcls = 0x7fffffff;
          uint32_t tied = 0;
          for (int q = 0; q < nd; ++q) {
            const uint32_t mv = v & sm.smsk[g * K + q];
            const int cnt = __popc(mv);
            const int cq = sm.scls[g * K + q];
            if (cnt > bc) { bc = cnt; bcls = cq; tied = mv; }
            else if (cnt == bc && cnt > 0) { tied |= mv; bcls = min(bcls, cq); }
          }
          // BEST_MEMBER: best-ranked member among the tied voters (reading Q2); LOWEST_CLASS: min class
          const int winner = (p.tie == 0) ? sm.rtop[g * K + sm.best_of[tied]] : bcls;
          okv = (winner == y);
        }
        // A4: averaged probabilities
        if (fl & F_AVG_POSS) {
          if (__popc(v) == 1) {
            oka = (sm.rtop[g * K + (__ffs(v) - 1)] == y);  // softmax is monotone (invariant I1)
          } else {
            const int nc = sm.sncand[g];
            const int ys = sm.sys[g];
            float sy_ = 0.f, m2 = -1.f;
            if (fl & F_TABLES) {
              const float* TAg = sm.T + (size_t)g * TT * TSTR;
              const float* A = TAg + (size_t)(v & (TA - 1)) * TSTR;
              const float* B = TAg + (size_t)(TA + (v >> p.K1)) * TSTR;
              sy_ = A[ys] + B[ys];
              for (int c = 0; c < nc; ++c) {
                const float s = A[c] + B[c];
                if (c != ys) m2 = fmaxf(m2, s);
              }
            } else {
              const float* Pg = Pbase(g, fl);
              const int ps = Pstride(fl);
              for (int c = 0; c < nc; ++c) {
                float s = 0.f;
                for (uint32_t a = v; a; a &= a - 1) s += Pg[(size_t)(__ffs(a) - 1) * ps + c];
                if (c == ys) sy_ = s; else m2 = fmaxf(m2, s);
              }
            }
            if (m2 > sy_ * (1.f + p.band)) {
              oka = 0;
            } else if (m2 < sy_ * (1.f - p.band)) {
              oka = 1;
            } else {
              // fp64 recheck over the candidates within the band (rare)
              atomicAdd(p.n_recheck + (v - 1), 1ull);
              const int64_t n = n0 + g;
              const int32_t* Cg = (fl & F_OVF) ? p.scratch_cls + ((size_t)blockIdx.x * G + g) * (size_t)C
                                               : sm.ccls + (size_t)g * p.CAP;
              const float* Pg = Pbase(g, fl);
              const int ps = Pstride(fl);
              const float lo = sy_ * (1.f - p.band);
              double best = -1.0;
              int bestc = 0x7fffffff;
              const int nv = __popc(v);
              for (int c = 0; c < nc; ++c) {
                float s32 = 0.f;
                if (fl & F_TABLES) {
                  const float* TAg = sm.T + (size_t)g * TT * TSTR;
                  s32 = TAg[(size_t)(v & (TA - 1)) * TSTR + c] + TAg[(size_t)(TA + (v >> p.K1)) * TSTR + c];
                } else {
                  for (uint32_t a = v; a; a &= a - 1) s32 += Pg[(size_t)(__ffs(a) - 1) * ps + c];
                }
                if (c != ys && s32 < lo) continue;
                const int cls = Cg[c];
                double s = 0.0;
                for (uint32_t a = v; a; a &= a - 1) {
                  const int m = __ffs(a) - 1;
                  double L = sm.lse64[g * K + m];
                  if (isnan(L)) {
                    L = row_lse64(p.logits + (n * K + m) * p.ldc, C);
                    sm.lse64[g * K + m] = L;  // benign race: every writer stores the same value
                  }
                  s += exp((double)p.logits[(n * K + m) * p.ldc + cls] - L);
                }
                const double a64 = s / (double)nv;
                if (a64 > best || (a64 == best && cls < bestc)) { best = a64; bestc = cls; }
              }
              oka = (bestc == y);
            }
          }
        }
        if (G == 1) {  // exclusive ownership: pair index == v-1
          sm.grpcnt[v - 1] += okv;
          sm.cta_avg[v - 1] += oka;
        } else {
          // register slot counters; i < NIMAX guaranteed by the host
#pragma unroll
          for (int q = 0; q < NIMAX; ++q)
            if (q == i) { slot_vote[q] += okv; slot_avg[q] += oka; }
        }
        if (okv && sm.stail[g]) {
          const uint32_t tm = sm.stail[g];
          for (int bi = 0; bi < p.nB; ++bi)
            if ((tm >> bi) & 1u) atomicAdd(p.tail + (size_t)bi * S + (v - 1), 1ull);
        }
      }
    }  // tiles of the unit

    // ---- unit end: fold slot counters into group counts, write groups, CTA totals ----------------
    __syncthreads();
    if (G > 1) {
      const int GS = G * S;
#pragma unroll
      for (int q = 0; q < NIMAX; ++q) {
        const int pidx = t + q * kVoteThreads;
        if (pidx < GS) {
          const int g = pidx / S;
          const int v1 = pidx - g * S;
          const int grp = (p.gs > 0 && G > p.gs) ? g / p.gs : 0;
          if (slot_vote[q]) atomicAdd(&sm.grpcnt[grp * S + v1], slot_vote[q]);
          if (slot_avg[q]) atomicAdd(&sm.cta_avg[v1], slot_avg[q]);
        }
        slot_vote[q] = 0;
        slot_avg[q] = 0;
      }
      __syncthreads();
    }
    {
      uint32_t unisum = 0;
      for (int q = 0; q < NGU; ++q) unisum += sm.uni[q];
      const int64_t ngroups_total = p.gs > 0 ? (N + p.gs - 1) / p.gs : 0;
      for (int v1 = t; v1 < S; v1 += kVoteThreads) {
        uint32_t tot = 0;
        for (int q = 0; q < NGU; ++q) {
          const uint32_t val = sm.grpcnt[q * S + v1] + sm.uni[q];
          tot += val;
          sm.grpcnt[q * S + v1] = 0;
          if (p.grp) {
            const int64_t gi = unit * NGU + q;
            if (gi < ngroups_total) p.grp[gi * S + v1] = (uint8_t)val;
          }
        }
        sm.cta_vote[v1] += tot;
        sm.cta_avg[v1] += unisum;
      }
      __syncthreads();
      for (int q = t; q < NGU; q += kVoteThreads) sm.uni[q] = 0;
    }
  }  // units

  __syncthreads();
  for (int v1 = t; v1 < S; v1 += kVoteThreads) {
    if (sm.cta_vote[v1]) atomicAdd(p.cnt_vote + v1, (unsigned long long)sm.cta_vote[v1]);
    if (sm.cta_avg[v1]) atomicAdd(p.cnt_avg + v1, (unsigned long long)sm.cta_avg[v1]);
  }
}

template <int VPL, int RP, bool STATS>
cudaError_t launch_t(const VoteParams& p, const VoteLayout& L, cudaStream_t st) {
  auto k = vote_kernel<VPL, RP, STATS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
  if (e != cudaSuccess) return e;
  k<<<L.grid, kVoteThreads, L.smem, st>>>(p);
  return cudaGetLastError();
}

template <bool STATS>
cudaError_t launch_s(const VoteParams& p, const VoteLayout& L, cudaStream_t st) {
  const int key = L.VPL * 10 + L.RP;
  switch (key) {
    case 11: return launch_t<1, 1, STATS>(p, L, st);
    case 12: return launch_t<1, 2, STATS>(p, L, st);
    case 21: return launch_t<2, 1, STATS>(p, L, st);
    case 22: return launch_t<2, 2, STATS>(p, L, st);
    case 41: return launch_t<4, 1, STATS>(p, L, st);
    case 42: return launch_t<4, 2, STATS>(p, L, st);
    case 81: return launch_t<8, 1, STATS>(p, L, st);
    case 82: return launch_t<8, 2, STATS>(p, L, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

size_t vote_smem_bytes(const VoteParams& p) { return carve(p, nullptr, nullptr); }
size_t vote_slot_bytes(const VoteParams& p) { return al128(4 * tile_floats(p)); }

static int pow2ceil(int x) { int r = 1; while (r < x) r <<= 1; return r; }

VoteLayout choose_vote_layout(int K, int C, int ldc, int gs, int sm_count) {
  VoteLayout best{};
  double best_score = -1.0;
  const int F = ldc / 4;
  const int S = (1 << K) - 1;
  for (int LPR = 32; LPR >= 1; LPR >>= 1) {
    const int VPL = pow2ceil((F + LPR - 1) / LPR);
    if (VPL > 8) continue;
    const int RS = kVoteThreads / LPR;
    for (int RP = 1; RP <= 2; ++RP) {
      int G = 1;
      while (G * 2 * K <= RS * RP && G * 2 <= 64) G *= 2;
      if (G * K > RS * RP) continue;  // one sample must fit
      while (G > 1 && G * S > 4 * kVoteThreads) G >>= 1;  // register slot counters limit
      while (G > 1 && (size_t)G * K * ldc * 4 > 24 * 1024) G >>= 1;  // ring slot size
      const double util = double(G * K) / double(RS * RP);
      const double lane_util = double(F) / double(LPR * VPL);
      // prefer utilisation, then fewer registers, then wide rows (coalescing)
      const double score = util * lane_util * 1000.0 - VPL * RP * 1.0 + LPR * 0.01;
      if (score > best_score) {
        best_score = score;
        best.LPR = LPR; best.VPL = VPL; best.RP = RP; best.RS = RS; best.G = G; best.NV = VPL * RP;
      }
    }
  }
  (void)gs;
  best.grid = sm_count;
  return best;
}

cudaError_t launch_vote(const VoteParams& p, const VoteLayout& L, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  return p.lse_in ? launch_s<true>(p, L, st) : launch_s<false>(p, L, st);
}

// ---- rk_predict: per-sample outputs of one action v (plain, one warp per sample) -------------------
__global__ void predict_kernel(const PredictParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int K = p.K, C = p.C;
  for (int64_t n = warp; n < p.N; n += nwarps) {
    int top[kMaxK];
    float lse[kMaxK];
    for (int m = 0; m < K; ++m) {
      const float* row = p.logits + (n * K + m) * p.ldc;
      float mx = -INFINITY;
      int arg = 0x7fffffff;
      for (int c = lane; c < C; c += 32) {
        const float x = row[c];
        if (x > mx) { mx = x; arg = c; }
      }
      for (int off = 16; off; off >>= 1) {
        const float om = __shfl_xor_sync(FULL, mx, off);
        const int oa = __shfl_xor_sync(FULL, arg, off);
        if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
      }
      float s = 0.f;
      for (int c = lane; c < C; c += 32) s += __expf(row[c] - mx);
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
      top[m] = arg;
      lse[m] = p.lse_in ? p.lse_in[n * K + m] : mx + logf(s);
    }
    // vote
    if (p.pred_vote && lane == 0) {
      int bestc = -1, bestcnt = 0;
      uint32_t tied = 0;
      for (int m = 0; m < K; ++m) {
        if (!((p.v >> m) & 1u)) continue;
        uint32_t mk = 0;
        for (int q = 0; q < K; ++q)
          if (((p.v >> q) & 1u) && top[q] == top[m]) mk |= 1u << q;
        const int cnt = __popc(mk);
        if (cnt > bestcnt || (cnt == bestcnt && top[m] < bestc)) { bestcnt = cnt; bestc = top[m]; }
      }
      for (int m = 0; m < K; ++m) {
        if (!((p.v >> m) & 1u)) continue;
        uint32_t mk = 0;
        for (int q = 0; q < K; ++q)
          if (((p.v >> q) & 1u) && top[q] == top[m]) mk |= 1u << q;
        if (__popc(mk) == bestcnt) tied |= 1u << m;
      }
      p.pred_vote[n] = p.tie == 0 ? top[p.best_of[tied]] : bestc;
    }
    // average (fp32 probabilities; lowest class on ties)
    if (p.pred_avg || p.avgprob) {
      const float inv = 1.f / (float)__popc(p.v);
      float bm = -1.f;
      int bc = 0x7fffffff;
      for (int c = lane; c < C; c += 32) {
        float s = 0.f;
        for (int m = 0; m < K; ++m)
          if ((p.v >> m) & 1u) s += expf(p.logits[(n * K + m) * p.ldc + c] - lse[m]);
        const float a = s * inv;
        if (p.avgprob) p.avgprob[n * C + c] = a;
        if (a > bm) { bm = a; bc = c; }
      }
      for (int off = 16; off; off >>= 1) {
        const float om = __shfl_xor_sync(FULL, bm, off);
        const int oc = __shfl_xor_sync(FULL, bc, off);
        if (om > bm || (om == bm && oc < bc)) { bm = om; bc = oc; }
      }
      if (p.pred_avg && lane == 0) p.pred_avg[n] = bc;
    }
  }
}

cudaError_t launch_predict(const PredictParams& p, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  int64_t blocks = (p.N + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  predict_kernel<<<(int)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rk
