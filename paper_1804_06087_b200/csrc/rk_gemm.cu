// rk_gemm.cu — step A1 (+A2 fused): K synthetic dense classifier heads on the 5th-generation
// tensor cores, with the per-(row, model) softmax normaliser and top-1 fused in the epilogue.
//
//   logit[n][m][c] = 2^s * sum_d X[n][d] * W[m][c][d] + bias[m][c]
//   top1[n][m]     = lowest c attaining max_c logit          (reading Q4)
//   rmax[n][m]     = max_c logit[n][m][c]
//   lsum[n][m]     = log sum_c exp(logit[n][m][c] - rmax[n][m])  (softmax normaliser, PAPER.md:72;
//                    relative to the max so p = exp((l - rmax) - lsum) stays exact for any offset)
// The heads stand in for the classifier layer of the paper's ConvNets (the
// inference time "depends on the model complexity, hardware efficiency ... and the batch size",
// PAPER.md:361).
//
// sm_100a design:
//   * persistent, one CTA per SM, 6 warps: warp 0 = TMA producer, warp 1 = tcgen05.mma issuer and
//     TMEM owner, warps 2-5 = epilogue (TMEM lane quarter = warp % 4).
//   * default: CTA pairs (cluster of 2) computing 256 rows x up to 256 columns of ONE model with
//     tcgen05.mma.cta_group::2 (each CTA stages its 128 X rows and half of the W tile; 6-stage
//     32 KB smem ring fed by TMA); single-CTA variant: 128 x 256 tiles, 4-stage 48 KB ring.
//     K-block 64, 128-byte swizzle, cp.async.bulk.tensor + mbarrier complete_tx.
//   * fp32 accumulators in TMEM, double-buffered (2 x 256 columns) so the epilogue of tile i
//     overlaps the MMAs of tile i+1.
//   * a work unit is (128-row block (CL rows blocks for a pair), model): the CTA walks the model's column tiles in ascending
//     order, so the epilogue keeps an ONLINE max / lowest-index argmax / rescaled sum-exp per row
//     in registers and writes top1/lsum/rmax once per unit; logits leave through swizzled smem staging
//     and TMA bulk tensor stores (rows >= N and columns >= C are clipped by the tensor map).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "rk_internal.h"

namespace rk {
namespace {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB: this CTA's 128 rows of X
constexpr int EPI_WARPS = 4;
constexpr int STG_BYTES = 32 * 32 * 4;  // one 32x32 fp32 staging box (packed mode: two 32x16 boxes)
#ifndef RK_EPI_PACK
#define RK_EPI_PACK 12
#endif
constexpr int EPI_PACK = RK_EPI_PACK;    // packed mode: EPI_PACK / 4 epilogue warps per TMEM lane quarter
constexpr int NHP = EPI_PACK / 4;
static_assert(EPI_PACK == 8 || EPI_PACK == 12 || EPI_PACK == 16, "packed epilogue: 2, 3 or 4 warps per lane quarter");
constexpr int XCH_BYTES = 4 * 32 * 12;   // (max, sum, argmax) hand-over per quarter and partner part
// CL = 1: one CTA computes a 128 x 256 tile (W tile 256 rows in its smem, 4 stages of 48 KB).
// CL = 2: a CTA pair computes a 256 x 256 tile with tcgen05.mma.cta_group::2 (M = 256): each CTA
// holds its 128 X rows and HALF of the W tile (128 rows), 6 stages of 32 KB.
// FUSED (NEXT-3): 8 epilogue warps (two per TMEM lane quarter, alternate 16-column halves of each chunk);
// the staging region holds the per-thread candidate queues ([16 entries][256 threads] values and classes)
// and a per-quarter hand-over of (max, sum, argmax, l_y, flag, T values, T classes) per row.
constexpr int FUSED_EPI = 8;
constexpr int XF = 6 + 2 * kFuseT;  // words per row in the fused hand-over
// Fused epilogue: a thread starts each row of a model with the threshold it ended its previous row of that
// model at, minus a margin (the 16th-largest logit varies little between rows, std ~0.45 at c4): only the
// elements above it are inserted into the top-T list instead of ~16 + 16 ln(504/16). A list left short
// (fewer than T elements above the threshold) is completed by a bound entry (class kFuseNone, value = the
// threshold: every unlisted class lies at or below it) and the next row's threshold backs off. Margins
// 1.5 / 0.75 / 0.25 / 0.1 measured fused GEMM 21.1 / 20.6 / 19.9-20.2 / 19.9 ms per 1M with the fallback
// fraction 3.623 / 3.624 / 3.635 / 3.659 %; 0.25 is the default.
#ifndef RK_T0_MARGIN
#define RK_T0_MARGIN 0.25f
#endif
#ifndef RK_T0_BACKOFF
#define RK_T0_BACKOFF (2.0f * RK_T0_MARGIN)
#endif
constexpr float kT0Margin = RK_T0_MARGIN, kT0Backoff = RK_T0_BACKOFF;
template <int CL, bool PACK = false, bool FUSED = false>
struct Tile {
  static constexpr int B_ROWS = BN / CL;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // packed mode with 3 or 4 warps per quarter: EPI_PACK x 4 KB of store staging
  static constexpr bool WIDE = (PACK && NHP >= 3) || FUSED;
#ifndef RK_GEMM_NS
#define RK_GEMM_NS 6
#endif
  static constexpr int STG_TOTAL = FUSED ? 16 * 256 * 8 : (WIDE ? EPI_PACK * 2 * (32 * 16 * 4) : EPI_WARPS * 2 * STG_BYTES);
  static constexpr int XCH_TOTAL = FUSED ? 4 * 32 * XF * 4 : XCH_BYTES * (PACK ? NHP - 1 : 1);
  // operand stages: as many as the remaining shared memory holds (<= RK_GEMM_NS): 6 for the per-model
  // CTA-pair tile, 5 (3 warps per quarter) or 4 (4 warps) for the packed one, 4 / 3 single-CTA
  static constexpr int NS_FIT = (232448 - 1024 - STG_TOTAL - 256 - XCH_TOTAL) / STAGE_BYTES;
  static constexpr int NS = NS_FIT < RK_GEMM_NS ? NS_FIT : RK_GEMM_NS;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + NS * STAGE_BYTES + STG_TOTAL + 256 + XCH_TOTAL;
};
static_assert(RK_GEMM_NS < 6 || (Tile<2>::NS == 6 && Tile<1>::NS == 4 && Tile<2, false, true>::NS == 5 &&
                                 Tile<1, false, true>::NS == 3 && Tile<2, true>::NS == (NHP == 4 ? 4 : NHP == 3 ? 5 : 6)),
              "operand stages of each tile shape");
template <bool PACK, bool FUSED>
__host__ __device__ constexpr int epi_warps() { return PACK ? EPI_PACK : (FUSED ? FUSED_EPI : EPI_WARPS); }
static_assert(Tile<1>::SMEM_BYTES <= 232448 && Tile<2>::SMEM_BYTES <= 232448 && Tile<1, true>::SMEM_BYTES <= 232448 &&
                  Tile<2, true>::SMEM_BYTES <= 232448 && Tile<1, false, true>::SMEM_BYTES <= 232448 &&
                  Tile<2, false, true>::SMEM_BYTES <= 232448,
              "smem");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// Logits leave with an L2 evict-first policy: the 32 GB output stream must not evict the X / W
// operand tiles that other CTAs are about to re-read from L2.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                             uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
                   map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::f16, A/B = BF16, D = F32, both K-major, M = m (128, or 256 for a pair), N = n.
__device__ __forceinline__ uint32_t umma_idesc(int n, int m) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2 (what __expf uses after its multiply)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kL2E = 1.4426950408889634f;
constexpr float kLN2 = 0.6931471805599453f;
// Sum-exp bookkeeping that stays exact relative to the row max for ANY logit offset: the terms are
// 2^(l*L2E + nml(mx)) with nml(mx) = rnd(-mx*L2E) (one FFMA each); a new running max rescales the sum by
// 2^(nml(new) - nml(old)) (the same rounded values the terms used, so no |mx|-sized error enters); at the
// end ln sum_c exp(l - mx) = ln(sum) - d*ln2 with d = mx*L2E + nml(mx), the rounding residual of nml,
// which one FMA yields exactly. (Using exp(mx_old - mx_new) for the rescale, or ignoring d, would
// leave an error of about |mx| * 2^-24 in the normaliser -- 1e-3 relative at |logits| ~ 1e4.)
__device__ __forceinline__ float nml_of(float mx) { return __fmul_rn(-mx, kL2E); }
__device__ __forceinline__ float rescale_factor(float mx_old, float mx_new) {
  return ex2_approx(nml_of(mx_new) - nml_of(mx_old));  // mx_old = -inf -> 2^-inf = 0
}
__device__ __forceinline__ float lsum_of(float sum, float mx) {
  return logf(sum) - fmaf(mx, kL2E, nml_of(mx)) * kLN2;
}
// Sum of one chunk's terms as a 4-way tree of partial sums, added to the row's running sum once per chunk:
// a C-column row then sees ~n/4 + 2 + C/n roundings on any path instead of C (recursive summation), which
// keeps lsum within ~1e-6 of the fp64 value for the 1000-class rows (the fp32 averaging band is 2e-5).
template <int NV>
__device__ __forceinline__ float chunk_sum(const float* v, float nml) {
  float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < NV; ++i) p[i & 3] += ex2_approx(fmaf(v[i], kL2E, nml));
  return (p[0] + p[1]) + (p[2] + p[3]);
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[32]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
#pragma unroll
  for (int i = 16; i < 32; ++i) v[i] = -INFINITY;
}

struct GemmArgs {
  int64_t N;
  int K, C, Cp, D, nt, scale_log2;
  int ng, gcols;  // work-unit column groups: K groups of Cp columns, or (packed) 1 group of K*Cp
  const float* bias;
  int32_t* top1;
  float* lsum;
  float* rmax;
  float* rs2;  // [N][K] second-largest logit (non-packed, non-fused epilogue; null = not written)
  // fused forward + vote (NEXT-3; FUSED instantiation): labels [N]; outputs the label's logit ly [N][K]
  // and the top-kFuseT logits per (row, model), values tv [N][K][T] (descending) and classes ti [N][K][T]
  const int32_t* labels;
  float* ly;
  float* tv;
  uint16_t* ti;
};

// CTA-pair (cta_group::2) forms. The TMA load lands in this CTA's shared memory but signals the
// LEADER CTA's mbarrier (shared::cluster address from mapa), so the leader's full barrier counts
// the bytes of both halves; the MMA commit arrives on the same barrier offset in both CTAs.
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {  // arrives on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// CL = 1: one CTA per work unit (128 rows, model). CL = 2: a CTA pair (cluster of 2 on one TPC)
// per work unit (256 rows, model) with tcgen05.mma.cta_group::2: the leader (rank 0) issues M = 256
// MMAs reading A (128 rows) and half of B (N/2 rows of W) from EACH CTA's shared memory, so every
// operand byte crosses L2 -> smem once per pair instead of once per CTA (B traffic halved, smem
// stage 32 KB instead of 48 KB -> 6 stages). Each CTA's TMEM receives its own 128 rows x N
// accumulator and its epilogue is unchanged.
// Accumulator stage `as` drained by this epilogue warp. CL = 1: one arrive per warp. CL = 2: the pair's
// barrier lives in the leader, whose MMAs refill both CTAs' TMEM: the leader's warps arrive locally, the
// peer's warps meet at a named barrier and ONE thread arrives remotely (release.cluster arrives are
// costly: one per warp and tile was 20 % of the packed epilogue's stall samples).
template <int CL, int EPI>
__device__ __forceinline__ void release_tmem_stage(uint64_t* tempty, uint32_t as, int crank, int lane) {
  tc_fence_before();
  __syncwarp();
  if (CL == 1 || crank == 0) {
    if (lane == 0) mbar_arrive(&tempty[as]);
  } else {
    asm volatile("bar.sync 12, %0;" ::"n"(EPI * 32) : "memory");
    if (threadIdx.x == 64) mbar_arrive_cluster(map_to_rank(smem_u32(&tempty[as]), 0));  // first epilogue thread
  }
}

// Packed-mode epilogue (see gemm_heads_kernel): 16-column blocks of the flattened column space; the
// two warps of a TMEM lane quarter (half h) take alternating blocks and keep per-model online
// (max, lowest argmax, sum-exp); at each model boundary half 1 hands its part to half 0 (named
// barrier per quarter), which merges and writes top1/lsum/max. Logits leave through a 32-row x
// 16-column staging box (64-byte rows, 16-byte chunks XOR (row >> 1) & 3: the 64B TMA swizzle)
// and a 3-D TMA store (class, model, row).
template <int CL>
__device__ __forceinline__ void epilogue_packed(const GemmArgs& a, const CUtensorMap& tmo16, uint64_t* tfull,
                                                uint64_t* tempty, uint32_t tmem_base, int q, int h, int lane,
                                                uint8_t* stg, float* xch, int64_t ucl0, int64_t units, int64_t ucls,
                                                int crank, float scale, uint64_t store_policy) {
  constexpr int SBOX = 32 * 16 * 4;
  uint32_t tc = 0, nstore = 0, nclose = 0;
  const int row_in_tile = q * 32 + lane;
  float* xb = xch + q * 96 * (NHP - 1);
  for (int64_t u = ucl0; u < units; u += ucls) {
    const int mt = (int)(u / a.ng) * CL + crank;
    const int64_t row = (int64_t)mt * BM + row_in_tile;
    float mx = -INFINITY, sum = 0.f;
    int arg = 0x7fffffff, cur = -1;
    auto close = [&](int m) {  // every part calls this at the same model boundaries
      if (m < 0) return;
      constexpr int NT = 32 * NHP;  // threads of the quarter's warps (named barriers 1+q, 5+q)
      if (h > 0) {
        if (nclose > 0) asm volatile("bar.sync %0, %1;" ::"r"(5 + q), "n"(NT) : "memory");  // part 0 read the last one
        float* xs = xb + (h - 1) * 96;
        xs[lane] = mx; xs[32 + lane] = sum; xs[64 + lane] = __int_as_float(arg);
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "n"(NT) : "memory");
      if (h == 0) {
        float mk[NHP - 1], sk[NHP - 1];
        int ak[NHP - 1];
#pragma unroll
        for (int k = 0; k < NHP - 1; ++k) {
          mk[k] = xb[k * 96 + lane]; sk[k] = xb[k * 96 + 32 + lane]; ak[k] = __float_as_int(xb[k * 96 + 64 + lane]);
        }
        asm volatile("bar.arrive %0, %1;" ::"r"(5 + q), "n"(NT) : "memory");
        float M = mx;
        int A = arg;
#pragma unroll
        for (int k = 0; k < NHP - 1; ++k) {  // the lowest column among the parts' maxima (Q4)
          if (mk[k] > M) { M = mk[k]; A = ak[k]; }
          else if (mk[k] == M && ak[k] < A) A = ak[k];
        }
        float S = 0.f;  // every part's sum moved to the base nml(M) (see rescale_factor)
        if (mx != -INFINITY) S += sum * rescale_factor(mx, M);
#pragma unroll
        for (int k = 0; k < NHP - 1; ++k)
          if (mk[k] != -INFINITY) S += sk[k] * rescale_factor(mk[k], M);
        if (row < a.N) {
          a.top1[row * a.K + m] = A;
          a.lsum[row * a.K + m] = lsum_of(S, M);  // log-sum relative to the row max (exact p below)
          a.rmax[row * a.K + m] = M;
        }
      }
      ++nclose;
    };
    uint32_t blk = 0;  // global 16-column block counter of this unit (dealt round-robin to the parts)
    // gc / Cp by a multiply-shift: with inv = ceil(2^20 / Cp), floor(gc * inv / 2^20) = floor(gc / Cp) for
    // gc < 2^12, Cp <= 128 (the error gc * (inv - 2^20 / Cp) / 2^20 < 1/256 is below the 1/Cp spacing)
    const uint32_t cp_inv = ((1u << 20) + (uint32_t)a.Cp - 1u) / (uint32_t)a.Cp;
    for (int j = 0; j < a.nt; ++j, ++tc) {
      const int width = min(BN, a.gcols - j * BN);
      const uint32_t as = tc & 1;
      mbar_wait(&tfull[as], (tc >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
      for (int c0 = 0; c0 < width; c0 += 16, ++blk) {
        const int gc = j * BN + c0;
        const int model = (int)(((uint32_t)gc * cp_inv) >> 20), cm = gc - model * a.Cp;
        if (model != cur) {  // first block of the next model: close the previous one
          close(cur);
          mx = -INFINITY; sum = 0.f; arg = 0x7fffffff; cur = model;
        }
        if ((int)(blk % NHP) != h) continue;
        float v[32];
        tmem_ld16(tbase + c0, v);
        const float4* bptr = reinterpret_cast<const float4*>(a.bias + (size_t)model * a.Cp + cm);
        float cmax = -INFINITY;
        int carg = 0;
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {
          const float4 b4 = __ldg(bptr + i4);  // -inf on padding columns
          const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) v[4 * i4 + e] = fmaf(v[4 * i4 + e], scale, bb[e]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) cmax = fmaxf(cmax, v[i]);
        if (cmax > mx) {  // new running max of this model: its lowest column (Q4)
#pragma unroll
          for (int i = 15; i >= 0; --i) carg = v[i] == cmax ? cm + i : carg;
          sum = sum * rescale_factor(mx, cmax);
          mx = cmax;
          arg = carg;
        }
        if (mx != -INFINITY) {
          const float nml = nml_of(mx);
          sum += chunk_sum<16>(v, nml);
        }
        uint8_t* buf = stg + (nstore & 1) * SBOX;
        if (lane == 0 && nstore >= 2) tma_store_wait_read1();
        __syncwarp();
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int phys = c4 ^ ((lane >> 1) & 3);
          *reinterpret_cast<float4*>(buf + lane * 64 + phys * 16) =
              make_float4(v[c4 * 4], v[c4 * 4 + 1], v[c4 * 4 + 2], v[c4 * 4 + 3]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&tmo16, buf, cm, model, (int)(mt * BM + q * 32), store_policy);
          tma_store_commit();
        }
        ++nstore;
      }
      release_tmem_stage<CL, EPI_PACK>(tempty, as, crank, lane);
    }
    close(cur);
  }
  if (lane == 0) tma_store_wait_all();
  __syncwarp();
}

// PACK (Cp <= 128): a work unit covers ALL K models -- the tiles walk the flattened [K*Cp] column
// space, so each X tile is staged once per 256 columns instead of once per model; the epilogue works
// in 16-column blocks (each inside one model, Cp % 16 == 0) and closes a model's online statistics
// when the next model's first block arrives.
// Fused epilogue (NEXT-3, FUSED instantiation, per-model column tiles). The two warps of a TMEM lane
// quarter (half h) take the alternate 16-column halves of every 32-column chunk; per row each keeps the
// online (max, lowest argmax, sum-exp) of its columns, the label's logit if it sees column y, and a
// descending list of its kFuseT largest logits: a chunk's candidates (above the list's last value) are
// queued per thread in shared memory in column order and inserted by a compare-exchange chain, so the
// warp iterates the longest queue of its lanes instead of every column some lane needs. At the unit end
// half 1 hands its part to half 0 (named barriers per quarter), which merges statistics and lists and
// writes top1 / lsum / rmax / l_y / the top-T values and classes. No logits are stored.
__device__ __forceinline__ void topk_insert(float (&tv)[kFuseT], int (&ti)[kFuseT], float cv, int cc) {
#pragma unroll
  for (int t = 0; t < kFuseT; ++t) {
    const bool sw = cv > tv[t];
    const float t1 = tv[t];
    const int t2 = ti[t];
    tv[t] = sw ? cv : t1;
    ti[t] = sw ? cc : t2;
    cv = sw ? t1 : cv;
    cc = sw ? t2 : cc;
  }
}

template <int CL>
__device__ __forceinline__ void epilogue_fused(const GemmArgs& a, uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                                               int q, int h, int lane, uint8_t* staging, float* xch, int64_t ucl0,
                                               int64_t units, int64_t ucls, int crank, float scale) {
  uint32_t tc = 0, nunit = 0;
  const int row_in_tile = q * 32 + lane;
  const int tid = h * 128 + row_in_tile;  // queue column (256 epilogue threads)
  float* qv = reinterpret_cast<float*>(staging);
  int* qc = reinterpret_cast<int*>(staging + 16 * 256 * 4);
  float* xb = xch + q * 32 * XF;          // hand-over of this quarter: [XF][32]
  constexpr int NT = 64;                  // threads of the quarter's two warps (named barriers 1+q, 5+q)
  float t0m[8];                           // carried starting threshold per model (K <= 8 on this path)
#pragma unroll
  for (int k = 0; k < 8; ++k) t0m[k] = -INFINITY;
  for (int64_t u = ucl0; u < units; u += ucls, ++nunit) {
    const int mt = (int)(u / a.ng) * CL + crank, model = (int)(u % a.ng);
    const int64_t row = (int64_t)mt * BM + row_in_tile;
    const int yl = row < a.N ? a.labels[row] : -1;
    float mx = -INFINITY, sum = 0.f, lyv = 0.f;
    int arg = 0x7fffffff, lyset = 0;
    float thr0 = -INFINITY;
#pragma unroll
    for (int k = 0; k < 8; ++k) thr0 = k == model ? t0m[k] : thr0;
    float tv[kFuseT];
    int ti[kFuseT];
#pragma unroll
    for (int k = 0; k < kFuseT; ++k) { tv[k] = -INFINITY; ti[k] = kFuseNone; }
    for (int j = 0; j < a.nt; ++j, ++tc) {
      const int width = min(BN, a.Cp - j * BN);
      const uint32_t as = tc & 1;
      mbar_wait(&tfull[as], (tc >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
      for (int c0 = 16 * h; c0 < width; c0 += 32) {
        float v[32];
        tmem_ld16(tbase + c0, v);
        const int colbase = j * BN + c0;
        const float4* bptr = reinterpret_cast<const float4*>(a.bias + (size_t)model * a.Cp + colbase);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) {  // Cp % 16 == 0: the 16 columns are inside the model
          const float4 b4 = __ldg(bptr + i4);
          const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) v[4 * i4 + e] = fmaf(v[4 * i4 + e], scale, bb[e]);
        }
        float cmax = -INFINITY;
#pragma unroll
        for (int i = 0; i < 16; ++i) cmax = fmaxf(cmax, v[i]);
        if (cmax > mx) {
          int carg = 0;
#pragma unroll
          for (int i = 15; i >= 0; --i) carg = v[i] == cmax ? colbase + i : carg;
          sum = sum * rescale_factor(mx, cmax);
          mx = cmax;
          arg = carg;
        }
        if (mx != -INFINITY) sum += chunk_sum<16>(v, nml_of(mx));
        const int yo = yl - colbase;
        if (yo >= 0 && yo < 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) lyv = (i == yo) ? v[i] : lyv;
          lyset = 1;
        }
        const float thr = fmaxf(tv[kFuseT - 1], thr0);
        int qn = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (v[i] > thr) { qv[qn * 256 + tid] = v[i]; qc[qn * 256 + tid] = colbase + i; ++qn; }
        const int qmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)qn);
        for (int k = 0; k < qmax; ++k)
          if (k < qn) topk_insert(tv, ti, qv[k * 256 + tid], qc[k * 256 + tid]);
        __syncwarp();
      }
      release_tmem_stage<CL, FUSED_EPI>(tempty, as, crank, lane);
    }
    // this half's unlisted elements are <= hb (its 16th value, or its threshold when the list is short)
    const bool short_h = !(tv[kFuseT - 1] > -INFINITY);
    const float hb = short_h ? thr0 : -INFINITY;
    {
      const float nt0 = short_h ? thr0 - kT0Backoff : tv[kFuseT - 1] - kT0Margin;
#pragma unroll
      for (int k = 0; k < 8; ++k) t0m[k] = k == model ? nt0 : t0m[k];
    }
    // merge the two halves of the row
    if (h == 1) {
      if (nunit > 0) asm volatile("bar.sync %0, %1;" ::"r"(5 + q), "n"(NT) : "memory");  // half 0 read the last one
      xb[0 * 32 + lane] = mx; xb[1 * 32 + lane] = sum; xb[2 * 32 + lane] = __int_as_float(arg);
      xb[3 * 32 + lane] = lyv; xb[4 * 32 + lane] = __int_as_float(lyset);
      xb[(5 + 2 * kFuseT) * 32 + lane] = hb;
#pragma unroll
      for (int k = 0; k < kFuseT; ++k) {
        xb[(5 + k) * 32 + lane] = tv[k];
        xb[(5 + kFuseT + k) * 32 + lane] = __int_as_float(ti[k]);
      }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "n"(NT) : "memory");
    if (h == 0) {
      const float m1 = xb[lane], s1 = xb[32 + lane];
      const int a1 = __float_as_int(xb[64 + lane]);
      const float ly1 = xb[96 + lane];
      const int set1 = __float_as_int(xb[128 + lane]);
      float M = mx;
      int A = arg;
      if (m1 > M) { M = m1; A = a1; }
      else if (m1 == M && a1 < A) A = a1;
      float S = 0.f;
      if (mx != -INFINITY) S += sum * rescale_factor(mx, M);
      if (m1 != -INFINITY) S += s1 * rescale_factor(m1, M);
      if (set1) lyv = ly1;
#pragma unroll
      for (int k = 0; k < kFuseT; ++k) {
        const float cv = xb[(5 + k) * 32 + lane];
        if (cv > tv[kFuseT - 1]) topk_insert(tv, ti, cv, __float_as_int(xb[(5 + kFuseT + k) * 32 + lane]));
      }
      // bound for every unlisted class: the merged 16th value, or a short half's threshold if higher; the
      // last slot then carries it as a bound-only entry (a listed 16th value below it becomes unlisted)
      const float bnd = fmaxf(hb, xb[(5 + 2 * kFuseT) * 32 + lane]);
      if (!(tv[kFuseT - 1] >= bnd)) { tv[kFuseT - 1] = bnd; ti[kFuseT - 1] = kFuseNone; }
      asm volatile("bar.arrive %0, %1;" ::"r"(5 + q), "n"(NT) : "memory");
      if (row < a.N) {
        const size_t o = (size_t)row * a.K + model;
        a.top1[o] = A;
        a.lsum[o] = lsum_of(S, M);
        a.rmax[o] = M;
        a.ly[o] = lyv;
        float4* tv4 = reinterpret_cast<float4*>(a.tv + o * kFuseT);
#pragma unroll
        for (int k = 0; k < kFuseT / 4; ++k) tv4[k] = make_float4(tv[4 * k], tv[4 * k + 1], tv[4 * k + 2], tv[4 * k + 3]);
        uint4* ti4 = reinterpret_cast<uint4*>(a.ti + o * kFuseT);
#pragma unroll
        for (int k = 0; k < kFuseT / 8; ++k)
          ti4[k] = make_uint4((uint32_t)ti[8 * k] | ((uint32_t)ti[8 * k + 1] << 16),
                              (uint32_t)ti[8 * k + 2] | ((uint32_t)ti[8 * k + 3] << 16),
                              (uint32_t)ti[8 * k + 4] | ((uint32_t)ti[8 * k + 5] << 16),
                              (uint32_t)ti[8 * k + 6] | ((uint32_t)ti[8 * k + 7] << 16));
      }
    }
  }
}

template <int CL, bool PACK, bool FUSED = false>
__global__ void __launch_bounds__(64 + 32 * epi_warps<PACK, FUSED>(), 1)
    gemm_heads_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                      const __grid_constant__ CUtensorMap tmo, const __grid_constant__ CUtensorMap tmo16,
                      const GemmArgs a) {
  using T = Tile<CL, PACK, FUSED>;
  constexpr int NS = T::NS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stages = smem;
  uint8_t* staging = smem + NS * T::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + T::STG_TOTAL);
  uint64_t* full = bars;            // [NS]  (CL = 2: only the leader's are waited on)
  uint64_t* empty = bars + NS;      // [NS]
  uint64_t* tfull = bars + 2 * NS;  // [2]
  uint64_t* tempty = bars + 2 * NS + 2;  // [2]  (CL = 2: the leader's counts both epilogues)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 4);
  float* xch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [4][NHP-1][3][32] (packed)
  constexpr int EPI = epi_warps<PACK, FUSED>();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mtiles = (a.N + BM - 1) / BM;
  // work unit = (group of CL adjacent row tiles, model); CTA `crank` of the pair takes row tile
  // CL * (u / K) + crank. Both CTAs of a pair walk the same unit sequence.
  const int64_t units = ((mtiles + CL - 1) / CL) * a.ng;
  const int64_t ucl0 = blockIdx.x / CL, ucls = gridDim.x / CL;
  const int crank = CL > 1 ? (int)cluster_rank() : 0;
  const int kblocks = a.D / BK;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], CL == 1 ? EPI : EPI + 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmx) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmw) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmo) : "memory");
    if (PACK) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmo16) : "memory");
  }
  if (warp == 1) {  // CL = 2: both CTAs allocate collectively (same warp id, same smem slot)
    if (CL == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CL > 1) cluster_sync_all();  // both CTAs' barriers and TMEM exist before any cross-CTA signal
  __syncthreads();  // (CL = 2: implied by the cluster barrier; explicit so racecheck sees the ordering of
                    // the tcgen05.alloc write of tmem_slot before its reads)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer (both CTAs of a pair: each loads its own A rows and its half of B) =====
    if (lane == 0) {
      // W (re-read by every row block) is kept in L2 against the 32 KB/sample logits stream:
      // measured -18% GEMM DRAM reads (ncu, N = 65,536), time unchanged
      const uint64_t pol_w = policy_evict_last();
      const uint64_t pol_x = policy_evict_normal();
      uint32_t it = 0;
      for (int64_t u = ucl0; u < units; u += ucls) {
        const int mt = (int)(u / a.ng) * CL + crank, grp = (int)(u % a.ng);
        for (int j = 0; j < a.nt; ++j) {
          const int width = min(BN, a.gcols - j * BN);
          const int col0 = grp * a.gcols + j * BN + crank * (width / CL);
          for (int kb = 0; kb < kblocks; ++kb, ++it) {
            const int s = it % NS;
            const uint32_t ph = (it / NS) & 1;
            mbar_wait(&empty[s], ph ^ 1);  // the MMAs that read stage s are complete
            uint8_t* sa = stages + s * T::STAGE_BYTES;
            uint8_t* sb = sa + A_BYTES;
            if (CL == 1) {
              mbar_expect_tx(&full[s], T::STAGE_BYTES);
              tma_load_2d(sa, &tmx, &full[s], kb * BK, mt * BM);
              tma_load_2d(sb, &tmw, &full[s], kb * BK, col0);
            } else {
              const uint32_t lbar = map_to_rank(smem_u32(&full[s]), 0);
              if (crank == 0) mbar_expect_tx(&full[s], CL * T::STAGE_BYTES);  // both halves' bytes
              tma_load_2d_pair(sa, &tmx, lbar, kb * BK, mt * BM, pol_x);
              tma_load_2d_pair(sb, &tmw, lbar, kb * BK, col0, pol_w);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (CL = 2: leader only) =====
    if (lane == 0 && crank == 0) {
      uint32_t it = 0, tc = 0;
      for (int64_t u = ucl0; u < units; u += ucls) {
        for (int j = 0; j < a.nt; ++j, ++tc) {
          const int width = min(BN, a.gcols - j * BN);
          const uint32_t idesc = umma_idesc(width, BM * CL);
          const uint32_t as = tc & 1;
          mbar_wait(&tempty[as], ((tc >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dtm = tmem_base + as * BN;
          for (int kb = 0; kb < kblocks; ++kb, ++it) {
            const int s = it % NS;
            mbar_wait(&full[s], (it / NS) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(stages + s * T::STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // advance 16 bf16 = 32 bytes inside the 128-byte swizzle atom
              if (CL == 1) umma_bf16(dtm, umma_desc(sa + k * 32), umma_desc(sb + k * 32), idesc, (kb | k) ? 1u : 0u);
              else umma_bf16_pair(dtm, umma_desc(sa + k * 32), umma_desc(sb + k * 32), idesc, (kb | k) ? 1u : 0u);
            }
            // smem slot reusable once these MMAs complete (CL = 2: in both CTAs)
            if (CL == 1) umma_commit(&empty[s]);
            else umma_commit_pair(&empty[s]);
          }
          if (CL == 1) umma_commit(&tfull[as]);  // accumulator ready for the epilogue(s)
          else umma_commit_pair(&tfull[as]);
        }
      }
    }
  } else {
    // ===== epilogue: TMEM -> registers -> (stats, swizzled smem) -> TMA store =====
    const int q = warp & 3;  // TMEM lane quarter accessible by this warp
    const int row_in_tile = q * 32 + lane;
    uint8_t* stg = staging + (warp - 2) * (T::STG_TOTAL / EPI);
    const float scale = ldexpf(1.0f, a.scale_log2);
    const uint64_t store_policy = policy_evict_first();
    uint32_t tc = 0, nstore = 0;
    if (PACK) {
      epilogue_packed<CL>(a, tmo16, tfull, tempty, tmem_base, q, (warp - 2) >> 2, lane, stg, xch, ucl0, units, ucls,
                          crank, scale, store_policy);
    } else if (FUSED) {
      epilogue_fused<CL>(a, tfull, tempty, tmem_base, q, (warp - 2) >> 2, lane, staging, xch, ucl0, units, ucls, crank,
                         scale);
    } else
    for (int64_t u = ucl0; u < units; u += ucls) {
      const int mt = (int)(u / a.ng) * CL + crank, model = (int)(u % a.ng);
      const int64_t row = (int64_t)mt * BM + row_in_tile;
      float mx = -INFINITY, sum = 0.f, s2 = -INFINITY;  // s2: max over the row without one occurrence of mx
      int arg = 0;
      for (int j = 0; j < a.nt; ++j, ++tc) {
        const int width = min(BN, a.Cp - j * BN);
        const uint32_t as = tc & 1;
        mbar_wait(&tfull[as], (tc >> 1) & 1);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
        for (int c0 = 0; c0 < width; c0 += 32) {
          float v[32];
          if (width - c0 >= 32) tmem_ld32(tbase + c0, v);
          else tmem_ld16(tbase + c0, v);
          const int colbase = j * BN + c0;  // column inside the model
          const float4* bptr = reinterpret_cast<const float4*>(a.bias + (size_t)model * a.Cp + colbase);
          float cmax = -INFINITY;
          int carg = 0;
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {  // bias: -inf on padding columns; groups of 4 never straddle Cp
            const float4 b4 = colbase + 4 * i4 < a.Cp ? __ldg(bptr + i4)
                                                      : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) v[4 * i4 + e] = fmaf(v[4 * i4 + e], scale, bb[e]);  // exact product, one rounding
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) cmax = fmaxf(cmax, v[i]);
          if (cmax > mx) {  // new running max (rare after the first chunks): its lowest column (Q4)
#pragma unroll
            for (int i = 31; i >= 0; --i) carg = v[i] == cmax ? colbase + i : carg;
            float c2 = -INFINITY;  // this chunk's largest value other than the argmax position
#pragma unroll
            for (int i = 0; i < 32; ++i) c2 = fmaxf(c2, colbase + i == carg ? -INFINITY : v[i]);
            s2 = fmaxf(mx, c2);
            sum = sum * rescale_factor(mx, cmax);
            mx = cmax;
            arg = carg;
          } else {
            s2 = fmaxf(s2, cmax);
          }
          if (mx != -INFINITY) {
            const float nml = nml_of(mx);
            sum += chunk_sum<32>(v, nml);
          }
          // stage 32 rows x 32 cols (128B-swizzled) and store with TMA. (Coalesced st.global.cs
          // from the same staging box measured 18% slower for the whole kernel: DESIGN.md §6.)
          uint8_t* buf = stg + (nstore & 1) * STG_BYTES;
          if (lane == 0 && nstore >= 2) tma_store_wait_read1();
          __syncwarp();
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const int phys = c4 ^ (lane & 7);
            float4 w4 = make_float4(v[c4 * 4], v[c4 * 4 + 1], v[c4 * 4 + 2], v[c4 * 4 + 3]);
            *reinterpret_cast<float4*>(buf + lane * 128 + phys * 16) = w4;
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmo, buf, colbase, model, (int)(mt * BM + q * 32), store_policy);
            tma_store_commit();
          }
          ++nstore;
        }
        release_tmem_stage<CL, EPI_WARPS>(tempty, as, crank, lane);
      }
      if (row < a.N) {
        a.top1[row * a.K + model] = arg;
        a.lsum[row * a.K + model] = lsum_of(sum, mx);  // relative to the row max
        a.rmax[row * a.K + model] = mx;
        if (a.rs2) a.rs2[row * a.K + model] = s2;
      }
    }
    if (lane == 0) tma_store_wait_all();
    __syncwarp();
  }
  tc_fence_before();
  if (CL > 1) cluster_sync_all();  // no CTA leaves while a peer may still signal its barriers
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CL == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// ---- host: tensor maps through the driver entry point (no libcuda link dependency) -------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

}  // namespace

int gemm_build_tmaps(GemmParams& p, const void* X, const void* W, float* logits, void* storage) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return -1;
  CUtensorMap* maps = reinterpret_cast<CUtensorMap*>(storage);
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.D, (cuuint64_t)p.N};
    cuuint64_t strides[1] = {(cuuint64_t)p.D * 2};
    cuuint32_t box[2] = {BK, BM};
    cuuint32_t es[2] = {1, 1};
    if (enc(&maps[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -2;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.D, (cuuint64_t)p.K * p.Cp};
    cuuint64_t strides[1] = {(cuuint64_t)p.D * 2};
    cuuint32_t box[2] = {BK, (cuuint32_t)(BN / (p.cluster > 1 ? p.cluster : 1))};  // W tile (or its half)
    cuuint32_t es[2] = {1, 1};
    if (enc(&maps[1], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(W), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -3;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.C, (cuuint64_t)p.K, (cuuint64_t)p.N};
    cuuint64_t strides[2] = {(cuuint64_t)p.ldc * 4, (cuuint64_t)p.K * p.ldc * 4};
    cuuint32_t box[3] = {32, 1, 32};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&maps[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, logits, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -4;
  }
  {  // 16-column store boxes for the packed mode (64-byte rows, 64B swizzle)
    cuuint64_t dims[3] = {(cuuint64_t)p.C, (cuuint64_t)p.K, (cuuint64_t)p.N};
    cuuint64_t strides[2] = {(cuuint64_t)p.ldc * 4, (cuuint64_t)p.K * p.ldc * 4};
    cuuint32_t box[3] = {16, 1, 32};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&maps[3], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, logits, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -5;
  }
  p.tmap_x = &maps[0];
  p.tmap_w = &maps[1];
  p.tmap_out = &maps[2];
  p.tmap_out16 = &maps[3];
  return 0;
}

template <int CL, bool PACK, bool FUSED = false>
static cudaError_t launch_t(const GemmArgs& a, const GemmParams& p, int sm_count, cudaStream_t st) {
  const CUtensorMap& mx = *reinterpret_cast<const CUtensorMap*>(p.tmap_x);
  const CUtensorMap& mw = *reinterpret_cast<const CUtensorMap*>(p.tmap_w);
  const CUtensorMap& mo = *reinterpret_cast<const CUtensorMap*>(p.tmap_out);
  const CUtensorMap& m16 = *reinterpret_cast<const CUtensorMap*>(p.tmap_out16);
  cudaError_t e = cudaFuncSetAttribute(gemm_heads_kernel<CL, PACK, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Tile<CL, PACK, FUSED>::SMEM_BYTES);
#ifdef RK_CARVEOUT
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_heads_kernel<CL, PACK, FUSED>, cudaFuncAttributePreferredSharedMemoryCarveout, RK_CARVEOUT);
#endif
  if (e != cudaSuccess) return e;
  const int64_t units = ((p.N + CL * BM - 1) / (CL * BM)) * a.ng;
  if (CL == 1) {
    const int grid = (int)(units < sm_count ? units : sm_count);
    gemm_heads_kernel<CL, PACK, FUSED><<<grid, 64 + 32 * epi_warps<PACK, FUSED>(), Tile<CL, PACK, FUSED>::SMEM_BYTES, st>>>(
        mx, mw, mo, m16, a);
    return cudaGetLastError();
  }
  // CTA pairs: clusters of 2 (one CTA per SM)
  const int64_t clusters = units < sm_count / 2 ? units : sm_count / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * clusters));
  cfg.blockDim = dim3(64 + 32 * epi_warps<PACK, FUSED>());
  cfg.dynamicSmemBytes = Tile<CL, PACK, FUSED>::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, gemm_heads_kernel<CL, PACK, FUSED>, mx, mw, mo, m16, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmParams& p, int sm_count, cudaStream_t st) {
  if (p.N <= 0) return cudaSuccess;
  GemmArgs a;
  a.N = p.N; a.K = p.K; a.C = p.C; a.Cp = p.Cp; a.D = p.D;
  a.scale_log2 = p.scale_log2; a.bias = p.bias; a.top1 = p.top1; a.lsum = p.lsum; a.rmax = p.rmax; a.rs2 = p.rs2;
  a.labels = p.labels; a.ly = p.ly; a.tv = p.tv; a.ti = p.ti;
  const bool pack = p.Cp <= 128;  // small heads: tiles span several models
  a.ng = pack ? 1 : p.K;
  a.gcols = pack ? p.K * p.Cp : p.Cp;
  a.nt = (a.gcols + BN - 1) / BN;
  if (p.labels) {  // fused forward + vote (NEXT-3): per-model column tiles only
    if (pack) return cudaErrorInvalidValue;
    return p.cluster <= 1 ? launch_t<1, false, true>(a, p, sm_count, st) : launch_t<2, false, true>(a, p, sm_count, st);
  }
  if (p.cluster <= 1) return pack ? launch_t<1, true>(a, p, sm_count, st) : launch_t<1, false>(a, p, sm_count, st);
  return pack ? launch_t<2, true>(a, p, sm_count, st) : launch_t<2, false>(a, p, sm_count, st);
}

}  // namespace rk
