/* rk_gen.h — seeded, counter-based synthetic input generators.
 *
 * This module is shared by the CPU oracle (oracle/) and by the GPU test/bench
 * harness. It holds NONE of the method's arithmetic (no argmax, softmax, vote,
 * average, counting or reward): it only turns (seed, index) into input values.
 * Every value is produced with integer arithmetic and ONE exact-or-RNE
 * integer->float conversion, so host and device generate bit-identical arrays.
 *
 * Workloads (recipe stated in DESIGN.md "Input recipe"):
 *  - labels y_n uniform in [0,C)                     (ImageNet-val shape)
 *  - logits  (SURVEY.md §8(d) formula, dyadic version):
 *      logit[n][m][c] = 3*( 15/16 g[n][c] + 5/16 h[n][m][c]
 *                           + [c==y_n]*(mu_m + 7/8 u[n] + 7/16 e[n][m]) )
 *      g,h,u,e ~ Irwin-Hall(4) "normals" (variance 1.02), mu_m = mu0 + dmu*(K-1-m)
 *      (shared class noise g and shared difficulty u make errors correlated across
 *       models, the same idea as SPEC.md:551)
 *  - GEMM features / weights for the synthetic dense heads (int mode: values in
 *    {-1,0,1}, so fp32 accumulation is exact; real mode: non-integer bf16).
 */
#ifndef RK_GEN_H
#define RK_GEN_H
#include <stdint.h>

#if defined(__CUDACC__)
#define RKG_FN static __host__ __device__ __forceinline__
#else
#define RKG_FN static inline
#endif

/* SplitMix64 finalizer. */
RKG_FN uint64_t rkg_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* Counter-based hash of (seed, tag, a, b). */
RKG_FN uint64_t rkg_hash(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  return rkg_mix64(rkg_mix64(rkg_mix64(seed ^ (tag * 0xD1B54A32D192ED03ull)) ^ a) + b);
}
/* Irwin-Hall(4) integer: sum of four 16-bit fields minus their mean, in [-131070,131070].
 * The unit normal it stands for is z * 7 / 2^18 (variance 7^2/2^36 * 4*(2^32-1)/12 ~ 1.02). */
RKG_FN int64_t rkg_ih4(uint64_t h) {
  return (int64_t)(h & 0xffff) + (int64_t)((h >> 16) & 0xffff) + (int64_t)((h >> 32) & 0xffff) +
         (int64_t)(h >> 48) - 131070;
}
/* Uniform integer in [0, n) by multiply-shift of the high 32 bits. */
RKG_FN uint32_t rkg_below(uint64_t h, uint32_t n) {
  return (uint32_t)(((h >> 32) * (uint64_t)n) >> 32);
}

enum { RKG_TAG_LABEL = 1, RKG_TAG_G = 2, RKG_TAG_H = 3, RKG_TAG_U = 4, RKG_TAG_E = 5,
       RKG_TAG_PROTO = 10, RKG_TAG_FLIP = 11, RKG_TAG_X = 12, RKG_TAG_XR = 13, RKG_TAG_WR = 14,
       RKG_TAG_BIAS = 15 };

RKG_FN int32_t rkg_label(uint64_t seed, int64_t n, int C) {
  return (int32_t)rkg_below(rkg_hash(seed, RKG_TAG_LABEL, (uint64_t)n, 0), (uint32_t)C);
}

/* Logit parameters in units of 2^-24 (mu0, dmu are dyadic). */
typedef struct { int64_t mu0_q24; int64_t dmu_q24; } rkg_logit_params;

/* One logit value. Integer numerator in units of 2^-24, times 3, converted once (RNE). */
RKG_FN float rkg_logit(uint64_t seed, int64_t n, int m, int c, int K, int y, rkg_logit_params prm) {
  int64_t num = 420 * rkg_ih4(rkg_hash(seed, RKG_TAG_G, (uint64_t)n, (uint64_t)c)) +
                140 * rkg_ih4(rkg_hash(seed, RKG_TAG_H, (uint64_t)n, ((uint64_t)m << 32) | (uint64_t)c));
  if (c == y) {
    num += prm.mu0_q24 + prm.dmu_q24 * (int64_t)(K - 1 - m) +
           392 * rkg_ih4(rkg_hash(seed, RKG_TAG_U, (uint64_t)n, 0)) +
           196 * rkg_ih4(rkg_hash(seed, RKG_TAG_E, (uint64_t)n, (uint64_t)m));
  }
  /* |3*num| < 2^31; int64 -> float rounds to nearest even; * 2^-24 is exact. */
  return (float)(3 * num) * 5.9604644775390625e-08f;
}

/* ---- GEMM inputs (synthetic dense classifier heads) ----------------------------------
 * Class prototype mu_c[d] = +-1. Model m's head row W[m][c][d] = mu_c[d], sign-flipped with
 * probability flip_q16(m)/65536 (worse models flip more). Feature X[n][d] = mu_{y_n}[d] with
 * probability psig_q16/65536, else uniform in {-1,0,1}. Int mode returns these integers;
 * real mode perturbs them by Irwin-Hall noise (non-integer bf16 values). */
/* The class prototypes are a fixed property of the synthetic "world" (shared by every X and
 * W seed), so features and heads drawn with different seeds still agree on what class c is. */
#define RKG_WORLD_SEED 0x5EEDull
RKG_FN int rkg_proto(uint64_t seed, int c, int d) {
  (void)seed;
  return (rkg_hash(RKG_WORLD_SEED, RKG_TAG_PROTO, (uint64_t)c, (uint64_t)d) >> 63) ? 1 : -1;
}
RKG_FN int rkg_w_int(uint64_t seed, int m, int c, int d, uint32_t flip_q16) {
  int p = rkg_proto(seed, c, d);
  uint32_t r = (uint32_t)(rkg_hash(seed, RKG_TAG_FLIP, ((uint64_t)m << 32) | (uint64_t)c, (uint64_t)d) & 0xffff);
  return r < flip_q16 ? -p : p;
}
/* psig_q16 packs two probabilities (units of 1/65536): bits 0..15 = P(prototype-matched dim);
 * bits 16..31 = P(noise dim is +-1) -- 0 keeps the original uniform {-1, 0, 1} noise. A sparser noise
 * lowers the spread of the wrong-class logits at the same signal, i.e. a softer softmax for a given
 * accuracy (the calibration knob between the power-of-two logit scales). */
RKG_FN int rkg_x_int(uint64_t seed, int64_t n, int d, int y, uint32_t psig_q16) {
  uint64_t h = rkg_hash(seed, RKG_TAG_X, (uint64_t)n, (uint64_t)d);
  if ((uint32_t)(h & 0xffff) < (psig_q16 & 0xffffu)) return rkg_proto(seed, y, d);
  const uint32_t pnz = psig_q16 >> 16;
  if (pnz == 0) return (int)rkg_below(h, 3) - 1;
  if ((uint32_t)((h >> 16) & 0xffff) >= pnz) return 0;
  return (h >> 63) ? 1 : -1;
}
/* float -> bf16 bits, round to nearest even (inputs are finite). */
RKG_FN uint16_t rkg_f32_to_bf16(float f) {
  union { float f; uint32_t u; } v; v.f = f;
  uint32_t u = v.u;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
RKG_FN uint16_t rkg_int_to_bf16(int v) { return rkg_f32_to_bf16((float)v); }
/* Real mode: x = 3/4*x_int + 1/2*z, w = w_int + 1/4*z (z: Irwin-Hall unit normal), rounded to bf16. */
RKG_FN uint16_t rkg_x_real(uint64_t seed, int64_t n, int d, int y, uint32_t psig_q16) {
  int64_t z = rkg_ih4(rkg_hash(seed, RKG_TAG_XR, (uint64_t)n, (uint64_t)d));
  /* value = 0.75*xi + 0.5*z*7/2^18, exact in fp32 (|num| < 2^24 in units of 2^-19) */
  int64_t num = (int64_t)rkg_x_int(seed, n, d, y, psig_q16) * 393216 + z * 7;
  return rkg_f32_to_bf16((float)num * 1.9073486328125e-06f);
}
RKG_FN uint16_t rkg_w_real(uint64_t seed, int m, int c, int d, uint32_t flip_q16) {
  int64_t z = rkg_ih4(rkg_hash(seed, RKG_TAG_WR, ((uint64_t)m << 32) | (uint64_t)c, (uint64_t)d));
  /* value = wi + 0.25*z*7/2^18 in units of 2^-20 */
  int64_t num = (int64_t)rkg_w_int(seed, m, c, d, flip_q16) * 1048576 + z * 7;
  return rkg_f32_to_bf16((float)num * 9.5367431640625e-07f);
}
/* Bias: int mode small integers in [-2,2]; real mode dyadic z/16. */
RKG_FN float rkg_bias(uint64_t seed, int m, int c, int real_mode) {
  uint64_t h = rkg_hash(seed, RKG_TAG_BIAS, (uint64_t)m, (uint64_t)c);
  if (!real_mode) return (float)((int)rkg_below(h, 5) - 2);
  return (float)(rkg_ih4(h) * 7) * 2.384185791015625e-07f; /* z*7/2^18 / 16 */
}
/* Default per-model flip probability: worse models (higher m) flip more. */
RKG_FN uint32_t rkg_flip_q16(int m, uint32_t flip0_q16, uint32_t dflip_q16) {
  return flip0_q16 + dflip_q16 * (uint32_t)m;
}
#endif
