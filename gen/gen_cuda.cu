// gen_cuda.cu — device-side fill of the synthetic inputs defined in rk_gen.h (bit-identical to
// gen_host.c). Used by the GPU tests and bench.py to create full-size inputs in HBM quickly.
// Holds no method arithmetic; not part of librk.so.
#include <cuda_runtime.h>
#include <math.h>
#include "rk_gen.h"

__global__ void k_labels(uint64_t seed, int64_t n0, int64_t n, int C, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rkg_label(seed, n0 + i, C);
}

__global__ void k_logits(uint64_t seed, int64_t n0, int64_t n, int K, int C, int ldc, int64_t mu0, int64_t dmu,
                         const int32_t* labels, float* out) {
  const int64_t per = (int64_t)K * ldc;
  const int64_t total = n * per;
  rkg_logit_params prm = {mu0, dmu};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = i / per;
    int r = (int)(i - s * per);
    int m = r / ldc, c = r - m * ldc;
    int y = labels ? labels[s] : rkg_label(seed, n0 + s, C);
    out[i] = c < C ? rkg_logit(seed, n0 + s, m, c, K, y, prm) : __int_as_float(0x7fc00000);
  }
}

__global__ void k_x(uint64_t seed, int64_t n0, int64_t n, int D, int C, uint32_t psig, int real,
                    const int32_t* labels, uint16_t* out) {
  const int64_t total = n * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = i / D;
    int d = (int)(i - s * D);
    int y = labels ? labels[s] : rkg_label(seed, n0 + s, C);
    out[i] = real ? rkg_x_real(seed, n0 + s, d, y, psig) : rkg_int_to_bf16(rkg_x_int(seed, n0 + s, d, y, psig));
  }
}

static int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return (int)(g > 148 * 64 ? 148 * 64 : (g < 1 ? 1 : g));
}

extern "C" {
int rkg_dev_fill_labels(uint64_t seed, int64_t n0, int64_t n, int C, int32_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  k_labels<<<grid_for(n), 256, 0, st>>>(seed, n0, n, C, out);
  return (int)cudaGetLastError();
}
int rkg_dev_fill_logits(uint64_t seed, int64_t n0, int64_t n, int K, int C, int ldc, int64_t mu0_q24, int64_t dmu_q24,
                        const int32_t* labels, float* out, cudaStream_t st) {
  if (n <= 0) return 0;
  k_logits<<<grid_for(n * K * ldc), 256, 0, st>>>(seed, n0, n, K, C, ldc, mu0_q24, dmu_q24, labels, out);
  return (int)cudaGetLastError();
}
int rkg_dev_fill_x(uint64_t seed, int64_t n0, int64_t n, int D, int C, uint32_t psig_q16, int real,
                   const int32_t* labels, uint16_t* out, cudaStream_t st) {
  if (n <= 0) return 0;
  k_x<<<grid_for(n * D), 256, 0, st>>>(seed, n0, n, D, C, psig_q16, real, labels, out);
  return (int)cudaGetLastError();
}
}
