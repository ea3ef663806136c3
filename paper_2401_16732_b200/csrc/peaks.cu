// peaks.cu — integer-pipe micro-benchmarks that define the roofline
// denominators MEASURED_PEAKS.json does not carry:
//   * mad.wide.s32 (IMAD.WIDE) issue rate — the K1 conv inner operation
//   * register-resident Harvey/Shoup forward butterfly rate — the K2 NTT op
// Both run register-resident (no memory traffic) with many independent
// chains per thread; bench.py times them with CUDA events.
#include "common.cuh"

namespace fhe {

__global__ void peak_imad_wide_kernel(int iters, long long* sink) {
  long long acc[16];
  int w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    acc[j] = j;
    w[j] = (int)(threadIdx.x * 7 + j * 131) - 1000;
  }
  int d = (int)(blockIdx.x * 977 + threadIdx.x);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] += (long long)w[j] * d;  // IMAD.WIDE
    d = (int)__byte_perm((unsigned)d, (unsigned)d, 0x0321);     // non-affine step
  }
  long long s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s ^= acc[j];
  if (s == 0x5eed) sink[0] = s;
}

__global__ void peak_butterfly_kernel(int iters, uint64_t q, uint64_t w, uint64_t wp, uint64_t* sink) {
  uint64_t x[8], y[8];
  const uint64_t q2 = 2 * q;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = (threadIdx.x * 1315423911ull + j) % q;
    y[j] = (blockIdx.x * 2654435761ull + 7 * j) % q;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint64_t X = x[j] >= q2 ? x[j] - q2 : x[j];
      const uint64_t T = shoup_lazy(y[j], w, wp, q);
      x[j] = X + T;
      y[j] = X - T + q2;
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s ^= x[j] ^ y[j];
  if (s == 0x5eed) sink[0] = s;
}

}  // namespace fhe

using namespace fhe;

extern "C" {

int fhe_peak_imad_wide(int blocks, int threads, int iters, int64_t* sink, void* stream) {
  if (blocks < 1 || threads < 1 || iters < 1 || !sink) return fail(FHE_ERR_VALUE, "bad peak arguments");
  peak_imad_wide_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, (long long*)sink);
  FHE_CHECK_LAUNCH("peak_imad_wide_kernel");
  return FHE_OK;
}

int fhe_peak_butterfly(int blocks, int threads, int iters, uint64_t q, uint64_t* sink, void* stream) {
  if (blocks < 1 || threads < 1 || iters < 1 || !sink || q < 3 || q >= (1ull << 62))
    return fail(FHE_ERR_VALUE, "bad peak arguments");
  const uint64_t w = q / 3 + 1;
  peak_butterfly_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, q, w, h_shoup(w, q), sink);
  FHE_CHECK_LAUNCH("peak_butterfly_kernel");
  return FHE_OK;
}

}  // extern "C"
