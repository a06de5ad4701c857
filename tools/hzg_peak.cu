// FP64 tensor-pipe (DMMA) peak, measured live by bench.py in the same GPU
// lease as the GSVD numbers it is the denominator for (built into
// paper_1909_00101_b200/_lib/libhzg_peak.so by build(); not on the solve path).
#include <cuda_runtime.h>

namespace {

__global__ void k_dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) d[t][0] = d[t][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

extern "C" {

// Sustained DMMA.8x8x4 throughput over about `seconds` of back-to-back
// launches (4 CTAs x 128 threads per SM); *tflops = 2*8*8*4 flops per warp
// instruction.  Returns 0 on success.
int hzg_fp64_peak(int device, double seconds, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int bs = 128, grid = sms * 4, iters = 1 << 16;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * grid * bs) != cudaSuccess) return 3;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dmma_loop<<<grid, bs>>>(out, iters);  // warm-up, also sizes the run
  cudaEventRecord(e0);
  k_dmma_loop<<<grid, bs>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  int reps = ms > 0 ? (int)(seconds * 1e3 / ms) : 1;
  if (reps < 1) reps = 1;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_dmma_loop<<<grid, bs>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)grid * bs / 32.0;
  const double flops = (double)reps * warps * iters * 8 * (2.0 * 8 * 8 * 4);
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaError_t e = cudaGetLastError();
  cudaFree(out);
  return e == cudaSuccess ? 0 : 3;
}

}  // extern "C"
