// FP64 FMA throughput of the B200 (the 3D stencils' second roofline; SURVEY §7
// "FP64 peak is not measured in MEASURED_PEAKS.json; measure it").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
// 8 independent DFMA chains per thread, 148 x 8 CTAs of 256 threads; timed with
// CUDA events after a warm-up launch; prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keep the chains alive
}

int main() {
  double *out;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int blocks = 148 * 8, threads = 256, iters = 1 << 16;
  dfma_loop<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fmas = (double)blocks * threads * iters * 8;
  printf("{\"kernel\": \"dfma_loop\", \"ms\": %.4f, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, "
         "\"dfma_per_clk_per_sm_at_1965MHz\": %.2f}\n",
         best, fmas / (best * 1e-3), 2.0 * fmas / (best * 1e-3) / 1e12,
         fmas / (best * 1e-3) / (148.0 * 1.965e9));
  return cudaGetLastError() != cudaSuccess;
}
