// FP64 FMA throughput microbenchmark (SURVEY §8d "FP64 check": the measured FP64 peak the
// force and pair kernels are compared with, to show the ALU bound is not the binding one).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
// Prints one JSON line: dense DFMA rate (2 flop per FMA), best of 5, CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * kChains * kIters * (double)threads * blocks;
  std::printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"sm_clock_mhz_attr\": %d, \"ms\": %.4f, "
              "\"how\": \"%d independent DFMA chains x %d iterations per thread, %d x %d threads, best of 5\"}\n",
              flops / (best * 1e-3) / 1e12, sms, clk / 1000, best, kChains, kIters, blocks, threads);
  return 0;
}
