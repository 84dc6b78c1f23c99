// FP64 (DFMA) peak of this GPU, measured: the denominator of the FD
// gradient's FP64 roofline (bench.py "fp64_roofline"; MEASURED_PEAKS.json has
// no FP64 figure).  Every thread runs 8 independent DFMA chains (enough ILP to
// cover the DFMA latency at full occupancy) for ITERS iterations; grid = SMs x
// 8 CTAs of 256 threads.  FLOP = 2 per DFMA.  Best of 10 launches, CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak            -> one JSON line
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) k_dfma(double *out, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double *out;
  cudaMalloc(&out, 8);
  const int grid = nsm * 8, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma<<<grid, block>>>(out, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<grid, block>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flop = 2.0 * CHAINS * ITERS * (double)grid * block;
  const double tf = flop / (best * 1e-3) / 1e12;
  const double per_sm_clk = flop / 2.0 / (best * 1e-3) / nsm / (clk * 1e3);
  printf("{\"fp64_tflops\": %.3f, \"dfma_per_sm_per_clk_at_max_clock\": %.2f, \"ms\": %.4f, "
         "\"sms\": %d, \"max_clock_mhz\": %.0f, \"how\": \"%d CTAs x %d threads, %d independent "
         "DFMA chains x %d iterations per thread, best of 10, CUDA events\"}\n",
         tf, per_sm_clk, best, nsm, clk / 1e3, grid, block, CHAINS, ITERS);
  return cudaGetLastError() != cudaSuccess;
}
