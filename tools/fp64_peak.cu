// FP64 pipe peak on this GPU: DFMA, DMUL and DADD
// throughput with enough independent chains per thread to cover the pipe
// latency, every SM busy.  Writes one JSON object to stdout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/_build/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int OP>
__global__ void k_fp64(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) x[c] = fma(x[c], a, b);          // DFMA: 2 flops
      else if (OP == 1) x[c] = x[c] * a;            // DMUL
      else x[c] = x[c] + b;                         // DADD
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;  // keep the chains alive
}

template <int OP>
double run(int blocks, int threads, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64<OP><<<blocks, threads>>>(d, 0.999999, 1e-9);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_fp64<OP><<<blocks, threads>>>(d, 0.999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 5.0 * blocks * threads * static_cast<double>(kIters) * kChains;
  return ops / (ms * 1e-3);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* d = nullptr;
  cudaMalloc(&d, sizeof(double));
  const int threads = 256, blocks = sms * 8;
  const double fma_ops = run<0>(blocks, threads, d);
  const double mul_ops = run<1>(blocks, threads, d);
  const double add_ops = run<2>(blocks, threads, d);
  std::printf("{\"sms\": %d, \"clock_khz\": %d, \"dfma_per_s\": %.6e, \"dmul_per_s\": %.6e, \"dadd_per_s\": %.6e, "
              "\"fp64_tflops_fma\": %.4f, \"fp64_tflops_nofma\": %.4f, \"dfma_per_clk_per_sm\": %.2f}\n",
              sms, clk, fma_ops, mul_ops, add_ops, 2.0 * fma_ops / 1e12, add_ops / 1e12,
              fma_ops / (static_cast<double>(clk) * 1e3 * sms));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
