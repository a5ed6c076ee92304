// Measured FP32 peak of this B200 (the flop side of the per-step roofline,
// "P_fp32 is not in MEASURED_PEAKS; measure it with an
// FFMA-chain microbenchmark").
//
// Every thread runs 16 independent FFMA chains (enough to cover the 4-cycle
// FMA latency at any occupancy), grid = 148 SMs x 8 CTAs x 256 threads.  Flops
// counted as 2 per FFMA; CUDA events around the launch, best of 10 after a
// warm-up.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak scripts/probes/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 16;

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const int threads = 256, blocks = sms * 8, iters = 1 << 16;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_ffma<<<blocks, threads>>>(out, iters, 0.999999f, 1e-6f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, iters, 0.999999f, 1e-6f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    fprintf(stderr, "fp32_peak: %s\n", cudaGetErrorString(err));
    return 1;
  }
  const double flops = 2.0 * kChains * (double)iters * threads * blocks;
  const double tf = flops / (best * 1e-3) / 1e12;
  // nominal: 128 FP32 lanes x 2 flops per SM per clock
  const double nominal = 2.0 * 128 * sms * (clk_khz * 1e3) / 1e12;
  printf("{\"fp32_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"clock_mhz_attr\": %.0f, "
         "\"nominal_tflops_at_attr_clock\": %.3f, \"frac_of_nominal\": %.4f, "
         "\"how\": \"%d independent FFMA chains/thread, %d CTAs x %d threads x %d iters, "
         "2 flops/FFMA, best of 10 (CUDA events)\"}\n",
         tf, best, sms, clk_khz / 1e3, nominal, tf / nominal, kChains, blocks, threads, iters);
  return 0;
}
