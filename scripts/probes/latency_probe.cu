// Per-step floor of a dependent kernel chain on B200: CUDA graph of K launches,
// with and without programmatic dependent launch, empty vs. load/store 4096 envs.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
}

__global__ void k_copy(float* s, int n, int rows, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = r < rows ? s[r * n + i] : 0.f;
#pragma unroll
  for (int r = 0; r < 32; ++r)
    if (r < rows) s[r * n + i] = v[r] * 1.0001f + 1e-7f;
}

template <typename F>
float chain(F launch, cudaStream_t st, int K) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < K; ++k) launch();
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best * 1000.f / K;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int n = 4096, K = 1000;
  float* buf;
  cudaMalloc(&buf, sizeof(float) * n * 32);
  cudaMemset(buf, 0, sizeof(float) * n * 32);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    auto mk = [&](dim3 g) {
      cudaLaunchConfig_t c = {};
      c.gridDim = g;
      c.blockDim = dim3(128);
      c.stream = st;
      c.attrs = attr;
      c.numAttrs = pdl ? 1 : 0;
      return c;
    };
    float e1 = chain([&] { auto c = mk(dim3(1)); cudaLaunchKernelEx(&c, k_empty, pdl); }, st, K);
    float e32 = chain([&] { auto c = mk(dim3(32)); cudaLaunchKernelEx(&c, k_empty, pdl); }, st, K);
    float c19 = chain([&] { auto c = mk(dim3(32)); cudaLaunchKernelEx(&c, k_copy, buf, n, 19, pdl); }, st, K);
    float c25 = chain([&] { auto c = mk(dim3(32)); cudaLaunchKernelEx(&c, k_copy, buf, n, 25, pdl); }, st, K);
    printf("pdl=%d empty(1 CTA) %.2f us  empty(32 CTA) %.2f us  copy19 %.2f us  copy25 %.2f us\n",
           pdl, e1, e32, c19, c25);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
