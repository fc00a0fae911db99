// FP32 pipe microbenchmark: independent FADD / FFMA chains per thread (B200).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OPK>
__global__ void __launch_bounds__(256) chains(float* sink, float seed, int iters) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; k++) a[k] = seed + threadIdx.x * 1e-7f + k;
  const float m = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      if (OPK == 0) a[k] = __fadd_rn(a[k], c);
      else if (OPK == 1) a[k] = __fmaf_rn(a[k], m, c);
      else a[k] = __fmul_rn(a[k], m);
    }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += a[k];
  if (s == 12345.f) sink[0] = s;
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, blocks = sms * 8;
  const char* names[3] = {"FADD", "FFMA", "FMUL"};
  for (int op = 0; op < 3; op++) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a);
      if (op == 0) chains<0><<<blocks, 256>>>(sink, 1.f, iters);
      else if (op == 1) chains<1><<<blocks, 256>>>(sink, 1.f, iters);
      else chains<2><<<blocks, 256>>>(sink, 1.f, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double instr = (double)blocks * 256 * iters * 8;
    printf("%s %.2f T instr/s (%.1f ms)\n", names[op], instr / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}
