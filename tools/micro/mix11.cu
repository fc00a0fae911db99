// 1:1 read/write-mix streaming microbenchmark (B200): NI f64 planes in, NO planes out, one
// CTA per 256*U vectors (the lean elementwise design), varying
//   VB  bytes per vector: 16 (LDG.128) or 32 (LDG.256)
//   U   vectors per plane per thread, all loads issued before any math
//   OP  0 = lane-wise add (free arithmetic), 12 = the vtsqrt1 core (tf_math.cuh)
// Question (round 2 session 5): the 16-byte one-vector-per-thread conversion kernels
// stream a 1:1 mix at 7.0 TB/s while the 32-byte lean kernels (vmem copy, vtsqrt1) sit
// at 6.86-6.93 — is finer per-thread granularity the better design at this mix?
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 -fmad=false \
//          -prec-div=true -prec-sqrt=true mix11.cu -o mix11
#include <cuda_runtime.h>

#include "../../paper_1401_6235_b200/csrc/tf_math.cuh"

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

template <int VB>
struct alignas(VB) Vec {
  double v[VB / 8];
};
__device__ __forceinline__ Vec<32> ldg(const Vec<32>* p) {
  Vec<32> r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
               : "l"(p));
  return r;
}
__device__ __forceinline__ Vec<16> ldg(const Vec<16>* p) {
  Vec<16> r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.v[0]), "=d"(r.v[1])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(Vec<32>* p, const Vec<32>& r) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]),
               "d"(r.v[2]), "d"(r.v[3])
               : "memory");
}
__device__ __forceinline__ void stg(Vec<16>* p, const Vec<16>& r) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]) : "memory");
}

template <int NI, int NO>
struct Args {
  const double* in[NI];
  double* out[NO];
};

template <int OP, int NI, int NO, int VB, int U, int MINB, int TPB = 256>
__global__ void __launch_bounds__(TPB, MINB) k(Args<NI, NO> a, int64_t nvec) {
  using V = Vec<VB>;
  constexpr int E = VB / 8;
  const int64_t base = (int64_t)blockIdx.x * (TPB * U) + threadIdx.x;
  V r[U][NI];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t j = base + u * TPB;
    if (j < nvec) {
#pragma unroll
      for (int q = 0; q < NI; q++) r[u][q] = ldg(reinterpret_cast<const V*>(a.in[q]) + j);
    }
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t j = base + u * TPB;
    if (j < nvec) {
      V o[NO];
#pragma unroll
      for (int e = 0; e < E; e++) {
        if constexpr (OP == 0) {
          double s = 0;
#pragma unroll
          for (int q = 0; q < NI; q++) s += r[u][q].v[e];
#pragma unroll
          for (int q = 0; q < NO; q++) o[q].v[e] = s;
        } else {
          double v[NI];
#pragma unroll
          for (int q = 0; q < NI; q++) v[q] = r[u][q].v[e];
          tf::P<double> z = tf::apply<double, OP>(v);
          o[0].v[e] = z.a;
          o[1].v[e] = z.b;
        }
      }
#pragma unroll
      for (int q = 0; q < NO; q++) stg(reinterpret_cast<V*>(a.out[q]) + j, o[q]);
    }
  }
}

static double* buf[6];
static int64_t N;

template <int OP, int NI, int NO, int VB, int U, int MINB, int TPB = 256>
static void run(const char* name) {
  Args<NI, NO> a;
  for (int q = 0; q < NI; q++) a.in[q] = buf[q];
  for (int q = 0; q < NO; q++) a.out[q] = buf[NI + q];
  const int64_t nvec = N / (VB / 8);
  const int64_t blocks = (nvec + TPB * U - 1) / (TPB * U);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k<OP, NI, NO, VB, U, MINB, TPB>);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<OP, NI, NO, VB, U, MINB, TPB>, TPB, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<OP, NI, NO, VB, U, MINB, TPB><<<(unsigned)blocks, TPB>>>(a, nvec);
  std::vector<float> ts;
  for (int i = 0; i < 15; i++) {
    cudaEventRecord(e0);
    k<OP, NI, NO, VB, U, MINB, TPB><<<(unsigned)blocks, TPB>>>(a, nvec);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  const double bytes = (double)(NI + NO) * N * 8;
  printf("%-28s regs %3d  ctas/sm %d  median %.4f ms  %.0f GB/s  best %.0f GB/s  (%s)\n", name,
         fa.numRegs, occ, ts[ts.size() / 2], bytes / ts[ts.size() / 2] / 1e6, bytes / ts[0] / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  if (cudaDeviceSynchronize() != cudaSuccess) exit(2);
}

int main(int argc, char** argv) {
  N = 1ll << (argc > 1 ? atoi(argv[1]) : 28);
  for (int q = 0; q < 6; q++) {
    if (cudaMalloc(&buf[q], N * 8) != cudaSuccess) {
      printf("cudaMalloc failed\n");
      return 1;
    }
    std::vector<double> h(1 << 20);
    for (size_t i = 0; i < h.size(); i++) h[i] = 1.0 + (double)((i * 2654435761u) % 1000003) / 1e6;
    for (int64_t off = 0; off < N; off += (int64_t)h.size())
      cudaMemcpy(buf[q] + off, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  }
  // tails plane: small relative to heads (vtsqrt1 input error plane)
  if (argc > 2) {  // threads per CTA for the light 16-byte design (session 5)
    for (int rep = 0; rep < 3; rep++) {
      printf("-- threads per CTA, VB16 U1\n");
      run<0, 4, 2, 16, 1, 8, 256>("add 4/2 tpb256 (8 CTAs)");
      run<0, 4, 2, 16, 1, 4, 512>("add 4/2 tpb512 (4 CTAs)");
      run<0, 4, 2, 16, 1, 16, 128>("add 4/2 tpb128 (16 CTAs)");
      run<0, 4, 2, 16, 1, 2, 1024>("add 4/2 tpb1024 (2 CTAs)");
      run<12, 2, 2, 16, 1, 8, 256>("vtsqrt1 tpb256 (8 CTAs)");
      run<12, 2, 2, 16, 1, 4, 512>("vtsqrt1 tpb512 (4 CTAs)");
      run<12, 2, 2, 16, 1, 16, 128>("vtsqrt1 tpb128 (16 CTAs)");
      run<12, 2, 2, 16, 1, 2, 1024>("vtsqrt1 tpb1024 (2 CTAs)");
      run<3, 4, 2, 16, 1, 5, 256>("vtdiv2 tpb256 (5 CTAs)");
      run<3, 4, 2, 16, 1, 2, 512>("vtdiv2 tpb512 (2 CTAs)");
      run<3, 4, 2, 16, 1, 10, 128>("vtdiv2 tpb128 (10 CTAs)");
    }
    return 0;
  }
  for (int rep = 0; rep < 2; rep++) {
    printf("-- copy 1 in / 1 out (vmem)\n");
    run<0, 1, 1, 16, 1, 1>("copy 1/1 VB16 U1");
    run<0, 1, 1, 16, 2, 1>("copy 1/1 VB16 U2");
    run<0, 1, 1, 16, 4, 1>("copy 1/1 VB16 U4");
    run<0, 1, 1, 32, 1, 1>("copy 1/1 VB32 U1");
    run<0, 1, 1, 32, 2, 1>("copy 1/1 VB32 U2");
    run<0, 1, 1, 32, 4, 1>("copy 1/1 VB32 U4");
    printf("-- add 2 in / 2 out\n");
    run<0, 2, 2, 16, 1, 1>("add 2/2 VB16 U1");
    run<0, 2, 2, 16, 2, 1>("add 2/2 VB16 U2");
    run<0, 2, 2, 32, 1, 1>("add 2/2 VB32 U1");
    run<0, 2, 2, 32, 2, 1>("add 2/2 VB32 U2");
    printf("-- vtsqrt1 core 2 in / 2 out\n");
    run<12, 2, 2, 16, 1, 1>("vtsqrt1 VB16 U1");
    run<12, 2, 2, 16, 1, 6>("vtsqrt1 VB16 U1 minb6");
    run<12, 2, 2, 16, 1, 8>("vtsqrt1 VB16 U1 minb8");
    run<12, 2, 2, 16, 2, 1>("vtsqrt1 VB16 U2");
    run<12, 2, 2, 32, 1, 1>("vtsqrt1 VB32 U1");
    run<12, 2, 2, 32, 1, 5>("vtsqrt1 VB32 U1 minb5");
    printf("-- add 4 in / 2 out (the 48 B ops' mix)\n");
    run<0, 4, 2, 16, 1, 1>("add 4/2 VB16 U1");
    run<0, 4, 2, 16, 2, 1>("add 4/2 VB16 U2");
    run<0, 4, 2, 32, 1, 1>("add 4/2 VB32 U1");
  }
  return 0;
}
