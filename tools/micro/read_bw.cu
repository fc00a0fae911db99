// Read-only streaming microbenchmark (B200): how fast can one or two f64 planes of 2^30
// elements be READ, as the reductions read them?  Each thread loads NV 16-byte vectors per
// plane, B at a time (all B loads issued before they are consumed), adds them up, and the CTA
// writes one partial.  One CTA per 256*NV vectors.  NV = 128, B = 8/16 is reduce_kernel's
// geometry (64K-element tiles); small NV are the "light" designs.  MINB = launch bound.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 read_bw.cu -o read_bw
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct alignas(16) V2 {
  double v[2];
};
__device__ __forceinline__ V2 ldg(const V2* p) {
  V2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.v[0]), "=d"(r.v[1])
               : "l"(p));
  return r;
}

template <int NP, int NV, int B, int MINB>
__global__ void __launch_bounds__(256, MINB) k(const double* a, const double* b, double* out,
                                               int64_t nvec) {
  const int64_t base = (int64_t)blockIdx.x * (256LL * NV) + threadIdx.x;
  double s0 = 0, s1 = 0;
#pragma unroll 1
  for (int k0 = 0; k0 < NV; k0 += B) {
    V2 r[B][NP];
#pragma unroll
    for (int u = 0; u < B; u++) {
      const int64_t j = base + (int64_t)(k0 + u) * 256;
      if (j < nvec) {
        r[u][0] = ldg(reinterpret_cast<const V2*>(a) + j);
        if (NP == 2) r[u][NP - 1] = ldg(reinterpret_cast<const V2*>(b) + j);
      } else {
        for (int q = 0; q < NP; q++) r[u][q].v[0] = r[u][q].v[1] = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < B; u++)
#pragma unroll
      for (int q = 0; q < NP; q++) {
        s0 += r[u][q].v[0];
        s1 += r[u][q].v[1];
      }
  }
  double s = s0 + s1;
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  __shared__ double sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < 8; w++) t += sm[w];
    out[blockIdx.x] = t;
  }
}

static double *A, *Bp, *O;
static int64_t N;

template <int NP, int NV, int B, int MINB>
static void run(const char* name) {
  const int64_t nvec = N / 2;
  const int64_t blocks = (nvec + 256LL * NV - 1) / (256LL * NV);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k<NP, NV, B, MINB>);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<NP, NV, B, MINB>, 256, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<NP, NV, B, MINB><<<(unsigned)blocks, 256>>>(A, Bp, O, nvec);
  std::vector<float> ts;
  for (int i = 0; i < 15; i++) {
    cudaEventRecord(e0);
    k<NP, NV, B, MINB><<<(unsigned)blocks, 256>>>(A, Bp, O, nvec);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  const double bytes = (double)NP * N * 8;
  printf("%-30s regs %3d ctas/sm %d  median %.4f ms  %.0f GB/s  best %.0f GB/s (%s)\n", name,
         fa.numRegs, occ, ts[ts.size() / 2], bytes / ts[ts.size() / 2] / 1e6, bytes / ts[0] / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  if (cudaDeviceSynchronize() != cudaSuccess) exit(2);
}

int main(int argc, char** argv) {
  N = 1ll << (argc > 1 ? atoi(argv[1]) : 30);
  if (cudaMalloc(&A, N * 8) != cudaSuccess || cudaMalloc(&Bp, N * 8) != cudaSuccess ||
      cudaMalloc(&O, (N / 512 + 1) * 8) != cudaSuccess) {
    printf("cudaMalloc failed\n");
    return 1;
  }
  cudaMemset(A, 0, N * 8);
  cudaMemset(Bp, 0, N * 8);
  for (int rep = 0; rep < 2; rep++) {
    printf("-- one plane (vtsum's traffic)\n");
    run<1, 128, 16, 1>("1 plane NV128 B16 (reduce)");
    run<1, 128, 8, 1>("1 plane NV128 B8");
    run<1, 128, 32, 1>("1 plane NV128 B32");
    run<1, 32, 16, 1>("1 plane NV32 B16");
    run<1, 16, 16, 1>("1 plane NV16 B16");
    run<1, 8, 8, 1>("1 plane NV8 B8");
    run<1, 4, 4, 1>("1 plane NV4 B4");
    run<1, 2, 2, 1>("1 plane NV2 B2");
    run<1, 1, 1, 8>("1 plane NV1 B1 minb8");
    printf("-- two planes (vtdot's traffic)\n");
    run<2, 128, 8, 1>("2 planes NV128 B8 (reduce)");
    run<2, 128, 16, 1>("2 planes NV128 B16");
    run<2, 128, 4, 1>("2 planes NV128 B4");
    run<2, 16, 8, 1>("2 planes NV16 B8");
    run<2, 4, 4, 1>("2 planes NV4 B4");
    run<2, 2, 2, 1>("2 planes NV2 B2");
    run<2, 1, 1, 8>("2 planes NV1 B1 minb8");
  }
  return 0;
}
