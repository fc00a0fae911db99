// Read/write-mix streaming microbenchmark (B200): how fast can a kernel stream
// NI input planes and NO output planes of f64, 2^28 elements each, with
//   reg  : 256-bit LDG -> registers -> 256-bit STG (the elementwise kernels' design)
//   tma  : cp.async.bulk global->smem ring, registers, st.shared, then
//          cp.async.bulk smem->global (bulk stores, TMA engine both ways)
//   tmal : bulk loads, 256-bit STG from registers (ew_bulk_kernel's design)
// The op is a trivial lane-wise add so the arithmetic is free; the question is
// the DRAM efficiency of each path at 1:1 (2 in / 2 out, vtsqrt1's mix) and
// 2:1 (4 in / 2 out, the 48 B/element ops).
// OP selects the per-lane work: 0 = a plain add (free), 12 = the vtsqrt1 core
// (2 in / 2 out), 3 = the vtdiv2 core (4 in / 2 out) — tf_math.cuh, intrinsics.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 -fmad=false \
//          -prec-div=true -prec-sqrt=true copy_mix.cu -o copy_mix
#include <cuda_runtime.h>

#include "../../paper_1401_6235_b200/csrc/tf_math.cuh"

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

struct alignas(32) V4 {
  double v[4];
};
__device__ __forceinline__ V4 ldg(const V4* p) {
  V4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(V4* p, const V4& r) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]),
               "d"(r.v[2]), "d"(r.v[3])
               : "memory");
}
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int OP, int NI, int NO>
__device__ __forceinline__ void lane_op(const V4 (&r)[NI], V4 (&o)[NO]) {
#pragma unroll
  for (int e = 0; e < 4; e++) {
    if constexpr (OP == 0) {
      double s = 0;
#pragma unroll
      for (int k = 0; k < NI; k++) s += r[k].v[e];
#pragma unroll
      for (int k = 0; k < NO; k++) o[k].v[e] = s;
    } else {
      double v[NI];
#pragma unroll
      for (int k = 0; k < NI; k++) v[k] = r[k].v[e];
      tf::P<double> z = tf::apply<double, OP>(v);
      o[0].v[e] = z.a;
      o[1].v[e] = z.b;
    }
  }
}

template <int NI, int NO>
struct Args {
  const V4* in[NI];
  V4* out[NO];
};

template <int OP, int NI, int NO>
__global__ void __launch_bounds__(256) reg_kernel(Args<NI, NO> a, int64_t nvec) {
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (j >= nvec) return;
  V4 r[NI];
#pragma unroll
  for (int k = 0; k < NI; k++) r[k] = ldg(a.in[k] + j);
  V4 o[NO];
  lane_op<OP, NI, NO>(r, o);
#pragma unroll
  for (int k = 0; k < NO; k++) stg(a.out[k] + j, o[k]);
}

// TMA both ways.  MODE 0: bulk stores from smem; MODE 1: 256-bit STG from registers.
template <int OP, int NI, int NO, int NST, int MODE>
__global__ void __launch_bounds__(256) tma_kernel(Args<NI, NO> a, int64_t nvec, int reps) {
  constexpr int TILE = 256 * 32;
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* sin = sm;                          // NST * NI tiles
  unsigned char* sout = sm + NST * NI * TILE;       // 2 * NO tiles (double-buffered)
  __shared__ __align__(8) uint64_t bar[NST];
  const int64_t ntile = (nvec + 255) / 256;
  const int64_t t0 = (int64_t)blockIdx.x * reps;
  if (t0 >= ntile) return;
  const int cnt = (int)(ntile - t0 < reps ? ntile - t0 : reps);
  if (threadIdx.x == 0) {
    for (int q = 0; q < NST; q++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int j, int buf) {
    const int64_t v0 = (t0 + j) * 256;
    const int64_t left = nvec - v0;
    const uint32_t bytes = (uint32_t)(left < 256 ? left : 256) * 32u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[buf])),
                 "r"(bytes * NI)
                 : "memory");
    for (int k = 0; k < NI; k++)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(sin + (buf * NI + k) * TILE)),
          "l"(a.in[k] + v0), "r"(bytes), "r"(su32(&bar[buf]))
          : "memory");
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < NST && q < cnt; q++) issue(q, q);
  for (int j = 0; j < cnt; j++) {
    const int buf = j % NST;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar[buf])),
        "r"((uint32_t)((j / NST) & 1))
        : "memory");
    const int64_t v0 = (t0 + j) * 256;
    const int64_t jv = v0 + threadIdx.x;
    const bool act = jv < nvec;
    V4 o[NO];
    if (act) {
      V4 r[NI];
#pragma unroll
      for (int k = 0; k < NI; k++) r[k] = *reinterpret_cast<const V4*>(sin + (buf * NI + k) * TILE + threadIdx.x * 32);
      lane_op<OP, NI, NO>(r, o);
    }
    if constexpr (MODE == 1) {
      if (act)
        for (int k = 0; k < NO; k++) stg(a.out[k] + jv, o[k]);
      __syncthreads();
    } else {
      const int ob = j & 1;
      // the bulk store that last read this output buffer (tile j-2) must be done
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
      if (act)
        for (int k = 0; k < NO; k++)
          *reinterpret_cast<V4*>(sout + (ob * NO + k) * TILE + threadIdx.x * 32) = o[k];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        const int64_t left = nvec - v0;
        const uint32_t bytes = (uint32_t)(left < 256 ? left : 256) * 32u;
        for (int k = 0; k < NO; k++)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.out[k] + v0),
                       "r"(su32(sout + (ob * NO + k) * TILE)), "r"(bytes)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0 && j + NST < cnt) issue(j + NST, buf);
  }
  if (MODE == 0 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
static void timeit(const char* name, double bytes, F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 5; i++) f();
  std::vector<float> ms;
  for (int r = 0; r < 30; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    ms.push_back(t);
  }
  std::sort(ms.begin(), ms.end());
  cudaError_t e = cudaGetLastError();
  printf("%-28s median %7.1f GB/s  best %7.1f GB/s  %s\n", name, bytes / (ms[15] * 1e-3) / 1e9,
         bytes / (ms[0] * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int OP, int NI, int NO, int NST, int MODE>
static void run_tma(const Args<NI, NO>& a, int64_t nvec, int reps, double bytes, const char* tag,
                    const char* what) {
  const int smem = NST * NI * 8192 + (MODE == 0 ? 2 * NO * 8192 : 0);
  cudaFuncSetAttribute(tma_kernel<OP, NI, NO, NST, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  const int64_t ntile = (nvec + 255) / 256;
  char nm[64];
  snprintf(nm, sizeof nm, "%s %s st%d r%d", tag, what, NST, reps);
  timeit(nm, bytes, [&] {
    tma_kernel<OP, NI, NO, NST, MODE><<<(unsigned)((ntile + reps - 1) / reps), 256, smem>>>(a, nvec,
                                                                                        reps);
  });
}

template <int OP, int NI, int NO>
static void run(const char* tag, double** planes, int64_t n) {
  Args<NI, NO> a;
  for (int k = 0; k < NI; k++) a.in[k] = reinterpret_cast<const V4*>(planes[k]);
  for (int k = 0; k < NO; k++) a.out[k] = reinterpret_cast<V4*>(planes[NI + k]);
  const int64_t nvec = n / 4;
  const double bytes = (double)(NI + NO) * 8.0 * n;
  char nm[64];
  snprintf(nm, sizeof nm, "%s reg", tag);
  timeit(nm, bytes, [&] { reg_kernel<OP, NI, NO><<<(unsigned)((nvec + 255) / 256), 256>>>(a, nvec); });
  for (int reps : {1, 2, 4}) {
    run_tma<OP, NI, NO, 2, 0>(a, nvec, reps, bytes, tag, "tma-bulkst");
    run_tma<OP, NI, NO, 2, 1>(a, nvec, reps, bytes, tag, "tma-ldonly");
  }
}

int main() {
  const int64_t n = 1LL << 28;
  double* planes[6];
  for (int k = 0; k < 6; k++) {
    cudaMalloc(&planes[k], n * 8);
    cudaMemset(planes[k], 0, n * 8);
  }
  cudaDeviceSynchronize();
  // inputs: positive values ~1 for the sqrt / division cores
  {
    std::vector<double> h(1 << 20);
    for (size_t i = 0; i < h.size(); i++) h[i] = 1.0 + (double)(i % 1000) * 1e-3;
    for (int k = 0; k < 6; k++)
      for (int64_t o = 0; o < n; o += (int64_t)h.size())
        cudaMemcpy(planes[k] + o, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  }
  for (int pass = 0; pass < 2; pass++) {
    run<0, 2, 2>("add 1:1 (2/2)", planes, n);
    run<0, 4, 2>("add 2:1 (4/2)", planes, n);
    run<12, 2, 2>("vtsqrt1 (2/2)", planes, n);
    run<3, 4, 2>("vtdiv2 (4/2)", planes, n);
    run<0, 1, 1>("copy 1:1 (1/1)", planes, n);
  }
  return 0;
}
