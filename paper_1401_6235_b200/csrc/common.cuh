// common.cuh — status/error plumbing and small device helpers shared by the
// libtwofold_b200 translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/twofold_b200.h"

// store cache hint (".cs" streaming by default; A/B builds may override)
#ifndef TF_ST_HINT
#define TF_ST_HINT ".cs"
#endif

namespace tf {

// thread-local last error, surfaced through tf_last_error()
void set_error(const std::string& msg);
void clear_error();

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

inline int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return TF_OK;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? TF_ENOMEM : TF_ECUDA;
}

// launch-error check right after a <<<>>> launch
inline int launch_status(const char* where) { return cuda_status(cudaGetLastError(), where); }

// SM count of the current device (cached per device)
int sm_count();

// ---- programmatic dependent launch (PDL) ----------------------------------------
// A kernel launched with the programmatic-stream-serialization attribute may be
// scheduled while its predecessor on the stream is still draining.  pdl_wait()
// at the very top (before ANY global-memory access) blocks until the predecessor
// grid has completed and its writes are visible, so the launch is correct
// whatever the predecessor was (our kernel, a torch kernel, a memcpy); what
// overlaps is only the dependent grid's launch and CTA scheduling with the
// predecessor's tail.  pdl_trigger() lets the next PDL launch start early.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// TF_PDL=0 disables the attribute (A/B runs); default on
bool pdl_enabled();
// cudaLaunchKernel with the PDL attribute when enabled
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                       cudaStream_t stream);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- streaming memory helpers --------------------------------------------------
// Inputs are read once: ld.global.nc with L1::no_allocate keeps them out of L1
// and lets L2 evict them first.  Outputs are written once: st.global.cs.
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global" TF_ST_HINT ".v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global" TF_ST_HINT ".v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global" TF_ST_HINT ".f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_stream(float* p, float v) {
  asm volatile("st.global" TF_ST_HINT ".f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// 16-byte vector of a plane type
template <class T>
struct Vec16;
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int N = 2;
};
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int N = 4;
};

template <class T>
__device__ __forceinline__ T lane(const typename Vec16<T>::type& v, int j);
template <>
__device__ __forceinline__ double lane<double>(const double2& v, int j) {
  return j == 0 ? v.x : v.y;
}
template <>
__device__ __forceinline__ float lane<float>(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
template <class T>
__device__ __forceinline__ void set_lane(typename Vec16<T>::type& v, int j, T x);
template <>
__device__ __forceinline__ void set_lane<double>(double2& v, int j, double x) {
  if (j == 0) v.x = x; else v.y = x;
}
template <>
__device__ __forceinline__ void set_lane<float>(float4& v, int j, float x) {
  if (j == 0) v.x = x; else if (j == 1) v.y = x; else if (j == 2) v.z = x; else v.w = x;
}

// 32-byte vector (sm_100 256-bit LDG/STG: LDG.E.*.256 / STG.E.*.256)
template <class T>
struct alignas(32) Vec32 {
  static constexpr int N = 32 / sizeof(T);
  T v[N];
};
__device__ __forceinline__ Vec32<double> ld_stream(const Vec32<double>* p) {
  Vec32<double> r;
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
      : "l"(p));
  return r;
}
__device__ __forceinline__ Vec32<float> ld_stream(const Vec32<float>* p) {
  Vec32<float> r;
  asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
        "=f"(r.v[6]), "=f"(r.v[7])
      : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(Vec32<double>* p, const Vec32<double>& r) {
  asm volatile("st.global" TF_ST_HINT ".v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]),
               "d"(r.v[2]), "d"(r.v[3])
               : "memory");
}
__device__ __forceinline__ void st_stream(Vec32<float>* p, const Vec32<float>& r) {
  asm volatile("st.global" TF_ST_HINT ".v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
               "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]),
               "f"(r.v[7])
               : "memory");
}
// 16-byte array vector (same LDG.128/STG.128 as double2/float4, indexable)
template <class T>
struct alignas(16) Vec16A {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};
__device__ __forceinline__ Vec16A<double> ld_stream(const Vec16A<double>* p) {
  Vec16A<double> r;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  return r;
}
__device__ __forceinline__ Vec16A<float> ld_stream(const Vec16A<float>* p) {
  Vec16A<float> r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
      : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(Vec16A<double>* p, const Vec16A<double>& r) {
  asm volatile("st.global" TF_ST_HINT ".v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]) : "memory");
}
__device__ __forceinline__ void st_stream(Vec16A<float>* p, const Vec16A<float>& r) {
  asm volatile("st.global" TF_ST_HINT ".v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]),
               "f"(r.v[2]), "f"(r.v[3])
               : "memory");
}
template <class T, int VB>
struct VecSel {
  using type = Vec32<T>;
};
template <class T>
struct VecSel<T, 16> {
  using type = Vec16A<T>;
};
template <class T, int VB>
using VecN = typename VecSel<T, VB>::type;

// ---- bulk async copies (TMA engine, UBLKCP) + mbarriers ---------------------------
// One elected thread arms an mbarrier with the byte count of a stage and issues
// one cp.async.bulk per plane; the copy engine completes the transaction on the
// barrier, and the consumers wait on its phase parity.  Addresses and sizes are
// multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) accesses that a barrier makes dependent on them
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// evict-first L2 policy for streamed-once inputs (bulk copies take it as a hint)
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

// RAII device switch for host entry points that take a device ordinal
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace tf
