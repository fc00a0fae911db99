// common.cuh — status/error plumbing and small device helpers shared by the
// libtwofold_b200 translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/twofold_b200.h"

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
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_stream(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
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
