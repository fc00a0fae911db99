// horner.cu — twofold Horner evaluation, one point per lane-slot.
//
// Per point: r = (c_d, +0); for k = d-1..0: r = _tadd1(_tmul1(r, x), c_k)
// (MTF1.1 arith.py:97-101, then ATF1.1 arith.py:67-71).  z0 is bitwise the
// plain (unfused) Horner value; z1 flags its cancellation.
//
// Compute-bound on the FP64 pipe: each step is 4 (tmul1: DMUL, DFMA, DMUL,
// DADD) + 7 (tadd1: TwoSum 6 + 1) = 11 FP64 instructions, 220 per point at
// degree 20, against 24 bytes of HBM traffic.  Each thread carries ILP
// independent points so the dependent DADD/DFMA chains overlap; coefficients
// are kernel parameters (constant bank operands).  Degree 20 — the benchmark
// polynomial (x-1)^20 — gets a fully unrolled instantiation.
#include <cuda_runtime.h>

#include "common.cuh"
#include "tf_math.cuh"

namespace tf {

template <class T>
struct Coeffs {
  T c[TF_HORNER_MAX_DEGREE + 1];
};

template <class T, int ILP, int DEG>
__global__ void __launch_bounds__(256) horner_kernel(const T* __restrict__ x, T* __restrict__ o0,
                                                     T* __restrict__ o1, int64_t n, int degree,
                                                     const __grid_constant__ Coeffs<T> c) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int d = DEG >= 0 ? DEG : degree;
  for (int64_t base = gtid; base < n; base += gstride * ILP) {
    T xv[ILP];
    P<T> r[ILP];
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const int64_t i = base + u * gstride;
      xv[u] = i < n ? ld_stream(x + i) : T(0);
      r[u] = P<T>{c.c[d], T(0)};
    }
    if constexpr (DEG >= 0) {
#pragma unroll
      for (int k = DEG - 1; k >= 0; k--) {
#pragma unroll
        for (int u = 0; u < ILP; u++) {
          r[u] = tmul1(r[u].a, r[u].b, xv[u]);
          r[u] = tadd1(r[u].a, r[u].b, c.c[k]);
        }
      }
    } else {
#pragma unroll 1
      for (int k = d - 1; k >= 0; k--) {
        const T ck = c.c[k];
#pragma unroll
        for (int u = 0; u < ILP; u++) {
          r[u] = tmul1(r[u].a, r[u].b, xv[u]);
          r[u] = tadd1(r[u].a, r[u].b, ck);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const int64_t i = base + u * gstride;
      if (i < n) {
        st_stream(o0 + i, r[u].a);
        st_stream(o1 + i, r[u].b);
      }
    }
  }
}

template <class T>
static int horner_t(int64_t n, const void* x, const double* coeffs, int degree, void* o0,
                    void* o1, cudaStream_t s) {
  Coeffs<T> c;
  for (int k = 0; k <= degree; k++) c.c[k] = (T)coeffs[k];
  for (int k = degree + 1; k <= TF_HORNER_MAX_DEGREE; k++) c.c[k] = T(0);
  constexpr int ILP = 4;
  int64_t blocks = (n + 256 * ILP - 1) / (256 * ILP);
  // one CTA per 256*ILP points (hardware-balanced, no idle-SM tail)
  blocks = blocks > 0x7fffffffLL ? 0x7fffffffLL : (blocks < 1 ? 1 : blocks);
  const T* px = static_cast<const T*>(x);
  T* p0 = static_cast<T*>(o0);
  T* p1 = static_cast<T*>(o1);
  if (degree == 20)
    horner_kernel<T, ILP, 20><<<(unsigned)blocks, 256, 0, s>>>(px, p0, p1, n, degree, c);
  else
    horner_kernel<T, ILP, -1><<<(unsigned)blocks, 256, 0, s>>>(px, p0, p1, n, degree, c);
  return launch_status("tf_horner");
}

int horner_launch(int dtype, int64_t n, const void* x, const double* coeffs, int degree,
                  void* o0, void* o1, cudaStream_t s) {
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_horner: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_horner: negative length");
  if (degree < 0 || degree > TF_HORNER_MAX_DEGREE)
    return fail(TF_EINVAL, "tf_horner: degree out of range");
  if (!coeffs) return fail(TF_EINVAL, "tf_horner: null coefficients");
  if (n == 0) return TF_OK;
  if (!x || !o0 || !o1) return fail(TF_EINVAL, "tf_horner: null plane");
  return dtype == TF_F64 ? horner_t<double>(n, x, coeffs, degree, o0, o1, s)
                         : horner_t<float>(n, x, coeffs, degree, o0, o1, s);
}

}  // namespace tf
