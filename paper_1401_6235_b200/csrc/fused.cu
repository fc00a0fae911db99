// fused.cu — fused twofold expression kernels.
//
// The reference chains scalar twofold ops in its application studies
// (demos.py:153-199 Gauss elimination, demos.py:211-238 quadratic roots).  Run
// over n independent instances, each chain becomes one data-parallel kernel
// that keeps every intermediate in registers instead of a round trip through
// HBM per op.  The op sequence and association order are the demos', op for op,
// so results equal composing the elementwise kernels (and the reference) bit
// for bit.
//
//   TF_FAXPY    z = tadd(tmul(a, x), y)                         6 in, 2 out planes
//   TF_FSUBMUL  z = tsub(c, tmul(a, b))  (elimination update,   6 in, 2 out
//               demos.py:182-184)
//   TF_FQUAD    roots of a x^2 + b x + c (demos.py:222-229):    6 in, 6 out
//               disc = tsub(tmul(b,b), tmul(tmul(4,a),c)); d = tsqrt(disc);
//               x0 = tdiv(tsub(-b,d), tmul(2,a)); x1 = tdiv(tadd(-b,d), tmul(2,a))
//   TF_FGAUSS3  naive 3x3 Gauss elimination + back substitution (demos.py:175-192)
//               in: A value/error (9 planes each, row-major), f value/error (3);
//               out: x value/error (3 planes each)
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "tf_math.cuh"

namespace tf {

template <class T>
struct TF {
  T a, b;
};
template <class T>
__device__ __forceinline__ TF<T> mk(P<T> p) {
  return {p.a, p.b};
}
template <class T>
__device__ __forceinline__ TF<T> Tmul(TF<T> x, TF<T> y) {
  return mk(tmul(x.a, x.b, y.a, y.b));
}
template <class T>
__device__ __forceinline__ TF<T> Tadd(TF<T> x, TF<T> y) {
  return mk(tadd(x.a, x.b, y.a, y.b));
}
template <class T>
__device__ __forceinline__ TF<T> Tsub(TF<T> x, TF<T> y) {
  return mk(tsub(x.a, x.b, y.a, y.b));
}
template <class T>
__device__ __forceinline__ TF<T> Tdiv(TF<T> x, TF<T> y) {
  return mk(tdiv(x.a, x.b, y.a, y.b));
}
template <class T>
__device__ __forceinline__ TF<T> Tsqrt(TF<T> x) {
  return mk(tsqrt(x.a, x.b));
}

template <class T>
__device__ __forceinline__ TF<T> ld2(const T* v, const T* e, int64_t i) {
  return {ld_stream(v + i), ld_stream(e + i)};
}
template <class T>
__device__ __forceinline__ void st2(T* v, T* e, int64_t i, TF<T> z) {
  st_stream(v + i, z.a);
  st_stream(e + i, z.b);
}

#ifndef TF_FQUAD_VB
#define TF_FQUAD_VB 16  // quadratic: 16-byte vectors (6 in + 6 out planes per thread)
#endif

struct FArgs {
  const void* in[6];
  void* out[6];
};

// One instance of a fused chain: v = the 6 input values, z = the outputs.
template <class T, int FOP>
__device__ __forceinline__ void fused_elem(const T* v, T* z) {
  const TF<T> a{v[0], v[1]}, x{v[2], v[3]}, y{v[4], v[5]};
  if constexpr (FOP == TF_FAXPY) {
    const TF<T> r = Tadd(Tmul(a, x), y);
    z[0] = r.a;
    z[1] = r.b;
  } else if constexpr (FOP == TF_FSUBMUL) {
    const TF<T> r = Tsub(a, Tmul(x, y));  // a is c here: c - a*b
    z[0] = r.a;
    z[1] = r.b;
  } else {  // TF_FQUAD: a x^2 + b x + c with (a, b, c) = (a, x, y)
    const TF<T> four{T(4), T(0)}, two{T(2), T(0)};
    const TF<T> disc = Tsub(Tmul(x, x), Tmul(Tmul(four, a), y));
    const TF<T> d = Tsqrt(disc);
    const TF<T> nb{-x.a, -x.b};  // tneg (arith.py:838-842): exact sign flips
    const TF<T> two_a = Tmul(two, a);
    const TF<T> x0 = Tdiv(Tsub(nb, d), two_a);
    const TF<T> x1 = Tdiv(Tadd(nb, d), two_a);
    z[0] = d.a;
    z[1] = d.b;
    z[2] = x0.a;
    z[3] = x0.b;
    z[4] = x1.a;
    z[5] = x1.b;
  }
}

// axpy / submul / quadratic over n instances: one VB-byte vector per plane per
// thread (the twofold kernels' memory design), one CTA per 256 vectors; planes
// that are not all VB-aligned (and the n % E tail) take the scalar path.
template <class T, int FOP, int VB>
__global__ void __launch_bounds__(256) fused_ew_kernel(FArgs p, int64_t n, int64_t nvec) {
  constexpr int NI = 6, NO = FOP == TF_FQUAD ? 6 : 2;
  using V = VecN<T, VB>;
  constexpr int E = V::N;
  const T* const* in = reinterpret_cast<const T* const*>(p.in);
  T* const* out = reinterpret_cast<T* const*>(p.out);
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = gtid; j < nvec; j += gstride) {
    V r[NI];
#pragma unroll
    for (int k = 0; k < NI; k++) r[k] = ld_stream(reinterpret_cast<const V*>(in[k]) + j);
    V o[NO];
#pragma unroll
    for (int e = 0; e < E; e++) {
      T v[NI], z[NO];
#pragma unroll
      for (int k = 0; k < NI; k++) v[k] = r[k].v[e];
      fused_elem<T, FOP>(v, z);
#pragma unroll
      for (int k = 0; k < NO; k++) o[k].v[e] = z[k];
    }
#pragma unroll
    for (int k = 0; k < NO; k++) st_stream(reinterpret_cast<V*>(out[k]) + j, o[k]);
  }
  for (int64_t i = nvec * E + gtid; i < n; i += gstride) {
    T v[NI], z[NO];
#pragma unroll
    for (int k = 0; k < NI; k++) v[k] = ld_stream(in[k] + i);
    fused_elem<T, FOP>(v, z);
#pragma unroll
    for (int k = 0; k < NO; k++) st_stream(out[k] + i, z[k]);
  }
}

template <class T, int FOP, int VB>
static void launch_fused_ew(const FArgs& p, int64_t n, cudaStream_t s) {
  constexpr int E = VecN<T, VB>::N;
  constexpr int NO = FOP == TF_FQUAD ? 6 : 2;
  bool aligned = true;
  for (int k = 0; k < 6; k++) aligned = aligned && (reinterpret_cast<uintptr_t>(p.in[k]) % VB == 0);
  for (int k = 0; k < NO; k++) aligned = aligned && (reinterpret_cast<uintptr_t>(p.out[k]) % VB == 0);
  const int64_t nvec = aligned ? n / E : 0;
  int64_t blocks = nvec > 0 ? (nvec + 255) / 256 : (n + 255) / 256;
  blocks = blocks > 0x7fffffffLL ? 0x7fffffffLL : (blocks < 1 ? 1 : blocks);
  fused_ew_kernel<T, FOP, VB><<<(unsigned)blocks, 256, 0, s>>>(p, n, nvec);
}

template <class T>
__global__ void __launch_bounds__(128) gauss3_kernel(const T* __restrict__ Av,
                                                     const T* __restrict__ Ae,
                                                     const T* __restrict__ fv,
                                                     const T* __restrict__ fe, T* __restrict__ xv,
                                                     T* __restrict__ xe, int64_t n) {
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gstride) {
    TF<T> a[3][3], f[3], x[3];
#pragma unroll
    for (int r = 0; r < 3; r++) {
#pragma unroll
      for (int c = 0; c < 3; c++) a[r][c] = ld2(Av + (3 * r + c) * n, Ae + (3 * r + c) * n, s);
      f[r] = ld2(fv + r * n, fe + r * n, s);
    }
    // forward elimination, natural order, no pivoting (demos.py:177-185)
#pragma unroll
    for (int k = 0; k < 3; k++) {
#pragma unroll
      for (int i = k + 1; i < 3; i++) {
        TF<T> m = Tdiv(a[i][k], a[k][k]);
#pragma unroll
        for (int j = k; j < 3; j++) a[i][j] = Tsub(a[i][j], Tmul(m, a[k][j]));
        f[i] = Tsub(f[i], Tmul(m, f[k]));
      }
    }
    // back substitution (demos.py:187-192)
#pragma unroll
    for (int i = 2; i >= 0; i--) {
      TF<T> acc = f[i];
#pragma unroll
      for (int j = i + 1; j < 3; j++) acc = Tsub(acc, Tmul(a[i][j], x[j]));
      x[i] = Tdiv(acc, a[i][i]);
    }
#pragma unroll
    for (int r = 0; r < 3; r++) st2(xv + r * n, xe + r * n, s, x[r]);
  }
}

// axpy / submul run on 16-byte vectors, the lighter-thread design that won for the
// registry kernels (ew_step16_kernel): f64 48 registers instead of 66, 6.95 -> 7.30 TB/s
// at 2^27 (+5%; profiles/r2s5_fused_vb_ab.txt).  TF_FUSED_VB=32 selects the 32-byte
// vectors again (A/B).
static bool fused_vb16() {
  static const bool v = [] {
    const char* e = getenv("TF_FUSED_VB");
    return !(e && atoi(e) == 32);
  }();
  return v;
}

int fused_launch(int fop, int dtype, int64_t n, const void* const* in, void* const* out,
                 cudaStream_t s) {
  if (fop < 0 || fop > 3) return fail(TF_EINVAL, "tf_fused: unknown fused op id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_fused: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_fused: negative length");
  if (n == 0) return TF_OK;
  static const int nin[4] = {6, 6, 6, 4}, nout[4] = {2, 2, 6, 2};
  if (!in || !out) return fail(TF_EINVAL, "tf_fused: null plane");
  for (int k = 0; k < nin[fop]; k++)
    if (!in[k]) return fail(TF_EINVAL, "tf_fused: null plane");
  for (int k = 0; k < nout[fop]; k++)
    if (!out[k]) return fail(TF_EINVAL, "tf_fused: null plane");
  FArgs p{};
  for (int k = 0; k < nin[fop]; k++) p.in[k] = in[k];
  for (int k = 0; k < nout[fop]; k++) p.out[k] = out[k];
  const int threads = 128;  // gauss3 (the others: launch_fused_ew)
  int64_t blocks = (n + threads - 1) / threads;
  blocks = blocks > 0x7fffffffLL ? 0x7fffffffLL : blocks;  // one CTA per chunk
  const bool f64 = dtype == TF_F64;
  switch (fop) {
    case TF_FAXPY:
      if (fused_vb16()) {
        if (f64) launch_fused_ew<double, TF_FAXPY, 16>(p, n, s);
        else launch_fused_ew<float, TF_FAXPY, 16>(p, n, s);
      } else if (f64) launch_fused_ew<double, TF_FAXPY, 32>(p, n, s);
      else launch_fused_ew<float, TF_FAXPY, 32>(p, n, s);
      break;
    case TF_FSUBMUL:
      if (fused_vb16()) {
        if (f64) launch_fused_ew<double, TF_FSUBMUL, 16>(p, n, s);
        else launch_fused_ew<float, TF_FSUBMUL, 16>(p, n, s);
      } else if (f64) launch_fused_ew<double, TF_FSUBMUL, 32>(p, n, s);
      else launch_fused_ew<float, TF_FSUBMUL, 32>(p, n, s);
      break;
    case TF_FQUAD:
      if (f64) launch_fused_ew<double, TF_FQUAD, TF_FQUAD_VB>(p, n, s);
      else launch_fused_ew<float, TF_FQUAD, TF_FQUAD_VB>(p, n, s);
      break;
    default:
      if (f64)
        gauss3_kernel<double><<<(unsigned)blocks, threads, 0, s>>>(
            (const double*)in[0], (const double*)in[1], (const double*)in[2],
            (const double*)in[3], (double*)out[0], (double*)out[1], n);
      else
        gauss3_kernel<float><<<(unsigned)blocks, threads, 0, s>>>(
            (const float*)in[0], (const float*)in[1], (const float*)in[2], (const float*)in[3],
            (float*)out[0], (float*)out[1], n);
  }
  return launch_status("tf_fused");
}

}  // namespace tf
