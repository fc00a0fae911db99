// interleaved.cu — the 24 elementwise ops over the INTERLEAVED (AoS) layout,
// plus split<->interleaved conversion kernels.
//
// Interleaved: a twofold operand or result is one array of n (value, error)
// pairs, the paper's twofold<T> struct {value, error}.  Scalar
// (non-twofold) operands stay plain 1-D planes.  A binary twofold op streams 3
// arrays instead of 6 planes; the bytes per element are the same
// ((NIN+2)*sizeof(T)), and so is the arithmetic: apply<T,OP> from tf_math.cuh,
// i.e. the reference cores (arith.py:61-218) bit for bit.
//
// Vector body: each step covers E = 16/sizeof(T) elements — one 16-byte load
// per plain plane, two per interleaved operand, two 16-byte stores for the
// result.  Requires 16-byte aligned arrays; otherwise a scalar grid-stride path
// (same launch).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "tf_math.cuh"

namespace tf {

template <class T>
struct ILArgs {
  const T* a;  // x: pairs if twofold (22, 21, u2), else plain
  const T* b;  // y: pairs if 22, plain if 21/11, unused for unary
  T* out;      // pairs
};

template <class T, int OP>
__device__ __forceinline__ void il_gather(const ILArgs<T>& p, int64_t i, T* v) {
  constexpr int AR = OpInfo<OP>::ARITY;
  if constexpr (AR == 22) {
    v[0] = ld_stream(p.a + 2 * i);
    v[1] = ld_stream(p.a + 2 * i + 1);
    v[2] = ld_stream(p.b + 2 * i);
    v[3] = ld_stream(p.b + 2 * i + 1);
  } else if constexpr (AR == 21) {
    v[0] = ld_stream(p.a + 2 * i);
    v[1] = ld_stream(p.a + 2 * i + 1);
    v[2] = ld_stream(p.b + i);
  } else if constexpr (AR == 11) {
    v[0] = ld_stream(p.a + i);
    v[1] = ld_stream(p.b + i);
  } else if constexpr (AR == 2) {
    v[0] = ld_stream(p.a + 2 * i);
    v[1] = ld_stream(p.a + 2 * i + 1);
  } else {
    v[0] = ld_stream(p.a + i);
  }
}

#ifndef TF_IL_MIN_BLOCKS
#define TF_IL_MIN_BLOCKS 4  // <= 64 registers: vtmul1 f64 otherwise took 122 (2 CTAs/SM)
#endif

template <class T, int OP>
__global__ void __launch_bounds__(256, TF_IL_MIN_BLOCKS) ew_il_kernel(ILArgs<T> p, int64_t n, int vec) {
  constexpr int NIN = OpInfo<OP>::NIN;
  constexpr int AR = OpInfo<OP>::ARITY;
  constexpr int E = Vec16<T>::N;
  using V = typename Vec16<T>::type;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvec = vec ? n / E : 0;

  // one step = E elements: a pair operand is one 32-byte vector (E pairs,
  // sm_100 256-bit LDG), a plain plane one 16-byte vector; the result one
  // 32-byte store.
  using VP = Vec32<T>;   // E pairs
  using VS = Vec16A<T>;  // E scalars
  constexpr bool XP = (AR == 22 || AR == 21 || AR == 2);
  // steps in flight per thread (all loads issue before any math); the one-plane
  // op (vtsqrt: 16 bytes in per step) carries 4 to keep enough bytes in flight
  constexpr int U = AR == 1 ? 4 : 2;
  // CTA-chunked, as the split kernels: chunk = 256*U consecutive steps per CTA,
  // thread t takes steps t and t+256 (coalesced, contiguous per CTA)
  const int64_t CH = 256LL * U;
  for (int64_t cb = (int64_t)blockIdx.x * CH; cb < nvec; cb += (int64_t)gridDim.x * CH) {
    const int64_t base = cb + threadIdx.x;
    VP xp[U], yp[U];
    VS xs[U], ys[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        if constexpr (XP) xp[u] = ld_stream(reinterpret_cast<const VP*>(p.a) + j);
        else xs[u] = ld_stream(reinterpret_cast<const VS*>(p.a) + j);
        if constexpr (AR == 22) yp[u] = ld_stream(reinterpret_cast<const VP*>(p.b) + j);
        else if constexpr (AR == 21 || AR == 11) ys[u] = ld_stream(reinterpret_cast<const VS*>(p.b) + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j >= nvec) continue;
      VP o;
      T v[E][NIN];
#pragma unroll
      for (int e = 0; e < E; e++) {
        if constexpr (XP) {
          v[e][0] = xp[u].v[2 * e];
          v[e][1] = xp[u].v[2 * e + 1];
        } else {
          v[e][0] = xs[u].v[e];
        }
        if constexpr (AR == 22) {
          v[e][2] = yp[u].v[2 * e];
          v[e][3] = yp[u].v[2 * e + 1];
        } else if constexpr (AR == 21) {
          v[e][2] = ys[u].v[e];
        } else if constexpr (AR == 11) {
          v[e][1] = ys[u].v[e];
        }
      }
      P<T> z[E];
      apply_lanes<T, OP, E>(v, z);
#pragma unroll
      for (int e = 0; e < E; e++) {
        o.v[2 * e] = z[e].a;
        o.v[2 * e + 1] = z[e].b;
      }
      st_stream(reinterpret_cast<VP*>(p.out) + j, o);
    }
  }
  // scalar remainder (or everything, when unaligned)
  for (int64_t i = nvec * E + gtid; i < n; i += gstride) {
    T v[NIN];
    il_gather<T, OP>(p, i, v);
    P<T> z = apply<T, OP>(v);
    st_stream(p.out + 2 * i, z.a);
    st_stream(p.out + 2 * i + 1, z.b);
  }
}

// Lean variant (aligned arrays; the default only where it measured faster, see
// il_lean_default): one CTA per 256*U
// steps, no chunk or grid-stride loops; the n % E remainder rides in one extra CTA
// as a masked step through the same per-lane compute (as ew_step_kernel).
#ifndef TF_IL_STEP_MIN_BLOCKS
#define TF_IL_STEP_MIN_BLOCKS 4
#endif
template <class T, int OP>
__global__ void __launch_bounds__(256, TF_IL_STEP_MIN_BLOCKS) ew_il_step_kernel(ILArgs<T> p, int64_t n, int64_t nblk) {
  constexpr int NIN = OpInfo<OP>::NIN;
  constexpr int AR = OpInfo<OP>::ARITY;
  constexpr int E = Vec16<T>::N;
  const int64_t nvec = n / E;

  // one step = E elements: a pair operand is one 32-byte vector (E pairs,
  // sm_100 256-bit LDG), a plain plane one 16-byte vector; the result one
  // 32-byte store.
  using VP = Vec32<T>;   // E pairs
  using VS = Vec16A<T>;  // E scalars
  constexpr bool XP = (AR == 22 || AR == 21 || AR == 2);
  // steps in flight per thread (all loads issue before any math); the one-plane
  // op (vtsqrt: 16 bytes in per step) carries 4 to keep enough bytes in flight
  constexpr int U = AR == 1 ? 4 : 2;
  // CTA-chunked, as the split kernels: chunk = 256*U consecutive steps per CTA,
  // thread t takes steps t and t+256 (coalesced, contiguous per CTA)
  const int64_t CH = 256LL * U;
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t cb = (int64_t)blockIdx.x * CH;
    const int64_t base = cb + threadIdx.x;
    VP xp[U], yp[U];
    VS xs[U], ys[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        if constexpr (XP) xp[u] = ld_stream(reinterpret_cast<const VP*>(p.a) + j);
        else xs[u] = ld_stream(reinterpret_cast<const VS*>(p.a) + j);
        if constexpr (AR == 22) yp[u] = ld_stream(reinterpret_cast<const VP*>(p.b) + j);
        else if constexpr (AR == 21 || AR == 11) ys[u] = ld_stream(reinterpret_cast<const VS*>(p.b) + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j >= nvec) continue;
      VP o;
      T v[E][NIN];
#pragma unroll
      for (int e = 0; e < E; e++) {
        if constexpr (XP) {
          v[e][0] = xp[u].v[2 * e];
          v[e][1] = xp[u].v[2 * e + 1];
        } else {
          v[e][0] = xs[u].v[e];
        }
        if constexpr (AR == 22) {
          v[e][2] = yp[u].v[2 * e];
          v[e][3] = yp[u].v[2 * e + 1];
        } else if constexpr (AR == 21) {
          v[e][2] = ys[u].v[e];
        } else if constexpr (AR == 11) {
          v[e][1] = ys[u].v[e];
        }
      }
      P<T> z[E];
      apply_lanes<T, OP, E>(v, z);
#pragma unroll
      for (int e = 0; e < E; e++) {
        o.v[2 * e] = z[e].a;
        o.v[2 * e + 1] = z[e].b;
      }
      st_stream(reinterpret_cast<VP*>(p.out) + j, o);
    }
  } else if (threadIdx.x == 0) {
    // the n % E remainder as one masked step (inactive lanes compute on 1.0)
    const int64_t i0 = nvec * E;
    const int cnt = (int)(n - i0);
    if (cnt > 0) {
      T v[E][NIN];
#pragma unroll
      for (int e = 0; e < E; e++) {
        if (e < cnt) {
          il_gather<T, OP>(p, i0 + e, v[e]);
        } else {
#pragma unroll
          for (int k = 0; k < NIN; k++) v[e][k] = T(1);
        }
      }
      P<T> z[E];
      apply_lanes<T, OP, E>(v, z);
#pragma unroll
      for (int e = 0; e < E; e++)
        if (e < cnt) {
          st_stream(p.out + 2 * (i0 + e), z[e].a);
          st_stream(p.out + 2 * (i0 + e) + 1, z[e].b);
        }
    }
  }
}

template <class T>
__global__ void __launch_bounds__(256) interleave_kernel(const T* __restrict__ v,
                                                         const T* __restrict__ e,
                                                         T* __restrict__ out, int64_t n,
                                                         int vec) {
  using Vt = typename Vec16<T>::type;
  constexpr int E = Vec16<T>::N;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvec = vec ? n / E : 0;
  for (int64_t j = gtid; j < nvec; j += gstride) {
    Vt a = ld_stream(reinterpret_cast<const Vt*>(v) + j);
    Vt b = ld_stream(reinterpret_cast<const Vt*>(e) + j);
    Vt o0, o1;
#pragma unroll
    for (int k = 0; k < E; k++) {
      Vt& o = (2 * k < E) ? o0 : o1;
      set_lane<T>(o, (2 * k) % E, lane<T>(a, k));
      set_lane<T>(o, (2 * k + 1) % E, lane<T>(b, k));
    }
    Vt* po = reinterpret_cast<Vt*>(out) + 2 * j;
    st_stream(po, o0);
    st_stream(po + 1, o1);
  }
  for (int64_t i = nvec * E + gtid; i < n; i += gstride) {
    st_stream(out + 2 * i, ld_stream(v + i));
    st_stream(out + 2 * i + 1, ld_stream(e + i));
  }
}

template <class T>
__global__ void __launch_bounds__(256) deinterleave_kernel(const T* __restrict__ in,
                                                           T* __restrict__ v, T* __restrict__ e,
                                                           int64_t n, int vec) {
  using Vt = typename Vec16<T>::type;
  constexpr int E = Vec16<T>::N;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvec = vec ? n / E : 0;
  for (int64_t j = gtid; j < nvec; j += gstride) {
    const Vt* pi = reinterpret_cast<const Vt*>(in) + 2 * j;
    Vt r0 = ld_stream(pi), r1 = ld_stream(pi + 1);
    Vt a, b;
#pragma unroll
    for (int k = 0; k < E; k++) {
      const Vt& r = (2 * k < E) ? r0 : r1;
      set_lane<T>(a, k, lane<T>(r, (2 * k) % E));
      set_lane<T>(b, k, lane<T>(r, (2 * k + 1) % E));
    }
    st_stream(reinterpret_cast<Vt*>(v) + j, a);
    st_stream(reinterpret_cast<Vt*>(e) + j, b);
  }
  for (int64_t i = nvec * E + gtid; i < n; i += gstride) {
    st_stream(v + i, ld_stream(in + 2 * i));
    st_stream(e + i, ld_stream(in + 2 * i + 1));
  }
}

// ---- lean conversions (the default for 32-byte-aligned arrays) ---------------------
// One CTA per 256*2 vector steps and no loops: a step moves E = 32/sizeof(T)
// elements — two 32-byte loads (one per plane, or two adjacent pair vectors) and two
// 32-byte stores, both steps' loads issued before any store.  The n % E tail rides in
// one extra CTA, one element per thread.  Pure data movement at the vmem copy's 1:1
// read/write mix (16 B in, 16 B out per f64 element).  Measured at 2^27/2^28
// (tools/convert_bench.py, profiles/r2s5_convert_ab.txt): f64 interleave 6.54 ->
// 6.92 TB/s (+6%); the other three conversions ran 1.4-2.3% faster on the 16-byte
// grid-stride kernels above (6.87-7.07 TB/s), so those keep them.  TF_CONV_LEAN=1 /
// =0 force either variant for every conversion (A/B, tests).
template <class T>
__global__ void __launch_bounds__(256) interleave_step_kernel(const T* __restrict__ v,
                                                              const T* __restrict__ e,
                                                              T* __restrict__ out, int64_t n,
                                                              int64_t nvec, int64_t nblk) {
  using V = Vec32<T>;
  constexpr int E = V::N;
  constexpr int U = 2;
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t base = (int64_t)blockIdx.x * (256 * U) + threadIdx.x;
    V a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        a[u] = ld_stream(reinterpret_cast<const V*>(v) + j);
        b[u] = ld_stream(reinterpret_cast<const V*>(e) + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        V o0, o1;
#pragma unroll
        for (int k = 0; k < E / 2; k++) {
          o0.v[2 * k] = a[u].v[k];
          o0.v[2 * k + 1] = b[u].v[k];
          o1.v[2 * k] = a[u].v[E / 2 + k];
          o1.v[2 * k + 1] = b[u].v[E / 2 + k];
        }
        V* po = reinterpret_cast<V*>(out) + 2 * j;
        st_stream(po, o0);
        st_stream(po + 1, o1);
      }
    }
  } else {
    const int64_t i = nvec * E + threadIdx.x;
    if (i < n) {
      st_stream(out + 2 * i, ld_stream(v + i));
      st_stream(out + 2 * i + 1, ld_stream(e + i));
    }
  }
}

template <class T>
__global__ void __launch_bounds__(256) deinterleave_step_kernel(const T* __restrict__ in,
                                                                T* __restrict__ v,
                                                                T* __restrict__ e, int64_t n,
                                                                int64_t nvec, int64_t nblk) {
  using V = Vec32<T>;
  constexpr int E = V::N;
  constexpr int U = 2;
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t base = (int64_t)blockIdx.x * (256 * U) + threadIdx.x;
    V r0[U], r1[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        const V* pi = reinterpret_cast<const V*>(in) + 2 * j;
        r0[u] = ld_stream(pi);
        r1[u] = ld_stream(pi + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        V a, b;
#pragma unroll
        for (int k = 0; k < E / 2; k++) {
          a.v[k] = r0[u].v[2 * k];
          b.v[k] = r0[u].v[2 * k + 1];
          a.v[E / 2 + k] = r1[u].v[2 * k];
          b.v[E / 2 + k] = r1[u].v[2 * k + 1];
        }
        st_stream(reinterpret_cast<V*>(v) + j, a);
        st_stream(reinterpret_cast<V*>(e) + j, b);
      }
    }
  } else {
    const int64_t i = nvec * E + threadIdx.x;
    if (i < n) {
      st_stream(v + i, ld_stream(in + 2 * i));
      st_stream(e + i, ld_stream(in + 2 * i + 1));
    }
  }
}

// ---- dispatch ------------------------------------------------------------------

struct IlEntry {
  const void* fn;
  const void* step_fn;  // lean variant (aligned arrays)
  bool lean_default;    // the lean variant measured faster for this op
};

// Ops whose lean interleaved kernel is the default: f32 vtsqrt1 and vtdiv (+4.6%,
// +2.1% at 2^27); for the rest ew_il_kernel was 0.3-1.5% faster
// (profiles/r2s3_il_lean_ab.txt).  TF_IL_LEAN=1 / =0 force either for every op.
template <class T, int OP>
constexpr bool il_lean_default() {
  return sizeof(T) == 4 && (OP == 11 || OP == 12);
}

template <class T, int OP>
IlEntry make_il() {
  return IlEntry{reinterpret_cast<const void*>(&ew_il_kernel<T, OP>),
                 reinterpret_cast<const void*>(&ew_il_step_kernel<T, OP>),
                 il_lean_default<T, OP>()};
}
template <class T, int... OPS>
struct IlTable {
  static IlEntry* get() {
    static IlEntry t[] = {make_il<T, OPS>()...};
    return t;
  }
};
static IlEntry* il_table(int dtype) {
  if (dtype == TF_F64)
    return IlTable<double, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19,
                   20, 21, 22, 23>::get();
  return IlTable<float, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
                 21, 22, 23>::get();
}

// one CTA per 256 work items: the hardware block scheduler balances the SMs
// (a grid capped at the resident CTAs leaves a tail of idle SMs, -6% on B200)
static int64_t grid_for(int64_t work) {
  int64_t blocks = (work + 255) / 256;
  if (blocks > 0x7fffffffLL) blocks = 0x7fffffffLL;
  return blocks < 1 ? 1 : blocks;
}

int il_launch(int op, int dtype, int64_t n, const void* a, const void* b, void* out,
              cudaStream_t s) {
  if (op < 0 || op >= TF_NUM_OPS) return fail(TF_EINVAL, "tf_elementwise_il: unknown op id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_elementwise_il: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_elementwise_il: negative length");
  if (n == 0) return TF_OK;
  static const int nin_of[TF_NUM_OPS] = {4, 4, 4, 4, 3, 3, 3, 3, 2, 2, 2, 2,
                                         2, 1, 4, 4, 4, 4, 3, 3, 3, 3, 2, 1};
  const bool binary = nin_of[op] >= 2 && op != TF_VTSQRT1;
  if (!a || !out || (binary && !b)) return fail(TF_EINVAL, "tf_elementwise_il: null array");
  const IlEntry& ent = il_table(dtype)[op];
  // pair arrays need 32-byte alignment, plain planes 16-byte
  const int ar = nin_of[op] == 4 ? 22 : nin_of[op] == 3 ? 21 : op == TF_VTSQRT1 ? 2 : nin_of[op] == 2 ? 11 : 1;
  const bool xpairs = ar == 22 || ar == 21 || ar == 2;
  int vec = (xpairs ? aligned32(a) : aligned16(a)) && aligned32(out) &&
            (!binary || (ar == 22 ? aligned32(b) : aligned16(b)));
  const int E = dtype == TF_F64 ? 2 : 4;
  ILArgs<double> p{static_cast<const double*>(a), static_cast<const double*>(b ? b : a),
                   static_cast<double*>(out)};
  const int U = ar == 1 ? 4 : 2;  // steps per thread, as in ew_il_kernel
  static const int lean_env = [] {  // -1 per-op default, 0 never, 1 always
    const char* e = getenv("TF_IL_LEAN");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool lean = lean_env < 0 ? ent.lean_default : lean_env == 1;
  if (vec && lean && n >= E) {
    const int64_t nblk = (n / E + 256LL * U - 1) / (256LL * U);
    const int64_t extra = n % E ? 1 : 0;
    if (nblk + extra <= 0x7fffffffLL) {
      int64_t nb = nblk;
      void* args[] = {&p, &n, &nb};
      return cuda_status(
          cudaLaunchKernel(ent.step_fn, dim3((unsigned)(nblk + extra)), dim3(256), args, 0, s),
          "tf_elementwise_il: launch");
    }
  }
  const int64_t blocks = grid_for(vec ? (n / E + U - 1) / U : n);
  void* args[] = {&p, &n, &vec};
  return cuda_status(cudaLaunchKernel(ent.fn, dim3((unsigned)blocks), dim3(256), args, 0, s),
                     "tf_elementwise_il: launch");
}

int convert_launch(int to_interleaved, int dtype, int64_t n, const void* a, const void* b,
                   void* c, cudaStream_t s) {
  if ((dtype != TF_F32 && dtype != TF_F64) || n < 0)
    return fail(TF_EINVAL, "tf_interleave: bad arguments");
  if (n == 0) return TF_OK;
  const int E = dtype == TF_F64 ? 2 : 4;
  if (!a || !b || !c)
    return fail(TF_EINVAL, to_interleaved ? "tf_interleave: null array"
                                          : "tf_deinterleave: null array");
  static const int lean_env = [] {  // -1 per-conversion default, 0 never, 1 always
    const char* e = getenv("TF_CONV_LEAN");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool lean = lean_env < 0 ? (to_interleaved && dtype == TF_F64) : lean_env == 1;
  const int64_t E32 = 2 * E;  // elements per 32-byte vector
  if (lean && n >= E32 && aligned32(a) && aligned32(b) && aligned32(c)) {
    const int64_t nvec = n / E32;
    const int64_t nblk = (nvec + 511) / 512;
    const int64_t extra = n % E32 ? 1 : 0;
    if (nblk + extra <= 0x7fffffffLL) {
      const unsigned grid = (unsigned)(nblk + extra);
      if (to_interleaved) {
        if (dtype == TF_F64)
          interleave_step_kernel<double><<<grid, 256, 0, s>>>((const double*)a, (const double*)b,
                                                             (double*)c, n, nvec, nblk);
        else
          interleave_step_kernel<float><<<grid, 256, 0, s>>>((const float*)a, (const float*)b,
                                                            (float*)c, n, nvec, nblk);
      } else {
        if (dtype == TF_F64)
          deinterleave_step_kernel<double><<<grid, 256, 0, s>>>(
              (const double*)a, (double*)const_cast<void*>(b), (double*)c, n, nvec, nblk);
        else
          deinterleave_step_kernel<float><<<grid, 256, 0, s>>>(
              (const float*)a, (float*)const_cast<void*>(b), (float*)c, n, nvec, nblk);
      }
      return launch_status(to_interleaved ? "tf_interleave" : "tf_deinterleave");
    }
  }
  if (to_interleaved) {  // a = value, b = error, c = pairs
    if (!a || !b || !c) return fail(TF_EINVAL, "tf_interleave: null array");
    int vec = aligned16(a) && aligned16(b) && aligned16(c);
    const int64_t blocks = grid_for(vec ? n / E : n);
    if (dtype == TF_F64)
      interleave_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(
          (const double*)a, (const double*)b, (double*)c, n, vec);
    else
      interleave_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)a, (const float*)b,
                                                                 (float*)c, n, vec);
  } else {  // a = pairs, b = value out, c = error out
    if (!a || !b || !c) return fail(TF_EINVAL, "tf_deinterleave: null array");
    int vec = aligned16(a) && aligned16(b) && aligned16(c);
    const int64_t blocks = grid_for(vec ? n / E : n);
    if (dtype == TF_F64)
      deinterleave_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(
          (const double*)a, (double*)const_cast<void*>(b), (double*)c, n, vec);
    else
      deinterleave_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
          (const float*)a, (float*)const_cast<void*>(b), (float*)c, n, vec);
  }
  return launch_status(to_interleaved ? "tf_interleave" : "tf_deinterleave");
}

}  // namespace tf
