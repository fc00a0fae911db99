// batch.cu — several registry ops over the same device planes in ONE launch
// (tf_elementwise_batch): the device twin of tf_elementwise_host_batch.
//
// The reference runs each kernel as its own loop over memory (kernels.py:79-113);
// a caller that applies several ops to the same operands (the bench's config-2
// step: add, sub, mul, div over x and y) re-reads every operand plane once per
// op.  Here thread t of chunk c walks vectors j and, for each j, runs every op
// of the batch in order: the first op's 32-byte loads of a plane come from HBM,
// later ops' loads of the same vector hit L1 (or L2), so HBM moves each
// distinct input plane once plus every output plane once.  Per element and op
// the arithmetic is the registry core (apply<T, OP>), so every output is
// bit-identical to running the ops one by one.  No output may overlap any input
// of the batch (no intra-batch chains), checked before the launch.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "tf_math.cuh"

// minimum resident CTAs requested for the batch kernels (A/B builds)
#ifndef TF_BATCH_MINB
#define TF_BATCH_MINB 1
#endif
#ifndef TF_BATCH_STEP_MINB
#define TF_BATCH_STEP_MINB 4
#endif

namespace tf {

constexpr int BMAX = 8;  // ops per launch

template <class T>
struct BatchOp {
  const T* in[4];
  T* out[2];
  int op;
};

template <class T>
struct BatchArgs {
  BatchOp<T> o[BMAX];
  int nops;
};

// Cached read-only 32-byte load: unlike ld_stream it allocates in L1 (and keeps
// the default L2 policy), because the batch's later ops re-read the vector.
__device__ __forceinline__ Vec32<double> ld_keep(const Vec32<double>* p) {
  Vec32<double> r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
      : "l"(p));
  return r;
}
__device__ __forceinline__ Vec32<float> ld_keep(const Vec32<float>* p) {
  Vec32<float> r;
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
        "=f"(r.v[6]), "=f"(r.v[7])
      : "l"(p));
  return r;
}

__device__ __forceinline__ Vec16A<double> ld_keep(const Vec16A<double>* p) {
  Vec16A<double> r;
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  return r;
}
__device__ __forceinline__ Vec16A<float> ld_keep(const Vec16A<float>* p) {
  Vec16A<float> r;
  asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
      : "l"(p));
  return r;
}

template <class T, int OP, class V = Vec32<T>>
__device__ __forceinline__ void batch_vec(const BatchOp<T>& b, int64_t head, int64_t j) {
  constexpr int NIN = OpInfo<OP>::NIN;
  V r[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++) r[k] = ld_keep(reinterpret_cast<const V*>(b.in[k] + head) + j);
  V o0, o1;
  apply_vec<T, OP, V, false>(r, o0, o1);  // intrinsics: fewer registers (A/B r2)
  st_stream(reinterpret_cast<V*>(b.out[0] + head) + j, o0);
  st_stream(reinterpret_cast<V*>(b.out[1] + head) + j, o1);
}

// cnt (< E) elements from s0 as one masked vector (inactive lanes compute on 1.0
// and are not stored): the lean kernel's scalar head and tail
template <class T, int OP>
__device__ __forceinline__ void batch_masked(const BatchOp<T>& b, int64_t s0, int cnt) {
  constexpr int NIN = OpInfo<OP>::NIN;
  using V = Vec32<T>;
  constexpr int E = V::N;
  V r[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++)
#pragma unroll
    for (int e = 0; e < E; e++) r[k].v[e] = e < cnt ? b.in[k][s0 + e] : T(1);
  V o0, o1;
  apply_vec<T, OP, V, false>(r, o0, o1);
#pragma unroll
  for (int e = 0; e < E; e++)
    if (e < cnt) {
      st_stream(b.out[0] + s0 + e, o0.v[e]);
      st_stream(b.out[1] + s0 + e, o1.v[e]);
    }
}

template <class T, int OP>
__device__ __forceinline__ void batch_elem(const BatchOp<T>& b, int64_t i) {
  constexpr int NIN = OpInfo<OP>::NIN;
  T v[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++) v[k] = b.in[k][i];
  P<T> z = apply<T, OP>(v);
  st_stream(b.out[0] + i, z.a);
  st_stream(b.out[1] + i, z.b);
}

#define TF_BATCH_CASES(F) \
  F(0) F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) \
  F(12) F(13) F(14) F(15) F(16) F(17) F(18) F(19) F(20) F(21) F(22) F(23)

template <class T>
__device__ __forceinline__ void dispatch_vec(const BatchOp<T>& b, int64_t head, int64_t j) {
  switch (b.op) {  // warp-uniform
#define TF_CASE(ID) \
  case ID:          \
    batch_vec<T, ID>(b, head, j); \
    break;
    TF_BATCH_CASES(TF_CASE)
#undef TF_CASE
  }
}

template <class T>
__device__ __forceinline__ void dispatch_vec16(const BatchOp<T>& b, int64_t head, int64_t j) {
  switch (b.op) {  // warp-uniform
#define TF_CASE(ID) \
  case ID:          \
    batch_vec<T, ID, Vec16A<T>>(b, head, j); \
    break;
    TF_BATCH_CASES(TF_CASE)
#undef TF_CASE
  }
}

template <class T>
__device__ __forceinline__ void dispatch_masked(const BatchOp<T>& b, int64_t s0, int cnt) {
  switch (b.op) {
#define TF_CASE(ID) \
  case ID:          \
    batch_masked<T, ID>(b, s0, cnt); \
    break;
    TF_BATCH_CASES(TF_CASE)
#undef TF_CASE
  }
}

template <class T>
__device__ __forceinline__ void dispatch_elem(const BatchOp<T>& b, int64_t i) {
  switch (b.op) {
#define TF_CASE(ID) \
  case ID:          \
    batch_elem<T, ID>(b, i); \
    break;
    TF_BATCH_CASES(TF_CASE)
#undef TF_CASE
  }
}

// One CTA per chunk of 256*reps vectors (as ew_kernel); for each vector every op
// of the batch runs in order, so one plane's re-reads are a few hundred cycles
// apart and hit L1.  Scalar head (common misalignment) and tail in the same launch.
template <class T>
__global__ void __launch_bounds__(256, TF_BATCH_MINB) batch_kernel(BatchArgs<T> a, int64_t n, int64_t head,
                                                    int64_t nvec, int reps) {
  constexpr int E = Vec32<T>::N;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int nops = a.nops;
  for (int64_t i = gtid; i < head; i += gstride)
    for (int o = 0; o < nops; o++) dispatch_elem<T>(a.o[o], i);
  for (int64_t i = head + nvec * E + gtid; i < n; i += gstride)
    for (int o = 0; o < nops; o++) dispatch_elem<T>(a.o[o], i);
  const int64_t CH = 256LL * reps;
  for (int64_t cb = (int64_t)blockIdx.x * CH; cb < nvec; cb += (int64_t)gridDim.x * CH) {
#pragma unroll 1
    for (int rr = 0; rr < reps; rr++) {
      const int64_t j = cb + (int64_t)rr * 256 + threadIdx.x;
      if (j < nvec)
#pragma unroll 1
        for (int o = 0; o < nops; o++) dispatch_vec<T>(a.o[o], head, j);
    }
  }
}

// (Tried and removed, session 5: prefetch.global.L2 of the later ops' first-read planes
// at thread start — config 2 -6%, configs 1 and 3 flat, profiles/r2s5_batch_prefetch_ab.txt.)
// Lean variant (the f64 default when every plane shares the 32-byte alignment): one
// CTA per 256 vectors and no loops but the ops, the scalar head and tail as masked
// vectors in one extra CTA (thread 0 head, thread 1 tail) — the loops of
// batch_kernel cost registers the vector body pays for (as ew_step_kernel).
template <class T>
__global__ void __launch_bounds__(256, TF_BATCH_STEP_MINB) batch_step_kernel(BatchArgs<T> a, int64_t n,
                                                                        int64_t head, int64_t nvec,
                                                                        int64_t nblk) {
  constexpr int E = Vec32<T>::N;
  const int nops = a.nops;
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j < nvec)
#pragma unroll 1
      for (int o = 0; o < nops; o++) dispatch_vec<T>(a.o[o], head, j);
  } else if (threadIdx.x < 2) {
    const int64_t s0 = threadIdx.x == 0 ? 0 : head + nvec * E;
    const int cnt = (int)(threadIdx.x == 0 ? head : n - s0);
    if (cnt > 0)
#pragma unroll 1
      for (int o = 0; o < nops; o++) dispatch_masked<T>(a.o[o], s0, cnt);
  }
}

// Lean 16-byte variant: one 16-byte vector per plane per thread, as ew_step16_kernel —
// lighter threads, more resident CTAs.  The f32 default (config 3's three-op batch
// 428.0 -> 430.7 G elem-ops/s); f64 keeps the 32-byte lean kernel (config 2's five-op
// batch 237.7 -> 228-233 at any register cap; profiles/r2s5_batch_v16_ab.txt).
// TF_BATCH_V16=1 / =0 force it on / off for both dtypes (A/B).  Head and tail elements
// (fewer than 32/sizeof(T) each) run scalar in one extra CTA, one element per thread.
#ifndef TF_BATCH_V16_MINB
#define TF_BATCH_V16_MINB 6
#endif
template <class T>
__global__ void __launch_bounds__(256, TF_BATCH_V16_MINB) batch_step16_kernel(BatchArgs<T> a, int64_t n,
                                                                        int64_t head,
                                                                        int64_t nvec16,
                                                                        int64_t nblk) {
  constexpr int E = Vec16A<T>::N;
  const int nops = a.nops;
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j < nvec16)
#pragma unroll 1
      for (int o = 0; o < nops; o++) dispatch_vec16<T>(a.o[o], head, j);
  } else {
    const int64_t t0 = head + nvec16 * E;
    const int64_t i = (int64_t)threadIdx.x < head ? (int64_t)threadIdx.x
                                                  : t0 + ((int64_t)threadIdx.x - head);
    if (i < head || (i >= t0 && i < n))
#pragma unroll 1
      for (int o = 0; o < nops; o++) dispatch_elem<T>(a.o[o], i);
  }
}

int ew_num_inputs(int op);

template <class T>
static int launch_batch(int nops, const int* ops, int64_t n, const void* const* in,
                        void* const* out, cudaStream_t s) {
  static std::atomic<int> mbs_cache{0};
  BatchArgs<T> a{};
  a.nops = nops;
  const size_t tsz = sizeof(T);
  const uintptr_t amask = 31;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(out[0]) & amask;
  bool same = (mis % tsz) == 0;
  for (int o = 0; o < nops; o++) {
    const int nin = ew_num_inputs(ops[o]);
    a.o[o].op = ops[o];
    for (int k = 0; k < nin; k++) {
      a.o[o].in[k] = static_cast<const T*>(in[4 * o + k]);
      same = same && (reinterpret_cast<uintptr_t>(in[4 * o + k]) & amask) == mis;
    }
    for (int k = 0; k < 2; k++) {
      a.o[o].out[k] = static_cast<T*>(out[2 * o + k]);
      same = same && (reinterpret_cast<uintptr_t>(out[2 * o + k]) & amask) == mis;
    }
  }
  const int64_t E = 32 / (int64_t)tsz;
  int64_t head = n, nvec = 0;
  if (same) {
    head = mis ? (int64_t)((32 - mis) / tsz) : 0;
    if (head > n) head = n;
    nvec = (n - head) / E;
  }
  static const bool lean = [] {  // TF_BATCH_LEAN=0 / TF_BATCH_REPS select batch_kernel (A/B)
    const char* e = getenv("TF_BATCH_LEAN");
    const char* r = getenv("TF_BATCH_REPS");
    return !(e && e[0] == '0') && !(r && atoi(r) >= 1);
  }();
  static const int v16_env = [] {  // -1 per-dtype default, 0 never, 1 always
    const char* e = getenv("TF_BATCH_V16");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  const bool v16 = v16_env < 0 ? (lean && sizeof(T) == 4) : v16_env == 1;
  if (v16 && nvec > 0) {
    const int64_t nvec16 = nvec * 2;
    const int64_t nblk = (nvec16 + 255) / 256;
    const int64_t extra = (head > 0 || n - head - nvec * E > 0) ? 1 : 0;
    if (nblk + extra <= 0x7fffffffLL) {
      batch_step16_kernel<T><<<(unsigned)(nblk + extra), 256, 0, s>>>(a, n, head, nvec16, nblk);
      return launch_status("tf_elementwise_batch: launch");
    }
  }
  // f64 only: +1.8% on config 2's five-op batch, while f32 measured 2% slower than
  // batch_kernel on config 3 (profiles/r2s3_batch_ab.txt)
  if (lean && nvec > 0 && sizeof(T) == 8) {
    const int64_t nblk = (nvec + 255) / 256;
    const int64_t extra = (head > 0 || n - head - nvec * E > 0) ? 1 : 0;
    if (nblk + extra <= 0x7fffffffLL) {
      batch_step_kernel<T><<<(unsigned)(nblk + extra), 256, 0, s>>>(a, n, head, nvec, nblk);
      return launch_status("tf_elementwise_batch: launch");
    }
  }
  int mbs = mbs_cache.load(std::memory_order_relaxed);
  if (mbs == 0) {
    int b = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, batch_kernel<T>, 256, 0);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_batch: occupancy");
    mbs = b > 0 ? b : 1;
    mbs_cache.store(mbs, std::memory_order_relaxed);
  }
  const int64_t resident = (int64_t)sm_count() * mbs;
  static const int reps_env = [] {  // TF_BATCH_REPS: A/B of the chunk length (1..64)
    const char* e = getenv("TF_BATCH_REPS");
    const int r = e ? atoi(e) : 0;
    return (r >= 1 && r <= 64) ? r : 0;
  }();
  int reps = reps_env ? reps_env : 1;  // 1 step per CTA: +0.6% over 4 (profiles/r1s2_chunk_reps_hbm.txt)
  while (reps > 1 && nvec / (256LL * reps) < 2 * resident) reps >>= 1;
  const int64_t chunk = 256LL * reps;
  int64_t blocks = nvec > 0 ? (nvec + chunk - 1) / chunk : (n + 255) / 256;
  if (nvec == 0 && blocks > resident) blocks = resident;
  if (blocks > 0x7fffffffLL) blocks = 0x7fffffffLL;
  if (blocks < 1) blocks = 1;
  batch_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(a, n, head, nvec, reps);
  return launch_status("tf_elementwise_batch: launch");
}

}  // namespace tf

using namespace tf;

// nops registry ops over device planes of one length and dtype, ONE launch on
// `stream`.  in: 4 pointers per op (unused trailing inputs NULL), out: 2 per op.
extern "C" int tf_elementwise_batch(int nops, const int* ops, int dtype, int64_t n,
                                    const void* const* in, void* const* out, void* stream) {
  const char* who = "tf_elementwise_batch";
  if (nops < 1 || nops > BMAX || !ops)
    return fail(TF_EINVAL, std::string(who) + ": 1..8 ops per batch");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, std::string(who) + ": planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, std::string(who) + ": negative length");
  for (int o = 0; o < nops; o++)
    if (ew_num_inputs(ops[o]) < 0) return fail(TF_EINVAL, std::string(who) + ": unknown op id");
  if (n == 0) return TF_OK;  // as tf_elementwise: nothing is read or written
  if (!in || !out) return fail(TF_EINVAL, std::string(who) + ": null plane");
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  const uintptr_t span = (uintptr_t)n * tsz;
  for (int o = 0; o < nops; o++) {
    const int nin = ew_num_inputs(ops[o]);
    if (!out[2 * o] || !out[2 * o + 1]) return fail(TF_EINVAL, std::string(who) + ": null plane");
    for (int k = 0; k < nin; k++)
      if (!in[4 * o + k]) return fail(TF_EINVAL, std::string(who) + ": null plane");
  }
  // outputs either coincide (later ops overwrite, as run one by one) or are
  // disjoint: a partial overlap has no per-element order that matches
  for (int w = 0; w < 2 * nops; w++)
    for (int v = w + 1; v < 2 * nops; v++) {
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(out[w]);
      const uintptr_t b0 = reinterpret_cast<uintptr_t>(out[v]);
      if (a0 != b0 && a0 < b0 + span && b0 < a0 + span)
        return fail(TF_EINVAL, std::string(who) + ": out planes overlap each other");
    }
  // no op may read what any op of the batch writes (no intra-batch chains)
  for (int w = 0; w < 2 * nops; w++) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(out[w]);
    for (int o = 0; o < nops; o++)
      for (int k = 0; k < ew_num_inputs(ops[o]); k++) {
        const uintptr_t b0 = reinterpret_cast<uintptr_t>(in[4 * o + k]);
        if (a0 < b0 + span && b0 < a0 + span)
          return fail(TF_EINVAL, std::string(who) + ": out must not alias an input");
      }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dtype == TF_F64 ? launch_batch<double>(nops, ops, n, in, out, s)
                         : launch_batch<float>(nops, ops, n, in, out, s);
}
