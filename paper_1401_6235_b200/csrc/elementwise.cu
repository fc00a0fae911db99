// elementwise.cu — the 22 twofold kernels (+ the two raw exact-transform loops)
// over split (value, error) planes, f32 and f64.
//
// Replaces the reference loop drivers _loop22/_loop21/_loop11/_loop1u
// (kernels.py:79-113): out[i] = core(in[i]) for every i, each output index
// written exactly once.  HBM-bound: per element the kernel moves
// (NIN + 2) * sizeof(T) bytes and nothing else.
//
// Layout in HBM: each plane is one contiguous 1-D array (SoA, kernels.py:3-5).
// Kernels, all one launch per call and bit-identical to one another:
//   ew_step16_kernel  the default for most ops: one CTA per 256 16-byte vectors, one
//                     vector per plane per thread, <= 32 registers, 8 CTAs per SM
//   ew_step_kernel    32-byte vectors (sm_100's 256-bit LDG.E.NA.EFL2.256 /
//                     STG.E.EF.ENL2.256), one CTA per 256*U vectors; the default for
//                     the one-plane square roots and f32 vtsqrt1
//   ew_kernel         chunked / persistent / 16-byte A/B variants and the all-scalar
//                     path for planes with different misalignments
//   ew_bulk_kernel    TMA-staged inputs (cp.async.bulk ring, mbarriers), opt-in
// Planes that share a common misalignment get a scalar head up to the 32-byte boundary;
// the remainder below one vector is a scalar tail — both inside the same launch.  One
// CTA per chunk lets the hardware block scheduler balance the 148 SMs (a persistent grid
// left a tail of idle SMs: -6..7 points of bandwidth, profiles/README.md).
// TF_EW_V16, TF_EW_LEAN, TF_VEC_BYTES=16, TF_EW_SCHED=persistent, TF_EW_REPS and
// TF_EW_BULK select the variants for A/B measurements.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "tf_math.cuh"

// minimum resident CTAs requested for the vtsqrt1 vector kernel (A/B builds)
#ifndef TF_SQRT_MINB
#define TF_SQRT_MINB 1
#endif
// minimum resident CTAs requested for the other 32-byte-vector kernels (A/B builds)
#ifndef TF_EW_MINB
#define TF_EW_MINB 1
#endif
// minimum resident CTAs requested for the vtdiv2 vector kernel: 4 caps it at 64
// registers (68 otherwise: 3 CTAs/SM) without spilling; +1.0% on config 2's vtdiv2
// (6933 -> 7002 GB/s, profiles/r2s3_minb_ab.txt).  Capping every kernel at 64 lost
// on vtdiv/vtsqrt (spills) and on the batch kernel.
#ifndef TF_DIV2_MINB
#define TF_DIV2_MINB 4
#endif
// 32-byte vectors in flight per plane per thread for vtsqrt1: 1 (two IEEE square
// roots and a division per element keep more elements in flight than registers
// allow: U = 1 holds 56 registers, 4 CTAs per SM; U = 2 held 80-84, 3 CTAs, and
// ran 13% slower — profiles/r2_sqrt_ab.txt)
#ifndef TF_SQRT_U
#define TF_SQRT_U 1
#endif
// 32-byte vectors in flight per thread for the one-plane ops (vtsqrt, sqrt_resid), which
// stay on the 32-byte kernel (A/B builds)
#ifndef TF_U_NIN1
#define TF_U_NIN1 2
#endif
// ... f64: 4 (vtsqrt 6.81 -> 6.84 TB/s; 1 loses 13%; f32 flat — profiles/r2s5_u_nin1_ab.txt)
#ifndef TF_U_NIN1_F64
#define TF_U_NIN1_F64 4
#endif

// shared-memory stages of the TMA-staged variant, by input-plane count (A/B builds)
#ifndef TF_BULK_NST2
#define TF_BULK_NST2 3
#endif
#ifndef TF_BULK_NST3
#define TF_BULK_NST3 3
#endif
#ifndef TF_BULK_NST4
#define TF_BULK_NST4 2
#endif

namespace tf {

template <class T>
struct Planes {
  const T* in[4];
  T* out[2];
};

template <int NIN>
struct Unroll {
  static constexpr int U = NIN >= 4 ? 2 : (NIN == 3 ? 2 : 4);
};

template <class T, int OP>
__device__ __forceinline__ void scalar_elem(const Planes<T>& p, int64_t i) {
  constexpr int NIN = OpInfo<OP>::NIN;
  T v[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++) v[k] = ld_stream(p.in[k] + i);
  P<T> z = apply<T, OP>(v);
  st_stream(p.out[0] + i, z.a);
  st_stream(p.out[1] + i, z.b);
}

// The register path takes the branch-free f64 fast paths (tf_math.cuh
// div_fast/sqrt_fast, all lanes of a vector interleaved) only where that beat the
// intrinsics at the hbm size (profiles/r2_fastpath_ab.txt): vtdiv and vtsqrt,
// +12% and +6%.  For vtdiv2 and vtsqrt1 the interleaved lanes raise registers
// past four resident CTAs per SM and cost more bytes in flight than the ILP
// gains; those keep the intrinsics.
template <int OP>
__host__ __device__ constexpr bool reg_fast_op() {
  return OP == 11 || OP == 13;
}

template <class T, int OP, int VB, int U>
__device__ __forceinline__ void compute_store(const VecN<T, VB> (&r)[U][OpInfo<OP>::NIN],
                                              int64_t base, int64_t nvec, VecN<T, VB>* vo0,
                                              VecN<T, VB>* vo1) {
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t j = base + u * 256;
    if (j < nvec) {
      VecN<T, VB> o0, o1;
      apply_vec<T, OP, VecN<T, VB>, reg_fast_op<OP>()>(r[u], o0, o1);
      st_stream(vo0 + j, o0);
      st_stream(vo1 + j, o1);
    }
  }
}

template <class T, int OP, int VB>
__global__ void __launch_bounds__(256, (OP == 12 && VB == 32) ? TF_SQRT_MINB
                                      : (OP == 3 && VB == 32) ? TF_DIV2_MINB
                                      : VB == 32 ? TF_EW_MINB : 1) ew_kernel(Planes<T> p, int64_t n, int64_t head,
                                                 int64_t nvec, int reps) {
  constexpr int NIN = OpInfo<OP>::NIN;
  using V = VecN<T, VB>;
  constexpr int E = V::N;
  constexpr int U = (VB == 32) ? (OP == 12 ? TF_SQRT_U : (NIN >= 3 ? 1 : (NIN == 1 ? (sizeof(T) == 8 ? TF_U_NIN1_F64 : TF_U_NIN1) : 2))) : Unroll<NIN>::U;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  // PDL (launched with programmatic stream serialization): nothing touches
  // global memory before the predecessor grid has completed; then let the next
  // launch on the stream be scheduled during this grid's tail
  pdl_wait();
  pdl_trigger();

  // scalar head (common misalignment) — or everything, when nvec == 0
  for (int64_t i = gtid; i < head; i += gstride) scalar_elem<T, OP>(p, i);
  // scalar tail
  const int64_t tail0 = head + nvec * E;
  for (int64_t i = tail0 + gtid; i < n; i += gstride) scalar_elem<T, OP>(p, i);

  // vector body: U steps of one VB-byte vector per plane, all loads first
  const V* vin[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++) vin[k] = reinterpret_cast<const V*>(p.in[k] + head);
  V* vo0 = reinterpret_cast<V*>(p.out[0] + head);
  V* vo1 = reinterpret_cast<V*>(p.out[1] + head);

  // CTA-chunked: chunk c = vectors [c*CH, (c+1)*CH), CH = 256*U*reps; thread t
  // takes t, t+256, ... (coalesced).  With one CTA per chunk the hardware block
  // scheduler balances SMs dynamically (no tail of idle SMs); a capped grid
  // strides over chunks.  reps is 1 (2 for vtsqrt1), halved on small planes so
  // that the grid still covers every SM evenly.
  const int64_t CH = 256LL * U * reps;
  for (int64_t cb = (int64_t)blockIdx.x * CH; cb < nvec; cb += (int64_t)gridDim.x * CH) {
#pragma unroll 1
    for (int rr = 0; rr < reps; rr++) {
      const int64_t base = cb + (int64_t)rr * 256 * U + threadIdx.x;
      V r[U][NIN];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t j = base + u * 256;
        if (j < nvec) {
#pragma unroll
          for (int k = 0; k < NIN; k++) r[u][k] = ld_stream(vin[k] + j);
        }
      }
      compute_store<T, OP, VB, U>(r, base, nvec, vo0, vo1);
    }
  }
}

// The scalar head (common misalignment, < E elements) and tail (< E) as two
// masked vectors, thread 0 the head and thread 1 the tail, through the vector
// compute path (inactive lanes compute on 1.0 and are not stored).
template <class T, int OP>
__device__ __forceinline__ void head_tail(const Planes<T>& p, int64_t n, int64_t head,
                                          int64_t nvec) {
  constexpr int NIN = OpInfo<OP>::NIN;
  using V = Vec32<T>;
  constexpr int E = V::N;
  if (threadIdx.x >= 2) return;
  const int64_t s0 = threadIdx.x == 0 ? 0 : head + nvec * E;
  const int64_t cnt = threadIdx.x == 0 ? head : n - s0;
  if (cnt <= 0) return;
  V r[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++)
#pragma unroll
    for (int e = 0; e < E; e++) r[k].v[e] = e < cnt ? p.in[k][s0 + e] : T(1);
  V o0, o1;
  apply_vec<T, OP, V, reg_fast_op<OP>()>(r, o0, o1);
#pragma unroll
  for (int e = 0; e < E; e++)
    if (e < cnt) {
      st_stream(p.out[0] + s0 + e, o0.v[e]);
      st_stream(p.out[1] + s0 + e, o1.v[e]);
    }
}

// ---- lean single-step kernel (the default for 32-byte vectors) ------------------
// One CTA per 256*U vectors and nothing else: no chunk loop, no grid-stride
// loops.  The scalar head (common misalignment, < E elements) and tail (< E)
// ride in ONE extra CTA as two masked vectors — thread 0 the head, thread 1 the
// tail — through the same per-lane compute, so the launch stays single.  Both
// loops cost registers that the vector body pays for even when they never run:
// vtsqrt1 holds 46 here against 56 in ew_kernel (5 resident CTAs per SM instead of
// 4); ew_kernel stays for TF_EW_SCHED=persistent, TF_EW_REPS, 16-byte vectors and
// mixed misalignment (profiles/r2s3_lean_ab.txt).
template <class T, int OP>
__global__ void __launch_bounds__(256, OP == 3 ? TF_DIV2_MINB : TF_EW_MINB)
    ew_step_kernel(Planes<T> p, int64_t n, int64_t head, int64_t nvec, int64_t nblk) {
  constexpr int NIN = OpInfo<OP>::NIN;
  using V = Vec32<T>;
  constexpr int U = (OP == 12 ? TF_SQRT_U : (NIN >= 3 ? 1 : (NIN == 1 ? (sizeof(T) == 8 ? TF_U_NIN1_F64 : TF_U_NIN1) : 2)));
  pdl_wait();
  pdl_trigger();
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t base = (int64_t)blockIdx.x * (256 * U) + threadIdx.x;
    V r[U][NIN];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
#pragma unroll
        for (int k = 0; k < NIN; k++)
          r[u][k] = ld_stream(reinterpret_cast<const V*>(p.in[k] + head) + j);
      }
    }
    compute_store<T, OP, 32, U>(r, base, nvec, reinterpret_cast<V*>(p.out[0] + head),
                                reinterpret_cast<V*>(p.out[1] + head));
  } else {
    head_tail<T, OP>(p, n, head, nvec);
  }
}

// ---- lean 16-byte variant (the default for most ops, see v16_default_op) ------------
// The same single-step structure with ONE 16-byte vector per plane per thread and a
// 32-register cap (__launch_bounds__(256, 8): eight resident CTAs, 2048 threads per SM).
// More, lighter threads beat fewer, fatter ones: latency (HBM, and vtsqrt1's two IEEE
// square roots and a division per element) is hidden by occupancy instead of per-thread
// ILP, and twice as many, half as long CTAs drain a grid with a shorter tail
// (tools/micro/mix11.cu: vtsqrt1 7.01-7.03 TB/s against 6.74-6.83 for the 32-byte
// kernel; profiles/r2s5_mix11.txt).  Alignment contract as ew_step_kernel (head to the
// 32-byte boundary, nvec counts 32-byte vectors); the head and tail elements run scalar
// in one extra CTA, one element per thread.  TF_EW_V16 selects the ops (A/B): unset =
// the per-op default, 0 = none, all = every op.
// (the three- and four-plane division ops spill at 32 registers: 40-48 for those)
template <class T, int OP>
__global__ void __launch_bounds__(256, OP == 3 ? 5 : (OP == 7 || OP == 17 || OP == 21) ? 6 : 8)
    ew_step16_kernel(Planes<T> p, int64_t n, int64_t head, int64_t nvec16, int64_t nblk) {
  constexpr int NIN = OpInfo<OP>::NIN;
  using V = Vec16A<T>;
  constexpr int E = V::N;
  pdl_wait();
  pdl_trigger();
  if ((int64_t)blockIdx.x < nblk) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j < nvec16) {
      V r[NIN];
#pragma unroll
      for (int k = 0; k < NIN; k++) r[k] = ld_stream(reinterpret_cast<const V*>(p.in[k] + head) + j);
      V o0, o1;
      apply_vec<T, OP, V, false>(r, o0, o1);
      st_stream(reinterpret_cast<V*>(p.out[0] + head) + j, o0);
      st_stream(reinterpret_cast<V*>(p.out[1] + head) + j, o1);
    }
  } else {
    // head: elements [0, head); tail: [head + nvec16*E, n) — fewer than 32/sizeof(T) each
    const int64_t t0 = head + nvec16 * E;
    const int64_t i = (int64_t)threadIdx.x < head ? (int64_t)threadIdx.x
                                                  : t0 + ((int64_t)threadIdx.x - head);
    if (i < head || (i >= t0 && i < n)) scalar_elem<T, OP>(p, i);
  }
}

// ---- TMA-staged variant: bulk async copies into a shared-memory ring ------------
// Inputs arrive through cp.async.bulk (the TMA engine's UBLKCP) into NST stages of
// one 256-vector tile (8 KB) per input plane.  Each thread reads its 32-byte
// vectors from shared memory, computes and stores; then the CTA syncs and one
// thread refills the slot with the tile NST ahead — so NST-1 tiles per CTA stay
// in flight while every warp computes, bounded by shared memory instead of
// registers.  That is what vtsqrt1 lacks on the register
// path: two IEEE square roots and a division per element (~41 FP64 instructions)
// leave warps computing, not loading, for most of their time.  Outputs leave as
// 256-bit streaming stores straight from registers.  One CTA per chunk of `reps`
// tiles (the hardware block scheduler balances the SMs); the scalar head and tail
// in one extra CTA (head_tail).  Same per-element core, so outputs are
// bit-identical to ew_kernel.
template <class T, int OP>
struct BulkEw {
  static constexpr int NIN = OpInfo<OP>::NIN;
  static constexpr int TILE = 256 * 32;  // bytes per plane per tile
  static constexpr int NST = NIN <= 2 ? TF_BULK_NST2 : (NIN == 3 ? TF_BULK_NST3 : TF_BULK_NST4);
  static constexpr int SMEM = NST * NIN * TILE;  // 32 KB (2 planes) .. 64 KB (4 planes)
};

template <class T, int OP>
__global__ void __launch_bounds__(256) ew_bulk_kernel(Planes<T> p, int64_t n, int64_t head,
                                                      int64_t nvec, int reps) {
  using B = BulkEw<T, OP>;
  constexpr int NIN = B::NIN;
  using V = Vec32<T>;
  constexpr int E = V::N;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[B::NST];
  pdl_wait();
  pdl_trigger();
  const int64_t ntile = (nvec + 255) / 256;
  const int64_t t0 = (int64_t)blockIdx.x * reps;
  if (t0 >= ntile) {  // the one extra CTA: scalar head and tail
    head_tail<T, OP>(p, n, head, nvec);
    return;
  }
  const int cnt = (int)(ntile - t0 < reps ? ntile - t0 : reps);
  const T* src[NIN];
#pragma unroll
  for (int k = 0; k < NIN; k++) src[k] = p.in[k] + head;
  V* vo0 = reinterpret_cast<V*>(p.out[0] + head);
  V* vo1 = reinterpret_cast<V*>(p.out[1] + head);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < B::NST; q++) mbar_init(&bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int j, int buf) {
    const int64_t v0 = (t0 + j) * 256;
    const int64_t left = nvec - v0;
    const uint32_t bytes = (uint32_t)(left < 256 ? left : 256) * 32u;
    const uint64_t pol = l2_evict_first_policy();
    mbar_expect_tx(&bar[buf], bytes * NIN);
#pragma unroll
    for (int k = 0; k < NIN; k++)
      bulk_g2s_hint(smem + (buf * NIN + k) * B::TILE, src[k] + v0 * E, bytes, &bar[buf], pol);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < B::NST && q < cnt; q++) issue(q, q);
#pragma unroll 1
  for (int j = 0; j < cnt; j++) {
    const int buf = j % B::NST;
    mbar_wait(&bar[buf], (uint32_t)((j / B::NST) & 1));
    const int64_t jv = (t0 + j) * 256 + threadIdx.x;
    const bool act = jv < nvec;
    if (act) {
      V r[NIN];
#pragma unroll
      for (int k = 0; k < NIN; k++)
        r[k] = *reinterpret_cast<const V*>(smem + (buf * NIN + k) * B::TILE + threadIdx.x * 32);
      V o0, o1;
      apply_vec<T, OP, V, reg_fast_op<OP>()>(r, o0, o1);
      st_stream(vo0 + jv, o0);
      st_stream(vo1 + jv, o1);
    }
    // Refill this slot only after every thread has USED its vectors: the refill
    // is an async-proxy write into the slot, and bar.sync alone does not wait
    // for a shared-memory read's data to come back — a read still in flight
    // when thread 0 issued the copy returned the NEXT tile (seen on vtsqrt1,
    // tools/bulk_debug.py).  The other NST-1 slots stay in flight meanwhile.
    __syncthreads();
    if (threadIdx.x == 0 && j + B::NST < cnt) issue(j + B::NST, buf);
  }
}

// ---- dispatch ------------------------------------------------------------------

struct EwEntry {
  const void* fn;  // kernel symbol
  int nin;
  int unroll;
  int reps;  // default chunk length in 256*unroll-vector steps (hbm sweep, profiles)
  std::atomic<int> max_blocks_per_sm;  // occupancy, filled lazily (idempotent)
  const void* step_fn;  // lean single-step kernel (ew_step_kernel), 32-byte vectors only
  const void* bulk_fn;  // TMA-staged variant (ew_bulk_kernel), 32-byte vectors only
  int bulk_smem;
  int bulk_default;  // the bulk variant is the default for this op
  int bulk_reps;     // tiles per CTA
  std::atomic<unsigned> bulk_attr_set;  // per-device bit: max dynamic smem raised
  const void* step16_fn;  // lean 16-byte variant
  bool v16_default;       // ... is the default for this op
};

// Ops whose lean 16-byte kernel is the default: every op but the one-plane square
// roots (vtsqrt, sqrt_resid) and f32 vtsqrt1.  Measured with the 22 registry ops
// launched one after another, as a caller and bench.py run them (2 GiB planes, three
// alternating runs, profiles/r2s5_v16_ab.txt): +0.2...+2.0% for every other op (f64
// vtsqrt1 6.87 -> 7.01 TB/s, vtdiv2 7.02 -> 7.12; bench.py config 2 155.2 -> 157.0 G
// elem-ops/s, config 3 291.5 -> 293.3), -1.7% / -3.4% for vtsqrt and -6.5% for f32
// vtsqrt1 (too few bytes in flight per thread for their latency).  In gpubench's
// context (graph replays of ONE kernel back to back, best of 7) the 32-byte kernel stays
// 0.3-0.6% ahead on the four-plane ops; both records are kept.
template <class T, int OP>
constexpr bool v16_default_op() {
  return OP != 13 && OP != 23 && !(sizeof(T) == 4 && OP == 12);
}

// Ops whose TMA-staged variant is the default: none.  Measured against the
// register path at 2^27/2^28 (profiles/r2_bulk_ab.txt): it wins only while the
// SM clock sits at the power cap (vtsqrt1 +3.5% in a sustained loop) and loses
// 0.5-5% at the bench's clocks, where the register path already keeps enough
// bytes in flight.  TF_EW_BULK=all selects it for every op (A/B runs, tests).
template <class T, int OP>
constexpr bool bulk_default_op() {
  return false;
}

template <class T, int OP, int VB>
EwEntry make_entry() {
  constexpr int NIN = OpInfo<OP>::NIN;
  constexpr int U = (VB == 32) ? (OP == 12 ? TF_SQRT_U : (NIN >= 3 ? 1 : (NIN == 1 ? (sizeof(T) == 8 ? TF_U_NIN1_F64 : TF_U_NIN1) : 2))) : Unroll<NIN>::U;
  // one 256*U-vector step per CTA was fastest for every op at 2^27 (6.9-7.0 TB/s
  // for the 48 B/element ops; profiles/r1s2_chunk_reps_hbm.txt), except vtsqrt1
  // (div + 2 sqrt per element, U = 1): four steps (profiles/r2_sqrt_ab.txt)
  constexpr int REPS = OP == 12 ? 4 : 1;
  return EwEntry{reinterpret_cast<const void*>(&ew_kernel<T, OP, VB>),
                 NIN,
                 U,
                 REPS,
                 {0},
                 reinterpret_cast<const void*>(&ew_step_kernel<T, OP>),
                 reinterpret_cast<const void*>(&ew_bulk_kernel<T, OP>),
                 BulkEw<T, OP>::SMEM,
                 bulk_default_op<T, OP>(),
                 NIN <= 2 ? 8 : 4,
                 {0u},
                 reinterpret_cast<const void*>(&ew_step16_kernel<T, OP>),
                 v16_default_op<T, OP>()};
}

template <class T, int VB, int... OPS>
struct Table {
  static EwEntry* get() {
    static EwEntry t[] = {make_entry<T, OPS, VB>()...};
    return t;
  }
};

#define TF_ALL_OPS 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23
static EwEntry* table_for(int dtype, int vb) {
  if (dtype == TF_F64)
    return vb == 32 ? Table<double, 32, TF_ALL_OPS>::get() : Table<double, 16, TF_ALL_OPS>::get();
  return vb == 32 ? Table<float, 32, TF_ALL_OPS>::get() : Table<float, 16, TF_ALL_OPS>::get();
}

// vector width of the split-layout body: 32-byte (sm_100 256-bit LDG/STG) by
// default; TF_VEC_BYTES=16 selects the 128-bit variant (A/B measurements)
static int vec_bytes() {
  static const int vb = [] {  // thread-safe one-time init
    const char* e = getenv("TF_VEC_BYTES");
    return (e && atoi(e) == 16) ? 16 : 32;
  }();
  return vb;
}

int ew_num_inputs(int op) {
  static const int nin[TF_NUM_OPS] = {4, 4, 4, 4, 3, 3, 3, 3, 2, 2, 2, 2,
                                      2, 1, 4, 4, 4, 4, 3, 3, 3, 3, 2, 1};
  if (op < 0 || op >= TF_NUM_OPS) return TF_EINVAL;
  return nin[op];
}

int ew_launch(int op, int dtype, int64_t n, const void* const* in, void* const* out,
              cudaStream_t stream) {
  if (op < 0 || op >= TF_NUM_OPS) return fail(TF_EINVAL, "tf_elementwise: unknown op id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_elementwise: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_elementwise: negative length");
  if (n == 0) return TF_OK;
  const int VBYTES = vec_bytes();
  EwEntry& ent = table_for(dtype, VBYTES)[op];
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  const int E = (int)(VBYTES / tsz);
  if (!in || !out || !out[0] || !out[1]) return fail(TF_EINVAL, "tf_elementwise: null plane");
  for (int k = 0; k < ent.nin; k++)
    if (!in[k]) return fail(TF_EINVAL, "tf_elementwise: null plane");

  // common misalignment -> scalar head, else all-scalar
  const uintptr_t amask = (uintptr_t)VBYTES - 1;
  uintptr_t mis = reinterpret_cast<uintptr_t>(out[0]) & amask;
  bool same = (mis % tsz) == 0 && (reinterpret_cast<uintptr_t>(out[1]) & amask) == mis;
  for (int k = 0; k < ent.nin; k++)
    same = same && (reinterpret_cast<uintptr_t>(in[k]) & amask) == mis;
  int64_t head, nvec;
  if (same) {
    head = mis ? (int64_t)((VBYTES - mis) / tsz) : 0;
    if (head > n) head = n;
    nvec = (n - head) / E;
  } else {
    head = n;
    nvec = 0;
  }

  // TMA-staged variant (ew_bulk_kernel): TF_EW_BULK=0 never, =all for every op,
  // default per op (bulk_default); chunk = TF_EW_BULK_REPS tiles (default 8 for
// one- and two-plane ops, 4 for three and four planes: profiles/r2_bulk_ab.txt)
  static const int bulk_mode = [] {  // 0 never, 1 default ops, 2 all ops
    const char* e = getenv("TF_EW_BULK");
    if (!e) return 1;
    if (e[0] == '0') return 0;
    if (e[0] == 'a') return 2;
    return 1;
  }();
  if (VBYTES == 32 && nvec > 0 && (bulk_mode == 2 || (bulk_mode == 1 && ent.bulk_default))) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise: device");
    const unsigned bit = 1u << (dev & 31);
    if (!(ent.bulk_attr_set.load(std::memory_order_acquire) & bit)) {
      e = cudaFuncSetAttribute(ent.bulk_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               ent.bulk_smem);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise: smem attribute");
      ent.bulk_attr_set.fetch_or(bit, std::memory_order_acq_rel);
    }
    static const int breps = [] {
      const char* r = getenv("TF_EW_BULK_REPS");
      const int v = r ? atoi(r) : 0;
      return (v >= 1 && v <= 256) ? v : 0;
    }();
    const int64_t ntile = (nvec + 255) / 256;
    // keep at least ~4 CTAs per SM worth of chunks on small planes
    int reps = breps ? breps : ent.bulk_reps;
    while (reps > 1 && ntile / reps < 4LL * sm_count()) reps >>= 1;
    int64_t blocks = (ntile + reps - 1) / reps;  // >= 1: nvec > 0 here
    if (head > 0 || n - head - nvec * E > 0) blocks++;  // the head_tail CTA
    if (blocks > 0x7fffffffLL) return fail(TF_EINVAL, "tf_elementwise: plane too long");
    Planes<double> p{};
    for (int k = 0; k < ent.nin; k++) p.in[k] = static_cast<const double*>(in[k]);
    p.out[0] = static_cast<double*>(out[0]);
    p.out[1] = static_cast<double*>(out[1]);
    void* args[] = {&p, &n, &head, &nvec, &reps};
    e = launch_pdl(ent.bulk_fn, dim3((unsigned)blocks), dim3(256), args, ent.bulk_smem, stream);
    return cuda_status(e, "tf_elementwise: launch");
  }

  // lean single-step kernel: the default for 32-byte vectors (TF_EW_LEAN=0, a
  // TF_EW_REPS override or TF_EW_SCHED=persistent select ew_kernel)
  static const bool lean = [] {
    const char* e = getenv("TF_EW_LEAN");
    return !(e && e[0] == '0');
  }();
  static const bool reps_override = [] {
    const char* e = getenv("TF_EW_REPS");
    return e && atoi(e) >= 1;
  }();
  static const bool persistent_env = [] {
    const char* e = getenv("TF_EW_SCHED");
    return e && e[0] == 'p';
  }();
  static const int v16_mode = [] {  // 0 never, 1 per-op default, 2 every op
    const char* e = getenv("TF_EW_V16");
    if (!e) return 1;
    if (e[0] == '0') return 0;
    return e[0] == 'a' ? 2 : 1;
  }();
  if (VBYTES == 32 && nvec > 0 && lean && !reps_override && !persistent_env &&
      (v16_mode == 2 || (v16_mode == 1 && ent.v16_default))) {
    const int64_t nvec16 = nvec * 2;
    const int64_t nblk = (nvec16 + 255) / 256;
    const int64_t extra = (head > 0 || n - head - nvec * E > 0) ? 1 : 0;
    if (nblk + extra <= 0x7fffffffLL) {
      Planes<double> p{};
      for (int k = 0; k < ent.nin; k++) p.in[k] = static_cast<const double*>(in[k]);
      p.out[0] = static_cast<double*>(out[0]);
      p.out[1] = static_cast<double*>(out[1]);
      int64_t nb = nblk, nv = nvec16;
      void* args[] = {&p, &n, &head, &nv, &nb};
      cudaError_t e = launch_pdl(ent.step16_fn, dim3((unsigned)(nblk + extra)), dim3(256), args,
                                 0, stream);
      return cuda_status(e, "tf_elementwise: launch");
    }
  }
  if (VBYTES == 32 && nvec > 0 && lean && !reps_override && !persistent_env) {
    const int64_t per = 256LL * ent.unroll;
    const int64_t nblk = (nvec + per - 1) / per;
    const int64_t extra = (head > 0 || n - head - nvec * E > 0) ? 1 : 0;
    if (nblk + extra <= 0x7fffffffLL) {
      Planes<double> p{};
      for (int k = 0; k < ent.nin; k++) p.in[k] = static_cast<const double*>(in[k]);
      p.out[0] = static_cast<double*>(out[0]);
      p.out[1] = static_cast<double*>(out[1]);
      int64_t nb = nblk;
      void* args[] = {&p, &n, &head, &nvec, &nb};
      cudaError_t e = launch_pdl(ent.step_fn, dim3((unsigned)(nblk + extra)), dim3(256), args, 0,
                                 stream);
      return cuda_status(e, "tf_elementwise: launch");
    }
  }

  int mbs = ent.max_blocks_per_sm.load(std::memory_order_relaxed);
  if (mbs == 0) {
    int b = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ent.fn, 256, 0);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise: occupancy");
    mbs = b > 0 ? b : 1;
    ent.max_blocks_per_sm.store(mbs, std::memory_order_relaxed);
  }
  // one CTA per chunk of 256*U*reps vectors (hardware-balanced); reps per op
  // (ent.reps), halved while that leaves fewer than two full waves of resident
  // CTAs (small planes).  TF_EW_REPS overrides it for A/B runs;
  // TF_EW_SCHED=persistent caps the grid at the resident CTAs (A/B runs).
  const int64_t resident = (int64_t)sm_count() * mbs;
  static const int reps_env = [] {  // thread-safe one-time init
    const char* e = getenv("TF_EW_REPS");
    const int r = e ? atoi(e) : 0;
    return (r >= 1 && r <= 64) ? r : 0;
  }();
  int reps = reps_env ? reps_env : ent.reps;
  while (reps > 1 && nvec / (256LL * ent.unroll * reps) < 2 * resident) reps >>= 1;
  const int64_t chunk = 256LL * ent.unroll * reps;
  int64_t blocks = nvec > 0 ? (nvec + chunk - 1) / chunk : (n + 255) / 256;
  static const bool persistent = [] {
    const char* e = getenv("TF_EW_SCHED");
    return e && e[0] == 'p';
  }();
  const int64_t cap = persistent || nvec == 0 ? resident : (int64_t)0x7fffffff;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;

  Planes<double> p{};  // bit-identical layout for float: only pointers
  for (int k = 0; k < ent.nin; k++) p.in[k] = static_cast<const double*>(in[k]);
  p.out[0] = static_cast<double*>(out[0]);
  p.out[1] = static_cast<double*>(out[1]);
  void* args[] = {&p, &n, &head, &nvec, &reps};
  cudaError_t e = launch_pdl(ent.fn, dim3((unsigned)blocks), dim3(256), args, 0, stream);
  return cuda_status(e, "tf_elementwise: launch");
}

// ---- dotted baselines + copy (bench.py:56-87) --------------------------------

template <class T, int BASE>
__global__ void __launch_bounds__(256) dotted_kernel(const T* __restrict__ x,
                                                     const T* __restrict__ y, T* __restrict__ r,
                                                     int64_t n) {
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gtid; i < n; i += gstride) {
    T a = ld_stream(x + i), v;
    if constexpr (BASE == 0) v = add(a, ld_stream(y + i));
    else if constexpr (BASE == 1) v = mul(a, ld_stream(y + i));
    else if constexpr (BASE == 2) v = dvd(a, ld_stream(y + i));
    else if constexpr (BASE == 3) v = sqr(a);
    else v = a;
    st_stream(r + i, v);
  }
}

// The dotted baselines get the same memory design as the twofold kernels (32-byte
// vectors, one CTA per chunk of 256*U vectors), so the ratio column compares like
// with like.
template <class T, int BASE>
__global__ void __launch_bounds__(256) dotted_vec_kernel(const Vec32<T>* __restrict__ x,
                                                         const Vec32<T>* __restrict__ y,
                                                         Vec32<T>* __restrict__ r, int64_t nvec) {
  constexpr int E = Vec32<T>::N;
  constexpr int U = 2;
  const int64_t CH = 256LL * U;
  for (int64_t cb = (int64_t)blockIdx.x * CH; cb < nvec; cb += (int64_t)gridDim.x * CH) {
    Vec32<T> a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = cb + u * 256 + threadIdx.x;
      if (j < nvec) {
        a[u] = ld_stream(x + j);
        if constexpr (BASE <= 2) b[u] = ld_stream(y + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t j = cb + u * 256 + threadIdx.x;
      if (j < nvec) {
        Vec32<T> o;
#pragma unroll
        for (int e = 0; e < E; e++) {
          const T s = a[u].v[e];
          T v;
          if constexpr (BASE == 0) v = add(s, b[u].v[e]);
          else if constexpr (BASE == 1) v = mul(s, b[u].v[e]);
          else if constexpr (BASE == 2) v = dvd(s, b[u].v[e]);
          else if constexpr (BASE == 3) v = sqr(s);
          else v = s;
          o.v[e] = v;
        }
        st_stream(r + j, o);
      }
    }
  }
}

template <class T, int BASE>
static int dotted_t(int64_t n, const void* x, const void* y, void* r, cudaStream_t s) {
  constexpr int E = Vec32<T>::N;
  const int64_t cap = 0x7fffffffLL;  // one CTA per chunk: hardware-balanced
  const bool vec = aligned32(x) && aligned32(r) && (BASE > 2 || aligned32(y)) && n % E == 0;
  if (vec) {
    const int64_t nvec = n / E;
    int64_t blocks = (nvec + 511) / 512;
    blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
    dotted_vec_kernel<T, BASE><<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<const Vec32<T>*>(x), static_cast<const Vec32<T>*>(y ? y : x),
        static_cast<Vec32<T>*>(r), nvec);
  } else {
    int64_t blocks = (n + 255) / 256;
    blocks = blocks < 1 ? 1 : (blocks > cap ? cap : blocks);
    dotted_kernel<T, BASE><<<(unsigned)blocks, 256, 0, s>>>(
        static_cast<const T*>(x), static_cast<const T*>(y ? y : x), static_cast<T*>(r), n);
  }
  return launch_status("tf_dotted");
}

int dotted_launch(int base, int dtype, int64_t n, const void* x, const void* y, void* r,
                  cudaStream_t s) {
  if (n < 0 || (dtype != TF_F32 && dtype != TF_F64) || base < 0 || base > 4 || !x || !r)
    return fail(TF_EINVAL, "tf_dotted: bad arguments");
  if (n == 0) return TF_OK;
  if (base <= 2 && !y) return fail(TF_EINVAL, "tf_dotted: null y");
#define D(B)                                                                       \
  case B:                                                                          \
    return dtype == TF_F64 ? dotted_t<double, B>(n, x, y, r, s) : dotted_t<float, B>(n, x, y, r, s);
  switch (base) { D(0) D(1) D(2) D(3) D(4) }
#undef D
  return TF_EINVAL;
}

}  // namespace tf
