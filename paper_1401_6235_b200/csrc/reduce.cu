// reduce.cu — twofold sum / twofold-input sum / dot in the canonical order, and
// the cross-shard combine.
//
// The reference has no reduction API; its only reduction is the serial
// _accumulate fold of _tadd (demos.py:107-113).  These kernels compose the same
// cores (_tadd1, _tadd, _two_prod: arith.py:61-71, fp_core.py:170-173) in a
// fixed, data-parallel order that the CPU oracle restates exactly:
//
//   tile t holds elements [t*L, (t+1)*L), L = V*W*K (V elements per 16-byte
//   vector, W = 256 lanes, K = 128 vectors per lane);
//   lane w folds elements t*L + V*(w + W*k) + v, k-major then v, starting from
//   its first element ((x,+0) | (x0,x1) | TwoProd(x,y));
//   lanes, then tiles, combine in the adjacent-pair (stride-doubling) _tadd tree,
//   lower index on the left, absent nodes skipped (never padded).
//
// One CTA per tile: 256 threads issue 8 x 16-byte loads each per batch
// (coalesced: consecutive lanes read consecutive vectors), fold in registers,
// reduce through warp shuffles and shared memory, and publish a 16-byte tile
// partial.  The last CTA to finish (atomic ticket, never arrival order for the
// arithmetic) folds all tile partials with the same tree, so the whole reduction
// is one launch and bit-deterministic.  HBM-bound: sizeof(T) bytes per element
// per input plane.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "reduce_impl.cuh"
#include "tf_math.cuh"

namespace tf {

// ---- variant 1: register path (LDG.128 batches) --------------------------------
template <class T, int ROP, bool VEC>
__global__ void __launch_bounds__(RW) reduce_kernel(const T* __restrict__ a,
                                                    const T* __restrict__ b, int64_t n,
                                                    int64_t ntiles, P<T>* tiles,
                                                    unsigned* counter, T* out) {
  reduce_tile<T, ROP, VEC>(a, b, n, ntiles, tiles, counter, out, blockIdx.x);
}

// ---- two reductions over the same planes in one pass (tf_reduce_pair) -----------
template <class T, int R1, int R2, bool VEC>
__global__ void __launch_bounds__(RW) reduce_pair_kernel(const T* __restrict__ a,
                                                         const T* __restrict__ b, int64_t n,
                                                         int64_t ntiles, P<T>* tiles1,
                                                         P<T>* tiles2, unsigned* counter,
                                                         T* out1, T* out2) {
  reduce_tile2<T, R1, R2, VEC>(a, b, n, ntiles, tiles1, tiles2, counter, out1, out2, blockIdx.x);
}

// ---- variant 2: TMA bulk-copy path (cp.async.bulk -> smem ring, mbarriers) ------
// A tile is streamed through shared memory in stages of KS k-steps (KS*4 KB per
// plane): one elected thread arms an mbarrier with the byte count and issues
// one bulk copy per plane (UBLKCP); lanes read their 16-byte vectors back from
// shared memory in exactly the canonical order (bank-conflict free: lane w reads
// bytes [16w, 16w+16) of each 4 KB k-row).  NST stages in flight per CTA, two
// CTAs per SM.
// (smem_u32 / mbar_* / bulk_g2s: common.cuh)

template <int ROP>
struct BulkGeo {
  static constexpr int NPL = ROP == TF_RSUM ? 1 : 2;  // planes
  static constexpr int KS = ROP == TF_RSUM ? 8 : 4;   // k-steps per stage
  static constexpr int NST = 3;                        // stages in flight
  static constexpr int STAGE = RW * 16 * KS;           // bytes per plane per stage
  static constexpr int SMEM = NST * NPL * STAGE;       // 96 KB: two CTAs per SM
};

template <class T, int ROP>
__global__ void __launch_bounds__(RW) reduce_bulk_kernel(const T* __restrict__ a,
                                                         const T* __restrict__ b, int64_t n,
                                                         int64_t ntiles, P<T>* tiles,
                                                         unsigned* counter, T* out) {
  using G = BulkGeo<ROP>;
  constexpr int V = Geo<T>::V;
  constexpr int64_t L = Geo<T>::L;
  constexpr int NSTAGES = RK / G::KS;
  using Vt = typename Vec16<T>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[G::NST];
  const int w = threadIdx.x;
  const int64_t t = blockIdx.x;
  const int64_t base = t * L;
  P<T> acc{T(0), T(0)};
  int have = 0;

  if (base + L <= n) {
    const T* planes[2] = {a + base, (ROP == TF_RSUM ? a : b) + base};
    if (w == 0) {
      for (int q = 0; q < G::NST; q++) mbar_init(&bar[q], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int stage, int buf) {
      mbar_expect_tx(&bar[buf], G::NPL * G::STAGE);
#pragma unroll
      for (int pl = 0; pl < G::NPL; pl++)
        bulk_g2s(smem + (buf * G::NPL + pl) * G::STAGE,
                 planes[pl] + (int64_t)stage * G::KS * RW * V, G::STAGE, &bar[buf]);
    };
    if (w == 0)
      for (int q = 0; q < G::NST && q < NSTAGES; q++) issue(q, q);
#pragma unroll 1
    for (int j = 0; j < NSTAGES; j++) {
      const int buf = j % G::NST;
      mbar_wait(&bar[buf], (uint32_t)((j / G::NST) & 1));
      const Vt* sa = reinterpret_cast<const Vt*>(smem + (buf * G::NPL) * G::STAGE) + w;
      const Vt* sb = reinterpret_cast<const Vt*>(smem + (buf * G::NPL + G::NPL - 1) * G::STAGE) + w;
#pragma unroll
      for (int kl = 0; kl < G::KS; kl++) {
        Vt ra = sa[kl * RW];
        Vt rb = ROP == TF_RSUM ? ra : sb[kl * RW];
#pragma unroll
        for (int e = 0; e < V; e++) {
          T x = lane<T>(ra, e);
          T y = (ROP == TF_RSUM) ? x : lane<T>(rb, e);
          if (j == 0 && kl == 0 && e == 0) acc = first_term<T, ROP>(x, y);
          else acc = fold<T, ROP>(acc, x, y);
        }
      }
      fence_proxy_async_smem();  // generic reads before the async-proxy refill
      __syncthreads();  // every lane is done with this buffer
      if (w == 0 && j + G::NST < NSTAGES) issue(j + G::NST, buf);
    }
    have = 1;
  } else {
    fold_scalar<T, ROP>(a, b, n, base, acc, have);
  }
  finish_tile(acc, have, t, ntiles, tiles, counter, out);
}

struct ShardIdx {
  short v[1024];  // indices of the non-empty shards, in shard order
  int m;
};

template <class T>
__global__ void combine_kernel(const T* partials, ShardIdx idx, T* out) {
  // one thread: the skip tree over the m non-empty shards, in shard order
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int m = idx.m;
  if (m == 0) {
    out[0] = T(0);
    out[1] = T(0);
    return;
  }
  P<T> st[40];
  int lv[40];
  int sp = 0;
  for (int q = 0; q < m; q++) {
    P<T> v{partials[2 * idx.v[q]], partials[2 * idx.v[q] + 1]};
    int l = 0;
    while (sp > 0 && lv[sp - 1] == l) {
      v = comb(st[sp - 1], v);
      sp--;
      l++;
    }
    st[sp] = v;
    lv[sp] = l;
    sp++;
  }
  P<T> acc = st[sp - 1];
  for (int s = sp - 2; s >= 0; s--) acc = comb(st[s], acc);
  out[0] = acc.a;
  out[1] = acc.b;
}

// ---- host side -------------------------------------------------------------------

static int64_t tiles_for(int dtype, int64_t n) {
  const int64_t L = dtype == TF_F64 ? Geo<double>::L : Geo<float>::L;
  return (n + L - 1) / L;
}

size_t reduce_ws_bytes(int dtype, int64_t n) {
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  return 256 + (size_t)tiles_for(dtype, n) * 2 * tsz;
}

int reduce_geometry(int dtype, int* V, int* W, int* K) {
  if (dtype != TF_F32 && dtype != TF_F64) return fail(TF_EINVAL, "tf_reduce_geometry: dtype");
  if (V) *V = dtype == TF_F64 ? Geo<double>::V : Geo<float>::V;
  if (W) *W = RW;
  if (K) *K = RK;
  return TF_OK;
}

// Both full-tile paths sit at the read-bandwidth wall (config 4, n=2^30:
// register path 7256 GB/s, bulk path 7191 GB/s); the register path is the
// default, TF_REDUCE_PATH=bulk selects the TMA bulk-copy path.
static bool use_bulk() {
  static const bool v = [] {  // thread-safe one-time init
    const char* e = getenv("TF_REDUCE_PATH");
    return e && e[0] == 'b';
  }();
  return v;
}

template <class T, int ROP>
static int reduce_t(int64_t n, const void* a, const void* b, void* out, void* ws,
                    cudaStream_t s) {
  const int64_t nt = tiles_for(sizeof(T) == 8 ? TF_F64 : TF_F32, n);
  unsigned* counter = static_cast<unsigned*>(ws);
  P<T>* tiles = reinterpret_cast<P<T>*>(static_cast<char*>(ws) + 256);
  const bool vec = aligned16(a) && (ROP == TF_RSUM || aligned16(b));
  const T* pa = static_cast<const T*>(a);
  const T* pb = static_cast<const T*>(b ? b : a);
  T* po = static_cast<T*>(out);
  if (vec && use_bulk()) {
    // per call: the attribute is per device, and the call is cheap
    cudaError_t e = cudaFuncSetAttribute(reduce_bulk_kernel<T, ROP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         BulkGeo<ROP>::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "tf_reduce: smem attribute");
    reduce_bulk_kernel<T, ROP><<<(unsigned)nt, RW, BulkGeo<ROP>::SMEM, s>>>(pa, pb, n, nt, tiles,
                                                                           counter, po);
  } else if (vec) {
    reduce_kernel<T, ROP, true><<<(unsigned)nt, RW, 0, s>>>(pa, pb, n, nt, tiles, counter, po);
  } else {
    reduce_kernel<T, ROP, false><<<(unsigned)nt, RW, 0, s>>>(pa, pb, n, nt, tiles, counter, po);
  }
  return launch_status("tf_reduce");
}

int reduce_launch(int rop, int dtype, int64_t n, const void* a, const void* b, void* out,
                  void* ws, size_t ws_bytes, cudaStream_t s) {
  if (rop < 0 || rop >= TF_NUM_ROPS) return fail(TF_EINVAL, "tf_reduce: unknown reduction id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_reduce: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_reduce: negative length");
  if (!out) return fail(TF_EINVAL, "tf_reduce: null output");
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  if (n == 0) return cuda_status(cudaMemsetAsync(out, 0, 2 * tsz, s), "tf_reduce: zero");
  if (!a || (rop != TF_RSUM && !b)) return fail(TF_EINVAL, "tf_reduce: null plane");
  if (!ws || ws_bytes < reduce_ws_bytes(dtype, n))
    return fail(TF_EINVAL, "tf_reduce: workspace too small");
  if (tiles_for(dtype, n) > 0x7fffffffLL) return fail(TF_EINVAL, "tf_reduce: too many tiles");
#define R(ROP)                                                            \
  case ROP:                                                               \
    return dtype == TF_F64 ? reduce_t<double, ROP>(n, a, b, out, ws, s)   \
                           : reduce_t<float, ROP>(n, a, b, out, ws, s);
  switch (rop) { R(TF_RSUM) R(TF_RSUM2) R(TF_RDOT) }
#undef R
  return TF_EINVAL;
}

template <class T, int R1, int R2>
static int reduce_pair_t(int64_t n, const void* a, const void* b, void* out, void* ws,
                         cudaStream_t s) {
  const int64_t nt = tiles_for(sizeof(T) == 8 ? TF_F64 : TF_F32, n);
  unsigned* counter = static_cast<unsigned*>(ws);
  P<T>* tiles1 = reinterpret_cast<P<T>*>(static_cast<char*>(ws) + 256);
  P<T>* tiles2 = tiles1 + nt;
  constexpr bool NEED_B = R1 != TF_RSUM || R2 != TF_RSUM;
  const bool vec = aligned16(a) && (!NEED_B || aligned16(b));
  const T* pa = static_cast<const T*>(a);
  const T* pb = static_cast<const T*>(b ? b : a);
  T* po = static_cast<T*>(out);
  if (vec)
    reduce_pair_kernel<T, R1, R2, true><<<(unsigned)nt, RW, 0, s>>>(pa, pb, n, nt, tiles1, tiles2,
                                                                   counter, po, po + 2);
  else
    reduce_pair_kernel<T, R1, R2, false><<<(unsigned)nt, RW, 0, s>>>(pa, pb, n, nt, tiles1,
                                                                    tiles2, counter, po, po + 2);
  return launch_status("tf_reduce_pair");
}

int reduce_pair_launch(int r1, int r2, int dtype, int64_t n, const void* a, const void* b,
                       void* out, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (r1 < 0 || r1 >= TF_NUM_ROPS || r2 < 0 || r2 >= TF_NUM_ROPS)
    return fail(TF_EINVAL, "tf_reduce_pair: unknown reduction id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_reduce_pair: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_reduce_pair: negative length");
  if (!out) return fail(TF_EINVAL, "tf_reduce_pair: null output");
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  if (n == 0) return cuda_status(cudaMemsetAsync(out, 0, 4 * tsz, s), "tf_reduce_pair: zero");
  if (!a || ((r1 != TF_RSUM || r2 != TF_RSUM) && !b))
    return fail(TF_EINVAL, "tf_reduce_pair: null plane");
  if (!ws || ws_bytes < 2 * reduce_ws_bytes(dtype, n))
    return fail(TF_EINVAL, "tf_reduce_pair: workspace too small");
  if (tiles_for(dtype, n) > 0x7fffffffLL) return fail(TF_EINVAL, "tf_reduce_pair: too many tiles");
#define RP2(A, B)                                                                    \
  if (r1 == A && r2 == B)                                                            \
    return dtype == TF_F64 ? reduce_pair_t<double, A, B>(n, a, b, out, ws, s)        \
                           : reduce_pair_t<float, A, B>(n, a, b, out, ws, s);
#define RP(A) RP2(A, TF_RSUM) RP2(A, TF_RSUM2) RP2(A, TF_RDOT)
  RP(TF_RSUM) RP(TF_RSUM2) RP(TF_RDOT)
#undef RP
#undef RP2
  return TF_EINVAL;
}

int combine_launch(int dtype, int g, const void* partials, const int64_t* counts, void* out,
                   cudaStream_t s) {
  if (dtype != TF_F32 && dtype != TF_F64) return fail(TF_EINVAL, "tf_combine: dtype");
  if (g < 0 || g > 1024) return fail(TF_EINVAL, "tf_combine: shard count out of range");
  if (!out || (g > 0 && (!partials || !counts))) return fail(TF_EINVAL, "tf_combine: null pointer");
  ShardIdx idx;
  idx.m = 0;
  for (int r = 0; r < g; r++)
    if (counts[r] > 0) idx.v[idx.m++] = (short)r;
  if (dtype == TF_F64)
    combine_kernel<double><<<1, 32, 0, s>>>(static_cast<const double*>(partials), idx,
                                            static_cast<double*>(out));
  else
    combine_kernel<float><<<1, 32, 0, s>>>(static_cast<const float*>(partials), idx,
                                           static_cast<float*>(out));
  return launch_status("tf_combine");
}

}  // namespace tf
