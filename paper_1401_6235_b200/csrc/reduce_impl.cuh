// reduce_impl.cuh — the canonical-order reduction machinery shared by the
// reduction kernels (reduce.cu) and the fused reduce + NVLink exchange kernel
// (xgpu.cu).  See reduce.cu for the order itself.
#pragma once

#include "common.cuh"
#include "tf_math.cuh"

namespace tf {

constexpr int RW = 256;  // lanes per tile
constexpr int RK = 128;  // vectors per lane
constexpr int RKB = 8;   // vectors per load batch (two planes)
#ifndef TF_RKB_SUM
#define TF_RKB_SUM 16        // one plane: twice the batch keeps the same bytes in flight
#endif

template <class T>
struct Geo {
  static constexpr int V = Vec16<T>::N;
  static constexpr int64_t L = (int64_t)V * RW * RK;
};

// fold one element into a lane accumulator
template <class T, int ROP>
__device__ __forceinline__ P<T> first_term(T x, T y) {
  if constexpr (ROP == TF_RSUM) return {x, T(0)};
  else if constexpr (ROP == TF_RSUM2) return {x, y};
  else return two_prod(x, y);
}
template <class T, int ROP>
__device__ __forceinline__ P<T> fold(P<T> acc, T x, T y) {
  if constexpr (ROP == TF_RSUM) return tadd1(acc.a, acc.b, x);
  else if constexpr (ROP == TF_RSUM2) return tadd(acc.a, acc.b, x, y);
  else {
    P<T> p = two_prod(x, y);
    return tadd(acc.a, acc.b, p.a, p.b);
  }
}

template <class T>
__device__ __forceinline__ P<T> comb(P<T> l, P<T> r) {
  return tadd(l.a, l.b, r.a, r.b);
}

// adjacent-pair tree across the 32 lanes of a warp (absent lanes form a suffix)
template <class T>
__device__ __forceinline__ void warp_tree(P<T>& acc, int& have, int lane, int width) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    if (off >= width) break;
    T oa = __shfl_down_sync(0xffffffffu, acc.a, off);
    T ob = __shfl_down_sync(0xffffffffu, acc.b, off);
    int oh = __shfl_down_sync(0xffffffffu, have, off);
    if ((lane & (2 * off - 1)) == 0 && oh && (lane + off) < width) {
      acc = comb(acc, P<T>{oa, ob});
    }
  }
}

// Sequential evaluation of the skip tree over items [lo, hi) of an aligned block:
// binary-counter stack, then a right fold of what is left.
template <class T>
__device__ __forceinline__ P<T> block_tree(const P<T>* items, int64_t lo, int64_t hi) {
  P<T> st[40];
  int lv[40];
  int sp = 0;
  for (int64_t i = lo; i < hi; i++) {
    P<T> v = P<T>{__ldcg(&items[i].a), __ldcg(&items[i].b)};
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
  return acc;
}

// CTA-wide skip tree over one value per thread (threads with have==0 form a suffix)
template <class T>
__device__ __forceinline__ P<T> cta_tree(P<T> acc, int have, int* have_out) {
  __shared__ T sa[RW / 32], sb[RW / 32];
  __shared__ int sh[RW / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_tree(acc, have, lane, 32);
  if (lane == 0) {
    sa[warp] = acc.a;
    sb[warp] = acc.b;
    sh[warp] = have;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = RW / 32;
    P<T> w = lane < nw ? P<T>{sa[lane], sb[lane]} : P<T>{T(0), T(0)};
    int h = lane < nw ? sh[lane] : 0;
    warp_tree(w, h, lane, nw);
    acc = w;
    have = h;
  }
  *have_out = have;
  return acc;
}

// partial tile or unaligned planes: the canonical order, scalar loads, bounds checked
template <class T, int ROP>
__device__ __forceinline__ void fold_scalar(const T* a, const T* b, int64_t n, int64_t base,
                                            P<T>& acc, int& have) {
  constexpr int V = Geo<T>::V;
  const int w = threadIdx.x;
  for (int k = 0; k < RK; k++) {
    for (int e = 0; e < V; e++) {
      const int64_t i = base + (int64_t)V * (w + (int64_t)RW * k) + e;
      if (i >= n) continue;
      T x = ld_stream(a + i);
      T y = (ROP == TF_RSUM) ? x : ld_stream(b + i);
      if (!have) {
        acc = first_term<T, ROP>(x, y);
        have = 1;
      } else {
        acc = fold<T, ROP>(acc, x, y);
      }
    }
  }
}

// lane tree -> tile partial; the last CTA (atomic ticket) runs the tile tree
template <class T>
__device__ __forceinline__ bool finish_tile(P<T> acc, int have, int64_t t, int64_t ntiles,
                                            P<T>* tiles, unsigned* counter, T* out) {
  int h;
  acc = cta_tree(acc, have, &h);

  __shared__ int is_last;
  if (threadIdx.x == 0) {
    tiles[t].a = acc.a;
    tiles[t].b = acc.b;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    is_last = (prev == (unsigned)(ntiles - 1));
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();

  // last CTA: the tile tree.  Thread j owns the aligned block of B2 tiles
  // [j*B2, (j+1)*B2); blocks are complete subtrees, so block trees followed by
  // the CTA tree reproduce the global adjacent-pair tree exactly.
  int64_t per = (ntiles + RW - 1) / RW;
  int64_t B2 = 1;
  while (B2 < per) B2 <<= 1;
  const int64_t lo = (int64_t)threadIdx.x * B2;
  const int64_t hi = lo + B2 < ntiles ? lo + B2 : ntiles;
  P<T> part{T(0), T(0)};
  int ph = 0;
  if (lo < ntiles) {
    part = block_tree(tiles, lo, hi);
    ph = 1;
  }
  __syncthreads();  // shared scratch of cta_tree is reused
  part = cta_tree(part, ph, &h);
  if (threadIdx.x == 0) {
    out[0] = part.a;
    out[1] = part.b;
    *counter = 0u;  // leave the workspace ready for the next call
  }
  return true;
}

// ---- variant 1: register path (LDG.128 batches) --------------------------------
// Tile t, one per CTA; returns true in the last CTA (after it wrote out[0..1]).
template <class T, int ROP, bool VEC>
__device__ __forceinline__ bool reduce_tile(const T* __restrict__ a, const T* __restrict__ b,
                                            int64_t n, int64_t ntiles, P<T>* tiles,
                                            unsigned* counter, T* out, int64_t t) {
  constexpr int V = Geo<T>::V;
  constexpr int64_t L = Geo<T>::L;
  using Vt = typename Vec16<T>::type;
  const int w = threadIdx.x;
  const int64_t base = t * L;
  P<T> acc{T(0), T(0)};
  int have = 0;

  if (VEC && base + L <= n) {
    // full tile, 16-byte aligned planes
    const Vt* va = reinterpret_cast<const Vt*>(a + base) + w;
    const Vt* vb = reinterpret_cast<const Vt*>((ROP == TF_RSUM ? a : b) + base) + w;
    constexpr int KB = ROP == TF_RSUM ? TF_RKB_SUM : RKB;
#pragma unroll 1
    for (int k0 = 0; k0 < RK; k0 += KB) {
      Vt ra[KB], rb[ROP == TF_RSUM ? 1 : KB];
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
        ra[kb] = ld_stream(va + (int64_t)RW * (k0 + kb));
        if constexpr (ROP != TF_RSUM) rb[kb] = ld_stream(vb + (int64_t)RW * (k0 + kb));
      }
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
#pragma unroll
        for (int e = 0; e < V; e++) {
          T x = lane<T>(ra[kb], e);
          T y = x;
          if constexpr (ROP != TF_RSUM) y = lane<T>(rb[kb], e);
          if (k0 == 0 && kb == 0 && e == 0) acc = first_term<T, ROP>(x, y);
          else acc = fold<T, ROP>(acc, x, y);
        }
      }
    }
    have = 1;
  } else {
    fold_scalar<T, ROP>(a, b, n, base, acc, have);
  }
  return finish_tile(acc, have, t, ntiles, tiles, counter, out);
}



// ---- two reductions in one pass -------------------------------------------------
// Lane fold of two reductions over the same planes (a, b): each accumulator in its
// own canonical order, so each result is bit-identical to its single reduction;
// the planes are read once.
template <class T, int R1, int R2>
__device__ __forceinline__ void fold2(P<T>& acc1, P<T>& acc2, int& have, T x, T y) {
  if (!have) {
    acc1 = first_term<T, R1>(x, y);
    acc2 = first_term<T, R2>(x, y);
    have = 1;
  } else {
    acc1 = fold<T, R1>(acc1, x, y);
    acc2 = fold<T, R2>(acc2, x, y);
  }
}

// lane trees -> two tile partials; the last CTA (one ticket) runs both tile trees
template <class T>
__device__ __forceinline__ bool finish_tile2(P<T> acc1, P<T> acc2, int have, int64_t t,
                                             int64_t ntiles, P<T>* tiles1, P<T>* tiles2,
                                             unsigned* counter, T* out1, T* out2) {
  int h;
  acc1 = cta_tree(acc1, have, &h);
  __syncthreads();  // shared scratch of cta_tree is reused
  acc2 = cta_tree(acc2, have, &h);
  __shared__ int is_last;
  if (threadIdx.x == 0) {
    tiles1[t] = acc1;
    tiles2[t] = acc2;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    is_last = (prev == (unsigned)(ntiles - 1));
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  int64_t per = (ntiles + RW - 1) / RW;
  int64_t B2 = 1;
  while (B2 < per) B2 <<= 1;
  const int64_t lo = (int64_t)threadIdx.x * B2;
  const int64_t hi = lo + B2 < ntiles ? lo + B2 : ntiles;
  P<T>* const tl[2] = {tiles1, tiles2};
  T* const outs[2] = {out1, out2};
#pragma unroll 1
  for (int r = 0; r < 2; r++) {
    P<T> part{T(0), T(0)};
    int ph = 0;
    if (lo < ntiles) {
      part = block_tree(tl[r], lo, hi);
      ph = 1;
    }
    __syncthreads();
    part = cta_tree(part, ph, &h);
    if (threadIdx.x == 0) {
      outs[r][0] = part.a;
      outs[r][1] = part.b;
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

template <class T, int R1, int R2, bool VEC>
__device__ __forceinline__ bool reduce_tile2(const T* __restrict__ a, const T* __restrict__ b,
                                             int64_t n, int64_t ntiles, P<T>* tiles1,
                                             P<T>* tiles2, unsigned* counter, T* out1, T* out2,
                                             int64_t t) {
  constexpr int V = Geo<T>::V;
  constexpr int64_t L = Geo<T>::L;
  constexpr bool ONE = R1 == TF_RSUM && R2 == TF_RSUM;  // only plane a is read
  using Vt = typename Vec16<T>::type;
  const int w = threadIdx.x;
  const int64_t base = t * L;
  P<T> acc1{T(0), T(0)}, acc2{T(0), T(0)};
  int have = 0;
  if (VEC && base + L <= n) {
    const Vt* va = reinterpret_cast<const Vt*>(a + base) + w;
    const Vt* vb = reinterpret_cast<const Vt*>((ONE ? a : b) + base) + w;
    constexpr int KB = ONE ? TF_RKB_SUM : RKB;
#pragma unroll 1
    for (int k0 = 0; k0 < RK; k0 += KB) {
      Vt ra[KB], rb[ONE ? 1 : KB];
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
        ra[kb] = ld_stream(va + (int64_t)RW * (k0 + kb));
        if constexpr (!ONE) rb[kb] = ld_stream(vb + (int64_t)RW * (k0 + kb));
      }
#pragma unroll
      for (int kb = 0; kb < KB; kb++) {
#pragma unroll
        for (int e = 0; e < V; e++) {
          T x = lane<T>(ra[kb], e);
          T y = x;
          if constexpr (!ONE) y = lane<T>(rb[kb], e);
          if (k0 == 0 && kb == 0 && e == 0) {
            acc1 = first_term<T, R1>(x, y);
            acc2 = first_term<T, R2>(x, y);
          } else {
            acc1 = fold<T, R1>(acc1, x, y);
            acc2 = fold<T, R2>(acc2, x, y);
          }
        }
      }
    }
    have = 1;
  } else {
    for (int k = 0; k < RK; k++) {
      for (int e = 0; e < V; e++) {
        const int64_t i = base + (int64_t)V * (w + (int64_t)RW * k) + e;
        if (i >= n) continue;
        T x = ld_stream(a + i);
        T y = ONE ? x : ld_stream(b + i);
        fold2<T, R1, R2>(acc1, acc2, have, x, y);
      }
    }
  }
  return finish_tile2(acc1, acc2, have, t, ntiles, tiles1, tiles2, counter, out1, out2);
}

}  // namespace tf
