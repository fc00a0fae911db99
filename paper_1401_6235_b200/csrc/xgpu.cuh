// xgpu.cuh — the NVLink mailbox exchange protocol (see xgpu.cu), as a device
// function shared by the exchange kernel, the one-GPU emulation and the fused
// reduce + exchange kernel.
#pragma once

#include "common.cuh"
#include "tf_math.cuh"

namespace tf {

constexpr int XG_MAXG = 64;

struct Slot {
  double z0, z1;
  unsigned long long seq;
  unsigned long long pad;
};

struct XArgs {
  Slot* box[XG_MAXG];  // mailbox base of every rank, as mapped on this device
  int rank, world;
  unsigned long long epoch;
  unsigned long long nonempty_lo, nonempty_hi;  // bitmask of ranks with count > 0
};

template <class T>
__device__ __forceinline__ P<T> xcomb(P<T> l, P<T> r) {
  return tadd(l.a, l.b, r.a, r.b);
}

// The protocol, for one rank; run by one thread.  Shared by the real transport
// kernel (one rank per GPU) and the one-GPU emulation (one rank per block).
// Phase 1 (publish): this rank's partial into every mailbox, one system fence,
// then the epoch flags.
template <class T>
__device__ void xgpu_publish(const T* out, const XArgs& x) {
  const int par = (int)(x.epoch & 1);
  const volatile T* mine_v = out;
  const double z0 = (double)mine_v[0], z1 = (double)mine_v[1];
  for (int r = 0; r < x.world; r++) {
    volatile Slot* s = x.box[r] + par * XG_MAXG + x.rank;
    s->z0 = z0;
    s->z1 = z1;
  }
  __threadfence_system();
  for (int r = 0; r < x.world; r++) {
    volatile Slot* s = x.box[r] + par * XG_MAXG + x.rank;
    s->seq = x.epoch;
  }
}

// Phase 2 (collect): wait (bounded) for every rank's slot of this epoch in the
// local mailbox, then fold the non-empty ranks' partials into out.
template <class T>
__device__ void xgpu_collect(T* out, const XArgs& x, int* status) {
  const int par = (int)(x.epoch & 1);
  volatile Slot* mine = x.box[x.rank] + par * XG_MAXG;
  const long long t0 = clock64();
  for (int r = 0; r < x.world; r++) {
    while (mine[r].seq != x.epoch) {
      if (clock64() - t0 > 20000000000LL) {  // ~10 s at 2 GHz: give up, never hang
        out[0] = out[1] = T(NAN);
        *status = 1;
        return;
      }
    }
  }
  __threadfence_system();
  // skip tree over the non-empty ranks, in rank order (as tf_combine)
  P<T> st[8];
  int lv[8];
  int sp = 0, m = 0;
  for (int r = 0; r < x.world; r++) {
    const bool present = r < 64 && ((r < 32 ? (x.nonempty_lo >> r) : (x.nonempty_hi >> (r - 32))) & 1ull);
    if (!present) continue;
    P<T> v{(T)mine[r].z0, (T)mine[r].z1};
    m++;
    int l = 0;
    while (sp > 0 && lv[sp - 1] == l) {
      v = xcomb(st[sp - 1], v);
      sp--;
      l++;
    }
    st[sp] = v;
    lv[sp] = l;
    sp++;
  }
  if (m == 0) {
    out[0] = T(0);
    out[1] = T(0);
    return;
  }
  P<T> acc = st[sp - 1];
  for (int s = sp - 2; s >= 0; s--) acc = xcomb(st[s], acc);
  out[0] = acc.a;
  out[1] = acc.b;
}

template <class T>
__device__ void xgpu_exchange(T* out, const XArgs& x, int* status) {
  xgpu_publish(out, x);
  xgpu_collect(out, x, status);
}

}  // namespace tf
