// xgpu.cu — cross-GPU combine of reduction partials over NVLink peer memory,
// without NCCL (opt-in transport; the default multi-GPU path all-gathers the
// 16-byte partials with NCCL and runs tf_combine).
//
// Every rank owns a mailbox in its HBM: Slot[2][MAXG] (double-buffered by epoch
// parity).  The mailboxes are shared through CUDA IPC and mapped into every
// peer (NVLink/NVSwitch P2P).  After its local canonical-order reduction, each
// rank runs ONE thread of xgpu_exchange_kernel that
//   1. stores its partial into slot [parity][rank] of every peer's mailbox
//      (P2P stores over NVLink), then __threadfence_system(), then the epoch
//      flag of those slots;
//   2. spins on its own mailbox until all G flags carry this epoch;
//   3. folds the non-empty ranks' partials with the adjacent-pair _tadd tree
//      (the same skip tree as tf_combine), so the result is bit-identical to
//      the NCCL path and to the one-GPU reduction.
// A rank can be at most one epoch ahead of any other (its call only completes
// after reading everyone's current epoch), so two parity buffers suffice.  The
// spin is bounded (~10 s): on timeout the result is NaN and tf_xgpu_status
// reports the failure instead of hanging the device.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "reduce_impl.cuh"
#include "tf_math.cuh"
#include "xgpu.cuh"

namespace tf {

// The split (two-phase) form: XM_PUBLISH stores this rank's partial and flags
// and returns; XM_COLLECT later waits for and folds the peers'.  The caller
// orders the phases across ranks (a host barrier in between), so no kernel
// ever waits on another rank's kernel.
enum { XM_FULL = 0, XM_PUBLISH = 1, XM_COLLECT = 2 };

template <class T>
__device__ __forceinline__ void xgpu_run(T* out, const XArgs& x, int* status, int mode) {
  if (mode != XM_COLLECT) xgpu_publish(out, x);
  if (mode != XM_PUBLISH) xgpu_collect(out, x, status);
}

template <class T>
__global__ void xgpu_exchange_kernel(T* out, XArgs x, int* status, int mode) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  xgpu_run(out, x, status, mode);
}

// Reduction fused with the exchange: every CTA reduces its tile as in
// reduce_kernel; the last CTA, having folded the tile tree into out[0..1], runs
// the mailbox protocol from the same thread — the local result goes straight to
// the peers over NVLink and the global result lands in out, in ONE launch.
template <class T, int ROP, bool VEC>
__global__ void __launch_bounds__(RW) reduce_xgpu_kernel(const T* __restrict__ a,
                                                         const T* __restrict__ b, int64_t n,
                                                         int64_t ntiles, P<T>* tiles,
                                                         unsigned* counter, T* out, XArgs x,
                                                         int* status, int mode) {
  if (reduce_tile<T, ROP, VEC>(a, b, n, ntiles, tiles, counter, out, blockIdx.x) &&
      threadIdx.x == 0)
    xgpu_run(out, x, status, mode);
}

// One-GPU emulation of the FUSED path for `world` ranks: one grid, tpr CTAs per
// rank (block r*tpr + t is tile t of rank r's contiguous shard), per-rank
// workspaces, and the mailboxes of every rank in this GPU's memory.  Each
// rank's last CTA runs the exchange exactly as reduce_xgpu_kernel does.  At most
// `world` CTAs ever spin, far fewer than the resident slots, so every other CTA
// keeps making progress on one device.
struct EmuShards {
  int64_t lo[XG_MAXG], n[XG_MAXG];
};

template <class T, int ROP>
__global__ void __launch_bounds__(RW) reduce_xgpu_emulate_kernel(const T* a, const T* b,
                                                                  EmuShards sh, int64_t tpr,
                                                                  P<T>* tiles, unsigned* counters,
                                                                  T* outs, XArgs base,
                                                                  int* status) {
  const int r = (int)(blockIdx.x / tpr);
  const int64_t t = blockIdx.x % tpr;
  const int64_t n = sh.n[r];
  const int64_t nt = (n + Geo<T>::L - 1) / Geo<T>::L;
  XArgs x = base;
  x.rank = r;
  T* out = outs + 2 * r;
  if (n == 0) {  // an empty shard still takes part in the exchange
    if (t == 0 && threadIdx.x == 0) {
      out[0] = T(0);
      out[1] = T(0);
      xgpu_exchange(out, x, status);
    }
    return;
  }
  if (t >= nt) return;
  if (reduce_tile<T, ROP, false>(a + sh.lo[r], b + sh.lo[r], n, nt, tiles + r * tpr,
                                 counters + r, out, t) &&
      threadIdx.x == 0)
    xgpu_exchange(out, x, status);
}

// One-GPU emulation of `world` ranks: block r plays rank r over mailboxes that
// all live in this GPU's memory, for `epochs` back-to-back exchanges (both
// parity buffers).  All blocks of one small grid are co-resident, so the spin
// waits between them are safe on one device (unlike separate launches).
template <class T>
__global__ void xgpu_emulate_kernel(T* io, XArgs base, int epochs, int* status) {
  if (threadIdx.x != 0) return;
  XArgs x = base;
  x.rank = blockIdx.x;
  T* out = io + 2 * blockIdx.x;
  const T p0 = out[0], p1 = out[1];
  for (int e = 0; e < epochs; e++) {
    out[0] = p0;  // every epoch starts from this rank's own partial
    out[1] = p1;
    x.epoch = base.epoch + e;
    xgpu_exchange(out, x, status);
  }
}

struct XCtx {
  std::mutex mu;
  Slot* own = nullptr;
  Slot* box[XG_MAXG] = {};
  int rank = -1, world = 0;
  unsigned long long epoch = 0;
  int* status = nullptr;
  XArgs published{};  // the exchange a split-form publish left for its collect
  bool pending = false;
};
static XCtx g_x[64];

// Arguments of this rank's next exchange (caller holds c.mu): one epoch per call.
static XArgs next_exchange(XCtx& c, const int64_t* counts) {
  XArgs x{};
  for (int r = 0; r < c.world; r++) x.box[r] = c.box[r];
  x.rank = c.rank;
  x.world = c.world;
  x.epoch = ++c.epoch;
  for (int r = 0; r < c.world; r++)
    if (counts[r] > 0) {
      if (r < 32) x.nonempty_lo |= 1ull << r;
      else x.nonempty_hi |= 1ull << (r - 32);
    }
  return x;
}

static XCtx* ctx_for_current(int* dev_out) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (dev_out) *dev_out = dev;
  return &g_x[dev];
}

}  // namespace tf

using namespace tf;

// Allocate (once) this device's mailbox and return its 64-byte IPC handle.
extern "C" int tf_xgpu_mailbox(int device, void* handle64) {
  DeviceGuard g(device);
  XCtx* c = ctx_for_current(nullptr);
  if (!c || !handle64) return fail(TF_EINVAL, "tf_xgpu_mailbox: bad arguments");
  std::lock_guard<std::mutex> lock(c->mu);
  if (!c->own) {
    cudaError_t e = cudaMalloc(&c->own, sizeof(Slot) * 2 * XG_MAXG);
    if (e == cudaSuccess) e = cudaMemset(c->own, 0xff, sizeof(Slot) * 2 * XG_MAXG);  // seq = ~0
    if (e == cudaSuccess) e = cudaMalloc(&c->status, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->status, 0, sizeof(int));
    if (e != cudaSuccess) return cuda_status(e, "tf_xgpu_mailbox");
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->own);
  if (e != cudaSuccess) return cuda_status(e, "tf_xgpu_mailbox: ipc handle");
  std::memcpy(handle64, &h, sizeof h);
  return TF_OK;
}

// Map every peer's mailbox (handles: world x 64 bytes, rank order).
extern "C" int tf_xgpu_open(int device, int world, int rank, const void* handles) {
  DeviceGuard g(device);
  XCtx* c = ctx_for_current(nullptr);
  if (!c || world < 1 || world > XG_MAXG || rank < 0 || rank >= world || !handles)
    return fail(TF_EINVAL, "tf_xgpu_open: bad arguments");
  std::lock_guard<std::mutex> lock(c->mu);
  if (!c->own) return fail(TF_EINVAL, "tf_xgpu_open: call tf_xgpu_mailbox first");
  // A second transport in the same job (same group): the peers' mailboxes are
  // process-lifetime allocations, already mapped — reuse them.
  if (c->world == world && c->rank == rank) return TF_OK;
  if (c->world > 1) return fail(TF_EINVAL, "tf_xgpu_open: already open for another group");
  for (int r = 0; r < world; r++) {
    if (r == rank) {
      c->box[r] = c->own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * r, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "tf_xgpu_open: ipc open");
    c->box[r] = static_cast<Slot*>(p);
  }
  c->rank = rank;
  c->world = world;
  return TF_OK;
}

namespace tf {
size_t reduce_ws_bytes(int dtype, int64_t n);

template <class T>
static void launch_exchange(void* out, const XArgs& x, int* status, int mode, cudaStream_t s) {
  xgpu_exchange_kernel<T><<<1, 32, 0, s>>>(static_cast<T*>(out), x, status, mode);
}

template <class T, int ROP>
static void launch_reduce_xgpu(int64_t n, const void* a, const void* b, void* out, void* ws,
                               const XArgs& x, int* status, int mode, cudaStream_t s) {
  const int64_t nt = (n + Geo<T>::L - 1) / Geo<T>::L;
  unsigned* counter = static_cast<unsigned*>(ws);
  P<T>* tiles = reinterpret_cast<P<T>*>(static_cast<char*>(ws) + 256);
  const T* pa = static_cast<const T*>(a);
  const T* pb = static_cast<const T*>(b ? b : a);
  T* po = static_cast<T*>(out);
  if (aligned16(a) && (ROP == TF_RSUM || aligned16(b)))
    reduce_xgpu_kernel<T, ROP, true><<<(unsigned)nt, RW, 0, s>>>(pa, pb, n, nt, tiles, counter,
                                                                 po, x, status, mode);
  else
    reduce_xgpu_kernel<T, ROP, false><<<(unsigned)nt, RW, 0, s>>>(pa, pb, n, nt, tiles, counter,
                                                                  po, x, status, mode);
}

// The epoch of a new exchange (caller holds c.mu).  A split-form publish leaves
// it pending until tf_xgpu_collect; nothing else may start in between.
static int begin_exchange(XCtx& c, const int64_t* counts, int mode, const char* who,
                          XArgs* x) {
  if (c.pending)
    return fail(TF_EINVAL, std::string(who) + ": a published exchange awaits tf_xgpu_collect");
  *x = next_exchange(c, counts);
  if (mode == XM_PUBLISH) {
    c.published = *x;
    c.pending = true;
  }
  return TF_OK;
}

// Launch status of an exchange; a publish that never reached the device leaves
// nothing pending to collect.
static int end_exchange(XCtx& c, int mode, const char* who) {
  const int rc = launch_status(who);
  if (rc && mode == XM_PUBLISH) c.pending = false;
  return rc;
}

static int xgpu_combine_impl(int dtype, void* out, const int64_t* counts, void* stream, int mode,
                             const char* who) {
  XCtx* c = ctx_for_current(nullptr);
  if (!c || c->world < 1) return fail(TF_EINVAL, std::string(who) + ": transport not open");
  if ((dtype != TF_F32 && dtype != TF_F64) || !out || !counts)
    return fail(TF_EINVAL, std::string(who) + ": bad arguments");
  std::lock_guard<std::mutex> lock(c->mu);
  XArgs x;
  if (int rc = begin_exchange(*c, counts, mode, who, &x)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == TF_F64) launch_exchange<double>(out, x, c->status, mode, s);
  else launch_exchange<float>(out, x, c->status, mode, s);
  return end_exchange(*c, mode, who);
}

static int xgpu_reduce_impl(int rop, int dtype, int64_t n, const void* a, const void* b,
                            void* out, void* ws, size_t ws_bytes, const int64_t* counts,
                            void* stream, int mode, const char* who) {
  const std::string w(who);
  XCtx* c = ctx_for_current(nullptr);
  if (!c || c->world < 1) return fail(TF_EINVAL, w + ": transport not open");
  if (rop < 0 || rop >= TF_NUM_ROPS) return fail(TF_EINVAL, w + ": unknown reduction id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, w + ": planes must be float32 or float64");
  if (n < 0 || !out || !counts) return fail(TF_EINVAL, w + ": bad arguments");
  if (n > 0 && (!a || (rop != TF_RSUM && !b))) return fail(TF_EINVAL, w + ": null plane");
  if (n > 0 && (!ws || ws_bytes < reduce_ws_bytes(dtype, n)))
    return fail(TF_EINVAL, w + ": workspace too small");
  const int64_t L = dtype == TF_F64 ? Geo<double>::L : Geo<float>::L;
  if ((n + L - 1) / L > 0x7fffffffLL) return fail(TF_EINVAL, w + ": too many tiles");
  std::lock_guard<std::mutex> lock(c->mu);
  XArgs x;
  if (int rc = begin_exchange(*c, counts, mode, who, &x)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  if (n == 0) {  // nothing to reduce: (+0, +0), skipped by the fold (count 0)
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * tsz, s);
    if (e != cudaSuccess) {
      if (mode == XM_PUBLISH) c->pending = false;
      return cuda_status(e, who);
    }
    if (dtype == TF_F64) launch_exchange<double>(out, x, c->status, mode, s);
    else launch_exchange<float>(out, x, c->status, mode, s);
    return end_exchange(*c, mode, who);
  }
#define XR(ROP)                                                                                   \
  case ROP:                                                                                       \
    if (dtype == TF_F64) launch_reduce_xgpu<double, ROP>(n, a, b, out, ws, x, c->status, mode, s); \
    else launch_reduce_xgpu<float, ROP>(n, a, b, out, ws, x, c->status, mode, s);                 \
    break;
  switch (rop) { XR(TF_RSUM) XR(TF_RSUM2) XR(TF_RDOT) }
#undef XR
  return end_exchange(*c, mode, who);
}
}  // namespace tf

// Exchange + combine: out (device, 2 x dtype) holds this rank's partial on entry
// and the global result on exit.  counts: host array of world shard sizes.
extern "C" int tf_xgpu_combine(int dtype, void* out, const int64_t* counts, void* stream) {
  return xgpu_combine_impl(dtype, out, counts, stream, XM_FULL, "tf_xgpu_combine");
}

// Reduce this rank's shard AND exchange/combine over NVLink in one launch:
// tf_reduce followed by tf_xgpu_combine, fused (the last CTA publishes the local
// result to the peers' mailboxes, waits for theirs and folds them).  Same
// arguments as tf_reduce plus the host array of world shard sizes; out holds the
// global result on completion.  Collective, like tf_xgpu_combine.
extern "C" int tf_xgpu_reduce(int rop, int dtype, int64_t n, const void* a, const void* b,
                              void* out, void* ws, size_t ws_bytes, const int64_t* counts,
                              void* stream) {
  return xgpu_reduce_impl(rop, dtype, n, a, b, out, ws, ws_bytes, counts, stream, XM_FULL,
                          "tf_xgpu_reduce");
}

// Split form, phase 1: as tf_xgpu_combine / tf_xgpu_reduce, but the device
// thread only publishes this rank's partial (data, fence, epoch flags) and
// returns; out keeps the local partial.  Once the caller knows every rank's
// publish has completed (e.g. stream sync + host barrier), tf_xgpu_collect
// waits for nothing and folds.  No kernel ever waits on another rank's kernel,
// so ranks may even share one GPU (how the IPC mapping is tested here).
extern "C" int tf_xgpu_publish(int dtype, void* out, const int64_t* counts, void* stream) {
  return xgpu_combine_impl(dtype, out, counts, stream, XM_PUBLISH, "tf_xgpu_publish");
}

extern "C" int tf_xgpu_reduce_publish(int rop, int dtype, int64_t n, const void* a,
                                      const void* b, void* out, void* ws, size_t ws_bytes,
                                      const int64_t* counts, void* stream) {
  return xgpu_reduce_impl(rop, dtype, n, a, b, out, ws, ws_bytes, counts, stream, XM_PUBLISH,
                          "tf_xgpu_reduce_publish");
}

// Split form, phase 2: fold the pending exchange's partials into out (2 x dtype,
// device); dtype must match the publish.
extern "C" int tf_xgpu_collect(int dtype, void* out, void* stream) {
  XCtx* c = ctx_for_current(nullptr);
  if (!c || c->world < 1) return fail(TF_EINVAL, "tf_xgpu_collect: transport not open");
  if ((dtype != TF_F32 && dtype != TF_F64) || !out)
    return fail(TF_EINVAL, "tf_xgpu_collect: bad arguments");
  std::lock_guard<std::mutex> lock(c->mu);
  if (!c->pending) return fail(TF_EINVAL, "tf_xgpu_collect: no published exchange");
  c->pending = false;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == TF_F64) launch_exchange<double>(out, c->published, c->status, XM_COLLECT, s);
  else launch_exchange<float>(out, c->published, c->status, XM_COLLECT, s);
  return launch_status("tf_xgpu_collect");
}

// Test entry: the fused reduce + exchange for `world` emulated ranks on this
// GPU.  Rank r's shard is the next counts[r] elements of the device planes a
// (and b); outs (device, world x 2) receives every rank's global result.
// Synchronous.
extern "C" int tf_xgpu_reduce_emulate(int rop, int dtype, int world, const void* a,
                                      const void* b, const int64_t* counts, void* outs,
                                      void* stream) {
  if (rop < 0 || rop >= TF_NUM_ROPS || (dtype != TF_F32 && dtype != TF_F64) || world < 1 ||
      world > XG_MAXG || !counts || !outs || !a || (rop != TF_RSUM && !b))
    return fail(TF_EINVAL, "tf_xgpu_reduce_emulate: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  const int64_t L = dtype == TF_F64 ? Geo<double>::L : Geo<float>::L;
  EmuShards sh{};
  int64_t off = 0, tpr = 1;
  XArgs x{};
  for (int r = 0; r < world; r++) {
    if (counts[r] < 0) return fail(TF_EINVAL, "tf_xgpu_reduce_emulate: negative count");
    sh.lo[r] = off;
    sh.n[r] = counts[r];
    off += counts[r];
    const int64_t nt = (counts[r] + L - 1) / L;
    if (nt > tpr) tpr = nt;
    if (counts[r] > 0) {
      if (r < 32) x.nonempty_lo |= 1ull << r;
      else x.nonempty_hi |= 1ull << (r - 32);
    }
  }
  if (tpr * world > 0x7fffffffLL) return fail(TF_EINVAL, "tf_xgpu_reduce_emulate: too large");
  Slot* boxes = nullptr;
  void* tiles = nullptr;
  unsigned* counters = nullptr;
  int* status = nullptr;
  const size_t bbytes = sizeof(Slot) * 2 * XG_MAXG * world;
  cudaError_t e = cudaMalloc(&boxes, bbytes);
  if (e == cudaSuccess) e = cudaMemset(boxes, 0xff, bbytes);
  if (e == cudaSuccess) e = cudaMalloc(&tiles, (size_t)world * tpr * 2 * tsz);
  if (e == cudaSuccess) e = cudaMalloc(&counters, sizeof(unsigned) * world);
  if (e == cudaSuccess) e = cudaMemset(counters, 0, sizeof(unsigned) * world);
  if (e == cudaSuccess) e = cudaMalloc(&status, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(status, 0, sizeof(int));
  int rc = e == cudaSuccess ? TF_OK : cuda_status(e, "tf_xgpu_reduce_emulate");
  if (!rc) {
    for (int r = 0; r < world; r++) x.box[r] = boxes + (size_t)r * 2 * XG_MAXG;
    x.world = world;
    x.epoch = 1;
    const unsigned grid = (unsigned)(tpr * world);
#define XE(ROP)                                                                               \
  case ROP:                                                                                   \
    if (dtype == TF_F64)                                                                      \
      reduce_xgpu_emulate_kernel<double, ROP><<<grid, RW, 0, s>>>(                            \
          static_cast<const double*>(a), static_cast<const double*>(b ? b : a), sh, tpr,      \
          static_cast<P<double>*>(tiles), counters, static_cast<double*>(outs), x, status);   \
    else                                                                                      \
      reduce_xgpu_emulate_kernel<float, ROP><<<grid, RW, 0, s>>>(                             \
          static_cast<const float*>(a), static_cast<const float*>(b ? b : a), sh, tpr,        \
          static_cast<P<float>*>(tiles), counters, static_cast<float*>(outs), x, status);     \
    break;
    switch (rop) { XE(TF_RSUM) XE(TF_RSUM2) XE(TF_RDOT) }
#undef XE
    rc = launch_status("tf_xgpu_reduce_emulate");
  }
  int h = 0;
  if (!rc) {
    e = cudaMemcpyAsync(&h, status, sizeof h, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_status(e, "tf_xgpu_reduce_emulate");
  }
  cudaFree(boxes);
  cudaFree(tiles);
  cudaFree(counters);
  cudaFree(status);
  if (!rc && h) rc = fail(TF_ECUDA, "tf_xgpu_reduce_emulate: exchange timed out");
  return rc;
}

// 0 = OK, 1 = a combine timed out waiting for a peer (synchronous read).
extern "C" int tf_xgpu_status(int device) {
  DeviceGuard g(device);
  XCtx* c = ctx_for_current(nullptr);
  if (!c || !c->status) return 0;
  int v = 0;
  cudaMemcpy(&v, c->status, sizeof v, cudaMemcpyDeviceToHost);
  return v;
}

// Test entry: emulate `world` ranks on this GPU.  io (device, world x 2 of dtype)
// holds each rank's partial on entry and each rank's combined result on exit.
extern "C" int tf_xgpu_emulate(int dtype, int world, void* io, const int64_t* counts,
                               int epochs, void* stream) {
  if ((dtype != TF_F32 && dtype != TF_F64) || world < 1 || world > XG_MAXG || !io || !counts ||
      epochs < 1)
    return fail(TF_EINVAL, "tf_xgpu_emulate: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Slot* boxes = nullptr;
  int* status = nullptr;
  const size_t bytes = sizeof(Slot) * 2 * XG_MAXG * world;
  cudaError_t e = cudaMalloc(&boxes, bytes);
  if (e == cudaSuccess) e = cudaMemset(boxes, 0xff, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&status, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(status, 0, sizeof(int));
  if (e != cudaSuccess) return cuda_status(e, "tf_xgpu_emulate");
  XArgs x{};
  for (int r = 0; r < world; r++) x.box[r] = boxes + (size_t)r * 2 * XG_MAXG;
  x.world = world;
  x.epoch = 1;
  for (int r = 0; r < world; r++)
    if (counts[r] > 0) {
      if (r < 32) x.nonempty_lo |= 1ull << r;
      else x.nonempty_hi |= 1ull << (r - 32);
    }
  if (dtype == TF_F64)
    xgpu_emulate_kernel<double><<<world, 32, 0, s>>>(static_cast<double*>(io), x, epochs, status);
  else
    xgpu_emulate_kernel<float><<<world, 32, 0, s>>>(static_cast<float*>(io), x, epochs, status);
  int rc = launch_status("tf_xgpu_emulate");
  int h = 0;
  if (!rc) {
    e = cudaMemcpyAsync(&h, status, sizeof h, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_status(e, "tf_xgpu_emulate");
  }
  cudaFree(boxes);
  cudaFree(status);
  if (!rc && h) rc = fail(TF_ECUDA, "tf_xgpu_emulate: exchange timed out");
  return rc;
}
