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
template <class T>
__device__ void xgpu_exchange(T* out, const XArgs& x, int* status) {
  const int par = (int)(x.epoch & 1);
  const volatile T* mine_v = out;
  const double z0 = (double)mine_v[0], z1 = (double)mine_v[1];
  // 1. publish: data everywhere, one system fence, then the flags
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
  // 2. wait for every rank's slot of this epoch in the local mailbox
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
  // 3. skip tree over the non-empty ranks, in rank order (as tf_combine)
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
__global__ void xgpu_exchange_kernel(T* out, XArgs x, int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
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
};
static XCtx g_x[64];

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

// Exchange + combine: out (device, 2 x dtype) holds this rank's partial on entry
// and the global result on exit.  counts: host array of world shard sizes.
extern "C" int tf_xgpu_combine(int dtype, void* out, const int64_t* counts, void* stream) {
  XCtx* c = ctx_for_current(nullptr);
  if (!c || c->world < 1) return fail(TF_EINVAL, "tf_xgpu_combine: transport not open");
  if ((dtype != TF_F32 && dtype != TF_F64) || !out || !counts)
    return fail(TF_EINVAL, "tf_xgpu_combine: bad arguments");
  std::lock_guard<std::mutex> lock(c->mu);
  XArgs x{};
  for (int r = 0; r < c->world; r++) x.box[r] = c->box[r];
  x.rank = c->rank;
  x.world = c->world;
  x.epoch = ++c->epoch;
  for (int r = 0; r < c->world; r++)
    if (counts[r] > 0) {
      if (r < 32) x.nonempty_lo |= 1ull << r;
      else x.nonempty_hi |= 1ull << (r - 32);
    }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == TF_F64)
    xgpu_exchange_kernel<double><<<1, 32, 0, s>>>(static_cast<double*>(out), x, c->status);
  else
    xgpu_exchange_kernel<float><<<1, 32, 0, s>>>(static_cast<float*>(out), x, c->status);
  return launch_status("tf_xgpu_combine");
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
