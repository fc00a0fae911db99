// hostpipe.cu — tf_elementwise_host: the reference's calling convention (numpy
// planes in host memory, kernels.py:191-239) served by the device.
//
// The planes are cut into chunks that flow through S slots, each with its own
// stream and device buffers:  H2D(inputs) -> kernel -> D2H(outputs).  Slots
// overlap, so the copy engines (both directions) and the SMs work concurrently
// and the call runs at the host-link bound.
//
// Pinned (page-locked / registered) planes are DMA'd directly.  Pageable planes
// (plain numpy) cannot be DMA'd asynchronously, and the driver's own staging
// runs at ~13 GB/s; here a pool of host threads copies them through
// library-owned pinned staging buffers instead, overlapped with the transfers
// of the other slots.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tf {

int ew_num_inputs(int op);
int ew_launch(int op, int dtype, int64_t n, const void* const* in, void* const* out,
              cudaStream_t stream);
constexpr int TF_BATCH_MAX_OPS = 8;  // tf_elementwise_batch's limit

// ---- a small persistent thread pool for parallel host memcpy ------------------
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; i++) th_.emplace_back([this, i] { worker(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  // run f(part) for part in [0, parts) on the workers and the calling thread
  void run(int parts, const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f;
      parts_ = parts;
      next_ = 0;
      pending_ = parts;
      gen_++;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void drain() {
    for (;;) {
      int k;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> g(m_);
        if (!job_ || next_ >= parts_) return;
        k = next_++;
        f = job_;
      }
      (*f)(k);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  void worker(int) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || (gen_ != seen && job_ && next_ < parts_); });
        if (stop_) return;
        seen = gen_;
      }
      drain();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

static void par_memcpy(CopyPool& pool, void* dst, const void* src, size_t bytes) {
  const size_t grain = 1 << 20;
  int parts = (int)((bytes + grain - 1) / grain);
  if (parts > pool.size() * 2) parts = pool.size() * 2;
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = ((bytes / parts) + 63) & ~size_t(63);
  pool.run(parts, [&](int k) {
    const size_t lo = (size_t)k * per;
    if (lo >= bytes) return;
    const size_t len = (lo + per > bytes) ? bytes - lo : per;
    std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, len);
  });
}

// ---- per-device pipeline state -------------------------------------------------
struct HostPipe {
  static constexpr int MAX_SLOTS = 8;
  int slots = 3;
  int64_t chunk_bytes = 32ll << 20;  // per plane per slot (sweep: 32 MB best, r1 profiles)
  int64_t min_chunks = 8;             // split smaller planes into this many chunks ...
  int64_t min_chunk_bytes = 1 << 20;  // ... of at least this many bytes (sweep: r1s2_host_chunk_sweep.txt)
  int64_t zerocopy_bytes = 16ll << 20;  // pinned planes up to this size: zero-copy kernel
  std::mutex mu;
  bool ready = false;
  cudaStream_t st[MAX_SLOTS] = {};
  cudaEvent_t done[MAX_SLOTS] = {};
  // per slot: one device arena and one pinned arena (pageable planes only),
  // carved per call into NP plane buffers of `plane` bytes; grown on demand
  void* darena[MAX_SLOTS] = {};
  void* harena[MAX_SLOTS] = {};
  size_t dcap = 0, hcap = 0;
  CopyPool* pool = nullptr;
};
// Staging memory a call may use across all slots (device; the same again in
// pinned host memory for pageable planes): a batch of many ops gets shorter
// chunks instead of NP x 32 MB x slots of staging.
constexpr int64_t STAGING_BUDGET = 3ll << 30;
static HostPipe g_pipe[64];

static int pipe_init(HostPipe& p) {
  if (p.ready) return TF_OK;
  if (const char* v = getenv("TF_HOST_SLOTS")) {
    int k = atoi(v);
    if (k >= 2 && k <= HostPipe::MAX_SLOTS) p.slots = k;
  }
  if (const char* v = getenv("TF_HOST_CHUNK_MB")) {
    long k = atol(v);
    if (k >= 1 && k <= 1024) p.chunk_bytes = (int64_t)k << 20;
  }
  if (const char* v = getenv("TF_HOST_ZEROCOPY_MB")) {
    long k = atol(v);
    if (k >= 0 && k <= 4096) p.zerocopy_bytes = (int64_t)k << 20;
  }
  if (const char* v = getenv("TF_HOST_MIN_CHUNKS")) {
    long k = atol(v);
    if (k >= 1 && k <= 64) p.min_chunks = k;
  }
  if (const char* v = getenv("TF_HOST_MIN_CHUNK_KB")) {
    long k = atol(v);
    if (k >= 4 && k <= (1 << 20)) p.min_chunk_bytes = (int64_t)k << 10;
  }
  for (int s = 0; s < p.slots; s++) {
    cudaError_t e = cudaStreamCreateWithFlags(&p.st[s], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.done[s], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: stream");
  }
  p.ready = true;
  return TF_OK;
}

// Bytes per plane per slot for a call staging NP planes of `total` bytes each:
// the configured chunk, shortened (4 KB multiples) so that NP planes x slots fit
// the staging budget, and so that a plane of a few chunks still splits into
// min_chunks (of >= min_chunk_bytes each): with one chunk, H2D, kernel and D2H run back
// to back and the two link directions never overlap.
static int64_t plane_bytes(const HostPipe& p, int NP, int64_t total) {
  int64_t b = STAGING_BUDGET / ((int64_t)NP * p.slots);
  if (b > p.chunk_bytes) b = p.chunk_bytes;
  int64_t split = (total + p.min_chunks - 1) / p.min_chunks;
  if (split < p.min_chunk_bytes) split = p.min_chunk_bytes;
  if (b > split) b = split;
  b = (b + 4095) & ~int64_t(4095);
  return b < 4096 ? 4096 : b;
}

// Grow the slot arenas to hold `need` bytes each (calls are synchronous and
// serialised by p.mu, so nothing is in flight when an arena is replaced).
static int ensure_arenas(HostPipe& p, size_t need, bool pinned_staging) {
  if (p.dcap < need) {
    for (int s = 0; s < p.slots; s++) {
      if (p.darena[s]) cudaFree(p.darena[s]);
      p.darena[s] = nullptr;
    }
    p.dcap = 0;
    for (int s = 0; s < p.slots; s++) {
      cudaError_t e = cudaMalloc(&p.darena[s], need);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: staging alloc");
    }
    p.dcap = need;
  }
  if (pinned_staging && p.hcap < need) {
    for (int s = 0; s < p.slots; s++) {
      if (p.harena[s]) cudaFreeHost(p.harena[s]);
      p.harena[s] = nullptr;
    }
    p.hcap = 0;
    for (int s = 0; s < p.slots; s++) {
      cudaError_t e = cudaHostAlloc(&p.harena[s], need, cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: pinned staging alloc");
    }
    p.hcap = need;
  }
  return TF_OK;
}

static int ensure_pool(HostPipe& p) {
  if (!p.pool) {
    unsigned hw = std::thread::hardware_concurrency();
    int nt = hw ? (int)hw : 4;
    if (const char* v = getenv("TF_HOST_THREADS")) nt = atoi(v) > 0 ? atoi(v) : nt;
    if (nt > 32) nt = 32;
    p.pool = new CopyPool(nt > 1 ? nt - 1 : 0);
  }
  return TF_OK;
}

static bool is_pinned(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();  // clear
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// On an error return, wait for everything already queued on the slot streams:
// copies into the caller's host planes must not land after we have returned.
struct DrainOnError {
  HostPipe& p;
  bool ok = false;
  ~DrainOnError() {
    if (ok) return;
    for (int s = 0; s < p.slots; s++)
      if (p.st[s]) cudaStreamSynchronize(p.st[s]);
  }
};

// Run `nops` ops over the same n elements of host planes in one pipelined pass.
// Distinct input planes (by address) cross the host link once per chunk however
// many ops read them; every op's two outputs come back, in op order.
using HostLaunch = std::function<int(int, int64_t, const void* const*, void* const*, cudaStream_t)>;

static int host_batch(int nops, const int* ops, int dtype, int64_t n, const void* const* in,
                      void* const* out, int device, const char* who,
                      const HostLaunch* launch = nullptr, int nin_all = -1) {
  if (nops < 1 || nops > 64) return fail(TF_EINVAL, std::string(who) + ": 1..64 ops per batch");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, std::string(who) + ": planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, std::string(who) + ": negative length");
  if (!in || !out) return fail(TF_EINVAL, std::string(who) + ": null plane");
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  // distinct inputs; per op the index of each of its inputs among them
  std::vector<const void*> uniq;
  std::vector<int> idx((size_t)nops * 4, -1);
  for (int o = 0; o < nops; o++) {
    const int nin = nin_all >= 0 ? nin_all : ew_num_inputs(ops[o]);
    if (nin < 0) return fail(TF_EINVAL, std::string(who) + ": unknown op id");
    if (!out[2 * o] || !out[2 * o + 1]) return fail(TF_EINVAL, std::string(who) + ": null plane");
    for (int k = 0; k < nin; k++) {
      const void* ptr = in[4 * o + k];
      if (!ptr) return fail(TF_EINVAL, std::string(who) + ": null plane");
      int u = -1;
      for (size_t q = 0; q < uniq.size(); q++)
        if (uniq[q] == ptr) u = (int)q;
      if (u < 0) {
        u = (int)uniq.size();
        uniq.push_back(ptr);
      }
      idx[4 * o + k] = u;
    }
  }
  // outputs either coincide (later ops overwrite, as run one by one) or are
  // disjoint: a partial overlap has no chunk order that matches
  const uintptr_t span = (uintptr_t)n * tsz;
  for (int w = 0; w < 2 * nops && n; w++)
    for (int v = w + 1; v < 2 * nops; v++) {
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(out[w]);
      const uintptr_t b0 = reinterpret_cast<uintptr_t>(out[v]);
      if (a0 != b0 && a0 < b0 + span && b0 < a0 + span)
        return fail(TF_EINVAL, std::string(who) + ": out planes overlap each other");
    }
  // no op may read what another op of the batch writes (no intra-batch chains)
  for (int o = 0; o < 2 * nops; o++) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(out[o]);
    for (const void* u : uniq) {
      const uintptr_t b0 = reinterpret_cast<uintptr_t>(u);
      if (n && a0 < b0 + span && b0 < a0 + span)
        return fail(TF_EINVAL, std::string(who) + ": out must not alias an input");
    }
  }
  if (n == 0) return TF_OK;

  DeviceGuard g(device);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(TF_EINVAL, std::string(who) + ": device ordinal");
  HostPipe& p = g_pipe[dev];
  std::lock_guard<std::mutex> lock(p.mu);
  int rc = pipe_init(p);
  if (rc) return rc;
  DrainOnError guard{p};

  const int U = (int)uniq.size();
  const int NP = U + 2 * nops;  // staging planes per slot: inputs, then outputs
  std::vector<char> pin_in(U), pin_out(2 * nops);
  bool any_pageable = false;
  for (int q = 0; q < U; q++) any_pageable |= !(pin_in[q] = is_pinned(uniq[q]));
  for (int o = 0; o < 2 * nops; o++) any_pageable |= !(pin_out[o] = is_pinned(out[o]));
  // Small calls over pinned planes: zero-copy.  ONE batch kernel reads and writes
  // the host planes in place over PCIe (UVA-mapped), with no staging copies and
  // no chunk pipeline; below ~16 MB per plane this beats the copy engines'
  // fill/drain (profiles/r1s2_zerocopy.json).  Large calls keep the pipeline.
  if (!launch && !any_pageable && nops <= TF_BATCH_MAX_OPS &&
      n * (int64_t)tsz <= p.zerocopy_bytes) {
    std::vector<const void*> zin((size_t)nops * 4, nullptr);
    std::vector<void*> zout((size_t)nops * 2, nullptr);
    bool mapped = true;
    auto dev_ptr = [&](const void* h) -> void* {
      void* d = nullptr;
      if (cudaHostGetDevicePointer(&d, const_cast<void*>(h), 0) != cudaSuccess) {
        cudaGetLastError();
        mapped = false;
      }
      return d;
    };
    for (int o = 0; o < nops && mapped; o++) {
      for (int k = 0; k < 4; k++)
        if (idx[4 * o + k] >= 0) zin[4 * o + k] = dev_ptr(in[4 * o + k]);
      for (int k = 0; k < 2; k++) zout[2 * o + k] = dev_ptr(out[2 * o + k]);
    }
    if (mapped) {
      rc = tf_elementwise_batch(nops, ops, dtype, n, zin.data(), zout.data(), p.st[0]);
      if (rc) return rc;
      cudaError_t e = cudaStreamSynchronize(p.st[0]);
      if (e != cudaSuccess) return cuda_status(e, who);
      guard.ok = true;
      return TF_OK;
    }
  }
  const int64_t pb = plane_bytes(p, NP, n * (int64_t)tsz);
  if ((rc = ensure_arenas(p, (size_t)pb * NP, any_pageable))) return rc;
  if (any_pageable && (rc = ensure_pool(p))) return rc;
  auto dplane = [&](int s, int q) { return static_cast<char*>(p.darena[s]) + (size_t)q * pb; };
  auto hplane = [&](int s, int q) { return static_cast<char*>(p.harena[s]) + (size_t)q * pb; };

  const int64_t chunk = pb / (int64_t)tsz;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const int S = p.slots;
  std::vector<int64_t> slot_off(S, -1);  // chunk offset in flight in each slot

  auto finish = [&](int s) -> int {  // wait for slot s; unstage pageable outputs in op order
    if (slot_off[s] < 0) return TF_OK;
    cudaError_t e = cudaEventSynchronize(p.done[s]);
    if (e != cudaSuccess) return cuda_status(e, who);
    const int64_t off = slot_off[s];
    const int64_t m = (n - off) < chunk ? (n - off) : chunk;
    for (int o = 0; o < 2 * nops; o++)
      if (!pin_out[o])
        par_memcpy(*p.pool, static_cast<char*>(out[o]) + off * tsz, hplane(s, U + o),
                   (size_t)m * tsz);
    slot_off[s] = -1;
    return TF_OK;
  };

  for (int64_t c = 0; c < nchunks; c++) {
    const int s = (int)(c % S);
    if ((rc = finish(s))) return rc;
    const int64_t off = c * chunk;
    const int64_t m = (n - off) < chunk ? (n - off) : chunk;
    const size_t bytes = (size_t)m * tsz;
    cudaStream_t st = p.st[s];
    for (int q = 0; q < U; q++) {
      const void* src = static_cast<const char*>(uniq[q]) + off * tsz;
      if (!pin_in[q]) {
        par_memcpy(*p.pool, hplane(s, q), src, bytes);
        src = hplane(s, q);
      }
      cudaError_t e = cudaMemcpyAsync(dplane(s, q), src, bytes, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_status(e, who);
    }
    for (int o = 0; o < nops; o++) {
      const void* din[4] = {nullptr, nullptr, nullptr, nullptr};
      for (int k = 0; k < 4; k++)
        if (idx[4 * o + k] >= 0) din[k] = dplane(s, idx[4 * o + k]);
      void* dout[2] = {dplane(s, U + 2 * o), dplane(s, U + 2 * o + 1)};
      rc = launch ? (*launch)(o, m, din, dout, st) : ew_launch(ops[o], dtype, m, din, dout, st);
      if (rc) return rc;
    }
    for (int o = 0; o < 2 * nops; o++) {
      void* dst = pin_out[o] ? static_cast<char*>(out[o]) + off * tsz : hplane(s, U + o);
      cudaError_t e = cudaMemcpyAsync(dst, dplane(s, U + o), bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_status(e, who);
    }
    cudaError_t e = cudaEventRecord(p.done[s], st);
    if (e != cudaSuccess) return cuda_status(e, who);
    slot_off[s] = off;
  }
  // drain in chunk order
  for (int64_t c = nchunks; c < nchunks + S; c++)
    if ((rc = finish((int)(c % S)))) return rc;
  guard.ok = true;
  return TF_OK;
}

}  // namespace tf

using namespace tf;

extern "C" int tf_elementwise_host(int op, int dtype, int64_t n, const void* const* in,
                                   void* const* out, int device) {
  const int nin = ew_num_inputs(op);
  if (nin < 0) return fail(TF_EINVAL, "tf_elementwise_host: unknown op id");
  if (!in || !out) return fail(TF_EINVAL, "tf_elementwise_host: null plane");
  const void* in4[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int k = 0; k < nin; k++) in4[k] = in[k];
  return host_batch(1, &op, dtype, n, in4, out, device, "tf_elementwise_host");
}

namespace tf {
int horner_launch(int dtype, int64_t n, const void* x, const double* coeffs, int degree,
                  void* o0, void* o1, cudaStream_t s);
}

// Twofold Horner over HOST planes through the same pipeline (x in, z0/z1 out).
extern "C" int tf_horner_host(int dtype, int64_t n, const void* x, const double* coeffs,
                              int degree, void* out0, void* out1, int device) {
  if (!coeffs || degree < 0 || degree > TF_HORNER_MAX_DEGREE)
    return fail(TF_EINVAL, "tf_horner_host: degree out of range or null coefficients");
  std::vector<double> c(coeffs, coeffs + degree + 1);
  HostLaunch fn = [&](int, int64_t m, const void* const* din, void* const* dout,
                      cudaStream_t st) {
    return horner_launch(dtype, m, din[0], c.data(), degree, dout[0], dout[1], st);
  };
  const void* in4[4] = {x, nullptr, nullptr, nullptr};
  void* out2[2] = {out0, out1};
  int op = 0;
  return host_batch(1, &op, dtype, n, in4, out2, device, "tf_horner_host", &fn, 1);
}

extern "C" int tf_elementwise_host_batch(int nops, const int* ops, int dtype, int64_t n,
                                         const void* const* in, void* const* out, int device) {
  if (!ops) return fail(TF_EINVAL, "tf_elementwise_host_batch: null op list");
  return host_batch(nops, ops, dtype, n, in, out, device, "tf_elementwise_host_batch");
}

// ---- reductions over host planes --------------------------------------------------
namespace tf {
size_t reduce_ws_bytes(int dtype, int64_t n);
int reduce_geometry(int dtype, int* V, int* W, int* K);
int reduce_launch(int rop, int dtype, int64_t n, const void* a, const void* b, void* out,
                  void* ws, size_t ws_bytes, cudaStream_t s);
int combine_launch(int dtype, int g, const void* partials, const int64_t* counts, void* out,
                   cudaStream_t s);

constexpr int RED_MAX_BATCH = 16;

struct RedStage {  // per device: staging planes per slot (grown on demand)
  int64_t plane_bytes = 0;
  std::vector<void*> d[HostPipe::MAX_SLOTS];  // device planes
  std::vector<void*> h[HostPipe::MAX_SLOTS];  // pinned staging (pageable inputs)
  void* ws[HostPipe::MAX_SLOTS] = {};         // one per slot: its reductions run in order
  size_t ws_bytes = 0;
};
static RedStage g_red[64];

static void red_free(RedStage& R) {
  for (int s = 0; s < HostPipe::MAX_SLOTS; s++) {
    for (void* d : R.d[s]) cudaFree(d);
    for (void* h : R.h[s]) cudaFreeHost(h);
    R.d[s].clear();
    R.h[s].clear();
    if (R.ws[s]) cudaFree(R.ws[s]);
    R.ws[s] = nullptr;
  }
  R.plane_bytes = 0;
  R.ws_bytes = 0;
}

// Reduce n elements of HOST planes in the canonical order, `nred` reductions in
// one pass: chunks of C tiles (C a power of two, so every chunk is a complete
// subtree of the tile tree) stream through the slots; each distinct input plane
// crosses the host link once per chunk however many reductions read it; each
// chunk's subtree value lands in a device array and the combine kernel folds
// them with the same adjacent-pair tree — every result is bit-identical to
// tf_reduce on device planes.  Synchronous; writes out[2r..2r+1] (host, dtype).
static int reduce_host_batch(int nred, const int* rops, int dtype, int64_t n,
                             const void* const* a, const void* const* b, void* out,
                             int device, const char* who) {
  const std::string w(who);
  if (nred < 1 || nred > RED_MAX_BATCH) return fail(TF_EINVAL, w + ": 1..16 reductions per batch");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, w + ": planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, w + ": negative length");
  if (!out || !rops || !a) return fail(TF_EINVAL, w + ": null argument");
  for (int r = 0; r < nred; r++)
    if (rops[r] < 0 || rops[r] >= TF_NUM_ROPS) return fail(TF_EINVAL, w + ": unknown reduction id");
  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  if (n == 0) {
    std::memset(out, 0, 2 * tsz * nred);
    return TF_OK;
  }
  // distinct planes; per reduction the index of each operand among them
  std::vector<const void*> uniq;
  std::vector<int> ia(nred), ib(nred, -1);
  auto intern = [&](const void* ptr) {
    for (size_t q = 0; q < uniq.size(); q++)
      if (uniq[q] == ptr) return (int)q;
    uniq.push_back(ptr);
    return (int)uniq.size() - 1;
  };
  for (int r = 0; r < nred; r++) {
    if (!a[r] || (rops[r] != TF_RSUM && (!b || !b[r]))) return fail(TF_EINVAL, w + ": null plane");
    ia[r] = intern(a[r]);
    if (rops[r] != TF_RSUM) ib[r] = intern(b[r]);
  }
  const int U = (int)uniq.size();

  DeviceGuard g(device);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(TF_EINVAL, w + ": device ordinal");
  HostPipe& p = g_pipe[dev];
  RedStage& R = g_red[dev];
  std::lock_guard<std::mutex> lock(p.mu);
  int rc = pipe_init(p);
  if (rc) return rc;
  DrainOnError guard{p};

  int V = 0, W = 0, K = 0;
  reduce_geometry(dtype, &V, &W, &K);
  const int64_t L = (int64_t)V * W * K;
  const int64_t T = (n + L - 1) / L;
  int64_t C = 1;  // tiles per chunk: a power of two near the staging chunk size
  while (C * L * (int64_t)tsz < p.chunk_bytes) C <<= 1;
  while ((T + C - 1) / C > 1024) C <<= 1;  // the combine folds <= 1024 partials
  const int64_t chunk = C * L;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const int64_t pbytes = chunk * (int64_t)tsz;

  std::vector<char> pin(U);
  bool pageable = false;
  for (int q = 0; q < U; q++) pageable |= !(pin[q] = is_pinned(uniq[q]));
  const size_t need_ws = reduce_ws_bytes(dtype, chunk);  // f64 needs twice f32's
  if (R.plane_bytes < pbytes || R.ws_bytes < need_ws) {
    red_free(R);  // set up again below; a failed setup leaves it empty and retries
    for (int s = 0; s < p.slots; s++) {
      cudaError_t e = cudaMalloc(&R.ws[s], need_ws);
      if (e == cudaSuccess) e = cudaMemset(R.ws[s], 0, need_ws);
      if (e != cudaSuccess) {
        red_free(R);
        return cuda_status(e, who);
      }
    }
    R.plane_bytes = pbytes;
    R.ws_bytes = need_ws;
  }
  for (int s = 0; s < p.slots; s++) {
    while ((int)R.d[s].size() < U) {
      void* d = nullptr;
      cudaError_t e = cudaMalloc(&d, R.plane_bytes);
      if (e != cudaSuccess) return cuda_status(e, who);
      R.d[s].push_back(d);
    }
    while (pageable && (int)R.h[s].size() < U) {
      void* h = nullptr;
      cudaError_t e = cudaHostAlloc(&h, R.plane_bytes, cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_status(e, who);
      R.h[s].push_back(h);
    }
  }
  if (pageable && (rc = ensure_pool(p))) return rc;  // the copy pool

  void* parts = nullptr;  // nred x nchunks x 2 of dtype, then nred result pairs
  cudaError_t e = cudaMalloc(&parts, (size_t)nred * (nchunks + 1) * 2 * tsz);
  if (e != cudaSuccess) return cuda_status(e, who);
  auto part_at = [&](int r, int64_t c) {
    return static_cast<char*>(parts) + ((size_t)r * nchunks + (size_t)c) * 2 * tsz;
  };
  char* res = static_cast<char*>(parts) + (size_t)nred * nchunks * 2 * tsz;
  std::vector<int64_t> counts(nchunks);
  const int S = p.slots;
  std::vector<char> busy(S, 0);
  for (int64_t c = 0; c < nchunks && !rc; c++) {
    const int s = (int)(c % S);
    if (busy[s]) {  // the slot's previous chunk must be done before its buffers are reused
      e = cudaEventSynchronize(p.done[s]);
      if (e != cudaSuccess) { rc = cuda_status(e, who); break; }
    }
    const int64_t off = c * chunk;
    const int64_t m = (n - off) < chunk ? (n - off) : chunk;
    counts[c] = m;
    const size_t bytes = (size_t)m * tsz;
    cudaStream_t st = p.st[s];
    for (int q = 0; q < U && !rc; q++) {
      const void* from = static_cast<const char*>(uniq[q]) + off * tsz;
      if (!pin[q]) {
        par_memcpy(*p.pool, R.h[s][q], from, bytes);
        from = R.h[s][q];
      }
      e = cudaMemcpyAsync(R.d[s][q], from, bytes, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) rc = cuda_status(e, who);
    }
    for (int r = 0; r < nred && !rc; r++)
      rc = reduce_launch(rops[r], dtype, m, R.d[s][ia[r]], ib[r] >= 0 ? R.d[s][ib[r]] : nullptr,
                         part_at(r, c), R.ws[s], R.ws_bytes, st);
    if (!rc && (e = cudaEventRecord(p.done[s], st)) != cudaSuccess) rc = cuda_status(e, who);
    busy[s] = 1;
  }
  for (int s = 0; s < S && !rc; s++)
    if (busy[s] && (e = cudaEventSynchronize(p.done[s])) != cudaSuccess) rc = cuda_status(e, who);
  for (int r = 0; r < nred && !rc; r++)
    rc = combine_launch(dtype, (int)nchunks, part_at(r, 0), counts.data(), res + (size_t)r * 2 * tsz,
                        p.st[0]);
  if (!rc) {
    e = cudaMemcpyAsync(out, res, (size_t)nred * 2 * tsz, cudaMemcpyDeviceToHost, p.st[0]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p.st[0]);
    if (e != cudaSuccess) rc = cuda_status(e, who);
  }
  if (!rc) guard.ok = true;
  else
    for (int s = 0; s < p.slots; s++) cudaStreamSynchronize(p.st[s]);
  cudaFree(parts);
  return rc;
}
}  // namespace tf

extern "C" int tf_reduce_host(int rop, int dtype, int64_t n, const void* a, const void* b,
                              void* out, int device) {
  const void* bb[1] = {b};
  return reduce_host_batch(1, &rop, dtype, n, &a, bb, out, device, "tf_reduce_host");
}

extern "C" int tf_reduce_host_batch(int nred, const int* rops, int dtype, int64_t n,
                                    const void* const* a, const void* const* b, void* out,
                                    int device) {
  return reduce_host_batch(nred, rops, dtype, n, a, b, out, device, "tf_reduce_host_batch");
}

// ---- page-locking of reused pageable planes ------------------------------------
// Pageable planes cross the link through staging copies (host DRAM traffic x3);
// registering a plane that is reused makes it DMA-able in place.  The Python
// layer decides what to register (second use, size, budget) and unregisters it
// before its memory is released.
extern "C" int tf_host_register(void* ptr, size_t bytes) {
  if (!ptr || !bytes) return fail(TF_EINVAL, "tf_host_register: bad arguments");
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_status(e, "tf_host_register");
  }
  return TF_OK;
}

extern "C" int tf_host_unregister(void* ptr) {
  if (!ptr) return fail(TF_EINVAL, "tf_host_unregister: null pointer");
  // A host call on another thread may be DMA-ing this plane in place (it was
  // pinned when that call checked).  Host calls hold their device's pipe lock
  // for their whole duration, so taking every pipe lock (in index order; a call
  // holds only one) waits for them; later calls see the plane as pageable.
  std::vector<std::unique_lock<std::mutex>> held;
  held.reserve(64);
  for (auto& pp : g_pipe) held.emplace_back(pp.mu);
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_status(e, "tf_host_unregister");
  }
  return TF_OK;
}
