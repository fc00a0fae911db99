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
  int64_t chunk_bytes = 16ll << 20;  // per plane per slot
  std::mutex mu;
  bool ready = false;
  cudaStream_t st[MAX_SLOTS] = {};
  cudaEvent_t done[MAX_SLOTS] = {};
  void* dbuf[MAX_SLOTS][6] = {};  // device: 4 inputs + 2 outputs
  void* hbuf[MAX_SLOTS][6] = {};  // pinned staging for pageable planes (lazy)
  CopyPool* pool = nullptr;
};
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
  for (int s = 0; s < p.slots; s++) {
    cudaError_t e = cudaStreamCreateWithFlags(&p.st[s], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.done[s], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: stream");
    for (int k = 0; k < 6; k++) {
      e = cudaMalloc(&p.dbuf[s][k], p.chunk_bytes);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: staging alloc");
    }
  }
  p.ready = true;
  return TF_OK;
}

static int ensure_host_staging(HostPipe& p) {
  if (p.hbuf[0][0]) return TF_OK;
  for (int s = 0; s < p.slots; s++)
    for (int k = 0; k < 6; k++) {
      cudaError_t e = cudaHostAlloc(&p.hbuf[s][k], p.chunk_bytes, cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: pinned staging alloc");
    }
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

}  // namespace tf

using namespace tf;

extern "C" int tf_elementwise_host(int op, int dtype, int64_t n, const void* const* in,
                                   void* const* out, int device) {
  const int nin = ew_num_inputs(op);
  if (nin < 0) return fail(TF_EINVAL, "tf_elementwise_host: unknown op id");
  if (dtype != TF_F32 && dtype != TF_F64)
    return fail(TF_EINVAL, "tf_elementwise_host: planes must be float32 or float64");
  if (n < 0) return fail(TF_EINVAL, "tf_elementwise_host: negative length");
  if (n == 0) return TF_OK;
  if (!in || !out || !out[0] || !out[1]) return fail(TF_EINVAL, "tf_elementwise_host: null plane");
  for (int k = 0; k < nin; k++)
    if (!in[k]) return fail(TF_EINVAL, "tf_elementwise_host: null plane");
  DeviceGuard g(device);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(TF_EINVAL, "tf_elementwise_host: device ordinal");
  HostPipe& p = g_pipe[dev];
  std::lock_guard<std::mutex> lock(p.mu);
  int rc = pipe_init(p);
  if (rc) return rc;

  bool pin_in[4] = {true, true, true, true}, pin_out[2];
  bool any_pageable = false;
  for (int k = 0; k < nin; k++) any_pageable |= !(pin_in[k] = is_pinned(in[k]));
  for (int k = 0; k < 2; k++) any_pageable |= !(pin_out[k] = is_pinned(out[k]));
  if (any_pageable && (rc = ensure_host_staging(p))) return rc;

  const size_t tsz = dtype == TF_F64 ? 8 : 4;
  const int64_t chunk = p.chunk_bytes / (int64_t)tsz;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const int S = p.slots;
  std::vector<int64_t> slot_off(S, -1);  // chunk offset in flight in each slot

  auto finish = [&](int s) -> int {  // wait for slot s; unstage pageable outputs
    if (slot_off[s] < 0) return TF_OK;
    cudaError_t e = cudaEventSynchronize(p.done[s]);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: sync");
    const int64_t off = slot_off[s];
    const int64_t m = (n - off) < chunk ? (n - off) : chunk;
    for (int k = 0; k < 2; k++)
      if (!pin_out[k])
        par_memcpy(*p.pool, static_cast<char*>(out[k]) + off * tsz, p.hbuf[s][4 + k],
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
    const void* din[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int k = 0; k < nin; k++) {
      const void* src = static_cast<const char*>(in[k]) + off * tsz;
      if (!pin_in[k]) {
        par_memcpy(*p.pool, p.hbuf[s][k], src, bytes);
        src = p.hbuf[s][k];
      }
      cudaError_t e = cudaMemcpyAsync(p.dbuf[s][k], src, bytes, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: H2D");
      din[k] = p.dbuf[s][k];
    }
    void* dout[2] = {p.dbuf[s][4], p.dbuf[s][5]};
    if ((rc = ew_launch(op, dtype, m, din, dout, st))) return rc;
    for (int k = 0; k < 2; k++) {
      void* dst = pin_out[k] ? static_cast<char*>(out[k]) + off * tsz : p.hbuf[s][4 + k];
      cudaError_t e = cudaMemcpyAsync(dst, dout[k], bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: D2H");
    }
    cudaError_t e = cudaEventRecord(p.done[s], st);
    if (e != cudaSuccess) return cuda_status(e, "tf_elementwise_host: event");
    slot_off[s] = off;
  }
  // drain in chunk order
  for (int64_t c = nchunks; c < nchunks + S; c++)
    if ((rc = finish((int)(c % S)))) return rc;
  return TF_OK;
}
