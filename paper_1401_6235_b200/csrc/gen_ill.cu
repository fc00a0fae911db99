// gen_ill.cu — seeded ill-conditioned inputs for BASELINE config 4 (twofold dot
// and sum at n = 2^30, cond ~ 1e16), generated identically on the host and on
// the device (workload tool; the reference repository has no generator).
//
// Method: the Ogita-Rump-Oishi generators ("Accurate sum and dot product",
// SIAM J. Sci. Comput. 26(6), 2005: GenDot, Alg. 6.1, and its summation
// analogue), applied block by block.  The global problem of n_total elements is
// cut into blocks of TF_GEN_BLOCK = 65536 (the f64 reduction tile); in each block
//   * the first half of the terms (dot: pairs x_i, y_i sharing an exponent;
//     sum: terms p_i) are random, mantissa U(-1, 1) and exponent
//     e_i ~ round(U[emin, emax]) — BASELINE's "half the pairs have random
//     exponents in [-50, 50]";
//   * the second half is chosen to cancel the block's running value (carried in
//     double-double, exact TwoSum / TwoProd updates): element i takes a target
//     t = U(-1, 1) * 2^e with e falling linearly from emax to emin, and
//     y_i = (t - cur) / x_i (dot) or p_i = t - cur (sum);
//   * the block's LAST target is calibrated, +c * sum|terms_block| / cond with
//     c = 2 (dot: cond = 2 sum|x_i y_i| / |sum x_i y_i|) or 1 (sum:
//     cond = sum|p_i| / |sum p_i|), always positive.
// Every block — and so every prefix of whole blocks, and the whole problem —
// therefore has the requested condition number, and a block depends only on
// (seed, its global element indices).  Any contiguous run of whole blocks can
// be generated alone: each rank of a multi-GPU run generates exactly its shard
// of one global problem, bit-identical to the N = 1 planes.
//
// The same __host__ __device__ code runs on both sides; no contraction
// (-fmad=false on the device, -ffp-contract=off for the host compiler and no
// FMA in the x86-64 baseline ISA), explicit correctly rounded fma, IEEE
// division, exact ldexp/round: host and device planes are bit-identical
// (tests/test_gpu_gen_ill.py).  Cost: one serial chain per block (latency-bound,
// ~ms on the device for 2^30 elements, seconds on the host threads).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tf {
namespace {

constexpr int64_t GEN_BLOCK = TF_GEN_BLOCK;

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// exact: a 53-bit integer times 2^-53
__host__ __device__ inline double unit(uint64_t key, uint64_t i) {
  return (double)(mix64(key ^ i) >> 11) * 0x1p-53;
}
// U(-1, 1) with 53 random bits (2u - 1 is exact)
__host__ __device__ inline double sym(uint64_t key, uint64_t i) { return 2.0 * unit(key, i) - 1.0; }

struct DDAcc {  // running value s + c, exact updates (TwoSum / TwoProd)
  double s, c, abs_sum;
  __host__ __device__ void add(double p) {
    const double t = s + p;
    const double bv = t - s;
    const double av = t - bv;
    const double e = (s - av) + (p - bv);
    s = t;
    c += e;
  }
};

template <int KIND>  // 0 = dot (x, y), 1 = sum (x only)
__host__ __device__ void gen_block(int64_t g0, int64_t m, double cond, uint64_t key, int emin,
                                   int emax, double* x, double* y) {
  DDAcc acc{0.0, 0.0, 0.0};
  const int64_t h = m / 2;
  const double span = (double)(emax - emin);
  for (int64_t i = 0; i < h; i++) {
    const uint64_t g = (uint64_t)(g0 + i);
    const double e = round((double)emin + unit(key, 4 * g) * span);
    const double sc = ldexp(1.0, (int)e);
    if (KIND == 0) {
      const double xi = sym(key, 4 * g + 1) * sc;
      const double yi = sym(key, 4 * g + 2) * sc;
      x[i] = xi;
      y[i] = yi;
      const double p = xi * yi;
      acc.add(p);
      acc.c += fma(xi, yi, -p);
      acc.abs_sum += fabs(p);
    } else {
      const double p = sym(key, 4 * g + 1) * sc;
      x[i] = p;
      acc.add(p);
      acc.abs_sum += fabs(p);
    }
  }
  const int64_t r = m - h;
  for (int64_t j = 0; j < r; j++) {
    const int64_t i = h + j;
    const uint64_t g = (uint64_t)(g0 + i);
    const double frac = r > 1 ? (double)j / (double)(r - 1) : 1.0;
    const double e = round((double)emax - frac * span);
    const double sc = ldexp(1.0, (int)e);
    double target = sym(key, 4 * g + 2) * sc;
    if (j == r - 1) target = (KIND == 0 ? 2.0 : 1.0) * acc.abs_sum / cond;
    const double cur = acc.s + acc.c;
    if (KIND == 0) {
      double xi = sym(key, 4 * g + 1) * sc;
      if (xi == 0.0) xi = sc;
      const double yi = (target - cur) / xi;
      x[i] = xi;
      y[i] = yi;
      const double p = xi * yi;
      acc.add(p);
      acc.c += fma(xi, yi, -p);
      acc.abs_sum += fabs(p);
    } else {
      const double p = target - cur;
      x[i] = p;
      acc.add(p);
      acc.abs_sum += fabs(p);
    }
  }
}

template <int KIND>
__global__ void gen_ill_kernel(int64_t n_total, int64_t first, int64_t nblocks, double cond,
                               uint64_t key, int emin, int emax, double* x, double* y) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const int64_t g0 = first + b * GEN_BLOCK;
  const int64_t m = n_total - g0 < GEN_BLOCK ? n_total - g0 : GEN_BLOCK;
  gen_block<KIND>(g0, m, cond, key, emin, emax, x + b * GEN_BLOCK,
                  KIND == 0 ? y + b * GEN_BLOCK : nullptr);
}

int check_args(int kind, int64_t n_total, int64_t first, int64_t count, double cond, int emin,
               int emax, const double* x, const double* y) {
  if (kind != 0 && kind != 1) return fail(TF_EINVAL, "tf_gen_ill: kind must be 0 (dot) or 1 (sum)");
  if (n_total < 0 || first < 0 || count < 0 || first + count > n_total)
    return fail(TF_EINVAL, "tf_gen_ill: range outside the global problem");
  if (first % GEN_BLOCK != 0 || ((first + count) % GEN_BLOCK != 0 && first + count != n_total))
    return fail(TF_EINVAL, "tf_gen_ill: the range must cover whole blocks of TF_GEN_BLOCK elements");
  if (!(cond > 1.0)) return fail(TF_EINVAL, "tf_gen_ill: cond must exceed 1");
  if (emin > emax || emin < -500 || emax > 500)
    return fail(TF_EINVAL, "tf_gen_ill: exponent range must satisfy -500 <= emin <= emax <= 500");
  if (count > 0 && (!x || (kind == 0 && !y))) return fail(TF_EINVAL, "tf_gen_ill: null plane");
  return TF_OK;
}

inline uint64_t stream_key(int kind, uint64_t seed) { return mix64(seed * 2 + (uint64_t)kind); }

}  // namespace
}  // namespace tf

using namespace tf;

extern "C" int tf_gen_ill(int kind, int64_t n_total, int64_t first, int64_t count, double cond,
                          uint64_t seed, int emin, int emax, double* x, double* y, void* stream) {
  int rc = check_args(kind, n_total, first, count, cond, emin, emax, x, y);
  if (rc) return rc;
  if (count == 0) return TF_OK;
  const int64_t nblocks = (count + GEN_BLOCK - 1) / GEN_BLOCK;
  const uint64_t key = stream_key(kind, seed);
  const unsigned threads = 64;  // a few blocks per SM: the chains are latency-bound
  const unsigned grid = (unsigned)((nblocks + threads - 1) / threads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (kind == 0)
    gen_ill_kernel<0><<<grid, threads, 0, s>>>(n_total, first, nblocks, cond, key, emin, emax, x, y);
  else
    gen_ill_kernel<1><<<grid, threads, 0, s>>>(n_total, first, nblocks, cond, key, emin, emax, x, y);
  return launch_status("tf_gen_ill");
}

extern "C" int tf_gen_ill_host(int kind, int64_t n_total, int64_t first, int64_t count,
                               double cond, uint64_t seed, int emin, int emax, double* x,
                               double* y, int nthreads) {
  int rc = check_args(kind, n_total, first, count, cond, emin, emax, x, y);
  if (rc) return rc;
  if (count == 0) return TF_OK;
  const int64_t nblocks = (count + GEN_BLOCK - 1) / GEN_BLOCK;
  const uint64_t key = stream_key(kind, seed);
  int nt = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > nblocks) nt = (int)nblocks;
  auto work = [&](int t) {
    for (int64_t b = t; b < nblocks; b += nt) {
      const int64_t g0 = first + b * GEN_BLOCK;
      const int64_t m = std::min<int64_t>(GEN_BLOCK, n_total - g0);
      if (kind == 0)
        gen_block<0>(g0, m, cond, key, emin, emax, x + b * GEN_BLOCK, y + b * GEN_BLOCK);
      else
        gen_block<1>(g0, m, cond, key, emin, emax, x + b * GEN_BLOCK, nullptr);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; t++) th.emplace_back(work, t);
  work(0);
  for (auto& t : th) t.join();
  return TF_OK;
}
