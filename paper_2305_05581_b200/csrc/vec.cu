// vec.cu — Krylov vector algebra for the device Lanczos / Davidson loop
// (dmrg.py:43 lanczos_ground: dot, axpy, full reorthogonalisation, norms).
//
// All reductions run in a fixed order (per-block partials over a fixed grid,
// then one warp per output summing partials in index order), so results are
// bitwise reproducible run to run and identical on every rank that holds the
// same vectors (replicated Krylov space across GPUs).
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "../../include/sdmrg_b200.h"
#include "runtime.h"

namespace sdmrg {

constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// partial[row * gridDim.x + blockIdx.x] = sum over this block's chunk of
// V_row . w   (blockIdx.y = row)
__global__ void dots_partial(int64_t n, const double* __restrict__ v, int64_t ldv,
                             const double* __restrict__ w, double* __restrict__ partial) {
  const int row = blockIdx.y;
  const double* vr = v + (int64_t)row * ldv;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += vr[i] * w[i];
  s = warp_sum(s);
  __shared__ double red[kRedThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[(int64_t)row * gridDim.x + blockIdx.x] = t;
  }
}

// out[row] = sum_b partial[row*nb + b]   (one warp per row, fixed order)
__global__ void dots_final(int rows, int nb, const double* __restrict__ partial,
                           double* __restrict__ out, int sqrt_out) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += partial[(int64_t)row * nb + b];
  s = warp_sum(s);
  if (lane == 0) out[row] = sqrt_out ? sqrt(s) : s;
}

// w[j] += sign * sum_i coef[i] * V[i][j]
__global__ void gemv_n_kernel(int k, int64_t n, const double* __restrict__ v, int64_t ldv,
                              const double* __restrict__ coef, double sign,
                              double* __restrict__ w) {
  extern __shared__ double sc[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) sc[i] = coef[i];
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += sc[i] * v[(int64_t)i * ldv + j];
    w[j] += sign * s;
  }
}

__global__ void scal_dev_kernel(int64_t n, const double* __restrict__ num,
                                const double* __restrict__ den, int invert, double* x) {
  double s = num ? *num : 1.0;
  if (den) s = invert ? s / *den : s * *den;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= s;
}

__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (b == 0.0) ? a * x[i] : a * x[i] + b * y[i];  // b == 0: y may be garbage
}

// Krylov basis as up to kMaxSlabs slabs of slab_rows contiguous vectors
// (lanczos.py KrylovBasis): one launch per reduction / update over all of
// them instead of one per slab.
constexpr int kMaxSlabs = 16;
struct SlabTable {
  const double* p[kMaxSlabs];
};

__global__ void dots_partial_slabs(int64_t n, SlabTable t, int slab_rows,
                                   const double* __restrict__ w, double* __restrict__ partial) {
  const int row = blockIdx.y;
  const double* vr = t.p[row / slab_rows] + (int64_t)(row % slab_rows) * n;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += vr[i] * w[i];
  s = warp_sum(s);
  __shared__ double red[kRedThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double u = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
    u = warp_sum(u);
    if (threadIdx.x == 0) partial[(int64_t)row * gridDim.x + blockIdx.x] = u;
  }
}

// w[j] -= sum_i coef[i] V_i[j] over all slabs; optionally the per-block
// partial sums of the updated w[j]^2 (the norm of the projected vector,
// fused into the same pass over w)
__global__ void gemv_n_slabs(int k, int64_t n, SlabTable t, int slab_rows,
                             const double* __restrict__ coef, double* __restrict__ w,
                             double* __restrict__ sq_partial) {
  extern __shared__ double sc[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) sc[i] = coef[i];
  __syncthreads();
  double sq = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int sl = 0, i0 = 0; i0 < k; ++sl, i0 += slab_rows) {
      const double* v = t.p[sl] + j;
      const int ie = min(k - i0, slab_rows);
      for (int i = 0; i < ie; ++i) s += sc[i0 + i] * v[(int64_t)i * n];
    }
    const double x = w[j] - s;
    w[j] = x;
    sq += x * x;
  }
  if (sq_partial) {
    sq = warp_sum(sq);
    __shared__ double red[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x < 32) {
      double u = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
      u = warp_sum(u);
      if (threadIdx.x == 0) sq_partial[blockIdx.x] = u;
    }
  }
}

static int grid_for_n(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
}

// Reduction partials: one grow-only device buffer per (device, stream),
// reused by every call on that stream (stream order makes reuse safe).  A
// per-call cudaMallocAsync measured ~90 ms per Lanczos reorthogonalisation
// pass once the plan's large allocations had pushed the async pool to
// return memory at every host synchronisation.
static int partials_for(cudaStream_t stream, size_t doubles, double** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<double*, size_t>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = cache[{dev, stream}];
  if (slot.second < doubles) {
    if (slot.first) {
      cudaStreamSynchronize(stream);
      cudaFree(slot.first);
      slot = {nullptr, 0};
    }
    const size_t want = std::max<size_t>(doubles, 64 * kRedBlocks);
    int rc = cuda_check(cudaMalloc(&slot.first, sizeof(double) * want), "cudaMalloc partials");
    if (rc) return rc;
    slot.second = want;
  }
  *out = slot.first;
  return SDMRG_OK;
}

static int dots(int k, int64_t n, const double* v, int64_t ldv, const double* w, double* out,
                int sqrt_out, cudaStream_t stream) {
  if (k <= 0) return SDMRG_OK;
  double* partial = nullptr;
  int rc = partials_for(stream, (size_t)k * kRedBlocks, &partial);
  if (rc) return rc;
  dots_partial<<<dim3(kRedBlocks, k), kRedThreads, 0, stream>>>(n, v, ldv, w, partial);
  dots_final<<<(k + 7) / 8, 256, 0, stream>>>(k, kRedBlocks, partial, out, sqrt_out);
  count_launch(2);
  return cuda_check(cudaGetLastError(), "dots launch");
}

}  // namespace sdmrg

using namespace sdmrg;

extern "C" {

int sdmrg_dot(int64_t n, const double* x, const double* y, double* out_dev, void* stream) {
  if (n < 0) return fail(SDMRG_EINVAL, "dot: negative length");
  return dots(1, n, x, n, y, out_dev, 0, static_cast<cudaStream_t>(stream));
}

int sdmrg_nrm2(int64_t n, const double* x, double* out_dev, void* stream) {
  if (n < 0) return fail(SDMRG_EINVAL, "nrm2: negative length");
  return dots(1, n, x, n, x, out_dev, 1, static_cast<cudaStream_t>(stream));
}

int sdmrg_gemv_t(int k, int64_t n, const double* v, int64_t ldv, const double* w,
                 double* coef_dev, void* stream) {
  if (k < 0 || n < 0 || ldv < n) return fail(SDMRG_EINVAL, "gemv_t: bad dimensions");
  return dots(k, n, v, ldv, w, coef_dev, 0, static_cast<cudaStream_t>(stream));
}

int sdmrg_gemv_n(int k, int64_t n, const double* v, int64_t ldv, const double* coef_dev,
                 double sign, double* w, void* stream) {
  if (k < 0 || n < 0 || ldv < n) return fail(SDMRG_EINVAL, "gemv_n: bad dimensions");
  if (k == 0 || n == 0) return SDMRG_OK;
  gemv_n_kernel<<<grid_for_n(n), 256, sizeof(double) * k, static_cast<cudaStream_t>(stream)>>>(
      k, n, v, ldv, coef_dev, sign, w);
  count_launch();
  return cuda_check(cudaGetLastError(), "gemv_n launch");
}

int sdmrg_krylov_project(int nslabs, const double* const* slabs, int slab_rows, int k, int64_t n,
                         double* w, double* coef_dev, double* norm_dev, void* stream_) {
  if (k < 0 || n < 0 || slab_rows <= 0 || nslabs < 0 || nslabs > kMaxSlabs ||
      (int64_t)nslabs * slab_rows < k || (k > 0 && !slabs))
    return fail(SDMRG_EINVAL, "krylov_project: bad arguments");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  SlabTable t{};
  for (int i = 0; i < nslabs; ++i) t.p[i] = slabs[i];
  const int gn = grid_for_n(n);
  double* partial = nullptr;
  int rc = partials_for(stream, (size_t)std::max(k, 1) * kRedBlocks + gn, &partial);
  if (rc) return rc;
  double* sq = partial + (size_t)std::max(k, 1) * kRedBlocks;
  if (k > 0) {
    dots_partial_slabs<<<dim3(kRedBlocks, k), kRedThreads, 0, stream>>>(n, t, slab_rows, w, partial);
    dots_final<<<(k + 7) / 8, 256, 0, stream>>>(k, kRedBlocks, partial, coef_dev, 0);
    count_launch(2);
  }
  if (n > 0 && (k > 0 || norm_dev)) {
    gemv_n_slabs<<<gn, kRedThreads, sizeof(double) * std::max(k, 1), stream>>>(
        k, n, t, slab_rows, coef_dev, w, norm_dev ? sq : nullptr);
    count_launch();
  }
  if (norm_dev) {
    if (n == 0) return cuda_check(cudaMemsetAsync(norm_dev, 0, sizeof(double), stream), "norm");
    dots_final<<<1, 32, 0, stream>>>(1, gn, sq, norm_dev, 1);
    count_launch();
  }
  return cuda_check(cudaGetLastError(), "krylov_project launch");
}

// Davidson correction with the diagonal preconditioner:
// t[j] = r[j] / (theta - diag[j]), |theta - diag[j]| floored at 1e-3 (a
// tiny floor lets the few diagonal entries nearest θ dominate the
// correction and steer the search space off the ground state)
__global__ void davidson_precond_kernel(int64_t n, const double* __restrict__ r,
                                        const double* __restrict__ diag, double theta,
                                        double* __restrict__ t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double den = theta - diag[i];
    if (fabs(den) < 1e-3) den = den < 0.0 ? -1e-3 : 1e-3;
    t[i] = r[i] / den;
  }
}

int sdmrg_davidson_precond(int64_t n, const double* r, const double* diag, double theta,
                           double* t, void* stream) {
  if (n < 0 || (n > 0 && (!r || !diag || !t))) return fail(SDMRG_EINVAL, "davidson_precond: bad arguments");
  if (n == 0) return SDMRG_OK;
  davidson_precond_kernel<<<grid_for_n(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, r, diag,
                                                                                        theta, t);
  count_launch();
  return cuda_check(cudaGetLastError(), "davidson_precond launch");
}

int sdmrg_scal_dev(int64_t n, const double* num_dev, const double* den_dev, int invert_den,
                   double* x, void* stream) {
  if (n < 0) return fail(SDMRG_EINVAL, "scal: negative length");
  if (n == 0) return SDMRG_OK;
  scal_dev_kernel<<<grid_for_n(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n, num_dev, den_dev, invert_den, x);
  count_launch();
  return cuda_check(cudaGetLastError(), "scal launch");
}

int sdmrg_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream) {
  if (n < 0) return fail(SDMRG_EINVAL, "axpby: negative length");
  if (n == 0) return SDMRG_OK;
  axpby_kernel<<<grid_for_n(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, a, x, b, y);
  count_launch();
  return cuda_check(cudaGetLastError(), "axpby launch");
}

}  // extern "C"
