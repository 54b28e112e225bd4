// solver.cu -- device vector kernels of the reconstruction protocol
// (SURVEY.md §8(f) row 1): Nesterov-accelerated Tikhonov least squares
// (reference solver.cpp:17-75) and the spectral-norm power iteration
// (projector.cpp:262-280), both driven by capi.cu over the K3/K4 (CSR) or
// K5/K6 (matrix-free) projectors.
//
// All reductions are deterministic: a fixed grid of kRedBlocks blocks reduces
// in a fixed order into per-block partials, which one block then sums in a
// fixed tree order (no float atomics), so the solver iterates are identical
// run to run. Compiled with -fmad=false like the reference's host code
// (-ffp-contract=off): the elementwise update evaluates the reference's
// expressions operation for operation.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace ctsmb {
namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 4;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  __syncthreads();
  return s;  // valid in thread 0
}

// partial[b] = sum over the block's grid-stride elements of f(i)
template <typename F>
__device__ __forceinline__ void reduce_partial(uint64_t n, double* partial, F&& f) {
  __shared__ double sh[kRedThreads / 32];
  double acc = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += f(i);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out[k] = sum of partial[k * kRedBlocks .. (k+1) * kRedBlocks), k < n_sums;
// optional sqrt. One block.
__global__ void finish_sums_kernel(const double* partial, int n_sums, double* out, int take_sqrt) {
  __shared__ double sh[kRedThreads / 32];
  for (int k = 0; k < n_sums; ++k) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += blockDim.x) acc += partial[k * kRedBlocks + i];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[k] = take_sqrt ? sqrt(s) : s;
  }
}

// NAG step (solver.cpp:39-50): with m = (t-1)/t_next and L = 1 + lambda,
//   y = (1+m) u - m u_prev,  grad = (1+m)(h + lam u) - m (h_prev + lam u_prev) - q,
//   u_prev = u, h_prev = h, u = y - grad / L.
__global__ void nag_step_kernel(uint64_t n, double m, double lam, double L, double* u,
                                double* u_prev, double* h, double* h_prev, const double* q) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double ui = u[i], upi = u_prev[i], hi = h[i], hpi = h_prev[i];
    const double yi = (1.0 + m) * ui - m * upi;
    const double gi = (1.0 + m) * (hi + lam * ui) - m * (hpi + lam * upi) - q[i];
    u_prev[i] = ui;
    h_prev[i] = hi;
    u[i] = yi - gi / L;
  }
}

// h <- hs * h (operator scale), then partial of sum (h + lam u - q)^2
// (solver.cpp:54-58).
__global__ void nag_grad_kernel(uint64_t n, double hs, double lam, double* h, const double* u,
                                const double* q, double* partial) {
  reduce_partial(n, partial, [&](uint64_t i) {
    const double hi = hs == 1.0 ? h[i] : hs * h[i];
    if (hs != 1.0) h[i] = hi;
    const double g = hi + lam * u[i] - q[i];
    return g * g;
  });
}

// partial of sum (vs v - p)^2 (v <- vs v in place) and of sum u^2 (trace row,
// solver.cpp:61-65); partial2 = partial + kRedBlocks.
__global__ void resid_kernel(uint64_t n_rows, double vs, double* v, const double* p,
                             double* partial) {
  reduce_partial(n_rows, partial, [&](uint64_t r) {
    const double vr = vs == 1.0 ? v[r] : vs * v[r];
    if (vs != 1.0) v[r] = vr;
    const double d = vr - p[r];
    return d * d;
  });
}

__global__ void sumsq_kernel(uint64_t n, const double* a, double scale, double* partial) {
  reduce_partial(n, partial, [&](uint64_t i) {
    const double v = scale * a[i];
    return v * v;
  });
}

// v = u / lam (lam = *lam_dev; the power iteration's normalisation,
// projector.cpp:276). A zero lam flags ZeroMatrix and leaves v untouched.
__global__ void normalize_kernel(uint64_t n, const double* u, double us, const double* lam_dev,
                                 double* v, int* status) {
  const double lam = *lam_dev;
  if (lam == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(status, 0, CTSM_ERR_ZERO_MATRIX);
    return;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (us == 1.0 ? u[i] : us * u[i]) / lam;
}

__global__ void scale_kernel(uint64_t n, double* v, double f) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] *= f;
}

unsigned ew_grid(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  const uint64_t cap = 148ull * 16;
  return (unsigned)(b == 0 ? 1 : (b < cap ? b : cap));
}

}  // namespace

size_t solver_partial_doubles() { return 2 * (size_t)kRedBlocks; }

cudaError_t nag_step(uint64_t n, double m, double lam, double L, double* u, double* u_prev,
                     double* h, double* h_prev, const double* q, cudaStream_t st) {
  nag_step_kernel<<<ew_grid(n), 256, 0, st>>>(n, m, lam, L, u, u_prev, h, h_prev, q);
  count_launch();
  return cudaGetLastError();
}

cudaError_t nag_grad_sq(uint64_t n, double hs, double lam, double* h, const double* u,
                        const double* q, double* partial, double* out_dev, cudaStream_t st) {
  nag_grad_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, hs, lam, h, u, q, partial);
  finish_sums_kernel<<<1, kRedThreads, 0, st>>>(partial, 1, out_dev, 0);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t nag_trace_sums(uint64_t n_rows, uint64_t n_cols, double vs, double* v,
                           const double* p, const double* u, double* partial, double* out_dev,
                           cudaStream_t st) {
  resid_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n_rows, vs, v, p, partial);
  sumsq_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n_cols, u, 1.0, partial + kRedBlocks);
  finish_sums_kernel<<<1, kRedThreads, 0, st>>>(partial, 2, out_dev, 0);
  count_launch(3);
  return cudaGetLastError();
}

cudaError_t norm2(uint64_t n, const double* a, double scale, double* partial, double* out_dev,
                  cudaStream_t st) {
  sumsq_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, a, scale, partial);
  finish_sums_kernel<<<1, kRedThreads, 0, st>>>(partial, 1, out_dev, 1);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t normalize_by(uint64_t n, const double* u, double us, const double* lam_dev,
                         double* v, int* status, cudaStream_t st) {
  normalize_kernel<<<ew_grid(n), 256, 0, st>>>(n, u, us, lam_dev, v, status);
  count_launch();
  return cudaGetLastError();
}

cudaError_t scale_in_place(uint64_t n, double* v, double f, cudaStream_t st) {
  scale_kernel<<<ew_grid(n), 256, 0, st>>>(n, v, f);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ctsmb
