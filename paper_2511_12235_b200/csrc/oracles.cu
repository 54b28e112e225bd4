// oracles.cu -- the reference's independent numerical oracles on the device
// (oracle.cpp:70-196), for batches of (voxel box, cell)
// cases so the 3D oracle suite (validate.cpp:167-293) scales to many cases:
//   * mc_volume_3d: uniform point sampling with the reference's 16 mt19937_64
//     sub-streams (seed + shard) -- one thread per (case, shard) runs its
//     stream, so the hit count is the reference's, bit for bit (compiled with
//     -fmad=false; cos / sin of phi from crmath);
//   * multiline_volume_3d: k x k Gauss-Legendre ray grid, one block per case,
//     fixed-order reduction (deterministic; equals the reference's sequential
//     sum up to rounding);
//   * gauss_legendre: the reference's Newton iteration, on the host.
#include <cmath>

#include "common.cuh"
#include "crmath.h"
#include "kernels.h"

namespace ctsmb {
namespace {

struct Mt64 {  // std::mt19937_64
  unsigned long long mt[312];
  int idx;
  __device__ void seed(unsigned long long s) {
    mt[0] = s;
    for (int i = 1; i < 312; ++i)
      mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (unsigned long long)i;
    idx = 312;
  }
  __device__ unsigned long long next() {
    if (idx >= 312) {
      for (int i = 0; i < 312; ++i) {
        const unsigned long long x =
            (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
        mt[i] = mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
      }
      idx = 0;
    }
    unsigned long long x = mt[idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
  }
  __device__ double u01() { return (double)(next() >> 11) * 0x1.0p-53; }  // oracle.cpp:46-49
};

constexpr int kShards = 16;  // oracle.cpp:75

// mc_volume_3d (oracle.cpp:70-98): thread = (case, shard)
__global__ void __launch_bounds__(64) mc_volume_kernel(long long n_cases,
                                                       const double* __restrict__ box,
                                                       const double* __restrict__ phi, double s,
                                                       double d, double d_y, double d_z,
                                                       const int* __restrict__ my,
                                                       const int* __restrict__ mz,
                                                       unsigned long long n_samples,
                                                       unsigned long long seed,
                                                       unsigned long long* hits) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_cases * kShards) return;
  const long long c = t / kShards;
  const int shard = (int)(t % kShards);
  const double x0 = box[6 * c], x1 = box[6 * c + 1], y0 = box[6 * c + 2], y1 = box[6 * c + 3];
  const double zb = box[6 * c + 4], zt = box[6 * c + 5];
  const double cp = crm_cos(phi[c]), sp = crm_sin(phi[c]);
  const int m_y = my[c], m_z = mz[c];
  Mt64 rng;
  rng.seed(seed + (unsigned long long)shard);
  const unsigned long long count =
      n_samples / kShards + (shard < (int)(n_samples % kShards) ? 1 : 0);
  unsigned long long h = 0;
  for (unsigned long long i = 0; i < count; ++i) {
    const double x = x0 + (x1 - x0) * rng.u01();
    const double y = y0 + (y1 - y0) * rng.u01();
    const double z = zb + (zt - zb) * rng.u01();
    const double depth = s - x * cp - y * sp;
    const double uy = (s + d) / depth * (y * cp - x * sp) / d_y;
    const double uz = (s + d) / depth * z / d_z;
    if (uy >= m_y && uy < m_y + 1 && uz >= m_z && uz < m_z + 1) ++h;
  }
  if (h) atomicAdd(&hits[c], h);
}

__device__ __forceinline__ double omin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double omax(double a, double b) { return (a < b) ? b : a; }

// multiline_volume_3d (oracle.cpp:124-196): block = case
constexpr int kGlThreads = 256;
__global__ void __launch_bounds__(kGlThreads) multiline_volume_kernel(
    const double* __restrict__ box, const double* __restrict__ phi, double s, double d, double d_y,
    double d_z, const int* __restrict__ my, const int* __restrict__ mz, int k,
    const double* __restrict__ nodes, const double* __restrict__ wts, double* out) {
  __shared__ double red[kGlThreads];
  const long long c = blockIdx.x;
  const double x0 = box[6 * c], x1 = box[6 * c + 1], y0 = box[6 * c + 2], y1 = box[6 * c + 3];
  const double zb = box[6 * c + 4], zt = box[6 * c + 5];
  const double cp = crm_cos(phi[c]), sp = crm_sin(phi[c]);
  const double sx = s * cp, sy = s * sp;
  double u_min = 0, u_max = 0, v_min = 0, v_max = 0;
  bool first = true;
  const double vxs[2] = {x0, x1}, vys[2] = {y0, y1}, vzs[2] = {zb, zt};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const double depth = s - vxs[a] * cp - vys[b] * sp;
      const double u = (s + d) / depth * (vys[b] * cp - vxs[a] * sp) / d_y;
      u_min = first ? u : omin(u_min, u);
      u_max = first ? u : omax(u_max, u);
      for (int e = 0; e < 2; ++e) {
        const double v = (s + d) / depth * vzs[e] / d_z;
        if (first) {
          v_min = v_max = v;
        } else {
          v_min = omin(v_min, v);
          v_max = omax(v_max, v);
        }
        first = false;
      }
    }
  const double u_lo = omax((double)my[c], u_min), u_hi = omin((double)my[c] + 1.0, u_max);
  const double v_lo = omax((double)mz[c], v_min), v_hi = omin((double)mz[c] + 1.0, v_max);
  if (u_hi <= u_lo || v_hi <= v_lo) {  // uniform over the block
    if (threadIdx.x == 0) out[c] = 0.0;
    return;
  }
  const double uc = 0.5 * (u_lo + u_hi), ur = 0.5 * (u_hi - u_lo);
  const double vc = 0.5 * (v_lo + v_hi), vr = 0.5 * (v_hi - v_lo);
  // One thread per ray of the k x k grid (strided); a ray S + t (D - S) meets
  // the box in the parameter interval common to the three axis slabs, and its
  // share of the cone volume over that interval is (t1^3 - t0^3) / 3.
  double total = 0.0;
  const long long n_rays = (long long)k * k;
  const double src[3] = {sx, sy, 0.0};
  const double bmin[3] = {x0, y0, zb}, bmax[3] = {x1, y1, zt};
  for (long long r = threadIdx.x; r < n_rays; r += kGlThreads) {
    const int i = (int)(r / k), j = (int)(r % k);
    const double ey = (uc + ur * nodes[i]) * d_y;
    const double ez = (vc + vr * nodes[j]) * d_z;
    // detector point of the ray, minus the source
    const double dir[3] = {(-d * cp - ey * sp) - sx, (-d * sp + ey * cp) - sy, ez};
    double t_in = 0.0, t_out = INFINITY;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (fabs(dir[ax]) < 1e-300) {  // parallel to the slab: inside or never
        if (src[ax] < bmin[ax] || src[ax] > bmax[ax]) {
          t_in = 1.0;
          t_out = 0.0;
        }
        continue;
      }
      const double ta = (bmin[ax] - src[ax]) / dir[ax];
      const double tb = (bmax[ax] - src[ax]) / dir[ax];
      t_in = omax(t_in, ta > tb ? tb : ta);
      t_out = omin(t_out, ta > tb ? ta : tb);
    }
    if (t_out > t_in)
      total += wts[i] * wts[j] * (t_out * t_out * t_out - t_in * t_in * t_in) / 3.0;
  }
  red[threadIdx.x] = total;
  __syncthreads();
  for (int o = kGlThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    out[c] = d_y * d_z * (s + d) * red[0] * ur * vr / ((x1 - x0) * (y1 - y0) * (zt - zb));
}

}  // namespace

cudaError_t mc_volume_batch(long long n_cases, const double* box, const double* phi, double s,
                            double d, double d_y, double d_z, const int* my, const int* mz,
                            unsigned long long n_samples, unsigned long long seed,
                            unsigned long long* hits, cudaStream_t st) {
  if (n_cases <= 0) return cudaSuccess;
  const long long threads = n_cases * kShards;
  mc_volume_kernel<<<(unsigned)((threads + 63) / 64), 64, 0, st>>>(n_cases, box, phi, s, d, d_y,
                                                                   d_z, my, mz, n_samples, seed,
                                                                   hits);
  count_launch();
  return cudaGetLastError();
}

cudaError_t multiline_volume_batch(long long n_cases, const double* box, const double* phi,
                                   double s, double d, double d_y, double d_z, const int* my,
                                   const int* mz, int k, const double* nodes, const double* wts,
                                   double* out, cudaStream_t st) {
  if (n_cases <= 0) return cudaSuccess;
  multiline_volume_kernel<<<(unsigned)n_cases, kGlThreads, 0, st>>>(box, phi, s, d, d_y, d_z, my,
                                                                    mz, k, nodes, wts, out);
  count_launch();
  return cudaGetLastError();
}

// gauss_legendre (oracle.cpp:100-122)
void gauss_legendre_host(int k, double* x, double* w) {
  for (int i = 0; i < k; ++i) {
    double t = std::cos(kPi * (i + 0.75) / (k + 0.5));
    double pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 0; j < k; ++j) {
        const double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j + 1.0) * t * p1 - j * p2) / (j + 1.0);
      }
      pp = k * (t * p0 - p1) / (t * t - 1.0);
      const double dt = p0 / pp;
      t -= dt;
      if (std::fabs(dt) < 1e-15) break;
    }
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * pp * pp);
  }
}

}  // namespace ctsmb
