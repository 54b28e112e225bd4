// line.cu -- the paper's comparison method on the device: line and
// multiline(k) system matrices (baseline.cpp:13-128),
// as CSR (bit-exact) and as matrix-free A x / A^T y.
//
// One thread owns one detector cell (row) and traces its 1, k or k*k rays
// through the grid exactly as trace_ray / cell_ray do (baseline.cpp:13-79):
// same IEEE operations in the same order, compiled with -fmad=false, with the
// per-angle sin/cos from a correctly rounded table (crmath.h). The row's
// hits are then put in the reference's order -- merge_hits (81-94: stable sort
// by column, lengths of equal columns summed in emission order) and
// build_angle_block's stable column sort (projector.cpp:100-102) -- by a
// warp-per-row (<= 1024 hits) or block-per-row (<= 8192 hits) bitonic sort on
// (column, emission index) keys in shared memory.
//
// Matrix-free: A x is a per-row gather (no atomics, deterministic); A^T y is a
// per-row scatter into an int64 fixed-point volume (integer adds commute, so
// the result is independent of the schedule), converted once at the end.
#include "common.cuh"
#include "crmath.h"
#include "kernels.h"

namespace ctsmb {

namespace {

// Per-angle ray table: correctly rounded (cos, sin) of phi_i
// (geometry.hpp:50-52); the reference evaluates std::cos/std::sin of phi in
// cell_ray and detector_point (same argument, same value).
struct RayAngle {
  double cp, sp;
};

__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max

// trace_ray (baseline.cpp:13-67) from (ox, oy, 0) along the unit (ux, uy, uz);
// emit(column, length * scale) per crossed voxel in ray order.
template <typename Emit>
__device__ __forceinline__ void trace_ray(const DevGeom& g, double ox, double oy, double ux,
                                          double uy, double uz, double scale, Emit&& emit) {
  const double lo0 = face(0, g.n_x, g.a), lo1 = face(0, g.n_y, g.b), lo2 = face(0, g.n_z, g.c);
  const double hi0 = face(g.n_x, g.n_x, g.a), hi1 = face(g.n_y, g.n_y, g.b),
               hi2 = face(g.n_z, g.n_z, g.c);
  const double oz = 0.0;
  double tmin = 0.0, tmax = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  // slab clipping per axis (17-32)
  auto clip = [&](double org, double dir, double lo, double hi) -> bool {
    if (fabs(dir) < 1e-15) return !(org < lo || org > hi);
    double ta = (lo - org) / dir;
    double tb = (hi - org) / dir;
    if (ta > tb) {
      const double t = ta;
      ta = tb;
      tb = t;
    }
    tmin = dmax(tmin, ta);
    tmax = dmin(tmax, tb);
    return true;
  };
  if (!clip(ox, ux, lo0, hi0)) return;
  if (!clip(oy, uy, lo1, hi1)) return;
  if (!clip(oz, uz, lo2, hi2)) return;
  if (tmax <= tmin) return;
  const double eps = 1e-12 * dmin(dmin(g.a, g.b), g.c);  // std::min({a,b,c})
  int i0 = (int)floor((ox + (tmin + eps) * ux - lo0) / g.a);
  int i1 = (int)floor((oy + (tmin + eps) * uy - lo1) / g.b);
  int i2 = (int)floor((oz + (tmin + eps) * uz - lo2) / g.c);
  const int s0 = ux > 0 ? 1 : -1, s1 = uy > 0 ? 1 : -1, s2 = uz > 0 ? 1 : -1;
  const int f0 = ux > 0 ? 1 : 0, f1 = uy > 0 ? 1 : 0, f2 = uz > 0 ? 1 : 0;
  double t = tmin;
  while (t < tmax - eps) {
    if (!(i0 >= 0 && i0 < g.n_x && i1 >= 0 && i1 < g.n_y && i2 >= 0 && i2 < g.n_z)) break;
    double tn = tmax;
    int step_ax = -1;
    if (ux != 0.0) {
      const double tc = (lo0 + (i0 + f0) * g.a - ox) / ux;
      if (tc < tn) {
        tn = tc;
        step_ax = 0;
      }
    }
    if (uy != 0.0) {
      const double tc = (lo1 + (i1 + f1) * g.b - oy) / uy;
      if (tc < tn) {
        tn = tc;
        step_ax = 1;
      }
    }
    if (uz != 0.0) {
      const double tc = (lo2 + (i2 + f2) * g.c - oz) / uz;
      if (tc < tn) {
        tn = tc;
        step_ax = 2;
      }
    }
    if (tn > t)
      emit((uint32_t)(((uint64_t)i2 * g.n_y + i1) * g.n_x + i0), (tn - t) * scale);
    if (step_ax < 0 || tn >= tmax) break;
    if (step_ax == 0)
      i0 += s0;
    else if (step_ax == 1)
      i1 += s1;
    else
      i2 += s2;
    t = tn;
  }
}

// cell_ray (baseline.cpp:69-79) with detector_point (geometry.hpp:108-113);
// (cp, sp) = correctly rounded (cos, sin) of phi_i.
template <typename Emit>
__device__ __forceinline__ void cell_ray(const DevGeom& g, const RayAngle& A, double e_y,
                                         double e_z, double scale, Emit&& emit) {
  const double cp = A.cp, sp = A.sp;
  const double ox = g.s * cp, oy = g.s * sp;
  const double dx = -g.d * cp - e_y * g.d_y * sp, dy = -g.d * sp + e_y * g.d_y * cp;
  const double dz = e_z * g.d_z;
  double ux = dx - ox, uy = dy - oy, uz = dz;
  const double nrm = sqrt(ux * ux + uy * uy + uz * uz);
  ux /= nrm;
  uy /= nrm;
  uz /= nrm;
  trace_ray(g, ox, oy, ux, uy, uz, scale, emit);
}

// The rays of one detector cell: line_weights (98-110) or multiline_weights
// (112-126), in the reference's emission order.
template <typename Emit>
__device__ __forceinline__ void cell_rays(const DevGeom& g, const RayAngle& A, int mode, int k,
                                          int m_y, int m_z, Emit&& emit) {
  const bool two_d = g.n_z == 1 && g.n_det_z == 1;
  if (mode == CTSM_MODE_LINE || k == 1) {
    cell_ray(g, A, m_y + 0.5, two_d ? 0.0 : (m_z + 0.5), 1.0, emit);
    return;
  }
  if (two_d) {
    for (int i = 0; i < k; ++i) cell_ray(g, A, m_y + (i + 0.5) / k, 0.0, 1.0 / k, emit);
  } else {
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        cell_ray(g, A, m_y + (i + 0.5) / k, m_z + (j + 0.5) / k, 1.0 / ((double)k * k), emit);
  }
}

struct RowId {
  int ka, m_y, m_z;
};
__device__ __forceinline__ RowId row_id(const DevGeom& g, uint64_t r) {
  const int rpa = g.rows_per_angle;
  RowId id;
  id.ka = (int)(r / rpa);
  const int rr = (int)(r % rpa);
  id.m_z = rr / g.n_det_y - g.n_det_z / 2;
  id.m_y = rr % g.n_det_y - g.n_det_y / 2;
  return id;
}

__global__ void __launch_bounds__(128) ray_count_kernel(DevGeom g, const RayAngle* angs,
                                                        int mode, int k, uint64_t n_rows,
                                                        unsigned* counts) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const RowId id = row_id(g, r);
  const RayAngle A = angs[id.ka];
  unsigned n = 0;
  cell_rays(g, A, mode, k, id.m_y, id.m_z, [&](uint32_t, double) { ++n; });
  counts[r] = n;
}

__global__ void __launch_bounds__(128) ray_fill_kernel(DevGeom g, const RayAngle* angs,
                                                       int mode, int k, uint64_t n_rows,
                                                       const uint64_t* __restrict__ start,
                                                       uint32_t* col, double* val) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const RowId id = row_id(g, r);
  const RayAngle A = angs[id.ka];
  uint64_t p = start[r];
  cell_rays(g, A, mode, k, id.m_y, id.m_z, [&](uint32_t c, double w) {
    col[p] = c;
    val[p] = w;
    ++p;
  });
}

// ---- per-row stable column sort + merge of equal columns -------------------
constexpr int kMergeWarps = 2;
constexpr int kMergeWarpCap = 1024;
constexpr int kMergeBlockCap = 8192;
constexpr int kMergeBlockThreads = 512;

__device__ __forceinline__ void bitonic(unsigned long long* key, int n2, int tid, int nthreads,
                                        bool block) {
  for (int kk = 2; kk <= n2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < n2; i += nthreads) {
        const int p = i ^ j;
        if (p > i) {
          const unsigned long long a = key[i], b = key[p];
          if ((a > b) == ((i & kk) == 0)) {
            key[i] = b;
            key[p] = a;
          }
        }
      }
      if (block)
        __syncthreads();
      else
        __syncwarp();
    }
  }
}

// Sorted keys (col << 32 | emission index) + values by index -> merged row
// written from col[b] / val[b] on; returns the merged count (warp variant).
__device__ __forceinline__ unsigned merge_sorted_warp(const unsigned long long* key,
                                                      const double* sval, int n, uint64_t b,
                                                      uint32_t* col, double* val, int lane) {
  unsigned base = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < n;
    const uint32_t c = valid ? (uint32_t)(key[i] >> 32) : 0u;
    const bool head = valid && (i == 0 || (uint32_t)(key[i - 1] >> 32) != c);
    const unsigned mask = __ballot_sync(0xffffffffu, head);
    if (head) {
      double v = sval[key[i] & 0xffffffffu];
      for (int q = i + 1; q < n && (uint32_t)(key[q] >> 32) == c; ++q) v += sval[key[q] & 0xffffffffu];
      const unsigned pos = base + __popc(mask & ((1u << lane) - 1u));
      col[b + pos] = c;
      val[b + pos] = v;
    }
    base += __popc(mask);
  }
  return base;
}

__global__ void __launch_bounds__(kMergeWarps * 32) sort_merge_warp_kernel(
    uint64_t n_rows, const uint64_t* __restrict__ start, unsigned* counts, uint32_t* col,
    double* val, unsigned* long_rows, unsigned* n_long) {
  __shared__ unsigned long long skey[kMergeWarps][kMergeWarpCap];
  __shared__ double sval[kMergeWarps][kMergeWarpCap];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * kMergeWarps;
  for (uint64_t r = (uint64_t)blockIdx.x * kMergeWarps + wid; r < n_rows; r += warps_total) {
    const uint64_t b = start[r];
    const int n = (int)(start[r + 1] - b);
    if (n <= 1) {
      if (lane == 0) counts[r] = (unsigned)n;
      continue;
    }
    if (n > kMergeWarpCap) {
      if (lane == 0) long_rows[atomicAdd(n_long, 1u)] = (unsigned)r;
      continue;
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = lane; i < n2; i += 32) {
      if (i < n) {
        skey[wid][i] = ((unsigned long long)col[b + i] << 32) | (unsigned)i;
        sval[wid][i] = val[b + i];
      } else {
        skey[wid][i] = ~0ull;
      }
    }
    __syncwarp();
    bitonic(skey[wid], n2, lane, 32, false);
    const unsigned m = merge_sorted_warp(skey[wid], sval[wid], n, b, col, val, lane);
    if (lane == 0) counts[r] = m;
    __syncwarp();
  }
}

// Long rows: one block each (dynamic shared memory: keys + values).
__global__ void __launch_bounds__(kMergeBlockThreads) sort_merge_block_kernel(
    const unsigned* long_rows, const unsigned* n_long, const uint64_t* __restrict__ start,
    unsigned* counts, uint32_t* col, double* val, int* status) {
  extern __shared__ __align__(16) unsigned char dyn[];
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(dyn);
  double* sval = reinterpret_cast<double*>(dyn + sizeof(unsigned long long) * kMergeBlockCap);
  __shared__ unsigned warp_heads[kMergeBlockThreads / 32];
  __shared__ unsigned s_base;
  const unsigned nl = *n_long;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (unsigned q = blockIdx.x; q < nl; q += gridDim.x) {
    const uint64_t r = long_rows[q];
    const uint64_t b = start[r];
    const int n = (int)(start[r + 1] - b);
    if (n > kMergeBlockCap) {
      if (tid == 0) raise_status(status, CTSM_ERR_TOO_LARGE);
      continue;
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int i = tid; i < n2; i += blockDim.x) {
      if (i < n) {
        skey[i] = ((unsigned long long)col[b + i] << 32) | (unsigned)i;
        sval[i] = val[b + i];
      } else {
        skey[i] = ~0ull;
      }
    }
    if (tid == 0) s_base = 0;
    __syncthreads();
    bitonic(skey, n2, tid, blockDim.x, true);
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
      const int i = i0 + tid;
      const bool valid = i < n;
      const uint32_t c = valid ? (uint32_t)(skey[i] >> 32) : 0u;
      const bool head = valid && (i == 0 || (uint32_t)(skey[i - 1] >> 32) != c);
      const unsigned mask = __ballot_sync(0xffffffffu, head);
      if (lane == 0) warp_heads[wid] = __popc(mask);
      __syncthreads();
      unsigned off = s_base;
      for (int w = 0; w < wid; ++w) off += warp_heads[w];
      if (head) {
        double v = sval[skey[i] & 0xffffffffu];
        for (int p = i + 1; p < n && (uint32_t)(skey[p] >> 32) == c; ++p)
          v += sval[skey[p] & 0xffffffffu];
        const unsigned pos = off + __popc(mask & ((1u << lane) - 1u));
        col[b + pos] = c;
        val[b + pos] = v;
      }
      __syncthreads();
      if (tid == 0) {
        unsigned tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += warp_heads[w];
        s_base += tot;
      }
      __syncthreads();
    }
    if (tid == 0) counts[r] = s_base;
    __syncthreads();
  }
}

// merged rows [raw_start[r], + count) -> [row_start[r], ...) (warp per row)
__global__ void compact_rows_kernel(uint64_t n_rows, const uint64_t* __restrict__ raw_start,
                                    const uint64_t* __restrict__ row_start,
                                    const uint32_t* __restrict__ rcol,
                                    const double* __restrict__ rval, uint32_t* col,
                                    double* val) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps_total) {
    const uint64_t s = raw_start[r], d = row_start[r], n = row_start[r + 1] - d;
    for (uint64_t j = lane; j < n; j += 32) {
      col[d + j] = rcol[s + j];
      val[d + j] = rval[s + j];
    }
  }
}

// ---- matrix-free ------------------------------------------------------------
// Shard rows: local row r -> angle slot ka (angle angle_begin + ka * step).
template <typename T>
__global__ void __launch_bounds__(128) ray_fwd_kernel(DevGeom g, const RayAngle* angs, int mode,
                                                      int k, int angle_begin, int angle_step,
                                                      uint64_t n_rows, const T* __restrict__ x,
                                                      T* y, unsigned long long* n_upd,
                                                      int* status) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned cnt = 0;
  if (r < n_rows) {
    const RowId id = row_id(g, r);
    const RayAngle A = angs[id.ka];
    double acc = 0.0;
    cell_rays(g, A, mode, k, id.m_y, id.m_z, [&](uint32_t c, double w) {
      acc += w * (double)x[c];
      ++cnt;
    });
    const uint64_t row = (uint64_t)(angle_begin + id.ka * angle_step) * g.rows_per_angle +
                         (r % (uint64_t)g.rows_per_angle);
    y[row] = (T)acc;
    if (!isfinite(acc)) raise_status(status, CTSM_ERR_NON_FINITE);
  }
  // updates counter (one atomic per warp)
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_upd, (unsigned long long)cnt);
}

template <typename T>
__global__ void __launch_bounds__(128) ray_bwd_kernel(DevGeom g, const RayAngle* angs, int mode,
                                                      int k, int angle_begin, int angle_step,
                                                      uint64_t n_rows, const T* __restrict__ y,
                                                      unsigned long long* acc, double scale) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const RowId id = row_id(g, r);
  const uint64_t row = (uint64_t)(angle_begin + id.ka * angle_step) * g.rows_per_angle +
                       (r % (uint64_t)g.rows_per_angle);
  const double ys = (double)y[row] * scale;
  if (ys == 0.0) return;
  const RayAngle A = angs[id.ka];
  cell_rays(g, A, mode, k, id.m_y, id.m_z, [&](uint32_t c, double w) {
    atomicAdd(&acc[c], (unsigned long long)__double2ll_rn(w * ys));
  });
}

template <typename T>
__global__ void fixed_to_t_kernel(uint64_t n, const unsigned long long* acc, double inv_scale,
                                  T* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)((double)(long long)acc[i] * inv_scale);
}

// RayAngle table for a strided shard (angle_begin + k * step)
__global__ void strided_angle_table(DevGeom g, int angle_begin, int step, int n, RayAngle* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = angle_begin + k * step;
  const double phi = g.angle_start + (g.angle_end - g.angle_start) * i / g.n_angles;
  RayAngle A;
  A.cp = crm_cos(phi);
  A.sp = crm_sin(phi);
  out[k] = A;
}

unsigned grid1(uint64_t n, int bs) {
  const uint64_t b = (n + bs - 1) / bs;
  return (unsigned)(b ? b : 1);
}

}  // namespace

size_t ray_angle_bytes() { return sizeof(RayAngle); }

cudaError_t ray_angle_table(const DevGeom& g, int angle_begin, int angle_step, int n_sel,
                            void* angles_dev, cudaStream_t st) {
  if (n_sel <= 0) return cudaSuccess;
  strided_angle_table<<<grid1(n_sel, 128), 128, 0, st>>>(g, angle_begin, angle_step, n_sel,
                                                        (RayAngle*)angles_dev);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ray_count(const DevGeom& g, const void* angles_dev, int mode, int k, uint64_t n_rows,
                      unsigned* counts, cudaStream_t st) {
  if (n_rows == 0) return cudaSuccess;
  ray_count_kernel<<<grid1(n_rows, 128), 128, 0, st>>>(g, (const RayAngle*)angles_dev, mode, k,
                                                       n_rows, counts);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ray_fill(const DevGeom& g, const void* angles_dev, int mode, int k, uint64_t n_rows,
                     const uint64_t* start, uint32_t* col, double* val, cudaStream_t st) {
  if (n_rows == 0) return cudaSuccess;
  ray_fill_kernel<<<grid1(n_rows, 128), 128, 0, st>>>(g, (const RayAngle*)angles_dev, mode, k,
                                                      n_rows, start, col, val);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ray_sort_merge(uint64_t n_rows, const uint64_t* start, unsigned* counts, uint32_t* col,
                           double* val, unsigned* long_rows, unsigned* n_long, int* status,
                           cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(n_long, 0, sizeof(unsigned), st);
  if (e != cudaSuccess || n_rows == 0) return e;
  const uint64_t blocks = (n_rows + kMergeWarps - 1) / kMergeWarps;
  const unsigned grid = (unsigned)(blocks < 148ull * 8 ? blocks : 148ull * 8);
  sort_merge_warp_kernel<<<grid, kMergeWarps * 32, 0, st>>>(n_rows, start, counts, col, val,
                                                            long_rows, n_long);
  const size_t smem = (sizeof(unsigned long long) + sizeof(double)) * kMergeBlockCap;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(sort_merge_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  sort_merge_block_kernel<<<148, kMergeBlockThreads, smem, st>>>(long_rows, n_long, start, counts,
                                                                 col, val, status);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t ray_compact(uint64_t n_rows, const uint64_t* raw_start, const uint64_t* row_start,
                        const uint32_t* rcol, const double* rval, uint32_t* col, double* val,
                        cudaStream_t st) {
  if (n_rows == 0) return cudaSuccess;
  const uint64_t blocks = (n_rows + 7) / 8;
  const unsigned grid = (unsigned)(blocks < 148ull * 32 ? blocks : 148ull * 32);
  compact_rows_kernel<<<grid, 256, 0, st>>>(n_rows, raw_start, row_start, rcol, rval, col, val);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ray_fwd_mf(const DevGeom& g, int dtype, const void* angles_dev, int mode, int k,
                       int angle_begin, int angle_step, int n_sel, const void* x, void* y,
                       unsigned long long* n_upd, int* status, cudaStream_t st) {
  const uint64_t n_rows = (uint64_t)n_sel * g.rows_per_angle;
  if (n_rows == 0) return cudaSuccess;
  const RayAngle* A = (const RayAngle*)angles_dev;
  if (dtype == CTSM_F64)
    ray_fwd_kernel<double><<<grid1(n_rows, 128), 128, 0, st>>>(
        g, A, mode, k, angle_begin, angle_step, n_rows, (const double*)x, (double*)y, n_upd, status);
  else
    ray_fwd_kernel<float><<<grid1(n_rows, 128), 128, 0, st>>>(
        g, A, mode, k, angle_begin, angle_step, n_rows, (const float*)x, (float*)y, n_upd, status);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ray_bwd_mf(const DevGeom& g, int dtype, const void* angles_dev, int mode, int k,
                       int angle_begin, int angle_step, int n_sel, const void* y,
                       unsigned long long* acc, double scale, void* x, cudaStream_t st) {
  const uint64_t n_rows = (uint64_t)n_sel * g.rows_per_angle;
  const RayAngle* A = (const RayAngle*)angles_dev;
  const uint64_t nv = (uint64_t)g.n_vox;
  cudaError_t e = cudaMemsetAsync(acc, 0, nv * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (n_rows > 0) {
    if (dtype == CTSM_F64)
      ray_bwd_kernel<double><<<grid1(n_rows, 128), 128, 0, st>>>(
          g, A, mode, k, angle_begin, angle_step, n_rows, (const double*)y, acc, scale);
    else
      ray_bwd_kernel<float><<<grid1(n_rows, 128), 128, 0, st>>>(
          g, A, mode, k, angle_begin, angle_step, n_rows, (const float*)y, acc, scale);
    count_launch();
  }
  const unsigned gc = grid1(nv, 256) < 148u * 16 ? grid1(nv, 256) : 148u * 16;
  if (dtype == CTSM_F64)
    fixed_to_t_kernel<double><<<gc, 256, 0, st>>>(nv, acc, 1.0 / scale, (double*)x);
  else
    fixed_to_t_kernel<float><<<gc, 256, 0, st>>>(nv, acc, 1.0 / scale, (float*)x);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ctsmb
