// weights.cu -- the reference's weight API on the device (bit-exact path,
// compiled with -fmad=false):
//   * pixel_area_factors (weights2d.cpp:105-129) and voxel_volume_factors
//     (weights3d.cpp:354-462) for a batch of (voxel, phi) queries, one thread
//     per query, results in the reference's order (ascending m_y, then m_z);
//   * detail::angle_block_entries (projector.cpp:44-84): the entries of one
//     angle block reordered from emission records into the reference's
//     emission order (voxels z -> y -> x, each voxel's weights by (m_y, m_z)).
// These serve callers of the reference's weight API (validate.cpp,
// acceptance.cpp:92-95) and the C++ drop-in; the hot paths are csr.cu / mf.cu.
#include "exact.cuh"
#include "kernels.h"

namespace ctsmb {

namespace {

using exact::EdgeAngle;
using exact::ExactAngle;
using exact::Sweep;

// ExactAngle of an arbitrary phi (the reference's functions take phi, not an
// angle index): phi and its sequential quarter turns (geometry.cpp:85-91).
__device__ ExactAngle angle_of_phi(double phi) {
  ExactAngle A;
  double f = phi;
  for (int r = 0; r < 4; ++r) {
    A.fphi[r] = f;
    A.sn[r] = crm_sin(f);
    A.cs[r] = crm_cos(f);
    f -= kPi / 2;
  }
  return A;
}

struct Slab {
  int cap;
  int* count;
  int* my;
  int* mz;
  double* w;
  __device__ void push(long long q, int& n, int m_y, int m_z, double v) const {
    if (n < cap) {
      my[q * cap + n] = m_y;
      mz[q * cap + n] = m_z;
      w[q * cap + n] = v;
    }
    ++n;
  }
};

__global__ void __launch_bounds__(64) weights_batch_kernel(DevGeom g,
                                                           const EdgeAngle* __restrict__ edges,
                                                           long long n_q, const int* __restrict__ ix,
                                                           const int* __restrict__ iy,
                                                           const int* __restrict__ iz,
                                                           const double* __restrict__ phi,
                                                           Slab out, int* status) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_q) return;
  const bool two_d = (g.n_z == 1 && g.n_det_z == 1);
  const ExactAngle A = angle_of_phi(phi[q]);
  const double s = g.s;
  int n = 0;
  out.count[q] = 0;
  Sweep sw;
  if (!exact::strip_sweep(g, A, edges, face(ix[q], g.n_x, g.a), face(ix[q] + 1, g.n_x, g.a),
                          face(iy[q], g.n_y, g.b), face(iy[q] + 1, g.n_y, g.b), sw, status))
    return;
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  if (two_d) {
    // pixel_area_factors (weights2d.cpp:105-129)
    bool have = false;
    int cur = 0;
    double cw = 0.0;
    exact::AreaCache ac;
    for (int p = 0; p < sw.np; ++p) {
      const int cell = sw.pcell[p];
      if (cell < cell_lo || cell > cell_hi) continue;
      double w = exact::piece_area_cached(sw, p, s, status, ac);
      if (w < 0.0) {
        if (w < kNegClamp2D) raise_status(status, CTSM_ERR_NON_FINITE);
        w = 0.0;
      }
      if (have && cur == cell) {
        cw += w;
      } else {
        if (have && !(cw <= kEpsWeight)) out.push(q, n, cur, 0, cw);
        cur = cell;
        cw = w;
        have = true;
      }
    }
    if (have && !(cw <= kEpsWeight)) out.push(q, n, cur, 0, cw);
    out.count[q] = n;
    return;
  }
  // voxel_volume_factors (weights3d.cpp:354-462), in the reference's order
  const double a = sw.x1 - sw.x0, b = sw.y1 - sw.y0;
  const double zb = face(iz[q], g.n_z, g.c), zt = face(iz[q] + 1, g.n_z, g.c);
  const double cz = zt - zb;
  const double sdd = g.s + g.d;
  double m_min = 0.0, m_max = 0.0;
  {
    bool first = true;
    const double vx[2] = {sw.x0, sw.x1}, vy[2] = {sw.y0, sw.y1}, vz[2] = {zb, zt};
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        const double depth = s - vx[i] * sw.C - vy[j] * sw.S;
        if (depth <= kEpsDenRel * s) {
          raise_status(status, CTSM_ERR_DEGENERATE_GEOMETRY);
          return;
        }
        for (int r = 0; r < 2; ++r) {
          const double m = sdd / g.d_z * vz[r] / depth;
          m_min = first ? m : exact::dmin(m_min, m);
          m_max = first ? m : exact::dmax(m_max, m);
          first = false;
        }
      }
  }
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  int i = 0;
  exact::AreaCache ac;
  while (i < sw.np) {
    int j = i;
    while (j < sw.np && sw.pcell[j] == sw.pcell[i]) ++j;
    const int cell = sw.pcell[i];
    if (cell >= cell_lo && cell <= cell_hi) {
      double w2d = 0.0;
      for (int p = i; p < j; ++p) w2d += exact::piece_area_cached(sw, p, s, status, ac);
      if (w2d < 0.0) w2d = 0.0;
      auto above = [&](double kk) -> double {
        if (kk <= m_min) return w2d;
        if (kk >= m_max) return 0.0;
        if (kk == 0.0) {
          if (zb >= 0.0) return w2d;
          if (zt <= 0.0) return 0.0;
          return w2d * zt / (zt - zb);
        }
        if (kk > 0.0) {
          const double tan_a = kk * g.d_z / sdd;
          return exact::atom_sum(sw, i, j, s, a, b, cz, tan_a, zt) -
                 exact::atom_sum(sw, i, j, s, a, b, cz, tan_a, zb);
        }
        const double tan_a = -kk * g.d_z / sdd;
        return w2d - (exact::atom_sum(sw, i, j, s, a, b, cz, tan_a, -zb) -
                      exact::atom_sum(sw, i, j, s, a, b, cz, tan_a, -zt));
      };
      const int fl = (int)floor(m_min);
      const int k_lo = fl < row_lo ? row_lo : fl;
      const int ch = (int)ceil(m_max) - 1;
      const int k_hi = ch < row_hi ? ch : row_hi;
      if (k_hi >= k_lo) {
        double prev = above((double)k_lo);
        for (int L = k_lo; L <= k_hi; ++L) {
          const double next = above((double)(L + 1));
          const double v = prev - next;
          if (v > kEpsWeight) out.push(q, n, cell, L, v);
          else if (v < kNegClamp3D) raise_status(status, CTSM_ERR_NON_FINITE);
          prev = next;
        }
      }
    }
    i = j;
  }
  out.count[q] = n;
}

// ---- angle_block_entries: records -> emission order -----------------------
__global__ void __launch_bounds__(256) count_columns_kernel(const uint4* __restrict__ rec,
                                                            const unsigned long long* n_dev,
                                                            unsigned long long cap,
                                                            unsigned* counts) {
  const unsigned long long n = *n_dev < cap ? *n_dev : cap;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint4 r = rec[i];
    if (r.x != 0xffffffffu) atomicAdd(&counts[r.y], 1u);
  }
}

__global__ void __launch_bounds__(256) scatter_columns_kernel(const uint4* __restrict__ rec,
                                                              const unsigned long long* n_dev,
                                                              unsigned long long cap,
                                                              unsigned* cursor, uint4* tmp) {
  const unsigned long long n = *n_dev < cap ? *n_dev : cap;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint4 r = rec[i];
    if (r.x == 0xffffffffu) continue;
    tmp[atomicAdd(&cursor[r.y], 1u)] = r;
  }
}

// After the scatter cursor[c] is the end of column c's range (and the start
// of column c + 1's): order each column's entries by (m_y, m_z) and write the
// three output arrays.
__global__ void __launch_bounds__(256) order_columns_kernel(uint64_t n_cols,
                                                            const unsigned* __restrict__ cursor,
                                                            uint4* tmp, int n_det_y, int n_det_z,
                                                            uint32_t* raster, uint32_t* col,
                                                            double* w) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const unsigned b = c == 0 ? 0u : cursor[c - 1], e = cursor[c];
  auto key = [&](const uint4& r) { return (r.x % (unsigned)n_det_y) * (unsigned)n_det_z + r.x / (unsigned)n_det_y; };
  for (unsigned i = b + 1; i < e; ++i) {
    const uint4 r = tmp[i];
    const unsigned kr = key(r);
    unsigned j = i;
    while (j > b && key(tmp[j - 1]) > kr) {
      tmp[j] = tmp[j - 1];
      --j;
    }
    tmp[j] = r;
  }
  for (unsigned i = b; i < e; ++i) {
    const uint4 r = tmp[i];
    raster[i] = r.x;
    col[i] = r.y;
    w[i] = __hiloint2double((int)r.w, (int)r.z);
  }
}

__global__ void __launch_bounds__(256) expand_rows_kernel(uint64_t n_rows,
                                                          const uint64_t* __restrict__ rs,
                                                          uint32_t* raster) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps)
    for (uint64_t j = rs[r] - rs[0] + lane; j < rs[r + 1] - rs[0]; j += 32) raster[j] = (uint32_t)r;
}

}  // namespace

cudaError_t weights_batch(const DevGeom& g, const void* edges_dev, long long n_q, const int* ix,
                          const int* iy, const int* iz, const double* phi, int cap, int* count,
                          int* my, int* mz, double* w, int* status, cudaStream_t st) {
  if (n_q <= 0) return cudaSuccess;
  Slab out{cap, count, my, mz, w};
  weights_batch_kernel<<<(unsigned)((n_q + 63) / 64), 64, 0, st>>>(
      g, (const exact::EdgeAngle*)edges_dev, n_q, ix, iy, iz, phi, out, status);
  count_launch();
  return cudaGetLastError();
}

cudaError_t records_to_emission_order(const void* rec, const unsigned long long* n_dev,
                                      unsigned long long cap, uint64_t n_cols, unsigned* counts,
                                      uint64_t* scan_tmp, void* scan_scratch, void* tmp,
                                      int n_det_y, int n_det_z, uint32_t* raster, uint32_t* col,
                                      double* w, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(counts, 0, n_cols * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  count_columns_kernel<<<148 * 16, 256, 0, st>>>((const uint4*)rec, n_dev, cap, counts);
  e = exclusive_scan_u32_u64(counts, n_cols, scan_tmp, scan_scratch, st, 0, nullptr, counts);
  if (e != cudaSuccess) return e;
  scatter_columns_kernel<<<148 * 16, 256, 0, st>>>((const uint4*)rec, n_dev, cap, counts,
                                                   (uint4*)tmp);
  order_columns_kernel<<<(unsigned)((n_cols + 255) / 256), 256, 0, st>>>(
      n_cols, counts, (uint4*)tmp, n_det_y, n_det_z, raster, col, w);
  count_launch(3);
  return cudaGetLastError();
}

cudaError_t expand_row_index(uint64_t n_rows, const uint64_t* row_start, uint32_t* raster,
                             cudaStream_t st) {
  if (n_rows == 0) return cudaSuccess;
  const uint64_t blocks = (n_rows + 7) / 8;
  expand_rows_kernel<<<(unsigned)(blocks < 148ull * 16 ? blocks : 148ull * 16), 256, 0, st>>>(
      n_rows, row_start, raster);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ctsmb
