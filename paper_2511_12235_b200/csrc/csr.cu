#include <climits>
// csr.cu -- K1/K2 consistent system-matrix CSR emission (bit-exact) and the
// K3/K4 CSR appliers. Compiled with -fmad=false (see exact.cuh).
//
// Emission (build_system_matrix, projector.cpp:144-201) runs in two passes
// over (voxel column, angle) work items, both evaluating exactly the same
// weights: pass 1 counts entries per row, a scan yields row_start, pass 2
// scatters (col, w) into per-row slots, and a per-row sort restores the
// reference's strictly ascending column order (projector.cpp:100-102).
#include "exact.cuh"
#include "kernels.h"

namespace ctsmb {

using exact::EdgeAngle;
using exact::ExactAngle;
using exact::Sweep;

size_t exact_angle_bytes() { return sizeof(ExactAngle); }
size_t edge_angle_bytes() { return sizeof(EdgeAngle); }

cudaError_t build_exact_tables(const DevGeom& g, int angle_begin, int n_sel, void* angles_dev,
                               void* edges_dev, cudaStream_t st) {
  if (n_sel > 0) {
    exact::build_angle_table<<<(n_sel + 127) / 128, 128, 0, st>>>(g, angle_begin, n_sel,
                                                                 (ExactAngle*)angles_dev);
    count_launch();
  }
  if (g.n_edges > 0) {
    exact::build_edge_table<<<(g.n_edges + 127) / 128, 128, 0, st>>>(g, (EdgeAngle*)edges_dev);
    count_launch();
  }
  return cudaGetLastError();
}

namespace {

struct Emitter {
  int mode;
  unsigned* row_counter;
  const uint64_t* row_start;
  uint32_t* col;
  double* val;
  __device__ __forceinline__ void operator()(uint64_t row_local, uint32_t column, double w) const {
    if (mode == 0) {
      atomicAdd(&row_counter[row_local], 1u);
    } else {
      const unsigned slot = atomicAdd(&row_counter[row_local], 1u);
      const uint64_t pos = row_start[row_local] + slot;
      col[pos] = column;
      val[pos] = w;
    }
  }
};

// One thread per (pixel, angle): pixel_area_factors (weights2d.cpp:105-129)
// -> emit (projector.cpp:53-60).
#ifndef CTSM_CSR2_MINB
#define CTSM_CSR2_MINB 8  // 64 registers: C0 assembly 42.9 -> 40.5 ms
#endif
__global__ void __launch_bounds__(128, CTSM_CSR2_MINB) csr2d_kernel(DevGeom g, const ExactAngle* __restrict__ angs,
                                                    const EdgeAngle* __restrict__ edges,
                                                    Emitter em, int* status) {
  const long long pix = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= (long long)g.n_x * g.n_y) return;
  const int k = blockIdx.y;
  const int ix = (int)(pix % g.n_x), iy = (int)(pix / g.n_x);
  const ExactAngle A = angs[k];
  const double x0 = face(ix, g.n_x, g.a), x1 = face(ix + 1, g.n_x, g.a);
  const double y0 = face(iy, g.n_y, g.b), y1 = face(iy + 1, g.n_y, g.b);
  Sweep sw;
  if (!exact::strip_sweep(g, A, edges, x0, x1, y0, y1, sw, status)) return;
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  const uint64_t row_base = (uint64_t)k * g.rows_per_angle + (uint64_t)(g.n_det_z / 2) * g.n_det_y;
  const uint32_t column = (uint32_t)pix;
  bool have = false;
  int cur = 0;
  double cw = 0.0;
  for (int p = 0; p < sw.np; ++p) {
    const int cell = sw.pcell[p];
    if (cell < cell_lo || cell > cell_hi) continue;
    double w = exact::piece_area(sw, p, g.s, status);
    if (w < 0.0) {
      if (w < kNegClamp2D) raise_status(status, CTSM_ERR_NON_FINITE);
      w = 0.0;
    }
    if (have && cur == cell) {
      cw += w;
    } else {
      if (have && !(cw <= kEpsWeight)) em(row_base + (cur + g.n_det_y / 2), column, cw);
      cur = cell;
      cw = w;
      have = true;
    }
  }
  if (have && !(cw <= kEpsWeight)) em(row_base + (cur + g.n_det_y / 2), column, cw);
}

// One thread per (voxel column (ix, iy), angle); walks iz. The xy sweep, the
// per-cell 2D weights and the corner depths are shared along the column
// (identical computations), then voxel_volume_factors (weights3d.cpp:354-462)
// runs per voxel.
#ifndef CTSM_CSR3_MINB
#define CTSM_CSR3_MINB 4  // 128 registers (small spills): C2 assembly 2.73 -> 2.51 s
#endif
__global__ void __launch_bounds__(128, CTSM_CSR3_MINB) csr3d_kernel(DevGeom g, const ExactAngle* __restrict__ angs,
                                                    const EdgeAngle* __restrict__ edges,
                                                    Emitter em, int* status) {
  const long long colxy = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (colxy >= (long long)g.n_x * g.n_y) return;
  const int k = blockIdx.y;
  const int ix = (int)(colxy % g.n_x), iy = (int)(colxy / g.n_x);
  const ExactAngle A = angs[k];
  const double s = g.s;
  Sweep sw;
  if (!exact::strip_sweep(g, A, edges, face(ix, g.n_x, g.a), face(ix + 1, g.n_x, g.a),
                          face(iy, g.n_y, g.b), face(iy + 1, g.n_y, g.b), sw, status))
    return;
  const double a = sw.x1 - sw.x0, b = sw.y1 - sw.y0;
  const double sdd = g.s + g.d;
  // depths of the four xy corners (weights3d.cpp:367-371), order x0y0,x0y1,x1y0,x1y1
  double dep[4];
  {
    const double vx[2] = {sw.x0, sw.x1}, vy[2] = {sw.y0, sw.y1};
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        const double depth = s - vx[i] * sw.C - vy[j] * sw.S;
        if (depth <= kEpsDenRel * s) {
          raise_status(status, CTSM_ERR_DEGENERATE_GEOMETRY);
          return;
        }
        dep[2 * i + j] = depth;
      }
  }
  // cell groups with their 2D weight (weights3d.cpp:385-397)
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  int ng = 0;
  unsigned char gbeg[kMaxBrk], gend[kMaxBrk];
  int gcell[kMaxBrk];
  double gw2d[kMaxBrk];
  {
    int i = 0;
    while (i < sw.np) {
      int j = i;
      while (j < sw.np && sw.pcell[j] == sw.pcell[i]) ++j;
      const int cell = sw.pcell[i];
      if (cell >= cell_lo && cell <= cell_hi) {
        double w2d = 0.0;
        for (int p = i; p < j; ++p) w2d += exact::piece_area(sw, p, s, status);
        if (w2d < 0.0) w2d = 0.0;
        gbeg[ng] = (unsigned char)i;
        gend[ng] = (unsigned char)j;
        gcell[ng] = cell;
        gw2d[ng] = w2d;
        ++ng;
      }
      i = j;
    }
  }
  if (ng == 0) return;
  const uint64_t row_base = (uint64_t)k * g.rows_per_angle;
  const double sdd_dz = sdd / g.d_z;
  // Cell group outer, voxel inner (the emission order within a row does not
  // matter: rows are sorted by column afterwards). Along z the top face of
  // voxel iz is the bottom face of voxel iz+1: atom_sum(..., cz, tan_a, zt)
  // of voxel iz and atom_sum(..., cz', tan_a, zb') of voxel iz+1 are the same
  // operation on the same operands whenever cz' == cz bitwise (zb' is
  // face(iz+1) in both), so the value is reused -- bit-identical to
  // recomputing it. Up to 4 row edges are cached per voxel.
  for (int q = 0; q < ng; ++q) {
    const int pi = gbeg[q], pj = gend[q];
    const double w2d = gw2d[q];
    int cL[4] = {INT_MIN, INT_MIN, INT_MIN, INT_MIN};
    double cF[4] = {0.0, 0.0, 0.0, 0.0};
    double ccz = -1.0;  // cz of the cached faces
    for (int iz = 0; iz < g.n_z; ++iz) {
      const double zb = face(iz, g.n_z, g.c), zt = face(iz + 1, g.n_z, g.c);
      const double cz = zt - zb;
      double m_min = 0.0, m_max = 0.0;
      bool first = true;
      for (int qq = 0; qq < 4; ++qq) {
        const double depth = dep[qq];
        const double vz[2] = {zb, zt};
        for (int r = 0; r < 2; ++r) {
          const double m = sdd_dz * vz[r] / depth;
          m_min = first ? m : exact::dmin(m_min, m);
          m_max = first ? m : exact::dmax(m_max, m);
          first = false;
        }
      }
      const uint32_t column = (uint32_t)(((uint64_t)iz * g.n_y + iy) * g.n_x + ix);
      const int fl = (int)floor(m_min);
      const int k_lo = (fl < row_lo) ? row_lo : fl;
      const int ch = (int)ceil(m_max) - 1;
      const int k_hi = (ch < row_hi) ? ch : row_hi;
      const bool reuse = (cz == ccz);
      int nL[4] = {INT_MIN, INT_MIN, INT_MIN, INT_MIN};
      double nF[4] = {0.0, 0.0, 0.0, 0.0};
      int nn = 0;
      if (k_hi >= k_lo) {
        // above(k) lambda (weights3d.cpp:426-440); F(L, z) is atom_sum at
        // zref = z (L > 0) or -z (L < 0); the bottom-face value of edge L
        // comes from the cache when voxel iz-1 computed it as its top face
        auto above = [&](double kk) -> double {
          if (kk <= m_min) return w2d;
          if (kk >= m_max) return 0.0;
          if (kk == 0.0) {
            if (zb >= 0.0) return w2d;
            if (zt <= 0.0) return 0.0;
            return w2d * zt / (zt - zb);
          }
          const int L = (int)kk;
          const double tan_a = kk > 0.0 ? kk * g.d_z / sdd : -kk * g.d_z / sdd;
          const double zt_s = kk > 0.0 ? zt : -zt, zb_s = kk > 0.0 ? zb : -zb;
          double Fb;
          bool hit = false;
          if (reuse) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (!hit && cL[c] == L) {
                Fb = cF[c];
                hit = true;
              }
          }
#ifdef CTSM_CSR3_TWO_SITES
          const double Ft = exact::atom_sum(sw, pi, pj, s, a, b, cz, tan_a, zt_s);
          if (!hit) Fb = exact::atom_sum(sw, pi, pj, s, a, b, cz, tan_a, zb_s);
#else
          // one call site of the (large) atom sum: instruction-cache bound
          // kernel; the same calls on the same operands as two sites
          double Ft = 0.0;
#pragma unroll 1
          for (int f = hit ? 1 : 0; f < 2; ++f) {
            const double r = exact::atom_sum(sw, pi, pj, s, a, b, cz, tan_a, f == 0 ? zb_s : zt_s);
            if (f == 0) Fb = r; else Ft = r;
          }
#endif
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c == nn) {
              nL[c] = L;
              nF[c] = Ft;
            }
          ++nn;
          // weights3d.cpp:432-438: k > 0 -> F(zt) - F(zb); k < 0 -> w2d - (F(-zb) - F(-zt))
          return kk > 0.0 ? Ft - Fb : w2d - (Fb - Ft);
        };
#ifdef CTSM_CSR3_TWO_SITES
        double prev = above((double)k_lo);
        for (int L = k_lo; L <= k_hi; ++L) {
          const double next = above((double)(L + 1));
#else
        // one call site of above(): edges k_lo .. k_hi+1 in order (the same
        // calls as above(k_lo) followed by above(L+1) per row)
        double prev = 0.0;
#pragma unroll 1
        for (int L = k_lo - 1; L <= k_hi; ++L) {
          const double next = above((double)(L + 1));
          if (L < k_lo) {
            prev = next;
            continue;
          }
#endif
          const double v = prev - next;
          if (v > kEpsWeight) {
            em(row_base + (uint64_t)(L + g.n_det_z / 2) * g.n_det_y + (gcell[q] + g.n_det_y / 2),
               column, v);
          } else if (v < kNegClamp3D) {
            raise_status(status, CTSM_ERR_NON_FINITE);
          }
          prev = next;
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        cL[c] = nL[c];
        cF[c] = nF[c];
      }
      ccz = cz;
    }
  }
}

}  // namespace

cudaError_t csr_emit(const DevGeom& g, const void* angles_dev, const void* edges_dev,
                     int angle_begin, int n_sel, int mode, unsigned* row_counter,
                     const uint64_t* row_start, uint32_t* col, double* val, int* status,
                     cudaStream_t st) {
  (void)angle_begin;
  if (n_sel <= 0) return cudaSuccess;
  Emitter em{mode, row_counter, row_start, col, val};
  const long long nxy = (long long)g.n_x * g.n_y;
  dim3 grid((unsigned)((nxy + 127) / 128), (unsigned)n_sel);
  const bool two_d = (g.n_z == 1 && g.n_det_z == 1);
  if (two_d)
    csr2d_kernel<<<grid, 128, 0, st>>>(g, (const ExactAngle*)angles_dev,
                                       (const EdgeAngle*)edges_dev, em, status);
  else
    csr3d_kernel<<<grid, 128, 0, st>>>(g, (const ExactAngle*)angles_dev,
                                       (const EdgeAngle*)edges_dev, em, status);
  count_launch();
  return cudaGetLastError();
}

// ---- exclusive scan u32 -> u64 (three-phase, block size 1024) --------------
namespace {
constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;  // per thread
constexpr int kScanTile = kScanBlock * kScanItems;

__device__ __forceinline__ uint64_t block_scan_excl(uint64_t v, uint64_t* smem, uint64_t* total) {
  // Hillis-Steele over warps via shuffles, then across warps.
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = (lane < (int)(blockDim.x >> 5)) ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint64_t warp_off = wid > 0 ? smem[wid - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_off + x - v;
}

__global__ void scan_reduce_kernel(const unsigned* in, uint64_t n, uint64_t* tile_sums) {
  __shared__ uint64_t smem[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + i;
    if (idx < n) s += in[idx];
  }
  uint64_t total;
  block_scan_excl(s, smem, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void scan_tiles_kernel(uint64_t* tile_sums, uint64_t n_tiles) {
  // single block: sequential over chunks of 1024 tiles
  __shared__ uint64_t smem[32];
  uint64_t carry = 0;
  for (uint64_t base = 0; base < n_tiles; base += blockDim.x) {
    const uint64_t idx = base + threadIdx.x;
    const uint64_t v = idx < n_tiles ? tile_sums[idx] : 0;
    uint64_t total;
    const uint64_t ex = block_scan_excl(v, smem, &total);
    if (idx < n_tiles) tile_sums[idx] = carry + ex;
    carry += total;
    __syncthreads();
  }
}

__global__ void scan_down_kernel(const unsigned* in, uint64_t n, const uint64_t* tile_offs,
                                 uint64_t* out) {
  __shared__ uint64_t smem[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t vals[kScanItems];
  uint64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + i;
    vals[i] = idx < n ? in[idx] : 0;
    s += vals[i];
  }
  uint64_t total;
  uint64_t off = block_scan_excl(s, smem, &total) + tile_offs[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + i;
    if (idx < n) out[idx] = off;
    off += vals[i];
    if (idx + 1 == n) out[n] = off;
  }
}
}  // namespace

size_t scan_scratch_bytes(uint64_t n) {
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile + 1;
  return tiles * sizeof(uint64_t);
}

cudaError_t exclusive_scan_u32_u64(const unsigned* counts, uint64_t n, uint64_t* row_start,
                                   void* scratch, cudaStream_t st) {
  if (n == 0) return cudaMemsetAsync(row_start, 0, sizeof(uint64_t), st);
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  uint64_t* ts = (uint64_t*)scratch;
  scan_reduce_kernel<<<(unsigned)tiles, kScanBlock, 0, st>>>(counts, n, ts);
  scan_tiles_kernel<<<1, kScanBlock, 0, st>>>(ts, tiles);
  scan_down_kernel<<<(unsigned)tiles, kScanBlock, 0, st>>>(counts, n, ts, row_start);
  count_launch(3);
  return cudaGetLastError();
}

// ---- per-row sort by column ---------------------------------------------
namespace {
constexpr int kSortWarps = 2;
constexpr int kWarpCap = 1024;  // rows up to this length are sorted by one warp

__device__ __forceinline__ void bitonic_warp(unsigned long long* key, int n2) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < n2; i += 32) {
        const int p = i ^ j;
        if (p > i) {
          const unsigned long long a = key[i], b = key[p];
          const bool up = ((i & k) == 0);
          if ((a > b) == up) {
            key[i] = b;
            key[p] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kSortWarps * 32) sort_rows_warp(uint64_t n_rows,
                                                                  const uint64_t* __restrict__ rs,
                                                                  uint32_t* col, double* val,
                                                                  unsigned* long_rows,
                                                                  unsigned* n_long) {
  __shared__ unsigned long long skey[kSortWarps][kWarpCap];
  __shared__ double sval[kSortWarps][kWarpCap];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * kSortWarps;
  for (uint64_t r = (uint64_t)blockIdx.x * kSortWarps + wid; r < n_rows; r += warps_total) {
    const uint64_t b = rs[r], e = rs[r + 1];
    const int n = (int)(e - b);
    if (n <= 1) continue;
    if (n > kWarpCap) {
      if (lane == 0) long_rows[atomicAdd(n_long, 1u)] = (unsigned)r;
      continue;
    }
    // already sorted? (cheap check, common for rows from few columns)
    bool sorted = true;
    for (int i = lane; i + 1 < n; i += 32)
      if (col[b + i] > col[b + i + 1]) sorted = false;
    if (__all_sync(0xffffffffu, sorted)) continue;
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
    bitonic_warp(skey[wid], n2);
    for (int i = lane; i < n; i += 32) {
      const unsigned long long kk = skey[wid][i];
      col[b + i] = (uint32_t)(kk >> 32);
      val[b + i] = sval[wid][kk & 0xffffffffu];
    }
    __syncwarp();
  }
}

// Long rows: one block each, shell-sort in global memory by a single thread
// (rare; keeps correctness for any geometry).
__global__ void sort_rows_long(const unsigned* long_rows, const unsigned* n_long,
                               const uint64_t* __restrict__ rs, uint32_t* col, double* val) {
  const unsigned nl = *n_long;
  for (unsigned q = blockIdx.x; q < nl; q += gridDim.x) {
    if (threadIdx.x != 0) continue;
    const uint64_t r = long_rows[q];
    const uint64_t b = rs[r];
    const long long n = (long long)(rs[r + 1] - b);
    long long gap = 1;
    while (gap < n / 3) gap = 3 * gap + 1;
    for (; gap > 0; gap /= 3)
      for (long long i = gap; i < n; ++i) {
        const uint32_t c = col[b + i];
        const double v = val[b + i];
        long long j = i;
        while (j >= gap && col[b + j - gap] > c) {
          col[b + j] = col[b + j - gap];
          val[b + j] = val[b + j - gap];
          j -= gap;
        }
        col[b + j] = c;
        val[b + j] = v;
      }
  }
}
}  // namespace

cudaError_t csr_sort_rows(uint64_t n_rows, const uint64_t* row_start, uint32_t* col,
                          double* val, unsigned* long_rows, unsigned* n_long, int* status,
                          cudaStream_t st) {
  (void)status;
  cudaError_t e = cudaMemsetAsync(n_long, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  if (n_rows == 0) return cudaSuccess;
  const uint64_t blocks = (n_rows + kSortWarps - 1) / kSortWarps;
  const unsigned grid = (unsigned)(blocks < 148ull * 16 ? blocks : 148ull * 16);
  sort_rows_warp<<<grid, kSortWarps * 32, 0, st>>>(n_rows, row_start, col, val, long_rows, n_long);
  sort_rows_long<<<148, 32, 0, st>>>(long_rows, n_long, row_start, col, val);
  count_launch(2);
  return cudaGetLastError();
}

// ---- K3: y = A x, one warp per row, fixed reduction tree (deterministic) ---
namespace {
__global__ void __launch_bounds__(256) spmv_kernel(uint64_t n_rows, const uint64_t* __restrict__ rs,
                                                   const uint32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x, double* y,
                                                   int* status) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps_total) {
    const uint64_t b = rs[r], e = rs[r + 1];
    double acc = 0.0;
    // col / val are read once: streaming (evict-first) loads keep x in
    // L2 (C2: 12.7 -> 11.9-12.1 ms, 67 -> 70-72 % of HBM; a second
    // accumulator with two rounds in flight, prefetching the next row's
    // bounds, or one resident wave of blocks were all slower)
    for (uint64_t j = b + lane; j < e; j += 32) acc += __ldcs(&val[j]) * __ldg(&x[__ldcs(&col[j])]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      y[r] = acc;
      if (!isfinite(acc)) raise_status(status, CTSM_ERR_NON_FINITE);
    }
  }
}

__global__ void colsum_abs_kernel(uint64_t n_rows, const uint64_t* __restrict__ rs,
                                  const uint32_t* __restrict__ col, const double* __restrict__ val,
                                  double* colsum) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps_total) {
    for (uint64_t j = rs[r] + lane; j < rs[r + 1]; j += 32)
      atomicAdd(&colsum[__ldcs(&col[j])], fabs(__ldcs(&val[j])));
  }
}

// K4 scatter in fixed point: x_acc[c] += round(val * y[r] * scale). Integer
// addition is associative, so the result is independent of execution order.
__global__ void spmvt_fixed_kernel(uint64_t n_rows, const uint64_t* __restrict__ rs,
                                   const uint32_t* __restrict__ col,
                                   const double* __restrict__ val, const double* __restrict__ y,
                                   unsigned long long* acc, double scale) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps_total) {
    const double yr = y[r];
    if (yr == 0.0) continue;  // projector.cpp:226
    const double ys = yr * scale;
    for (uint64_t j = rs[r] + lane; j < rs[r + 1]; j += 32)
      atomicAdd(&acc[__ldcs(&col[j])], (unsigned long long)__double2ll_rn(__ldcs(&val[j]) * ys));
  }
}
}  // namespace

static unsigned row_grid(uint64_t n_rows, int warps_per_block, int blocks_per_sm = 32) {
  const uint64_t blocks = (n_rows + warps_per_block - 1) / warps_per_block;
  const uint64_t cap = 148ull * blocks_per_sm;
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

cudaError_t spmv_csr(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                     const double* val, const double* x, double* y, int* status,
                     cudaStream_t st) {
  spmv_kernel<<<row_grid(n_rows, 8), 256, 0, st>>>(n_rows, row_start, col, val, x, y, status);
  count_launch();
  return cudaGetLastError();
}

cudaError_t colsum_abs(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                       const double* val, double* colsum, cudaStream_t st) {
  colsum_abs_kernel<<<row_grid(n_rows, 8), 256, 0, st>>>(n_rows, row_start, col, val, colsum);
  count_launch();
  return cudaGetLastError();
}

cudaError_t spmvt_csr_fixed(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                            const double* val, const double* y, unsigned long long* acc,
                            double scale, cudaStream_t st) {
  spmvt_fixed_kernel<<<row_grid(n_rows, 8), 256, 0, st>>>(n_rows, row_start, col, val, y, acc,
                                                          scale);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ctsmb
