// csr.cu -- K1/K2 consistent system-matrix CSR emission (bit-exact) and the
// K3/K4 CSR appliers. Compiled with -fmad=false (see exact.cuh).
//
// Emission (build_system_matrix, projector.cpp:144-201) either evaluates each
// weight once into records that are then grouped by row (ctsm_csr_build), or
// runs twice over the same weights (the count / fill protocol: pass 1 counts
// entries per row, a scan yields row_start, pass 2 writes row-grouped
// entries); in both cases a per-row radix sort restores the reference's
// strictly ascending column order (projector.cpp:100-102).
#include <climits>
#include <cstdlib>

#include "exact.cuh"
#include "csr3d.cuh"
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

using k2::Sink;

// One thread per (pixel, angle): pixel_area_factors (weights2d.cpp:105-129)
// -> emit (projector.cpp:53-60).
#ifndef CTSM_CSR2_MINB
#define CTSM_CSR2_MINB 8  // 64 registers: C0 assembly 42.9 -> 40.5 ms
#endif
__global__ void __launch_bounds__(128, CTSM_CSR2_MINB) csr2d_kernel(DevGeom g, const ExactAngle* __restrict__ angs,
                                                    const EdgeAngle* __restrict__ edges,
                                                    Sink em, int* status) {
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
  exact::AreaCache ac;
  for (int p = 0; p < sw.np; ++p) {
    const int cell = sw.pcell[p];
    if (cell < cell_lo || cell > cell_hi) continue;
    double w = exact::piece_area_cached(sw, p, g.s, status, ac);
    if (w < 0.0) {
      if (w < kNegClamp2D) raise_status(status, CTSM_ERR_NON_FINITE);
      w = 0.0;
    }
    if (have && cur == cell) {
      cw += w;
    } else {
      if (have && !(cw <= kEpsWeight)) k2::emit_any(em, row_base + (cur + g.n_det_y / 2), column, cw);
      cur = cell;
      cw = w;
      have = true;
    }
  }
  if (have && !(cw <= kEpsWeight)) k2::emit_any(em, row_base + (cur + g.n_det_y / 2), column, cw);
}

}  // namespace

cudaError_t selftest_division(unsigned long long n, unsigned long long seed,
                              unsigned long long* mismatches_dev, cudaStream_t st) {
  k2::selftest_division_kernel<<<148 * 8, 256, 0, st>>>(n, seed, mismatches_dev);
  count_launch();
  return cudaGetLastError();
}

size_t csr_plan_bytes(const DevGeom& g, int n_sel) {
  if (g.n_z == 1 && g.n_det_z == 1) return 0;
  return (size_t)g.n_x * g.n_y * (size_t)n_sel * sizeof(k2::ColPlan);
}

// Emission of angles [0, n_sel) of the prepared tables (rows local to the
// shard). 3D: plan kernel + warp-per-column kernel (csr3d.cuh); `plans` needs
// csr_plan_bytes(g, n_sel) bytes.
cudaError_t csr_emit(const DevGeom& g, const void* angles_dev, const void* edges_dev, int n_sel,
                     const CsrSink& out, void* plans, int* status, cudaStream_t st) {
  if (n_sel <= 0) return cudaSuccess;
  Sink em{out.mode, out.row_counter, out.row_start, (uint4*)out.grp, (uint4*)out.rec,
          out.cursor, out.cap, 0u, out.pos_base};
  const long long nxy = (long long)g.n_x * g.n_y;
  const bool two_d = (g.n_z == 1 && g.n_det_z == 1);
  const ExactAngle* angs = (const ExactAngle*)angles_dev;
  const EdgeAngle* edges = (const EdgeAngle*)edges_dev;
  // gridDim.y <= 65535: launch the angles in slices
  for (int k0 = 0; k0 < n_sel; k0 += 32768) {
    const int nk = n_sel - k0 < 32768 ? n_sel - k0 : 32768;
    Sink e2 = em;
    const uint64_t row_off = (uint64_t)k0 * g.rows_per_angle;
    e2.row_counter = em.row_counter + row_off;
    if (em.row_start) e2.row_start = em.row_start + row_off;
    e2.row_bias = (unsigned)row_off;
    dim3 grid((unsigned)((nxy + 127) / 128), (unsigned)nk);
    if (two_d) {
      csr2d_kernel<<<grid, 128, 0, st>>>(g, angs + k0, edges, e2, status);
      count_launch();
    } else {
      k2::ColPlan* pl = (k2::ColPlan*)plans + (size_t)k0 * nxy;
      k2::plan3d_kernel<<<grid, 128, 0, st>>>(g, angs + k0, edges, pl, status);
      const long long items = nxy * nk;
      const long long blocks = (items + k2::kEmitWarps - 1) / k2::kEmitWarps;
      static const int per_sm = [] {  // experiment knob: emission blocks per SM
        const char* e = getenv("CTSM_EMIT3_BLOCKS");
        return e ? atoi(e) : CTSM_EMIT3_MINB;
      }();
      const long long cap = 148ll * per_sm;  // one resident wave, warps stride
      k2::emit3d_kernel<<<(unsigned)(blocks < cap ? blocks : cap), k2::kEmitWarps * 32, 0, st>>>(
          g, pl, nk, e2, status);
      count_launch(2);
    }
  }
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
                                 uint64_t* out, uint64_t out_base, const uint64_t* base_dev,
                                 unsigned* local_out) {
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
  uint64_t loc = block_scan_excl(s, smem, &total) + tile_offs[blockIdx.x];
  uint64_t off = loc + out_base + (base_dev ? *base_dev : 0);
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + i;
    if (idx < n) out[idx] = off;
    // the shard-local offset (may alias the counts: each thread has read its items)
    if (idx < n && local_out) local_out[idx] = (unsigned)loc;
    loc += vals[i];
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
                                   void* scratch, cudaStream_t st, uint64_t base,
                                   const uint64_t* base_dev, unsigned* local_out) {
  if (n == 0) {
    if (base_dev) return cudaMemcpyAsync(row_start, base_dev, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st);
    return cudaMemcpyAsync(row_start, &base, sizeof(uint64_t), cudaMemcpyHostToDevice, st);
  }
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  uint64_t* ts = (uint64_t*)scratch;
  scan_reduce_kernel<<<(unsigned)tiles, kScanBlock, 0, st>>>(counts, n, ts);
  scan_tiles_kernel<<<1, kScanBlock, 0, st>>>(ts, tiles);
  scan_down_kernel<<<(unsigned)tiles, kScanBlock, 0, st>>>(counts, n, ts, row_start, base, base_dev,
                                                           local_out);
  count_launch(3);
  return cudaGetLastError();
}

// ---- single-evaluation build: records -> rows -> sorted rows ---------------
namespace {
// Step P: each record goes to its row's range of the (unsorted) row-grouped
// array: `cursor` holds the rows' shard-local start offsets (written by the
// scan) and hands out the slots, so a record costs one atomic and one 16-byte
// store {col, -, val}.
__global__ void __launch_bounds__(256) scatter_records_kernel(const uint4* __restrict__ rec,
                                                              const unsigned long long* n_dev,
                                                              unsigned long long cap,
                                                              unsigned* cursor, uint4* grp,
                                                              uint64_t grp_cap) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long n = *n_dev < cap ? *n_dev : cap;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint4 r = __ldcs(&rec[i]);
    if (r.x == k2::kInvalidRow) continue;
    const uint64_t pos = atomicAdd(&cursor[r.x], 1u);
    if (pos >= grp_cap) continue;  // only after dropped records; the host redoes the build
    grp[pos] = make_uint4(r.y, 0u, r.z, r.w);
  }
}

// Step Q: per-row LSD radix sort by column, one warp per row, out of place
// (grouped arrays -> final arrays). The digits that are equal in all keys of a
// row are skipped; each 8-bit pass is histogram, scan, and a stable scatter
// (32 keys at a time: match_any ranks equal digits within the chunk).
constexpr int kRsWarps = 4;
constexpr int kRsCap = 1024;  // longer rows go to sort_rows_block
constexpr int kRsIdxBits = 10;
// kPacked (columns below 2^22, e.g. C0 and C2): a key and its entry index
// travel as one 32-bit word (column << 10 | index): one shared-memory array
// pair instead of two, 9 instead of 13 KB per warp.
template <bool kPacked>
struct RsWarp {
  uint32_t key[2][kRsCap];
  uint16_t idx[kPacked ? 1 : 2][kPacked ? 1 : kRsCap];
  uint32_t hist[256];
};

template <bool kPacked>
__global__ void __launch_bounds__(kRsWarps * 32) sort_rows_radix(
    uint64_t n_rows, const uint64_t* __restrict__ rs, const uint4* __restrict__ grp,
    uint32_t* __restrict__ col_out, double* __restrict__ val_out, uint64_t out_cap,
    uint64_t grp_cap, unsigned* long_rows, unsigned* n_long) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  RsWarp<kPacked>& w = reinterpret_cast<RsWarp<kPacked>*>(rs_smem)[wid];
  const unsigned full = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  constexpr int kS = kPacked ? kRsIdxBits : 0;  // the column starts at this bit of a key
  const uint64_t warps_total = (uint64_t)gridDim.x * kRsWarps;
  const uint64_t base = rs[0];  // the grouped arrays start at the chunk's first entry
  for (uint64_t r = (uint64_t)blockIdx.x * kRsWarps + wid; r < n_rows; r += warps_total) {
    const uint64_t b = rs[r] - base;
    const uint64_t n64 = rs[r + 1] - rs[r];
    if (n64 == 0) continue;
    if (rs[r + 1] > out_cap || b + n64 > grp_cap) continue;  // beyond the caller's arrays
    if (n64 > (uint64_t)kRsCap) {
      if (lane == 0) long_rows[atomicAdd(n_long, 1u)] = (unsigned)r;
      continue;
    }
    const int n = (int)n64;
    uint32_t kor = 0u, kand = ~0u;
    for (int i = lane; i < n; i += 32) {
      const uint32_t k = grp[b + i].x;
      w.key[0][i] = kPacked ? ((k << kRsIdxBits) | (uint32_t)i) : k;
      if (!kPacked) w.idx[0][i] = (uint16_t)i;
      kor |= k;
      kand &= k;
    }
    __syncwarp();
    bool sorted = true;
    for (int i = lane; i + 1 < n; i += 32)
      if (w.key[0][i] > w.key[0][i + 1]) sorted = false;
    int cur = 0;
    if (!__all_sync(full, sorted)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        kor |= __shfl_xor_sync(full, kor, o);
        kand &= __shfl_xor_sync(full, kand, o);
      }
      const uint32_t diff = kor ^ kand;
      for (int shift = 0; shift < 32 - kS; shift += 8) {
        if (((diff >> shift) & 0xffu) == 0u) continue;
        for (int j = lane; j < 256; j += 32) w.hist[j] = 0u;
        __syncwarp();
        for (int i = lane; i < n; i += 32)
          atomicAdd(&w.hist[(w.key[cur][i] >> (shift + kS)) & 0xffu], 1u);
        __syncwarp();
        {
          unsigned loc[8], sum = 0u;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            loc[j] = w.hist[lane * 8 + j];
            sum += loc[j];
          }
          unsigned incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(full, incl, o);
            if (lane >= o) incl += y;
          }
          unsigned run = incl - sum;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            w.hist[lane * 8 + j] = run;
            run += loc[j];
          }
        }
        __syncwarp();
        for (int c = 0; c < n; c += 32) {
          const int i = c + lane;
          const bool valid = i < n;
          const uint32_t k = valid ? w.key[cur][i] : 0u;
          uint16_t id = 0;
          if (!kPacked) id = valid ? w.idx[cur][i] : (uint16_t)0;
          const unsigned d = valid ? ((k >> (shift + kS)) & 0xffu) : (256u + (unsigned)lane);
          const unsigned peers = __match_any_sync(full, d);
          const unsigned rank = __popc(peers & lt);
          if (valid) {
            const unsigned pos = w.hist[d] + rank;
            w.key[cur ^ 1][pos] = k;
            if (!kPacked) w.idx[cur ^ 1][pos] = id;
          }
          __syncwarp();
          if (valid && rank == 0u) w.hist[d] += __popc(peers);
          __syncwarp();
        }
        cur ^= 1;
      }
    }
    for (int i = lane; i < n; i += 32) {
      const uint32_t k = w.key[cur][i];
      const unsigned src = kPacked ? (k & ((1u << kRsIdxBits) - 1u)) : (unsigned)w.idx[cur][i];
      const uint4 e = grp[b + src];
      col_out[base + b + i] = kPacked ? (k >> kRsIdxBits) : k;
      val_out[base + b + i] = __hiloint2double((int)e.w, (int)e.z);
    }
    __syncwarp();
  }
}

// Rows longer than kRsCap: one block per row, bitonic sort of (column, index)
// keys in shared memory up to kLongCap entries; beyond that a shell sort in
// global memory by one thread (kept for completeness).
constexpr int kLongCap = 16384;
constexpr int kLongThreads = 512;
__global__ void __launch_bounds__(kLongThreads) sort_rows_block(
    const unsigned* __restrict__ long_rows, const unsigned* __restrict__ n_long,
    const uint64_t* __restrict__ rs, const uint4* __restrict__ grp,
    uint32_t* __restrict__ col_out_g, double* __restrict__ val_out_g, uint64_t out_cap,
    uint64_t grp_cap) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(rs_smem);
  const unsigned nl = *n_long;
  const uint64_t base = rs[0];
  uint32_t* col_out = col_out_g + base;
  double* val_out = val_out_g + base;
  for (unsigned q = blockIdx.x; q < nl; q += gridDim.x) {
    const uint64_t r = long_rows[q];
    const uint64_t b = rs[r] - base;
    const uint64_t n = rs[r + 1] - rs[r];
    if (rs[r + 1] > out_cap || b + n > grp_cap) continue;
    if (n <= (uint64_t)kLongCap) {
      int n2 = 1;
      while ((uint64_t)n2 < n) n2 <<= 1;
      for (int i = threadIdx.x; i < n2; i += kLongThreads)
        key[i] = (uint64_t)i < n ? (((unsigned long long)grp[b + i].x << 32) | (unsigned)i) : ~0ull;
      __syncthreads();
      for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = threadIdx.x; i < n2; i += kLongThreads) {
            const int p = i ^ j;
            if (p > i) {
              const unsigned long long x = key[i], y = key[p];
              if ((x > y) == ((i & k) == 0)) {
                key[i] = y;
                key[p] = x;
              }
            }
          }
          __syncthreads();
        }
      for (uint64_t i = threadIdx.x; i < n; i += kLongThreads) {
        const unsigned long long kk = key[i];
        const uint4 e = grp[b + (kk & 0xffffffffu)];
        col_out[b + i] = (uint32_t)(kk >> 32);
        val_out[b + i] = __hiloint2double((int)e.w, (int)e.z);
      }
      __syncthreads();
    } else {
      for (uint64_t i = threadIdx.x; i < n; i += kLongThreads) {
        const uint4 e = grp[b + i];
        col_out[b + i] = e.x;
        val_out[b + i] = __hiloint2double((int)e.w, (int)e.z);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        long long gap = 1;
        while (gap < (long long)n / 3) gap = 3 * gap + 1;
        for (; gap > 0; gap /= 3)
          for (long long i = gap; i < (long long)n; ++i) {
            const uint32_t c = col_out[b + i];
            const double v = val_out[b + i];
            long long j = i;
            while (j >= gap && col_out[b + j - gap] > c) {
              col_out[b + j] = col_out[b + j - gap];
              val_out[b + j] = val_out[b + j - gap];
              j -= gap;
            }
            col_out[b + j] = c;
            val_out[b + j] = v;
          }
      }
      __syncthreads();
    }
  }
}
}  // namespace

cudaError_t csr_scatter_records(const void* rec, const unsigned long long* n_dev,
                                unsigned long long cap, unsigned* cursor, void* grp,
                                uint64_t grp_cap, cudaStream_t st) {
  if (cap == 0) return cudaSuccess;
#ifndef CTSM_SCATTER_BLOCKS
#define CTSM_SCATTER_BLOCKS 32
#endif
  scatter_records_kernel<<<148 * CTSM_SCATTER_BLOCKS, 256, 0, st>>>((const uint4*)rec, n_dev, cap, cursor,
                                                   (uint4*)grp, grp_cap);
  count_launch();
  return cudaGetLastError();
}

cudaError_t csr_sort_rows_radix(uint64_t n_rows, const uint64_t* row_start, const void* grp,
                                uint32_t* col_out, double* val_out, uint64_t out_cap,
                                uint64_t grp_cap, unsigned* long_rows, unsigned* n_long,
                                cudaStream_t st, uint64_t n_cols) {
  const bool packed = n_cols != 0 && n_cols <= (1ull << (32 - kRsIdxBits));
  {  // per device (function attributes are not shared between devices): set on every call
    cudaError_t e = packed
                        ? cudaFuncSetAttribute(sort_rows_radix<true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kRsWarps * sizeof(RsWarp<true>)))
                        : cudaFuncSetAttribute(sort_rows_radix<false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kRsWarps * sizeof(RsWarp<false>)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sort_rows_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kLongCap * sizeof(unsigned long long)));
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaMemsetAsync(n_long, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  if (n_rows == 0) return cudaSuccess;
  const uint64_t blocks = (n_rows + kRsWarps - 1) / kRsWarps;
#ifndef CTSM_SORT_BLOCKS
#define CTSM_SORT_BLOCKS 0  // blocks per SM in the grid; 0: what the shared memory allows
#endif
  // 37 KB (packed) / 53 KB of shared memory per block
  const uint64_t per_sm = CTSM_SORT_BLOCKS ? CTSM_SORT_BLOCKS : (packed ? 6 : 4);
  const unsigned grid = (unsigned)(blocks < 148ull * per_sm ? blocks : 148ull * per_sm);
  if (packed)
    sort_rows_radix<true><<<grid, kRsWarps * 32, kRsWarps * sizeof(RsWarp<true>), st>>>(
        n_rows, row_start, (const uint4*)grp, col_out, val_out, out_cap, grp_cap, long_rows,
        n_long);
  else
    sort_rows_radix<false><<<grid, kRsWarps * 32, kRsWarps * sizeof(RsWarp<false>), st>>>(
        n_rows, row_start, (const uint4*)grp, col_out, val_out, out_cap, grp_cap, long_rows,
        n_long);
  sort_rows_block<<<148, kLongThreads, kLongCap * sizeof(unsigned long long), st>>>(
      long_rows, n_long, row_start, (const uint4*)grp, col_out, val_out, out_cap, grp_cap);
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
// ---- K4 as a gather: CSC transpose of a device CSR --------------------------
// The scatter above is bound by the L2's 64-bit reductions (4.6 G of them for
// C2: 49 % of the HBM time of the matrix). With the transpose kept beside the
// CSR (C2: 2 x 55 GB of 180) A^T y reads each entry once and gathers y.
// csc_count / csc_scatter build it: column counts, their scan (the caller),
// then every CSR entry takes a slot of its column from a cursor. The order of
// a column's entries depends on the schedule; the applier sums the same
// rounded fixed-point integers as the scatter, so its result does not, and it
// is bit-identical to spmvt_fixed_kernel's.
__global__ void csc_count_kernel(uint64_t nnz, const uint32_t* __restrict__ col,
                                 unsigned* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += stride)
    atomicAdd(&counts[__ldcs(&col[j])], 1u);
}

__global__ void csc_scatter_kernel(uint64_t n_rows, const uint64_t* __restrict__ rs,
                                   const uint32_t* __restrict__ col,
                                   const double* __restrict__ val,
                                   const uint64_t* __restrict__ col_start, unsigned* cursor,
                                   uint32_t* __restrict__ row_out, double* __restrict__ val_out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps_total) {
    for (uint64_t j = rs[r] + lane; j < rs[r + 1]; j += 32) {
      const uint32_t c = __ldcs(&col[j]);
      const uint64_t pos = col_start[c] + atomicAdd(&cursor[c], 1u);
      row_out[pos] = (uint32_t)r;
      val_out[pos] = __ldcs(&val[j]);
    }
  }
}

// warp per column: acc = sum_j round(val_j * (y[row_j] * scale)), the
// scatter's integers (spmvt_fixed_kernel) in another order
__global__ void spmvt_csc_fixed_kernel(uint64_t n_cols, const uint64_t* __restrict__ cs,
                                       const uint32_t* __restrict__ row,
                                       const double* __restrict__ val,
                                       const double* __restrict__ y,
                                       unsigned long long* __restrict__ acc, double scale) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t c = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n_cols;
       c += warps_total) {
    long long a = 0;
    for (uint64_t j = cs[c] + lane; j < cs[c + 1]; j += 32)
      a += __double2ll_rn(__ldcs(&val[j]) * (__ldg(&y[__ldcs(&row[j])]) * scale));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) acc[c] = (unsigned long long)a;
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

cudaError_t csc_count(uint64_t nnz, const uint32_t* col, unsigned* counts, cudaStream_t st) {
  const uint64_t blocks = (nnz + 255) / 256;
  csc_count_kernel<<<(unsigned)(blocks < 148ull * 32 ? (blocks ? blocks : 1) : 148ull * 32), 256, 0,
                     st>>>(nnz, col, counts);
  count_launch();
  return cudaGetLastError();
}

cudaError_t csc_scatter(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                        const double* val, const uint64_t* col_start, unsigned* cursor,
                        uint32_t* row_out, double* val_out, cudaStream_t st) {
  csc_scatter_kernel<<<row_grid(n_rows, 8), 256, 0, st>>>(n_rows, row_start, col, val, col_start,
                                                          cursor, row_out, val_out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t spmvt_csc_fixed(uint64_t n_cols, const uint64_t* col_start, const uint32_t* row,
                            const double* val, const double* y, unsigned long long* acc,
                            double scale, cudaStream_t st) {
  spmvt_csc_fixed_kernel<<<row_grid(n_cols, 8), 256, 0, st>>>(n_cols, col_start, row, val, y, acc,
                                                              scale);
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
