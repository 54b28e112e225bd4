// mf.cu -- K5/K6 matrix-free projectors (forward_project_matrix_free,
// projector.cpp:235-260, and its adjoint) plus the SIRT elementwise kernels.
//
// Weights are regenerated on the fly in FP64 (fast2d.cuh / fast3d.cuh) and
// never stored. Forward (A x) is voxel-driven: each thread owns one
// (pixel/voxel column, angle) work item and scatters w * x into a fixed-point
// int64 sinogram accumulator (integer adds commute, so the result is
// bit-reproducible for any schedule or GPU count). Backward (A^T y) is a
// voxel-driven gather: each thread owns one pixel/voxel, loops over the angle
// shard and accumulates in FP64 registers -- no atomics, deterministic.
#include "fast2d.cuh"
#include "fast3dw.cuh"
#include "kernels.h"

namespace ctsmb {

int mf3d_max_pieces() { return fast::kMaxPieces; }

namespace {

__global__ void angle_cs_kernel(DevGeom g, int angle_begin, int angle_step, int n, AngleCS* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = angle_begin + k * angle_step;
  const double phi = g.angle_start + (g.angle_end - g.angle_start) * i / g.n_angles;
  double S, C;
  sincos(phi, &S, &C);
  out[k] = AngleCS{C, S};
}

template <typename T>
__device__ __forceinline__ double ld(const T* p) {
  return (double)__ldg(p);
}

// Voxel-ray update counter: nonzero weights applied in a forward call (the
// metric's unit, measured live). One atomic per warp.
__device__ __forceinline__ void count_updates(unsigned long long* n_upd, unsigned cnt) {
  if (!n_upd) return;
  const unsigned tot = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(n_upd, (unsigned long long)tot);
}

// 2D pixel tile per block: 16 x 8 pixels, 128 threads.
// G consecutive values (16-byte aligned) with 128-bit read-only loads.
template <typename T, int G>
__device__ __forceinline__ void load_vec(const T* p, T (&v)[G]) {
#ifndef CTSM_NO_LDG256
  // 32-byte aligned vectors: sm_100 256-bit loads (LDG.E.ENL2.256), one per
  // 8 floats / 4 doubles
  if constexpr (G % (32 / sizeof(T)) == 0) {
#pragma unroll
    for (int c = 0; c < G / (32 / (int)sizeof(T)); ++c) {
      if constexpr (sizeof(T) == 4) {
        float* o = reinterpret_cast<float*>(v) + 8 * c;
        asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]),
              "=f"(o[7])
            : "l"(reinterpret_cast<const float*>(p) + 8 * c));
      } else {
        double* o = reinterpret_cast<double*>(v) + 4 * c;
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
            : "l"(reinterpret_cast<const double*>(p) + 4 * c));
      }
    }
    return;
  }
#endif
  constexpr int per = 16 / sizeof(T);
#pragma unroll
  for (int c = 0; c < G / per; ++c) {
    if constexpr (sizeof(T) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p) + c);
      v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
    } else {
      const double2 q = __ldg(reinterpret_cast<const double2*>(p) + c);
      v[2 * c] = q.x; v[2 * c + 1] = q.y;
    }
  }
}
// z-mirror reuse in the 3D symmetric kernels (CTSM_NO_ZMIRROR: off)
__device__ __forceinline__ bool zmirror_on() {
#ifdef CTSM_NO_ZMIRROR
  return false;
#else
  return true;
#endif
}

constexpr int kTx = 16, kTy = 8;

// Forward 2D: block = 16x8 pixel tile x a chunk of kFwdAngles angles; each
// thread loops over its chunk's angles (x and the per-angle cos/sin are loaded
// once per thread / prefetched, amortising the load latency).
constexpr int kFwdAngles = 4;

template <typename T>
__global__ void __launch_bounds__(128, 8) fwd2d_kernel(DevGeom g, const AngleCS* __restrict__ cs,
                                                    int angle_begin, int angle_step, int n_sel,
                                                    const T* __restrict__ x,
                                                    unsigned long long* __restrict__ yacc,
                                                    double scale, unsigned long long* n_upd,
                                                    int* status) {
  const int tiles_x = (g.n_x + kTx - 1) / kTx;
  const int ix = (blockIdx.x % tiles_x) * kTx + (threadIdx.x % kTx);
  const int iy = (blockIdx.x / tiles_x) * kTy + (threadIdx.x / kTx);
  unsigned cnt = 0;
  if (ix < g.n_x && iy < g.n_y) {
    const double xs = ld(&x[(long long)iy * g.n_x + ix]) * scale;
    const int k0 = blockIdx.y * kFwdAngles;
    const int k1 = min(k0 + kFwdAngles, n_sel);
    AngleCS a = cs[k0];
    for (int k = k0; k < k1; ++k) {
      const AngleCS an = cs[min(k + 1, n_sel - 1)];  // prefetch
      const int ip = angle_begin + k * angle_step;
      unsigned long long* yrow = yacc + (long long)ip * g.rows_per_angle + g.n_det_y / 2;
      fast::pixel_weights(g, a.C, a.S, ix, iy, status, [&](int m, double w) {
        ++cnt;
        if (xs != 0.0) atomicAdd(&yrow[m], (unsigned long long)__double2ll_rn(w * xs));
      });
      a = an;
    }
  }
  count_updates(n_upd, cnt);
}

// Backward 2D: block = pixel tile x angle chunk. With n_chunks > 1 each chunk
// writes its partial sum to part[chunk][pixel] and bwd_reduce adds the chunks
// in fixed order (deterministic); with one chunk x is written directly.
template <typename T>
__global__ void __launch_bounds__(128, 8) bwd2d_kernel(DevGeom g, const AngleCS* __restrict__ cs,
                                                    int angle_begin, int angle_step, int n_sel,
                                                    int chunk, const T* __restrict__ y,
                                                    T* __restrict__ x, double* __restrict__ part,
                                                    int* status) {
  const int tiles_x = (g.n_x + kTx - 1) / kTx;
  const int ix = (blockIdx.x % tiles_x) * kTx + (threadIdx.x % kTx);
  const int iy = (blockIdx.x / tiles_x) * kTy + (threadIdx.x / kTx);
  if (ix >= g.n_x || iy >= g.n_y) return;
  const int k0 = blockIdx.y * chunk;
  const int k1 = min(k0 + chunk, n_sel);
  double acc = 0.0;
  for (int k = k0; k < k1; ++k) {
    const int ip = angle_begin + k * angle_step;
    const AngleCS a = cs[k];
    const T* yrow = y + (long long)ip * g.rows_per_angle + g.n_det_y / 2;
    fast::pixel_weights(g, a.C, a.S, ix, iy, status,
                        [&](int m, double w) { acc += w * ld(&yrow[m]); });
  }
  const long long pix = (long long)iy * g.n_x + ix;
  if (part)
    part[(long long)blockIdx.y * g.n_x * g.n_y + pix] = acc;
  else
    x[pix] = (T)acc;
}

template <typename T>
__global__ void bwd_reduce_kernel(long long n, int n_chunks, const double* __restrict__ part,
                                  T* __restrict__ x) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < n_chunks; ++c) acc += part[(long long)c * n + i];
    x[i] = (T)acc;
  }
}

// 3D (K5/K6): one warp per voxel column; the warp loops over the angle
// shard, plans the column once per angle (sweep + atom coefficients in shared
// memory, fast3dw.cuh) and its lanes evaluate contiguous z-chunks of voxels.
// Forward scatters w*x into the fixed-point sinogram accumulator; backward
// accumulates w*y per voxel in shared memory in a fixed order (deterministic).
// Per-group piecewise-cubic tables of a planned (column, angle)
// (fast3dw.cuh), opt-in with CTSM_TABLE3D: measured slower than the per-piece
// atom evaluation with its linear / zero short cuts at C3 (fwd 402 vs 332 ms,
// bwd 344 vs 290 ms per projection, r1o), so the default keeps the atoms.
#ifdef CTSM_TABLE3D
#define CTSM_TABLE_DECL(n) __shared__ fast::GroupTable stab[n]
#define CTSM_TABLE_PTR (&stab[warp])
#else
#define CTSM_TABLE_PTR nullptr
#define CTSM_TABLE_DECL(n)
#endif
__device__ __forceinline__ const fast::GroupTable* table3d(const fast::ColumnHead& H,
                                                           const fast::PieceCoef* P,
                                                           fast::GroupTable* T, int lane) {
#ifdef CTSM_TABLE3D
  fast::build_group_tables(H, P, *T, lane);
  return T;
#else
  return nullptr;
#endif
}

// flattened (voxel, row edge) walk of the symmetric kernels (fast3dw.cuh
// chunk_weights_flat); 0 = the lockstep per-voxel walk
#ifndef CTSM_FLAT
#define CTSM_FLAT 1  // C3 fwd 90 -> 89, bwd 104 -> 102 ms per projection
#endif
// flattened walk of the back-projection: row vectors loaded before the weight
// is evaluated
#ifndef CTSM_BWD3_EARLY_LOAD
#define CTSM_BWD3_EARLY_LOAD 1  // C3 bwd 97 -> 92 ms per projection
#endif
// flattened walk of the forward: row runs flushed at the end of their cell group
// (An fp32 forward without row runs -- every weight reduced to memory
// directly, no pending sums, no flush branch, 16 registers fewer -- issues 1.3x
// the vector reductions and is 26 % slower, 99 vs 78 ms per projection: the
// forward runs close to the SM's global-reduction throughput.)
#ifndef CTSM_FWD3_GEND
#define CTSM_FWD3_GEND 1  // C3 fwd 85 -> 83 ms per projection
#endif
// warp-batched cubic faces (fast3dw.cuh CubicBatch); CTSM_NO_BATCH: in place
#ifndef CTSM_NO_BATCH
#define CTSM_BATCH_DECL(n) __shared__ fast::CubicBatch sbat[n]
#define CTSM_BATCH_PTR (&sbat[warp])
#else
#define CTSM_BATCH_DECL(n)
#define CTSM_BATCH_PTR nullptr
#endif

#ifndef CTSM_KW3
#define CTSM_KW3 4
#endif
constexpr int kWarps3 = CTSM_KW3;
constexpr int kZcMax = 16;  // voxels per lane per z-block (z-block = 512 voxels)

// ---- plan pass of the 3D kernels --------------------------------
// Planning a (column, base angle) -- the xy sweep, the pieces' G-independent
// coefficients, the group short cuts -- does not depend on z. Inside the
// projection kernels it was done by the whole warp (every lane computing the
// same sweep), 26 % of a C3 projection. plan3d_fast_kernel plans all (column,
// base angle) pairs of a launch with ONE THREAD each (full lanes instead of 32
// redundant copies) into global memory; the projection kernels then load the
// plan (coalesced, ~1-3 KB) into shared memory instead of computing it.
struct FastPlan {
  fast::ColumnHead H;
  fast::PieceCoef P[fast::kMaxPieces];
};
static_assert(sizeof(fast::ColumnHead) % 32 == 0 && sizeof(fast::PieceCoef) % 32 == 0,
              "plans are stored as 32-byte vectors and loaded as 16-byte vectors");

__global__ void __launch_bounds__(128) plan3d_fast_kernel(DevGeom g, const AngleCS* __restrict__ cs,
                                                          int n_base, FastPlan* __restrict__ plans,
                                                          int* status) {
  const long long nxy = (long long)g.n_x * g.n_y;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nxy * n_base) return;
  const int kk = (int)(t / nxy);
  const long long col = t - (long long)kk * nxy;
  FastPlan* out = plans + t;
  // the head is assembled in thread-local memory (small fields written all
  // over it) and leaves as 32-byte stores; the pieces are stored from
  // registers by plan_column
  fast::ColumnHead Hl;
  fast::plan_column<true>(g, cs[kk].C, cs[kk].S, (int)(col % g.n_x), (int)(col / g.n_x), status,
                          Hl, out->P, 0);
  const double* src = reinterpret_cast<const double*>(&Hl);
  double* dst = reinterpret_cast<double*>(&out->H);
#pragma unroll 1
  for (int i = 0; i < (int)(sizeof(fast::ColumnHead) / 8); i += 4)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + i), "d"(src[i]),
                 "d"(src[i + 1]), "d"(src[i + 2]), "d"(src[i + 3])
                 : "memory");
}

// Plans are read once per z-block: streaming (evict-first) loads keep them
// from displacing the forward's reduction rows in L2 (CTSM_PLAN_STREAM)
#ifndef CTSM_PLAN_STREAM
#define CTSM_PLAN_STREAM 1  // C3 bwd 74.2 -> 73.7 ms; an evict-last hint on the forward's reductions: no gain
#endif
#if CTSM_PLAN_STREAM
#define CTSM_PLAN_LD(p) __ldcs(p)
#else
#define CTSM_PLAN_LD(p) __ldg(p)
#endif
// Loads the plan of (column, slot kk) into the warp's shared head / pieces.
// Returns false for a column without work (failed sweep or no cell group).
__device__ __forceinline__ bool load_plan(const FastPlan* __restrict__ plans, long long idx,
                                          fast::ColumnHead& H, fast::PieceCoef* P, int lane) {
  const FastPlan* src = plans + idx;
  {
    const double2* s2 = reinterpret_cast<const double2*>(&src->H);
    double2* d2 = reinterpret_cast<double2*>(&H);
    for (int i = lane; i < (int)(sizeof(fast::ColumnHead) / 16); i += 32) d2[i] = CTSM_PLAN_LD(&s2[i]);
  }
  __syncwarp();
  const int np = H.np;
  {
    const double2* s2 = reinterpret_cast<const double2*>(src->P);
    double2* d2 = reinterpret_cast<double2*>(P);
    for (int i = lane; i < np * (int)(sizeof(fast::PieceCoef) / 16); i += 32) d2[i] = CTSM_PLAN_LD(&s2[i]);
  }
  return H.ng > 0;
}

// Prefetch of the plan a warp loads next (CTSM_PLAN_PREFETCH: 1 = into L2,
// 2 = into L1): the plans stream from DRAM, each read once per z-block, and
// load_plan is a dependent load the warp waits for (~5 % of the samples).
#ifndef CTSM_PLAN_PREFETCH
#define CTSM_PLAN_PREFETCH 1  // C3 fwd 90 -> 88 ms per projection (L1: the same)
#endif
__device__ __forceinline__ void prefetch_plan(const FastPlan* __restrict__ plans, long long idx,
                                              int lane) {
#if CTSM_PLAN_PREFETCH
  // head (~0.7 KB) + the first pieces: 32 lanes x 128-byte lines = 4 KB covers a whole plan
  const char* p = reinterpret_cast<const char*>(plans + idx) + lane * 128;
  if (lane * 128 < (int)sizeof(FastPlan)) {
#if CTSM_PLAN_PREFETCH == 2
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
  }
#endif
}

static cudaError_t plan_pass(const DevGeom& g, const AngleCS* cs, int nk, void* plans, int* status,
                             cudaStream_t st) {
  if (!plans) return cudaSuccess;
  const long long n = (long long)g.n_x * g.n_y * nk;
  plan3d_fast_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(g, cs, nk, (FastPlan*)plans,
                                                                  status);
  count_launch();
  return cudaGetLastError();
}

template <typename T, bool kFwd>
__global__ void __launch_bounds__(kWarps3 * 32, 4) proj3d_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, int angle_begin, int angle_step, int n_sel,
    const T* __restrict__ in, T* __restrict__ xout, unsigned long long* __restrict__ yacc,
    double scale, unsigned long long* n_upd, int accumulate, int* status,
    const FastPlan* __restrict__ plans = nullptr) {
  __shared__ __align__(32) fast::ColumnHead sh[kWarps3];
  __shared__ __align__(32) fast::PieceCoef sp[kWarps3][fast::kMaxPieces];
  __shared__ double sacc[kWarps3][kZcMax][32];
  CTSM_TABLE_DECL(kWarps3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nxy = (long long)g.n_x * g.n_y;
  const long long col = (long long)blockIdx.x * kWarps3 + warp;
  if (col >= nxy) return;  // whole warp
  const int ix = (int)(col % g.n_x), iy = (int)(col / g.n_x);
  const long long plane = nxy;
  const int rpa = g.rows_per_angle;
  const int hy = g.n_det_y / 2, hz = g.n_det_z / 2;
  unsigned cnt = 0;
  for (int zb0 = 0; zb0 < g.n_z; zb0 += 32 * kZcMax) {
    const int nzb = min(32 * kZcMax, g.n_z - zb0);
    const int zc = (nzb + 31) / 32;
    const int z0 = zb0 + lane * zc, z1 = min(z0 + zc, zb0 + nzb);
    if (!kFwd)
      for (int i = 0; i < zc; ++i) sacc[warp][i][lane] = 0.0;
    for (int k = 0; k < n_sel; ++k) {
      const int ip = angle_begin + k * angle_step;
      const AngleCS a = cs[k];
      __syncwarp();
      const bool ok = plans ? load_plan(plans, (long long)k * nxy + col, sh[warp], sp[warp], lane)
                            : fast::plan_column(g, a.C, a.S, ix, iy, status, sh[warp], sp[warp],
                                                lane);
      __syncwarp();
      if (!ok) continue;
      const fast::ColumnHead& H = sh[warp];
      const fast::PieceCoef* P = sp[warp];
      const fast::GroupTable* TB = table3d(H, P, CTSM_TABLE_PTR, lane);
      if (kFwd) {
        unsigned long long* yb = yacc + (long long)ip * rpa;
        // consecutive emits of a lane often hit the same (row, cell) as z
        // advances: merge them (integer sums of the rounded contributions, so
        // the result equals the unmerged atomics) before one atomic.
        long long pr = -1, pv = 0;
        fast::chunk_weights(g, H, P, z0, z1, [&](int iz, int my, int mz, double w) {
          ++cnt;
          const double xs = ld(&in[iz * plane + col]) * scale;
          const long long r = (long long)(mz + hz) * g.n_det_y + (my + hy);
          const long long v = __double2ll_rn(w * xs);
          if (r == pr) {
            pv += v;
          } else {
            if (pr >= 0 && pv != 0) atomicAdd(&yb[pr], (unsigned long long)pv);
            pr = r;
            pv = v;
          }
        }, TB);
        if (pr >= 0 && pv != 0) atomicAdd(&yb[pr], (unsigned long long)pv);
      } else {
        const T* yb = in + (long long)ip * rpa;
        fast::chunk_weights(g, H, P, z0, z1, [&](int iz, int my, int mz, double w) {
          sacc[warp][iz - z0][lane] += w * ld(&yb[(long long)(mz + hz) * g.n_det_y + (my + hy)]);
        }, TB);
      }
    }
    if (!kFwd)
      for (int iz = z0; iz < z1; ++iz) {
        double v = sacc[warp][iz - z0][lane];
        if (accumulate) v += (double)xout[iz * plane + col];
        xout[iz * plane + col] = (T)v;
      }
  }
  if (kFwd) count_updates(n_upd, cnt);
}

// ---- quarter-turn symmetric kernels --------------------------------------
// For a square grid (n_x == n_y, a == b) and angles uniform over a full turn
// with n_angles % 4 == 0, rotating the scanner by a quarter turn maps the
// setup onto itself: pixel (ix, iy) at angle i + n/4 sees exactly the weights
// of pixel R^-1(ix, iy) at angle i, with R(ix, iy) = (n-1-iy, ix). Each weight
// evaluation therefore serves four (pixel, angle) pairs; the kernels below
// evaluate weights at the "base" angles i < n/4 only and apply every weight to
// its four images. The updates applied are the same as in the general
// kernels; only repeated weight evaluations are avoided.
__device__ __forceinline__ void rot_pixel(int n, int ix, int iy, int k, int& ox, int& oy) {
  int x = ix, y = iy;
  for (int r = 0; r < k; ++r) {
    const int t = x;
    x = n - 1 - y;
    y = t;
  }
  ox = x;
  oy = y;
}

// Forward: thread = (pixel p, chunk of base angles); scatters w * x[R^k p] to
// the rows of angle i + k n/4.
template <typename T>
__global__ void __launch_bounds__(128) fwd2d_sym_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    const T* __restrict__ x, unsigned long long* __restrict__ yacc, double scale,
    unsigned long long* n_upd, int* status) {
  const int tiles_x = (g.n_x + kTx - 1) / kTx;
  const int ix = (blockIdx.x % tiles_x) * kTx + (threadIdx.x % kTx);
  const int iy = (blockIdx.x / tiles_x) * kTy + (threadIdx.x / kTx);
  unsigned cnt = 0;
  if (ix < g.n_x && iy < g.n_y) {
    const int n = g.n_x;
    double xs[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int rx, ry;
      rot_pixel(n, ix, iy, k, rx, ry);
      xs[k] = ld(&x[(long long)ry * n + rx]) * scale;
    }
    const int q = g.n_angles / 4;
    const int k0 = blockIdx.y * kFwdAngles;
    const int k1 = min(k0 + kFwdAngles, n_base);
    for (int kk = k0; kk < k1; ++kk) {
      const AngleCS a = cs[kk];
      const int i = base[kk];
      unsigned long long* rows[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        rows[k] = yacc + (long long)((i + k * q) % g.n_angles) * g.rows_per_angle + g.n_det_y / 2;
      fast::pixel_weights(g, a.C, a.S, ix, iy, status, [&](int m, double w) {
        cnt += 4;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (xs[k] != 0.0) atomicAdd(&rows[k][m], (unsigned long long)__double2ll_rn(w * xs[k]));
      });
    }
  }
  count_updates(n_upd, cnt);
}

// Backward: thread = quarter-turn orbit {p, Rp, R^2p, R^3p} of a pixel of the
// first quadrant x a chunk of base angles; every weight set of orbit member j
// at base angle i is gathered against the rows of angles i + k n/4 into the
// accumulator of member j + k.
template <typename T>
__global__ void __launch_bounds__(128) bwd2d_sym_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    int chunk, const T* __restrict__ y, T* __restrict__ x, double* __restrict__ part,
    int* status) {
  const int h = g.n_x / 2;
  const int tiles_x = (h + kTx - 1) / kTx;
  const int ix = (blockIdx.x % tiles_x) * kTx + (threadIdx.x % kTx);
  const int iy = (blockIdx.x / tiles_x) * kTy + (threadIdx.x / kTx);
  if (ix >= h || iy >= h) return;
  const int n = g.n_x, q = g.n_angles / 4;
  int px[4], py[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) rot_pixel(n, ix, iy, j, px[j], py[j]);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int k0 = blockIdx.y * chunk;
  const int k1 = min(k0 + chunk, n_base);
  for (int kk = k0; kk < k1; ++kk) {
    const AngleCS a = cs[kk];
    const int i = base[kk];
    const T* rows[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      rows[k] = y + (long long)((i + k * q) % g.n_angles) * g.rows_per_angle + g.n_det_y / 2;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      fast::pixel_weights(g, a.C, a.S, px[j], py[j], status, [&](int m, double w) {
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[(j + k) & 3] += w * ld(&rows[k][m]);
      });
    }
  }
  const long long npix = (long long)n * n;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long long pix = (long long)py[j] * n + px[j];
    if (part)
      part[(long long)blockIdx.y * npix + pix] = acc[j];
    else
      x[pix] = (T)acc[j];
  }
}

// ---- dihedral (8-fold) symmetric 2D kernels --------------------------------
// With additionally angle_start == 0 and n_angles % 8 == 0, the reflection M
// (y -> -y) maps the scan onto itself too: angle i -> n - i, pixel
// (ix, iy) -> (ix, n-1-iy), detector cell m -> -1-m. The dihedral group D4 =
// {R^k M^f} has 8 elements e = k + 4 f acting on pixels (apply M if f, then R
// k times), angles (i -> (f ? -i : i) + k n/4) and cells (m -> f ? -1-m : m),
// with w(e p, e i, e m) = w(p, i, m). Weights are evaluated at the base angles
// 0 <= i <= n/8 only; the two self-symmetric base angles 0 and n/8 use the 4
// rotations (their reflections coincide with rotations).
__device__ __forceinline__ void d4_pixel(int n, int ix, int iy, int e, int& ox, int& oy) {
  int x = ix, y = (e >= 4) ? n - 1 - iy : iy;
  for (int r = 0; r < (e & 3); ++r) {
    const int t = x;
    x = n - 1 - y;
    y = t;
  }
  ox = x;
  oy = y;
}
__device__ __forceinline__ int d4_angle(int n_angles, int i, int e) {
  // 0 <= i <= n/8: no integer division
  const int b = (e >= 4 && i != 0) ? n_angles - i : i;
  const int r = b + (e & 3) * (n_angles >> 2);
  return r >= n_angles ? r - n_angles : r;
}
// composition g o h (apply h, then g)
__host__ __device__ constexpr int d4_compose(int g, int h) {
  return ((((g & 3) + ((g >= 4) ? (4 - (h & 3)) : (h & 3))) & 3) + 4 * (((g >> 2) ^ (h >> 2)) & 1));
}

// Forward: block = 16x8 pixel tile x a chunk of base angles. The tile's cell
// weights of one base angle are summed in a shared-memory window of detector
// cells (fixed point, exact integer adds) shared by the 8 images -- image e's
// cell is m or -1-m -- and flushed once per cell to global memory: ~10x fewer
// global atomics than one per weight. The window [clo, clo + W) is the
// projection of the tile's corners (same t expressions as the pixel sweeps),
// computed identically by every thread; a tile whose shadow exceeds the window
// falls back to direct global atomics. Shared memory has no native 64-bit
// atomic add, so the host caps the fixed-point scale so that every single
// contribution is below 2^47 (f64; 2^23 for f32) -- a resolution of 2^-47
// max|x| per weight, far below the f64 rounding of the sums -- and the window
// holds 32-bit limbs: the low 24 bits and the signed rest (f64), or one signed
// limb (f32). With <= 128 adds per cell (one per tile pixel) no limb
// overflows; the flush recombines them exactly into the 64-bit accumulator.
#ifndef CTSM_D8F_MINB
#define CTSM_D8F_MINB 8  // with 16-angle chunks: C1 fwd 1.003 -> 0.975 ms (f64), 0.747 -> 0.727 (f32)
#endif
#ifndef CTSM_D8B_MINB
#define CTSM_D8B_MINB 7
#endif
#ifndef CTSM_D8ANG
#define CTSM_D8ANG 16  // base angles per block (<= 32: one lane per angle computes the shadow)
#endif
constexpr int kD8Angles = CTSM_D8ANG;
#ifndef CTSM_D8WIN
#define CTSM_D8WIN 64
#endif
constexpr int kD8Win = CTSM_D8WIN;
// tile width of the dihedral forward per dtype (128-pixel tiles): 32 x 4 for
// fp64 (C1 fwd 1.078 -> 1.035 ms: shorter shadows per tile row, fewer window
// cells per flush), 16 x 8 for fp32 (0.815 vs 0.823 ms at 32 x 4)
#ifndef CTSM_D8TX_F64
#define CTSM_D8TX_F64 32
#endif
#ifndef CTSM_D8TX_F32
#define CTSM_D8TX_F32 16
#endif
template <typename T>
__host__ __device__ constexpr int d8_tx() { return sizeof(T) == 8 ? CTSM_D8TX_F64 : CTSM_D8TX_F32; }
// warp footprint width in the tile: full 32-pixel rows for fp64 (8 x 4 warps:
// 1.040 vs 1.052 ms), 8 x 4 pixel warps for fp32 (C1 fwd 0.817 -> 0.795 ms)
#ifndef CTSM_D8WX_F64
#define CTSM_D8WX_F64 32
#endif
#ifndef CTSM_D8WX_F32
#define CTSM_D8WX_F32 8
#endif
template <typename T>
__host__ __device__ constexpr int d8_wx() { return sizeof(T) == 8 ? CTSM_D8WX_F64 : CTSM_D8WX_F32; }
// w * xs rounded to the nearest integer (|.| < 2^47) by the 1.5 * 2^52 shift:
// the low 51 mantissa bits then hold the integer + 2^51 -- one DFMA instead of
// a 64-bit float->int conversion.
template <int L>
__device__ __forceinline__ void limb_add(unsigned* w, double wv, double xsv) {
  const double sh = fma(wv, xsv, 6755399441055744.0);  // 1.5 * 2^52
  const unsigned lo = (unsigned)__double2loint(sh);
  if (L == 1) {
    atomicAdd(w, lo);  // |value| < 2^23: the low word is its two's complement
  } else {
    const unsigned hi = (unsigned)__double2hiint(sh) & 0xFFFFFu;
    atomicAdd(w, lo & 0xFFFFFFu);
    atomicAdd(w + kD8Win, ((lo >> 24) | (hi << 8)) - (1u << 27));  // (value >> 24), signed
  }
}

template <typename T>
__global__ void __launch_bounds__(128, CTSM_D8F_MINB) fwd2d_d8_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    const T* __restrict__ x, unsigned long long* __restrict__ yacc, double scale,
    unsigned long long* n_upd, int* status) {
  constexpr int L = sizeof(T) == 8 ? 2 : 1;  // limbs per window cell
  __shared__ unsigned win[2][8][L][kD8Win];
  for (int j = threadIdx.x; j < 2 * 8 * L * kD8Win; j += blockDim.x) (&win[0][0][0][0])[j] = 0u;
  constexpr int kTx = d8_tx<T>(), kTy = 128 / kTx;
  const int tiles_x = (g.n_x + kTx - 1) / kTx;
  const int tx0 = (blockIdx.x % tiles_x) * kTx, ty0 = (blockIdx.x / tiles_x) * kTy;
  // warp footprint kWx x (32 / kWx) pixels inside the tile: fewer lanes on
  // one detector cell (same-address shared atomics) when the rays run along
  // a tile row
  constexpr int kWx = d8_wx<T>() < kTx ? d8_wx<T>() : kTx;
  const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int ix = tx0 + (wid % (kTx / kWx)) * kWx + ln % kWx;
  const int iy = ty0 + (wid / (kTx / kWx)) * (32 / kWx) + ln / kWx;
  const int n = g.n_x;
  const bool inside = ix < n && iy < g.n_y;
  double xs[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    int rx, ry;
    d4_pixel(n, ix, iy, e, rx, ry);
    xs[e] = inside ? ld(&x[(long long)ry * n + rx]) * scale : 0.0;
  }
  // tile corners (world coordinates)
  const double X0 = (tx0 - n / 2.0) * g.a, X1 = (min(tx0 + kTx, n) - n / 2.0) * g.a;
  const double Y0 = (ty0 - g.n_y / 2.0) * g.b, Y1 = (min(ty0 + kTy, g.n_y) - g.n_y / 2.0) * g.b;
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  const long long rpa = g.rows_per_angle;
  unsigned cnt = 0;
  __syncthreads();
  const int k0 = blockIdx.y * kD8Angles;
  const int k1 = min(k0 + kD8Angles, n_base);
  // shadow of the tile (t over the 4 corners; depths checked by the sweeps)
  // per angle of the chunk: uniform across the block, so lane j of every
  // warp computes angle k0 + j once and the loop reads it by shuffle
  static_assert(kD8Angles <= 32, "one lane per angle of the chunk");
  int sh_clo = 0, sh_w = 0;
  {
    const int kk = k0 + (int)(threadIdx.x & 31);
    if ((threadIdx.x & 31) < kD8Angles && kk < k1) {
      const AngleCS a = cs[kk];
      const double s = g.s;
      const double t0 = (Y0 * a.C - X0 * a.S) * fast::frcp(s - X0 * a.C - Y0 * a.S);
      const double t1 = (Y0 * a.C - X1 * a.S) * fast::frcp(s - X1 * a.C - Y0 * a.S);
      const double t2 = (Y1 * a.C - X1 * a.S) * fast::frcp(s - X1 * a.C - Y1 * a.S);
      const double t3 = (Y1 * a.C - X0 * a.S) * fast::frcp(s - X0 * a.C - Y1 * a.S);
      const double tmin = fmin(fmin(t0, t1), fmin(t2, t3));
      const double tmax = fmax(fmax(t0, t1), fmax(t2, t3));
      sh_clo = max((int)floor(tmin * g.u_scale) - 1, cell_lo);
      const int chi = min((int)ceil(tmax * g.u_scale) + 1, cell_hi);
      sh_w = chi - sh_clo + 1;
    }
  }
  for (int kk = k0; kk < k1; ++kk) {
    const int buf = (kk - k0) & 1;
    const AngleCS a = cs[kk];
    const int i = base[kk];
    const bool full = (i != 0) && (8 * i != g.n_angles);
    const int clo = __shfl_sync(0xffffffffu, sh_clo, kk - k0);
    const int W = __shfl_sync(0xffffffffu, sh_w, kk - k0);
    const bool use_win = W <= kD8Win;
    if (inside) {
      unsigned* wb = &win[buf][0][0][0] - clo;
      fast::pixel_weights(g, a.C, a.S, ix, iy, status, [&](int m, double w) {
        cnt += full ? 8 : 4;
        if (use_win) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e < 4 || full)
              limb_add<L>(wb + e * L * kD8Win + m, w, xs[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e < 4 || full) {
              unsigned long long* row =
                  yacc + (long long)d4_angle(g.n_angles, i, e) * rpa + g.n_det_y / 2;
              atomicAdd(row + (e >= 4 ? -1 - m : m),
                        (unsigned long long)__double2ll_rn(w * xs[e]));
            }
        }
      });
    }
    __syncthreads();
    if (use_win) {
#pragma unroll
      for (int j0 = 0; j0 < 8 * kD8Win; j0 += 128) {
        const int j = j0 + threadIdx.x;
        const int e = j / kD8Win, c = j % kD8Win;
        if (c < W && (e < 4 || full)) {
          unsigned long long v;
          if (L == 1) {
            v = (unsigned long long)(long long)(int)win[buf][e][0][c];
          } else {
            v = (unsigned long long)win[buf][e][0][c] +
                ((unsigned long long)(long long)(int)win[buf][e][L - 1][c] << 24);
            win[buf][e][L - 1][c] = 0u;
          }
          win[buf][e][0][c] = 0u;
          if (v) {
            const int m = clo + c;
            unsigned long long* row =
                yacc + (long long)d4_angle(g.n_angles, i, e) * rpa + g.n_det_y / 2;
            atomicAdd(row + (e >= 4 ? -1 - m : m), v);
          }
        }
      }
    }
  }
  count_updates(n_upd, cnt);
}

// Backward: thread = D4 orbit of a pixel p0 of the fundamental triangle
// (iy0 <= ix0 < n/2); members p_h = h p0 (the 4 rotations only when p0 lies
// on the diagonal, whose reflections coincide with rotations). The weight set
// of member h at base angle i is gathered against angle g i, cell g m for
// every group element g into the accumulator of pixel (g o h) p0.
//
// TR: y is the base angles' image rows interleaved, yt[k][m][e] (image e >= 4
// at the mirrored cell, transpose_images_kernel): a weight reads the 8 image
// values with vector loads instead of 8 scattered ones.
template <typename T, bool TR>
__global__ void __launch_bounds__(128, CTSM_D8B_MINB) bwd2d_d8_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    int chunk, const T* __restrict__ y, T* __restrict__ x, double* __restrict__ part,
    int* status) {
  const int h = g.n_x / 2;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)h * (h + 1) / 2) return;
  // triangular index -> (ix0 >= iy0)
  int ix0 = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((long long)(ix0 + 1) * (ix0 + 2) / 2 <= t) ++ix0;
  while ((long long)ix0 * (ix0 + 1) / 2 > t) --ix0;
  const int iy0 = (int)(t - (long long)ix0 * (ix0 + 1) / 2);
  const bool diag = (ix0 == iy0);
  const int n = g.n_x;
  int px[8], py[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) d4_pixel(n, ix0, iy0, e, px[e], py[e]);
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  const int k0 = blockIdx.y * chunk;
  const int k1 = min(k0 + chunk, n_base);
  for (int kk = k0; kk < k1; ++kk) {
    const AngleCS a = cs[kk];
    const int i = base[kk];
    const bool full = (i != 0) && (8 * i != g.n_angles);
    // 2D sinograms are < 2^31 entries: 32-bit row offsets
    int rows[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      rows[e] = TR ? 0 : d4_angle(g.n_angles, i, e) * g.rows_per_angle + g.n_det_y / 2;
    // one inlined sweep for all members (small code: the member loop is not
    // unrolled); tsum[ge] collects member hm's sums per group element and is
    // folded into acc[ge o hm] by a static permutation per member.
    const int n_mem = diag ? 4 : 8;
#pragma unroll 1
    for (int hm = 0; hm < n_mem; ++hm) {
      int mx, my;
      d4_pixel(n, ix0, iy0, hm, mx, my);
      double tsum[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) tsum[e] = 0.0;
      const T* yk = y + ((long long)kk * g.n_det_y + g.n_det_y / 2) * 8;
      fast::pixel_weights(g, a.C, a.S, mx, my, status, [&](int m, double w) {
        if (TR) {
          T v[8];
          load_vec<T, 8>(yk + (long long)m * 8, v);
#pragma unroll
          for (int ge = 0; ge < 8; ++ge)
            if (ge < 4 || full) tsum[ge] += w * (double)v[ge];
        } else {
#pragma unroll
          for (int ge = 0; ge < 4; ++ge) tsum[ge] += w * ld(&y[rows[ge] + m]);
          if (full) {
#pragma unroll
            for (int ge = 4; ge < 8; ++ge) tsum[ge] += w * ld(&y[rows[ge] - 1 - m]);
          }
        }
      });
      switch (hm) {
#define CTSM_FOLD(H)                                                      \
  case H:                                                                 \
    _Pragma("unroll") for (int ge = 0; ge < 8; ++ge) acc[d4_compose(ge, H)] += tsum[ge]; \
    break;
        CTSM_FOLD(0) CTSM_FOLD(1) CTSM_FOLD(2) CTSM_FOLD(3)
        CTSM_FOLD(4) CTSM_FOLD(5) CTSM_FOLD(6) CTSM_FOLD(7)
#undef CTSM_FOLD
      }
    }
  }
  const long long npix = (long long)n * n;
  auto put = [&](int e, double v) {
    const long long pix = (long long)py[e] * n + px[e];
    if (part)
      part[(long long)blockIdx.y * npix + pix] = v;
    else
      x[pix] = (T)v;
  };
  if (diag) {
    // pixel of e equals pixel of e o (R M) (= e o 5): fold the aliases
#pragma unroll
    for (int e = 0; e < 4; ++e) put(e, acc[e] + acc[d4_compose(e, 5)]);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) put(e, acc[e]);
  }
}

// 3D symmetric forward (group order G = 4: quarter turns, base angles < n/4;
// G = 8: dihedral, base angles 0..n/8, see the 2D kernels above): warp =
// column c, base angles only; each weight of c at base angle i is scattered
// to the rows of the image angles e i (image detector column -1-m_y for the
// reflections) with the voxel values of the image columns e c.
//
// The voxel values of the G image columns are staged in shared memory once
// per z-block ([image][slot][lane], conflict-free) and reused for all base
// angles: the per-weight reads are shared-memory hits instead of G scattered
// global loads.
#ifndef CTSM_KZCF
#define CTSM_KZCF 8
#endif
#ifndef CTSM_FWD3_MINB
#define CTSM_FWD3_MINB 3
#endif
#ifndef CTSM_FWD3_MINB_F
#define CTSM_FWD3_MINB_F 4  // fp32: 128 registers (small spills) beat 160 (C3 fwd 253 -> 227 ms)
#endif
template <typename T, int G>
constexpr int fwd3_minb() { return G == 8 ? (sizeof(T) == 4 ? CTSM_FWD3_MINB_F : CTSM_FWD3_MINB) : 4; }
#ifndef CTSM_KZCF_F
#define CTSM_KZCF_F CTSM_KZCF
#endif
// z-block of 32 * zc voxels for the staged values (per dtype)
template <typename T>
__host__ __device__ constexpr int fwd3_zc() { return sizeof(T) == 4 ? CTSM_KZCF_F : CTSM_KZCF; }

template <typename T, int G>
constexpr size_t fwd3d_sym_dyn_smem() { return sizeof(T) * kWarps3 * G * fwd3_zc<T>() * 32; }

//
// FA (fp32 volumes, G = 8): the row runs go with two 16-byte vector float
// reductions (red.global.add.v4.f32) into the launch's image-interleaved rows
// yt[k][my][mz][e] (the layout of the back-projection's transposed input)
// instead of 8 scalar 64-bit fixed-point atomics; fwd3d_uninterleave then
// writes the sinogram rows. The fp32 sums are order-dependent at the fp32
// rounding level (the fp64 path stays fixed point and bit-reproducible).
template <typename T, int G, bool FA = false>
__global__ void __launch_bounds__(kWarps3 * 32, fwd3_minb<T, G>()) fwd3d_sym_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    const T* __restrict__ in, unsigned long long* __restrict__ yacc, double scale,
    unsigned long long* n_upd, int* status, float* __restrict__ yt = nullptr,
    const FastPlan* __restrict__ plans = nullptr) {
  __shared__ __align__(16) fast::ColumnHead sh[kWarps3];
  __shared__ __align__(16) fast::PieceCoef sp[kWarps3][fast::kMaxPieces];
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  // [warp][t][chunk][lane][V]: the G image values of (t, lane) as NC 16-byte
  // vectors, each chunk conflict-free across the lanes (one LDS.128 each)
  constexpr int V = 16 / sizeof(T), NC = G / V;
  constexpr int kZcF = fwd3_zc<T>();
  T* xsm = reinterpret_cast<T*>(dyn_smem) + (size_t)(threadIdx.x >> 5) * kZcF * G * 32;
  auto xidx = [&](int t, int e, int ln) { return ((t * NC + e / V) * 32 + ln) * V + e % V; };
  __shared__ long long sab[kWarps3][G];  // row base of every image angle of the base angle
  CTSM_BATCH_DECL(kWarps3);
  CTSM_TABLE_DECL(kWarps3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = g.n_x;
  const long long nxy = (long long)n * g.n_y;
  const long long col = (long long)blockIdx.x * kWarps3 + warp;
  if (col >= nxy) return;  // whole warp
  const int ix = (int)(col % n), iy = (int)(col / n);
  const int rpa = g.rows_per_angle, ndy = g.n_det_y;
  const int hy = g.n_det_y / 2, hz = g.n_det_z / 2;
  unsigned cnt = 0;
  // z mirror (even n_z): only the lower half of the column is evaluated;
  // each weight of voxel iz at row m_z also applies to voxel n_z-1-iz at row
  // -1-m_z, whose values are staged in the upper half of the slots
  const bool zmir = zmirror_on() && (g.n_z % 2 == 0);
  constexpr int kMF = kZcF / 2;
  const int zspan = zmir ? g.n_z / 2 : g.n_z;
  const int zbs = 32 * (zmir ? kMF : kZcF);
  for (int zb0 = 0; zb0 < zspan; zb0 += zbs) {
    const int nzb = min(zbs, zspan - zb0);
    const int zc = (nzb + 31) / 32;
    const int z0 = zb0 + lane * zc, z1 = min(z0 + zc, zb0 + nzb);
    __syncwarp();
#pragma unroll
    for (int e = 0; e < G; ++e) {
      int rx, ry;
      d4_pixel(n, ix, iy, e, rx, ry);
      // z-fastest volume: the lane's z-chunk is contiguous (its sectors are
      // re-hit in L1 across t), instead of one sector per voxel
      const T* src = in + ((long long)ry * n + rx) * g.n_z;
#pragma unroll 1
      for (int t = 0; t < zc; ++t) {
        xsm[xidx(t, e, lane)] = (z0 + t < z1) ? src[z0 + t] : (T)0;
        if (zmir) xsm[xidx(kMF + t, e, lane)] = (z0 + t < z1) ? src[g.n_z - 1 - (z0 + t)] : (T)0;
      }
    }
    __syncwarp();
    for (int kk = 0; kk < n_base; ++kk) {
      const int i = base[kk];
      const AngleCS a = cs[kk];
      const bool full = G == 4 || ((i != 0) && (8 * i != g.n_angles));
      const int ne = full ? G : 4;
      __syncwarp();
      if (lane < G) sab[warp][lane] = (long long)d4_angle(g.n_angles, i, lane) * rpa;
#ifdef CTSM_INKERNEL_PLAN
      const bool ok = plans ? load_plan(plans, (long long)kk * nxy + col, sh[warp], sp[warp], lane)
                            : fast::plan_column(g, a.C, a.S, ix, iy, status, sh[warp], sp[warp],
                                                lane);
#else
      (void)a;
      const bool ok = load_plan(plans, (long long)kk * nxy + col, sh[warp], sp[warp], lane);
      if (kk + 1 < n_base) prefetch_plan(plans, (long long)(kk + 1) * nxy + col, lane);
#endif
      __syncwarp();
      if (!ok) continue;
      const fast::GroupTable* TB = table3d(sh[warp], sp[warp], CTSM_TABLE_PTR, lane);
#ifdef CTSM_EXP_PLAN_ONLY
      continue;  // timing experiment: planning cost alone
#endif
      // pending merge of consecutive emits to one row (see proj3d_kernel):
      // row pr = (mz + hz) ndy + py, py = my + hy; reflections write -1-my
      // the run of one row is summed in FP64 (fixed lane order: deterministic)
      // and converted to fixed point once, at the flush
      // fp32 volumes sum a row run in fp32 (1-3 terms; converted to fixed
      // point at the flush), fp64 volumes in fp64
      using PT = T;
      const float scale_f = (float)scale;
      int pr = -1;
      PT pv[G], pm[G];  // run sums of the lower voxel and of its z mirror
      int py = 0, pz = 0;
#pragma unroll
      for (int e = 0; e < G; ++e) pv[e] = pm[e] = (PT)0;
      // one call site per side (no loop over a register-array selector)
      auto flush_side = [&](const PT* q, const int rz) {
        {
          if constexpr (FA) {
            // interleaved row (my, mz) of slot kk: all G images in one vector
            // (the launch's scratch holds < 2^31 floats: sym3d_chunk bounds it)
            float* dst = yt + (unsigned)(((kk * ndy + py) * g.n_det_z + rz) * G);
#pragma unroll
            for (int c = 0; c < G / 4; ++c)
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * c),
                           "f"((float)q[4 * c]), "f"((float)q[4 * c + 1]), "f"((float)q[4 * c + 2]),
                           "f"((float)q[4 * c + 3])
                           : "memory");
          } else {
#pragma unroll
            for (int e = 0; e < G; ++e)
              if (e < ne && q[e] != (PT)0) {
                const long long r = (long long)rz * ndy + ((e < 4) ? py : ndy - 1 - py);
#ifdef CTSM_EXP_NO_SCATTER
                if (q[e] == (PT)1.2345) yacc[r] = 1;  // timing experiment: no atomics
#else
                // fp32 runs convert in fp32 (2^-24 of the fixed-point range:
                // far below the fp32 output rounding)
                const long long iv = sizeof(T) == 4 ? __float2ll_rn((float)q[e] * scale_f)
                                                    : __double2ll_rn((double)q[e] * scale);
                atomicAdd(yacc + sab[warp][e] + r, (unsigned long long)iv);
#endif
              }
          }
        }
      };
      auto flush = [&]() {
        flush_side(pv, pz);
        if (zmir) flush_side(pm, g.n_det_z - 1 - pz);  // mirror row -1-mz
      };
      unsigned nw = 0;  // weights of this (column, angle); updates = nw * images * sides
      auto apply_weight = [&](const int iz, const PT wp) {
        auto acc_side = [&](PT* acc, const int slot) {
          const T* xv = xsm + xidx(slot, 0, lane);
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            T v[V];
            if constexpr (sizeof(T) == 4) {
              const float4 q = reinterpret_cast<const float4*>(xv)[c * 32];
              v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
            } else {
              const double2 q = reinterpret_cast<const double2*>(xv)[c * 32];
              v[0] = q.x; v[1] = q.y;
            }
            // FA: the interleaved scratch rows carry all G image slots and
            // fwd3d_uninterleave reads only the first 4 of a self-symmetric
            // base angle, so the other 4 may accumulate (unused) values
            if constexpr (FA && sizeof(T) == 4) {
              // packed fp32 FMAs (FFMA2, sm_100): two images per instruction,
              // each component rounded as the scalar FMA would
              const float2 w2 = make_float2((float)wp, (float)wp);
#pragma unroll
              for (int u = 0; u < V; u += 2) {
                const float2 r = __ffma2_rn(w2, make_float2((float)v[u], (float)v[u + 1]),
                                            make_float2((float)acc[c * V + u], (float)acc[c * V + u + 1]));
                acc[c * V + u] = (PT)r.x;
                acc[c * V + u + 1] = (PT)r.y;
              }
            } else {
#pragma unroll
              for (int u = 0; u < V; ++u)
                if (FA || c * V + u < ne) acc[c * V + u] += wp * v[u];
            }
          }
        };
        acc_side(pv, iz - z0);
        if (zmir) acc_side(pm, kMF + iz - z0);
      };
      auto on_weight = [&](int iz, int my, int mz, double w) {
        ++nw;
        const int r = (mz + hz) * ndy + (my + hy);  // < rows_per_angle < 2^31
        if (r != pr) {
          if (pr >= 0) flush();
          pr = r;
          py = my + hy;
          pz = mz + hz;
#pragma unroll
          for (int e = 0; e < G; ++e) pv[e] = pm[e] = (PT)0;
        }
        apply_weight(iz, (PT)w);
      };
#if CTSM_FLAT && !defined(CTSM_NO_BATCH) && !defined(CTSM_TABLE3D)
      (void)TB;
      {
#if CTSM_FWD3_GEND
      // runs end with their cell group: the pending run's cell is the group's
      // (py is loop-invariant in the walk; the flush address is rz * G off a
      // per-group base)
      int prz = -1;
      auto flush_g = [&](const int pyy) {
        py = pyy;
        flush_side(pv, prz);
        if (zmir) flush_side(pm, g.n_det_z - 1 - prz);
      };
      fast::chunk_weights_flat<true>(
          g, sh[warp], sp[warp], z0, z1,
          [&](int iz, int my, int mz, double w) {
            ++nw;
            const int rz = mz + hz;
            if (rz != prz) {
              if (prz >= 0) flush_g(my + hy);
              prz = rz;
#pragma unroll
              for (int e = 0; e < G; ++e) pv[e] = pm[e] = (PT)0;
            }
            apply_weight(iz, (PT)w);
          },
          CTSM_BATCH_PTR, lane, fast::NoPre(),
          [&](int cell) {
            if (prz >= 0) flush_g(cell + hy);
            prz = -1;
          });
      pr = -1;
#else
      fast::chunk_weights_flat(g, sh[warp], sp[warp], z0, z1, on_weight, CTSM_BATCH_PTR, lane);
#endif
      }
#else
      fast::chunk_weights(g, sh[warp], sp[warp], z0, z1, on_weight, TB, CTSM_BATCH_PTR, lane);
#endif
      if (pr >= 0) flush();
      cnt += nw * (unsigned)(zmir ? 2 * ne : ne);
    }
  }
  count_updates(n_upd, cnt);
}

// 3D symmetric backward: warp = orbit of a column of the fundamental domain
// (G = 4: first quadrant, members R^j c; G = 8: triangle iy0 <= ix0 < n/2,
// members h c, the 4 rotations only on the diagonal). Per base angle the
// members are planned in turn and every weight set of member h is gathered
// against the image angles e i into the shared-memory accumulator of member
// e o h (fixed order: deterministic).
#ifndef CTSM_KZCS
#define CTSM_KZCS 8
#endif
#ifndef CTSM_BWD3_MINB
#define CTSM_BWD3_MINB 8
#endif
#ifndef CTSM_KWS
#define CTSM_KWS 2
#endif
#ifndef CTSM_KWS_F
#define CTSM_KWS_F 2
#endif
#ifndef CTSM_BWD3_MINB_F
#define CTSM_BWD3_MINB_F 7  // with the early row-vector loads: C3 bwd 45.9 -> 45.1 ms per half scan (8: 45.9, 6: 51.2, 9: 63.9)
#endif
// warps (orbits) per block and min blocks per SM of the fp64 / fp32 variants
template <typename T>
__host__ __device__ constexpr int bwd3_warps() { return sizeof(T) == 4 ? CTSM_KWS_F : CTSM_KWS; }
template <typename T>
__host__ __device__ constexpr int bwd3_minb() { return sizeof(T) == 4 ? CTSM_BWD3_MINB_F : CTSM_BWD3_MINB; }
template <typename T>
struct BwdAcc {
  using type = double;
};
#ifndef CTSM_BWD3_ACC64
template <>
struct BwdAcc<float> {
  using type = float;
};
#endif
#ifndef CTSM_KZCS_F
#define CTSM_KZCS_F CTSM_KZCS
#endif
template <typename T>
__host__ __device__ constexpr int bwd3_zc() { return sizeof(T) == 4 ? CTSM_KZCS_F : CTSM_KZCS; }



// TR: `in` is the launch's image rows transposed per (base slot, image) into
// [k * G + e][my][mz] (mz fastest, transpose_images below): a lane walking up
// its z-chunk then reads consecutive addresses (shared sectors / L1 hits)
// instead of one 2 KB-strided sector per row.
template <typename T, int G, bool TR>
__global__ void __launch_bounds__(bwd3_warps<T>() * 32, bwd3_minb<T>()) bwd3d_sym_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    const T* __restrict__ in, T* __restrict__ xout, int accumulate, int* status,
    const FastPlan* __restrict__ plans = nullptr) {
  constexpr int kWarpsS = bwd3_warps<T>();
  __shared__ __align__(16) fast::ColumnHead sh[kWarpsS];
  __shared__ __align__(16) fast::PieceCoef sp[kWarpsS][fast::kMaxPieces];
  // fp32 volumes accumulate their per-launch sums in fp32 (fixed order, so
  // still deterministic): at most ~chunk * 12 terms per slot, an error far
  // below the fp32 tolerance, and half the shared memory -> more warps/SM
  using AccT = typename BwdAcc<T>::type;
  constexpr int kZcS = bwd3_zc<T>();
  __shared__ AccT sacc[kWarpsS][G][kZcS][32];
  CTSM_TABLE_DECL(kWarpsS);
// warp-batched cubic faces: neutral before the z mirror (C3 190 vs 194 ms),
// a gain with it (C3 bwd 148 -> 138 ms: every batched face now serves two
// voxels); CTSM_BWD3_NOBATCH evaluates them in place
#ifndef CTSM_BWD3_NOBATCH
  CTSM_BATCH_DECL(kWarpsS);
#define CTSM_BATCH_PTR_B CTSM_BATCH_PTR
#else
#define CTSM_BATCH_PTR_B nullptr
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = g.n_x, h = n / 2;
  // (dispatching the orbits from the centre of the grid outwards, most work
  // first, changed nothing: 85 vs 85 ms)
  const long long n_orb = G == 4 ? (long long)h * h : (long long)h * (h + 1) / 2;
  const long long orb = (long long)blockIdx.x * kWarpsS + warp;
  if (orb >= n_orb) return;  // whole warp
  int ix0, iy0;
  if (G == 4) {
    ix0 = (int)(orb % h);
    iy0 = (int)(orb / h);
  } else {
    ix0 = (int)((sqrt(8.0 * (double)orb + 1.0) - 1.0) * 0.5);
    while ((long long)(ix0 + 1) * (ix0 + 2) / 2 <= orb) ++ix0;
    while ((long long)ix0 * (ix0 + 1) / 2 > orb) --ix0;
    iy0 = (int)(orb - (long long)ix0 * (ix0 + 1) / 2);
  }
  const bool diag = G == 8 && ix0 == iy0;
  const int n_mem = (G == 4 || diag) ? 4 : 8;
  const int rpa = g.rows_per_angle;
  const int hy = g.n_det_y / 2, hz = g.n_det_z / 2;
  // z mirror (even n_z, TR): voxel iz at row m_z has the weight of voxel
  // n_z-1-iz at row -1-m_z (source and detector centred on z = 0), so only
  // the lower half of the column is evaluated and every weight is gathered
  // twice; the mirrored voxels use the upper half of the slots
  const bool zmir = TR && zmirror_on() && (g.n_z % 2 == 0);
  constexpr int kM = kZcS / 2;
  const int zspan = zmir ? g.n_z / 2 : g.n_z;
  const int zbs = 32 * (zmir ? kM : kZcS);
  for (int zb0 = 0; zb0 < zspan; zb0 += zbs) {
    const int nzb = min(zbs, zspan - zb0);
    const int zc = (nzb + 31) / 32;
    const int z0 = zb0 + lane * zc, z1 = min(z0 + zc, zb0 + nzb);
    for (int j = 0; j < G; ++j)
      for (int t = 0; t < zc; ++t) {
        sacc[warp][j][t][lane] = 0.0;
        if (zmir) sacc[warp][j][kM + t][lane] = 0.0;
      }
    for (int kk = 0; kk < n_base; ++kk) {
      const int i = base[kk];
      const AngleCS a = cs[kk];
      const bool full = G == 4 || ((i != 0) && (8 * i != g.n_angles));
      const T* yb[TR ? 1 : G];
      if (TR) {
        yb[0] = in + (long long)kk * G * rpa;
      } else {
#pragma unroll
        for (int e = 0; e < (TR ? 1 : G); ++e) yb[e] = in + (long long)d4_angle(g.n_angles, i, e) * rpa;
      }
#pragma unroll 1
      for (int hm = 0; hm < n_mem; ++hm) {
        int cx, cy;
        d4_pixel(n, ix0, iy0, hm, cx, cy);
        __syncwarp();
#ifdef CTSM_INKERNEL_PLAN
        const bool ok =
            plans ? load_plan(plans, (long long)kk * ((long long)n * g.n_y) + (long long)cy * n + cx,
                              sh[warp], sp[warp], lane)
                  : fast::plan_column(g, a.C, a.S, cx, cy, status, sh[warp], sp[warp], lane);
#else
        (void)a;
        const bool ok = load_plan(
            plans, (long long)kk * ((long long)n * g.n_y) + (long long)cy * n + cx, sh[warp],
            sp[warp], lane);
#if CTSM_PLAN_PREFETCH
        {
          // the next member of this base angle, or member 0 of the next one
          int nh = hm + 1, nk = kk;
          if (nh == n_mem) {
            nh = 0;
            ++nk;
          }
          if (nk < n_base) {
            int px, py;
            d4_pixel(n, ix0, iy0, nh, px, py);
            prefetch_plan(plans, (long long)nk * ((long long)n * g.n_y) + (long long)py * n + px,
                          lane);
          }
        }
#endif
#endif
        __syncwarp();
        if (!ok) continue;
        const fast::GroupTable* TB = table3d(sh[warp], sp[warp], CTSM_TABLE_PTR, lane);
#ifdef CTSM_EXP_PLAN_ONLY
        continue;  // timing experiment: planning cost alone
#endif
        // accumulator slots of the images, 3 bits each (one register: kept
        // live through the gathers instead of re-derived per weight)
        unsigned pk = 0;
#pragma unroll
        for (int e = 0; e < G; ++e) pk |= (unsigned)d4_compose(e, hm) << (3 * e);
#ifdef CTSM_EXP_NO_GATHER
#define CTSM_LDY(p) ((AccT)1)
#else
#define CTSM_LDY(p) ((AccT)__ldg(p))
#endif
        // consecutive weights of a lane often hit the same detector row (the
        // row shared by voxels iz and iz + 1): its image vectors are kept in
        // registers instead of being gathered again
        int prow = -1;
        T pv0[G], pv1[G];
        auto gather = [&](int t, int my, int mz, double w) {
          const AccT wa = (AccT)w;  // fp32 volumes: FFMA in fp32
          if (TR) {
            // the G image values of (my, mz): one contiguous vector; with
            // the z mirror also those of row -1-mz for voxel n_z-1-iz
            const int rowi = (my + hy) * g.n_det_z + (mz + hz);
            if (rowi != prow) {
              const T* rowp = yb[0] + (long long)(my + hy) * g.n_det_z * G;
              load_vec<T, G>(rowp + (long long)(mz + hz) * G, pv0);
              if (zmir) load_vec<T, G>(rowp + (long long)(g.n_det_z - 1 - (mz + hz)) * G, pv1);
              prow = rowi;
            }
            // one call site per side (no loop over a register-array selector)
            auto add_side = [&](const T* v, const int slot) {
              // the G slots are distinct (pk is a permutation): all loads,
              // then all adds, then all stores -- as one read-modify-write per
              // slot the compiler must assume aliasing and serialise them
              AccT* base = &sacc[warp][0][slot][lane];
              constexpr int kSlot = kZcS * 32;
              AccT cur[G];
#pragma unroll
              for (int e = 0; e < G; ++e) cur[e] = base[((pk >> (3 * e)) & 7) * kSlot];
#pragma unroll
              for (int e = 0; e < G; ++e)
                if (e < 4 || full) cur[e] += wa * (AccT)v[e];
#pragma unroll
              for (int e = 0; e < G; ++e) base[((pk >> (3 * e)) & 7) * kSlot] = cur[e];
            };
            add_side(pv0, t);
            if (zmir) add_side(pv1, kM + t);
          } else {
            const long long r = (long long)(mz + hz) * g.n_det_y + (my + hy);
#pragma unroll
            for (int e = 0; e < 4; ++e) sacc[warp][(pk >> (3 * e)) & 7][t][lane] += wa * CTSM_LDY(&yb[e][r]);
            if (G == 8 && full) {
              const long long rr = r + g.n_det_y - 1 - 2 * (my + hy);
#pragma unroll
              for (int e = 4; e < G; ++e) sacc[warp][(pk >> (3 * e)) & 7][t][lane] += wa * CTSM_LDY(&yb[e][rr]);
            }
          }
        };
#if CTSM_FLAT && !defined(CTSM_NO_BATCH) && !defined(CTSM_BWD3_NOBATCH) && !defined(CTSM_TABLE3D)
        (void)TB;
#if CTSM_BWD3_EARLY_LOAD
        // the row vectors of the weight about to be evaluated: loaded before
        // the evaluation (pv0 / pv1 are live across it anyway)
        auto pre_row = [&](int my, int mz) {
          if (TR) {
            const int rowi = (my + hy) * g.n_det_z + (mz + hz);
            if (rowi != prow) {
              const T* rowp = yb[0] + (long long)(my + hy) * g.n_det_z * G;
              load_vec<T, G>(rowp + (long long)(mz + hz) * G, pv0);
              if (zmir) load_vec<T, G>(rowp + (long long)(g.n_det_z - 1 - (mz + hz)) * G, pv1);
              prow = rowi;
            }
          }
        };
        fast::chunk_weights_flat(
            g, sh[warp], sp[warp], z0, z1,
            [&](int iz, int my, int mz, double w) { gather(iz - z0, my, mz, w); }, CTSM_BATCH_PTR_B,
            lane, pre_row);
#else
        fast::chunk_weights_flat(
            g, sh[warp], sp[warp], z0, z1,
            [&](int iz, int my, int mz, double w) { gather(iz - z0, my, mz, w); }, CTSM_BATCH_PTR_B,
            lane);
#endif
#else
        fast::chunk_weights(g, sh[warp], sp[warp], z0, z1,
                            [&](int iz, int my, int mz, double w) { gather(iz - z0, my, mz, w); }, TB,
                            CTSM_BATCH_PTR_B, lane);
#endif
      }
    }
    for (int e = 0; e < (diag ? 4 : G); ++e) {
      int cx, cy;
      d4_pixel(n, ix0, iy0, e, cx, cy);
      const long long c = (long long)cy * n + cx;
      const int e2 = d4_compose(e, 5);  // diagonal: e c == (e o 5) c
      for (int t = 0; t < zc; ++t) {
        const int iz = z0 + t;
        if (iz >= z1) break;
        for (int side = 0; side < (zmir ? 2 : 1); ++side) {
          const int sl = side == 0 ? t : kM + t;
          double v = (double)sacc[warp][e][sl][lane];
          if (diag) v += (double)sacc[warp][e2][sl][lane];
          T* dst = xout + c * g.n_z + (side == 0 ? iz : g.n_z - 1 - iz);  // z-fastest volume
          if (accumulate) v += (double)*dst;
          *dst = (T)v;
        }
      }
    }
  }
}

// Member-outer form of the symmetric back-projection (transposed image rows,
// flattened walk; CTSM_BWD3_VEC). In bwd3d_sym_kernel a weight of member h is
// added, per image e, to the accumulator of pixel (e o h) p0: a run-time
// permutation of 8 scalar shared-memory slots (3 integer instructions per
// slot to decode it, 8 LDS + 8 STS per side). Here the members are the OUTER
// loop: member h accumulates all its base angles in image order -- slot e
// holds image e, so the G slots of a voxel are one contiguous vector
// (2 LDS.128 + 2 STS.128 per side in fp32, no decoding) -- and its sums are
// added to the pixels (e o h) p0 of the z-fastest volume once per member and
// z-block. The orbit belongs to this warp alone, so those updates are plain
// loads and stores in a fixed order (deterministic).
#ifndef CTSM_BWD3_VEC
#define CTSM_BWD3_VEC 1  // C3 bwd 87 -> 85 ms per projection
#endif
#ifndef CTSM_BWD3_SPLIT
#define CTSM_BWD3_SPLIT 1  // C3 bwd 86 -> 79 ms per projection
#endif
template <typename T, int G>
__global__ void __launch_bounds__(bwd3_warps<T>() * 32, bwd3_minb<T>()) bwd3d_sym_v_kernel(
    DevGeom g, const AngleCS* __restrict__ cs, const int* __restrict__ base, int n_base,
    const T* __restrict__ in, T* __restrict__ xout, int accumulate, int* status,
    const FastPlan* __restrict__ plans) {
  constexpr int kWarpsS = bwd3_warps<T>();
  __shared__ __align__(16) fast::ColumnHead sh[kWarpsS];
  __shared__ __align__(16) fast::PieceCoef sp[kWarpsS][fast::kMaxPieces];
  using AccT = typename BwdAcc<T>::type;
  constexpr int kZcS = bwd3_zc<T>();
  constexpr int V = 16 / sizeof(AccT), NC = G / V;
  // [warp][slot][chunk][lane][V]: the G image sums of (slot, lane) as NC
  // 16-byte vectors, each conflict-free across the lanes
  __shared__ __align__(16) AccT sacc[kWarpsS][kZcS][NC][32][V];
  CTSM_BATCH_DECL(kWarpsS);
  (void)cs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = g.n_x, h = n / 2;
  const long long nxy = (long long)n * g.n_y;
  // CTSM_BWD3_SPLIT: an orbit is shared by the block's two warps, warp w
  // taking half of the members and folding into its own partial volume
  // (xout + w * n_vox; the host adds the two while transposing). A C3 launch
  // is 8,256 orbits on 16 resident warps x 148 SMs = 3.49 rounds, i.e. 4 with
  // the last one half empty (occupancy 14 of 16 warps, ncu); split, it is
  // 6.97 rounds of half-length units.
  const long long n_orb = G == 4 ? (long long)h * h : (long long)h * (h + 1) / 2;
#if CTSM_BWD3_SPLIT
  static_assert(kWarpsS == 2, "a warp pair per orbit");
  const long long orb = (long long)blockIdx.x;
#else
  const long long orb = (long long)blockIdx.x * kWarpsS + warp;
#endif
  if (orb >= n_orb) return;  // whole warp
  int ix0, iy0;
  if (G == 4) {
    ix0 = (int)(orb % h);
    iy0 = (int)(orb / h);
  } else {
    ix0 = (int)((sqrt(8.0 * (double)orb + 1.0) - 1.0) * 0.5);
    while ((long long)(ix0 + 1) * (ix0 + 2) / 2 <= orb) ++ix0;
    while ((long long)ix0 * (ix0 + 1) / 2 > orb) --ix0;
    iy0 = (int)(orb - (long long)ix0 * (ix0 + 1) / 2);
  }
  const bool diag = G == 8 && ix0 == iy0;
  const int n_mem = (G == 4 || diag) ? 4 : 8;
  const int rpa = g.rows_per_angle;
  const int hy = g.n_det_y / 2, hz = g.n_det_z / 2;
  const bool zmir = zmirror_on() && (g.n_z % 2 == 0);
  constexpr int kM = kZcS / 2;
  const int zspan = zmir ? g.n_z / 2 : g.n_z;
  const int zbs = 32 * (zmir ? kM : kZcS);
  for (int zb0 = 0; zb0 < zspan; zb0 += zbs) {
    const int nzb = min(zbs, zspan - zb0);
    const int zc = (nzb + 31) / 32;
    const int z0 = zb0 + lane * zc, z1 = min(z0 + zc, zb0 + nzb);
#if CTSM_BWD3_SPLIT
    const int m_lo = warp * (n_mem / 2), m_hi = m_lo + n_mem / 2;
    T* const xw = xout + (long long)warp * g.n_vox;
#else
    const int m_lo = 0, m_hi = n_mem;
    T* const xw = xout;
#endif
#pragma unroll 1
    for (int hm = m_lo; hm < m_hi; ++hm) {
      int cx, cy;
      d4_pixel(n, ix0, iy0, hm, cx, cy);
      const long long mcol = (long long)cy * n + cx;
      // this lane's slots (only this lane reads or writes them)
      for (int t = 0; t < zc; ++t)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int u = 0; u < V; ++u) {
            sacc[warp][t][c][lane][u] = (AccT)0;
            if (zmir) sacc[warp][kM + t][c][lane][u] = (AccT)0;
          }
#pragma unroll 1
      for (int kk = 0; kk < n_base; ++kk) {
        const int i = base[kk];
        const bool full = G == 4 || ((i != 0) && (8 * i != g.n_angles));
        const T* yb = in + (long long)kk * G * rpa;
        __syncwarp();
        const bool ok = load_plan(plans, (long long)kk * nxy + mcol, sh[warp], sp[warp], lane);
#if CTSM_PLAN_PREFETCH
        if (kk + 1 < n_base) {
          prefetch_plan(plans, (long long)(kk + 1) * nxy + mcol, lane);
        } else if (hm + 1 < m_hi) {
          int px, py;
          d4_pixel(n, ix0, iy0, hm + 1, px, py);
          prefetch_plan(plans, (long long)py * n + px, lane);
        }
#endif
        __syncwarp();
        if (!ok) continue;
        int prow = -1;
        T pv0[G], pv1[G];
        auto pre_row = [&](int my, int mz) {
          const int rowi = (my + hy) * g.n_det_z + (mz + hz);
          if (rowi != prow) {
            const T* rowp = yb + (long long)(my + hy) * g.n_det_z * G;
            load_vec<T, G>(rowp + (long long)(mz + hz) * G, pv0);
            if (zmir) load_vec<T, G>(rowp + (long long)(g.n_det_z - 1 - (mz + hz)) * G, pv1);
            prow = rowi;
          }
        };
        auto add_side = [&](const T* v, const int slot, const AccT wa) {
          AccT* sp0 = &sacc[warp][slot][0][lane][0];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (c * V < 4 || full) {
              if constexpr (sizeof(AccT) == 4) {
                float4* q = reinterpret_cast<float4*>(sp0 + c * 32 * V);
                float4 cur = *q;
                const float2 w2 = make_float2((float)wa, (float)wa);
                const float2 lo = __ffma2_rn(w2, make_float2((float)v[c * V], (float)v[c * V + 1]),
                                             make_float2(cur.x, cur.y));
                const float2 hi = __ffma2_rn(w2, make_float2((float)v[c * V + 2], (float)v[c * V + 3]),
                                             make_float2(cur.z, cur.w));
                *q = make_float4(lo.x, lo.y, hi.x, hi.y);
              } else {
                double2* q = reinterpret_cast<double2*>(sp0 + c * 32 * V);
                double2 cur = *q;
                cur.x += (double)wa * (double)v[c * V];
                cur.y += (double)wa * (double)v[c * V + 1];
                *q = cur;
              }
            }
          }
        };
        fast::chunk_weights_flat(
            g, sh[warp], sp[warp], z0, z1,
            [&](int iz, int my, int mz, double w) {
              // (pv0 / pv1 hold this row: the walk's pre() precedes every emit)
              const AccT wa = (AccT)w;
              // (loading both sides' vectors before updating either: no gain)
              add_side(pv0, iz - z0, wa);
              if (zmir) add_side(pv1, kM + iz - z0, wa);
            },
            CTSM_BATCH_PTR, lane, pre_row);
      }
      // member hm's sums of image e belong to pixel (e o hm) p0; the first
      // member initialises the pixels (on the diagonal the images e >= 4
      // alias the pixels of e < 4 and add to them)
#pragma unroll 1
      for (int e = 0; e < G; ++e) {
        int px, py;
        d4_pixel(n, ix0, iy0, d4_compose(e, hm), px, py);
        T* col = xw + ((long long)py * n + px) * g.n_z;  // z-fastest (partial) volume
        const bool init = hm == m_lo && !accumulate && (e < 4 || !diag);
        for (int t = 0; t < zc; ++t) {
          const int iz = z0 + t;
          if (iz >= z1) break;
          for (int side = 0; side < (zmir ? 2 : 1); ++side) {
            const int sl = side == 0 ? t : kM + t;
            double v = (double)sacc[warp][sl][e / V][lane][e % V];
            T* dst = col + (side == 0 ? iz : g.n_z - 1 - iz);
            if (!init) v += (double)*dst;
            *dst = (T)v;
          }
        }
      }
    }
  }
}

template <typename T>
__global__ void fixed_rows_kernel(int rpa, int angle_begin, int angle_step, int n_sel,
                                  unsigned long long* acc, double inv_scale, T* y) {
  const long long n = (long long)rpa * n_sel;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i / rpa);
    const long long r = (long long)(angle_begin + k * angle_step) * rpa + (i % rpa);
    const long long q = (long long)acc[r];
    y[r] = (T)((double)q * inv_scale);
  }
}

__global__ void zero_rows_kernel(int rpa, int angle_begin, int angle_step, int n_sel,
                                 unsigned long long* acc) {
  const long long n = (long long)rpa * n_sel;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i / rpa);
    acc[(long long)(angle_begin + k * angle_step) * rpa + (i % rpa)] = 0ull;
  }
}

__global__ void fixed_to_double_kernel(uint64_t n, const unsigned long long* acc, double inv_scale,
                                       double* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (double)(long long)acc[i] * inv_scale;
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // valid for v >= 0: IEEE ordering of non-negative doubles == integer ordering
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

template <typename T>
__global__ void max_abs_kernel(uint64_t n, const T* v, double* out) {
  double m = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double a = fabs((double)v[i]);
    if (!(a <= m)) m = a;  // NaN propagates as "larger"
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

template <typename T>
__global__ void invert_nonzero_kernel(uint64_t n, T* v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const T a = v[i];
    v[i] = a != (T)0 ? (T)(1.0 / (double)a) : (T)0;
  }
}

template <typename T>
__global__ void sirt_residual_kernel(int rpa, int angle_begin, int angle_step, int n_sel,
                                     const T* y, const T* rinv, T* ax) {
  const long long n = (long long)rpa * n_sel;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i / rpa);
    const long long r = (long long)(angle_begin + k * angle_step) * rpa + (i % rpa);
    ax[r] = rinv[r] * (y[r] - ax[r]);
  }
}

template <typename T>
__global__ void sirt_update_kernel(uint64_t n, const T* cinv, const T* bp, T* x) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    x[i] += cinv[i] * bp[i];
}

template <typename T>
__global__ void fill_kernel(uint64_t n, double v, T* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)v;
}

unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  const uint64_t cap = 148ull * 16;
  return (unsigned)(b == 0 ? 1 : (b < cap ? b : cap));
}

}  // namespace

cudaError_t build_angle_cs(const DevGeom& g, int angle_begin, int angle_step, int n_sel,
                           AngleCS* out, cudaStream_t st) {
  if (n_sel <= 0) return cudaSuccess;
  angle_cs_kernel<<<(n_sel + 127) / 128, 128, 0, st>>>(g, angle_begin, angle_step, n_sel, out);
  count_launch();
  return cudaGetLastError();
}

static dim3 tile_grid(const DevGeom& g, unsigned ydim, int tx = kTx) {
  const int ty = 128 / tx;
  const unsigned tiles = (unsigned)(((g.n_x + tx - 1) / tx) * ((g.n_y + ty - 1) / ty));
  return dim3(tiles, ydim);
}

// Angles per launch of the general 3D kernel: the rows of one launch's angles
// should stay L2-resident (~64 MB of the 126 MB L2), see sym3d_chunk below.
static int gen3d_chunk(const DevGeom& g, size_t elem_bytes) {
  int c = (int)((64.0 * (1 << 20)) / ((double)g.rows_per_angle * (double)elem_bytes));
  // ... and the launch's plans (one per column and angle) within ~2 GB
  const double plan_angle = (double)g.n_x * g.n_y * (double)sizeof(FastPlan);
  const int cp = (int)((2048.0 * (1 << 20)) / plan_angle);
  if (c > cp) c = cp;
  return c < 1 ? 1 : c;
}

cudaError_t fwd_mf(const DevGeom& g, int dtype, const AngleCS* cs, int angle_begin,
                   int angle_step, int n_sel, const void* x, unsigned long long* yacc,
                   double scale, unsigned long long* n_upd, int* status, cudaStream_t st,
                   void* plans) {
  if (n_sel <= 0) return cudaSuccess;
  const bool two_d = (g.n_z == 1 && g.n_det_z == 1);
  if (two_d) {
    const dim3 grid = tile_grid(g, (unsigned)((n_sel + kFwdAngles - 1) / kFwdAngles));
    if (dtype == CTSM_F64)
      fwd2d_kernel<double><<<grid, 128, 0, st>>>(g, cs, angle_begin, angle_step, n_sel,
                                                 (const double*)x, yacc, scale, n_upd, status);
    else
      fwd2d_kernel<float><<<grid, 128, 0, st>>>(g, cs, angle_begin, angle_step, n_sel,
                                                (const float*)x, yacc, scale, n_upd, status);
    count_launch();
  } else {
    const long long nxy = (long long)g.n_x * g.n_y;
    const unsigned blocks = (unsigned)((nxy + kWarps3 - 1) / kWarps3);
    const int chunk = gen3d_chunk(g, sizeof(unsigned long long));
    for (int k0 = 0; k0 < n_sel; k0 += chunk) {
      const int nk = n_sel - k0 < chunk ? n_sel - k0 : chunk;
      const int a0 = angle_begin + k0 * angle_step;
      {
        const cudaError_t e = plan_pass(g, cs + k0, nk, plans, status, st);
        if (e != cudaSuccess) return e;
      }
      if (dtype == CTSM_F64)
        proj3d_kernel<double, true><<<blocks, kWarps3 * 32, 0, st>>>(
            g, cs + k0, a0, angle_step, nk, (const double*)x, nullptr, yacc, scale, n_upd, 0,
            status, (const FastPlan*)plans);
      else
        proj3d_kernel<float, true><<<blocks, kWarps3 * 32, 0, st>>>(
            g, cs + k0, a0, angle_step, nk, (const float*)x, nullptr, yacc, scale, n_upd, 0,
            status, (const FastPlan*)plans);
      count_launch();
    }
  }
  return cudaGetLastError();
}

int bwd_chunks(const DevGeom& g, int n_sel) {
  const bool two_d = (g.n_z == 1 && g.n_det_z == 1);
  if (!two_d || n_sel <= 1) return 1;
  const long long tiles = (long long)((g.n_x + kTx - 1) / kTx) * ((g.n_y + kTy - 1) / kTy);
  // aim for >= ~16 resident-block waves (148 SMs x ~6 blocks of 128 threads)
  long long c = (16LL * 148 * 6 + tiles - 1) / tiles;
  if (c > n_sel) c = n_sel;
  if (c > 64) c = 64;
  return (int)(c < 1 ? 1 : c);
}

cudaError_t bwd_mf(const DevGeom& g, int dtype, const AngleCS* cs, int angle_begin,
                   int angle_step, int n_sel, const void* y, void* x, double* part, int n_chunks,
                   int* status, cudaStream_t st, void* plans) {
  const bool two_d = (g.n_z == 1 && g.n_det_z == 1);
  if (two_d) {
    const int chunk = (n_sel + n_chunks - 1) / (n_chunks > 0 ? n_chunks : 1);
    const int nc = chunk > 0 ? (n_sel + chunk - 1) / chunk : 1;
    const dim3 grid = tile_grid(g, (unsigned)(nc > 0 ? nc : 1));
    double* p = nc > 1 ? part : nullptr;
    if (dtype == CTSM_F64)
      bwd2d_kernel<double><<<grid, 128, 0, st>>>(g, cs, angle_begin, angle_step, n_sel, chunk,
                                                 (const double*)y, (double*)x, p, status);
    else
      bwd2d_kernel<float><<<grid, 128, 0, st>>>(g, cs, angle_begin, angle_step, n_sel, chunk,
                                                (const float*)y, (float*)x, p, status);
    count_launch();
    if (nc > 1) {
      const long long n = (long long)g.n_x * g.n_y;
      if (dtype == CTSM_F64)
        bwd_reduce_kernel<double><<<grid_for(n), 256, 0, st>>>(n, nc, part, (double*)x);
      else
        bwd_reduce_kernel<float><<<grid_for(n), 256, 0, st>>>(n, nc, part, (float*)x);
      count_launch();
    }
  } else {
    const long long nxy = (long long)g.n_x * g.n_y;
    const unsigned blocks = (unsigned)((nxy + kWarps3 - 1) / kWarps3);
    // angle chunks accumulate into x in ascending order (deterministic)
    const int chunk = gen3d_chunk(g, dtype == CTSM_F64 ? 8 : 4);
    for (int k0 = 0; k0 < (n_sel > 0 ? n_sel : 1); k0 += chunk) {
      const int nk = n_sel - k0 < chunk ? n_sel - k0 : chunk;
      const int a0 = angle_begin + k0 * angle_step;
      void* pl = n_sel > 0 ? plans : nullptr;
      {
        const cudaError_t e = plan_pass(g, cs + k0, nk > 0 ? nk : 0, pl, status, st);
        if (e != cudaSuccess) return e;
      }
      if (dtype == CTSM_F64)
        proj3d_kernel<double, false><<<blocks, kWarps3 * 32, 0, st>>>(
            g, cs + k0, a0, angle_step, nk, (const double*)y, (double*)x, nullptr, 1.0, nullptr,
            k0 > 0, status, (const FastPlan*)pl);
      else
        proj3d_kernel<float, false><<<blocks, kWarps3 * 32, 0, st>>>(
            g, cs + k0, a0, angle_step, nk, (const float*)y, (float*)x, nullptr, 1.0, nullptr,
            k0 > 0, status, (const FastPlan*)pl);
      count_launch();
    }
  }
  return cudaGetLastError();
}

cudaError_t fwd_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                       int n_base, const void* x, unsigned long long* yacc, double scale,
                       unsigned long long* n_upd, int* status, cudaStream_t st) {
  if (n_base <= 0) return cudaSuccess;
  const dim3 grid = tile_grid(g, (unsigned)((n_base + kFwdAngles - 1) / kFwdAngles));
  if (dtype == CTSM_F64)
    fwd2d_sym_kernel<double><<<grid, 128, 0, st>>>(g, cs, base, n_base, (const double*)x, yacc,
                                                   scale, n_upd, status);
  else
    fwd2d_sym_kernel<float><<<grid, 128, 0, st>>>(g, cs, base, n_base, (const float*)x, yacc,
                                                  scale, n_upd, status);
  count_launch();
  return cudaGetLastError();
}

// Base angles per launch of the symmetric 3D kernels: every warp touches the
// rows of all image angles of the launch's base angles, so a launch covering
// the whole scan streams the sinogram (fixed-point accumulator / input) from
// HBM with scattered accesses; chunks bound that working set (and the launch's
// plan and scratch buffers).
static int sym3d_chunk(const DevGeom& g, int order, size_t elem_bytes) {
  const double per_base = (double)order * g.rows_per_angle * (double)elem_bytes;
  // r2: 192 MB of image rows per launch. Round 1 kept a launch's rows within
  // ~64 MB of the L2; with the interleaved fp32 rows and the plan pass longer
  // launches pay instead (fewer launch tails): C3 189.6 -> 183.5 ms, C4 SIRT
  // 2.96 -> 2.74 s per iteration at 256 MB, flat beyond ~160 MB.
  // (measured on the fp32 paths; the fp64 fixed-point rows keep 64 MB)
  static const double mb_env = getenv("CTSM_SYM3D_CHUNK_MB") ? atof(getenv("CTSM_SYM3D_CHUNK_MB")) : 0.0;
  const double mb = mb_env > 0.0 ? mb_env : (elem_bytes == 4 ? 192.0 : 64.0);
  int c = (int)((mb * (1 << 20)) / per_base);
  // ... and the launch's plans (one per column and base angle) within ~6 GB
  const double plan_base = (double)g.n_x * g.n_y * (double)sizeof(FastPlan);
  const int cp = (int)((6144.0 * (1 << 20)) / plan_base);
  if (c > cp) c = cp;
  return c < 1 ? 1 : c;
}

// out[c][r] = in[r][c] for a rows x cols matrix (volume layout changes
// [n_z][n_y n_x] <-> [n_y n_x][n_z]); 32x32 tiles through shared memory.
template <typename T>
__global__ void transpose2d_kernel(const T* __restrict__ in, T* __restrict__ out, long long rows,
                                   long long cols) {
  __shared__ T tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long r = r0 + j, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[j][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long c = c0 + j, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][j];
  }
}

// out[c][r] = in[r][c] + in2[r][c] (the two partial volumes of the split
// back-projection), summed in fp64
template <typename T>
__global__ void transpose2d_add_kernel(const T* __restrict__ in, const T* __restrict__ in2,
                                       T* __restrict__ out, long long rows, long long cols) {
  __shared__ T tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long r = r0 + j, c = c0 + threadIdx.x;
    if (r < rows && c < cols)
      tile[j][threadIdx.x] = (T)((double)in[r * cols + c] + (double)in2[r * cols + c]);
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const long long c = c0 + j, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][j];
  }
}

static cudaError_t transpose2d_add(int dtype, const void* in, const void* in2, void* out,
                                   long long rows, long long cols, cudaStream_t st) {
  const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (dtype == CTSM_F64)
    transpose2d_add_kernel<double><<<grid, dim3(32, 8), 0, st>>>(
        (const double*)in, (const double*)in2, (double*)out, rows, cols);
  else
    transpose2d_add_kernel<float><<<grid, dim3(32, 8), 0, st>>>(
        (const float*)in, (const float*)in2, (float*)out, rows, cols);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t transpose2d(int dtype, const void* in, void* out, long long rows,
                               long long cols, cudaStream_t st) {
  const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (dtype == CTSM_F64)
    transpose2d_kernel<double><<<grid, dim3(32, 8), 0, st>>>((const double*)in, (double*)out,
                                                             rows, cols);
  else
    transpose2d_kernel<float><<<grid, dim3(32, 8), 0, st>>>((const float*)in, (float*)out, rows,
                                                            cols);
  count_launch();
  return cudaGetLastError();
}

// yt[k][myc][mz][e] (slot k of the launch) -> sinogram rows of the image
// angles: y[angle(k, e)][mz][my], myc = my (e < 4) or ndy-1-my (reflections).
// Block = 32 (my) x 32 (mz) tile of one slot, all G images: the interleaved
// rows are read as contiguous G*32-float runs, the sinogram rows written
// coalesced. Slots of the self-symmetric base angles (i = 0, 8i = n) have
// only the 4 rotations.
template <int G>
__global__ void fwd3d_uninterleave(const float* __restrict__ yt, const int* __restrict__ base,
                                   int n_angles, int ndy, int ndz, float* __restrict__ y) {
  __shared__ float tile[G][32][33];
  const int k = blockIdx.z;
  const int my0 = blockIdx.x * 32, mz0 = blockIdx.y * 32;
  const int i = base[k];
  const bool full = G == 4 || ((i != 0) && (8 * i != n_angles));
  const long long rpa = (long long)ndy * ndz;
  const float* src = yt + (long long)k * G * rpa;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  // rows my0..my0+31: for image e the interleaved row is my (e < 4) or
  // ndy-1-my (e >= 4); each row run is G*32 contiguous floats
  for (int half = 0; half < (G == 8 ? 2 : 1); ++half)
    for (int j = 0; j < 32; ++j) {
      const int my = my0 + j;
      if (my >= ndy) break;
      const int myc = half == 0 ? my : ndy - 1 - my;
      const float* row = src + ((long long)myc * ndz + mz0) * G;
      for (int t = tid; t < 32 * G; t += 256) {
        const int mz = t / G, e = t % G;
        if ((e < 4) == (half == 0) && mz0 + mz < ndz) tile[e][j][mz] = row[t];
      }
    }
  __syncthreads();
  for (int e = 0; e < (full ? G : 4); ++e) {
    const int a = d4_angle(n_angles, i, e);
    float* dst = y + (long long)a * rpa;
    for (int j = threadIdx.y; j < 32; j += 8) {
      const int mz = mz0 + j, my = my0 + threadIdx.x;
      if (mz < ndz && my < ndy) dst[(long long)mz * ndy + my] = tile[e][threadIdx.x][j];
    }
  }
}

// Bytes of the plan scratch of one launch of the symmetric 3D kernels (the
// fp32 chunking is the larger one).
size_t mf3d_plan_bytes(const DevGeom& g, int order) {
#ifdef CTSM_INKERNEL_PLAN
  static const bool off = getenv("CTSM_NO_PLAN_PASS") != nullptr;
  if (off) return 0;
#endif
  if (g.n_z == 1 && g.n_det_z == 1) return 0;
  return (size_t)g.n_x * g.n_y * (size_t)sym3d_chunk(g, order, 4) * sizeof(FastPlan);
}

// ... and of one launch of the general (per-angle) 3D kernel.
size_t mf3d_plan_bytes_general(const DevGeom& g) {
  if (g.n_z == 1 && g.n_det_z == 1) return 0;
  return (size_t)g.n_x * g.n_y * (size_t)gen3d_chunk(g, 4) * sizeof(FastPlan);
}

size_t fwd3d_f32_scratch_elems(const DevGeom& g, int order) {
  if (order != 8 || getenv("CTSM_FWD3_FIXED")) return 0;
  return (size_t)sym3d_chunk(g, order, 4) * order * g.rows_per_angle;
}

// fp32 dihedral forward with vector float reductions (see fwd3d_sym_kernel,
// FA): writes the image rows of every base angle into y (fp32).
cudaError_t fwd3d_mf_d8_f32(const DevGeom& g, const AngleCS* cs, const int* base, int n_base,
                            const float* x_in, float* y, unsigned long long* n_upd, int* status,
                            cudaStream_t st, void* vol_t, float* yt, void* plans) {
  if (n_base <= 0) return cudaSuccess;
  {
    const cudaError_t e = transpose2d(CTSM_F32, x_in, vol_t, g.n_z, (long long)g.n_x * g.n_y, st);
    if (e != cudaSuccess) return e;
  }
  const long long nxy = (long long)g.n_x * g.n_y;
  const unsigned blocks = (unsigned)((nxy + kWarps3 - 1) / kWarps3);
  const int chunk = sym3d_chunk(g, 8, 4);
  constexpr size_t smem = fwd3d_sym_dyn_smem<float, 8>();
  cudaFuncSetAttribute(fwd3d_sym_kernel<float, 8, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int k0 = 0; k0 < n_base; k0 += chunk) {
    const int nk = n_base - k0 < chunk ? n_base - k0 : chunk;
    cudaError_t e = cudaMemsetAsync(yt, 0, (size_t)nk * 8 * g.rows_per_angle * sizeof(float), st);
    if (e != cudaSuccess) return e;
    e = plan_pass(g, cs + k0, nk, plans, status, st);
    if (e != cudaSuccess) return e;
    fwd3d_sym_kernel<float, 8, true><<<blocks, kWarps3 * 32, smem, st>>>(
        g, cs + k0, base + k0, nk, (const float*)vol_t, nullptr, 1.0, n_upd, status, yt,
        (const FastPlan*)plans);
    count_launch();
    const dim3 ug((g.n_det_y + 31) / 32, (g.n_det_z + 31) / 32, (unsigned)nk);
    fwd3d_uninterleave<8><<<ug, dim3(32, 8), 0, st>>>(yt, base + k0, g.n_angles, g.n_det_y,
                                                       g.n_det_z, y);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t fwd3d_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                         int n_base, const void* x_in, unsigned long long* yacc, double scale,
                         unsigned long long* n_upd, int* status, cudaStream_t st, int order,
                         void* vol_t, void* plans) {
  if (n_base <= 0) return cudaSuccess;
  {
    const cudaError_t e = transpose2d(dtype, x_in, vol_t, g.n_z, (long long)g.n_x * g.n_y, st);
    if (e != cudaSuccess) return e;
  }
  const void* x = vol_t;
  const long long nxy = (long long)g.n_x * g.n_y;
  const unsigned blocks = (unsigned)((nxy + kWarps3 - 1) / kWarps3);
  const int chunk = sym3d_chunk(g, order, sizeof(unsigned long long));
  for (int k0 = 0; k0 < n_base; k0 += chunk) {
    const int nk = n_base - k0 < chunk ? n_base - k0 : chunk;
    {
      const cudaError_t e = plan_pass(g, cs + k0, nk, plans, status, st);
      if (e != cudaSuccess) return e;
    }
#define CTSM_LAUNCH(T, G)                                                                     \
  do {                                                                                        \
    constexpr size_t smem = fwd3d_sym_dyn_smem<T, G>();                                       \
    cudaFuncSetAttribute(fwd3d_sym_kernel<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                         (int)smem);                                                          \
    fwd3d_sym_kernel<T, G><<<blocks, kWarps3 * 32, smem, st>>>(                                \
        g, cs + k0, base + k0, nk, (const T*)x, yacc, scale, n_upd, status, nullptr,           \
        (const FastPlan*)plans);                                                              \
  } while (0)
    if (dtype == CTSM_F64) {
      if (order == 8) CTSM_LAUNCH(double, 8); else CTSM_LAUNCH(double, 4);
    } else {
      if (order == 8) CTSM_LAUNCH(float, 8); else CTSM_LAUNCH(float, 4);
    }
#undef CTSM_LAUNCH
    count_launch();
  }
  return cudaGetLastError();
}

// Image rows of base slots [0, nk) -> yt[k][my][mz][e] (tiled transpose, the
// G images of a base slot interleaved): image e >= 4 (a reflection) is stored
// at the mirrored detector column ndy-1-my, so one (my, mz) of the base angle
// reads the values of all its images as one contiguous G-vector.
template <typename T>
__global__ void transpose_images_kernel(const T* __restrict__ y, const int* __restrict__ base,
                                        int G, int n_angles, int ndy, int ndz,
                                        T* __restrict__ yt) {
  __shared__ T tile[32][33];
  const int slab = blockIdx.z;
  const int e = slab % G;
  const int a = d4_angle(n_angles, base[slab / G], e);
  const long long rpa = (long long)ndy * ndz;
  const T* src = y + (long long)a * rpa;
  T* dst = yt + (long long)(slab / G) * G * rpa + e;
  const int cx = blockIdx.x * 32 + threadIdx.x;  // my
  const int rz = blockIdx.y * 32 + threadIdx.y;  // mz
  for (int j = 0; j < 32; j += 8)
    if (cx < ndy && rz + j < ndz) tile[threadIdx.y + j][threadIdx.x] = src[(long long)(rz + j) * ndy + cx];
  __syncthreads();
  const int oz = blockIdx.y * 32 + threadIdx.x;  // mz
  const int oy = blockIdx.x * 32 + threadIdx.y;  // my
  for (int j = 0; j < 32; j += 8)
    if (oz < ndz && oy + j < ndy) {
      const int myc = e < 4 ? oy + j : ndy - 1 - (oy + j);
      dst[((long long)myc * ndz + oz) * G] = tile[threadIdx.x][threadIdx.y + j];
    }
}

size_t bwd3d_scratch_elems(const DevGeom& g, int order, int dtype) {
  if (getenv("CTSM_BWD3_PLAIN")) return 0;
  return (size_t)sym3d_chunk(g, order, dtype == CTSM_F64 ? 8 : 4) * order * g.rows_per_angle;
}

cudaError_t bwd3d_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                         int n_base, const void* y, void* x_out, int* status, cudaStream_t st,
                         int order, void* scratch, void* vol_t, void* plans) {
  void* x = vol_t;  // z-fastest accumulator, transposed into x_out at the end
  const long long h = g.n_x / 2;
  const long long n_orb = order == 8 ? h * (h + 1) / 2 : h * h;
  const int kWS = dtype == CTSM_F64 ? bwd3_warps<double>() : bwd3_warps<float>();
  const unsigned blocks = (unsigned)((n_orb + kWS - 1) / kWS);
  const int chunk = sym3d_chunk(g, order, dtype == CTSM_F64 ? 8 : 4);
  const bool tr = scratch != nullptr && n_base > 0;
  // split back-projection: a block per orbit, two partial volumes in vol_t
  const bool split = CTSM_BWD3_SPLIT && CTSM_BWD3_VEC && tr && plans != nullptr;
  const unsigned vblocks = split ? (unsigned)n_orb : blocks;
  // chunks accumulate into x in ascending order (deterministic)
  for (int k0 = 0; k0 < (n_base > 0 ? n_base : 1); k0 += chunk) {
    const int nk = n_base - k0 < chunk ? n_base - k0 : chunk;
    if (tr) {
      const dim3 tg((g.n_det_y + 31) / 32, (g.n_det_z + 31) / 32, (unsigned)(nk * order));
      if (dtype == CTSM_F64)
        transpose_images_kernel<double><<<tg, dim3(32, 8), 0, st>>>(
            (const double*)y, base + k0, order, g.n_angles, g.n_det_y, g.n_det_z, (double*)scratch);
      else
        transpose_images_kernel<float><<<tg, dim3(32, 8), 0, st>>>(
            (const float*)y, base + k0, order, g.n_angles, g.n_det_y, g.n_det_z, (float*)scratch);
      count_launch();
    }
    // the fp64 chunking is the smaller one: the plan scratch holds it
    void* pl = (n_base > 0) ? plans : nullptr;
    {
      const cudaError_t e = plan_pass(g, cs + k0, nk > 0 ? nk : 0, pl, status, st);
      if (e != cudaSuccess) return e;
    }
#define CTSM_LAUNCH(T, G)                                                                      \
  do {                                                                                         \
    if (tr && CTSM_BWD3_VEC && pl)                                                             \
      bwd3d_sym_v_kernel<T, G><<<vblocks, bwd3_warps<T>() * 32, 0, st>>>(                      \
          g, cs + k0, base + k0, nk, (const T*)scratch, (T*)x, k0 > 0, status,                 \
          (const FastPlan*)pl);                                                                \
    else if (tr)                                                                               \
      bwd3d_sym_kernel<T, G, true><<<blocks, bwd3_warps<T>() * 32, 0, st>>>(                           \
          g, cs + k0, base + k0, nk, (const T*)scratch, (T*)x, k0 > 0, status,                 \
          (const FastPlan*)pl);                                                                \
    else                                                                                       \
      bwd3d_sym_kernel<T, G, false><<<blocks, bwd3_warps<T>() * 32, 0, st>>>(                          \
          g, cs + k0, base + k0, nk, (const T*)y, (T*)x, k0 > 0, status, (const FastPlan*)pl); \
  } while (0)
    if (dtype == CTSM_F64) {
      if (order == 8) CTSM_LAUNCH(double, 8); else CTSM_LAUNCH(double, 4);
    } else {
      if (order == 8) CTSM_LAUNCH(float, 8); else CTSM_LAUNCH(float, 4);
    }
#undef CTSM_LAUNCH
    count_launch();
  }
  if (split)
    return transpose2d_add(dtype, vol_t,
                           (const char*)vol_t + (size_t)g.n_vox * (dtype == CTSM_F64 ? 8 : 4), x_out,
                           (long long)g.n_x * g.n_y, g.n_z, st);
  return transpose2d(dtype, vol_t, x_out, (long long)g.n_x * g.n_y, g.n_z, st);
}

cudaError_t fwd_mf_d8(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                      int n_base, const void* x, unsigned long long* yacc, double scale,
                      unsigned long long* n_upd, int* status, cudaStream_t st) {
  if (n_base <= 0) return cudaSuccess;
  const dim3 grid = tile_grid(g, (unsigned)((n_base + kD8Angles - 1) / kD8Angles),
                              dtype == CTSM_F64 ? d8_tx<double>() : d8_tx<float>());
  if (dtype == CTSM_F64)
    fwd2d_d8_kernel<double><<<grid, 128, 0, st>>>(g, cs, base, n_base, (const double*)x, yacc,
                                                  scale, n_upd, status);
  else
    fwd2d_d8_kernel<float><<<grid, 128, 0, st>>>(g, cs, base, n_base, (const float*)x, yacc,
                                                 scale, n_upd, status);
  count_launch();
  return cudaGetLastError();
}

int bwd_d8_chunks(const DevGeom& g, int n_base) {
  const long long h = g.n_x / 2;
  const long long blocks = (h * (h + 1) / 2 + 127) / 128;
#ifndef CTSM_BWD2_WAVES
#define CTSM_BWD2_WAVES 3  // C1 bwd 0.772 -> 0.761 ms (f64), 0.738 -> 0.725 (f32) vs 6
#endif
  long long c = (16LL * 148 * CTSM_BWD2_WAVES + blocks - 1) / blocks;
  if (c > n_base) c = n_base;
  if (c > 64) c = 64;
  return (int)(c < 1 ? 1 : c);
}

// 2D rows of the base angles -> yt[k][m][e] (8 images interleaved, e >= 4 at
// the mirrored cell): one thread per output element, coalesced writes.
template <typename T>
__global__ void interleave2d_kernel(const T* __restrict__ y, const int* __restrict__ base,
                                    int n_base, int n_angles, int ndy, T* __restrict__ yt) {
  const long long n = (long long)n_base * ndy * 8;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < n;
       o += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(o & 7);
    const long long km = o >> 3;
    const int k = (int)(km / ndy), m = (int)(km % ndy);
    const int a = d4_angle(n_angles, base[k], e);
    yt[o] = y[(long long)a * ndy + (e < 4 ? m : ndy - 1 - m)];
  }
}

// fp32 only: measured at C1, the interleaved rows speed up the fp32 gathers
// (0.81 -> 0.74 ms) but slow the fp64 ones (0.77 -> 0.92 ms; 64-byte vectors
// spread over more L1 sectors than the 8 nearly coalesced direct rows)
size_t bwd_d8_scratch_elems(const DevGeom& g, int n_base, int dtype) {
  if (dtype == CTSM_F64 || getenv("CTSM_BWD2_PLAIN")) return 0;
  return (size_t)n_base * 8 * g.rows_per_angle;
}

cudaError_t bwd_mf_d8(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                      int n_base, const void* y, void* x, double* part, int n_chunks,
                      int* status, cudaStream_t st, void* yt) {
  const long long h = g.n_x / 2;
  const unsigned blocks = (unsigned)((h * (h + 1) / 2 + 127) / 128);
  const int chunk = (n_base + n_chunks - 1) / (n_chunks > 0 ? n_chunks : 1);
  const int nc = chunk > 0 ? (n_base + chunk - 1) / chunk : 1;
  double* p = nc > 1 ? part : nullptr;
  const dim3 grid(blocks, (unsigned)(nc > 0 ? nc : 1));
  const bool tr = yt != nullptr && n_base > 0;
  if (tr) {
    const unsigned gb = grid_for((uint64_t)n_base * g.n_det_y * 8);
    if (dtype == CTSM_F64)
      interleave2d_kernel<double><<<gb, 256, 0, st>>>((const double*)y, base, n_base, g.n_angles,
                                                      g.n_det_y, (double*)yt);
    else
      interleave2d_kernel<float><<<gb, 256, 0, st>>>((const float*)y, base, n_base, g.n_angles,
                                                     g.n_det_y, (float*)yt);
    count_launch();
  }
#define CTSM_LAUNCH(T)                                                                        \
  do {                                                                                        \
    if (tr)                                                                                   \
      bwd2d_d8_kernel<T, true><<<grid, 128, 0, st>>>(g, cs, base, n_base, chunk, (const T*)yt, \
                                                     (T*)x, p, status);                       \
    else                                                                                      \
      bwd2d_d8_kernel<T, false><<<grid, 128, 0, st>>>(g, cs, base, n_base, chunk,             \
                                                      (const T*)y, (T*)x, p, status);         \
  } while (0)
  if (dtype == CTSM_F64) CTSM_LAUNCH(double); else CTSM_LAUNCH(float);
#undef CTSM_LAUNCH
  count_launch();
  if (nc > 1) {
    const long long np = (long long)g.n_x * g.n_y;
    if (dtype == CTSM_F64)
      bwd_reduce_kernel<double><<<grid_for(np), 256, 0, st>>>(np, nc, part, (double*)x);
    else
      bwd_reduce_kernel<float><<<grid_for(np), 256, 0, st>>>(np, nc, part, (float*)x);
    count_launch();
  }
  return cudaGetLastError();
}

// fixed-point rows of an explicit angle list (zero / convert)
template <typename T>
__global__ void rows_list_kernel(int rpa, const int* angles, int n_list, unsigned long long* acc,
                                 double inv_scale, T* y, int mode) {
  const long long n = (long long)rpa * n_list;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = (long long)angles[i / rpa] * rpa + (i % rpa);
    if (mode == 0)
      acc[r] = 0ull;
    else
      y[r] = (T)((double)(long long)acc[r] * inv_scale);
  }
}

cudaError_t rows_list(const DevGeom& g, int dtype, const int* angles, int n_list,
                      unsigned long long* acc, double scale, void* y, int mode, cudaStream_t st) {
  const uint64_t n = (uint64_t)g.rows_per_angle * n_list;
  if (n == 0) return cudaSuccess;
  if (dtype == CTSM_F64)
    rows_list_kernel<double><<<grid_for(n), 256, 0, st>>>(g.rows_per_angle, angles, n_list, acc,
                                                          1.0 / scale, (double*)y, mode);
  else
    rows_list_kernel<float><<<grid_for(n), 256, 0, st>>>(g.rows_per_angle, angles, n_list, acc,
                                                         1.0 / scale, (float*)y, mode);
  count_launch();
  return cudaGetLastError();
}

int bwd_sym_chunks(const DevGeom& g, int n_base) {
  const int h = g.n_x / 2;
  const long long tiles = (long long)((h + kTx - 1) / kTx) * ((h + kTy - 1) / kTy);
  long long c = (16LL * 148 * 6 + tiles - 1) / tiles;
  if (c > n_base) c = n_base;
  if (c > 64) c = 64;
  return (int)(c < 1 ? 1 : c);
}

cudaError_t bwd_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                       int n_base, const void* y, void* x, double* part, int n_chunks,
                       int* status, cudaStream_t st) {
  const int h = g.n_x / 2;
  const unsigned tiles = (unsigned)(((h + kTx - 1) / kTx) * ((h + kTy - 1) / kTy));
  const int chunk = (n_base + n_chunks - 1) / (n_chunks > 0 ? n_chunks : 1);
  const int nc = chunk > 0 ? (n_base + chunk - 1) / chunk : 1;
  double* p = nc > 1 ? part : nullptr;
  const dim3 grid(tiles, (unsigned)(nc > 0 ? nc : 1));
  if (dtype == CTSM_F64)
    bwd2d_sym_kernel<double><<<grid, 128, 0, st>>>(g, cs, base, n_base, chunk, (const double*)y,
                                                   (double*)x, p, status);
  else
    bwd2d_sym_kernel<float><<<grid, 128, 0, st>>>(g, cs, base, n_base, chunk, (const float*)y,
                                                  (float*)x, p, status);
  count_launch();
  if (nc > 1) {
    const long long n = (long long)g.n_x * g.n_y;
    if (dtype == CTSM_F64)
      bwd_reduce_kernel<double><<<grid_for(n), 256, 0, st>>>(n, nc, part, (double*)x);
    else
      bwd_reduce_kernel<float><<<grid_for(n), 256, 0, st>>>(n, nc, part, (float*)x);
    count_launch();
  }
  return cudaGetLastError();
}

// (cos, sin) of an explicit angle list
__global__ void angle_cs_list_kernel(DevGeom g, const int* idx, int n, AngleCS* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = idx[k];
  const double phi = g.angle_start + (g.angle_end - g.angle_start) * i / g.n_angles;
  double S, C;
  sincos(phi, &S, &C);
  out[k] = AngleCS{C, S};
}

cudaError_t build_angle_cs_list(const DevGeom& g, const int* idx, int n, AngleCS* out,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  angle_cs_list_kernel<<<(n + 127) / 128, 128, 0, st>>>(g, idx, n, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t fixed_to_float_rows(const DevGeom& g, int dtype, int angle_begin, int angle_step,
                                int n_sel, unsigned long long* acc, double scale, void* y,
                                cudaStream_t st) {
  const uint64_t n = (uint64_t)g.rows_per_angle * n_sel;
  if (dtype == CTSM_F64)
    fixed_rows_kernel<double><<<grid_for(n), 256, 0, st>>>(g.rows_per_angle, angle_begin,
                                                           angle_step, n_sel, acc, 1.0 / scale,
                                                           (double*)y);
  else
    fixed_rows_kernel<float><<<grid_for(n), 256, 0, st>>>(g.rows_per_angle, angle_begin,
                                                          angle_step, n_sel, acc, 1.0 / scale,
                                                          (float*)y);
  count_launch();
  return cudaGetLastError();
}

cudaError_t zero_rows_u64(const DevGeom& g, int angle_begin, int angle_step, int n_sel,
                          unsigned long long* acc, cudaStream_t st) {
  const uint64_t n = (uint64_t)g.rows_per_angle * n_sel;
  zero_rows_kernel<<<grid_for(n), 256, 0, st>>>(g.rows_per_angle, angle_begin, angle_step,
                                                n_sel, acc);
  count_launch();
  return cudaGetLastError();
}

cudaError_t fixed_to_double(uint64_t n, const unsigned long long* acc, double scale, double* out,
                            cudaStream_t st) {
  fixed_to_double_kernel<<<grid_for(n), 256, 0, st>>>(n, acc, 1.0 / scale, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t max_abs(int dtype, uint64_t n, const void* v, double* out_dev, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  if (n == 0) return cudaSuccess;
  if (dtype == CTSM_F64)
    max_abs_kernel<double><<<grid_for(n), 256, 0, st>>>(n, (const double*)v, out_dev);
  else
    max_abs_kernel<float><<<grid_for(n), 256, 0, st>>>(n, (const float*)v, out_dev);
  count_launch();
  return cudaGetLastError();
}

cudaError_t invert_nonzero(int dtype, uint64_t n, void* v, cudaStream_t st) {
  if (dtype == CTSM_F64)
    invert_nonzero_kernel<double><<<grid_for(n), 256, 0, st>>>(n, (double*)v);
  else
    invert_nonzero_kernel<float><<<grid_for(n), 256, 0, st>>>(n, (float*)v);
  count_launch();
  return cudaGetLastError();
}

cudaError_t sirt_residual(const DevGeom& g, int dtype, int angle_begin, int angle_step,
                          int n_sel, const void* y, const void* rinv, void* ax,
                          cudaStream_t st) {
  const uint64_t n = (uint64_t)g.rows_per_angle * n_sel;
  if (dtype == CTSM_F64)
    sirt_residual_kernel<double><<<grid_for(n), 256, 0, st>>>(
        g.rows_per_angle, angle_begin, angle_step, n_sel, (const double*)y, (const double*)rinv,
        (double*)ax);
  else
    sirt_residual_kernel<float><<<grid_for(n), 256, 0, st>>>(
        g.rows_per_angle, angle_begin, angle_step, n_sel, (const float*)y, (const float*)rinv,
        (float*)ax);
  count_launch();
  return cudaGetLastError();
}

cudaError_t sirt_update(int dtype, uint64_t n, const void* cinv, const void* bp, void* x,
                        cudaStream_t st) {
  if (dtype == CTSM_F64)
    sirt_update_kernel<double><<<grid_for(n), 256, 0, st>>>(n, (const double*)cinv,
                                                            (const double*)bp, (double*)x);
  else
    sirt_update_kernel<float><<<grid_for(n), 256, 0, st>>>(n, (const float*)cinv,
                                                           (const float*)bp, (float*)x);
  count_launch();
  return cudaGetLastError();
}

cudaError_t fill_value(int dtype, uint64_t n, double v, void* out, cudaStream_t st) {
  if (dtype == CTSM_F64)
    fill_kernel<double><<<grid_for(n), 256, 0, st>>>(n, v, (double*)out);
  else
    fill_kernel<float><<<grid_for(n), 256, 0, st>>>(n, v, (float*)out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ctsmb

// ---- FP64 peak microkernel (roofline denominator) ---------------
namespace ctsmb {
namespace {
__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double b, double c) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 1.2345) out[0] = s;
}
}  // namespace

double bench_dfma_tflops(int device) {
  cudaSetDevice(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 8192;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-9);  // warm-up
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  count_launch(2);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * (double)blocks * threads * iters;
  return ms > 0 ? flops / (ms * 1e-3) / 1e12 : 0.0;
}
}  // namespace ctsmb
