// csr3d.cuh -- K2: exact 3D emission, one warp per (voxel column, angle).
//
// voxel_volume_factors (weights3d.cpp:354-462) in two kernels:
//   plan3d_kernel  one thread per (column, angle): canonical frame, strip
//                  sweep, per-cell 2D weights (the crmath-heavy, z-independent
//                  part) -> ColPlan in global memory;
//   emit3d_kernel  one warp per (column, angle), plan in shared memory, lanes =
//                  the voxels of a 32-voxel z chunk. The warp walks the row
//                  edges of its voxels in rounds; in a round every lane
//                  evaluates the same sequence of atoms (the column's pieces)
//                  on its own (row edge, z face) pair, so the FP64 work is
//                  lane-uniform, and emits the row weights with warp-level
//                  compaction (ballot + prefix) into the output sink.
//
// Bit-exactness (compiled with -fmad=false): every value is produced by the
// reference's operations on the reference's operands. What changes is how
// often identical operations run:
//   * quantities that depend only on (column, angle, breakpoint) -- cr = C +
//     S t, P / cr, Q / sr, delta, S S delta^3, sr / C, P^3 (cr1 + cr2) /
//     (cr1 cr2)^2 -- are evaluated once per column (OpConsts) instead of in
//     every atom call (weights3d.cpp:63-168 recomputes them per call);
//   * G = zref / (a tan_a) is evaluated once per (row edge, z face) instead
//     of once per atom;
//   * tri_atom_cum at a breakpoint shared by two adjacent pieces of the same
//     kind (b_hi of one, b_lo of the next; weights3d.cpp:404-419) is evaluated
//     once.
#pragma once
#include "exact.cuh"

namespace ctsmb {
namespace k2 {

constexpr int kMaxGrp = kMaxBrk;  // cell groups of one column sweep
constexpr int kMaxOps = 32;       // distinct atoms per (row edge, z face)
constexpr int kOpc = 11;          // doubles per OpConsts record

struct ColPlan {
  double S, C;                      // sin / cos of the canonical angle
  double x0, x1, y0, y1;            // canonical frame (Frame2D)
  double apex1_x, apex4_x;
  double dep[4];                    // corner depths x0y0, x0y1, x1y0, x1y1
  double tbrk[kMaxBrk];             // tan of the sweep breakpoints
  double gw2d[kMaxGrp];             // 2D weight of each in-range cell group
  int gcell[kMaxGrp];
  unsigned char gbeg[kMaxGrp], gend[kMaxGrp];  // piece range of each group
  unsigned char pkind[kMaxBrk], pb[kMaxBrk];   // piece kind, lower breakpoint
  // distinct atoms of the in-range pieces, in piece order (see emit3d_kernel)
  unsigned char optype[kMaxOps];  // 0 tri at apex 1, 1 trap, 2 tri at apex 4
  unsigned char opb[kMaxOps];     // breakpoint (tri) / lower breakpoint (trap)
  unsigned char plo[kMaxBrk], phi[kMaxBrk];  // per piece: atoms at b_lo / b_hi (trap: plo)
  int ng, np, nops, pad;
};
static_assert(sizeof(ColPlan) % 8 == 0, "ColPlan is copied as doubles");

// Output sink of the emission kernels.
//   mode 0: count entries per row (row_counter += 1);
//   mode 1: write the row-grouped entry {col, val} at row_start[row] -
//           pos_base + slot, slot = row_counter++;
//   mode 2: count, and append the entry as a 16-byte record {row, col, val}
//           to `rec` (single-evaluation build: the records are grouped by row
//           and sorted afterwards). Records are allocated from *cursor; a
//           record whose index is >= cap is dropped (the host sees cursor >
//           cap and retries with a larger buffer).
struct Sink {
  int mode;
  unsigned* row_counter;
  const uint64_t* row_start;
  uint4* grp;   // mode 1: row-grouped {col, -, val} entries
  uint4* rec;
  unsigned long long* cursor;
  unsigned long long cap;
  unsigned row_bias;   // added to the row of a record (launch slices of a shard)
  uint64_t pos_base;   // mode 1: col / val start at this global offset
};

constexpr unsigned kInvalidRow = 0xffffffffu;
constexpr unsigned long long kSeg = 256;  // records a warp allocates at a time

__device__ __forceinline__ uint4 make_rec(unsigned row, uint32_t column, double w) {
  return make_uint4(row, column, (unsigned)__double2loint(w), (unsigned)__double2hiint(w));
}

// Divergent-safe emission (2D kernel): the lanes that call together
// aggregate their record allocation into one atomic.
__device__ __forceinline__ void emit_any(const Sink& sk, uint64_t row_local, uint32_t column,
                                         double w) {
  if (sk.mode == 0) {
    atomicAdd(&sk.row_counter[row_local], 1u);
  } else if (sk.mode == 1) {
    const unsigned slot = atomicAdd(&sk.row_counter[row_local], 1u);
    const uint64_t pos = sk.row_start[row_local] - sk.pos_base + slot;
    sk.grp[pos] = make_uint4(column, 0u, (unsigned)__double2loint(w), (unsigned)__double2hiint(w));
  } else {
    atomicAdd(&sk.row_counter[row_local], 1u);
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(sk.cursor, (unsigned long long)__popc(m));
    base = __shfl_sync(m, base, leader);
    const unsigned long long pos = base + __popc(m & ((1u << lane) - 1u));
    if (pos < sk.cap) sk.rec[pos] = make_rec((unsigned)row_local + sk.row_bias, column, w);
  }
}

// Warp-convergent emission (3D kernel): all 32 lanes call; `flag` lanes emit.
// In mode 2 the warp owns a segment [seg_pos, seg_end) of the record buffer
// (warp-uniform registers) and refills it from the global cursor, so the
// global atomic runs once per kSeg records.
__device__ __forceinline__ void emit_warp(const Sink& sk, bool flag, uint64_t row_local,
                                          uint32_t column, double w,
                                          unsigned long long& seg_pos,
                                          unsigned long long& seg_end) {
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  if (m == 0) return;
  const int lane = threadIdx.x & 31;
  if (sk.mode == 0) {
    if (flag) atomicAdd(&sk.row_counter[row_local], 1u);
    return;
  }
  if (sk.mode == 1) {
    if (flag) {
      const unsigned slot = atomicAdd(&sk.row_counter[row_local], 1u);
      const uint64_t pos = sk.row_start[row_local] - sk.pos_base + slot;
      sk.grp[pos] = make_uint4(column, 0u, (unsigned)__double2loint(w), (unsigned)__double2hiint(w));
    }
    return;
  }
  if (flag) atomicAdd(&sk.row_counter[row_local], 1u);
  const unsigned n = __popc(m);
  if (seg_pos + n > seg_end) {
    // retire the segment: unused slots become invalid records
    for (unsigned long long i = seg_pos + lane; i < seg_end; i += 32)
      if (i < sk.cap) sk.rec[i] = make_uint4(kInvalidRow, 0u, 0u, 0u);
    unsigned long long np = 0;
    if (lane == 0) np = atomicAdd(sk.cursor, kSeg);
    np = __shfl_sync(0xffffffffu, np, 0);
    seg_pos = np;
    seg_end = np + kSeg;
  }
  const unsigned long long pos = seg_pos + __popc(m & ((1u << lane) - 1u));
  if (flag && pos < sk.cap) sk.rec[pos] = make_rec((unsigned)row_local + sk.row_bias, column, w);
  seg_pos += n;
}

__device__ __forceinline__ void retire_segment(const Sink& sk, unsigned long long seg_pos,
                                               unsigned long long seg_end) {
  if (sk.mode != 2) return;
  const int lane = threadIdx.x & 31;
  for (unsigned long long i = seg_pos + lane; i < seg_end; i += 32)
    if (i < sk.cap) sk.rec[i] = make_uint4(kInvalidRow, 0u, 0u, 0u);
}

// ---- plan: the z-independent part of voxel_volume_factors ------------------
__global__ void __launch_bounds__(128) plan3d_kernel(DevGeom g,
                                                     const exact::ExactAngle* __restrict__ angs,
                                                     const exact::EdgeAngle* __restrict__ edges,
                                                     ColPlan* __restrict__ plans, int* status) {
  const long long nxy = (long long)g.n_x * g.n_y;
  const long long colxy = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (colxy >= nxy) return;
  const int k = blockIdx.y;
  ColPlan* out = plans + ((size_t)k * nxy + colxy);
  out->ng = 0;
  out->np = 0;
  const int ix = (int)(colxy % g.n_x), iy = (int)(colxy / g.n_x);
  const exact::ExactAngle A = angs[k];
  const double s = g.s;
  exact::Sweep sw;
  if (!exact::strip_sweep(g, A, edges, face(ix, g.n_x, g.a), face(ix + 1, g.n_x, g.a),
                          face(iy, g.n_y, g.b), face(iy + 1, g.n_y, g.b), sw, status))
    return;
  // depths of the four xy corners (weights3d.cpp:367-371)
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
  // cell groups inside the detector with their 2D weight (weights3d.cpp:385-397)
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  int ng = 0;
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
      out->gbeg[ng] = (unsigned char)i;
      out->gend[ng] = (unsigned char)j;
      out->gcell[ng] = cell;
      out->gw2d[ng] = w2d;
      ++ng;
    }
    i = j;
  }
  if (ng == 0) return;
  out->S = sw.S;
  out->C = sw.C;
  out->x0 = sw.x0;
  out->x1 = sw.x1;
  out->y0 = sw.y0;
  out->y1 = sw.y1;
  out->apex1_x = sw.apex1_x;
  out->apex4_x = sw.apex4_x;
  for (int q = 0; q < 4; ++q) out->dep[q] = dep[q];
  for (int b = 0; b < sw.nb; ++b) out->tbrk[b] = sw.tbrk[b];
  for (int p = 0; p < sw.np; ++p) {
    out->pkind[p] = sw.pkind[p];
    out->pb[p] = sw.pb[p];
  }
  // distinct atoms: a trapezoid per kind-1 piece, a corner triangle per
  // (apex, breakpoint) used by a kind-0 / kind-2 piece
  unsigned char map0[kMaxBrk], map4[kMaxBrk];
  for (int q = 0; q < kMaxBrk; ++q) map0[q] = map4[q] = 0xff;
  int nops = 0;
  for (int q = 0; q < ng; ++q)
    for (int p = out->gbeg[q]; p < out->gend[q]; ++p) {
      const int kind = sw.pkind[p], lo = sw.pb[p], hi = lo + 1;
      if (nops + 2 > kMaxOps) {
        raise_status(status, CTSM_ERR_TOO_LARGE);
        return;
      }
      if (kind == 1) {
        out->optype[nops] = 1;
        out->opb[nops] = (unsigned char)lo;
        out->plo[p] = out->phi[p] = (unsigned char)nops;
        ++nops;
      } else {
        unsigned char* map = (kind == 0) ? map0 : map4;
        for (int e = 0; e < 2; ++e) {
          const int bidx = e == 0 ? lo : hi;
          if (map[bidx] == 0xff) {
            map[bidx] = (unsigned char)nops;
            out->optype[nops] = (unsigned char)(kind == 0 ? 0 : 2);
            out->opb[nops] = (unsigned char)bidx;
            ++nops;
          }
        }
        out->plo[p] = map[lo];
        out->phi[p] = map[hi];
      }
    }
  out->nops = nops;
  out->np = sw.np;
  out->ng = ng;
}

// ---- atoms with per-column constants ---------------------------------------
// x / b with rb = RN(1 / b) supplied: q0 = RN(x rb), r = x - b q0 (exact, one
// fma), q = RN(q0 + r rb). By Markstein's theorem (rb correctly rounded, q0
// within one ulp of x / b) q is the correctly rounded quotient, i.e. the bits
// of the IEEE division the reference performs -- in 3 FP64 instructions
// instead of the ~25 of a full division. Every divisor of the atom loop (C,
// S, cr1 cr2) is a per-column or per-breakpoint constant. Checked against the
// IEEE division on 2^28 random operand pairs by ctsm_selftest_division
// (tests/test_gpu_parity.py). CTSM_EXACT_DIV=1 compiles the plain divisions.
__device__ __forceinline__ double div_by(double x, double b, double rb) {
#ifdef CTSM_EXACT_DIV
  (void)rb;
  return x / b;
#else
  const double q0 = x * rb;
  const double r = __fma_rn(-b, q0, x);
  return __fma_rn(r, rb, q0);
#endif
}

// OpConsts of a corner-triangle atom at breakpoint t (tri_flags_at /
// tri_atom_flags, weights3d.cpp:115-168): c0 crg, c1 srh, c2 P/crg, c3 Q/srh,
// c4 P C, c5 Q S, c6 delta, c7 S S delta^3, c8 srh/C, c9 t.
__device__ __forceinline__ double tri_eval(const double* __restrict__ c, double S, double C,
                                           double rS, double rC, bool flat, double G,
                                           double tan_a, double coef) {
  const double g = G - c[2];
  const double gg = G - c[4] - c[5];
  const double h = G - c[3];
  const bool fg = g > 0.0, fgg = gg > 0.0, fh = h > 0.0;
  if (!flat) {
    double pair;
    if (fg && fgg) {
      const double delta = c[6];
      pair = c[0] * (3.0 * gg * gg * delta + 3.0 * gg * S * delta * delta + c[7]) -
             div_by(exact::cube(gg) * c[1], C, rC);
    } else if (!fg && !fgg) {
      pair = 0.0;
    } else {
      double v = 0.0;
      if (fg) v += c[0] * exact::cube(g);
      if (fgg) v -= div_by(exact::cube(gg), C, rC);
      pair = div_by(v, S, rS);
    }
    const double tt = pair + (fh ? c[8] * exact::cube(h) : 0.0);
    return coef * fabs(tan_a * tt);
  }
  const double t = c[9];
  double tv = 0.0;
  if (fg) tv += g * g * (t * g - 3.0 * t * (g - h));
  if (fh) tv -= t * exact::cube(h);
  return coef * fabs(tan_a * tv);
}

// trap_face_part (weights3d.cpp:51-61) with P/cr1, P/cr2 and the P^3 term
// supplied.
__device__ __forceinline__ double face_part_pre(double G, double G3, double P, double S,
                                                double rS, double t12, double cr1, double cr2,
                                                double cr12, double rcr12, double Pd1,
                                                double Pd2, double K) {
  const double d1 = G - Pd1, d2 = G - Pd2;
  const bool f1 = d1 > 0.0, f2 = d2 > 0.0;
  if (f1 && f2) return t12 * (G3 - div_by(3.0 * G * P * P, cr12, rcr12) + K);
  if (!f1 && !f2) return 0.0;
  double v = 0.0;
  if (f1) v += cr1 * exact::cube(d1);
  if (f2) v -= cr2 * exact::cube(d2);
  return div_by(v, S, rS);
}

// OpConsts of a trapezoid atom over (t1, t2) (weights3d.cpp:63-107): c0 cr1,
// c1 cr2, c2 t1 - t2, c3 cr1 cr2, c4 Pg/cr1, c5 Pg/cr2, c6 Pf/cr1, c7 Pf/cr2,
// c8 Pg^3 (cr1 + cr2) / (cr1 cr2)^2, c9 the same for Pf, c10 1 / (cr1 cr2). cst:
// Pg, Pf and, for the flat branch, 3 (s C - x1) / a and 3 (s C - x0) / a.
__device__ __forceinline__ double trap_eval(const double* __restrict__ c,
                                            const double* __restrict__ cst, double S, double rS,
                                            bool flat, double G, double G3, double tan_a,
                                            double coef) {
  const double Pg = cst[0], Pf = cst[1];
  if (!flat) {
    const double pg =
        face_part_pre(G, G3, Pg, S, rS, c[2], c[0], c[1], c[3], c[10], c[4], c[5], c[8]);
    const double pf =
        face_part_pre(G, G3, Pf, S, rS, c[2], c[0], c[1], c[3], c[10], c[6], c[7], c[9]);
    return coef * fabs(tan_a * (pg - pf));
  }
  const double gv = G - Pg, fv = G - Pf;
  double t = 0.0;
  if (gv > 0.0) t += gv * gv * (gv + cst[2]);
  if (fv > 0.0) t -= fv * fv * (fv + cst[3]);
  return coef * fabs(tan_a * t * c[2]);
}

// Self-test of div_by against the IEEE division: pseudo-random numerators
// over 26 decades and divisors in the ranges of C, S and cr1 cr2.
__global__ void selftest_division_kernel(unsigned long long n, unsigned long long seed,
                                         unsigned long long* mismatches) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long bad = 0;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;  // splitmix64
    double u[3];
    for (int j = 0; j < 3; ++j) {
      z += 0x9E3779B97F4A7C15ull;
      unsigned long long t = z;
      t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ull;
      t = (t ^ (t >> 27)) * 0x94D049BB133111EBull;
      t ^= t >> 31;
      u[j] = (double)(t >> 11) * 0x1.0p-53;
    }
    const int sel = (int)(i % 3);
    double b = sel == 0 ? 0.02 + 0.98 * u[0] : (sel == 1 ? 1e-8 + u[0] : 0.25 + 3.75 * u[0]);
    if (i & 8) b = -b;
    double x = (2.0 * u[1] - 1.0) * exp10(-20.0 + 26.0 * u[2]);
    if (i % 5 == 0) x = b * floor(u[1] * 1048576.0) * (1.0 + ((i & 16) ? 0x1.0p-52 : 0.0));
    const double rb = 1.0 / b;
    const double q0 = x * rb;
    const double r = __fma_rn(-b, q0, x);
    const double q = __fma_rn(r, rb, q0);
    if (__double_as_longlong(q) != __double_as_longlong(x / b)) ++bad;
  }
  if (bad) atomicAdd(mismatches, bad);
}

constexpr int kEmitWarps = 4;

struct WarpShared {
  ColPlan plan;
  double opc[kMaxOps][kOpc];
  double cst[4];
};

#ifndef CTSM_EMIT3_MINB
#define CTSM_EMIT3_MINB 5  // 96 registers: C2 assembly 736 -> 454 ms (6: 458, 8: 477)
#endif
__global__ void __launch_bounds__(kEmitWarps * 32, CTSM_EMIT3_MINB)
    emit3d_kernel(DevGeom g, const ColPlan* __restrict__ plans, int n_sel, Sink sk, int* status) {
  __shared__ WarpShared wsm[kEmitWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpShared& ws = wsm[wid];
  const unsigned full = 0xffffffffu;
  const long long nxy = (long long)g.n_x * g.n_y;
  const long long n_items = nxy * n_sel;
  const long long warps_total = (long long)gridDim.x * kEmitWarps;
  const double s = g.s, sdd = g.s + g.d;
  const double sdd_dz = sdd / g.d_z;
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  unsigned long long seg_pos = 0, seg_end = 0;

  for (long long item = (long long)blockIdx.x * kEmitWarps + wid; item < n_items;
       item += warps_total) {
    const int k = (int)(item / nxy);
    const long long colxy = item - (long long)k * nxy;
    const int ix = (int)(colxy % g.n_x), iy = (int)(colxy / g.n_x);
    __syncwarp();
    {  // plan -> shared memory
      const double* src = reinterpret_cast<const double*>(plans + item);
      double* dst = reinterpret_cast<double*>(&ws.plan);
      for (int i = lane; i < (int)(sizeof(ColPlan) / 8); i += 32) dst[i] = src[i];
    }
    __syncwarp();
    const int ng = ws.plan.ng;
    if (ng == 0) continue;
    const double S = ws.plan.S, C = ws.plan.C;
    const double a = ws.plan.x1 - ws.plan.x0, b = ws.plan.y1 - ws.plan.y0;
    const bool flat = !(fabs(S) > kEpsSingular);
    const double rS = 1.0 / S, rC = 1.0 / C;
    if (lane == 0) {
      ws.cst[0] = (s * C - ws.plan.x1) / a;
      ws.cst[1] = (s * C - ws.plan.x0) / a;
      ws.cst[2] = 3.0 * (s * C - ws.plan.x1) / a;
      ws.cst[3] = 3.0 * (s * C - ws.plan.x0) / a;
    }
    const int nops = ws.plan.nops;
    for (int o = lane; o < nops; o += 32) {
      double* c = ws.opc[o];
      const int ty = ws.plan.optype[o];
      if (ty == 1) {
        const double t1 = ws.plan.tbrk[ws.plan.opb[o]], t2 = ws.plan.tbrk[ws.plan.opb[o] + 1];
        const double cr1 = C + S * t1, cr2 = C + S * t2;
        const double Pg = (s * C - ws.plan.x1) / a, Pf = (s * C - ws.plan.x0) / a;
        c[0] = cr1;
        c[1] = cr2;
        c[2] = t1 - t2;
        c[3] = cr1 * cr2;
        c[4] = Pg / cr1;
        c[5] = Pg / cr2;
        c[6] = Pf / cr1;
        c[7] = Pf / cr2;
        c[8] = exact::cube(Pg) * (cr1 + cr2) / exact::sq(cr1 * cr2);
        c[9] = exact::cube(Pf) * (cr1 + cr2) / exact::sq(cr1 * cr2);
        c[10] = 1.0 / (cr1 * cr2);
      } else {
        const double t = ws.plan.tbrk[ws.plan.opb[o]];
        const double xa = ty == 0 ? ws.plan.apex1_x : ws.plan.apex4_x;
        const double ya = ty == 0 ? ws.plan.y0 : ws.plan.y1;
        const double crg = C + S * t;
        const double srh = S - C * t;
        const double P = (s * C - xa) / a;
        const double Q = (s * S - ya) / a;
        const double delta = Q - P * srh / crg;
        c[0] = crg;
        c[1] = srh;
        c[2] = P / crg;
        c[3] = Q / srh;
        c[4] = P * C;
        c[5] = Q * S;
        c[6] = delta;
        c[7] = S * S * exact::cube(delta);
        c[8] = srh / C;
        c[9] = t;
      }
    }
    __syncwarp();

    const uint64_t row_base = (uint64_t)k * g.rows_per_angle;
    double dep_min = ws.plan.dep[0], dep_max = ws.plan.dep[0];
#pragma unroll
    for (int qq = 1; qq < 4; ++qq) {
      dep_min = exact::dmin(dep_min, ws.plan.dep[qq]);
      dep_max = exact::dmax(dep_max, ws.plan.dep[qq]);
    }
    for (int z0 = 0; z0 < g.n_z; z0 += 32) {
      const int iz = z0 + lane;
      const bool act = iz < g.n_z;
      const double zb = face(iz, g.n_z, g.c), zt = face(iz + 1, g.n_z, g.c);
      const double cz = zt - zb;
      // row magnification range over the 8 corners (weights3d.cpp:365-378):
      // m = sdd/d_z * z / depth. Correctly rounded division is monotone in
      // both operands, so the minimum over the corners is attained at the
      // bottom face and the largest (z >= 0) or smallest (z < 0) depth, the
      // maximum at the top face likewise -- the same two values the
      // reference's min/max over all 8 quotients return.
      const double szb = sdd_dz * zb, szt = sdd_dz * zt;
      const double m_min = szb / (szb >= 0.0 ? dep_max : dep_min);
      const double m_max = szt / (szt >= 0.0 ? dep_min : dep_max);
      const int fl = (int)floor(m_min);
      const int k_lo = (fl < row_lo) ? row_lo : fl;
      const int ch = (int)ceil(m_max) - 1;
      const int k_hi = (ch < row_hi) ? ch : row_hi;
      const int E = (act && k_hi >= k_lo) ? (k_hi - k_lo + 2) : 0;
      int maxE = E;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxE = max(maxE, __shfl_xor_sync(full, maxE, o));
      const double coef = a * a / (6.0 * b * cz);
      const uint32_t column = (uint32_t)(((uint64_t)iz * g.n_y + iy) * g.n_x + ix);
      double prev[kMaxGrp];

      for (int e = 0; e < maxE; ++e) {
        const bool on = e < E;
        const int L = k_lo + e;
        const double kk = (double)L;
        // above(k) (weights3d.cpp:426-440): 1 -> w2d, 2 -> 0, 3 -> central
        // plane, 4 -> atoms
        int cls = 0;
        if (on) {
          if (kk <= m_min) cls = 1;
          else if (kk >= m_max) cls = 2;
          else if (kk == 0.0) cls = 3;
          else cls = 4;
        }
        const bool need = cls == 4;
        const bool any_need = __any_sync(full, need);
        double tan_a = 1.0, Gb = 0.0, Gt = 0.0, Gb3 = 0.0, Gt3 = 0.0;
        if (need) {
          tan_a = kk > 0.0 ? kk * g.d_z / sdd : -kk * g.d_z / sdd;
          const double zt_s = kk > 0.0 ? zt : -zt, zb_s = kk > 0.0 ? zb : -zb;
          Gb = zb_s / (a * tan_a);
          Gt = zt_s / (a * tan_a);
          Gb3 = exact::cube(Gb);
          Gt3 = exact::cube(Gt);
        }
        // the last two corner-triangle atoms evaluated (warp-uniform tags)
        int tag0 = -1, tag1 = -1, lru = 0;
        double vb0 = 0.0, vt0 = 0.0, vb1 = 0.0, vt1 = 0.0;
        for (int q = 0; q < ng; ++q) {
          const double w2d = ws.plan.gw2d[q];
          double ab = 0.0;
          if (any_need) {
            double Fb = 0.0, Ft = 0.0;
            for (int p = ws.plan.gbeg[q]; p < ws.plan.gend[q]; ++p) {
              const int kind = ws.plan.pkind[p];
              if (kind == 1) {
                if (need) {
                  const double* c = ws.opc[ws.plan.plo[p]];
                  Fb += trap_eval(c, ws.cst, S, rS, flat, Gb, Gb3, tan_a, coef);
                  Ft += trap_eval(c, ws.cst, S, rS, flat, Gt, Gt3, tan_a, coef);
                }
              } else {
                // b_lo first, then b_hi: the next piece of the chain reuses b_hi
                double xb0 = 0.0, xt0 = 0.0, xb1 = 0.0, xt1 = 0.0;
#pragma unroll 1
                for (int side = 0; side < 2; ++side) {
                  const int op = side == 0 ? ws.plan.plo[p] : ws.plan.phi[p];
                  double rb = 0.0, rt = 0.0;
                  if (op == tag0) {
                    rb = vb0;
                    rt = vt0;
                    lru = 1;
                  } else if (op == tag1) {
                    rb = vb1;
                    rt = vt1;
                    lru = 0;
                  } else {
                    if (need) {
                      const double* c = ws.opc[op];
                      rb = tri_eval(c, S, C, rS, rC, flat, Gb, tan_a, coef);
                      rt = tri_eval(c, S, C, rS, rC, flat, Gt, tan_a, coef);
                    }
                    if (lru == 0) {
                      tag0 = op;
                      vb0 = rb;
                      vt0 = rt;
                      lru = 1;
                    } else {
                      tag1 = op;
                      vb1 = rb;
                      vt1 = rt;
                      lru = 0;
                    }
                  }
                  if (side == 0) {
                    xb0 = rb;
                    xt0 = rt;
                  } else {
                    xb1 = rb;
                    xt1 = rt;
                  }
                }
                // kind 0: tri(b_hi) - tri(b_lo); kind 2: tri(b_lo) - tri(b_hi)
                if (kind == 0) {
                  Fb += xb1 - xb0;
                  Ft += xt1 - xt0;
                } else {
                  Fb += xb0 - xb1;
                  Ft += xt0 - xt1;
                }
              }
            }
            // weights3d.cpp:432-438: k > 0 -> F(zt) - F(zb); k < 0 -> w2d - (F(-zb) - F(-zt))
            ab = kk > 0.0 ? Ft - Fb : w2d - (Fb - Ft);
          }
          if (cls == 1) {
            ab = w2d;
          } else if (cls == 2) {
            ab = 0.0;
          } else if (cls == 3) {
            if (zb >= 0.0) ab = w2d;
            else if (zt <= 0.0) ab = 0.0;
            else ab = w2d * zt / (zt - zb);
          }
          bool out = false;
          double v = 0.0;
          if (on && e >= 1) {
            v = prev[q] - ab;
            if (v > kEpsWeight) out = true;
            else if (v < kNegClamp3D) raise_status(status, CTSM_ERR_NON_FINITE);
          }
          prev[q] = ab;
          emit_warp(sk, out,
                    row_base + (uint64_t)(L - 1 + g.n_det_z / 2) * g.n_det_y +
                        (ws.plan.gcell[q] + g.n_det_y / 2),
                    column, v, seg_pos, seg_end);
        }
      }
    }
  }
  retire_segment(sk, seg_pos, seg_end);
}

}  // namespace k2
}  // namespace ctsmb
