// fast3d.cuh -- matrix-free evaluation of the 3D consistent weights (voxel
// volume fractions per detector cell) along a voxel column.
//
// Same quantity as voxel_volume_factors (weights3d.cpp:354-462):
//  * the xy sweep is done in the ray parameter t = tan(beta) (fast2d.cuh),
//    shared by all voxels of the column (it does not depend on iz);
//  * the canonical quarter-turn frame (geometry.cpp:76-97) is the one whose
//    y0 face is the "low" face (the face holding the two smallest-t corners);
//    phi' = phi - k pi/2 gives (sin, cos) = (S, C), (-C, S), (-S, -C), (C, -S);
//  * the z composition (weights3d.cpp:380-458) uses the reference's closed-form
//    trapezoid / corner-triangle atoms (atoms.cuh) with tan(beta) = t exactly
//    (no atan/tan round trip) and cell 2D weights from fast2d's area forms.
#pragma once
#include "atoms.cuh"
#include "common.cuh"
#include "fast2d.cuh"

namespace ctsmb {
namespace fast {

struct Piece3 {
  double tlo, thi;
  int cell;
  int kind;
};

// For every voxel iz in [z0, z1) of column (ix, iy): xfn(iz) -> value passed
// through to emit, then
// emit(iz, m_y, m_z, w, value) for each weight w > 1e-16, cells and rows
// clipped to the detector.
template <typename XFn, typename Emit>
__device__ __forceinline__ bool column_weights(const DevGeom& g, double C, double S, int ix,
                                               int iy, int z0, int z1, int* status, XFn&& xfn,
                                               Emit&& emit) {
  const double x0 = (ix - g.n_x / 2.0) * g.a, x1 = x0 + g.a;
  const double y0 = (iy - g.n_y / 2.0) * g.b, y1 = y0 + g.b;
  const double s = g.s;
  Sweep2 sw;
  if (!sweep_setup(g, C, S, x0, x1, y0, y1, status, sw)) return false;
  // canonical frame = low face at y0: kq quarter turns (x, y) -> (y, -x),
  // phi' = phi - kq pi/2 (geometry.cpp:85-91)
  const int kq = sw.low_face;
  double Sp, Cp;
  switch (kq) {
    case 0: Sp = S; Cp = C; break;
    case 1: Sp = -C; Cp = S; break;
    case 2: Sp = -S; Cp = -C; break;
    default: Sp = C; Cp = -S; break;
  }
  double fx0 = x0, fx1 = x1, fy0 = y0, fy1 = y1;
  double ax1 = sw.Ta_x, ay1 = sw.Ta_y, ax4 = sw.Tb_x, ay4 = sw.Tb_y;
  for (int r = 0; r < kq; ++r) {
    const double nx0 = fy0, nx1 = fy1, ny0 = -fx1, ny1 = -fx0;
    fx0 = nx0; fx1 = nx1; fy0 = ny0; fy1 = ny1;
    double t = ax1; ax1 = ay1; ay1 = -t;
    t = ax4; ax4 = ay4; ay4 = -t;
  }
  const double ca = fx1 - fx0, cb = fy1 - fy0;  // canonical pixel sizes
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;

  // pieces (in range cells only) and per-cell 2D weights
  Piece3 pc[kMaxBrk];
  int np = 0;
  int ng = 0, last_end = 0;
  unsigned char gbeg[kMaxBrk], gend[kMaxBrk];
  double gw2d[kMaxBrk];
  bool overflow = false;
  sweep_walk(
      g, C, S, sw,
      [&](int cell, double tlo, double thi, int zone, double) {
        if (cell < cell_lo || cell > cell_hi) return;
        if (np == kMaxBrk) {
          overflow = true;
          return;
        }
        pc[np].tlo = tlo;
        pc[np].thi = thi;
        pc[np].cell = cell;
        pc[np].kind = zone;
        ++np;
      },
      [&](int cell, double acc) {
        if (cell < cell_lo || cell > cell_hi) return;
        if (np > last_end) {
          gbeg[ng] = (unsigned char)last_end;
          gend[ng] = (unsigned char)np;
          gw2d[ng] = acc > 0.0 ? acc : 0.0;
          ++ng;
          last_end = np;
        }
      });
  if (overflow) {
    raise_status(status, CTSM_ERR_TOO_LARGE);
    return false;
  }
  if (ng == 0) return true;
  double inv_depth[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) inv_depth[k] = frcp(sw.D[k]);

  const double sdd = g.sdd;
  const double sdd_dz = sdd / g.d_z;
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  double dmin_inv = inv_depth[0], dmax_inv = inv_depth[0];
#pragma unroll
  for (int k = 1; k < 4; ++k) {
    dmin_inv = fmin(dmin_inv, inv_depth[k]);
    dmax_inv = fmax(dmax_inv, inv_depth[k]);
  }

  auto atom_sum = [&](int pi, int pj, double cz, double tan_a, double zref) {
    double v = 0.0;
    for (int k = pi; k < pj; ++k) {
      switch (pc[k].kind) {
        case 0:
          v += exact::tri_atom(Sp, Cp, s, ca, cb, cz, ax1, ay1, pc[k].thi, tan_a, zref) -
               exact::tri_atom(Sp, Cp, s, ca, cb, cz, ax1, ay1, pc[k].tlo, tan_a, zref);
          break;
        case 1:
          v += exact::trap_atom(Sp, Cp, s, ca, cb, cz, fx0, fx1, pc[k].tlo, pc[k].thi, tan_a, zref);
          break;
        default:
          v += exact::tri_atom(Sp, Cp, s, ca, cb, cz, ax4, ay4, pc[k].tlo, tan_a, zref) -
               exact::tri_atom(Sp, Cp, s, ca, cb, cz, ax4, ay4, pc[k].thi, tan_a, zref);
      }
    }
    return v;
  };

  for (int iz = z0; iz < z1; ++iz) {
    const double xv = xfn(iz);
    const double zb = (iz - g.n_z / 2.0) * g.c, zt = (iz + 1 - g.n_z / 2.0) * g.c;
    const double cz = zt - zb;
    // row magnification range over the 8 corners (weights3d.cpp:365-378)
    const double mb1 = sdd_dz * zb * dmin_inv, mb2 = sdd_dz * zb * dmax_inv;
    const double mt1 = sdd_dz * zt * dmin_inv, mt2 = sdd_dz * zt * dmax_inv;
    const double m_min = fmin(fmin(mb1, mb2), fmin(mt1, mt2));
    const double m_max = fmax(fmax(mb1, mb2), fmax(mt1, mt2));
    const int fl = (int)floor(m_min);
    const int k_lo = (fl < row_lo) ? row_lo : fl;
    const int chi = (int)ceil(m_max) - 1;
    const int k_hi = (chi < row_hi) ? chi : row_hi;
    if (k_hi < k_lo) continue;
    for (int q = 0; q < ng; ++q) {
      const int pi = gbeg[q], pj = gend[q];
      const double w2d = gw2d[q];
      const int cell = pc[pi].cell;
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
          return atom_sum(pi, pj, cz, tan_a, zt) - atom_sum(pi, pj, cz, tan_a, zb);
        }
        const double tan_a = -kk * g.d_z / sdd;
        return w2d - (atom_sum(pi, pj, cz, tan_a, -zb) - atom_sum(pi, pj, cz, tan_a, -zt));
      };
      double prev = above((double)k_lo);
      for (int L = k_lo; L <= k_hi; ++L) {
        const double next = above((double)(L + 1));
        const double v = prev - next;
        if (v > kEpsWeight) emit(iz, cell, L, v, xv);
        prev = next;
      }
    }
  }
  return true;
}

}  // namespace fast
}  // namespace ctsmb
