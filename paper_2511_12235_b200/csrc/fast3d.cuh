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
// through to emit (voxels with value 0 are skipped), then
// emit(iz, m_y, m_z, w, value) for each weight w > 1e-16, cells and rows
// clipped to the detector.
template <typename XFn, typename Emit>
__device__ __forceinline__ bool column_weights(const DevGeom& g, double C, double S, int ix,
                                               int iy, int z0, int z1, int* status, XFn&& xfn,
                                               Emit&& emit) {
  const double x0 = (ix - g.n_x / 2.0) * g.a, x1 = (ix + 1 - g.n_x / 2.0) * g.a;
  const double y0 = (iy - g.n_y / 2.0) * g.b, y1 = (iy + 1 - g.n_y / 2.0) * g.b;
  const double s = g.s;
  Corner c[4];
  const double xs[4] = {x0, x1, x1, x0};
  const double ys[4] = {y0, y0, y1, y1};
  double inv_depth[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double D = s - xs[k] * C - ys[k] * S;
    const double L = ys[k] * C - xs[k] * S;
    if (!(D > kEpsDenRel * s)) {
      raise_status(status, CTSM_ERR_DEGENERATE_GEOMETRY);
      return false;
    }
    c[k].t = fdiv(L, D);
    c[k].D = D;
    c[k].x = xs[k];
    c[k].y = ys[k];
    inv_depth[k] = 1.0 / D;
  }
  int i1 = 0;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (c[k].t < c[i1].t) i1 = k;
  const int na = (i1 + 1) & 3, nb = (i1 + 3) & 3, op = (i1 + 2) & 3;
  const int i2 = (c[na].t <= c[nb].t) ? na : nb;
  const int i3o = (i2 == na) ? nb : na;
  const int i4 = (c[op].t >= c[i3o].t) ? op : i3o;
  const int i3 = (i4 == op) ? i3o : op;
  const double T1 = c[i1].t, T4 = c[i4].t;
  double T2 = c[i2].t, T3 = c[i3].t;
  if (T3 < T2) {
    const double m = 0.5 * (T2 + T3);
    T2 = m;
    T3 = m;
  }
  // low face index: edge (i, i+1 mod 4) is face i (0 bottom, 1 right, 2 top, 3 left)
  const int kq = (i2 == ((i1 + 1) & 3)) ? i1 : i2;
  double Sp, Cp;
  switch (kq) {
    case 0: Sp = S; Cp = C; break;
    case 1: Sp = -C; Cp = S; break;
    case 2: Sp = -S; Cp = -C; break;
    default: Sp = C; Cp = -S; break;
  }
  // canonical frame: k quarter turns (x, y) -> (y, -x)
  double fx0 = x0, fx1 = x1, fy0 = y0, fy1 = y1;
  double ax1 = c[i1].x, ay1 = c[i1].y, ax4 = c[i4].x, ay4 = c[i4].y;
  for (int r = 0; r < kq; ++r) {
    const double nx0 = fy0, nx1 = fy1, ny0 = -fx1, ny1 = -fx0;
    fx0 = nx0; fx1 = nx1; fy0 = ny0; fy1 = ny1;
    double t = ax1; ax1 = ay1; ay1 = -t;
    t = ax4; ax4 = ay4; ay4 = -t;
  }
  const double ca = fx1 - fx0, cb = fy1 - fy0;  // canonical pixel sizes

  // 2D pieces (fast2d.cuh area forms)
  const bool low_horizontal = (c[i1].y == c[i2].y);
  const double inv2ab = 1.0 / (2.0 * g.a * g.b);
  const double K1 = c[i1].D * c[i1].D * inv2ab;
  const double K4 = c[i4].D * c[i4].D * inv2ab;
  const double band_k = low_horizontal ? fabs(s * C - 0.5 * (x0 + x1)) / g.b
                                       : fabs(s * S - 0.5 * (y0 + y1)) / g.a;
  auto tri_den = [&](double t) { return fabs((C + t * S) * (t * C - S)); };
  auto band_p = [&](double t) { return low_horizontal ? (C + t * S) : (t * C - S); };

  const double inv_scale = g.d_y / g.sdd;
  const double scl = g.sdd / g.d_y;
  const long long e_lo = (long long)floor(T1 * scl) + 1;
  const long long e_hi = (long long)ceil(T4 * scl) - 1;
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;

  Piece3 pc[kMaxBrk];
  int np = 0;
  {
    const double zt4[4] = {T1, T2, T3, T4};
    int zi = 1;
    long long e = e_lo;
    int cell = (int)(e_lo - 1);
    double tlo = T1;
    while (true) {
      const bool have_e = (e <= e_hi);
      const double te = have_e ? e * inv_scale : 0.0;
      double thi;
      bool is_edge;
      if (zi < 4 && (!have_e || !(te < zt4[zi]))) {
        thi = zt4[zi];
        is_edge = false;
      } else if (have_e) {
        thi = te;
        is_edge = true;
      } else {
        break;
      }
      if (thi > tlo && cell >= cell_lo && cell <= cell_hi) {
        if (np == kMaxBrk) {
          raise_status(status, CTSM_ERR_TOO_LARGE);
          return false;
        }
        pc[np].tlo = tlo;
        pc[np].thi = thi;
        pc[np].cell = cell;
        pc[np].kind = (thi <= T2) ? 0 : ((tlo >= T3) ? 2 : 1);
        ++np;
      }
      tlo = thi;
      if (is_edge) {
        ++cell;
        ++e;
      } else {
        ++zi;
      }
    }
  }
  if (np == 0) return true;
  // cell groups and their 2D weights
  int ng = 0;
  unsigned char gbeg[kMaxBrk], gend[kMaxBrk];
  double gw2d[kMaxBrk];
  for (int i = 0; i < np;) {
    int j = i;
    double w2d = 0.0;
    while (j < np && pc[j].cell == pc[i].cell) {
      const double tl = pc[j].tlo, th = pc[j].thi;
      double w;
      if (pc[j].kind == 0) {
        const double dh = th - T1, dl = tl - T1;
        w = (dh == 0.0 ? 0.0 : K1 * dh * dh / tri_den(th)) - (dl == 0.0 ? 0.0 : K1 * dl * dl / tri_den(tl));
      } else if (pc[j].kind == 2) {
        const double dh = T4 - th, dl = T4 - tl;
        w = (dl == 0.0 ? 0.0 : K4 * dl * dl / tri_den(tl)) - (dh == 0.0 ? 0.0 : K4 * dh * dh / tri_den(th));
      } else {
        w = (th - tl) * band_k / fabs(band_p(tl) * band_p(th));
      }
      w2d += w;
      ++j;
    }
    gbeg[ng] = (unsigned char)i;
    gend[ng] = (unsigned char)j;
    gw2d[ng] = w2d > 0.0 ? w2d : 0.0;
    ++ng;
    i = j;
  }

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
    if (xv == 0.0) continue;
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
