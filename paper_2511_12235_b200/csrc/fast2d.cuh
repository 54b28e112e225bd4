// fast2d.cuh -- transcendental-free evaluation of the 2D consistent weights
// (pixel area fractions per detector cell) for the matrix-free projectors.
//
// Same quantity as pixel_area_factors (weights2d.cpp:105-129), reformulated
// in the ray parameter t = tan(beta) (fan-angle tangent; detector coordinate
// e_y = t (s+d) / d_y):
//  * a point (x, y) projects to t = L / D with lateral L = y cos(phi) -
//    x sin(phi) and depth D = s - x cos(phi) - y sin(phi) (geometry.cpp:56-62);
//    t is invariant under the quarter-turn canonicalisation, so no frame
//    search (geometry.cpp:76-97) and no atan2 are needed: the "low" face (the
//    canonical y0 face) is the face whose larger corner t is smallest;
//  * detector edge e sits at t_e = e d_y / (s+d) exactly (no atan/tan pair);
//  * the corner-triangle area cut from apex corner (xa, ya) by the ray t
//    (paper A3, weights2d.cpp:8-16) is the cumulative
//        A(t) = Da^2 (t - ta)^2 / (2 a b |(C + t S)(t C - S)|),
//    and the band between rays t1 < t2 crossing both faces x = x0, x1
//    (paper A4, weights2d.cpp:19-27) is
//        |(t2 - t1)(s C - xm)| / (b |(C + t1 S)(C + t2 S)|)
//    (faces y = y0, y1: |(t2 - t1)(s S - ym)| / (a |(t1 C - S)(t2 C - S)|)).
// These are algebraically identical to the reference's sine/tangent forms.
// Each breakpoint costs one reciprocal; cumulative areas are carried from one
// piece to the next, so a pixel-angle needs no transcendental and ~10
// reciprocals. Results agree with the reference to ~1e-13 (tests check the
// 1e-10 fp64 tolerance against the oracle).
#pragma once
#include "common.cuh"

namespace ctsmb {
namespace fast {

// 1/x to ~1 ulp: hardware approximation + two Newton steps.
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Division used by the 3D atoms in the matrix-free path.
__device__ __forceinline__ double fdiv(double a, double b) { return a * frcp(b); }

// The sweep of one pixel at one angle in t-space (shared by 2D and 3D).
struct Sweep2 {
  double T1, T2, T3, T4;   // sorted corner parameters (T1 apex-low, T4 apex-high)
  double K1, K4;           // Da^2 / (2ab) of the two apex corners
  double band_k;           // |s C - xm| / b  or  |s S - ym| / a
  bool band_vertical;      // band crosses x = const faces (low face horizontal)
  int low_face;            // 0 bottom (y0), 1 right (x1), 2 top (y1), 3 left (x0)
  double Ta_x, Ta_y, Tb_x, Tb_y;  // apex-low / apex-high corner coordinates
  double D[4];             // corner depths (0 (x0,y0), 1 (x1,y0), 2 (x1,y1), 3 (x0,y1))
};

__device__ __forceinline__ bool sweep_setup(const DevGeom& g, double C, double S, double x0,
                                            double x1, double y0, double y1, int* status,
                                            Sweep2& w) {
  const double s = g.s;
  const double x0C = x0 * C, x1C = x1 * C, x0S = x0 * S, x1S = x1 * S;
  const double y0C = y0 * C, y1C = y1 * C, y0S = y0 * S, y1S = y1 * S;
  const double D0 = s - x0C - y0S, D1 = s - x1C - y0S, D2 = s - x1C - y1S, D3 = s - x0C - y1S;
  const double dmin = fmin(fmin(D0, D1), fmin(D2, D3));
  if (!(dmin > kEpsDenRel * s)) {
    raise_status(status, CTSM_ERR_DEGENERATE_GEOMETRY);
    return false;
  }
  w.D[0] = D0; w.D[1] = D1; w.D[2] = D2; w.D[3] = D3;
  // corner parameters; corners 0 (x0,y0), 1 (x1,y0), 2 (x1,y1), 3 (x0,y1)
  double ta = (y0C - x0S) * frcp(D0), tb = (y0C - x1S) * frcp(D1);
  double tc = (y1C - x1S) * frcp(D2), td = (y1C - x0S) * frcp(D3);
  double Da = D0, Db = D1, Dc = D2, Dd = D3;
  int ia = 0, ib = 1, ic = 2, id = 3;
  // 5-comparator sorting network on t, carrying depth and corner index
  auto ce = [](double& t0, double& t1, double& d0, double& d1, int& i0, int& i1) {
    const bool sw = t1 < t0;
    const double tt = sw ? t1 : t0, tu = sw ? t0 : t1;
    const double dd = sw ? d1 : d0, du = sw ? d0 : d1;
    const int ii = sw ? i1 : i0, iu = sw ? i0 : i1;
    t0 = tt; t1 = tu; d0 = dd; d1 = du; i0 = ii; i1 = iu;
  };
  ce(ta, tb, Da, Db, ia, ib);
  ce(tc, td, Dc, Dd, ic, id);
  ce(ta, tc, Da, Dc, ia, ic);
  ce(tb, td, Db, Dd, ib, id);
  ce(tb, tc, Db, Dc, ib, ic);
  // the two smallest corners must share a face (the canonical y0 face); at a
  // rounding-level tie they can come out diagonal: then the third-smallest
  // corner (a neighbour of the smallest) takes the second place.
  if ((ia ^ ib) == 2) {
    const double t = tb; tb = tc; tc = t;
    const int i = ib; ib = ic; ic = i;
  }
  w.T1 = ta;
  w.T2 = tb;
  w.T3 = tc;
  w.T4 = td;
  w.K1 = Da * Da * g.inv_2ab;
  w.K4 = Dd * Dd * g.inv_2ab;
  // low face: horizontal iff its corners share y (indices {0,1} or {2,3})
  const bool horiz = (ia >> 1) == (ib >> 1);
  w.band_vertical = horiz;
  w.low_face = horiz ? ((ia >> 1) == 0 ? 0 : 2) : ((ia == 1 || ia == 2) ? 1 : 3);
  w.Ta_x = (ia == 1 || ia == 2) ? x1 : x0;
  w.Ta_y = (ia >= 2) ? y1 : y0;
  w.Tb_x = (id == 1 || id == 2) ? x1 : x0;
  w.Tb_y = (id >= 2) ? y1 : y0;
  w.band_k = horiz ? fabs(s * C - 0.5 * (x0 + x1)) * g.inv_b
                   : fabs(s * S - 0.5 * (y0 + y1)) * g.inv_a;
  return true;
}

// Walks the pieces of the sweep in ascending t; calls
// piece(cell, tlo, thi, kind, w2d) for every piece of positive width and
// cell_done(cell, w) when a detector cell is complete (w = its area weight,
// possibly 0). Cells are not clipped here.
template <typename Piece, typename CellDone>
__device__ __forceinline__ void sweep_walk(const DevGeom& g, double C, double S, const Sweep2& w,
                                           Piece&& piece, CellDone&& cell_done) {
  const double scale = g.u_scale;
  const double inv_scale = g.t_scale;
  const double T1 = w.T1, T2 = w.T2, T3 = w.T3, T4 = w.T4;
  const int e_lo = (int)floor(T1 * scale) + 1;
  const int e_hi = (int)ceil(T4 * scale) - 1;
  int cell = e_lo - 1;
  const bool bv = w.band_vertical;
  // A ray parallel to a pixel face makes a factor vanish; the reference then
  // returns 0 for the triangle (|sin(beta - phi)| < 1e-12, weights2d.cpp:11)
  // and such a ray bounds no band piece (weights2d.cpp:22-23): guard likewise.
  auto pq_inv = [&](double t) {
    const double v = fabs((C + t * S) * (t * C - S));
    return v > kEpsAngle ? frcp(v) : 0.0;
  };
  auto p_inv = [&](double t) {
    const double v = fabs(bv ? (C + t * S) : (t * C - S));
    return v > kEpsAngle ? frcp(v) : 0.0;
  };
  // zone of the upcoming piece: 0 low triangle, 1 band, 2 high triangle
  int zone;
  double Aprev = 0.0, ipprev = 0.0;
  if (T1 < T2) {
    zone = 0;
  } else if (T2 < T3) {
    zone = 1;
    ipprev = p_inv(T1);
  } else {
    zone = 2;
    const double d = T4 - T1;
    Aprev = w.K4 * d * d * pq_inv(T1);
  }
  double prev = T1;
  double acc = 0.0;
  int zi = 1;  // next corner: 1 -> T2, 2 -> T3, 3 -> T4
  int e = e_lo;
  while (zi <= 3) {
    const double tz = zi == 1 ? T2 : (zi == 2 ? T3 : T4);
    const bool have_e = e <= e_hi;
    const double te = e * inv_scale;
    const bool is_edge = have_e && te < tz;
    const double b = is_edge ? te : tz;
    if (b > prev) {
      double wv;
      if (zone == 0) {
        const double d = b - T1;
        const double A = w.K1 * d * d * pq_inv(b);
        wv = A - Aprev;
        Aprev = A;
      } else if (zone == 1) {
        const double ip = p_inv(b);
        wv = w.band_k * (b - prev) * (ipprev * ip);
        ipprev = ip;
      } else {
        const double d = T4 - b;
        const double A = w.K4 * d * d * pq_inv(b);
        wv = Aprev - A;
        Aprev = A;
      }
      if (wv > 0.0) {
        acc += wv;
        piece(cell, prev, b, zone, wv);
      }
      prev = b;
    }
    if (is_edge) {
      cell_done(cell, acc);
      acc = 0.0;
      ++cell;
      ++e;
    } else {
      if (zi == 1) {  // leaving the low triangle
        if (T2 < T3) {
          zone = 1;
          ipprev = p_inv(T2);
        } else {
          zone = 2;
          const double d = T4 - T2;
          Aprev = w.K4 * d * d * pq_inv(T2);
        }
      } else if (zi == 2 && zone == 1) {  // leaving the band
        zone = 2;
        const double d = T4 - T3;
        Aprev = w.K4 * d * d * pq_inv(T3);
      }
      ++zi;
    }
  }
  cell_done(cell, acc);
}

// Streams the cell weights of pixel (ix, iy) at an angle with cos/sin (C, S)
// to emit(cell_m, w) in ascending cell order; cells outside the detector are
// skipped (weights2d.cpp:110-113), as are weights <= 1e-16 (125-127).
//
// Cell weights are differences of the cumulative area CA(t) (fraction of the
// pixel with ray parameter < t):
//   CA = A1(t)                             T1 <= t <= T2  (low corner triangle)
//      = A1(T2) + band(T2, t)              T2 <= t <= T3
//      = A1(T2) + band(T2, T3) + A4(T3) - A4(t)   T3 <= t <= T4
// so every detector edge costs one independent reciprocal (good ILP) and the
// zone constants four more.
template <typename Emit>
__device__ __forceinline__ bool pixel_weights(const DevGeom& g, double C, double S, int ix,
                                              int iy, int* status, Emit&& emit) {
  const double x0 = (ix - g.n_x / 2.0) * g.a, x1 = x0 + g.a;
  const double y0 = (iy - g.n_y / 2.0) * g.b, y1 = y0 + g.b;
  Sweep2 w;
  if (!sweep_setup(g, C, S, x0, x1, y0, y1, status, w)) return false;
  const double T1 = w.T1, T2 = w.T2, T3 = w.T3, T4 = w.T4;
  const bool bv = w.band_vertical;
  auto pq_inv = [&](double t) {
    const double v = fabs((C + t * S) * (t * C - S));
    return v > kEpsAngle ? frcp(v) : 0.0;
  };
  auto p_inv = [&](double t) {
    const double v = fabs(bv ? (C + t * S) : (t * C - S));
    return v > kEpsAngle ? frcp(v) : 0.0;
  };
  // zone constants (independent reciprocals)
  const double d12 = T2 - T1, d34 = T4 - T3, d23 = T3 - T2;
  const double A1T2 = d12 > 0.0 ? w.K1 * d12 * d12 * pq_inv(T2) : 0.0;
  const double A4T3 = d34 > 0.0 ? w.K4 * d34 * d34 * pq_inv(T3) : 0.0;
  const double ipT2 = d23 > 0.0 ? p_inv(T2) : 0.0;
  const double bandT = d23 > 0.0 ? w.band_k * d23 * ipT2 * p_inv(T3) : 0.0;
  const double base2 = A1T2 + bandT + A4T3;  // CA(T4) (== 1 up to rounding)
  // (a branch-free form -- one shared reciprocal, the zone's constant and
  // factor picked by selects -- was neutral: C1 1.705 vs 1.710 ms per step)
  auto CA = [&](double t) -> double {
    if (t <= T2) {
      const double d = t - T1;
      return d > 0.0 ? w.K1 * d * d * pq_inv(t) : 0.0;
    }
    if (t < T3) return A1T2 + w.band_k * (t - T2) * ipT2 * p_inv(t);
    const double d = T4 - t;
    return base2 - (d > 0.0 ? w.K4 * d * d * pq_inv(t) : 0.0);
  };
  const double scale = g.u_scale;
  const double inv_scale = g.t_scale;
  // |t| * scale is bounded by the edge-table extent (dev_geom), so 32-bit
  // edge indices suffice (cheaper int <-> double conversions)
  const int e_lo = (int)floor(T1 * scale) + 1;
  const int e_hi = (int)ceil(T4 * scale) - 1;
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  double prev = 0.0;  // CA(T1)
  int cell = e_lo - 1;
#pragma unroll 2
  for (int e = e_lo; e <= e_hi; ++e, ++cell) {
    const double cur = CA(e * inv_scale);  // CA clamps outside [T1, T4]
    const double wv = cur - prev;
    prev = cur;
    if (wv > kEpsWeight && cell >= cell_lo && cell <= cell_hi) emit(cell, wv);
  }
  const double wv = base2 - prev;
  if (wv > kEpsWeight && cell >= cell_lo && cell <= cell_hi) emit(cell, wv);
  return true;
}

}  // namespace fast
}  // namespace ctsmb
