// fast2d.cuh -- transcendental-free evaluation of the 2D consistent weights
// (pixel area fractions per detector cell) for the matrix-free projectors.
//
// Same quantity as pixel_area_factors (weights2d.cpp:105-129), reformulated
// in the ray parameter t = tan(beta) (fan-angle tangent, detector coordinate
// e_y = t (s+d) / d_y):
//  * a point (x, y) projects to t = L / D with lateral L = y cos(phi) -
//    x sin(phi) and depth D = s - x cos(phi) - y sin(phi) (geometry.cpp:56-62);
//    t is invariant under the quarter-turn canonicalisation, so no frame
//    search (geometry.cpp:76-97) and no atan2 are needed;
//  * detector edge e sits at t_e = e d_y / (s+d) exactly (no atan/tan pair);
//  * the corner-triangle area cut from apex corner (xa, ya) by the ray t
//    (paper A3, weights2d.cpp:8-16) is
//        A(t) = Da^2 (t - ta)^2 / (2 a b |(C + t S)(t C - S)|),
//    and the band between rays t1 < t2 crossing both faces x = x0, x1
//    (paper A4, weights2d.cpp:19-27) is
//        |(t2 - t1)(s C - xm)| / (b |(C + t1 S)(C + t2 S)|)
//    (faces y = y0, y1: |(t2 - t1)(s S - ym)| / (a |(t1 C - S)(t2 C - S)|)).
// These are algebraically identical to the reference's sine/tangent forms;
// results agree with the reference to ~1e-13 (checked by tests against the
// oracle at the 1e-10 fp64 tolerance).
#pragma once
#include "common.cuh"

namespace ctsmb {
namespace fast {

// Division in the matrix-free kernels: IEEE double division (the compiler's
// sequence). Kept in one place so it can be swapped for a reciprocal scheme.
__device__ __forceinline__ double fdiv(double a, double b) { return a / b; }

struct Corner {
  double t, D;
  double x, y;
};

// Streams the cell weights of pixel (ix, iy) at an angle with cos/sin (C, S)
// to emit(cell_m, w) in ascending cell order; cells outside the detector are
// skipped (weights2d.cpp:110-113), as are weights <= 0. Returns false and
// raises status on degenerate geometry.
template <typename Emit>
__device__ __forceinline__ bool pixel_weights(const DevGeom& g, double C, double S, int ix,
                                              int iy, int* status, Emit&& emit) {
  const double x0 = (ix - g.n_x / 2.0) * g.a, x1 = (ix + 1 - g.n_x / 2.0) * g.a;
  const double y0 = (iy - g.n_y / 2.0) * g.b, y1 = (iy + 1 - g.n_y / 2.0) * g.b;
  const double s = g.s;
  // corners counter-clockwise: 0 (x0,y0), 1 (x1,y0), 2 (x1,y1), 3 (x0,y1)
  Corner c[4];
  const double xs[4] = {x0, x1, x1, x0};
  const double ys[4] = {y0, y0, y1, y1};
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
  }
  // apex1 = corner with the smallest t; the low face joins it to its
  // neighbour with the smaller t; the high face is the opposite face.
  int i1 = 0;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (c[k].t < c[i1].t) i1 = k;
  const int na = (i1 + 1) & 3, nb = (i1 + 3) & 3, op = (i1 + 2) & 3;
  const int i2 = (c[na].t <= c[nb].t) ? na : nb;   // low-face partner
  const int i3o = (i2 == na) ? nb : na;            // remaining neighbour (high face)
  // high face = {op, i3o}
  const int i4 = (c[op].t >= c[i3o].t) ? op : i3o;
  const int i3 = (i4 == op) ? i3o : op;
  const double T1 = c[i1].t, T4 = c[i4].t;
  double T2 = c[i2].t, T3 = c[i3].t;
  if (T3 < T2) {  // rounding-level inconsistency at degenerate alignments
    const double m = 0.5 * (T2 + T3);
    T2 = m;
    T3 = m;
  }
  // low face horizontal (corners share y) -> band crosses the x = const faces
  const bool low_horizontal = (c[i1].y == c[i2].y);
  const double inv2ab = 1.0 / (2.0 * g.a * g.b);
  const double K1 = c[i1].D * c[i1].D * inv2ab;
  const double K4 = c[i4].D * c[i4].D * inv2ab;
  double band_k;  // band = (t2 - t1) * band_k / |p(t1) p(t2)|
  if (low_horizontal)
    band_k = fabs(s * C - 0.5 * (x0 + x1)) / g.b;
  else
    band_k = fabs(s * S - 0.5 * (y0 + y1)) / g.a;

  // cumulative-area helpers at a breakpoint t
  auto tri_den = [&](double t) { return fabs((C + t * S) * (t * C - S)); };
  auto band_p = [&](double t) { return low_horizontal ? (C + t * S) : (t * C - S); };

  // detector edges strictly inside (T1, T4)
  const double scale = g.sdd / g.d_y;   // t -> edge coordinate
  const double inv_scale = g.d_y / g.sdd;
  const double u_lo = T1 * scale, u_hi = T4 * scale;
  const long long e_lo = (long long)floor(u_lo) + 1;
  const long long e_hi = (long long)ceil(u_hi) - 1;
  int cell = (int)(e_lo - 1);
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;

  // walk merged breakpoints: corners T1 < T2 <= T3 < T4 and edges
  const double zt[4] = {T1, T2, T3, T4};
  int zi = 1;               // next corner breakpoint index (T1 is the start)
  long long e = e_lo;
  double tlo = T1;
  double acc = 0.0;         // current cell weight
  while (true) {
    const double te = (e <= e_hi) ? e * inv_scale : 0.0;
    const bool have_e = (e <= e_hi);
    double thi;
    bool is_edge;
    if (zi < 4 && (!have_e || !(te < zt[zi]))) {
      thi = zt[zi];
      is_edge = false;
    } else if (have_e) {
      thi = te;
      is_edge = true;
    } else {
      break;
    }
    if (thi > tlo) {
      // zone of the piece [tlo, thi]: 0 if thi <= T2, 2 if tlo >= T3, else band
      double w;
      if (thi <= T2) {
        const double dh = thi - T1, dl = tlo - T1;
        const double ah = dh == 0.0 ? 0.0 : fdiv(K1 * dh * dh, tri_den(thi));
        const double al = dl == 0.0 ? 0.0 : fdiv(K1 * dl * dl, tri_den(tlo));
        w = ah - al;
      } else if (tlo >= T3) {
        const double dh = T4 - thi, dl = T4 - tlo;
        const double ah = dh == 0.0 ? 0.0 : fdiv(K4 * dh * dh, tri_den(thi));
        const double al = dl == 0.0 ? 0.0 : fdiv(K4 * dl * dl, tri_den(tlo));
        w = al - ah;
      } else {
        w = fdiv((thi - tlo) * band_k, fabs(band_p(tlo) * band_p(thi)));
      }
      if (w > 0.0) acc += w;
    }
    tlo = thi;
    if (is_edge) {
      if (acc > 0.0 && cell >= cell_lo && cell <= cell_hi) emit(cell, acc);
      acc = 0.0;
      ++cell;
      ++e;
    } else {
      ++zi;
    }
  }
  if (acc > 0.0 && cell >= cell_lo && cell <= cell_hi) emit(cell, acc);
  return true;
}

}  // namespace fast
}  // namespace ctsmb
