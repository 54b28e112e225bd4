// atoms.cuh -- the reference's closed-form 3D volume atoms as pure device
// functions of (sin phi', cos phi', tan beta, tan alpha, zref) in the
// canonical frame. Shared by the bit-exact CSR kernels (compiled with
// -fmad=false, exact.cuh) and the matrix-free kernels (fast3d.cuh).
#pragma once
#include "common.cuh"

namespace ctsmb {
namespace exact {

__device__ __forceinline__ double cube(double v) { return v * v * v; }
__device__ __forceinline__ double sq(double v) { return v * v; }

// ---- 3D atoms (weights3d.cpp:51-168); S, C, tan(beta) supplied ------------

// trap_face_part (weights3d.cpp:51-61)
__device__ __forceinline__ double trap_face_part(double G, double P, double S, double t1,
                                                 double t2, double cr1, double cr2, int flag1,
                                                 int flag2) {
  if (flag1 && flag2)
    return (t1 - t2) *
           (cube(G) - 3.0 * G * P * P / (cr1 * cr2) + cube(P) * (cr1 + cr2) / sq(cr1 * cr2));
  if (!flag1 && !flag2) return 0.0;
  double v = 0.0;
  if (flag1) v += cr1 * cube(G - P / cr1);
  if (flag2) v -= cr2 * cube(G - P / cr2);
  return v / S;
}

// detail::trap_atom = trap_flags_at + trap_atom_flags (weights3d.cpp:63-107, 176-183)
__device__ __forceinline__ double trap_atom(double S, double C, double s, double a, double b,
                                            double c, double x0, double x1, double t1,
                                            double t2, double tan_a, double zref) {
  const double G = zref / (a * tan_a);
  if (fabs(S) > kEpsSingular) {
    const double cr1 = C + S * t1, cr2 = C + S * t2;
    const double Pg = (s * C - x1) / a, Pf = (s * C - x0) / a;
    const int g1 = (G - Pg / cr1) > 0.0;
    const int g2 = (G - Pg / cr2) > 0.0;
    const int f1 = (G - Pf / cr1) > 0.0;
    const int f2 = (G - Pf / cr2) > 0.0;
    const double pg = trap_face_part(G, Pg, S, t1, t2, cr1, cr2, g1, g2);
    const double pf = trap_face_part(G, Pf, S, t1, t2, cr1, cr2, f1, f2);
    return (a * a / (6.0 * b * c)) * fabs(tan_a * (pg - pf));
  }
  const int gs = (G - (s * C - x1) / a) > 0.0;
  const int fs = (G - (s * C - x0) / a) > 0.0;
  const double gv = G - (s * C - x1) / a;
  const double fv = G - (s * C - x0) / a;
  double t = 0.0;
  if (gs) t += gv * gv * (gv + 3.0 * (s * C - x1) / a);
  if (fs) t -= fv * fv * (fv + 3.0 * (s * C - x0) / a);
  return (a * a / (6.0 * b * c)) * fabs(tan_a * t * (t1 - t2));
}

// detail::tri_atom_cum = tri_flags_at + tri_atom_flags (weights3d.cpp:115-168, 185-190)
__device__ __forceinline__ double tri_atom(double S, double C, double s, double a, double b,
                                           double c, double xa, double ya, double t, double tan_a,
                                           double zref) {
  const double G = zref / (a * tan_a);
  const double crg = C + S * t;
  const double srh = S - C * t;
  const double P = (s * C - xa) / a;
  const double Q = (s * S - ya) / a;
  const double g = G - P / crg;
  const double gg = G - P * C - Q * S;
  const double h = G - Q / srh;
  const int fg = g > 0.0, fgg = gg > 0.0, fh = h > 0.0;
  if (fabs(S) > kEpsSingular) {
    double pair;
    if (fg && fgg) {
      const double delta = Q - P * srh / crg;
      pair = crg * (3.0 * gg * gg * delta + 3.0 * gg * S * delta * delta + S * S * cube(delta)) -
             cube(gg) * srh / C;
    } else if (!fg && !fgg) {
      pair = 0.0;
    } else {
      double v = 0.0;
      if (fg) v += crg * cube(g);
      if (fgg) v -= cube(gg) / C;
      pair = v / S;
    }
    const double tt = pair + (fh ? (srh / C) * cube(h) : 0.0);
    return (a * a / (6.0 * b * c)) * fabs(tan_a * tt);
  }
  double tv = 0.0;
  if (fg) tv += g * g * (t * g - 3.0 * t * (g - h));
  if (fh) tv -= t * cube(h);
  return (a * a / (6.0 * b * c)) * fabs(tan_a * tv);
}

}  // namespace exact
}  // namespace ctsmb
