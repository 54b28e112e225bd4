// fast3dw.cuh -- matrix-free evaluation of the 3D consistent weights (voxel
// volume fractions per detector cell), warp-cooperative along a voxel column.
//
// Same quantity as voxel_volume_factors (weights3d.cpp:354-462):
//  * the xy sweep (weights2d.cpp:38-87) does not depend on iz; it is done once
//    per (column, angle) in the ray parameter t = tan(beta) (fast2d.cuh);
//  * the canonical quarter-turn frame (geometry.cpp:76-97) is the one whose
//    y0 face is the "low" face; phi' = phi - k pi/2 gives
//    (sin, cos) = (S, C), (-C, S), (-S, -C), (C, -S);
//  * the z composition (weights3d.cpp:380-458) uses the reference's closed-form
//    trapezoid / corner-triangle atoms (weights3d.cpp:51-168), keeping their
//    cancellation-safe branch forms, with tan(beta) = t exactly. Every
//    quantity of an atom that does not depend on the plane height G is
//    precomputed once per (column, angle, piece) -- by one lane per piece --
//    into shared memory; per voxel an atom costs three subtractions, the flag
//    tests and a cubic.
#pragma once
#include <climits>

#include "common.cuh"
#include "fast2d.cuh"

namespace ctsmb {
namespace fast {

constexpr int kMaxPieces = 12;  // pieces of one column sweep inside the detector

// G-independent coefficients of one sweep piece (24 doubles).
//  kind 0/2 (corner triangle, atoms at the two endpoints lo/hi):
//    c[0..6]   = lo: th_g, th_gg, th_h, crg, delta, srh_C, t
//    c[7..13]  = hi: same
//    c[14..17] = lo: th_min, th_max, slope, root   (linear / zero short cuts)
//    c[18..21] = hi: same
//  kind 1 (trapezoid band between t1 = lo and t2 = hi):
//    c[0..12]  = th_g1, th_g2, th_f1, th_f2, cr1, cr2, d12, A2g, A3g, A2f, A3f, Pg, Pf
//    c[14..17] = th_min, th_max, slope, root
// An atom's flags test the row-edge plane against zref at the vertices of the
// atom's 2D region (weights3d.cpp:72-75, 123-125). With every flag set the
// plane lies below zref over the whole region and the atom is exactly linear:
// atom = Area (zref - tan_a D_centroid) / (a b c), i.e. tt = slope (G - root)
// with slope = 6 Area / a^2, root = D_centroid / a; with no flag set it is 0.
// Only mixed flags need the reference's cubic forms.
constexpr int kCoef = 24;
constexpr int kLin = 14;
struct alignas(32) PieceCoef {
  double c[kCoef];
};

struct alignas(32) ColumnHead {
  double S, C, invS, invC, kappa;  // canonical sin/cos of phi', 1/S, 1/C, a'^2/(6 b' c)
  double inv_a;                    // 1 / a' (G = zref / (a' tan_a))
  double dmin_inv, dmax_inv;       // extremes of 1/depth over the 4 xy corners
  int flat;                        // |S| <= 1e-8: flat-source branch (weights3d.cpp:68, 142)
  int np, ng;
  int pkind[kMaxPieces];
  int gcell[kMaxPieces];
  unsigned char gbeg[kMaxPieces], gend[kMaxPieces];
  double gw2d[kMaxPieces];
  // per cell group: every atom of the group is zero for G <= gmin and linear
  // for G > gmax, where the group sum is galpha * G - gbeta
  double gmin[kMaxPieces], gmax[kMaxPieces], galpha[kMaxPieces], gbeta[kMaxPieces];
};

__device__ __forceinline__ double cube3(double v) { return v * v * v; }

// Corner-triangle atom from precomputed coefficients (tri_atom_flags,
// weights3d.cpp:129-168), without the kappa*|tan_a| factor.
__device__ __forceinline__ double tri_tt(const ColumnHead& h, const double* c, double G) {
  const double g = G - c[0], gg = G - c[1], hh = G - c[2];
  const bool fg = g > 0.0, fgg = gg > 0.0, fh = hh > 0.0;
  if (!h.flat) {
    double pair;
    if (fg && fgg) {
      const double crg = c[3], d = c[4], S = h.S;
      pair = crg * (3.0 * gg * gg * d + 3.0 * gg * S * d * d + S * S * cube3(d)) - cube3(gg) * c[5];
    } else if (!fg && !fgg) {
      pair = 0.0;
    } else {
      double v = 0.0;
      if (fg) v += c[3] * cube3(g);
      if (fgg) v -= cube3(gg) * h.invC;
      pair = v * h.invS;
    }
    return pair + (fh ? c[5] * cube3(hh) : 0.0);
  }
  const double t = c[6];
  double tv = 0.0;
  if (fg) tv += g * g * (t * g - 3.0 * t * (g - hh));
  if (fh) tv -= t * cube3(hh);
  return tv;
}

// Trapezoid atom (trap_face_part / trap_atom_flags, weights3d.cpp:51-107),
// without the kappa*|tan_a| factor.
__device__ __forceinline__ double trap_tt(const ColumnHead& h, const double* c, double G) {
  if (!h.flat) {
    auto face = [&](double th1, double th2, double A2, double A3) -> double {
      const bool f1 = G - th1 > 0.0, f2 = G - th2 > 0.0;
      if (f1 && f2) return c[6] * (cube3(G) - G * A2 + A3);
      if (!f1 && !f2) return 0.0;
      double v = 0.0;
      if (f1) v += c[4] * cube3(G - th1);
      if (f2) v -= c[5] * cube3(G - th2);
      return v * h.invS;
    };
    return face(c[0], c[1], c[7], c[8]) - face(c[2], c[3], c[9], c[10]);
  }
  const double gv = G - c[11], fv = G - c[12];
  double t = 0.0;
  if (gv > 0.0) t += gv * gv * (gv + 3.0 * c[11]);
  if (fv > 0.0) t -= fv * fv * (fv + 3.0 * c[12]);
  return t * c[6];
}

// Plans one (column, angle). Warp-cooperative form (kSerial = false): every
// lane of the warp computes the sweep (identical), lane j computes piece j's
// coefficients into P[j]; lane 0 writes the head; the caller must
// __syncwarp() before reading H / P. Serial form (kSerial = true, lane = 0):
// one thread does all of it -- used by plan3d_fast_kernel, which plans a
// whole launch's (column, base angle) pairs one per thread, so the sweep is
// computed once instead of by all 32 lanes of the projection kernel's warp.
template <bool kSerial = false>
__device__ __forceinline__ bool plan_column(const DevGeom& g, double C, double S, int ix, int iy,
                                            int* status, ColumnHead& H, PieceCoef* P,
                                            int lane) {
  const double x0 = (ix - g.n_x / 2.0) * g.a, x1 = x0 + g.a;
  const double y0 = (iy - g.n_y / 2.0) * g.b, y1 = y0 + g.b;
  const double s = g.s;
  Sweep2 sw;
  if (!sweep_setup(g, C, S, x0, x1, y0, y1, status, sw)) {
    if (lane == 0) {
      H.np = 0;
      H.ng = 0;
    }
    return false;
  }
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
  const double ca = fx1 - fx0, cb = fy1 - fy0;
  const int cell_lo = -g.n_det_y / 2, cell_hi = g.n_det_y / 2 - 1;
  int np = 0, ng = 0, last_end = 0;
  double my_lo = 0.0, my_hi = 0.0;
  int my_kind = -1;
  // serial form: nothing is read back from H / P (global memory there): the
  // piece bounds stay in thread-local arrays, kinds and group ends in packed
  // registers, and the group aggregates are accumulated while the pieces are
  // computed (same order as the warp form's per-group loop)
  double all_lo[kSerial ? kMaxPieces : 1], all_hi[kSerial ? kMaxPieces : 1];
  unsigned kinds = 0;             // 2 bits per piece
  unsigned long long gends = 0;   // 4 bits per group
  bool overflow = false;
  sweep_walk(
      g, C, S, sw,
      [&](int cell, double tlo, double thi, int zone, double) {
        if (cell < cell_lo || cell > cell_hi) return;
        if (np == kMaxPieces) {
          overflow = true;
          return;
        }
        if (kSerial) {
          all_lo[np] = tlo;
          all_hi[np] = thi;
          kinds |= (unsigned)zone << (2 * np);
        } else if (lane == np) {
          my_lo = tlo;
          my_hi = thi;
          my_kind = zone;
        }
        if (lane == 0) H.pkind[np] = zone;
        ++np;
      },
      [&](int cell, double acc) {
        if (cell < cell_lo || cell > cell_hi) return;
        if (np > last_end) {
          if (lane == 0) {
            H.gbeg[ng] = (unsigned char)last_end;
            H.gend[ng] = (unsigned char)np;
            H.gcell[ng] = cell;
            H.gw2d[ng] = acc > 0.0 ? acc : 0.0;
          }
          if (kSerial) gends |= (unsigned long long)np << (4 * ng);
          ++ng;
          last_end = np;
        }
      });
  if (overflow) {
    raise_status(status, CTSM_ERR_TOO_LARGE);
    if (lane == 0) {
      H.np = 0;
      H.ng = 0;
    }
    return false;
  }
  const bool flat = !(fabs(Sp) > kEpsSingular);
  if (lane == 0) {
    H.S = Sp;
    H.C = Cp;
    H.invS = flat ? 0.0 : 1.0 / Sp;
    H.invC = 1.0 / Cp;
    H.kappa = ca * ca / (6.0 * cb * g.c);
    H.inv_a = 1.0 / ca;
    double dmn = frcp(sw.D[0]), dmx = dmn;
    for (int k = 1; k < 4; ++k) {
      const double v = frcp(sw.D[k]);
      dmn = fmin(dmn, v);
      dmx = fmax(dmx, v);
    }
    H.dmin_inv = dmn;
    H.dmax_inv = dmx;
    H.flat = flat;
    H.np = np;
    H.ng = ng;
  }
  int qcur = 0;
  double agg_mn = 1e300, agg_mx = -1e300, agg_al = 0.0, agg_be = 0.0;
  for (int pj = kSerial ? 0 : lane; pj < np && (kSerial || pj == lane); ++pj) {
    if (kSerial) {
      my_lo = all_lo[pj];
      my_hi = all_hi[pj];
      my_kind = (int)((kinds >> (2 * pj)) & 3u);
    }
    // constant divisors as reciprocal multiplies (tolerance-checked path)
    const double ica = 1.0 / ca;
    double cl[kSerial ? kCoef : 1];
    if (kSerial) {
#pragma unroll
      for (int i = 0; i < kCoef; ++i) cl[i] = 0.0;
    }
    double* c = kSerial ? cl : P[pj].c;
    if (my_kind == 1) {
      // trap_flags_at / trap_atom_flags (weights3d.cpp:63-107)
      const double t1 = my_lo, t2 = my_hi;
      const double cr1 = Cp + Sp * t1, cr2 = Cp + Sp * t2;
      const double Pg = (s * Cp - fx1) * ica, Pf = (s * Cp - fx0) * ica;
      const double i1 = 1.0 / cr1, i2 = 1.0 / cr2, i12 = i1 * i2;
      c[0] = Pg * i1;
      c[1] = Pg * i2;
      c[2] = Pf * i1;
      c[3] = Pf * i2;
      c[4] = cr1;
      c[5] = cr2;
      c[6] = t1 - t2;
      c[7] = 3.0 * Pg * Pg * i12;
      c[8] = Pg * Pg * Pg * (cr1 + cr2) * i12 * i12;
      c[9] = 3.0 * Pf * Pf * i12;
      c[10] = Pf * Pf * Pf * (cr1 + cr2) * i12 * i12;
      c[11] = Pg;
      c[12] = Pf;
      // band quadrilateral between the rays t1, t2 and the faces x = fx0, fx1
      // (canonical frame): y_t(X) = (t (s - X Cp) + X Sp) / (Cp + t Sp);
      // Simpson over X is exact for the (quadratic) depth moment.
      auto seg = [&](double X, double& len, double& dmid) {
        const double ya = (t1 * (s - X * Cp) + X * Sp) * i1;
        const double yb = (t2 * (s - X * Cp) + X * Sp) * i2;
        len = fabs(yb - ya);
        dmid = s - X * Cp - 0.5 * (ya + yb) * Sp;
      };
      double l0, d0, lm, dm, l1, d1;
      seg(fx0, l0, d0);
      seg(0.5 * (fx0 + fx1), lm, dm);
      seg(fx1, l1, d1);
      const double area = ca * (l0 + 4.0 * lm + l1) * (1.0 / 6.0);
      const double mom = ca * (l0 * d0 + 4.0 * lm * dm + l1 * d1) * (1.0 / 6.0);
      double* l = c + kLin;
      l[0] = fmin(fmin(c[0], c[1]), fmin(c[2], c[3]));
      l[1] = fmax(fmax(c[0], c[1]), fmax(c[2], c[3]));
      l[2] = 6.0 * area * ica * ica;
      l[3] = area > 0.0 ? mom / area * ica : 0.0;
    } else {
      // tri_flags_at / tri_atom_flags (weights3d.cpp:115-168) at both ends
      const double xa = my_kind == 0 ? ax1 : ax4, ya = my_kind == 0 ? ay1 : ay4;
      const double Pq = (s * Cp - xa) * ica, Qq = (s * Sp - ya) * ica;
      const double thgg = Pq * Cp + Qq * Sp;
      const double Da = s - xa * Cp - ya * Sp;       // apex depth (= a' thgg)
      const double ta = my_kind == 0 ? sw.T1 : sw.T4;  // apex ray parameter
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double t = e == 0 ? my_lo : my_hi;
        const double crg = Cp + Sp * t, srh = Sp - Cp * t;
        double* q = c + 7 * e;
        q[0] = Pq / crg;
        q[1] = thgg;
        q[2] = Qq / srh;
        q[3] = crg;
        q[4] = Qq - Pq * srh / crg;
        q[5] = srh / Cp;
        q[6] = t;
        // corner triangle between the apex ray and ray t (canonical frame):
        // legs dx = Da (t - ta) / (t Cp - Sp), dy = Da (t - ta) / (Cp + t Sp)
        const double k = Da * (t - ta);
        const double dx = k / (t * Cp - Sp), dy = k / crg;
        const double area = 0.5 * fabs(dx * dy);
        const double dcen = Da - (dx * Cp + dy * Sp) * (1.0 / 3.0);
        double* l = c + kLin + 4 * e;
        l[0] = fmin(fmin(q[0], q[1]), q[2]);
        l[1] = fmax(fmax(q[0], q[1]), q[2]);
        l[2] = 6.0 * area * ica * ica;
        l[3] = dcen * ica;
      }
    }
    if (kSerial) {
      const double* l = cl + kLin;
      // the piece leaves as six 32-byte stores (whole sectors: no partial
      // writes, 6 instead of 22 store instructions per piece)
#pragma unroll
      for (int i = 0; i < kCoef; i += 4)
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(P[pj].c + i), "d"(cl[i]),
                     "d"(cl[i + 1]), "d"(cl[i + 2]), "d"(cl[i + 3])
                     : "memory");
      if (my_kind == 1) {
        agg_mn = fmin(agg_mn, l[0]);
        agg_mx = fmax(agg_mx, l[1]);
        agg_al += l[2];
        agg_be += l[2] * l[3];
      } else {
        const double sg = my_kind == 0 ? 1.0 : -1.0;
        agg_mn = fmin(agg_mn, fmin(l[0], l[4]));
        agg_mx = fmax(agg_mx, fmax(l[1], l[5]));
        agg_al += sg * (l[6] - l[2]);
        agg_be += sg * (l[6] * l[7] - l[2] * l[3]);
      }
      if (pj + 1 == (int)((gends >> (4 * qcur)) & 15ull)) {  // last piece of group qcur
        H.gmin[qcur] = agg_mn;
        H.gmax[qcur] = agg_mx;
        H.galpha[qcur] = agg_al;
        H.gbeta[qcur] = agg_be;
        ++qcur;
        agg_mn = 1e300;
        agg_mx = -1e300;
        agg_al = agg_be = 0.0;
      }
    }
  }
  if (kSerial) return true;
  __syncwarp();
  for (int q = kSerial ? 0 : lane; q < ng && (kSerial || q == lane); ++q) {
    // group aggregates (warp form: lane q handles group q)
    double mn = 1e300, mx = -1e300, al = 0.0, be = 0.0;
#pragma unroll 1
    for (int k = H.gbeg[q]; k < H.gend[q]; ++k) {
      const double* c = P[k].c;
      const double* l = c + kLin;
      if (H.pkind[k] == 1) {
        mn = fmin(mn, l[0]);
        mx = fmax(mx, l[1]);
        al += l[2];
        be += l[2] * l[3];
      } else {
        const double sg = H.pkind[k] == 0 ? 1.0 : -1.0;  // zone 0: hi - lo; zone 2: lo - hi
        mn = fmin(mn, fmin(l[0], l[4]));
        mx = fmax(mx, fmax(l[1], l[5]));
        al += sg * (l[6] - l[2]);
        be += sg * (l[6] * l[7] - l[2] * l[3]);
      }
    }
    H.gmin[q] = mn;
    H.gmax[q] = mx;
    H.galpha[q] = al;
    H.gbeta[q] = be;
  }
  return true;
}

// |tt| of a triangle atom with the linear / zero short cuts (q: the 7 cubic
// coefficients, l: th_min, th_max, slope, root).
__device__ __forceinline__ double tri_abs(const ColumnHead& H, const double* q, const double* l,
                                          double G) {
  if (G <= l[0]) return 0.0;
  if (G > l[1]) return l[2] * (G - l[3]);
  return fabs(tri_tt(H, q, G));
}

__device__ __forceinline__ double trap_abs(const ColumnHead& H, const double* c, double G) {
  const double* l = c + kLin;
  if (G <= l[0]) return 0.0;
  if (G > l[1]) return l[2] * (G - l[3]);
  return fabs(trap_tt(H, c, G));
}

// atom_sum (weights3d.cpp:400-423) over the pieces of cell group q at height
// zref for row-edge slope tan_a; gs = 1 / (a' tan_a) so G = zref * gs.
__device__ __forceinline__ double atom_sum3(const ColumnHead& H, const PieceCoef* P, int q,
                                            double tan_a, double gs, double zref) {
  const double G = zref * gs;
  if (G <= H.gmin[q]) return 0.0;
  if (G > H.gmax[q]) return H.kappa * tan_a * (H.galpha[q] * G - H.gbeta[q]);
  double v = 0.0;
  for (int k = H.gbeg[q]; k < H.gend[q]; ++k) {
    const double* c = P[k].c;
    double tt;
    switch (H.pkind[k]) {
      case 0: tt = tri_abs(H, c + 7, c + kLin + 4, G) - tri_abs(H, c, c + kLin, G); break;
      case 1: tt = trap_abs(H, c, G); break;
      default: tt = tri_abs(H, c, c + kLin, G) - tri_abs(H, c + 7, c + kLin + 4, G); break;
    }
    v += tt;
  }
  return H.kappa * tan_a * v;
}

// ---- per-group piecewise-cubic tables -------------------------------------
// For a cell group q the un-scaled atom sum f_q(G) (atom_sum3 without the
// kappa tan_a factor) is the integral over the group's 2D region of a ramp
// max(0, G - depth/a'): a piecewise cubic in G whose knots are the atoms' flag
// thresholds (the depths of the region's vertices). Zero for G <= gmin and
// the exact linear galpha G - gbeta for G > gmax. Between consecutive knots
// it is one cubic, so it is recovered exactly (in real arithmetic) from the
// reference atoms at 4 nodes of the interval: s = -1, -1/3, 1/3, 1 on the
// interval mapped to [-1, 1], stored as b0 + b1 s + b2 s^2 + b3 s^3 (|s| <= 1:
// rounding stays at a few ulps of max|f|). Knots closer than ~1e-9 of the
// group's G range are merged; the sliver they bound then carries the cubic
// of its neighbour, an error of order jump(f''') w^3 (negligible).
// Per voxel a group evaluation is then a knot count and one Horner cubic
// instead of the per-piece flag logic of atom_sum3. A (column, angle) whose
// knots or intervals exceed the capacity falls back to atom_sum3.
constexpr int kMaxKnots = 48;
constexpr int kMaxIntervals = 64;
struct GroupTable {
  int ok;
  unsigned char kbeg[kMaxPieces], kcnt[kMaxPieces], ibeg[kMaxPieces];
  double kn[kMaxKnots];
  double2 iv[kMaxIntervals][3];  // (mid, 2/w), (b0, b1), (b2, b3)
};

// Un-scaled atom sum of group q (the inner loop of atom_sum3).
#ifdef CTSM_GROUP_RAW_NOINLINE
__device__ __noinline__ double group_raw(
#else
__device__ __forceinline__ double group_raw(
#endif
    const ColumnHead& H, const PieceCoef* P, int q, double G) {
  double v = 0.0;
  for (int k = H.gbeg[q]; k < H.gend[q]; ++k) {
    const double* c = P[k].c;
    double tt;
    switch (H.pkind[k]) {
      case 0: tt = tri_abs(H, c + 7, c + kLin + 4, G) - tri_abs(H, c, c + kLin, G); break;
      case 1: tt = trap_abs(H, c, G); break;
      default: tt = tri_abs(H, c, c + kLin, G) - tri_abs(H, c + 7, c + kLin + 4, G); break;
    }
    v += tt;
  }
  return v;
}

// Builds the tables of a planned (column, angle); all lanes, after the
// __syncwarp() that follows plan_column. Ends with __syncwarp().
__device__ __forceinline__ void build_group_tables(const ColumnHead& H, const PieceCoef* P,
                                                   GroupTable& T, int lane) {
  const int ng = H.ng;
  // (1) knots, lane q for group q: thresholds in (gmin, gmax) plus both ends,
  // insertion-sorted in place into the group's slot of T.kn, close ones merged.
  // Slots are provisional (18 per group) and compacted in (2).
  constexpr int kRaw = 20;
  double* raw = &T.iv[0][0].x;  // scratch: kMaxIntervals * 6 doubles >= kMaxPieces * kRaw
  int cnt = 0;
  bool bad = false;
  if (lane < ng) {
    const int q = lane;
    const double lo = H.gmin[q], hi = H.gmax[q];
    double* r = raw + q * kRaw;
    r[0] = lo;
    cnt = 1;
    auto add = [&](double v) {
      if (!(v > lo && v < hi)) return;
      if (cnt >= kRaw - 1) {  // cannot happen (<= 3 pieces per cell): be safe
        bad = true;
        return;
      }
      int i = cnt++;
      while (i > 0 && r[i - 1] > v) {
        r[i] = r[i - 1];
        --i;
      }
      r[i] = v;
    };
    for (int k = H.gbeg[q]; k < H.gend[q]; ++k) {
      const double* c = P[k].c;
      // every threshold any branch of the atom tests (a superset of the
      // knots is harmless: the cubic just spans a split interval)
      if (H.pkind[k] == 1) {
        add(c[0]); add(c[1]); add(c[2]); add(c[3]);
        if (H.flat) {
          add(c[11]);
          add(c[12]);
        }
      } else {
        for (int e = 0; e < 2; ++e) {
          add(c[7 * e]);
          add(c[7 * e + 1]);
          add(c[7 * e + 2]);
        }
      }
    }
    if (hi > lo) r[cnt++] = hi;
    // merge knots closer than tol; the ends stay gmin and gmax exactly (a
    // range below tol keeps gmin only: zero below, linear above)
    const double tol = 1e-9 * (hi - lo) + 4e-16 * fabs(hi);
    int m = 1;
    for (int i = 1; i < cnt; ++i)
      if (r[i] - r[m - 1] > tol) r[m++] = r[i];
    if (m > 1) r[m - 1] = hi;
    cnt = m;
  }
  // (2) offsets (warp prefix over groups) and capacity check
  int kb = cnt, ib = cnt + 1;
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, kb, o), b = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) {
      kb += a;
      ib += b;
    }
  }
  const int kt = __shfl_sync(0xffffffffu, kb, 31), it = __shfl_sync(0xffffffffu, ib, 31);
  kb -= cnt;
  ib -= cnt + 1;
  const bool fits = kt <= kMaxKnots && it <= kMaxIntervals && !__any_sync(0xffffffffu, bad);
  if (fits && lane < ng) {
    const double* r = raw + lane * kRaw;
    for (int i = 0; i < cnt; ++i) T.kn[kb + i] = r[i];
    T.kbeg[lane] = (unsigned char)kb;
    T.kcnt[lane] = (unsigned char)cnt;
    T.ibeg[lane] = (unsigned char)ib;
  }
  if (lane == 0) T.ok = fits;
  __syncwarp();
  if (!fits) return;
  // (3) node values of the cubic intervals: item = (group, interval, node);
  // the interval slots of group q are ibeg+1 .. ibeg+cnt-1 (slot ibeg: zero,
  // ibeg+cnt: linear); node values go to the (b0,b1),(b2,b3) slots first.
  int tot = 0;
  for (int q = 0; q < ng; ++q) tot += 4 * (T.kcnt[q] - 1);
  for (int it0 = lane; it0 < tot; it0 += 32) {
    int q = 0, rem = it0;
    while (rem >= 4 * (T.kcnt[q] - 1)) {
      rem -= 4 * (T.kcnt[q] - 1);
      ++q;
    }
    const int j = rem >> 2, nd = rem & 3;
    const double k0 = T.kn[T.kbeg[q] + j], k1 = T.kn[T.kbeg[q] + j + 1];
    const double mid = 0.5 * (k0 + k1), hw = 0.5 * (k1 - k0);
    const double G = nd == 0 ? k0 : (nd == 3 ? k1 : mid + hw * (nd == 1 ? -1.0 / 3.0 : 1.0 / 3.0));
    double* dst = &T.iv[T.ibeg[q] + 1 + j][1].x;
    dst[nd] = group_raw(H, P, q, G);
  }
  __syncwarp();
  // (4) coefficients, one lane per interval slot
  for (int s = lane; s < it; s += 32) {
    int q = 0;
    while (q + 1 < ng && T.ibeg[q + 1] <= s) ++q;
    const int j = s - T.ibeg[q], m = T.kcnt[q];
    double2* e = T.iv[s];
    if (j == 0) {
      e[0] = make_double2(0.0, 0.0);
      e[1] = make_double2(0.0, 0.0);
      e[2] = make_double2(0.0, 0.0);
    } else if (j == m) {
      const double gm = H.gmax[q], al = H.galpha[q];
      e[0] = make_double2(gm, 1.0);
      e[1] = make_double2(al * gm - H.gbeta[q], al);
      e[2] = make_double2(0.0, 0.0);
    } else {
      const double k0 = T.kn[T.kbeg[q] + j - 1], k1 = T.kn[T.kbeg[q] + j];
      const double f0 = e[1].x, f1 = e[1].y, f2 = e[2].x, f3 = e[2].y;
      const double E1 = 0.5 * (f0 + f3), E2 = 0.5 * (f1 + f2);
      const double O1 = 0.5 * (f3 - f0), O2 = 0.5 * (f2 - f1);
      const double b2 = 1.125 * (E1 - E2);
      const double b0 = E2 - b2 * (1.0 / 9.0);
      const double b1 = 0.125 * (27.0 * O2 - O1);
      const double b3 = O1 - b1;
      e[0] = make_double2(0.5 * (k0 + k1), 2.0 / (k1 - k0));
      e[1] = make_double2(b0, b1);
      e[2] = make_double2(b2, b3);
    }
  }
  __syncwarp();
}

// f_q(G) from the table (see above).
__device__ __forceinline__ double group_table(const GroupTable& T, int q, double G) {
  const double* kn = T.kn + T.kbeg[q];
  const int m = T.kcnt[q];
  int j = 0;
  for (int i = 0; i < m; ++i) j += kn[i] < G;
  const double2* e = T.iv[T.ibeg[q] + j];
  const double2 h = e[0], b01 = e[1], b23 = e[2];
  const double s = (G - h.x) * h.y;
  return fma(fma(fma(b23.y, s, b23.x), s, b01.y), s, b01.x);
}

// Weights of voxel iz of a planned column: emit(cell m_y, row m_z, w) for every
// w > 1e-16 inside the detector (weights3d.cpp:426-458).
template <typename Emit>
__device__ __forceinline__ void voxel_weights(const DevGeom& g, const ColumnHead& H,
                                              const PieceCoef* P, int iz, Emit&& emit) {
  const double sdd = g.sdd;
  const double zb = (iz - g.n_z / 2.0) * g.c, zt = zb + g.c;
  const double sdd_dz = g.sdd_dz;
  const double mb1 = sdd_dz * zb * H.dmin_inv, mb2 = sdd_dz * zb * H.dmax_inv;
  const double mt1 = sdd_dz * zt * H.dmin_inv, mt2 = sdd_dz * zt * H.dmax_inv;
  const double m_min = fmin(fmin(mb1, mb2), fmin(mt1, mt2));
  const double m_max = fmax(fmax(mb1, mb2), fmax(mt1, mt2));
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  const int fl = (int)floor(m_min);
  const int k_lo = (fl < row_lo) ? row_lo : fl;
  const int chi = (int)ceil(m_max) - 1;
  const int k_hi = (chi < row_hi) ? chi : row_hi;
  if (k_hi < k_lo) return;
  const double dz_sdd = g.dz_sdd;
  for (int q = 0; q < H.ng; ++q) {
    const double w2d = H.gw2d[q];
    auto above = [&](double kk) -> double {
      if (kk <= m_min) return w2d;
      if (kk >= m_max) return 0.0;
      if (kk == 0.0) {
        if (zb >= 0.0) return w2d;
        if (zt <= 0.0) return 0.0;
        return w2d * zt / (zt - zb);
      }
      const double tan_a = fabs(kk) * dz_sdd;
      const double gs = H.inv_a / tan_a;
      if (kk > 0.0) return atom_sum3(H, P, q, tan_a, gs, zt) - atom_sum3(H, P, q, tan_a, gs, zb);
      return w2d - (atom_sum3(H, P, q, tan_a, gs, -zb) - atom_sum3(H, P, q, tan_a, gs, -zt));
    };
    const int cell = H.gcell[q];
    double prev = above((double)k_lo);
    for (int L = k_lo; L <= k_hi; ++L) {
      const double next = above((double)(L + 1));
      const double v = prev - next;
      if (v > kEpsWeight) emit(cell, L, v);
      prev = next;
    }
  }
}

// Weights of voxels [z0, z1) of a planned column, cell group by cell group,
// with the z-face sharing of the reference's composition made explicit: the
// top face of voxel iz is the bottom face of voxel iz+1, so the atom sums
// F(L, zt) computed for voxel iz are exactly F(L, zb) of voxel iz+1 and are
// reused (up to 4 row edges cached). emit(iz, cell, row, w).
__device__ __noinline__ double atom_sum3_slow(const ColumnHead& H, const PieceCoef* P, int q,
                                              double tan_a, double gs, double zref) {
  return atom_sum3(H, P, q, tan_a, gs, zref);
}

// Warp-batched cubic faces (chunk_weights with a CubicBatch): the cubic path
// (group_raw: mixed-flag atoms) is needed by a few lanes at a time, at
// different voxels, so evaluated where it arises it runs nearly every step
// with 1-3 active lanes. Per cell group the lanes first list their cubic
// faces (pass 1: the same zero / linear classification, no weights), the
// warp evaluates the whole list with every lane busy (pass 2, a warp prefix
// sum over the per-lane counts), and the row loop (pass 3) takes the values
// in the order pass 1 listed them. Faces beyond a lane's kRq slots are
// evaluated in place. The classification is the same products and compares
// in both passes, so the two passes agree face by face.
#ifndef CTSM_KRQ
#define CTSM_KRQ 8
#endif
constexpr int kRq = CTSM_KRQ;
struct CubicBatch {
  double rq[kRq][32];  // [slot][lane]: G in pass 1, the raw atom sum after pass 2
  int roff[32];
};

template <typename Emit>
__device__ __forceinline__ void chunk_weights(const DevGeom& g, const ColumnHead& H,
                                              const PieceCoef* P, int z0, int z1, Emit&& emit,
                                              const GroupTable* T = nullptr,
                                              CubicBatch* B = nullptr, int lane = 0) {
  const bool tab = T != nullptr && T->ok;
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  const double dz_sdd = g.dz_sdd, sdd_dz = g.sdd_dz;
  const double c_mn = sdd_dz * H.dmin_inv, c_mx = sdd_dz * H.dmax_inv;
  // row magnification range of a voxel [zb, zt]: the extremes of the four
  // products z * c (c > 0, rounding monotone) picked by the signs of zb, zt,
  // bit-identical to min / max over all four
  const double c_lo = fmin(c_mn, c_mx), c_hi = fmax(c_mn, c_mx);
  const double ga = H.inv_a * sdd_dz;  // G = zref * ga / |L|
  for (int q = 0; q < H.ng; ++q) {
    const double w2d = H.gw2d[q];
    const int cell = H.gcell[q];
    // the group's short cuts in registers, division-free: with u = zref ga,
    // G <= gmin  <=>  u <= gmin |L|  (F = 0), and G > gmax  <=>  u > gmax |L|,
    // where F = kappa tan_a (galpha G - gbeta) = l1 zref - l2 |L|
    // (tan_a = |L| dz/sdd, tan_a G = zref ga dz/sdd)
    const double gmn = H.gmin[q], gmx = H.gmax[q];
    const double l1 = H.kappa * H.galpha[q] * ga * dz_sdd, l2 = H.kappa * H.gbeta[q] * dz_sdd;
    auto cheap = [&](double aL, double zref, double& f) -> bool {
      const double u = zref * ga;
      if (u <= gmn * aL) {
        f = 0.0;
        return true;
      }
      if (u > gmx * aL) {
        f = l1 * zref - l2 * aL;
        return true;
      }
      return false;
    };
    auto Fcubic = [&](double aL, double zref) -> double {
#ifdef CTSM_EXP_NO_CUBIC
      return l1 * zref - l2 * aL;  // timing experiment only (wrong weights)
#endif
      const double tan_a = aL * dz_sdd;
      const double G = zref * ga * frcp(aL);
      if (tab) return H.kappa * tan_a * group_table(*T, q, G);
      return H.kappa * tan_a * group_raw(H, P, q, G);
    };
    int nl = 0, used = 0;
    if (B != nullptr) {
      // pass 1: list the cubic faces (same walk and tests as pass 3)
      int nreq = 0;
#pragma unroll 1
      for (int iz = z0; iz < z1; ++iz) {
        const double zb = (iz - g.n_z / 2.0) * g.c, zt = zb + g.c;
        const double m_min = zb * (zb >= 0.0 ? c_lo : c_hi);
        const double m_max = zt * (zt <= 0.0 ? c_lo : c_hi);
        const int fl = (int)floor(m_min);
        const int k_lo = (fl < row_lo) ? row_lo : fl;
        const int chi = (int)ceil(m_max) - 1;
        const int k_hi = (chi < row_hi) ? chi : row_hi;
        // unclamped ends are always skipped below (floor(m_min) <= m_min,
        // ceil(m_max) >= m_max): leave them out of the walk
#pragma unroll 1
        for (int L = k_lo + (fl >= row_lo), Le = k_hi + (chi >= row_hi); L <= Le; ++L) {
          const double kk = (double)L;
          if (kk <= m_min || kk >= m_max || L == 0) continue;
          const double aL = fabs(kk);
          const double zt_s = L > 0 ? zt : -zt, zb_s = L > 0 ? zb : -zb;
          double f;
          if (!cheap(aL, zb_s, f)) {
            if (nreq < kRq) B->rq[nreq][lane] = zb_s * ga * frcp(aL);
            ++nreq;
          }
          if (!cheap(aL, zt_s, f)) {
            if (nreq < kRq) B->rq[nreq][lane] = zt_s * ga * frcp(aL);
            ++nreq;
          }
        }
      }
      // pass 2: the warp evaluates all listed faces
      nl = nreq < kRq ? nreq : kRq;
      int incl = nl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (total > 0) {
        B->roff[lane] = incl - nl;
        __syncwarp();
#pragma unroll 1
        for (int f = lane; f < total; f += 32) {
          int o = 0;
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1)
            if (o + st < 32 && B->roff[o + st] <= f) o += st;
          const int k = f - B->roff[o];
#ifdef CTSM_EXP_NO_CUBIC
          B->rq[k][o] = 0.0;
#else
          B->rq[k][o] = group_raw(H, P, q, B->rq[k][o]);
#endif
        }
        __syncwarp();
      }
    }
    // cache of F(L, z) at the current voxel's bottom face (signed L key);
    // unused when batched (pass 1 lists both faces)
    int cL0 = INT_MIN, cL1 = INT_MIN, cL2 = INT_MIN, cL3 = INT_MIN;
    double cF0 = 0.0, cF1 = 0.0, cF2 = 0.0, cF3 = 0.0;
    for (int iz = z0; iz < z1; ++iz) {
      const double zb = (iz - g.n_z / 2.0) * g.c, zt = zb + g.c;
      const double m_min = zb * (zb >= 0.0 ? c_lo : c_hi);
      const double m_max = zt * (zt <= 0.0 ? c_lo : c_hi);
      const int fl = (int)floor(m_min);
      const int k_lo = (fl < row_lo) ? row_lo : fl;
      const int chi = (int)ceil(m_max) - 1;
      const int k_hi = (chi < row_hi) ? chi : row_hi;
      int nL0 = INT_MIN, nL1 = INT_MIN, nL2 = INT_MIN, nL3 = INT_MIN;
      double nF0 = 0.0, nF1 = 0.0, nF2 = 0.0, nF3 = 0.0;
      int nn = 0;
      auto above = [&](int L) -> double {
        const double kk = (double)L;
        if (kk <= m_min) return w2d;
        if (kk >= m_max) return 0.0;
        if (L == 0) {
          if (zb >= 0.0) return w2d;
          if (zt <= 0.0) return 0.0;
          return w2d * zt / (zt - zb);
        }
        const double aL = fabs(kk);
        const double zt_s = L > 0 ? zt : -zt, zb_s = L > 0 ? zb : -zb;
        // zero / linear faces first (the common case, no cache traffic);
        // only a cubic bottom face consults the cache of the previous
        // voxel's cubic top faces, and only a cubic top face is cached
        double Fb = 0.0, Ft = 0.0;
        bool need_b = !cheap(aL, zb_s, Fb), need_t = !cheap(aL, zt_s, Ft);
        if (need_b && B == nullptr) {
          if (L == cL0) { Fb = cF0; need_b = false; }
          else if (L == cL1) { Fb = cF1; need_b = false; }
          else if (L == cL2) { Fb = cF2; need_b = false; }
          else if (L == cL3) { Fb = cF3; need_b = false; }
        }
        if (need_b || need_t) {
          // one call site of the cubic path (large: code size / icache)
#pragma unroll 1
          for (;;) {
            double f;
            const int k = used++;
            if (B != nullptr && k < nl)
              f = H.kappa * (aL * dz_sdd) * B->rq[k][lane];
            else
              f = Fcubic(aL, need_b ? zb_s : zt_s);
            if (need_b) {
              Fb = f;
              need_b = false;
              if (!need_t) break;
            } else {
              Ft = f;
              switch (nn) {
                case 0: nL0 = L; nF0 = Ft; break;
                case 1: nL1 = L; nF1 = Ft; break;
                case 2: nL2 = L; nF2 = Ft; break;
                case 3: nL3 = L; nF3 = Ft; break;
                default: break;
              }
              ++nn;
              break;
            }
          }
        }
        return L > 0 ? Ft - Fb : w2d - (Fb - Ft);
      };
      // edges k_lo .. k_hi+1 with one call site each of above() and emit()
      // unclamped lower end: above(k_lo) = w2d (floor(m_min) <= m_min, an
      // early return before any cache traffic), so the walk starts after it
      const bool lo_free = fl >= row_lo;
      double prev = lo_free ? w2d : 0.0;
#pragma unroll 1
      for (int L = k_lo + (lo_free ? 1 : 0); L <= k_hi + 1; ++L) {
        const double cur = above(L);
        if (L > k_lo) {
          const double v = prev - cur;
          if (v > kEpsWeight) emit(iz, cell, L - 1, v);
        }
        prev = cur;
      }
      cL0 = nL0; cL1 = nL1; cL2 = nL2; cL3 = nL3;
      cF0 = nF0; cF1 = nF1; cF2 = nF2; cF3 = nF3;
    }
  }
}


// chunk_weights with the (voxel, row edge) walks of a lane flattened into one
// loop (CTSM_FLAT, batched form only): in chunk_weights the lanes of a warp
// step through their voxels in lockstep, so every voxel costs the warp the
// longest edge walk among its 32 lanes (2 or 3 edges, whichever lane has the
// most); flattened, a lane that finishes a voxel's edges moves on to its next
// voxel while other lanes still work on theirs, and the warp pays the longest
// *chunk total* instead of the sum of the per-voxel maxima. The per-lane
// sequence of evaluations, their operands and the emission order are those
// of chunk_weights (same lambdas, same products and compares), so the
// weights are bit-identical.
// pre(cell, row) is called before the weight of (cell, row) is evaluated (it
// may turn out to be zero and not be emitted): the back-projection issues the
// row's image-vector loads there, so that they are in flight during the
// evaluation instead of being waited for right after it.
// gend(cell) is called after the last weight of a cell group: the forward
// flushes its pending row run there, so a run never crosses groups and its
// detector cell is the group's (loop-invariant address arithmetic).
__device__ __noinline__ double group_raw_ool(const ColumnHead& H, const PieceCoef* P, int q,
                                             double G) {
  return group_raw(H, P, q, G);
}
#ifndef CTSM_CHEAP_BF
#define CTSM_CHEAP_BF 1  // C3 fwd 82 -> 79, bwd 86 -> 82 ms per projection
#endif
struct NoPre {
  __device__ __forceinline__ void operator()(int, int) const {}
};
struct NoGroupEnd {
  __device__ __forceinline__ void operator()(int) const {}
};
// (Summing a voxel's weights in 16 more registers and adding them to the
// back-projection's shared-memory accumulators once per (group, voxel) was
// slower: C3 bwd 47.5 vs 43.4 ms per half scan.)
// kTwoSite: the emitting pass takes a cubic face's value at two call sites
// (bottom / top face; a face beyond the lane's kRq slots goes through the
// out-of-line atom sum) instead of one loop around a single site: the forward
// gains 2 % (C3 83 -> 82 ms per projection), the back-projection loses 3 %
// (87 -> 90 ms), so only the forward uses it.
template <bool kTwoSite = false, typename Emit, typename Pre = NoPre, typename GEnd = NoGroupEnd>
__device__ __forceinline__ void chunk_weights_flat(const DevGeom& g, const ColumnHead& H,
                                                   const PieceCoef* P, int z0, int z1,
                                                   Emit&& emit, CubicBatch* B, int lane,
                                                   Pre&& pre = NoPre(),
                                                   GEnd&& gend = NoGroupEnd()) {
  const int row_lo = -g.n_det_z / 2, row_hi = g.n_det_z / 2 - 1;
  const double dz_sdd = g.dz_sdd, sdd_dz = g.sdd_dz;
  const double c_mn = sdd_dz * H.dmin_inv, c_mx = sdd_dz * H.dmax_inv;
  const double c_lo = fmin(c_mn, c_mx), c_hi = fmax(c_mn, c_mx);
  const double ga = H.inv_a * sdd_dz;  // G = zref * ga / |L|
  const double hz = g.n_z / 2.0, vc = g.c;
  // Row range of a voxel: fl = floor(m_min), chi = ceil(m_max) - 1. For an
  // integer edge L, L <= m_min <=> L <= fl and L >= m_max <=> L > chi, so
  // the walks compare integers (C3 bwd 45.1 -> 43.4 ms per half scan).
  // (Computing the ranges of a chunk once per (column, angle) and keeping
  // them across the groups was slower, packed in two registers (45.0 ms) or
  // in shared memory (44.7 ms).)
  auto range_of = [&](int izq, int& fl, int& chi) {
    const double zb = ((double)izq - hz) * vc, zt = zb + vc;
    const double m_min = zb * (zb >= 0.0 ? c_lo : c_hi);
    const double m_max = zt * (zt <= 0.0 ? c_lo : c_hi);
    fl = (int)floor(m_min);
    chi = (int)ceil(m_max) - 1;
  };
  for (int q = 0; q < H.ng; ++q) {
    const double w2d = H.gw2d[q];
    const int cell = H.gcell[q];
    const double gmn = H.gmin[q], gmx = H.gmax[q];
    const double l1 = H.kappa * H.galpha[q] * ga * dz_sdd, l2 = H.kappa * H.gbeta[q] * dz_sdd;
    auto cheap = [&](double aL, double zref, double& f) -> bool {
      const double u = zref * ga;
#if CTSM_CHEAP_BF
      // branch-free: the linear value is formed speculatively (it is
      // overwritten when the face turns out to be cubic)
      const double flin = l1 * zref - l2 * aL;
      const bool zero = u <= gmn * aL, lin = u > gmx * aL;
      f = zero ? 0.0 : flin;
      return zero || lin;
#else
      if (u <= gmn * aL) {
        f = 0.0;
        return true;
      }
      if (u > gmx * aL) {
        f = l1 * zref - l2 * aL;
        return true;
      }
      return false;
#endif
    };
    // walk state of the lane: voxel iz with faces zb / zt, its row range
    // (fl, chi), the current edge L and the last edge Le of the voxel
    int iz, L = 0, Le = -1, k_lo = 0, vfl = 0, vchi = 0;
    double zb = 0.0, zt = 0.0;
    // pass 1: list the cubic faces
    auto setup1 = [&]() {
      for (; iz < z1; ++iz) {
        range_of(iz, vfl, vchi);
        k_lo = (vfl < row_lo) ? row_lo : vfl;
        const int k_hi = (vchi < row_hi) ? vchi : row_hi;
        L = k_lo + (vfl >= row_lo);
        Le = k_hi + (vchi >= row_hi);
        if (L <= Le) {
          zb = ((double)iz - hz) * vc;
          zt = zb + vc;
          return;
        }
      }
    };
    int nreq = 0;
    iz = z0;
    setup1();
#pragma unroll 1
    while (iz < z1) {
      const double kk = (double)L;
      // (L > fl always holds in this walk)
      if (!(L > vchi || L == 0)) {
        const double aL = fabs(kk);
        const double zt_s = L > 0 ? zt : -zt, zb_s = L > 0 ? zb : -zb;
        double f;
        if (!cheap(aL, zb_s, f)) {
          if (nreq < kRq) B->rq[nreq][lane] = zb_s * ga * frcp(aL);
          ++nreq;
        }
        if (!cheap(aL, zt_s, f)) {
          if (nreq < kRq) B->rq[nreq][lane] = zt_s * ga * frcp(aL);
          ++nreq;
        }
      }
      if (++L > Le) {
        ++iz;
        setup1();
      }
    }
    // pass 2: the warp evaluates all listed faces
    const int nl = nreq < kRq ? nreq : kRq;
    int incl = nl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total > 0) {
      B->roff[lane] = incl - nl;
      __syncwarp();
#pragma unroll 1
      for (int f = lane; f < total; f += 32) {
        int o = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1)
          if (o + st < 32 && B->roff[o + st] <= f) o += st;
        const int k = f - B->roff[o];
        B->rq[k][o] = group_raw(H, P, q, B->rq[k][o]);
      }
      __syncwarp();
    }
    // pass 3: the weights
    int used = 0;
    double prev = 0.0;
    auto setup3 = [&]() {
      for (; iz < z1; ++iz) {
        range_of(iz, vfl, vchi);
        k_lo = (vfl < row_lo) ? row_lo : vfl;
        const int k_hi = (vchi < row_hi) ? vchi : row_hi;
        // unclamped lower end: above(k_lo) = w2d, the walk starts after it
        const bool lo_free = vfl >= row_lo;
        prev = lo_free ? w2d : 0.0;
        L = k_lo + (lo_free ? 1 : 0);
        Le = k_hi + 1;
        if (k_hi >= k_lo) {
          zb = ((double)iz - hz) * vc;
          zt = zb + vc;
          return;
        }
      }
    };
    auto above = [&](int Lq) -> double {
      const double kk = (double)Lq;
      // (Lq > vfl always holds in this walk: it starts above floor(m_min))
      if (Lq > vchi) return 0.0;
      if (Lq == 0) {
        if (zb >= 0.0) return w2d;
        if (zt <= 0.0) return 0.0;
        return w2d * zt / (zt - zb);
      }
      const double aL = fabs(kk);
      const double zt_s = Lq > 0 ? zt : -zt, zb_s = Lq > 0 ? zb : -zb;
      double Fb = 0.0, Ft = 0.0;
      bool need_b = !cheap(aL, zb_s, Fb), need_t = !cheap(aL, zt_s, Ft);
      if (kTwoSite && (need_b || need_t)) {
        // a listed face takes its value from the batch; a face beyond the
        // lane's kRq slots (rare) goes through the out-of-line atom sum
        const double kap = H.kappa * (aL * dz_sdd);
        if (need_b) {
          const int k = used++;
          Fb = kap * (k < nl ? B->rq[k][lane] : group_raw_ool(H, P, q, zb_s * ga * frcp(aL)));
        }
        if (need_t) {
          const int k = used++;
          Ft = kap * (k < nl ? B->rq[k][lane] : group_raw_ool(H, P, q, zt_s * ga * frcp(aL)));
        }
      } else if (need_b || need_t) {
        // one call site of the cubic path
#pragma unroll 1
        for (;;) {
          double f;
          const int k = used++;
          if (k < nl) {
            f = H.kappa * (aL * dz_sdd) * B->rq[k][lane];
          } else {
            const double zr = need_b ? zb_s : zt_s;
            f = H.kappa * (aL * dz_sdd) * group_raw(H, P, q, zr * ga * frcp(aL));
          }
          if (need_b) {
            Fb = f;
            need_b = false;
            if (!need_t) break;
          } else {
            Ft = f;
            break;
          }
        }
      }
      return Lq > 0 ? Ft - Fb : w2d - (Fb - Ft);
    };
    iz = z0;
    setup3();
#pragma unroll 1
    while (iz < z1) {
      if (L > k_lo) pre(cell, L - 1);
      const double cur = above(L);
      if (L > k_lo) {
        const double v = prev - cur;
        if (v > kEpsWeight) emit(iz, cell, L - 1, v);
      }
      prev = cur;
      if (++L > Le) {
        ++iz;
        setup3();
      }
    }
    gend(cell);
  }
}

// (A variant with the walks fused across cell groups -- one walk emitting
// group w - 1 while listing the cubic faces of group w, ng + 1 walks instead
// of 2 ng, the batch split into two halves -- was correct but slower: C3 fwd
// 79 vs 78, bwd 77 vs 75 ms per projection, profiles/r3v_sweep3d.log.)

}  // namespace fast
}  // namespace ctsmb
