// exact.cuh -- bit-exact device evaluation of the reference's consistent
// weights, used by the CSR emission kernels (K1/K2).
//
// Contract: compiled with -fmad=false (no FMA contraction) and using the
// correctly rounded crmath.h for every transcendental, each function below
// performs the same IEEE operations, in the same order, on the same operands
// as the reference function it names (paths relative to
// /root/reference/proj/src). The only changes are bit-preserving hoists of
// identical computations:
//   * sin/cos of the (sequentially) quarter-turned angle phi' = phi - k*pi/2
//     are per-angle table lookups (ExactAngle), not per-call evaluations;
//   * edge angles atan(e*d_y/(s+d)) and their tangents are a per-geometry
//     table (edge_tab);
//   * vertex_angles is evaluated once per canonical try (the reference
//     re-evaluates the accepted try in strip_sweep, weights2d.cpp:42);
//   * tan() of every sweep breakpoint is evaluated once and reused by all
//     atoms; the xy sweep is shared by all voxels of a z column.
#pragma once
#include "common.cuh"
#include "crmath.h"
#include "atoms.cuh"

namespace ctsmb {
namespace exact {

// Per-angle table entry: phi_i (geometry.hpp:50-52) and the canonical angles
// phi - k*pi/2 obtained by k sequential subtractions (geometry.cpp:85-91).
struct ExactAngle {
  double fphi[4];
  double sn[4];  // crm_sin(fphi[k])
  double cs[4];  // crm_cos(fphi[k])
};

// Edge table entry for detector edge e: be = atan(e*d_y/(s+d))
// (weights2d.cpp:59) and tan(be) (used by the 3D atoms).
struct EdgeAngle {
  double be;
  double tbe;
};

__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max

// std::lround: round half away from zero.
__device__ __forceinline__ long long lround_exact(double v) {
  double r = trunc(v);
  if (fabs(v - r) >= 0.5) r += (v < 0 ? -1.0 : 1.0);
  return (long long)r;
}

// Table builders (one thread per entry).
static __global__ void build_angle_table(DevGeom g, int angle_begin, int n, ExactAngle* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = angle_begin + k;
  ExactAngle A;
  double fphi = g.angle_start + (g.angle_end - g.angle_start) * i / g.n_angles;
  for (int r = 0; r < 4; ++r) {
    A.fphi[r] = fphi;
    A.sn[r] = crm_sin(fphi);
    A.cs[r] = crm_cos(fphi);
    fphi -= kPi / 2;
  }
  out[k] = A;
}

static __global__ void build_edge_table(DevGeom g, EdgeAngle* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= g.n_edges) return;
  const long long e = (long long)g.edge_lo + k;
  EdgeAngle E;
  E.be = crm_atan(e * g.d_y / (g.s + g.d));
  E.tbe = crm_tan(E.be);
  out[k] = E;
}

// ---- geometry.cpp:56-97 ---------------------------------------------------
// point_angle with sin/cos of phi supplied (identical values).
__device__ __forceinline__ double point_angle(double x, double y, double s, double sp, double cp,
                                              int* status, bool* bad) {
  const double num = y * cp - x * sp;
  const double den = s - y * sp - x * cp;
  if (den <= kEpsDenRel * s) {
    raise_status(status, CTSM_ERR_DEGENERATE_GEOMETRY);
    *bad = true;
    return 0.0;
  }
  return crm_atan2(num, den);
}

struct Sweep {
  // canonical frame (Frame2D, geometry.hpp:124-129)
  double x0, x1, y0, y1, phi, S, C;
  double G1, G2, G3, G4;
  double apex1_x, apex4_x;
  int nb;
  double brk[kMaxBrk];
  double tbrk[kMaxBrk];  // tan(brk[i])
  int np;
  unsigned char pb[kMaxBrk];    // piece i spans brk[pb[i]] .. brk[pb[i] + 1]
  unsigned char pkind[kMaxBrk];
  int pcell[kMaxBrk];
};

// canonical_orientation (geometry.cpp:76-97) + strip_sweep (weights2d.cpp:38-87).
// Returns false (status raised) on failure.
static __device__ bool strip_sweep(const DevGeom& g, const ExactAngle& A, const EdgeAngle* edges,
                            double x0, double x1, double y0, double y1, Sweep& sw, int* status) {
  const double s = g.s;
  bool bad = false;
  // quadrant hint (geometry.cpp:78-82)
  const double cx = 0.5 * (x0 + x1), cy = 0.5 * (y0 + y1);
  const double chi = crm_atan2(s * A.sn[0] - cy, s * A.cs[0] - cx);
  const int k0 = ((int)lround_exact(chi / (kPi / 2)) % 4 + 4) % 4;
  const int tries[4] = {k0, (k0 + 1) % 4, (k0 + 3) % 4, (k0 + 2) % 4};
  double gm[4];
  bool found = false;
  for (int ti = 0; ti < 4 && !found; ++ti) {
    const int k = tries[ti];
    double fx0 = x0, fx1 = x1, fy0 = y0, fy1 = y1;
    for (int r = 0; r < k; ++r) {
      const double nx0 = fy0, nx1 = fy1, ny0 = -fx1, ny1 = -fx0;
      fx0 = nx0;
      fx1 = nx1;
      fy0 = ny0;
      fy1 = ny1;
    }
    const double sp = A.sn[k], cp = A.cs[k];
    gm[0] = point_angle(fx0, fy0, s, sp, cp, status, &bad);
    gm[1] = point_angle(fx1, fy0, s, sp, cp, status, &bad);
    gm[2] = point_angle(fx1, fy1, s, sp, cp, status, &bad);
    gm[3] = point_angle(fx0, fy1, s, sp, cp, status, &bad);
    if (bad) return false;
    if (dmax(gm[0], gm[1]) <= dmin(gm[2], gm[3]) + kCanonSlack) {
      sw.x0 = fx0;
      sw.x1 = fx1;
      sw.y0 = fy0;
      sw.y1 = fy1;
      sw.phi = A.fphi[k];
      sw.S = sp;
      sw.C = cp;
      found = true;
    }
  }
  if (!found) {
    raise_status(status, CTSM_ERR_DEGENERATE_GEOMETRY);
    return false;
  }
  sw.G1 = dmin(gm[0], gm[1]);
  sw.G2 = dmax(gm[0], gm[1]);
  sw.G3 = dmin(gm[2], gm[3]);
  sw.G4 = dmax(gm[2], gm[3]);
  sw.apex1_x = (gm[0] <= gm[1]) ? sw.x0 : sw.x1;
  sw.apex4_x = (gm[3] >= gm[2]) ? sw.x0 : sw.x1;

  // Breakpoints (weights2d.cpp:53-63): corner angles and interior edge angles,
  // sorted, exact duplicates removed. Edges ascend with e, so a merge of the
  // sorted corners with the edges yields the std::sort order.
  const double sdd = g.s + g.d;
  const double tG1 = crm_tan(sw.G1), tG4 = crm_tan(sw.G4);
  const double t_lo = tG1 * (s + g.d) / g.d_y;
  const double t_hi = tG4 * (s + g.d) / g.d_y;
  const long long e_lo = (long long)floor(t_lo) + 1;
  const long long e_hi = (long long)ceil(t_hi) - 1;
  (void)sdd;
  double cv[4] = {sw.G1, sw.G2, sw.G3, sw.G4};
  double ct[4];
  // tan of each corner: reuse tan(G1), tan(G4); G2, G3 evaluated here.
  ct[0] = tG1;
  ct[1] = crm_tan(sw.G2);
  ct[2] = crm_tan(sw.G3);
  ct[3] = tG4;
  // sort the four corner values (stable insertion sort; equal values are
  // identical doubles up to the sign of zero, which no later use observes)
  for (int i = 1; i < 4; ++i) {
    const double v = cv[i], tv = ct[i];
    int j = i - 1;
    while (j >= 0 && v < cv[j]) {
      cv[j + 1] = cv[j];
      ct[j + 1] = ct[j];
      --j;
    }
    cv[j + 1] = v;
    ct[j + 1] = tv;
  }
  int nb = 0;
  int ci = 0;
  long long e = e_lo;
  for (;;) {
    // next edge strictly inside (G1, G4)
    double ev = 0.0, et = 0.0;
    bool have_e = false;
    while (e <= e_hi) {
      const long long idx = e - g.edge_lo;
      if (idx < 0 || idx >= g.n_edges) {
        raise_status(status, CTSM_ERR_TOO_LARGE);
        return false;
      }
      const EdgeAngle E = edges[idx];
      if (sw.G1 < E.be && E.be < sw.G4) {
        ev = E.be;
        et = E.tbe;
        have_e = true;
        break;
      }
      ++e;
    }
    double v, tv;
    if (ci < 4 && (!have_e || !(ev < cv[ci]))) {
      v = cv[ci];
      tv = ct[ci];
      ++ci;
    } else if (have_e) {
      v = ev;
      tv = et;
      ++e;
    } else {
      break;
    }
    if (nb > 0 && sw.brk[nb - 1] == v) continue;  // std::unique
    if (nb == kMaxBrk) {
      raise_status(status, CTSM_ERR_TOO_LARGE);
      return false;
    }
    sw.brk[nb] = v;
    sw.tbrk[nb] = tv;
    ++nb;
  }
  sw.nb = nb;

  int np = 0;
  for (int i = 0; i + 1 < nb; ++i) {
    const double blo = sw.brk[i], bhi = sw.brk[i + 1];
    if (bhi - blo < kEpsPiece) continue;
    const double mid = 0.5 * (blo + bhi);
    sw.pb[np] = (unsigned char)i;
    sw.pcell[np] = (int)floor(crm_tan(mid) * (s + g.d) / g.d_y);
    sw.pkind[np] = (mid <= sw.G2) ? 0 : ((mid <= sw.G3) ? 1 : 2);
    ++np;
  }
  sw.np = np;
  return true;
}

// triangle_area_factor (weights2d.cpp:8-16)
__device__ __forceinline__ double triangle_area_factor(double phi, double gamma_far,
                                                       double gamma_near, double beta, double a,
                                                       double b) {
  if (fabs(crm_sin(gamma_near - gamma_far)) < kEpsAngle) return 0.0;
  if (fabs(crm_sin(beta - phi)) < kEpsAngle) return 0.0;
  const double den = fabs(crm_sin(2.0 * (phi - beta)));
  const double r =
      crm_sin(phi - gamma_near) * crm_sin(beta - gamma_far) / crm_sin(gamma_near - gamma_far);
  return (a / (b * den)) * r * r;
}

// band_area (weights2d.cpp:19-27); cos(phi) supplied (table value).
__device__ __forceinline__ double band_area(double phi, double cphi, double x0, double x1,
                                            double beta_lo, double beta_hi, double s, double b,
                                            int* status) {
  const double c1 = crm_cos(phi - beta_lo), c2 = crm_cos(phi - beta_hi);
  if (fabs(c1) < kEpsAngle || fabs(c2) < kEpsAngle) {
    raise_status(status, CTSM_ERR_RAY_PARALLEL_TO_FACE);
    return 0.0;
  }
  const double xm = 0.5 * (x0 + x1);
  return (1.0 / b) * fabs(s * cphi - xm) * fabs(crm_tan(phi - beta_lo) - crm_tan(phi - beta_hi));
}

// detail::piece_area (weights2d.cpp:89-101)
__device__ __forceinline__ double piece_area(const Sweep& sw, int p, double s, int* status) {
  const double a = sw.x1 - sw.x0, b = sw.y1 - sw.y0;
  const double blo = sw.brk[sw.pb[p]], bhi = sw.brk[sw.pb[p] + 1];
  switch (sw.pkind[p]) {
    case 0:
      return triangle_area_factor(sw.phi, sw.G1, sw.G2, bhi, a, b) -
             triangle_area_factor(sw.phi, sw.G1, sw.G2, blo, a, b);
    case 1:
      return band_area(sw.phi, sw.C, sw.x0, sw.x1, blo, bhi, s, b, status);
    default:
      return triangle_area_factor(sw.phi, sw.G4, sw.G3, blo, a, b) -
             triangle_area_factor(sw.phi, sw.G4, sw.G3, bhi, a, b);
  }
}

// piece_area with the identical sub-expressions of consecutive calls shared
// (bit-preserving: same operations on the same operands, evaluated once):
//   * sin(gamma_near - gamma_far) and sin(phi - gamma_near) depend only on
//     the pixel and the piece kind; the reference evaluates them in every
//     triangle_area_factor call (weights2d.cpp:10-14), twice per piece;
//   * triangle_area_factor at a breakpoint is needed as b_hi of one piece and
//     as b_lo of the next piece of the same kind (weights2d.cpp:93-99), and
//     cos / tan(phi - beta) of band_area (weights2d.cpp:21-26) likewise.
// A pixel's ~6 pieces then cost ~3 crmath calls each instead of 12.
struct AreaCache {
  int tag0 = -1, tag2 = -1, tagb = -1;  // breakpoint whose value is cached
  double val0 = 0.0, val2 = 0.0;        // triangle factor at tag0 (kind 0) / tag2 (kind 2)
  double cb = 0.0, tb = 0.0;            // cos / tan(phi - brk[tagb])
  bool have0 = false, have2 = false;
  double nf0 = 0.0, pn0 = 0.0, nf2 = 0.0, pn2 = 0.0;  // sin(gn - gf), sin(phi - gn) per kind
};

// triangle_area_factor(phi, gamma_far, gamma_near, brk[bi], a, b) for kind 0
// (gamma_far = G1, gamma_near = G2) or kind 2 (G4, G3).
__device__ __forceinline__ double tri_factor_at(const Sweep& sw, int kind, int bi, double a,
                                                double b, AreaCache& c) {
  const double gf = kind == 0 ? sw.G1 : sw.G4, gn = kind == 0 ? sw.G2 : sw.G3;
  double nf, pn;
  if (kind == 0) {
    if (!c.have0) {
      c.nf0 = crm_sin(gn - gf);
      c.pn0 = crm_sin(sw.phi - gn);
      c.have0 = true;
    }
    nf = c.nf0;
    pn = c.pn0;
  } else {
    if (!c.have2) {
      c.nf2 = crm_sin(gn - gf);
      c.pn2 = crm_sin(sw.phi - gn);
      c.have2 = true;
    }
    nf = c.nf2;
    pn = c.pn2;
  }
  const double beta = sw.brk[bi];
  if (fabs(nf) < kEpsAngle) return 0.0;
  if (fabs(crm_sin(beta - sw.phi)) < kEpsAngle) return 0.0;
  const double den = fabs(crm_sin(2.0 * (sw.phi - beta)));
  const double r = pn * crm_sin(beta - gf) / nf;
  return (a / (b * den)) * r * r;
}

__device__ __forceinline__ double piece_area_cached(const Sweep& sw, int p, double s, int* status,
                                                    AreaCache& c) {
  const double a = sw.x1 - sw.x0, b = sw.y1 - sw.y0;
  const int lo = sw.pb[p], hi = lo + 1;
  switch (sw.pkind[p]) {
    case 0: {
      const double tlo = c.tag0 == lo ? c.val0 : tri_factor_at(sw, 0, lo, a, b, c);
      const double thi = tri_factor_at(sw, 0, hi, a, b, c);
      c.tag0 = hi;
      c.val0 = thi;
      return thi - tlo;
    }
    case 1: {
      double c1, t1;
      if (c.tagb == lo) {
        c1 = c.cb;
        t1 = c.tb;
      } else {
        c1 = crm_cos(sw.phi - sw.brk[lo]);
        t1 = crm_tan(sw.phi - sw.brk[lo]);
      }
      const double c2 = crm_cos(sw.phi - sw.brk[hi]);
      const double t2 = crm_tan(sw.phi - sw.brk[hi]);
      c.tagb = hi;
      c.cb = c2;
      c.tb = t2;
      if (fabs(c1) < kEpsAngle || fabs(c2) < kEpsAngle) {
        raise_status(status, CTSM_ERR_RAY_PARALLEL_TO_FACE);
        return 0.0;
      }
      const double xm = 0.5 * (sw.x0 + sw.x1);
      return (1.0 / b) * fabs(s * sw.C - xm) * fabs(t1 - t2);
    }
    default: {
      const double tlo = c.tag2 == lo ? c.val2 : tri_factor_at(sw, 2, lo, a, b, c);
      const double thi = tri_factor_at(sw, 2, hi, a, b, c);
      c.tag2 = hi;
      c.val2 = thi;
      return tlo - thi;
    }
  }
}

// atom_sum lambda (weights3d.cpp:400-423) over pieces [i, j) of one cell.
__device__ __forceinline__ double atom_sum(const Sweep& sw, int i, int j, double s, double a,
                                           double b, double cz, double tan_a, double zref) {
  double v = 0.0;
  for (int k = i; k < j; ++k) {
    const int lo = sw.pb[k];
    const double t_lo = sw.tbrk[lo], t_hi = sw.tbrk[lo + 1];
    switch (sw.pkind[k]) {
      case 0:
        v += tri_atom(sw.S, sw.C, s, a, b, cz, sw.apex1_x, sw.y0, t_hi, tan_a, zref) -
             tri_atom(sw.S, sw.C, s, a, b, cz, sw.apex1_x, sw.y0, t_lo, tan_a, zref);
        break;
      case 1:
        v += trap_atom(sw.S, sw.C, s, a, b, cz, sw.x0, sw.x1, t_lo, t_hi, tan_a, zref);
        break;
      default:
        v += tri_atom(sw.S, sw.C, s, a, b, cz, sw.apex4_x, sw.y1, t_lo, tan_a, zref) -
             tri_atom(sw.S, sw.C, s, a, b, cz, sw.apex4_x, sw.y1, t_hi, tan_a, zref);
    }
  }
  return v;
}

}  // namespace exact
}  // namespace ctsmb
