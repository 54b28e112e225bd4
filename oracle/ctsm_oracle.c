/* ctsm_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's consistent system-matrix hot path.
 *
 * Every function names the reference lines it restates (paths relative to
 * /root/reference/proj). Floating-point expressions keep the reference's
 * operand order and association exactly, and the file
 * is compiled with -ffp-contract=off, so with the same libm the results are
 * bit-identical to the reference's. Two builds exist (oracle/Makefile):
 *   - glibc libm   (-> compare with oracle/_ref/libctsm_ref_glibc.so)
 *   - crmath libm  (-DCTSM_ORACLE_CRMATH; -> compare with libctsm_ref_cr.so
 *                   and, bit-exactly, with the GPU kernels).
 * Errors (the reference throws ctsm::Error, common.hpp:29-42) are raised by
 * longjmp to the entry point, which returns -(ErrorCode ordinal + 1).
 */
#define _GNU_SOURCE
#include "ctsm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <setjmp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef CTSM_ORACLE_CRMATH
#include "crmath.h"
#define O_SIN crm_sin
#define O_COS crm_cos
#define O_TAN crm_tan
#define O_ATAN crm_atan
#define O_ATAN2 crm_atan2
#else
#define O_SIN sin
#define O_COS cos
#define O_TAN tan
#define O_ATAN atan
#define O_ATAN2 atan2
#endif

/* ---- numeric contract (common.hpp:11-57) -------------------------------- */
enum {
  E_DegenerateGeometry = 0, E_RayParallelToFace, E_SingularPhi, E_CentralRow,
  E_ZRestrictionViolation, E_DimensionMismatch, E_NonFinite, E_ZeroMatrix, E_TooLarge,
  E_InvalidSpec, E_OutOfMemory, E_InvalidConfig, E_IoFailure
};
static const char* const k_err_names[] = {
    "DegenerateGeometry", "RayParallelToFace", "SingularPhi", "CentralRow",
    "ZRestrictionViolation", "DimensionMismatch", "NonFinite", "ZeroMatrix", "TooLarge",
    "InvalidSpec", "OutOfMemory", "InvalidConfig", "IoFailure"};

#define K_PI 3.14159265358979323846
#define EPS_DEN_REL 1e-12
#define EPS_ANGLE 1e-12
#define EPS_SINGULAR 1e-8
#define EPS_PIECE 1e-15
#define EPS_WEIGHT 1e-16
#define NEG_CLAMP_2D -1e-14
#define NEG_CLAMP_3D -1e-9
#define CANON_SLACK 1e-13

static double sq(double v) { return v * v; }
static double cube(double v) { return v * v * v; }
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

static __thread char t_err[512];
static __thread jmp_buf* t_jmp;
static __thread int t_code;

static void o_fail(int code, const char* msg) {
  snprintf(t_err, sizeof t_err, "%s: %s", k_err_names[code], msg);
  t_code = code;
  longjmp(*t_jmp, 1);
}

#define O_TRY(...)                              \
  do {                                          \
    jmp_buf jb__;                               \
    jmp_buf* prev__ = t_jmp;                    \
    t_jmp = &jb__;                              \
    if (setjmp(jb__) == 0) {                    \
      __VA_ARGS__                               \
      t_jmp = prev__;                           \
    } else {                                    \
      t_jmp = prev__;                           \
      return -(t_code + 1);                     \
    }                                           \
  } while (0)

const char* ref_last_error(void) { return t_err; }

/* ---- geometry (geometry.hpp:29-84, geometry.cpp:27-97) ------------------- */
static double g_angle(const o_geom* g, int i) {  /* geometry.hpp:50-52 */
  return g->angle_start + (g->angle_end - g->angle_start) * i / g->n_angles;
}
static double face_x(const o_geom* g, double ix) { return (ix - g->n_x / 2.0) * g->a; }
static double face_y(const o_geom* g, double iy) { return (iy - g->n_y / 2.0) * g->b; }
static double face_z(const o_geom* g, double iz) { return (iz - g->n_z / 2.0) * g->c; }
static int is_2d(const o_geom* g) { return g->n_z == 1 && g->n_det_z == 1; }

static void validate(const o_geom* g) {  /* geometry.cpp:27-54 */
  if (!(g->s > 0.0)) o_fail(E_InvalidSpec, "source distance s must be > 0");
  if (!(g->d >= 0.0)) o_fail(E_InvalidSpec, "detector distance d must be >= 0");
  if (!(g->d_y > 0.0) || !(g->d_z > 0.0)) o_fail(E_InvalidSpec, "detector pitches must be > 0");
  if (g->n_det_y <= 0 || g->n_det_z <= 0 || g->n_angles <= 0)
    o_fail(E_InvalidSpec, "detector and angle counts must be > 0");
  if (g->n_det_y % 2 != 0) o_fail(E_InvalidSpec, "n_det_y must be even (centered detector)");
  if (g->n_det_z != 1 && g->n_det_z % 2 != 0)
    o_fail(E_InvalidSpec, "n_det_z must be 1 (2D) or even (centered detector)");
  if (!(g->a > 0.0) || !(g->b > 0.0) || !(g->c > 0.0)) o_fail(E_InvalidSpec, "voxel sizes must be > 0");
  if (g->n_x <= 0 || g->n_y <= 0 || g->n_z <= 0) o_fail(E_InvalidSpec, "grid dimensions must be > 0");
  if (g->n_det_z == 1 && g->n_z > 1) o_fail(E_InvalidSpec, "volume grid requires n_det_z > 1");
  if (!(g->angle_end > g->angle_start)) o_fail(E_InvalidSpec, "angle_end must exceed angle_start");
  if (!isfinite(g->s) || !isfinite(g->d) || !isfinite(g->d_y) || !isfinite(g->d_z) ||
      !isfinite(g->a) || !isfinite(g->b) || !isfinite(g->c) || !isfinite(g->angle_start) ||
      !isfinite(g->angle_end))
    o_fail(E_NonFinite, "geometry parameters must be finite");
  const double rx = g->n_x * g->a / 2.0, ry = g->n_y * g->b / 2.0;
  if (g->s <= hypot(rx, ry)) o_fail(E_DegenerateGeometry, "source circle intersects the grid");
}

/* point_angle (geometry.cpp:56-62) */
static double point_angle(double x, double y, double s, double phi) {
  const double num = y * O_COS(phi) - x * O_SIN(phi);
  const double den = s - y * O_SIN(phi) - x * O_COS(phi);
  if (den <= EPS_DEN_REL * s) o_fail(E_DegenerateGeometry, "point on or behind the source plane");
  return O_ATAN2(num, den);
}

/* vertex_angles (geometry.cpp:64-68): corners (x0,y0),(x1,y0),(x1,y1),(x0,y1) */
static void vertex_angles(double x0, double x1, double y0, double y1, double s, double phi,
                          double gm[4]) {
  gm[0] = point_angle(x0, y0, s, phi);
  gm[1] = point_angle(x1, y0, s, phi);
  gm[2] = point_angle(x1, y1, s, phi);
  gm[3] = point_angle(x0, y1, s, phi);
}

typedef struct {
  double x0, x1, y0, y1, phi;
  int rotations;
} frame2d;

/* canonical_orientation (geometry.cpp:76-97) */
static frame2d canonical_orientation(double x0, double x1, double y0, double y1, double phi,
                                     double s) {
  const double cx = 0.5 * (x0 + x1), cy = 0.5 * (y0 + y1);
  const double chi = O_ATAN2(s * O_SIN(phi) - cy, s * O_COS(phi) - cx);
  const int k0 = ((int)lround(chi / (K_PI / 2)) % 4 + 4) % 4;
  const int tries[4] = {k0, (k0 + 1) % 4, (k0 + 3) % 4, (k0 + 2) % 4};
  for (int ti = 0; ti < 4; ++ti) {
    const int k = tries[ti];
    double fx0 = x0, fx1 = x1, fy0 = y0, fy1 = y1, fphi = phi;
    for (int r = 0; r < k; ++r) {
      const double nx0 = fy0, nx1 = fy1, ny0 = -fx1, ny1 = -fx0;
      fx0 = nx0; fx1 = nx1; fy0 = ny0; fy1 = ny1;
      fphi -= K_PI / 2;
    }
    double gm[4];
    vertex_angles(fx0, fx1, fy0, fy1, s, fphi, gm);
    if (dmax(gm[0], gm[1]) <= dmin(gm[2], gm[3]) + CANON_SLACK) {
      frame2d f = {fx0, fx1, fy0, fy1, fphi, k};
      return f;
    }
  }
  o_fail(E_DegenerateGeometry, "no canonical quadrant found");
  frame2d z = {0, 0, 0, 0, 0, 0};
  return z;
}

/* ---- 2D sweep and area factors (weights2d.cpp) --------------------------- */
#define MAX_BRK 64
typedef struct {
  int cell, kind;
  double apex_x, apex_y, b_lo, b_hi;
} piece;
typedef struct {
  frame2d f;
  double G1, G2, G3, G4;
  int n;
  piece p[MAX_BRK];
} sweep;

/* triangle_area_factor (weights2d.cpp:8-16) */
static double triangle_area_factor(double phi, double gamma_far, double gamma_near, double beta,
                                   double a, double b) {
  if (fabs(O_SIN(gamma_near - gamma_far)) < EPS_ANGLE) return 0.0;
  if (fabs(O_SIN(beta - phi)) < EPS_ANGLE) return 0.0;
  const double den = fabs(O_SIN(2.0 * (phi - beta)));
  const double r = O_SIN(phi - gamma_near) * O_SIN(beta - gamma_far) / O_SIN(gamma_near - gamma_far);
  return (a / (b * den)) * r * r;
}

/* band_area (weights2d.cpp:19-27) */
static double band_area(double phi, double x0, double x1, double beta_lo, double beta_hi, double s,
                        double b) {
  const double c1 = O_COS(phi - beta_lo), c2 = O_COS(phi - beta_hi);
  if (fabs(c1) < EPS_ANGLE || fabs(c2) < EPS_ANGLE)
    o_fail(E_RayParallelToFace, "band ray parallel to x-faces");
  const double xm = 0.5 * (x0 + x1);
  return (1.0 / b) * fabs(s * O_COS(phi) - xm) * fabs(O_TAN(phi - beta_lo) - O_TAN(phi - beta_hi));
}

/* detail::strip_sweep (weights2d.cpp:38-87) */
static void strip_sweep(double x0, double x1, double y0, double y1, double phi, double s,
                        double d, double d_y, sweep* sw) {
  sw->f = canonical_orientation(x0, x1, y0, y1, phi, s);
  double gm[4];
  vertex_angles(sw->f.x0, sw->f.x1, sw->f.y0, sw->f.y1, s, sw->f.phi, gm);
  sw->G1 = dmin(gm[0], gm[1]);
  sw->G2 = dmax(gm[0], gm[1]);
  sw->G3 = dmin(gm[2], gm[3]);
  sw->G4 = dmax(gm[2], gm[3]);
  const double apex1_x = (gm[0] <= gm[1]) ? sw->f.x0 : sw->f.x1;
  const double apex4_x = (gm[3] >= gm[2]) ? sw->f.x0 : sw->f.x1;

  double brk[MAX_BRK];
  int nb = 0;
  brk[nb++] = sw->G1;
  brk[nb++] = sw->G2;
  brk[nb++] = sw->G3;
  brk[nb++] = sw->G4;
  const double t_lo = O_TAN(sw->G1) * (s + d) / d_y;
  const double t_hi = O_TAN(sw->G4) * (s + d) / d_y;
  const long long e_lo = (long long)floor(t_lo) + 1;
  const long long e_hi = (long long)ceil(t_hi) - 1;
  for (long long e = e_lo; e <= e_hi; ++e) {
    const double be = O_ATAN(e * d_y / (s + d));
    if (sw->G1 < be && be < sw->G4) {
      if (nb == MAX_BRK) o_fail(E_TooLarge, "oracle sweep breakpoint capacity exceeded");
      brk[nb++] = be;
    }
  }
  /* std::sort + std::unique (weights2d.cpp:62-63) */
  for (int i = 1; i < nb; ++i) {
    const double v = brk[i];
    int j = i - 1;
    while (j >= 0 && v < brk[j]) {
      brk[j + 1] = brk[j];
      --j;
    }
    brk[j + 1] = v;
  }
  int nu = 0;
  for (int i = 0; i < nb; ++i)
    if (nu == 0 || !(brk[nu - 1] == brk[i])) brk[nu++] = brk[i];

  sw->n = 0;
  for (int i = 0; i + 1 < nu; ++i) {
    const double blo = brk[i], bhi = brk[i + 1];
    if (bhi - blo < EPS_PIECE) continue;
    const double mid = 0.5 * (blo + bhi);
    piece p;
    p.cell = (int)floor(O_TAN(mid) * (s + d) / d_y);
    p.b_lo = blo;
    p.b_hi = bhi;
    p.apex_x = 0;
    p.apex_y = 0;
    if (mid <= sw->G2) {
      p.kind = 0;
      p.apex_x = apex1_x;
      p.apex_y = sw->f.y0;
    } else if (mid <= sw->G3) {
      p.kind = 1;
    } else {
      p.kind = 2;
      p.apex_x = apex4_x;
      p.apex_y = sw->f.y1;
    }
    sw->p[sw->n++] = p;
  }
}

/* detail::piece_area (weights2d.cpp:89-101) */
static double piece_area(const sweep* sw, const piece* p, double s) {
  const double a = sw->f.x1 - sw->f.x0, b = sw->f.y1 - sw->f.y0;
  switch (p->kind) {
    case 0:
      return triangle_area_factor(sw->f.phi, sw->G1, sw->G2, p->b_hi, a, b) -
             triangle_area_factor(sw->f.phi, sw->G1, sw->G2, p->b_lo, a, b);
    case 1:
      return band_area(sw->f.phi, sw->f.x0, sw->f.x1, p->b_lo, p->b_hi, s, b);
    default:
      return triangle_area_factor(sw->f.phi, sw->G4, sw->G3, p->b_lo, a, b) -
             triangle_area_factor(sw->f.phi, sw->G4, sw->G3, p->b_hi, a, b);
  }
}

typedef struct {
  int m_y, m_z;
  double w;
} weight;
#define MAX_W 256

/* pixel_area_factors (weights2d.cpp:105-129) */
static int pixel_area_factors(int ix, int iy, double phi, const o_geom* g, weight* out) {
  sweep sw;
  strip_sweep(face_x(g, ix), face_x(g, ix + 1), face_y(g, iy), face_y(g, iy + 1), phi, g->s,
              g->d, g->d_y, &sw);
  const int cell_lo = -g->n_det_y / 2, cell_hi = g->n_det_y / 2 - 1;
  int n = 0;
  for (int i = 0; i < sw.n; ++i) {
    const piece* p = &sw.p[i];
    if (p->cell < cell_lo || p->cell > cell_hi) continue;
    double w = piece_area(&sw, p, g->s);
    if (w < 0.0) {
      if (w < NEG_CLAMP_2D) o_fail(E_NonFinite, "negative area weight beyond FP tolerance");
      w = 0.0;
    }
    if (n > 0 && out[n - 1].m_y == p->cell) {
      out[n - 1].w += w;
    } else {
      out[n].m_y = p->cell;
      out[n].m_z = 0;
      out[n].w = w;
      ++n;
    }
  }
  int k = 0; /* erase weights <= eps (weights2d.cpp:125-127) */
  for (int i = 0; i < n; ++i)
    if (!(out[i].w <= EPS_WEIGHT)) out[k++] = out[i];
  return k;
}

/* ---- 3D atoms (weights3d.cpp:42-168) ------------------------------------- */
typedef struct {
  int g1, f1, g2, f2;
} trap_flags;
typedef struct {
  int g, h, gg;
} tri_flags;

/* trap_face_part (weights3d.cpp:51-61) */
static double trap_face_part(double G, double P, double S, double t1, double t2, double cr1,
                             double cr2, int flag1, int flag2) {
  if (flag1 && flag2)
    return (t1 - t2) * (cube(G) - 3.0 * G * P * P / (cr1 * cr2) + cube(P) * (cr1 + cr2) / sq(cr1 * cr2));
  if (!flag1 && !flag2) return 0.0;
  double v = 0.0;
  if (flag1) v += cr1 * cube(G - P / cr1);
  if (flag2) v -= cr2 * cube(G - P / cr2);
  return v / S;
}

/* trap_flags_at (weights3d.cpp:63-83) */
static trap_flags trap_flags_at(double phi, double s, double a, double x0, double x1, double beta1,
                                double beta2, double tan_a, double zref) {
  const double S = O_SIN(phi), C = O_COS(phi);
  const double G = zref / (a * tan_a);
  trap_flags fl = {0, 0, 0, 0};
  if (fabs(S) > EPS_SINGULAR) {
    const double t1 = O_TAN(beta1), t2 = O_TAN(beta2);
    const double cr1 = C + S * t1, cr2 = C + S * t2;
    const double Pg = (s * C - x1) / a, Pf = (s * C - x0) / a;
    fl.g1 = (G - Pg / cr1) > 0.0;
    fl.g2 = (G - Pg / cr2) > 0.0;
    fl.f1 = (G - Pf / cr1) > 0.0;
    fl.f2 = (G - Pf / cr2) > 0.0;
  } else {
    const int gs = (G - (s * C - x1) / a) > 0.0;
    const int fs = (G - (s * C - x0) / a) > 0.0;
    fl.g1 = fl.g2 = gs;
    fl.f1 = fl.f2 = fs;
  }
  return fl;
}

/* trap_atom_flags (weights3d.cpp:85-107) */
static double trap_atom_flags(double phi, double s, double a, double b, double c, double x0,
                              double x1, double beta1, double beta2, double tan_a, double zref,
                              trap_flags fl) {
  const double S = O_SIN(phi), C = O_COS(phi);
  const double G = zref / (a * tan_a);
  const double t1 = O_TAN(beta1), t2 = O_TAN(beta2);
  if (fabs(S) > EPS_SINGULAR) {
    const double cr1 = C + S * t1, cr2 = C + S * t2;
    const double pg = trap_face_part(G, (s * C - x1) / a, S, t1, t2, cr1, cr2, fl.g1, fl.g2);
    const double pf = trap_face_part(G, (s * C - x0) / a, S, t1, t2, cr1, cr2, fl.f1, fl.f2);
    return (a * a / (6.0 * b * c)) * fabs(tan_a * (pg - pf));
  }
  const double g = G - (s * C - x1) / a;
  const double f = G - (s * C - x0) / a;
  double t = 0.0;
  if (fl.g1) t += g * g * (g + 3.0 * (s * C - x1) / a);
  if (fl.f1) t -= f * f * (f + 3.0 * (s * C - x0) / a);
  return (a * a / (6.0 * b * c)) * fabs(tan_a * t * (t1 - t2));
}

/* tri_flags_at (weights3d.cpp:115-127) */
static tri_flags tri_flags_at(double phi, double s, double a, double xa, double ya, double beta,
                              double tan_a, double zref) {
  const double S = O_SIN(phi), C = O_COS(phi);
  const double G = zref / (a * tan_a);
  const double t = O_TAN(beta);
  const double crg = C + S * t, srh = S - C * t;
  const double P = (s * C - xa) / a, Q = (s * S - ya) / a;
  tri_flags fl;
  fl.g = (G - P / crg) > 0.0;
  fl.gg = (G - P * C - Q * S) > 0.0;
  fl.h = (G - Q / srh) > 0.0;
  return fl;
}

/* tri_atom_flags (weights3d.cpp:129-168) */
static double tri_atom_flags(double phi, double s, double a, double b, double c, double xa,
                             double ya, double beta, double tan_a, double zref, tri_flags fl) {
  const double S = O_SIN(phi), C = O_COS(phi);
  const double G = zref / (a * tan_a);
  const double t = O_TAN(beta);
  const double crg = C + S * t;
  const double srh = S - C * t;
  const double P = (s * C - xa) / a;
  const double Q = (s * S - ya) / a;
  const double g = G - P / crg;
  const double gg = G - P * C - Q * S;
  const double h = G - Q / srh;
  if (fabs(S) > EPS_SINGULAR) {
    double pair;
    if (fl.g && fl.gg) {
      const double delta = Q - P * srh / crg;
      pair = crg * (3.0 * gg * gg * delta + 3.0 * gg * S * delta * delta + S * S * cube(delta)) -
             cube(gg) * srh / C;
    } else if (!fl.g && !fl.gg) {
      pair = 0.0;
    } else {
      double v = 0.0;
      if (fl.g) v += crg * cube(g);
      if (fl.gg) v -= cube(gg) / C;
      pair = v / S;
    }
    const double tt = pair + (fl.h ? (srh / C) * cube(h) : 0.0);
    return (a * a / (6.0 * b * c)) * fabs(tan_a * tt);
  }
  double tv = 0.0;
  if (fl.g) tv += g * g * (t * g - 3.0 * t * (g - h));
  if (fl.h) tv -= t * cube(h);
  return (a * a / (6.0 * b * c)) * fabs(tan_a * tv);
}

/* detail::trap_atom / detail::tri_atom_cum (weights3d.cpp:176-190) */
static double trap_atom(double phi, double s, double a, double b, double c, double x0, double x1,
                        double beta1, double beta2, double tan_alpha, double zref) {
  const trap_flags fl = trap_flags_at(phi, s, a, x0, x1, beta1, beta2, tan_alpha, zref);
  return trap_atom_flags(phi, s, a, b, c, x0, x1, beta1, beta2, tan_alpha, zref, fl);
}
static double tri_atom_cum(double phi, double s, double a, double b, double c, double xa,
                           double ya, double beta, double tan_alpha, double zref) {
  const tri_flags fl = tri_flags_at(phi, s, a, xa, ya, beta, tan_alpha, zref);
  return tri_atom_flags(phi, s, a, b, c, xa, ya, beta, tan_alpha, zref, fl);
}

/* atom_sum lambda (weights3d.cpp:400-423) over pieces [i, j) of one cell */
static double atom_sum(const sweep* sw, int i, int j, const o_geom* g, double a, double b,
                       double cz, double tan_a, double zref) {
  double v = 0.0;
  for (int k = i; k < j; ++k) {
    const piece* p = &sw->p[k];
    switch (p->kind) {
      case 0:
        v += tri_atom_cum(sw->f.phi, g->s, a, b, cz, p->apex_x, p->apex_y, p->b_hi, tan_a, zref) -
             tri_atom_cum(sw->f.phi, g->s, a, b, cz, p->apex_x, p->apex_y, p->b_lo, tan_a, zref);
        break;
      case 1:
        v += trap_atom(sw->f.phi, g->s, a, b, cz, sw->f.x0, sw->f.x1, p->b_lo, p->b_hi, tan_a, zref);
        break;
      default:
        v += tri_atom_cum(sw->f.phi, g->s, a, b, cz, p->apex_x, p->apex_y, p->b_lo, tan_a, zref) -
             tri_atom_cum(sw->f.phi, g->s, a, b, cz, p->apex_x, p->apex_y, p->b_hi, tan_a, zref);
    }
  }
  return v;
}

/* voxel_volume_factors (weights3d.cpp:354-462) */
static int voxel_volume_factors(int ix, int iy, int iz, double phi, const o_geom* g,
                                weight* out, int cap) {
  sweep sw;
  strip_sweep(face_x(g, ix), face_x(g, ix + 1), face_y(g, iy), face_y(g, iy + 1), phi, g->s,
              g->d, g->d_y, &sw);
  const double a = sw.f.x1 - sw.f.x0, b = sw.f.y1 - sw.f.y0;
  const double zb = face_z(g, iz), zt = face_z(g, iz + 1);
  const double cz = zt - zb;
  const double sdd = g->s + g->d;

  double m_min = 0.0, m_max = 0.0;
  int first = 1;
  const double vxs[2] = {sw.f.x0, sw.f.x1}, vys[2] = {sw.f.y0, sw.f.y1}, vzs[2] = {zb, zt};
  for (int ixc = 0; ixc < 2; ++ixc)
    for (int iyc = 0; iyc < 2; ++iyc) {
      const double depth = g->s - vxs[ixc] * O_COS(sw.f.phi) - vys[iyc] * O_SIN(sw.f.phi);
      if (depth <= EPS_DEN_REL * g->s) o_fail(E_DegenerateGeometry, "voxel corner on the source plane");
      for (int izc = 0; izc < 2; ++izc) {
        const double m = sdd / g->d_z * vzs[izc] / depth;
        m_min = first ? m : dmin(m_min, m);
        m_max = first ? m : dmax(m_max, m);
        first = 0;
      }
    }

  const int cell_lo = -g->n_det_y / 2, cell_hi = g->n_det_y / 2 - 1;
  const int row_lo = -g->n_det_z / 2, row_hi = g->n_det_z / 2 - 1;
  int n = 0;
  int i = 0;
  while (i < sw.n) {
    int j = i;
    while (j < sw.n && sw.p[j].cell == sw.p[i].cell) ++j;
    const int cell = sw.p[i].cell;
    if (cell < cell_lo || cell > cell_hi) {
      i = j;
      continue;
    }
    double w2d = 0.0;
    for (int k = i; k < j; ++k) w2d += piece_area(&sw, &sw.p[k], g->s);
    if (w2d < 0.0) w2d = 0.0;

    const int fl_lo = (int)floor(m_min);
    const int k_lo = (fl_lo < row_lo) ? row_lo : fl_lo; /* std::max */
    const int k_hi_raw = (int)ceil(m_max) - 1;
    const int k_hi = k_hi_raw < row_hi ? k_hi_raw : row_hi;
    if (k_hi < k_lo) {
      i = j;
      continue;
    }
    double edge_above[MAX_W + 2];
    if (k_hi - k_lo + 2 > MAX_W + 2) o_fail(E_TooLarge, "oracle row-edge capacity exceeded");
    for (int L = k_lo; L <= k_hi + 1; ++L) {
      const double k = (double)L;
      double v;
      /* above(k) lambda (weights3d.cpp:426-440) */
      if (k <= m_min) {
        v = w2d;
      } else if (k >= m_max) {
        v = 0.0;
      } else if (k == 0.0) {
        if (zb >= 0.0) v = w2d;
        else if (zt <= 0.0) v = 0.0;
        else v = w2d * zt / (zt - zb);
      } else if (k > 0.0) {
        const double tan_a = k * g->d_z / sdd;
        v = atom_sum(&sw, i, j, g, a, b, cz, tan_a, zt) - atom_sum(&sw, i, j, g, a, b, cz, tan_a, zb);
      } else {
        const double tan_a = -k * g->d_z / sdd;
        v = w2d - (atom_sum(&sw, i, j, g, a, b, cz, tan_a, -zb) -
                   atom_sum(&sw, i, j, g, a, b, cz, tan_a, -zt));
      }
      edge_above[L - k_lo] = v;
    }
    for (int L = k_lo; L <= k_hi; ++L) {
      const double v = edge_above[L - k_lo] - edge_above[L - k_lo + 1];
      if (v > EPS_WEIGHT) {
        if (n == cap) o_fail(E_TooLarge, "oracle weight capacity exceeded");
        out[n].m_y = cell;
        out[n].m_z = L;
        out[n].w = v;
        ++n;
      } else if (v < NEG_CLAMP_3D) {
        o_fail(E_NonFinite, "negative volume weight beyond FP tolerance");
      }
    }
    i = j;
  }
  return n;
}

/* ---- public weight entry points ----------------------------------------- */
int ref_validate(const o_geom* g) {
  O_TRY(validate(g););
  return 0;
}
double ref_angle(const o_geom* g, int i) { return g_angle(g, i); }

long ref_pixel_area_factors(const o_geom* g, int ix, int iy, double phi, int32_t* my, double* w,
                            long cap) {
  weight buf[MAX_W];
  int n = 0;
  O_TRY(n = pixel_area_factors(ix, iy, phi, g, buf););
  for (int i = 0; i < n && i < cap; ++i) {
    my[i] = buf[i].m_y;
    w[i] = buf[i].w;
  }
  return n;
}

long ref_voxel_volume_factors(const o_geom* g, int ix, int iy, int iz, double phi, int32_t* my,
                              int32_t* mz, double* w, long cap) {
  weight buf[MAX_W];
  int n = 0;
  O_TRY(n = voxel_volume_factors(ix, iy, iz, phi, g, buf, MAX_W););
  for (int i = 0; i < n && i < cap; ++i) {
    my[i] = buf[i].m_y;
    mz[i] = buf[i].m_z;
    w[i] = buf[i].w;
  }
  return n;
}

/* ---- angle blocks (projector.cpp:44-84) ---------------------------------- */
typedef void (*emit_fn)(void* ctx, uint32_t row, uint32_t col, double w);

/* Entries of the voxels with slow index (iz in 3D, iy in 2D) in [lo, hi), in
 * the reference's emission order; the full block is [0, n). Splitting a block
 * into slabs only parallelises the oracle; it does not change any weight. */
static void angle_block_entries_slab(const o_geom* g, int ip, int lo, int hi, emit_fn emit,
                                     void* ctx) {
  const double phi = g_angle(g, ip);
  weight buf[MAX_W];
  if (is_2d(g)) {
    for (int iy = lo; iy < hi; ++iy)
      for (int ix = 0; ix < g->n_x; ++ix) {
        const uint32_t col = (uint32_t)((uint64_t)iy * g->n_x + ix);
        const int n = pixel_area_factors(ix, iy, phi, g, buf);
        for (int k = 0; k < n; ++k)
          emit(ctx, (uint32_t)((0 + g->n_det_z / 2) * g->n_det_y + (buf[k].m_y + g->n_det_y / 2)),
               col, buf[k].w);
      }
  } else {
    for (int iz = lo; iz < hi; ++iz)
      for (int iy = 0; iy < g->n_y; ++iy)
        for (int ix = 0; ix < g->n_x; ++ix) {
          const uint32_t col = (uint32_t)(((uint64_t)iz * g->n_y + iy) * g->n_x + ix);
          const int n = voxel_volume_factors(ix, iy, iz, phi, g, buf, MAX_W);
          for (int k = 0; k < n; ++k)
            emit(ctx,
                 (uint32_t)((buf[k].m_z + g->n_det_z / 2) * g->n_det_y +
                            (buf[k].m_y + g->n_det_y / 2)),
                 col, buf[k].w);
        }
  }
}

static int slab_extent(const o_geom* g) { return is_2d(g) ? g->n_y : g->n_z; }

static void angle_block_entries(const o_geom* g, int ip, emit_fn emit, void* ctx) {
  angle_block_entries_slab(g, ip, 0, slab_extent(g), emit, ctx);
}

typedef struct {
  uint32_t* row;
  uint32_t* col;
  double* w;
  long n, cap;
} entry_sink;
static void sink_emit(void* ctx, uint32_t r, uint32_t c, double w) {
  entry_sink* s = (entry_sink*)ctx;
  if (s->n < s->cap) {
    s->row[s->n] = r;
    s->col[s->n] = c;
    s->w[s->n] = w;
  }
  s->n++;
}

long ref_angle_block_entries(const o_geom* g, int ip, uint32_t* row, uint32_t* col, double* w,
                             long cap) {
  entry_sink s = {row, col, w, 0, cap};
  O_TRY(angle_block_entries(g, ip, sink_emit, &s););
  return s.n;
}

/* growable per-angle entry list */
typedef struct {
  uint32_t* row;
  uint32_t* col;
  double* w;
  long n, cap;
} entry_vec;
static void vec_emit(void* ctx, uint32_t r, uint32_t c, double w) {
  entry_vec* v = (entry_vec*)ctx;
  if (v->n == v->cap) {
    long nc = v->cap ? 2 * v->cap : 4096;
    v->row = (uint32_t*)realloc(v->row, nc * sizeof(uint32_t));
    v->col = (uint32_t*)realloc(v->col, nc * sizeof(uint32_t));
    v->w = (double*)realloc(v->w, nc * sizeof(double));
    if (!v->row || !v->col || !v->w) o_fail(E_OutOfMemory, "host allocation failed");
    v->cap = nc;
  }
  v->row[v->n] = r;
  v->col[v->n] = c;
  v->w[v->n] = w;
  v->n++;
}
static void vec_free(entry_vec* v) {
  free(v->row);
  free(v->col);
  free(v->w);
  memset(v, 0, sizeof *v);
}

/* ---- thread pool over angles (ordered results, cf. projector.cpp:114-140) - */
typedef struct task task;
typedef void (*task_fn)(task* t, int item, int worker);
struct task {
  task_fn fn;
  const o_geom* g;
  int count, threads;
  int next;
  pthread_mutex_t mu;
  int err_code;
  char err[512];
  void* user;
};
typedef struct {
  task* t;
  int worker;
} worker_arg;

static void* worker_main(void* p) {
  worker_arg* wa = (worker_arg*)p;
  task* t = wa->t;
  for (;;) {
    pthread_mutex_lock(&t->mu);
    volatile int item = t->err_code >= 0 ? t->count : t->next++;
    pthread_mutex_unlock(&t->mu);
    if (item >= t->count) break;
    jmp_buf jb;
    jmp_buf* prev = t_jmp;
    t_jmp = &jb;
    if (setjmp(jb) == 0) {
      t->fn(t, item, wa->worker);
      t_jmp = prev;
    } else {
      t_jmp = prev;
      pthread_mutex_lock(&t->mu);
      if (t->err_code < 0) {
        t->err_code = t_code;
        memcpy(t->err, t_err, sizeof t->err);
      }
      pthread_mutex_unlock(&t->mu);
    }
  }
  return NULL;
}

/* runs fn(item) for all items; returns 0 or -(code+1) */
static int run_tasks(task* t) {
  t->next = 0;
  t->err_code = -1;
  pthread_mutex_init(&t->mu, NULL);
  int nth = t->threads < 1 ? 1 : t->threads;
  if (nth > t->count) nth = t->count;
  if (nth < 1) nth = 1;
  pthread_t th[256];
  worker_arg wa[256];
  if (nth > 256) nth = 256;
  for (int i = 0; i < nth; ++i) {
    wa[i].t = t;
    wa[i].worker = i;
    pthread_create(&th[i], NULL, worker_main, &wa[i]);
  }
  for (int i = 0; i < nth; ++i) pthread_join(th[i], NULL);
  pthread_mutex_destroy(&t->mu);
  if (t->err_code >= 0) {
    memcpy(t_err, t->err, sizeof t_err);
    return -(t->err_code + 1);
  }
  return 0;
}

/* angle_block_entries split into slabs on threads; the slab entry lists are
 * concatenated in slab order, so the result is identical (same entries, same
 * emission order) to the sequential reference loop. */
typedef struct {
  int ip, n_parts;
  entry_vec* parts;
} blockpar_user;
static void blockpar_task(task* t, int item, int worker) {
  (void)worker;
  blockpar_user* u = (blockpar_user*)t->user;
  const int n = slab_extent(t->g);
  const int lo = (int)((int64_t)n * item / u->n_parts), hi = (int)((int64_t)n * (item + 1) / u->n_parts);
  angle_block_entries_slab(t->g, u->ip, lo, hi, vec_emit, &u->parts[item]);
}

long ref_angle_block_entries_par(const o_geom* g, int ip, uint32_t* row, uint32_t* col, double* w,
                                 long cap, int threads) {
  O_TRY(validate(g););
  int n_parts = threads < 1 ? 1 : threads;
  if (n_parts > slab_extent(g)) n_parts = slab_extent(g);
  entry_vec* parts = (entry_vec*)calloc(n_parts, sizeof(entry_vec));
  blockpar_user u = {ip, n_parts, parts};
  task t;
  memset(&t, 0, sizeof t);
  t.fn = blockpar_task;
  t.g = g;
  t.count = n_parts;
  t.threads = threads;
  t.user = &u;
  const int st = run_tasks(&t);
  long n = 0;
  if (st == 0)
    for (int p = 0; p < n_parts; ++p)
      for (long k = 0; k < parts[p].n; ++k, ++n)
        if (n < cap) {
          row[n] = parts[p].row[k];
          col[n] = parts[p].col[k];
          w[n] = parts[p].w[k];
        }
  for (int p = 0; p < n_parts; ++p) vec_free(&parts[p]);
  free(parts);
  return st != 0 ? st : n;
}

/* ---- line / multiline baselines (baseline.cpp:13-128) --------------------
 * The paper's comparison method: exact intersection
 * lengths of one (line) or k resp. k*k (multiline) rays per detector cell. */
typedef struct {
  uint32_t col;
  double len;
  long seq; /* emission index: makes the column sort stable (merge_hits) */
} ray_hit;
typedef struct {
  ray_hit* h;
  long n, cap;
} hit_vec;
static void hit_push(hit_vec* v, uint32_t col, double len) {
  if (v->n == v->cap) {
    long nc = v->cap ? 2 * v->cap : 1024;
    v->h = (ray_hit*)realloc(v->h, nc * sizeof(ray_hit));
    if (!v->h) o_fail(E_OutOfMemory, "host allocation failed");
    v->cap = nc;
  }
  v->h[v->n].col = col;
  v->h[v->n].len = len;
  v->h[v->n].seq = v->n;
  v->n++;
}

/* trace_ray (baseline.cpp:13-67): incremental grid traversal from the origin
 * along a unit direction; (column, length * scale) for every crossed voxel. */
static void trace_ray(double ox, double oy, double oz, double ux, double uy, double uz,
                      const o_geom* g, double scale, hit_vec* out) {
  const double lo[3] = {face_x(g, 0), face_y(g, 0), face_z(g, 0)};
  const double hi[3] = {face_x(g, g->n_x), face_y(g, g->n_y), face_z(g, g->n_z)};
  const double org[3] = {ox, oy, oz};
  const double dir[3] = {ux, uy, uz};
  const double pitch[3] = {g->a, g->b, g->c};
  const int dims[3] = {g->n_x, g->n_y, g->n_z};
  double tmin = 0.0, tmax = INFINITY;
  for (int ax = 0; ax < 3; ++ax) {
    if (fabs(dir[ax]) < 1e-15) {
      if (org[ax] < lo[ax] || org[ax] > hi[ax]) return;
      continue;
    }
    double ta = (lo[ax] - org[ax]) / dir[ax];
    double tb = (hi[ax] - org[ax]) / dir[ax];
    if (ta > tb) {
      const double t = ta;
      ta = tb;
      tb = t;
    }
    tmin = dmax(tmin, ta);
    tmax = dmin(tmax, tb);
  }
  if (tmax <= tmin) return;
  const double eps = 1e-12 * dmin(dmin(g->a, g->b), g->c);
  int idx[3];
  for (int ax = 0; ax < 3; ++ax) {
    const double p = org[ax] + (tmin + eps) * dir[ax];
    idx[ax] = (int)floor((p - lo[ax]) / pitch[ax]);
  }
  double t = tmin;
  while (t < tmax - eps) {
    int inside = 1;
    for (int ax = 0; ax < 3; ++ax) inside = inside && idx[ax] >= 0 && idx[ax] < dims[ax];
    if (!inside) break;
    double tn = tmax;
    int step_ax = -1;
    for (int ax = 0; ax < 3; ++ax) {
      if (dir[ax] == 0.0) continue;
      const int f = idx[ax] + (dir[ax] > 0 ? 1 : 0);
      const double tc = (lo[ax] + f * pitch[ax] - org[ax]) / dir[ax];
      if (tc < tn) {
        tn = tc;
        step_ax = ax;
      }
    }
    if (tn > t)
      hit_push(out, (uint32_t)(((uint64_t)idx[2] * g->n_y + idx[1]) * g->n_x + idx[0]),
               (tn - t) * scale);
    if (step_ax < 0 || tn >= tmax) break;
    idx[step_ax] += dir[step_ax] > 0 ? 1 : -1;
    t = tn;
  }
}

/* cell_ray (baseline.cpp:69-79) with detector_point (geometry.hpp:108-113). */
static void cell_ray(double e_y, double e_z, int ip, const o_geom* g, double scale,
                     hit_vec* out) {
  const double phi = g_angle(g, ip);
  const double ox = g->s * O_COS(phi), oy = g->s * O_SIN(phi);
  const double cp = O_COS(phi), sp = O_SIN(phi);
  const double dx = -g->d * cp - e_y * g->d_y * sp, dy = -g->d * sp + e_y * g->d_y * cp,
               dz = e_z * g->d_z;
  double ux = dx - ox, uy = dy - oy, uz = dz;
  const double nrm = sqrt(ux * ux + uy * uy + uz * uz);
  ux /= nrm;
  uy /= nrm;
  uz /= nrm;
  trace_ray(ox, oy, 0.0, ux, uy, uz, g, scale, out);
}

static int hit_cmp(const void* a, const void* b) {
  const ray_hit* x = (const ray_hit*)a;
  const ray_hit* y = (const ray_hit*)b;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}
/* merge_hits (baseline.cpp:81-94): stable sort by column, lengths of equal
 * columns summed in emission order. */
static void merge_hits(hit_vec* v) {
  qsort(v->h, v->n, sizeof(ray_hit), hit_cmp);
  long m = 0;
  for (long i = 0; i < v->n; ++i) {
    if (m > 0 && v->h[m - 1].col == v->h[i].col)
      v->h[m - 1].len += v->h[i].len;
    else
      v->h[m++] = v->h[i];
  }
  v->n = m;
}

/* line_weights / multiline_weights (baseline.cpp:98-128). mode 1 = line,
 * 2 = multiline (MatrixMode order, projector.hpp:12-16). */
static void ray_weights(const o_geom* g, int mode, int k, int m_y, int m_z, int ip,
                        hit_vec* out) {
  out->n = 0;
  if (mode == 2 && k <= 0) o_fail(E_InvalidSpec, "multiline ray count must be > 0");
  if (m_y < -g->n_det_y / 2 || m_y >= g->n_det_y / 2)
    o_fail(E_InvalidSpec, "detector cell m_y out of range");
  if (is_2d(g) && m_z != 0) o_fail(E_InvalidSpec, "m_z must be 0 for a 2D scan");
  if (!is_2d(g) && (m_z < -g->n_det_z / 2 || m_z >= g->n_det_z / 2))
    o_fail(E_InvalidSpec, "detector cell m_z out of range");
  if (mode == 1 || k == 1) {
    cell_ray(m_y + 0.5, is_2d(g) ? 0.0 : (m_z + 0.5), ip, g, 1.0, out);
    if (mode == 2) merge_hits(out);
    return;
  }
  if (is_2d(g)) {
    for (int i = 0; i < k; ++i) cell_ray(m_y + (i + 0.5) / k, 0.0, ip, g, 1.0 / k, out);
  } else {
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j)
        cell_ray(m_y + (i + 0.5) / k, m_z + (j + 0.5) / k, ip, g, 1.0 / ((double)k * k), out);
  }
  merge_hits(out);
}

long ref_line_weights(const o_geom* g, int mode, int k, int m_y, int m_z, int ip, uint32_t* col,
                      double* len, long cap) {
  hit_vec v = {0};
  long n = 0;
  int st = 0;
  {
    jmp_buf jb;
    jmp_buf* prev = t_jmp;
    t_jmp = &jb;
    if (setjmp(jb) == 0) {
      ray_weights(g, mode, k, m_y, m_z, ip, &v);
      t_jmp = prev;
    } else {
      t_jmp = prev;
      st = -(t_code + 1);
    }
  }
  if (st == 0) {
    n = v.n;
    for (long i = 0; i < v.n && i < cap; ++i) {
      col[i] = v.h[i].col;
      len[i] = v.h[i].len;
    }
  }
  free(v.h);
  return st != 0 ? st : n;
}

/* angle_block_entries for the ray modes (projector.cpp:72-83): rows in raster
 * order (m_z outer, m_y inner), hits of each row in the ray's order. */
static void angle_block_entries_rays(const o_geom* g, int mode, int k, int ip, emit_fn emit,
                                     void* ctx) {
  const int mz_lo = is_2d(g) ? 0 : -g->n_det_z / 2;
  const int mz_hi = is_2d(g) ? 0 : g->n_det_z / 2 - 1;
  hit_vec v = {0};
  for (int m_z = mz_lo; m_z <= mz_hi; ++m_z)
    for (int m_y = -g->n_det_y / 2; m_y < g->n_det_y / 2; ++m_y) {
      ray_weights(g, mode, k, m_y, m_z, ip, &v);
      const uint32_t row =
          (uint32_t)((m_z + g->n_det_z / 2) * g->n_det_y + (m_y + g->n_det_y / 2));
      for (long i = 0; i < v.n; ++i) emit(ctx, row, v.h[i].col, v.h[i].len);
    }
  free(v.h);
}

static void angle_block_entries_mode(const o_geom* g, int mode, int k, int ip, emit_fn emit,
                                     void* ctx) {
  if (mode == 0)
    angle_block_entries(g, ip, emit, ctx);
  else
    angle_block_entries_rays(g, mode, k, ip, emit, ctx);
}

long ref_angle_block_entries_mode(const o_geom* g, int mode, int k, int ip, uint32_t* row,
                                  uint32_t* col, double* w, long cap) {
  entry_sink s = {row, col, w, 0, cap};
  O_TRY(validate(g); angle_block_entries_mode(g, mode, k, ip, sink_emit, &s););
  return s.n;
}

/* ---- build_system_matrix (projector.cpp:144-201) -------------------------- */
typedef struct {
  uint64_t n_rows, n_cols;
  uint64_t* row_start;
  uint32_t* col;
  double* val;
  uint64_t nnz;
} csr;

/* build_angle_block (projector.cpp:92-104): entries of one angle bucketed by
 * row; within a row the emission order is already ascending in column (voxels
 * are visited in column order and emit at most once per row), so a stable
 * counting sort by row reproduces the reference's stable_sort result. */
static void bucket_by_row(const entry_vec* v, uint64_t rpa, uint64_t* counts, uint32_t* col_out,
                          double* val_out, int sort_rows) {
  uint64_t* pos = (uint64_t*)calloc(rpa + 1, sizeof(uint64_t));
  for (long i = 0; i < v->n; ++i) pos[v->row[i] + 1]++;
  for (uint64_t r = 0; r < rpa; ++r) {
    counts[r] = pos[r + 1];
    pos[r + 1] += pos[r];
  }
  for (long i = 0; i < v->n; ++i) {
    const uint64_t p = pos[v->row[i]]++;
    col_out[p] = v->col[i];
    val_out[p] = v->w[i];
  }
  free(pos);
  if (!sort_rows) return;
  /* ray modes: a row's hits come in ray order -> stable_sort by column
   * (projector.cpp:100-102) */
  hit_vec tmp = {0};
  uint64_t off = 0;
  for (uint64_t r = 0; r < rpa; ++r) {
    tmp.n = 0;
    for (uint64_t j = off; j < off + counts[r]; ++j) hit_push(&tmp, col_out[j], val_out[j]);
    qsort(tmp.h, tmp.n, sizeof(ray_hit), hit_cmp);
    for (long j = 0; j < tmp.n; ++j) {
      col_out[off + j] = tmp.h[j].col;
      val_out[off + j] = tmp.h[j].len;
    }
    off += counts[r];
  }
  free(tmp.h);
}

typedef struct {
  entry_vec* blocks;
  int mode, k;
} build_user;
static void build_task(task* t, int item, int worker) {
  (void)worker;
  build_user* u = (build_user*)t->user;
  angle_block_entries_mode(t->g, u->mode, u->k, item, vec_emit, &u->blocks[item]);
}

void* ref_build_system_matrix(const o_geom* g, int threads, uint64_t budget, int* status) {
  return ref_build_system_matrix_mode(g, 0, 1, threads, budget, status);
}

void* ref_build_system_matrix_mode(const o_geom* g, int mode, int k, int threads, uint64_t budget,
                                   int* status) {
  *status = 0;
  csr* m = NULL;
  entry_vec first = {0};
  {
    jmp_buf jb;
    jmp_buf* prev = t_jmp;
    t_jmp = &jb;
    if (setjmp(jb) != 0) {
      t_jmp = prev;
      vec_free(&first);
      *status = -(t_code + 1);
      return NULL;
    }
    validate(g);
    const uint64_t nvox = (uint64_t)g->n_x * g->n_y * g->n_z;
    if (nvox > 0xffffffffull) o_fail(E_TooLarge, "grid exceeds 2^32 voxel columns");
    const uint64_t n_rows = (uint64_t)g->n_angles * g->n_det_y * g->n_det_z;
    angle_block_entries_mode(g, mode, k, 0, vec_emit, &first);
    const uint64_t est_nnz = (uint64_t)first.n * (uint64_t)g->n_angles;
    const uint64_t est_bytes = est_nnz * (4 + 8) + (n_rows + 1) * 8;
    if (est_bytes > budget) {
      char msg[256];
      snprintf(msg, sizeof msg, "estimated %llu entries (%llu MiB) exceed the budget of %llu MiB",
               (unsigned long long)est_nnz, (unsigned long long)(est_bytes >> 20),
               (unsigned long long)(budget >> 20));
      o_fail(E_OutOfMemory, msg);
    }
    t_jmp = prev;
    vec_free(&first);
  }
  const uint64_t rpa = (uint64_t)g->n_det_y * g->n_det_z;
  entry_vec* blocks = (entry_vec*)calloc(g->n_angles, sizeof(entry_vec));
  build_user u = {blocks, mode, k};
  task t;
  memset(&t, 0, sizeof t);
  t.fn = build_task;
  t.g = g;
  t.count = g->n_angles;
  t.threads = threads;
  t.user = &u;
  const int st = run_tasks(&t);
  if (st != 0) {
    for (int i = 0; i < g->n_angles; ++i) vec_free(&blocks[i]);
    free(blocks);
    *status = st;
    return NULL;
  }
  uint64_t nnz = 0;
  for (int i = 0; i < g->n_angles; ++i) nnz += (uint64_t)blocks[i].n;
  if (nnz == 0) {
    for (int i = 0; i < g->n_angles; ++i) vec_free(&blocks[i]);
    free(blocks);
    snprintf(t_err, sizeof t_err, "ZeroMatrix: system matrix has no entries");
    *status = -(E_ZeroMatrix + 1);
    return NULL;
  }
  m = (csr*)calloc(1, sizeof(csr));
  m->n_rows = (uint64_t)g->n_angles * rpa;
  m->n_cols = (uint64_t)g->n_x * g->n_y * g->n_z;
  m->nnz = nnz;
  m->row_start = (uint64_t*)malloc((m->n_rows + 1) * sizeof(uint64_t));
  m->col = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  m->val = (double*)malloc(nnz * sizeof(double));
  uint64_t* counts = (uint64_t*)malloc(rpa * sizeof(uint64_t));
  uint64_t off = 0;
  m->row_start[0] = 0;
  for (int ip = 0; ip < g->n_angles; ++ip) {
    bucket_by_row(&blocks[ip], rpa, counts, m->col + off, m->val + off, mode != 0);
    for (uint64_t r = 0; r < rpa; ++r) {
      const uint64_t row = (uint64_t)ip * rpa + r;
      m->row_start[row + 1] = m->row_start[row] + counts[r];
    }
    off += (uint64_t)blocks[ip].n;
    vec_free(&blocks[ip]);
  }
  free(counts);
  free(blocks);
  return m;
}

uint64_t ref_csr_nnz(void* h) { return ((csr*)h)->nnz; }
uint64_t ref_csr_rows(void* h) { return ((csr*)h)->n_rows; }
void ref_csr_copy(void* h, uint64_t* row_start, uint32_t* col, double* val) {
  csr* m = (csr*)h;
  memcpy(row_start, m->row_start, (m->n_rows + 1) * sizeof(uint64_t));
  memcpy(col, m->col, m->nnz * sizeof(uint32_t));
  memcpy(val, m->val, m->nnz * sizeof(double));
}
void ref_csr_free(void* h) {
  csr* m = (csr*)h;
  if (!m) return;
  free(m->row_start);
  free(m->col);
  free(m->val);
  free(m);
}

/* forward_project (projector.cpp:203-217) */
int ref_forward_project(void* h, const double* x, double* y) {
  const csr* m = (const csr*)h;
  for (uint64_t r = 0; r < m->n_rows; ++r) {
    double acc = 0.0;
    for (uint64_t j = m->row_start[r]; j < m->row_start[r + 1]; ++j) acc += m->val[j] * x[m->col[j]];
    y[r] = acc;
  }
  for (uint64_t r = 0; r < m->n_rows; ++r)
    if (!isfinite(y[r])) {
      snprintf(t_err, sizeof t_err, "NonFinite: forward projection not finite");
      return -(E_NonFinite + 1);
    }
  return 0;
}

/* back_project (projector.cpp:219-233) */
int ref_back_project(void* h, const double* y, double* x) {
  const csr* m = (const csr*)h;
  memset(x, 0, m->n_cols * sizeof(double));
  for (uint64_t r = 0; r < m->n_rows; ++r) {
    const double yr = y[r];
    if (yr == 0.0) continue;
    for (uint64_t j = m->row_start[r]; j < m->row_start[r + 1]; ++j) x[m->col[j]] += m->val[j] * yr;
  }
  for (uint64_t c = 0; c < m->n_cols; ++c)
    if (!isfinite(x[c])) {
      snprintf(t_err, sizeof t_err, "NonFinite: back projection not finite");
      return -(E_NonFinite + 1);
    }
  return 0;
}

/* ---- matrix-free A x (projector.cpp:235-260) ----------------------------- */
/* Work items are (angle, slab) pairs; with fewer angles than threads each
 * angle is split into slabs whose partial blocks are summed in slab order. */
typedef struct {
  const int32_t* angles;
  const double* x;
  double* parts; /* n_sel * n_parts blocks of rpa */
  int n_parts;
  uint64_t rpa;
  int mode, k;
  int zlo, zhi; /* slab range evaluated (whole grid by default) */
} fwd_user;
typedef struct {
  double* block;
  const double* x;
} fwd_ctx;
static void fwd_emit(void* ctx, uint32_t r, uint32_t c, double w) {
  fwd_ctx* f = (fwd_ctx*)ctx;
  f->block[r] += w * f->x[c];
}
static void fwd_task(task* t, int item, int worker) {
  (void)worker;
  fwd_user* u = (fwd_user*)t->user;
  const int k = item / u->n_parts, part = item % u->n_parts;
  const int n = u->zhi - u->zlo;
  const int lo = u->zlo + (int)((int64_t)n * part / u->n_parts),
            hi = u->zlo + (int)((int64_t)n * (part + 1) / u->n_parts);
  double* block = u->parts + (uint64_t)item * u->rpa;
  memset(block, 0, u->rpa * sizeof(double));
  fwd_ctx c = {block, u->x};
  if (u->mode != 0)
    angle_block_entries_rays(t->g, u->mode, u->k, u->angles[k], fwd_emit, &c);
  else
    angle_block_entries_slab(t->g, u->angles[k], lo, hi, fwd_emit, &c);
}

static int forward_mf_angles_impl(const o_geom* g, const int32_t* angles, int n_sel,
                                  const double* x, double* y_sel, int threads, int split,
                                  int mode, int k, int zlo, int zhi) {
  O_TRY(validate(g););
  const uint64_t rpa = (uint64_t)g->n_det_y * g->n_det_z;
  const int z0 = zlo < 0 ? 0 : zlo;
  const int z1r = (zhi < 0 || zhi > slab_extent(g)) ? slab_extent(g) : zhi;
  const int z1 = z1r < z0 ? z0 : z1r;
  int n_parts = 1;
  if (split && mode == 0 && n_sel > 0 && n_sel < threads) n_parts = (threads + n_sel - 1) / n_sel;
  if (n_parts > z1 - z0) n_parts = z1 - z0 > 0 ? z1 - z0 : 1;
  double* parts = y_sel;
  if (n_parts > 1) parts = (double*)malloc((uint64_t)n_sel * n_parts * rpa * sizeof(double));
  fwd_user u = {angles, x, parts, n_parts, rpa, mode, k, z0, z1};
  task t;
  memset(&t, 0, sizeof t);
  t.fn = fwd_task;
  t.g = g;
  t.count = n_sel * n_parts;
  t.threads = threads;
  t.user = &u;
  const int st = run_tasks(&t);
  if (n_parts > 1) {
    if (st == 0)
      for (int k = 0; k < n_sel; ++k) {
        double* out = y_sel + (uint64_t)k * rpa;
        memset(out, 0, rpa * sizeof(double));
        for (int p = 0; p < n_parts; ++p) {
          const double* b = parts + ((uint64_t)k * n_parts + p) * rpa;
          for (uint64_t r = 0; r < rpa; ++r) out[r] += b[r];
        }
      }
    free(parts);
  }
  return st;
}

/* Reference order (bit-exact with forward_project_matrix_free's per-angle
 * accumulation). */
int ref_forward_mf_angles(const o_geom* g, const int32_t* angles, int n_sel, const double* x,
                          double* y_sel, int threads) {
  return forward_mf_angles_impl(g, angles, n_sel, x, y_sel, threads, 0, 0, 1, 0, -1);
}
/* Same values up to summation order; angles split into slabs so that a few
 * large angle blocks use all threads (tolerance checks at C3/C4 scale). */
int ref_forward_mf_angles_par(const o_geom* g, const int32_t* angles, int n_sel, const double* x,
                              double* y_sel, int threads) {
  return forward_mf_angles_impl(g, angles, n_sel, x, y_sel, threads, 1, 0, 1, 0, -1);
}
/* A x rows of the listed angles from the voxels of z slabs [zlo, zhi) only
 * (x restricted to those slabs; 2D: pixel rows): BASELINE-scale parity checks
 * of the outer / central slabs without evaluating the whole grid. */
int ref_forward_mf_angles_slabs(const o_geom* g, const int32_t* angles, int n_sel, int zlo,
                                int zhi, const double* x, double* y_sel, int threads) {
  return forward_mf_angles_impl(g, angles, n_sel, x, y_sel, threads, 1, 0, 1, zlo, zhi);
}

int ref_forward_project_matrix_free(const o_geom* g, const double* x, double* y, int threads) {
  int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (g->n_angles > 0 ? g->n_angles : 1));
  for (int i = 0; i < g->n_angles; ++i) all[i] = i;
  const int st = ref_forward_mf_angles(g, all, g->n_angles, x, y, threads);
  free(all);
  return st;
}

/* ---- matrix-free A^T y restatement --------------------------- */
/* Per-angle partial volumes, summed in angle order; with fewer angles than
 * threads each angle's block is also split into slabs (disjoint voxels). */
typedef struct {
  const int32_t* angles;
  const double* y;
  double** part; /* per chunk slot */
  int base, n_parts;
  uint64_t rpa, nv;
  int mode, k;
  int zlo, zhi;
  int compact; /* y holds only the rows of the listed angles, in list order */
} bwd_user;
typedef struct {
  double* xpart;
  const double* yb;
} bwd_ctx;
static void bwd_emit(void* ctx, uint32_t r, uint32_t c, double w) {
  bwd_ctx* b = (bwd_ctx*)ctx;
  b->xpart[c] += w * b->yb[r];
}
static void bwd_task(task* t, int item, int worker) {
  (void)worker;
  bwd_user* u = (bwd_user*)t->user;
  const int k = item / u->n_parts, part = item % u->n_parts;
  const int n = u->zhi - u->zlo;
  const int lo = u->zlo + (int)((int64_t)n * part / u->n_parts),
            hi = u->zlo + (int)((int64_t)n * (part + 1) / u->n_parts);
  const uint64_t plane = t->g->n_z > 1 || t->g->n_det_z > 1 ? (uint64_t)t->g->n_x * t->g->n_y
                                                              : (uint64_t)t->g->n_x;
  double* p = u->part[k];
  memset(p + (uint64_t)lo * plane, 0, (uint64_t)(hi - lo) * plane * sizeof(double));
  const int ang = u->angles[u->base + k];
  bwd_ctx c = {p, u->y + (uint64_t)(u->compact ? u->base + k : ang) * u->rpa};
  if (u->mode != 0)
    angle_block_entries_rays(t->g, u->mode, u->k, ang, bwd_emit, &c);
  else
    angle_block_entries_slab(t->g, ang, lo, hi, bwd_emit, &c);
}

static int back_mf_angles_impl(const o_geom* g, const int32_t* angles, int n_sel,
                               const double* y, double* x, int threads, int split, int mode,
                               int k, int zlo, int zhi, int compact) {
  O_TRY(validate(g););
  const uint64_t nv = (uint64_t)g->n_x * g->n_y * g->n_z;
  const int z0 = zlo < 0 ? 0 : zlo;
  const int z1r = (zhi < 0 || zhi > slab_extent(g)) ? slab_extent(g) : zhi;
  const int z1 = z1r < z0 ? z0 : z1r;
  int n_parts = 1;
  if (split && mode == 0 && n_sel > 0 && n_sel < threads) n_parts = (threads + n_sel - 1) / n_sel;
  if (n_parts > z1 - z0) n_parts = z1 - z0 > 0 ? z1 - z0 : 1;
  const uint64_t plane = g->n_z > 1 || g->n_det_z > 1 ? (uint64_t)g->n_x * g->n_y : (uint64_t)g->n_x;
  const int chunk = n_parts > 1 ? n_sel : (threads < 1 ? 1 : threads);
  double** part = (double**)malloc(sizeof(double*) * (chunk > 0 ? chunk : 1));
  for (int i = 0; i < chunk; ++i) part[i] = (double*)malloc(nv * sizeof(double));
  memset(x, 0, nv * sizeof(double));
  int st = 0;
  for (int k0 = 0; k0 < n_sel && st == 0; k0 += chunk) {
    const int n = (n_sel - k0) < chunk ? (n_sel - k0) : chunk;
    bwd_user u = {angles, y, part, k0, n_parts, (uint64_t)g->n_det_y * g->n_det_z, nv, mode, k,
                  z0, z1, compact};
    task t;
    memset(&t, 0, sizeof t);
    t.fn = bwd_task;
    t.g = g;
    t.count = n * n_parts;
    t.threads = threads;
    t.user = &u;
    st = run_tasks(&t);
    if (st == 0)
      for (int k = 0; k < n; ++k)
        for (uint64_t i = (uint64_t)z0 * plane; i < (uint64_t)z1 * plane; ++i) x[i] += part[k][i];
  }
  for (int i = 0; i < chunk; ++i) free(part[i]);
  free(part);
  return st;
}

int ref_back_mf_angles(const o_geom* g, const int32_t* angles, int n_sel, const double* y,
                       double* x, int threads) {
  return back_mf_angles_impl(g, angles, n_sel, y, x, threads, 0, 0, 1, 0, -1, 0);
}
int ref_back_mf_angles_par(const o_geom* g, const int32_t* angles, int n_sel, const double* y,
                           double* x, int threads) {
  return back_mf_angles_impl(g, angles, n_sel, y, x, threads, 1, 0, 1, 0, -1, 0);
}
/* A^T y of the listed angles on the voxels of z slabs [zlo, zhi) (other
 * voxels 0); y_rows holds only the rows of the listed angles, in list order. */
int ref_back_mf_angles_slabs(const o_geom* g, const int32_t* angles, int n_sel, int zlo, int zhi,
                             const double* y_rows, double* x, int threads) {
  return back_mf_angles_impl(g, angles, n_sel, y_rows, x, threads, 1, 0, 1, zlo, zhi, 1);
}

int ref_back_project_matrix_free(const o_geom* g, const double* y, double* x, int threads) {
  int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (g->n_angles > 0 ? g->n_angles : 1));
  for (int i = 0; i < g->n_angles; ++i) all[i] = i;
  const int st = ref_back_mf_angles(g, all, g->n_angles, y, x, threads);
  free(all);
  return st;
}

/* forward_project_matrix_free / the a16 adjoint for any MatrixMode. */
static int32_t* all_angles(const o_geom* g) {
  int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (g->n_angles > 0 ? g->n_angles : 1));
  for (int i = 0; i < g->n_angles; ++i) all[i] = i;
  return all;
}
int ref_forward_mf_mode(const o_geom* g, int mode, int k, const double* x, double* y,
                        int threads) {
  int32_t* all = all_angles(g);
  const int st = forward_mf_angles_impl(g, all, g->n_angles, x, y, threads, 0, mode, k, 0, -1);
  free(all);
  return st;
}
int ref_back_mf_mode(const o_geom* g, int mode, int k, const double* y, double* x, int threads) {
  int32_t* all = all_angles(g);
  const int st = back_mf_angles_impl(g, all, g->n_angles, y, x, threads, 0, mode, k, 0, -1, 0);
  free(all);
  return st;
}

/* SIRT (BASELINE.json configs[4]) composed from the projector restatement. */
int ref_sirt(const o_geom* g, const double* y, double* x, int iters, int threads) {
  const uint64_t nv = (uint64_t)g->n_x * g->n_y * g->n_z;
  const uint64_t nm = (uint64_t)g->n_angles * g->n_det_y * g->n_det_z;
  double* R = (double*)malloc(nm * sizeof(double));
  double* C = (double*)malloc(nv * sizeof(double));
  double* ax = (double*)malloc(nm * sizeof(double));
  double* bp = (double*)malloc(nv * sizeof(double));
  double* ones_v = (double*)malloc(nv * sizeof(double));
  double* ones_m = (double*)malloc(nm * sizeof(double));
  for (uint64_t i = 0; i < nv; ++i) ones_v[i] = 1.0;
  for (uint64_t i = 0; i < nm; ++i) ones_m[i] = 1.0;
  int st = ref_forward_project_matrix_free(g, ones_v, R, threads);
  if (!st) st = ref_back_project_matrix_free(g, ones_m, C, threads);
  if (!st) {
    for (uint64_t i = 0; i < nm; ++i) R[i] = R[i] != 0.0 ? 1.0 / R[i] : 0.0;
    for (uint64_t i = 0; i < nv; ++i) C[i] = C[i] != 0.0 ? 1.0 / C[i] : 0.0;
  }
  for (int it = 0; it < iters && !st; ++it) {
    st = ref_forward_project_matrix_free(g, x, ax, threads);
    if (st) break;
    for (uint64_t i = 0; i < nm; ++i) ax[i] = R[i] * (y[i] - ax[i]);
    st = ref_back_project_matrix_free(g, ax, bp, threads);
    if (st) break;
    for (uint64_t i = 0; i < nv; ++i) x[i] += C[i] * bp[i];
  }
  free(R); free(C); free(ax); free(bp); free(ones_v); free(ones_m);
  return st;
}

/* angle_column_sums (projector.cpp:288-295) */
typedef struct {
  double* sums;
} colsum_ctx;
static void colsum_emit(void* ctx, uint32_t r, uint32_t c, double w) {
  (void)r;
  ((colsum_ctx*)ctx)->sums[c] += w;
}
int ref_angle_column_sums(const o_geom* g, int ip, double* sums) {
  memset(sums, 0, (uint64_t)g->n_x * g->n_y * g->n_z * sizeof(double));
  colsum_ctx c = {sums};
  O_TRY(angle_block_entries(g, ip, colsum_emit, &c););
  return 0;
}


/* ---- independent numerical oracles (oracle.cpp:70-196) --------------------
 * The reference's oracle.cpp includes <Eigen/Dense> (absent here), so it
 * cannot be compiled where it lies; the Eigen-free bodies of mc_volume_3d,
 * gauss_legendre and multiline_volume_3d are restated here. Pin: like the
 * reference's own tests (test_weights3d.cpp:198-212; validate.cpp:167-293)
 * they are checked against voxel_volume_factors (tests/test_oracle_pin.py):
 * MC within 4 standard errors + 1e-6, Gauss-Legendre within 1e-6. */

/* std::mt19937_64 (the 64-bit Mersenne Twister of Matsumoto & Nishimura). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;
static void mt64_seed(mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}
static uint64_t mt64_next(mt64* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      r->mt[i] = r->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}
static double mt64_u01(mt64* r) { return (double)(mt64_next(r) >> 11) * 0x1.0p-53; } /* oracle.cpp:46-49 */

/* mc_volume_3d (oracle.cpp:70-98): out[0] = value, out[1] = std_err, returns hits */
uint64_t ref_mc_volume_3d(const double* box, double phi, double s, double d, double d_y, double d_z,
                          int m_y, int m_z, uint64_t n_samples, uint64_t seed, double* out) {
  const double x0 = box[0], x1 = box[1], y0 = box[2], y1 = box[3], zb = box[4], zt = box[5];
  const double cp = O_COS(phi), sp = O_SIN(phi);
  const int n_shards = 16;
  uint64_t hits = 0, total = 0;
  mt64 rng;
  for (int shard = 0; shard < n_shards; ++shard) {
    mt64_seed(&rng, seed + (uint64_t)shard);
    const uint64_t count = n_samples / n_shards + (shard < (int)(n_samples % n_shards) ? 1 : 0);
    for (uint64_t i = 0; i < count; ++i) {
      const double x = x0 + (x1 - x0) * mt64_u01(&rng);
      const double y = y0 + (y1 - y0) * mt64_u01(&rng);
      const double z = zb + (zt - zb) * mt64_u01(&rng);
      const double depth = s - x * cp - y * sp;
      const double uy = (s + d) / depth * (y * cp - x * sp) / d_y;
      const double uz = (s + d) / depth * z / d_z;
      if (uy >= m_y && uy < m_y + 1 && uz >= m_z && uz < m_z + 1) ++hits;
    }
    total += count;
  }
  const double p = (double)hits / (double)total;
  const double var = p * (1.0 - p), fl = 1.0 / (double)total;
  out[0] = p;
  out[1] = sqrt((var > fl ? var : fl) / (double)total);
  return hits;
}

/* gauss_legendre (oracle.cpp:100-122) */
void ref_gauss_legendre(int k, double* x, double* w) {
  for (int i = 0; i < k; ++i) {
    double t = cos(K_PI * (i + 0.75) / (k + 0.5));
    double pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 0; j < k; ++j) {
        const double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j + 1.0) * t * p1 - j * p2) / (j + 1.0);
      }
      pp = k * (t * p0 - p1) / (t * t - 1.0);
      const double dt = p0 / pp;
      t -= dt;
      if (fabs(dt) < 1e-15) break;
    }
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * pp * pp);
  }
}

/* multiline_volume_3d (oracle.cpp:124-196) */
double ref_multiline_volume_3d(const double* box, double phi, double s, double d, double d_y,
                               double d_z, int m_y, int m_z, int k) {
  const double x0 = box[0], x1 = box[1], y0 = box[2], y1 = box[3], zb = box[4], zt = box[5];
  const double cp = O_COS(phi), sp = O_SIN(phi);
  const double sx = s * cp, sy = s * sp;
  double u_min = 0, u_max = 0, v_min = 0, v_max = 0;
  int first = 1;
  const double vxs[2] = {x0, x1}, vys[2] = {y0, y1}, vzs[2] = {zb, zt};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const double vx = vxs[a], vy = vys[b];
      const double depth = s - vx * cp - vy * sp;
      const double u = (s + d) / depth * (vy * cp - vx * sp) / d_y;
      u_min = first ? u : dmin(u_min, u);
      u_max = first ? u : dmax(u_max, u);
      for (int c = 0; c < 2; ++c) {
        const double v = (s + d) / depth * vzs[c] / d_z;
        if (first) {
          v_min = v_max = v;
        } else {
          v_min = dmin(v_min, v);
          v_max = dmax(v_max, v);
        }
        first = 0;
      }
    }
  const double u_lo = dmax((double)m_y, u_min), u_hi = dmin((double)m_y + 1.0, u_max);
  const double v_lo = dmax((double)m_z, v_min), v_hi = dmin((double)m_z + 1.0, v_max);
  if (u_hi <= u_lo || v_hi <= v_lo) return 0.0;
  double* nodes = (double*)malloc(2 * (size_t)k * sizeof(double));
  double* wts = nodes + k;
  ref_gauss_legendre(k, nodes, wts);
  const double uc = 0.5 * (u_lo + u_hi), ur = 0.5 * (u_hi - u_lo);
  const double vc = 0.5 * (v_lo + v_hi), vr = 0.5 * (v_hi - v_lo);
  double total = 0.0;
  for (int i = 0; i < k; ++i) {
    const double ey = (uc + ur * nodes[i]) * d_y;
    for (int j = 0; j < k; ++j) {
      const double ez = (vc + vr * nodes[j]) * d_z;
      const double dx = -d * cp - ey * sp, dy = -d * sp + ey * cp, dz = ez;
      double t0 = 0.0, t1 = INFINITY;
      const double org[3] = {sx, sy, 0.0};
      const double dir[3] = {dx - sx, dy - sy, dz};
      const double lo[3] = {x0, y0, zb}, hi[3] = {x1, y1, zt};
      for (int ax = 0; ax < 3; ++ax) {
        if (fabs(dir[ax]) < 1e-300) {
          if (org[ax] < lo[ax] || org[ax] > hi[ax]) {
            t0 = 1.0;
            t1 = 0.0;
            break;
          }
          continue;
        }
        double ta = (lo[ax] - org[ax]) / dir[ax];
        double tb = (hi[ax] - org[ax]) / dir[ax];
        if (ta > tb) {
          const double tmp = ta;
          ta = tb;
          tb = tmp;
        }
        t0 = dmax(t0, ta);
        t1 = dmin(t1, tb);
      }
      if (t1 > t0) total += wts[i] * wts[j] * (cube(t1) - cube(t0)) / 3.0;
    }
  }
  free(nodes);
  return d_y * d_z * (s + d) * total * ur * vr / ((x1 - x0) * (y1 - y0) * (zt - zb));
}

#ifdef CTSM_ORACLE_CRMATH
/* crmath entry points for tests/test_crmath.py (correct-rounding checks). */
void orc_crm_eval(int fn, const double* a, const double* b, double* out, long n) {
  for (long i = 0; i < n; ++i) {
    switch (fn) {
      case 0: out[i] = crm_sin(a[i]); break;
      case 1: out[i] = crm_cos(a[i]); break;
      case 2: out[i] = crm_tan(a[i]); break;
      case 3: out[i] = crm_atan(a[i]); break;
      default: out[i] = crm_atan2(a[i], b[i]); break;
    }
  }
}
#endif
