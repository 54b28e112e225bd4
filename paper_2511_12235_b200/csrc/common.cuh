// common.cuh -- shared device-side definitions for the ctsm-b200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ctsm_b200.h"

namespace ctsmb {

constexpr double kPi = 3.14159265358979323846;  // common/geometry.hpp:11
// Numeric guards (common.hpp:46-57).
constexpr double kEpsDenRel = 1e-12;
constexpr double kEpsAngle = 1e-12;
constexpr double kEpsSingular = 1e-8;
constexpr double kEpsPiece = 1e-15;
constexpr double kEpsWeight = 1e-16;
constexpr double kNegClamp2D = -1e-14;
constexpr double kNegClamp3D = -1e-9;
constexpr double kCanonSlack = 1e-13;

// Device capacity limits (checked; exceeding them raises TooLarge).
constexpr int kMaxBrk = 24;   // breakpoints of one pixel sweep (4 corners + edges)
constexpr int kMaxRowsPerVoxel = 64;

// Geometry passed by value to kernels: the ScanGeometry fields plus a few
// derived quantities. Values that enter bit-exact arithmetic are computed with
// the same expressions as the reference (see exact.cuh).
struct DevGeom {
  double s, d, d_y, d_z;
  int n_det_y, n_det_z, n_angles;
  double angle_start, angle_end;
  double a, b, c;
  int n_x, n_y, n_z;
  // derived
  double sdd;        // s + d
  int rows_per_angle;
  long long n_vox;
  int edge_lo;       // edge-angle table covers e in [edge_lo, edge_lo + n_edges)
  int n_edges;
  // host-precomputed constants for the matrix-free (fast) path only
  double inv_a, inv_b, inv_2ab;  // 1/a, 1/b, 1/(2ab)
  double u_scale, t_scale;       // (s+d)/d_y, d_y/(s+d)
  double sdd_dz, dz_sdd;         // (s+d)/d_z, d_z/(s+d)
};

inline DevGeom make_dev_geom(const ctsm_geometry& g) {
  DevGeom d;
  d.s = g.s;
  d.d = g.d;
  d.d_y = g.d_y;
  d.d_z = g.d_z;
  d.n_det_y = g.n_det_y;
  d.n_det_z = g.n_det_z;
  d.n_angles = g.n_angles;
  d.angle_start = g.angle_start;
  d.angle_end = g.angle_end;
  d.a = g.a;
  d.b = g.b;
  d.c = g.c;
  d.n_x = g.n_x;
  d.n_y = g.n_y;
  d.n_z = g.n_z;
  d.sdd = g.s + g.d;
  d.rows_per_angle = g.n_det_y * g.n_det_z;
  d.n_vox = (long long)g.n_x * g.n_y * g.n_z;
  d.edge_lo = 0;
  d.n_edges = 0;
  d.inv_a = 1.0 / g.a;
  d.inv_b = 1.0 / g.b;
  d.inv_2ab = 0.5 / (g.a * g.b);
  d.u_scale = d.sdd / g.d_y;
  d.t_scale = g.d_y / d.sdd;
  d.sdd_dz = d.sdd / g.d_z;
  d.dz_sdd = g.d_z / d.sdd;
  return d;
}

// Device status word: the first failing thread records its code (1-based
// ErrorCode ordinal, ctsm_b200.h); the host checks it after each call.
__device__ __forceinline__ void raise_status(int* status, int code) {
  atomicCAS(status, 0, code);
}

// face_x/face_y/face_z (geometry.hpp:53-55): (i - n/2.0) * pitch.
__device__ __forceinline__ double face(double i, int n, double pitch) {
  return (i - n / 2.0) * pitch;
}

}  // namespace ctsmb
