/* ctsm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (consistent, line and
 * multiline modes). It exports the same extern "C" entry points as
 * ref_shim.cpp, so tests can drive the restatement and the compiled reference
 * interchangeably. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product never links or calls it.
 *
 * Pinned against the reference itself: tests/test_oracle_pin.py checks it
 * bit-for-bit against oracle/_ref (the unmodified reference compiled here) and
 * against the committed golden fixtures in tests/golden/ (generated from the
 * reference by tests/golden/make_golden.py).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct o_geom {  /* layout == ctsm_geometry (include/ctsm_b200.h) */
  double s, d, d_y, d_z;
  int32_t n_det_y, n_det_z, n_angles, pad0;
  double angle_start, angle_end;
  double a, b, c;
  int32_t n_x, n_y, n_z, pad1;
} o_geom;

const char* ref_last_error(void);
int ref_validate(const o_geom* g);
double ref_angle(const o_geom* g, int i);
long ref_pixel_area_factors(const o_geom* g, int ix, int iy, double phi, int32_t* my,
                            double* w, long cap);
long ref_voxel_volume_factors(const o_geom* g, int ix, int iy, int iz, double phi,
                              int32_t* my, int32_t* mz, double* w, long cap);
long ref_angle_block_entries(const o_geom* g, int ip, uint32_t* row, uint32_t* col,
                             double* w, long cap);
void* ref_build_system_matrix(const o_geom* g, int threads, uint64_t budget, int* status);
uint64_t ref_csr_nnz(void* h);
uint64_t ref_csr_rows(void* h);
void ref_csr_copy(void* h, uint64_t* row_start, uint32_t* col, double* val);
void ref_csr_free(void* h);
int ref_forward_project(void* h, const double* x, double* y);
int ref_back_project(void* h, const double* y, double* x);
int ref_forward_project_matrix_free(const o_geom* g, const double* x, double* y, int threads);
int ref_forward_mf_angles(const o_geom* g, const int32_t* angles, int n_sel, const double* x,
                          double* y_sel, int threads);
int ref_back_mf_angles(const o_geom* g, const int32_t* angles, int n_sel, const double* y,
                       double* x, int threads);
int ref_back_project_matrix_free(const o_geom* g, const double* y, double* x, int threads);
/* Restatement-only variants that also split each angle block into slabs (same
 * values up to summation order) to use all threads on few large angles. */
int ref_forward_mf_angles_par(const o_geom* g, const int32_t* angles, int n_sel, const double* x,
                              double* y_sel, int threads);
int ref_back_mf_angles_par(const o_geom* g, const int32_t* angles, int n_sel, const double* y,
                           double* x, int threads);
/* slab-restricted variants (z slabs [zlo, zhi); 2D: pixel rows): forward from
 * the voxels of those slabs only; back-projection onto those voxels only, from
 * y_rows = the rows of the listed angles in list order */
int ref_forward_mf_angles_slabs(const o_geom* g, const int32_t* angles, int n_sel, int zlo,
                                int zhi, const double* x, double* y_sel, int threads);
int ref_back_mf_angles_slabs(const o_geom* g, const int32_t* angles, int n_sel, int zlo, int zhi,
                             const double* y_rows, double* x, int threads);
long ref_angle_block_entries_par(const o_geom* g, int ip, uint32_t* row, uint32_t* col, double* w,
                                 long cap, int threads);
int ref_sirt(const o_geom* g, const double* y, double* x, int iters, int threads);
int ref_angle_column_sums(const o_geom* g, int ip, double* sums);
/* line / multiline modes (baseline.cpp:13-128; mode 1 = line, 2 = multiline,
 * 0 = consistent as above). */
long ref_line_weights(const o_geom* g, int mode, int k, int m_y, int m_z, int ip, uint32_t* col,
                      double* len, long cap);
long ref_angle_block_entries_mode(const o_geom* g, int mode, int k, int ip, uint32_t* row,
                                  uint32_t* col, double* w, long cap);
void* ref_build_system_matrix_mode(const o_geom* g, int mode, int k, int threads, uint64_t budget,
                                   int* status);
int ref_forward_mf_mode(const o_geom* g, int mode, int k, const double* x, double* y, int threads);
int ref_back_mf_mode(const o_geom* g, int mode, int k, const double* y, double* x, int threads);

/* Independent numerical oracles (oracle.cpp:70-196; restatement only: the
 * reference's oracle.cpp needs Eigen). box = {x0, x1, y0, y1, zb, zt}. */
uint64_t ref_mc_volume_3d(const double* box, double phi, double s, double d, double d_y, double d_z,
                          int m_y, int m_z, uint64_t n_samples, uint64_t seed, double* out);
void ref_gauss_legendre(int k, double* x, double* w);
double ref_multiline_volume_3d(const double* box, double phi, double s, double d, double d_y,
                               double d_z, int m_y, int m_z, int k);

#ifdef __cplusplus
}
#endif
