/* ctsm_b200.h -- C-ABI of the B200-native consistent CT system-matrix library.
 *
 * This is the drop-in boundary for the reference's hot path (ctsm,
 * /root/reference/proj): the C++ API in include/ctsm_b200/projector.hpp and
 * the Python mirror (paper_2511_12235_b200) are thin layers over these entry
 * points. Plain pointers and sizes only; device pointers are CUDA global
 * memory on the context's device; `stream` is a cudaStream_t (NULL = legacy
 * default stream).
 *
 * Status convention: every call returns 0 on success or
 * (ctsm::ErrorCode ordinal + 1) (common.hpp:11-25), e.g. 10 = InvalidSpec,
 * 11 = OutOfMemory; CTSM_ERR_CUDA (100) for a CUDA runtime failure.
 * ctsm_last_error() returns the message of the calling thread's last failure.
 * In-kernel guards (depth <= 1e-12 s, 2D piece < -1e-14, 3D weight < -1e-9;
 * geometry.cpp:59-60, weights2d.cpp:115-118, weights3d.cpp:455-457) raise the
 * same codes through a device status word checked after each call.
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ScanGeometry (geometry.hpp:29-44); field order and meaning identical. */
typedef struct ctsm_geometry {
  double s, d, d_y, d_z;
  int32_t n_det_y, n_det_z, n_angles, pad0;
  double angle_start, angle_end;
  double a, b, c;
  int32_t n_x, n_y, n_z, pad1;
} ctsm_geometry;

enum {
  CTSM_OK = 0,
  CTSM_ERR_DEGENERATE_GEOMETRY = 1,
  CTSM_ERR_RAY_PARALLEL_TO_FACE = 2,
  CTSM_ERR_SINGULAR_PHI = 3,
  CTSM_ERR_CENTRAL_ROW = 4,
  CTSM_ERR_Z_RESTRICTION = 5,
  CTSM_ERR_DIMENSION_MISMATCH = 6,
  CTSM_ERR_NON_FINITE = 7,
  CTSM_ERR_ZERO_MATRIX = 8,
  CTSM_ERR_TOO_LARGE = 9,
  CTSM_ERR_INVALID_SPEC = 10,
  CTSM_ERR_OUT_OF_MEMORY = 11,
  CTSM_ERR_INVALID_CONFIG = 12,
  CTSM_ERR_IO_FAILURE = 13,
  CTSM_ERR_CUDA = 100
};

/* Element type of matrix-free operands (x, y). Weights are always evaluated in
 * FP64; the dtype is the storage/accumulation type. */
enum { CTSM_F64 = 0, CTSM_F32 = 1 };

typedef struct ctsm_ctx ctsm_ctx;

/* ---- context ------------------------------------------------------------ */
int ctsm_create(int device, ctsm_ctx** out);
int ctsm_destroy(ctsm_ctx* ctx);
const char* ctsm_last_error(void);
const char* ctsm_version(void);
/* Number of GPU kernel launches issued by this library in this process
 * (monotonic; used by bench.py to report gpu_launches). */
uint64_t ctsm_launch_count(void);

/* ScanGeometry::validate (geometry.cpp:27-54), plus the device-side
 * implementation limits (TooLarge). */
int ctsm_validate_geometry(const ctsm_geometry* g);

/* ---- K1/K2: consistent system-matrix CSR (build_system_matrix,
 * projector.hpp:41-44 / projector.cpp:144-201) ----------------------------
 * Builds the rows of angles [angle_begin, angle_end) (an angle shard: rows
 * are angle-major, geometry.hpp:79-84, so a shard is a contiguous row range).
 * Two phases:
 *   ctsm_csr_count: row_start_dev[0..n_rows] (u64, n_rows = (angle_end -
 *     angle_begin) * n_det_y * n_det_z) receives the exclusive prefix sum of
 *     per-row entry counts; *nnz_out (host) the total. Raises OutOfMemory if
 *     nnz * 12 + (n_rows + 1) * 8 exceeds memory_budget_bytes (cf.
 *     projector.cpp:155-169) and ZeroMatrix if the full matrix is empty.
 *   ctsm_csr_fill: fills col_dev (u32, voxel columns strictly ascending per
 *     row) and val_dev (f64) for the same shard.
 * Values are bit-identical to the reference evaluated with a correctly
 * rounded libm (crmath.h); see DESIGN.md. */
int ctsm_csr_count(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                   uint64_t memory_budget_bytes, uint64_t* row_start_dev, uint64_t* nnz_out,
                   void* stream);
int ctsm_csr_fill(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                  const uint64_t* row_start_dev, uint32_t* col_dev, double* val_dev,
                  void* stream);

/* Single-evaluation build of the same rows: every weight is evaluated once.
 * Per chunk of angles the kernel appends 16-byte records {row, col, val} and
 * counts the rows; after the row scan the records are scattered into
 * row-grouped scratch and each row is radix-sorted by column into the
 * caller's arrays. row_start_dev as ctsm_csr_count; col_dev / val_dev hold
 * `capacity` entries (ctsm_csr_angle_nnz(angle 0) * angles * 1.2 is a good
 * size). *nnz_out receives the shard's entry count; the arrays are complete
 * only if *nnz_out <= capacity (otherwise call again with larger arrays).
 * Errors as ctsm_csr_count. ctsm_csr_angle_nnz counts one angle's entries
 * (the reference's budget estimate uses angle 0, projector.cpp:155-169). */
int ctsm_csr_angle_nnz(ctsm_ctx* ctx, const ctsm_geometry* g, int angle, uint64_t* nnz_out,
                       void* stream);
int ctsm_csr_build(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                   uint64_t memory_budget_bytes, uint64_t* row_start_dev, uint32_t* col_dev,
                   double* val_dev, uint64_t capacity, uint64_t* nnz_out, void* stream);

/* ---- the reference's weight API -------------------------------------------
 * ctsm_weights_batch: pixel_area_factors (weights2d.hpp:31-32,
 * weights2d.cpp:105-129) / voxel_volume_factors (weights3d.hpp:90-91,
 * weights3d.cpp:354-462) for n (voxel, phi) queries given as HOST arrays (iz
 * may be NULL for 2D). Query q's weights are written, in the reference's
 * order (ascending m_y, then m_z), to entries [q*cap, q*cap + count[q]) of
 * the host arrays m_y, m_z (may be NULL for 2D) and w. Bit-identical to the
 * reference with a correctly rounded libm. TooLarge if a query has more than
 * cap weights; the reference's guards raise their codes.
 * ctsm_angle_block_entries: detail::angle_block_entries (projector.hpp:72-78,
 * projector.cpp:44-84): every (raster row, column, weight) entry of one angle
 * block into DEVICE arrays of `capacity` entries, in the reference's emission
 * order (consistent: voxels z -> y -> x, each voxel's weights by (m_y, m_z);
 * line / multiline: row by row). *n_out receives the entry count; the arrays
 * are complete only if it is <= capacity (ctsm_csr_angle_nnz gives the count
 * of the consistent mode beforehand). */
int ctsm_weights_batch(ctsm_ctx* ctx, const ctsm_geometry* g, uint64_t n, const int32_t* ix,
                       const int32_t* iy, const int32_t* iz, const double* phi, int cap,
                       int32_t* count, int32_t* m_y, int32_t* m_z, double* w);
int ctsm_angle_block_entries(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int angle,
                             uint64_t capacity, uint32_t* raster_dev, uint32_t* col_dev,
                             double* w_dev, uint64_t* n_out, void* stream);

/* ---- K3/K4: CSR appliers (forward_project / back_project,
 * projector.cpp:203-233). Deterministic; NonFinite check as the reference. */
int ctsm_spmv(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols, const uint64_t* row_start_dev,
              const uint32_t* col_dev, const double* val_dev, const double* x_dev,
              double* y_dev, void* stream);
int ctsm_spmv_t(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols, const uint64_t* row_start_dev,
                const uint32_t* col_dev, const double* val_dev, const double* y_dev,
                double* x_dev, void* stream);
/* K4 in two parts, for callers that keep the matrix: the column-sum bound
 * max_c sum_r |A_rc| (one pass over the CSR; a property of the matrix, valid
 * until its values change) and the scatter with a given bound. ctsm_spmv_t
 * is the two in sequence. */
int ctsm_csr_colsum_max(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                        const uint64_t* row_start_dev, const uint32_t* col_dev,
                        const double* val_dev, double* colsum_max, void* stream);
int ctsm_spmv_t_bound(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                      const uint64_t* row_start_dev, const uint32_t* col_dev,
                      const double* val_dev, double colsum_max, const double* y_dev,
                      double* x_dev, void* stream);

/* K4 as a gather: the CSC transpose of a device CSR (col_start u64[n_cols+1],
 * row u32[nnz], val f64[nnz], caller-allocated; the entries of a column come
 * in schedule order) and back_project through it (projector.cpp:219-233). It
 * sums the same fixed-point integers as ctsm_spmv_t_bound, so the two agree
 * bit for bit; it reads every entry once instead of issuing one 64-bit
 * reduction per entry. n_rows must be < 2^32. */
int ctsm_csc_build(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                   const uint64_t* row_start_dev, const uint32_t* col_dev, const double* val_dev,
                   uint64_t* col_start_dev, uint32_t* row_dev, double* valt_dev, void* stream);
int ctsm_spmv_t_csc(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                    const uint64_t* col_start_dev, const uint32_t* row_dev,
                    const double* valt_dev, double colsum_max, const double* y_dev,
                    double* x_dev, void* stream);

/* ---- K5/K6: matrix-free projectors (forward_project_matrix_free,
 * projector.hpp:56-59; back_project_matrix_free is the rebuild's addition).
 * The angle shard is {angle_begin + k * angle_step < angle_end}. Forward
 * writes the sinogram rows of those angles (other rows untouched). Backward
 * writes x = sum over the shard's angles (overwrites x). Layouts: x
 * [n_z][n_y][n_x], y [n_angles][n_det_z][n_det_y]. dtype: CTSM_F64/CTSM_F32.
 * Results are deterministic (fixed-point accumulation for the scatter). */
int ctsm_fwd_mf(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int angle_begin,
                int angle_end, int angle_step, const void* x_dev, void* y_dev, void* stream);
int ctsm_bwd_mf(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int angle_begin,
                int angle_end, int angle_step, const void* y_dev, void* x_dev, void* stream);

/* Quarter-turn symmetric scans (square grid with even side, a == b,
 * n_angles % 4 == 0, angles over exactly one turn): rotating the scanner by a
 * quarter turn maps the setup onto itself, so each weight evaluation serves
 * four (voxel, angle) pairs. ctsm_fwd_mf / ctsm_bwd_mf use this automatically
 * for shards closed under +n_angles/4 (e.g. the full scan; disable with the
 * environment variable CTSM_NO_SYMMETRY=1). The orbit entry points take the
 * shard as base angles {base_begin + k * base_step < n_angles / 4} plus their
 * quarter-turn images -- the load-balanced multi-GPU sharding of such scans.
 * ctsm_quarter_symmetric returns 1 if the scan qualifies.
 *
 * Scans that additionally start at angle 0 with n_angles % 8 == 0 are also
 * symmetric under the reflection phi -> -phi, y -> -y (dihedral group of
 * order 8; disable with CTSM_NO_DIHEDRAL=1): then only the full scan is detected
 * automatically and the orbit base set is {0 <= i <= n_angles / 8} with each
 * base angle's 8 images (4 for i = 0 and i = n_angles / 8).
 * ctsm_symmetry_order returns 8, 4 or 1. */
int ctsm_quarter_symmetric(const ctsm_geometry* g);
int ctsm_symmetry_order(const ctsm_geometry* g);
int ctsm_fwd_mf_orbits(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int base_begin,
                       int base_step, const void* x_dev, void* y_dev, void* stream);
int ctsm_bwd_mf_orbits(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int base_begin,
                       int base_step, const void* y_dev, void* x_dev, void* stream);

/* Voxel-ray updates (nonzero weights applied, i.e. nnz of the shard's rows of
 * A) counted live by the last successful ctsm_fwd_mf call on ctx. */
uint64_t ctsm_last_update_count(ctsm_ctx* ctx);

/* Kernel family of the last matrix-free call on ctx (CTSM_PATH_* bits):
 * GENERAL = per-angle kernels; QUARTER / DIHEDRAL = the symmetric production
 * kernels (4 / 8 (pixel, angle) pairs per weight evaluation); ZMIRROR = the
 * 3D z-mirror reuse (even n_z); F32_VECRED = the fp32 3D forward with
 * red.global.add.v4.f32 row runs. Lets tests assert which kernel ran. */
#define CTSM_PATH_GENERAL 1
#define CTSM_PATH_QUARTER 4
#define CTSM_PATH_DIHEDRAL 8
#define CTSM_PATH_ZMIRROR 16
#define CTSM_PATH_F32_VECRED 32
int ctsm_last_kernel_path(ctsm_ctx* ctx);

/* ---- K7/K8: SIRT pieces (BASELINE.json configs[4]) ----------------------
 * x <- x + C .* A^T (R .* (y - A x)), R = 1/(A 1), C = 1/(A^T 1), zero sums -> 0.
 * ctsm_sirt_residual: r = R .* (y - ax) over the shard's rows, with R
 * supplied as inverse row sums (elementwise, n = rows of the shard's angles).
 * ctsm_sirt_update: x += C .* bp; both arrays full-size. ctsm_invert_nonzero
 * turns sums into inverse sums (0 stays 0). Multi-GPU drivers all-reduce bp
 * (and A^T 1) between ctsm_bwd_mf and ctsm_sirt_update. */
int ctsm_invert_nonzero(ctsm_ctx* ctx, int dtype, uint64_t n, void* v_dev, void* stream);
int ctsm_sirt_residual(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int angle_begin,
                       int angle_end, int angle_step, const void* y_dev, const void* rinv_dev,
                       void* ax_inout_dev, void* stream);
int ctsm_sirt_update(ctsm_ctx* ctx, int dtype, uint64_t n, const void* cinv_dev,
                     const void* bp_dev, void* x_inout_dev, void* stream);
/* Full single-device SIRT driver: iters iterations from x_inout. */
int ctsm_sirt(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, const void* y_dev,
              void* x_inout_dev, int iters, void* stream);

/* ---- reconstruction protocol on device -----------
 * The solvers take a linear operator W: a device CSR matrix (K3/K4 appliers)
 * or the fp64 matrix-free projector of a scan (K5/K6) times `scale` (the
 * matrix-free analogue of scale_values). All vectors are fp64 device arrays;
 * reductions are deterministic (fixed-order), so results repeat bit for bit.
 */
enum { CTSM_OP_CSR = 0, CTSM_OP_MATRIX_FREE = 1 };
typedef struct ctsm_operator {
  int kind;
  int pad0;
  uint64_t n_rows, n_cols;          /* CSR (ignored for matrix-free) */
  const uint64_t* row_start;        /* CSR, device */
  const uint32_t* col;              /* CSR, device */
  const double* val;                /* CSR, device */
  const ctsm_geometry* geom;        /* matrix-free */
  double scale;                     /* matrix-free: W = scale * A (CSR: must be 1) */
  /* CSR, optional (all three or none; zero-initialise otherwise): the CSC
   * transpose of ctsm_csc_build; W^T then gathers instead of scattering,
   * with the same bits */
  const uint64_t* col_start;
  const uint32_t* trow;
  const double* tval;
} ctsm_operator;

/* spectral_norm_power (projector.cpp:262-280): v_inout holds the start vector
 * (the caller's normal_samples(n_cols, seed)); it is normalised, then `iters`
 * times v <- W^T W v / ||W^T W v||; *norm_out = sqrt(||W^T W v||) of the
 * last iteration. ZeroMatrix for an empty matrix or a collapsed iteration. */
int ctsm_spectral_norm_power(ctsm_ctx* ctx, const ctsm_operator* op, int iters,
                             double* v_inout_dev, double* norm_out, void* stream);
/* nag_tikhonov (solver.hpp:32-35, solver.cpp:17-75): minimises
 * 0.5 ||W u - p||^2 + 0.5 lambda ||u||^2 by Nesterov's method with the fixed
 * step 1 / (1 + lambda) (W scaled to unit spectral norm by the caller);
 * stops when ||W^T (W u - p) + lambda u||^2 < tol. u_dev receives the
 * iterate (starts at 0). trace_host, if not NULL, receives 3 doubles per
 * iteration: {iter, objective, grad_norm_sq} (SolveTraceRow). InvalidConfig
 * for negative lambda/tol/max_iter; NonFinite when the iterate diverges. */
int ctsm_nag_tikhonov(ctsm_ctx* ctx, const ctsm_operator* op, const double* p_dev,
                      double lambda, int max_iter, double tol, double* u_dev,
                      double* trace_host, int* iterations, int* converged, void* stream);
/* normal_samples (phantoms.cpp:78-87; host): mt19937_64(seed), Box-Muller
 * cosine branch -- the start vector of spectral_norm_power. */
void ctsm_normal_samples(uint64_t n, uint64_t seed, double* out_host);
/* scale_values (projector.cpp:282-286) on a device value array. */
int ctsm_scale_values(ctsm_ctx* ctx, uint64_t nnz, double* val_dev, double factor,
                      void* stream);

/* ---- CSM1 / CTT1 containers (io.hpp:31-48) -------
 * CSM1 (write_matrix / read_matrix, io.cpp:153-227): "CSM1", u64 n_rows,
 * n_cols, nnz, meta_len, meta, row_start[n_rows+1] u64, col[nnz] as u64,
 * val[nnz] f64 -- byte-identical to the reference writer. The device variants
 * stream a device CSR through pinned staging (no host copy of the matrix).
 * Reading: ctsm_csm1_header gives the sizes to allocate; the reader applies
 * the reference's checks (IoFailure: bad magic, short file, inconsistent or
 * decreasing row offsets, column out of range; TooLarge: n_cols >= 2^32). */
int ctsm_write_csm1_device(ctsm_ctx* ctx, const char* path, uint64_t n_rows, uint64_t n_cols,
                           const uint64_t* row_start_dev, const uint32_t* col_dev,
                           const double* val_dev, const char* meta, uint64_t meta_len,
                           void* stream);
int ctsm_csm1_header(const char* path, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz,
                     uint64_t* meta_len);
int ctsm_read_csm1_device(ctsm_ctx* ctx, const char* path, uint64_t* row_start_dev,
                          uint32_t* col_dev, double* val_dev, char* meta_out, void* stream);
/* CTT1 (write_tensor / read_tensor, io.cpp:229-270), host buffers. */
int ctsm_write_ctt1(const char* path, const uint64_t* dims, int rank, const double* data_host);
int ctsm_ctt1_header(const char* path, uint64_t* dims_out /* [8] */, int* rank_out);
int ctsm_read_ctt1(const char* path, double* data_host, uint64_t count);

/* ---- line / multiline(k) modes -------------------
 * The paper's comparison method (baseline.cpp:13-128): the exact intersection
 * lengths of the ray to the centre of each detector cell (line) or the average
 * over k (2D) / k*k (3D) uniformly placed rays (multiline), one device thread
 * per detector cell. mode = MatrixMode ordinal (projector.hpp:12-16); for
 * CTSM_MODE_CONSISTENT the calls forward to the entry points above (k ignored).
 *   ctsm_csr_count_mode / ctsm_csr_fill_mode: build_system_matrix(g, mode, k)
 *     rows of angles [angle_begin, angle_end), same protocol and errors as
 *     ctsm_csr_count / ctsm_csr_fill; bit-identical to the reference with a
 *     correctly rounded libm (merge_hits order and stable column sort kept).
 *     Rows longer than 8192 traced hits (before merging) raise TooLarge.
 *   ctsm_fwd_mf_mode / ctsm_bwd_mf_mode: forward_project_matrix_free(g, mode,
 *     k, x) (projector.cpp:235-260) and its adjoint on a strided angle shard,
 *     deterministic (gather / int64 fixed-point scatter). InvalidSpec for an
 *     unknown mode or k <= 0 in multiline mode. */
enum { CTSM_MODE_CONSISTENT = 0, CTSM_MODE_LINE = 1, CTSM_MODE_MULTILINE = 2 };
int ctsm_csr_count_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int angle_begin,
                        int angle_end, uint64_t memory_budget_bytes, uint64_t* row_start_dev,
                        uint64_t* nnz_out, void* stream);
int ctsm_csr_fill_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int angle_begin,
                       int angle_end, const uint64_t* row_start_dev, uint32_t* col_dev,
                       double* val_dev, void* stream);
int ctsm_fwd_mf_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int dtype,
                     int angle_begin, int angle_end, int angle_step, const void* x_dev,
                     void* y_dev, void* stream);
int ctsm_bwd_mf_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int dtype,
                     int angle_begin, int angle_end, int angle_step, const void* y_dev,
                     void* x_dev, void* stream);

/* ---- host-buffer entry points (the reference's value-semantics calls,
 * projector.cpp:235-260; used for end-to-end timing). fp64 host arrays in,
 * fp64 host arrays out; the copies and kernels run on the context's own
 * non-blocking stream and the call returns when the result is on the host,
 * so calls on two contexts from two host threads overlap. ---- */
int ctsm_forward_project_matrix_free_host(ctsm_ctx* ctx, const ctsm_geometry* g,
                                          const double* x_host, double* y_host);
int ctsm_back_project_matrix_free_host(ctsm_ctx* ctx, const ctsm_geometry* g,
                                       const double* y_host, double* x_host);
/* fp32 overloads: fp32 host arrays (BASELINE configs 3/4);
 * the weights are still evaluated in FP64. */
int ctsm_forward_project_matrix_free_host_f32(ctsm_ctx* ctx, const ctsm_geometry* g,
                                              const float* x_host, float* y_host);
int ctsm_back_project_matrix_free_host_f32(ctsm_ctx* ctx, const ctsm_geometry* g,
                                           const float* y_host, float* x_host);

/* ---- independent numerical oracles on the device (
 * oracle.hpp:24-45, oracle.cpp:70-196) ----------------------------------------
 * Batches of n cases given as HOST arrays: boxes[6n] = {x0, x1, y0, y1, zb, zt}
 * per case, phi[n], and the detector cell (m_y[n], m_z[n]) of each case.
 * ctsm_mc_volume_3d: McEstimate of mc_volume_3d -- the volume fraction of
 *   the box inside the cone wedge of the cell by uniform point sampling with
 *   the reference's 16 mt19937_64 sub-streams (seed + shard), so the estimate
 *   is deterministic and the hit count is the reference's for the same libm;
 *   value / std_err / hits (each may be NULL) receive n results.
 * ctsm_multiline_volume_3d: the k x k Gauss-Legendre ray-grid integral.
 * ctsm_gauss_legendre: nodes and weights on [-1, 1] (host). */
int ctsm_mc_volume_3d(ctsm_ctx* ctx, uint64_t n, const double* boxes, const double* phi, double s,
                      double d, double d_y, double d_z, const int32_t* m_y, const int32_t* m_z,
                      uint64_t n_samples, uint64_t seed, double* value, double* std_err,
                      uint64_t* hits);
int ctsm_multiline_volume_3d(ctsm_ctx* ctx, uint64_t n, const double* boxes, const double* phi,
                             double s, double d, double d_y, double d_z, const int32_t* m_y,
                             const int32_t* m_z, int k, double* out);
void ctsm_gauss_legendre(int k, double* x, double* w);

/* ---- multi-GPU context --------------------------
 * One process, n devices: each device gets its own ctsm_ctx and stream, the
 * angles are sharded over the devices (ctsm_shard_angles: by symmetry orbits
 * for quarter-turn / dihedral scans, else strided), A x needs no
 * communication, and A^T y / SIRT sum the partial volumes with ncclAllReduce
 * over the devices' communicators (ncclCommInitAll; NCCL is bound at run time
 * from libnccl.so.2). Operands are HOST arrays of the dtype; x is replicated.
 * With one device no NCCL call is made (unless CTSM_MULTI_FORCE_NCCL=1, which
 * runs the one-rank communicator: used by the tests on single-GPU boxes).
 * ctsm_shard_angles: the angles (ascending) of rank `rank` of `world`, their
 * count, and whether the shard is an orbit shard (base angles rank, rank +
 * world, ... with all their images) -- the partition torch.distributed
 * callers (paper_2511_12235_b200/dist.py) and this context share. */
typedef struct ctsm_multi ctsm_multi;
int ctsm_shard_angles(const ctsm_geometry* g, int rank, int world, int* angles_out, int* n_out,
                      int* orbits_out);
int ctsm_multi_create(const int* devices, int n, ctsm_multi** out);
int ctsm_multi_destroy(ctsm_multi* m);
int ctsm_multi_size(const ctsm_multi* m);
int ctsm_multi_nccl_version(const ctsm_multi* m); /* 0 if no communicator was created */
int ctsm_multi_forward_project_matrix_free_host(ctsm_multi* m, const ctsm_geometry* g, int dtype,
                                                const void* x_host, void* y_host);
int ctsm_multi_back_project_matrix_free_host(ctsm_multi* m, const ctsm_geometry* g, int dtype,
                                             const void* y_host, void* x_host);
int ctsm_multi_sirt_host(ctsm_multi* m, const ctsm_geometry* g, int dtype, const void* y_host,
                         void* x_inout_host, int iters);

/* ---- diagnostics ---------------------------------------------------------
 * ctsm_selftest_division: the exact 3D emission divides by per-column
 * constants with a precomputed correctly rounded reciprocal and one fma
 * correction (csr3d.cuh div_by), which returns the IEEE quotient; this runs
 * the sequence against the division instruction on n pseudo-random operand
 * pairs and reports the number of differing results (expected 0).
 *
 * Measured FP64 FMA throughput of `device` in TFLOP/s (FMA = 2 flops): the
 * FP64 roofline denominator used by bench.py (MEASURED_PEAKS.json has none). */
double ctsm_bench_dfma(int device);
int ctsm_selftest_division(ctsm_ctx* ctx, uint64_t n, uint64_t seed, uint64_t* mismatches);

#ifdef __cplusplus
}
#endif
