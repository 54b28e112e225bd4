// kernels.h -- host-side launchers shared between the compilation units.
// csr.cu (compiled with -fmad=false: bit-exact emission) and mf.cu (matrix-free
// projectors) implement them; capi.cu orchestrates.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "common.cuh"

struct ctsm_ctx;

namespace ctsmb {

namespace exact {
struct ExactAngle;
struct EdgeAngle;
}  // namespace exact

// Global launch counter (reported by ctsm_launch_count).
void count_launch(int n = 1);
// Sets the thread-local last-error message (ctsm_last_error) and returns code.
int set_error(int code, const char* msg);
inline int set_error(int code, const std::string& msg) { return set_error(code, msg.c_str()); }
// cudaSetDevice(ctx's device) (capi.cu); 0 or an error code.
int select_device(::ctsm_ctx* ctx);

// ---- csr.cu --------------------------------------------------------------
size_t exact_angle_bytes();
size_t edge_angle_bytes();
cudaError_t build_exact_tables(const DevGeom& g, int angle_begin, int n_sel, void* angles_dev,
                               void* edges_dev, cudaStream_t st);
// Output sink of the CSR emission kernels (csr3d.cuh Sink):
//   mode 0: count entries per row into row_counter (u32, zeroed by the caller);
//   mode 1: write row-grouped 16-byte entries {col, -, val} to grp at
//           row_start[row] - pos_base + slot, row_counter as slot cursors;
//   mode 2: count and append 16-byte records {row, col, val} to rec[0..cap),
//           allocated from *cursor (zeroed by the caller; cursor > cap means
//           records were dropped: retry with a larger buffer).
struct CsrSink {
  int mode;
  unsigned* row_counter;
  const uint64_t* row_start;
  void* grp;
  void* rec;
  unsigned long long* cursor;
  unsigned long long cap;
  uint64_t pos_base;
};
// div_by (csr3d.cuh) against the IEEE division on n pseudo-random operand
// pairs; adds the number of differing results to *mismatches_dev.
cudaError_t selftest_division(unsigned long long n, unsigned long long seed,
                              unsigned long long* mismatches_dev, cudaStream_t st);
// Bytes of the per-(column, angle) plan scratch of the 3D emission (0 for 2D).
size_t csr_plan_bytes(const DevGeom& g, int n_sel);
// Emits the rows of the n_sel angles of the prepared tables (rows local to
// the shard) into `out`.
cudaError_t csr_emit(const DevGeom& g, const void* angles_dev, const void* edges_dev, int n_sel,
                     const CsrSink& out, void* plans, int* status, cudaStream_t st);
// Single-evaluation build, after a mode-2 emission and the row scan: records
// -> row-grouped 16-byte entries (cursor = the rows' shard-local offsets, from
// the scan's local_out) -> per-row radix sort by column into the final arrays.
// row_start points at the chunk's first row and holds global offsets: the
// grouped array (grp_cap entries) starts at entry row_start[0], col_out /
// val_out are the whole matrix's arrays (out_cap
// entries; rows reaching beyond are skipped). The record count is read from
// device memory (*n_dev, clamped to cap), so the host never waits on a chunk.
// n_cols (if given and <= 2^22) lets the sort pack a key and its entry index
// into one 32-bit word.
cudaError_t csr_scatter_records(const void* rec, const unsigned long long* n_dev,
                                unsigned long long cap, unsigned* cursor, void* grp,
                                uint64_t grp_cap, cudaStream_t st);
cudaError_t csr_sort_rows_radix(uint64_t n_rows, const uint64_t* row_start, const void* grp,
                                uint32_t* col_out, double* val_out, uint64_t out_cap,
                                uint64_t grp_cap, unsigned* long_rows, unsigned* n_long,
                                cudaStream_t st, uint64_t n_cols = 0);
// row_start[0..n] = exclusive scan of counts[0..n-1] (u32 -> u64); scratch
// needs scan_scratch_bytes(n).
size_t scan_scratch_bytes(uint64_t n);
cudaError_t exclusive_scan_u32_u64(const unsigned* counts, uint64_t n, uint64_t* row_start,
                                   void* scratch, cudaStream_t st, uint64_t base = 0,
                                   const uint64_t* base_dev = nullptr,
                                   unsigned* local_out = nullptr);
cudaError_t spmv_csr(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                     const double* val, const double* x, double* y, int* status, cudaStream_t st);
cudaError_t colsum_abs(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                       const double* val, double* colsum, cudaStream_t st);
cudaError_t spmvt_csr_fixed(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                            const double* val, const double* y, unsigned long long* acc,
                            double scale, cudaStream_t st);
// K4 as a gather over a CSC transpose (csr.cu): column counts, slot scatter
// (after the caller's scan of the counts), and the fixed-point applier
cudaError_t csc_count(uint64_t nnz, const uint32_t* col, unsigned* counts, cudaStream_t st);
cudaError_t csc_scatter(uint64_t n_rows, const uint64_t* row_start, const uint32_t* col,
                        const double* val, const uint64_t* col_start, unsigned* cursor,
                        uint32_t* row_out, double* val_out, cudaStream_t st);
cudaError_t spmvt_csc_fixed(uint64_t n_cols, const uint64_t* col_start, const uint32_t* row,
                            const double* val, const double* y, unsigned long long* acc,
                            double scale, cudaStream_t st);

// ---- weights.cu: the reference's weight API on the device ------------------
// pixel_area_factors / voxel_volume_factors (weights2d.cpp:105-129,
// weights3d.cpp:354-462) for n_q (voxel, phi) queries (device arrays); query q
// writes its weights, in the reference's order, to slab q of `cap` entries
// and count[q] (which may exceed cap: the slab then holds the first cap).
cudaError_t weights_batch(const DevGeom& g, const void* edges_dev, long long n_q, const int* ix,
                          const int* iy, const int* iz, const double* phi, int cap, int* count,
                          int* my, int* mz, double* w, int* status, cudaStream_t st);
// Mode-2 emission records of ONE angle -> (raster, col, w) in the reference's
// emission order (projector.cpp:44-84): counting sort by column, then each
// column's entries by (m_y, m_z). counts: n_cols u32; scan_tmp: n_cols + 1
// u64; tmp: cap 16-byte records.
cudaError_t records_to_emission_order(const void* rec, const unsigned long long* n_dev,
                                      unsigned long long cap, uint64_t n_cols, unsigned* counts,
                                      uint64_t* scan_tmp, void* scan_scratch, void* tmp,
                                      int n_det_y, int n_det_z, uint32_t* raster, uint32_t* col,
                                      double* w, cudaStream_t st);
// raster[j] = r for the entries j of row r (CSR of one angle block).
cudaError_t expand_row_index(uint64_t n_rows, const uint64_t* row_start, uint32_t* raster,
                             cudaStream_t st);

// ---- oracles.cu: mc_volume_3d / multiline_volume_3d (oracle.cpp:70-196) -----
// Batches of cases (device arrays: box[6n] = x0 x1 y0 y1 zb zt, phi[n], my[n],
// mz[n]); hits[n] (zeroed by the caller) receives the MC hit counts.
cudaError_t mc_volume_batch(long long n_cases, const double* box, const double* phi, double s,
                            double d, double d_y, double d_z, const int* my, const int* mz,
                            unsigned long long n_samples, unsigned long long seed,
                            unsigned long long* hits, cudaStream_t st);
cudaError_t multiline_volume_batch(long long n_cases, const double* box, const double* phi,
                                   double s, double d, double d_y, double d_z, const int* my,
                                   const int* mz, int k, const double* nodes, const double* wts,
                                   double* out, cudaStream_t st);
void gauss_legendre_host(int k, double* x, double* w);

// ---- mf.cu ---------------------------------------------------------------
// Pieces one column sweep of the 3D matrix-free kernels may hold (fast3dw.cuh).
int mf3d_max_pieces();
struct AngleCS {
  double C, S;
};
cudaError_t build_angle_cs(const DevGeom& g, int angle_begin, int angle_step, int n_sel,
                           AngleCS* out, cudaStream_t st);
// dtype: CTSM_F64 / CTSM_F32
// Quarter-turn symmetric variants (square grid, full turn, n_angles % 4 == 0):
// weights are evaluated at the base angles base[0..n_base) (< n_angles / 4)
// and applied to all four quarter-turn images (angles base + k n_angles / 4).
cudaError_t build_angle_cs_list(const DevGeom& g, const int* idx, int n, AngleCS* out,
                                cudaStream_t st);
cudaError_t fwd_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                       int n_base, const void* x, unsigned long long* yacc, double scale,
                       unsigned long long* n_upd, int* status, cudaStream_t st);
int bwd_sym_chunks(const DevGeom& g, int n_base);
cudaError_t bwd_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                       int n_base, const void* y, void* x, double* part, int n_chunks,
                       int* status, cudaStream_t st);
// Dihedral (8-fold) 2D variants: base angles 0 <= i <= n/8 (3D: order 8 of
// fwd3d_mf_sym / bwd3d_mf_sym).
cudaError_t fwd_mf_d8(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                      int n_base, const void* x, unsigned long long* yacc, double scale,
                      unsigned long long* n_upd, int* status, cudaStream_t st);
int bwd_d8_chunks(const DevGeom& g, int n_base);
// yt: scratch of bwd_d8_scratch_elems() elements of the dtype (the base
// angles' rows with their 8 images interleaved), or null (direct gathers)
size_t bwd_d8_scratch_elems(const DevGeom& g, int n_base, int dtype);
cudaError_t bwd_mf_d8(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                      int n_base, const void* y, void* x, double* part, int n_chunks,
                      int* status, cudaStream_t st, void* yt);
// mode 0: zero the fixed-point rows of the listed angles; mode 1: convert them
cudaError_t rows_list(const DevGeom& g, int dtype, const int* angles, int n_list,
                      unsigned long long* acc, double scale, void* y, int mode, cudaStream_t st);
// The symmetric 3D kernels read / write the volume in the z-fastest layout
// [n_y][n_x][n_z] (a lane's z-chunk is contiguous): vol_t is an n_vox scratch
// of the dtype; fwd transposes x into it, bwd accumulates into it and
// transposes the result into x.
// fp32 dihedral 3D forward with vector float reductions into an interleaved
// scratch yt of fwd3d_f32_scratch_elems() floats (0: use fwd3d_mf_sym);
// writes y (fp32) directly for every image angle of the base angles.
size_t fwd3d_f32_scratch_elems(const DevGeom& g, int order);
cudaError_t fwd3d_mf_d8_f32(const DevGeom& g, const AngleCS* cs, const int* base, int n_base,
                            const float* x_in, float* y, unsigned long long* n_upd, int* status,
                            cudaStream_t st, void* vol_t, float* yt, void* plans = nullptr);
cudaError_t fwd3d_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                         int n_base, const void* x, unsigned long long* yacc, double scale,
                         unsigned long long* n_upd, int* status, cudaStream_t st, int order,
                         void* vol_t, void* plans = nullptr);
// scratch: bwd3d_scratch_elems(...) elements of the dtype (transposed image
// rows of one L2 chunk), or NULL for the untransposed gather.
size_t bwd3d_scratch_elems(const DevGeom& g, int order, int dtype);
cudaError_t bwd3d_mf_sym(const DevGeom& g, int dtype, const AngleCS* cs, const int* base,
                         int n_base, const void* y, void* x, int* status, cudaStream_t st,
                         int order, void* scratch, void* vol_t, void* plans = nullptr);
// Plan scratch of one launch of the symmetric 3D kernels (0: plan in-kernel):
// the (column, base angle) plans of a launch are computed one per thread by a
// plan pass instead of by every projection warp.
size_t mf3d_plan_bytes(const DevGeom& g, int order);
size_t mf3d_plan_bytes_general(const DevGeom& g);  // the per-angle kernels (fwd_mf / bwd_mf)
cudaError_t fwd_mf(const DevGeom& g, int dtype, const AngleCS* cs, int angle_begin,
                   int angle_step, int n_sel, const void* x, unsigned long long* yacc,
                   double scale, unsigned long long* n_upd, int* status, cudaStream_t st,
                   void* plans = nullptr);
// Backward uses n_chunks angle chunks (bwd_chunks) with a partial-sum buffer
// part of n_chunks * n_x * n_y doubles when n_chunks > 1 (2D only).
int bwd_chunks(const DevGeom& g, int n_sel);
cudaError_t bwd_mf(const DevGeom& g, int dtype, const AngleCS* cs, int angle_begin,
                   int angle_step, int n_sel, const void* y, void* x, double* part, int n_chunks,
                   int* status, cudaStream_t st, void* plans = nullptr);
// y rows of the shard <- acc / scale (and acc rows zeroed for reuse)
cudaError_t fixed_to_float_rows(const DevGeom& g, int dtype, int angle_begin, int angle_step,
                                int n_sel, unsigned long long* acc, double scale, void* y,
                                cudaStream_t st);
cudaError_t fixed_to_double(uint64_t n, const unsigned long long* acc, double scale, double* out,
                            cudaStream_t st);
cudaError_t zero_rows_u64(const DevGeom& g, int angle_begin, int angle_step, int n_sel,
                          unsigned long long* acc, cudaStream_t st);
// max |v| over n elements -> *out (device double), dtype-aware
cudaError_t max_abs(int dtype, uint64_t n, const void* v, double* out_dev, cudaStream_t st);
cudaError_t invert_nonzero(int dtype, uint64_t n, void* v, cudaStream_t st);
cudaError_t sirt_residual(const DevGeom& g, int dtype, int angle_begin, int angle_step,
                          int n_sel, const void* y, const void* rinv, void* ax,
                          cudaStream_t st);
cudaError_t sirt_update(int dtype, uint64_t n, const void* cinv, const void* bp, void* x,
                        cudaStream_t st);
cudaError_t fill_value(int dtype, uint64_t n, double v, void* out, cudaStream_t st);

// ---- line.cu: line / multiline(k) rays (baseline.cpp:13-128) --------------
size_t ray_angle_bytes();
cudaError_t ray_angle_table(const DevGeom& g, int angle_begin, int angle_step, int n_sel,
                            void* angles_dev, cudaStream_t st);
cudaError_t ray_count(const DevGeom& g, const void* angles_dev, int mode, int k, uint64_t n_rows,
                      unsigned* counts, cudaStream_t st);
cudaError_t ray_fill(const DevGeom& g, const void* angles_dev, int mode, int k, uint64_t n_rows,
                     const uint64_t* start, uint32_t* col, double* val, cudaStream_t st);
cudaError_t ray_sort_merge(uint64_t n_rows, const uint64_t* start, unsigned* counts, uint32_t* col,
                           double* val, unsigned* long_rows, unsigned* n_long, int* status,
                           cudaStream_t st);
cudaError_t ray_compact(uint64_t n_rows, const uint64_t* raw_start, const uint64_t* row_start,
                        const uint32_t* rcol, const double* rval, uint32_t* col, double* val,
                        cudaStream_t st);
cudaError_t ray_fwd_mf(const DevGeom& g, int dtype, const void* angles_dev, int mode, int k,
                       int angle_begin, int angle_step, int n_sel, const void* x, void* y,
                       unsigned long long* n_upd, int* status, cudaStream_t st);
cudaError_t ray_bwd_mf(const DevGeom& g, int dtype, const void* angles_dev, int mode, int k,
                       int angle_begin, int angle_step, int n_sel, const void* y,
                       unsigned long long* acc, double scale, void* x, cudaStream_t st);

}  // namespace ctsmb

namespace ctsmb {
// Measured FP64 FMA throughput of the device in TFLOP/s (FMA = 2 flops).
double bench_dfma_tflops(int device);
// ---- solver.cu (deterministic vector kernels of the solvers) --------------
size_t solver_partial_doubles();
cudaError_t nag_step(uint64_t n, double m, double lam, double L, double* u, double* u_prev,
                     double* h, double* h_prev, const double* q, cudaStream_t st);
cudaError_t nag_grad_sq(uint64_t n, double hs, double lam, double* h, const double* u,
                        const double* q, double* partial, double* out_dev, cudaStream_t st);
cudaError_t nag_trace_sums(uint64_t n_rows, uint64_t n_cols, double vs, double* v,
                           const double* p, const double* u, double* partial, double* out_dev,
                           cudaStream_t st);
cudaError_t norm2(uint64_t n, const double* a, double scale, double* partial, double* out_dev,
                  cudaStream_t st);
cudaError_t normalize_by(uint64_t n, const double* u, double us, const double* lam_dev,
                         double* v, int* status, cudaStream_t st);
cudaError_t scale_in_place(uint64_t n, double* v, double f, cudaStream_t st);

}  // namespace ctsmb
