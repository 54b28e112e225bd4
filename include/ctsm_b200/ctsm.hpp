// ctsm_b200/ctsm.hpp -- C++ drop-in for the reference's projector hot path.
//
// Same namespace, types and signatures as the reference headers
// (/root/reference/proj/include/ctsm/{common,geometry,projector}.hpp), so a
// caller of the reference switches by pointing its include path here and
// linking libctsm_b200.so instead of libctsm.a. Implemented in
// paper_2511_12235_b200/csrc/api.cpp over the C-ABI (include/ctsm_b200.h);
// all compute runs on the GPU (no CPU fallback).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ctsm {

// common.hpp:11-25
enum class ErrorCode {
  DegenerateGeometry,
  RayParallelToFace,
  SingularPhi,
  CentralRow,
  ZRestrictionViolation,
  DimensionMismatch,
  NonFinite,
  ZeroMatrix,
  TooLarge,
  InvalidSpec,
  OutOfMemory,
  InvalidConfig,
  IoFailure,
};

const char* error_code_name(ErrorCode code);

// common.hpp:29-38
class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(error_code_name(code)) + ": " + message), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

inline constexpr double k_pi = 3.14159265358979323846;

// geometry.hpp:29-64
struct ScanGeometry {
  double s = 0.0;
  double d = 0.0;
  double d_y = 1.0;
  double d_z = 1.0;
  int n_det_y = 0;
  int n_det_z = 1;
  int n_angles = 0;
  double angle_start = 0.0;
  double angle_end = 2.0 * k_pi;
  double a = 1.0;
  double b = 1.0;
  double c = 1.0;
  int n_x = 0;
  int n_y = 0;
  int n_z = 1;

  void validate() const;  // throws InvalidSpec / DegenerateGeometry / NonFinite

  bool is_2d() const { return n_z == 1 && n_det_z == 1; }
  double sdd() const { return s + d; }
  double angle(int i) const { return angle_start + (angle_end - angle_start) * i / n_angles; }
  double face_x(double ix) const { return (ix - n_x / 2.0) * a; }
  double face_y(double iy) const { return (iy - n_y / 2.0) * b; }
  double face_z(double iz) const { return (iz - n_z / 2.0) * c; }
  std::uint64_t n_voxels() const {
    return std::uint64_t(n_x) * std::uint64_t(n_y) * std::uint64_t(n_z);
  }
  std::uint64_t n_measurements() const {
    return std::uint64_t(n_angles) * std::uint64_t(n_det_y) * std::uint64_t(n_det_z);
  }
};

// geometry.hpp:66-84
struct VoxelIndex {
  int ix = 0, iy = 0, iz = 0;
};
struct DetectorIndex {
  int m_y = 0, m_z = 0;
};
inline std::uint64_t voxel_column(const ScanGeometry& g, const VoxelIndex& n) {
  return (std::uint64_t(n.iz) * g.n_y + n.iy) * g.n_x + n.ix;
}
inline std::uint64_t measurement_row(const ScanGeometry& g, int angle_index,
                                     const DetectorIndex& m) {
  const std::uint64_t raster =
      std::uint64_t(m.m_z + g.n_det_z / 2) * g.n_det_y + (m.m_y + g.n_det_y / 2);
  return std::uint64_t(angle_index) * g.n_det_y * g.n_det_z + raster;
}

// weights2d.hpp:20-32 / weights3d.hpp:82-91: the consistent weights of one
// pixel / voxel at fan angle phi, evaluated on the device (bit-identical to
// the reference with a correctly rounded libm), in the reference's order.
struct CellWeight {
  int m_y = 0;
  double w = 0;
};
struct VoxelWeight {
  int m_y = 0, m_z = 0;
  double w = 0;
};
std::vector<CellWeight> pixel_area_factors(const VoxelIndex& n, double phi, const ScanGeometry& g);
std::vector<VoxelWeight> voxel_volume_factors(const VoxelIndex& n, double phi,
                                              const ScanGeometry& g);
// Additions: many (voxel, phi) queries in one device launch.
std::vector<std::vector<CellWeight>> pixel_area_factors(const std::vector<VoxelIndex>& n,
                                                        const std::vector<double>& phi,
                                                        const ScanGeometry& g);
std::vector<std::vector<VoxelWeight>> voxel_volume_factors(const std::vector<VoxelIndex>& n,
                                                           const std::vector<double>& phi,
                                                           const ScanGeometry& g);

// projector.hpp:12-16
enum class MatrixMode { consistent, line, multiline };

MatrixMode parse_matrix_mode(const std::string& text, int* k);
std::string matrix_mode_name(MatrixMode mode, int k);

// projector.hpp:26-35
struct SparseSystemMatrix {
  std::uint64_t n_rows = 0;
  std::uint64_t n_cols = 0;
  std::vector<std::uint64_t> row_start;
  std::vector<std::uint32_t> col;
  std::vector<double> val;
  std::string meta;
  std::uint64_t nnz() const { return col.size(); }
};

// projector.hpp:41-70 (threads is accepted and ignored: the work runs on the
// GPU; line / multiline(k) run the device ray tracer of baseline.cpp:13-128).
SparseSystemMatrix build_system_matrix(const ScanGeometry& g, MatrixMode mode, int k = 1,
                                       int threads = 1,
                                       std::uint64_t memory_budget_bytes = 5ull << 30);
std::vector<double> forward_project(const SparseSystemMatrix& w, const std::vector<double>& x);
std::vector<double> back_project(const SparseSystemMatrix& w, const std::vector<double>& y);
std::vector<double> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                                const std::vector<double>& x, int threads = 1);
// Addition: matrix-free adjoint.
std::vector<double> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                             const std::vector<double>& y, int threads = 1);
double spectral_norm_power(const SparseSystemMatrix& w, int iters = 100, std::uint64_t seed = 7);
void scale_values(SparseSystemMatrix* w, double factor);
std::vector<double> angle_column_sums(const ScanGeometry& g, MatrixMode mode, int k,
                                      int angle_index);
namespace detail {
// projector.hpp:72-78: every (local row, column, weight) entry of one angle
// block, emitted in the reference's order (projector.cpp:44-84); the entries
// are evaluated and ordered on the device and streamed to the callback.
void angle_block_entries(const ScanGeometry& g, MatrixMode mode, int k, int angle_index,
                         const std::function<void(std::uint32_t, std::uint32_t, double)>& emit);
}  // namespace detail

// Additions: fp32 operands (BASELINE configs 3 and 4; the
// weights are still evaluated in FP64).
std::vector<float> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                               const std::vector<float>& x, int threads = 1);
std::vector<float> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                            const std::vector<float>& y, int threads = 1);

// Addition: a system matrix resident on the device. The value-semantics calls
// above upload the CSR on every call (as the reference's signatures demand);
// a DeviceSystemMatrix is uploaded (or built in place) once and applied many
// times -- the solver loops, spectral_norm_power, repeated projections.
class DeviceSystemMatrix {
 public:
  explicit DeviceSystemMatrix(const SparseSystemMatrix& w);  // upload
  // build_system_matrix on the device, the matrix never leaves it
  DeviceSystemMatrix(const ScanGeometry& g, MatrixMode mode, int k = 1,
                     std::uint64_t memory_budget_bytes = 5ull << 30);
  ~DeviceSystemMatrix();
  DeviceSystemMatrix(const DeviceSystemMatrix&) = delete;
  DeviceSystemMatrix& operator=(const DeviceSystemMatrix&) = delete;
  std::uint64_t n_rows() const;
  std::uint64_t n_cols() const;
  std::uint64_t nnz() const;
  const std::string& meta() const;
  SparseSystemMatrix download() const;
  void scale_values(double factor);
  // keeps a CSC transpose beside the CSR (the CSR's col / val bytes again):
  // back_project(*this, y) then gathers instead of scattering, same bits;
  // scale_values drops it
  void build_transpose();
  bool has_transpose() const;
  struct Impl;
  const Impl& impl() const { return *impl_; }

 private:
  std::unique_ptr<Impl> impl_;
};
std::vector<double> forward_project(const DeviceSystemMatrix& w, const std::vector<double>& x);
std::vector<double> back_project(const DeviceSystemMatrix& w, const std::vector<double>& y);
double spectral_norm_power(const DeviceSystemMatrix& w, int iters = 100, std::uint64_t seed = 7);

// Additions: multi-GPU variants taking a device list:
// angles sharded over the devices, A x without communication, A^T y and SIRT
// with an NCCL all-reduce of the partial volumes inside the library.
std::vector<double> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                                const std::vector<double>& x,
                                                const std::vector<int>& devices);
std::vector<double> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                             const std::vector<double>& y,
                                             const std::vector<int>& devices);
std::vector<float> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                               const std::vector<float>& x,
                                               const std::vector<int>& devices);
std::vector<float> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                            const std::vector<float>& y,
                                            const std::vector<int>& devices);

// oracle.hpp:24-45: the independent numerical oracles, evaluated on the device
// (the dense Eigen helpers of oracle.hpp are out of scope). The batch forms
// take n cases: boxes[6n] = {x0, x1, y0, y1, zb, zt} per case.
struct McEstimate {
  double value = 0;
  double std_err = 0;
};
McEstimate mc_volume_3d(double x0, double x1, double y0, double y1, double zb, double zt,
                        double phi, double s, double d, double d_y, double d_z, int m_y, int m_z,
                        std::uint64_t n_samples, std::uint64_t seed);
double multiline_volume_3d(double x0, double x1, double y0, double y1, double zb, double zt,
                           double phi, double s, double d, double d_y, double d_z, int m_y,
                           int m_z, int k = 200);
std::pair<std::vector<double>, std::vector<double>> gauss_legendre(int k);
std::vector<McEstimate> mc_volume_3d(const std::vector<double>& boxes,
                                     const std::vector<double>& phi, double s, double d,
                                     double d_y, double d_z, const std::vector<int>& m_y,
                                     const std::vector<int>& m_z, std::uint64_t n_samples,
                                     std::uint64_t seed);
std::vector<double> multiline_volume_3d(const std::vector<double>& boxes,
                                        const std::vector<double>& phi, double s, double d,
                                        double d_y, double d_z, const std::vector<int>& m_y,
                                        const std::vector<int>& m_z, int k = 200);

// solver.hpp:10-35: Nesterov-accelerated Tikhonov least squares; the iteration
// runs on the device (ctsm_nag_tikhonov).
struct SolveOptions {
  double lambda = 1e-4;
  int max_iter = 1000;
  double tol = 1e-9;
};
struct SolveTraceRow {
  int iter;
  double objective;
  double grad_norm_sq;
};
struct SolveResult {
  std::vector<double> u;
  int iterations = 0;
  bool converged = false;
  std::vector<SolveTraceRow> trace;
};
SolveResult nag_tikhonov(const SparseSystemMatrix& w, const std::vector<double>& p,
                         const SolveOptions& opt, bool keep_trace = false);
SolveResult nag_tikhonov(const DeviceSystemMatrix& w, const std::vector<double>& p,
                         const SolveOptions& opt, bool keep_trace = false);
// io.hpp:31-48: CSM1 matrices and CTT1 tensors (byte-identical containers).
void write_matrix(const std::string& path, const SparseSystemMatrix& w);
SparseSystemMatrix read_matrix(const std::string& path);
void write_tensor(const std::string& path, const std::vector<std::uint64_t>& dims,
                  const std::vector<double>& data);
std::vector<double> read_tensor(const std::string& path, std::vector<std::uint64_t>* dims);
// Addition: SIRT (BASELINE.json configs[4]) on one device.
std::vector<double> sirt(const ScanGeometry& g, const std::vector<double>& y,
                         const std::vector<double>& x0, int iters);
std::vector<float> sirt(const ScanGeometry& g, const std::vector<float>& y,
                        const std::vector<float>& x0, int iters);
// ... on a device list (rows sharded, x replicated, one all-reduce per iteration)
std::vector<double> sirt(const ScanGeometry& g, const std::vector<double>& y,
                         const std::vector<double>& x0, int iters,
                         const std::vector<int>& devices);
std::vector<float> sirt(const ScanGeometry& g, const std::vector<float>& y,
                        const std::vector<float>& x0, int iters, const std::vector<int>& devices);

}  // namespace ctsm
