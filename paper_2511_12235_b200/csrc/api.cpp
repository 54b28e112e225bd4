// api.cpp -- the reference's C++ projector API (include/ctsm_b200/ctsm.hpp)
// implemented over the C-ABI. Value semantics as the reference: host vectors
// in, host vectors out; device buffers are allocated per call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <random>
#include <sstream>

#include "../../include/ctsm_b200.h"
#include "../../include/ctsm_b200/ctsm.hpp"

namespace ctsm {

const char* error_code_name(ErrorCode code) {
  static const char* names[] = {"DegenerateGeometry", "RayParallelToFace", "SingularPhi",
                                "CentralRow",         "ZRestrictionViolation",
                                "DimensionMismatch",  "NonFinite",         "ZeroMatrix",
                                "TooLarge",           "InvalidSpec",       "OutOfMemory",
                                "InvalidConfig",      "IoFailure"};
  const int i = static_cast<int>(code);
  return (i >= 0 && i < 13) ? names[i] : "UnknownError";
}

namespace {

[[noreturn]] void raise(int status) {
  std::string msg = ctsm_last_error();
  const auto pos = msg.find(": ");
  if (pos != std::string::npos) msg = msg.substr(pos + 2);
  if (status >= 1 && status <= 13) throw Error(static_cast<ErrorCode>(status - 1), msg);
  throw std::runtime_error("CUDA error: " + msg);
}

void check(int status) {
  if (status != 0) raise(status);
}

ctsm_ctx* ctx() {
  static std::mutex mu;
  static ctsm_ctx* c = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!c) {
    int dev = 0;
    cudaGetDevice(&dev);
    check(ctsm_create(dev, &c));
  }
  return c;
}

ctsm_geometry to_c(const ScanGeometry& g) {
  ctsm_geometry c{};
  c.s = g.s;
  c.d = g.d;
  c.d_y = g.d_y;
  c.d_z = g.d_z;
  c.n_det_y = g.n_det_y;
  c.n_det_z = g.n_det_z;
  c.n_angles = g.n_angles;
  c.angle_start = g.angle_start;
  c.angle_end = g.angle_end;
  c.a = g.a;
  c.b = g.b;
  c.c = g.c;
  c.n_x = g.n_x;
  c.n_y = g.n_y;
  c.n_z = g.n_z;
  return c;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n && cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error(ErrorCode::OutOfMemory, "device allocation failed");
    }
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void reset(size_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    if (n && cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw Error(ErrorCode::OutOfMemory, "device allocation failed");
    }
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

template <typename T>
void h2d(T* d, const T* h, size_t n) {
  if (n && cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    throw std::runtime_error("cudaMemcpy H2D failed");
}
template <typename T>
void d2h(T* h, const T* d, size_t n) {
  if (n && cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
    throw std::runtime_error("cudaMemcpy D2H failed");
}

// MatrixMode ordinal for the C-ABI (CTSM_MODE_*; projector.hpp:12-16).
int mode_code(MatrixMode mode) { return static_cast<int>(mode); }

// phantoms.cpp:78-87 convention (mt19937_64, Box-Muller cosine branch)
std::vector<double> normal_samples(std::size_t n, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<double> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    const double u1 = ((rng() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (rng() >> 11) * 0x1.0p-53;
    out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * k_pi * u2);
  }
  return out;
}

}  // namespace

void ScanGeometry::validate() const {
  const ctsm_geometry c = to_c(*this);
  check(ctsm_validate_geometry(&c));
}

MatrixMode parse_matrix_mode(const std::string& text, int* k) {
  *k = 1;
  if (text == "consistent") return MatrixMode::consistent;
  if (text == "line") return MatrixMode::line;
  if (text.rfind("multiline:", 0) == 0) {
    try {
      *k = std::stoi(text.substr(10));
    } catch (const std::exception&) {
      throw Error(ErrorCode::InvalidConfig, "bad multiline ray count in '" + text + "'");
    }
    if (*k <= 0) throw Error(ErrorCode::InvalidConfig, "multiline ray count must be > 0");
    return MatrixMode::multiline;
  }
  throw Error(ErrorCode::InvalidConfig, "unknown matrix mode '" + text + "'");
}

std::string matrix_mode_name(MatrixMode mode, int k) {
  switch (mode) {
    case MatrixMode::consistent: return "consistent";
    case MatrixMode::line: return "line";
    case MatrixMode::multiline: return "multiline:" + std::to_string(k);
  }
  return "?";
}

SparseSystemMatrix build_system_matrix(const ScanGeometry& g, MatrixMode mode, int k, int threads,
                                       std::uint64_t memory_budget_bytes) {
  (void)threads;
  const ctsm_geometry c = to_c(g);
  check(ctsm_validate_geometry(&c));
  SparseSystemMatrix w;
  w.n_rows = g.n_measurements();
  w.n_cols = g.n_voxels();
  DevBuf<std::uint64_t> rs(w.n_rows + 1);
  std::uint64_t nnz = 0;
  DevBuf<std::uint32_t> col(0);
  DevBuf<double> val(0);
  if (mode == MatrixMode::consistent) {
    // single evaluation: arrays sized from the angle-0 estimate
    std::uint64_t nnz0 = 0;
    check(ctsm_csr_angle_nnz(ctx(), &c, 0, &nnz0, nullptr));
    std::uint64_t cap = (std::uint64_t)((double)nnz0 * g.n_angles * 1.2) + 65536;
    if (12 * nnz0 * (std::uint64_t)g.n_angles + 8 * (w.n_rows + 1) > memory_budget_bytes) cap = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      col.reset(cap);
      val.reset(cap);
      check(ctsm_csr_build(ctx(), &c, 0, g.n_angles, memory_budget_bytes, rs.p, col.p, val.p, cap,
                           &nnz, nullptr));
      if (nnz <= cap) break;
      cap = nnz;
    }
  } else {
    check(ctsm_csr_count_mode(ctx(), &c, mode_code(mode), k, 0, g.n_angles, memory_budget_bytes,
                              rs.p, &nnz, nullptr));
    col.reset(nnz);
    val.reset(nnz);
    check(ctsm_csr_fill_mode(ctx(), &c, mode_code(mode), k, 0, g.n_angles, rs.p, col.p, val.p,
                             nullptr));
  }
  w.row_start.resize(w.n_rows + 1);
  w.col.resize(nnz);
  w.val.resize(nnz);
  d2h(w.row_start.data(), rs.p, w.n_rows + 1);
  d2h(w.col.data(), col.p, nnz);
  d2h(w.val.data(), val.p, nnz);
  std::ostringstream meta;  // projector.cpp:191-199
  meta << "mode=" << matrix_mode_name(mode, k) << "\n";
  meta << "s=" << g.s << "\nd=" << g.d << "\ndy=" << g.d_y << "\ndz=" << g.d_z
       << "\nndy=" << g.n_det_y << "\nndz=" << g.n_det_z << "\nnp=" << g.n_angles
       << "\nangle_start=" << g.angle_start << "\nangle_end=" << g.angle_end << "\na=" << g.a
       << "\nb=" << g.b << "\nc=" << g.c << "\nnx=" << g.n_x << "\nny=" << g.n_y
       << "\nnz=" << g.n_z << "\n";
  w.meta = meta.str();
  return w;
}

namespace {
struct DevCsr {
  DevBuf<std::uint64_t> rs;
  DevBuf<std::uint32_t> col;
  DevBuf<double> val;
  explicit DevCsr(const SparseSystemMatrix& w)
      : rs(w.row_start.size()), col(w.col.size()), val(w.val.size()) {
    h2d(rs.p, w.row_start.data(), w.row_start.size());
    h2d(col.p, w.col.data(), w.col.size());
    h2d(val.p, w.val.data(), w.val.size());
  }
};
}  // namespace

std::vector<double> forward_project(const SparseSystemMatrix& w, const std::vector<double>& x) {
  if (x.size() != w.n_cols)
    throw Error(ErrorCode::DimensionMismatch, "image size does not match matrix columns");
  DevCsr m(w);
  DevBuf<double> xd(x.size()), yd(w.n_rows);
  h2d(xd.p, x.data(), x.size());
  check(ctsm_spmv(ctx(), w.n_rows, w.n_cols, m.rs.p, m.col.p, m.val.p, xd.p, yd.p, nullptr));
  std::vector<double> y(w.n_rows);
  d2h(y.data(), yd.p, y.size());
  return y;
}

std::vector<double> back_project(const SparseSystemMatrix& w, const std::vector<double>& y) {
  if (y.size() != w.n_rows)
    throw Error(ErrorCode::DimensionMismatch, "sinogram size does not match matrix rows");
  DevCsr m(w);
  DevBuf<double> yd(y.size()), xd(w.n_cols);
  h2d(yd.p, y.data(), y.size());
  check(ctsm_spmv_t(ctx(), w.n_rows, w.n_cols, m.rs.p, m.col.p, m.val.p, yd.p, xd.p, nullptr));
  std::vector<double> x(w.n_cols);
  d2h(x.data(), xd.p, x.size());
  return x;
}

std::vector<double> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                                const std::vector<double>& x, int threads) {
  (void)threads;
  g.validate();
  if (x.size() != g.n_voxels())
    throw Error(ErrorCode::DimensionMismatch, "image size does not match the grid");
  const ctsm_geometry c = to_c(g);
  std::vector<double> y(g.n_measurements());
  if (mode == MatrixMode::consistent) {
    check(ctsm_forward_project_matrix_free_host(ctx(), &c, x.data(), y.data()));
    return y;
  }
  DevBuf<double> xd(x.size()), yd(y.size());
  h2d(xd.p, x.data(), x.size());
  check(ctsm_fwd_mf_mode(ctx(), &c, mode_code(mode), k, CTSM_F64, 0, g.n_angles, 1, xd.p, yd.p,
                         nullptr));
  d2h(y.data(), yd.p, y.size());
  return y;
}

std::vector<double> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                             const std::vector<double>& y, int threads) {
  (void)threads;
  g.validate();
  if (y.size() != g.n_measurements())
    throw Error(ErrorCode::DimensionMismatch, "sinogram size does not match the scan");
  const ctsm_geometry c = to_c(g);
  std::vector<double> x(g.n_voxels());
  if (mode == MatrixMode::consistent) {
    check(ctsm_back_project_matrix_free_host(ctx(), &c, y.data(), x.data()));
    return x;
  }
  DevBuf<double> yd(y.size()), xd(x.size());
  h2d(yd.p, y.data(), y.size());
  check(ctsm_bwd_mf_mode(ctx(), &c, mode_code(mode), k, CTSM_F64, 0, g.n_angles, 1, yd.p, xd.p,
                         nullptr));
  d2h(x.data(), xd.p, x.size());
  return x;
}

// ---- io (CSM1 through the device streaming writer/reader; CTT1 host) ----
void write_matrix(const std::string& path, const SparseSystemMatrix& w) {
  if (w.row_start.size() != w.n_rows + 1)
    throw Error(ErrorCode::DimensionMismatch, "row offsets do not match the row count");
  DevCsr m(w);
  check(ctsm_write_csm1_device(ctx(), path.c_str(), w.n_rows, w.n_cols, m.rs.p, m.col.p,
                               m.val.p, w.meta.data(), w.meta.size(), nullptr));
}

SparseSystemMatrix read_matrix(const std::string& path) {
  std::uint64_t n_rows = 0, n_cols = 0, nnz = 0, meta_len = 0;
  check(ctsm_csm1_header(path.c_str(), &n_rows, &n_cols, &nnz, &meta_len));
  SparseSystemMatrix w;
  w.n_rows = n_rows;
  w.n_cols = n_cols;
  w.meta.assign(meta_len, '\0');
  DevBuf<std::uint64_t> rs(n_rows + 1);
  DevBuf<std::uint32_t> col(nnz);
  DevBuf<double> val(nnz);
  check(ctsm_read_csm1_device(ctx(), path.c_str(), rs.p, col.p, val.p,
                              meta_len ? &w.meta[0] : nullptr, nullptr));
  w.row_start.resize(n_rows + 1);
  w.col.resize(nnz);
  w.val.resize(nnz);
  d2h(w.row_start.data(), rs.p, w.row_start.size());
  d2h(w.col.data(), col.p, w.col.size());
  d2h(w.val.data(), val.p, w.val.size());
  return w;
}

void write_tensor(const std::string& path, const std::vector<std::uint64_t>& dims,
                  const std::vector<double>& data) {
  if (dims.empty() || dims.size() > 8)
    throw Error(ErrorCode::InvalidSpec, "tensor rank must be between 1 and 8");
  std::uint64_t count = 1;
  for (std::uint64_t d : dims) count *= d;
  if (count != data.size())
    throw Error(ErrorCode::DimensionMismatch, "tensor dims do not match payload size");
  check(ctsm_write_ctt1(path.c_str(), dims.data(), (int)dims.size(), data.data()));
}

std::vector<double> read_tensor(const std::string& path, std::vector<std::uint64_t>* dims) {
  std::uint64_t d[8];
  int rank = 0;
  check(ctsm_ctt1_header(path.c_str(), d, &rank));
  dims->assign(d, d + rank);
  std::uint64_t count = 1;
  for (int i = 0; i < rank; ++i) count *= d[i];
  std::vector<double> out(count);
  check(ctsm_read_ctt1(path.c_str(), out.data(), count));
  return out;
}

double spectral_norm_power(const SparseSystemMatrix& w, int iters, std::uint64_t seed) {
  if (w.nnz() == 0) throw Error(ErrorCode::ZeroMatrix, "matrix has no entries");
  const std::vector<double> v = normal_samples(w.n_cols, seed);
  DevCsr m(w);
  DevBuf<double> vd(w.n_cols);
  h2d(vd.p, v.data(), v.size());
  ctsm_operator op{};
  op.kind = CTSM_OP_CSR;
  op.n_rows = w.n_rows;
  op.n_cols = w.n_cols;
  op.row_start = m.rs.p;
  op.col = m.col.p;
  op.val = m.val.p;
  op.scale = 1.0;
  double out = 0.0;
  check(ctsm_spectral_norm_power(ctx(), &op, iters, vd.p, &out, nullptr));
  return out;
}

SolveResult nag_tikhonov(const SparseSystemMatrix& w, const std::vector<double>& p,
                         const SolveOptions& opt, bool keep_trace) {
  if (p.size() != w.n_rows)
    throw Error(ErrorCode::DimensionMismatch, "data size does not match matrix rows");
  if (!(opt.lambda >= 0.0) || !(opt.tol >= 0.0) || opt.max_iter < 0)
    throw Error(ErrorCode::InvalidConfig, "solver options must be nonnegative");
  SolveResult res;
  res.u.assign(w.n_cols, 0.0);
  if (w.nnz() == 0) throw Error(ErrorCode::ZeroMatrix, "matrix has no entries");
  DevCsr m(w);
  DevBuf<double> pd(w.n_rows), ud(w.n_cols);
  h2d(pd.p, p.data(), p.size());
  ctsm_operator op{};
  op.kind = CTSM_OP_CSR;
  op.n_rows = w.n_rows;
  op.n_cols = w.n_cols;
  op.row_start = m.rs.p;
  op.col = m.col.p;
  op.val = m.val.p;
  op.scale = 1.0;
  std::vector<double> tr(keep_trace ? 3 * (size_t)std::max(opt.max_iter, 1) : 0);
  int its = 0, conv = 0;
  check(ctsm_nag_tikhonov(ctx(), &op, pd.p, opt.lambda, opt.max_iter, opt.tol, ud.p,
                          keep_trace ? tr.data() : nullptr, &its, &conv, nullptr));
  d2h(res.u.data(), ud.p, res.u.size());
  res.iterations = its;
  res.converged = conv != 0;
  for (int i = 0; keep_trace && i < its; ++i)
    res.trace.push_back({(int)tr[3 * i], tr[3 * i + 1], tr[3 * i + 2]});
  return res;
}

void scale_values(SparseSystemMatrix* w, double factor) {
  if (!std::isfinite(factor)) throw Error(ErrorCode::NonFinite, "scale factor must be finite");
  for (double& v : w->val) v *= factor;
}

std::vector<double> angle_column_sums(const ScanGeometry& g, MatrixMode mode, int k,
                                      int angle_index) {
  g.validate();
  const ctsm_geometry c = to_c(g);
  DevBuf<double> yd(g.n_measurements()), xd(g.n_voxels());
  std::vector<double> ones(g.n_measurements(), 1.0), x(g.n_voxels());
  h2d(yd.p, ones.data(), ones.size());
  check(ctsm_bwd_mf_mode(ctx(), &c, mode_code(mode), k, CTSM_F64, angle_index, angle_index + 1,
                         1, yd.p, xd.p, nullptr));
  d2h(x.data(), xd.p, x.size());
  return x;
}

std::vector<double> sirt(const ScanGeometry& g, const std::vector<double>& y,
                         const std::vector<double>& x0, int iters) {
  g.validate();
  if (y.size() != g.n_measurements() || x0.size() != g.n_voxels())
    throw Error(ErrorCode::DimensionMismatch, "operand sizes do not match the scan");
  const ctsm_geometry c = to_c(g);
  DevBuf<double> yd(y.size()), xd(x0.size());
  h2d(yd.p, y.data(), y.size());
  h2d(xd.p, x0.data(), x0.size());
  check(ctsm_sirt(ctx(), &c, CTSM_F64, yd.p, xd.p, iters, nullptr));
  std::vector<double> x(x0.size());
  d2h(x.data(), xd.p, x.size());
  return x;
}

}  // namespace ctsm

extern "C" void ctsm_normal_samples(uint64_t n, uint64_t seed, double* out) {
  const std::vector<double> v = ctsm::normal_samples((std::size_t)n, seed);
  std::copy(v.begin(), v.end(), out);
}
