// api.cpp -- the reference's C++ projector API (include/ctsm_b200/ctsm.hpp)
// implemented over the C-ABI. Value semantics as the reference: host vectors
// in, host vectors out; device buffers are allocated per call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
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

// One context per (host thread, device): the reference's functions are
// re-entrant, and a ctsm_ctx owns scratch buffers, a status word and streams
// that must not be shared between concurrent calls. The context of the
// calling thread's current device is created on first use and destroyed when
// the thread exits.
struct ThreadContexts {
  std::map<int, ctsm_ctx*> by_device;
  ~ThreadContexts() {
    for (auto& kv : by_device) ctsm_destroy(kv.second);
  }
};

ctsm_ctx* ctx() {
  thread_local ThreadContexts tc;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error("CUDA error: no usable CUDA device (ctsm-b200 has no CPU fallback)");
  }
  auto it = tc.by_device.find(dev);
  if (it != tc.by_device.end()) return it->second;
  ctsm_ctx* c = nullptr;
  check(ctsm_create(dev, &c));
  tc.by_device[dev] = c;
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
  DevCsr() : rs(0), col(0), val(0) {}
};

std::string meta_text(const ScanGeometry& g, MatrixMode mode, int k) {  // projector.cpp:191-199
  std::ostringstream meta;
  meta << "mode=" << matrix_mode_name(mode, k) << "\n";
  meta << "s=" << g.s << "\nd=" << g.d << "\ndy=" << g.d_y << "\ndz=" << g.d_z
       << "\nndy=" << g.n_det_y << "\nndz=" << g.n_det_z << "\nnp=" << g.n_angles
       << "\nangle_start=" << g.angle_start << "\nangle_end=" << g.angle_end << "\na=" << g.a
       << "\nb=" << g.b << "\nc=" << g.c << "\nnx=" << g.n_x << "\nny=" << g.n_y
       << "\nnz=" << g.n_z << "\n";
  return meta.str();
}

// build_system_matrix on the device: row offsets in rs, entries in col / val
// (which may hold more than nnz entries); returns nnz.
std::uint64_t build_on_device(const ScanGeometry& g, const ctsm_geometry& c, MatrixMode mode, int k,
                              std::uint64_t memory_budget_bytes, DevBuf<std::uint64_t>& rs,
                              DevBuf<std::uint32_t>& col, DevBuf<double>& val) {
  const std::uint64_t n_rows = g.n_measurements();
  std::uint64_t nnz = 0;
  if (mode == MatrixMode::consistent) {
    // single evaluation: arrays sized from the angle-0 estimate
    std::uint64_t nnz0 = 0;
    check(ctsm_csr_angle_nnz(ctx(), &c, 0, &nnz0, nullptr));
    std::uint64_t cap = (std::uint64_t)((double)nnz0 * g.n_angles * 1.2) + 65536;
    if (12 * nnz0 * (std::uint64_t)g.n_angles + 8 * (n_rows + 1) > memory_budget_bytes) cap = 0;
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
  return nnz;
}
}  // namespace

SparseSystemMatrix build_system_matrix(const ScanGeometry& g, MatrixMode mode, int k, int threads,
                                       std::uint64_t memory_budget_bytes) {
  (void)threads;
  const ctsm_geometry c = to_c(g);
  check(ctsm_validate_geometry(&c));
  SparseSystemMatrix w;
  w.n_rows = g.n_measurements();
  w.n_cols = g.n_voxels();
  DevBuf<std::uint64_t> rs(w.n_rows + 1);
  DevBuf<std::uint32_t> col(0);
  DevBuf<double> val(0);
  const std::uint64_t nnz = build_on_device(g, c, mode, k, memory_budget_bytes, rs, col, val);
  w.row_start.resize(w.n_rows + 1);
  w.col.resize(nnz);
  w.val.resize(nnz);
  d2h(w.row_start.data(), rs.p, w.n_rows + 1);
  d2h(w.col.data(), col.p, nnz);
  d2h(w.val.data(), val.p, nnz);
  w.meta = meta_text(g, mode, k);
  return w;
}


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


// ---- weights (weights2d.hpp:31-32, weights3d.hpp:90-91) --------------------
namespace {
constexpr int kWeightSlab = 256;  // weights per query the batch call provides for

struct WeightBatch {
  std::vector<int> count, my, mz;
  std::vector<double> w;
};

WeightBatch weights_batch(const std::vector<VoxelIndex>& n, const std::vector<double>& phi,
                          const ScanGeometry& g) {
  if (n.size() != phi.size())
    throw Error(ErrorCode::DimensionMismatch, "one angle per voxel index is required");
  g.validate();
  const ctsm_geometry c = to_c(g);
  const size_t nq = n.size();
  std::vector<int> ix(nq), iy(nq), iz(nq);
  for (size_t q = 0; q < nq; ++q) {
    ix[q] = n[q].ix;
    iy[q] = n[q].iy;
    iz[q] = n[q].iz;
  }
  WeightBatch out;
  out.count.resize(nq);
  out.my.resize(nq * kWeightSlab);
  out.mz.resize(nq * kWeightSlab);
  out.w.resize(nq * kWeightSlab);
  check(ctsm_weights_batch(ctx(), &c, nq, ix.data(), iy.data(), iz.data(), phi.data(), kWeightSlab,
                           out.count.data(), out.my.data(), out.mz.data(), out.w.data()));
  return out;
}
}  // namespace

std::vector<std::vector<CellWeight>> pixel_area_factors(const std::vector<VoxelIndex>& n,
                                                        const std::vector<double>& phi,
                                                        const ScanGeometry& g) {
  const WeightBatch b = weights_batch(n, phi, g);
  std::vector<std::vector<CellWeight>> out(n.size());
  for (size_t q = 0; q < n.size(); ++q)
    for (int i = 0; i < b.count[q]; ++i)
      out[q].push_back({b.my[q * kWeightSlab + i], b.w[q * kWeightSlab + i]});
  return out;
}

std::vector<std::vector<VoxelWeight>> voxel_volume_factors(const std::vector<VoxelIndex>& n,
                                                           const std::vector<double>& phi,
                                                           const ScanGeometry& g) {
  if (g.is_2d()) throw Error(ErrorCode::InvalidSpec, "voxel_volume_factors needs a 3D scan");
  const WeightBatch b = weights_batch(n, phi, g);
  std::vector<std::vector<VoxelWeight>> out(n.size());
  for (size_t q = 0; q < n.size(); ++q)
    for (int i = 0; i < b.count[q]; ++i)
      out[q].push_back({b.my[q * kWeightSlab + i], b.mz[q * kWeightSlab + i],
                        b.w[q * kWeightSlab + i]});
  return out;
}

std::vector<CellWeight> pixel_area_factors(const VoxelIndex& n, double phi, const ScanGeometry& g) {
  return pixel_area_factors(std::vector<VoxelIndex>{n}, std::vector<double>{phi}, g)[0];
}

std::vector<VoxelWeight> voxel_volume_factors(const VoxelIndex& n, double phi,
                                              const ScanGeometry& g) {
  return voxel_volume_factors(std::vector<VoxelIndex>{n}, std::vector<double>{phi}, g)[0];
}

namespace detail {
void angle_block_entries(const ScanGeometry& g, MatrixMode mode, int k, int angle_index,
                         const std::function<void(std::uint32_t, std::uint32_t, double)>& emit) {
  g.validate();
  if (angle_index < 0 || angle_index >= g.n_angles)
    throw Error(ErrorCode::InvalidSpec, "angle index out of range");
  const ctsm_geometry c = to_c(g);
  std::uint64_t cap = 0;
  if (mode == MatrixMode::consistent)
    check(ctsm_csr_angle_nnz(ctx(), &c, angle_index, &cap, nullptr));
  std::uint64_t n = 0;
  DevBuf<std::uint32_t> raster(0), col(0);
  DevBuf<double> w(0);
  for (int attempt = 0; attempt < 2; ++attempt) {
    raster.reset(cap);
    col.reset(cap);
    w.reset(cap);
    check(ctsm_angle_block_entries(ctx(), &c, mode_code(mode), k, angle_index, cap, raster.p,
                                   col.p, w.p, &n, nullptr));
    if (n <= cap) break;
    cap = n;
  }
  std::vector<std::uint32_t> hr(n), hc(n);
  std::vector<double> hw(n);
  d2h(hr.data(), raster.p, n);
  d2h(hc.data(), col.p, n);
  d2h(hw.data(), w.p, n);
  for (std::uint64_t i = 0; i < n; ++i) emit(hr[i], hc[i], hw[i]);
}
}  // namespace detail

// ---- fp32 operands -----------------------------------------------------------
std::vector<float> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                               const std::vector<float>& x, int threads) {
  (void)threads;
  g.validate();
  if (x.size() != g.n_voxels())
    throw Error(ErrorCode::DimensionMismatch, "image size does not match the grid");
  const ctsm_geometry c = to_c(g);
  std::vector<float> y(g.n_measurements());
  if (mode == MatrixMode::consistent) {
    check(ctsm_forward_project_matrix_free_host_f32(ctx(), &c, x.data(), y.data()));
    return y;
  }
  DevBuf<float> xd(x.size()), yd(y.size());
  h2d(xd.p, x.data(), x.size());
  check(ctsm_fwd_mf_mode(ctx(), &c, mode_code(mode), k, CTSM_F32, 0, g.n_angles, 1, xd.p, yd.p,
                         nullptr));
  d2h(y.data(), yd.p, y.size());
  return y;
}

std::vector<float> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                            const std::vector<float>& y, int threads) {
  (void)threads;
  g.validate();
  if (y.size() != g.n_measurements())
    throw Error(ErrorCode::DimensionMismatch, "sinogram size does not match the scan");
  const ctsm_geometry c = to_c(g);
  std::vector<float> x(g.n_voxels());
  if (mode == MatrixMode::consistent) {
    check(ctsm_back_project_matrix_free_host_f32(ctx(), &c, y.data(), x.data()));
    return x;
  }
  DevBuf<float> yd(y.size()), xd(x.size());
  h2d(yd.p, y.data(), y.size());
  check(ctsm_bwd_mf_mode(ctx(), &c, mode_code(mode), k, CTSM_F32, 0, g.n_angles, 1, yd.p, xd.p,
                         nullptr));
  d2h(x.data(), xd.p, x.size());
  return x;
}

std::vector<float> sirt(const ScanGeometry& g, const std::vector<float>& y,
                        const std::vector<float>& x0, int iters) {
  g.validate();
  if (y.size() != g.n_measurements() || x0.size() != g.n_voxels())
    throw Error(ErrorCode::DimensionMismatch, "operand sizes do not match the scan");
  const ctsm_geometry c = to_c(g);
  DevBuf<float> yd(y.size()), xd(x0.size());
  h2d(yd.p, y.data(), y.size());
  h2d(xd.p, x0.data(), x0.size());
  check(ctsm_sirt(ctx(), &c, CTSM_F32, yd.p, xd.p, iters, nullptr));
  std::vector<float> x(x0.size());
  d2h(x.data(), xd.p, x.size());
  return x;
}

// ---- device-resident matrix ---------------------------------------------------
struct DeviceSystemMatrix::Impl {
  int device = 0;
  std::uint64_t n_rows = 0, n_cols = 0, nnz = 0;
  std::string meta;
  DevBuf<std::uint64_t> rs{0};
  DevBuf<std::uint32_t> col{0};
  DevBuf<double> val{0};
  // CSC transpose (build_transpose) and the column-sum bound of K4
  bool csc = false;
  double colsum_max = 0.0;
  DevBuf<std::uint64_t> cs{0};
  DevBuf<std::uint32_t> trow{0};
  DevBuf<double> tval{0};
  ctsm_operator op() const {
    ctsm_operator o{};
    o.kind = CTSM_OP_CSR;
    o.n_rows = n_rows;
    o.n_cols = n_cols;
    o.row_start = rs.p;
    o.col = col.p;
    o.val = val.p;
    o.scale = 1.0;
    if (csc) {
      o.col_start = cs.p;
      o.trow = trow.p;
      o.tval = tval.p;
    }
    return o;
  }
};

DeviceSystemMatrix::DeviceSystemMatrix(const SparseSystemMatrix& w) : impl_(new Impl) {
  if (w.row_start.size() != w.n_rows + 1)
    throw Error(ErrorCode::DimensionMismatch, "row offsets do not match the row count");
  ctx();
  cudaGetDevice(&impl_->device);
  impl_->n_rows = w.n_rows;
  impl_->n_cols = w.n_cols;
  impl_->nnz = w.nnz();
  impl_->meta = w.meta;
  impl_->rs.reset(w.row_start.size());
  impl_->col.reset(w.col.size());
  impl_->val.reset(w.val.size());
  h2d(impl_->rs.p, w.row_start.data(), w.row_start.size());
  h2d(impl_->col.p, w.col.data(), w.col.size());
  h2d(impl_->val.p, w.val.data(), w.val.size());
}

DeviceSystemMatrix::DeviceSystemMatrix(const ScanGeometry& g, MatrixMode mode, int k,
                                       std::uint64_t memory_budget_bytes)
    : impl_(new Impl) {
  const ctsm_geometry c = to_c(g);
  check(ctsm_validate_geometry(&c));
  ctx();
  cudaGetDevice(&impl_->device);
  impl_->n_rows = g.n_measurements();
  impl_->n_cols = g.n_voxels();
  impl_->rs.reset(impl_->n_rows + 1);
  impl_->nnz = build_on_device(g, c, mode, k, memory_budget_bytes, impl_->rs, impl_->col,
                               impl_->val);
  impl_->meta = meta_text(g, mode, k);
}

DeviceSystemMatrix::~DeviceSystemMatrix() = default;
std::uint64_t DeviceSystemMatrix::n_rows() const { return impl_->n_rows; }
std::uint64_t DeviceSystemMatrix::n_cols() const { return impl_->n_cols; }
std::uint64_t DeviceSystemMatrix::nnz() const { return impl_->nnz; }
const std::string& DeviceSystemMatrix::meta() const { return impl_->meta; }

SparseSystemMatrix DeviceSystemMatrix::download() const {
  SparseSystemMatrix w;
  w.n_rows = impl_->n_rows;
  w.n_cols = impl_->n_cols;
  w.meta = impl_->meta;
  w.row_start.resize(impl_->n_rows + 1);
  w.col.resize(impl_->nnz);
  w.val.resize(impl_->nnz);
  d2h(w.row_start.data(), impl_->rs.p, w.row_start.size());
  d2h(w.col.data(), impl_->col.p, w.col.size());
  d2h(w.val.data(), impl_->val.p, w.val.size());
  return w;
}

void DeviceSystemMatrix::scale_values(double factor) {
  if (!std::isfinite(factor)) throw Error(ErrorCode::NonFinite, "scale factor must be finite");
  check(ctsm_scale_values(ctx(), impl_->nnz, impl_->val.p, factor, nullptr));
  impl_->csc = false;  // the transpose held the old values
  impl_->cs.reset(0);
  impl_->trow.reset(0);
  impl_->tval.reset(0);
}

void DeviceSystemMatrix::build_transpose() {
  Impl& m = *impl_;
  m.cs.reset(m.n_cols + 1);
  m.trow.reset(m.nnz);
  m.tval.reset(m.nnz);
  check(ctsm_csc_build(ctx(), m.n_rows, m.n_cols, m.rs.p, m.col.p, m.val.p, m.cs.p, m.trow.p,
                       m.tval.p, nullptr));
  check(ctsm_csr_colsum_max(ctx(), m.n_rows, m.n_cols, m.rs.p, m.col.p, m.val.p, &m.colsum_max,
                            nullptr));
  m.csc = true;
}

bool DeviceSystemMatrix::has_transpose() const { return impl_->csc; }

std::vector<double> forward_project(const DeviceSystemMatrix& w, const std::vector<double>& x) {
  const auto& m = w.impl();
  if (x.size() != m.n_cols)
    throw Error(ErrorCode::DimensionMismatch, "image size does not match matrix columns");
  DevBuf<double> xd(x.size()), yd(m.n_rows);
  h2d(xd.p, x.data(), x.size());
  check(ctsm_spmv(ctx(), m.n_rows, m.n_cols, m.rs.p, m.col.p, m.val.p, xd.p, yd.p, nullptr));
  std::vector<double> y(m.n_rows);
  d2h(y.data(), yd.p, y.size());
  return y;
}

std::vector<double> back_project(const DeviceSystemMatrix& w, const std::vector<double>& y) {
  const auto& m = w.impl();
  if (y.size() != m.n_rows)
    throw Error(ErrorCode::DimensionMismatch, "sinogram size does not match matrix rows");
  DevBuf<double> yd(y.size()), xd(m.n_cols);
  h2d(yd.p, y.data(), y.size());
  if (m.csc)
    check(ctsm_spmv_t_csc(ctx(), m.n_rows, m.n_cols, m.cs.p, m.trow.p, m.tval.p, m.colsum_max,
                          yd.p, xd.p, nullptr));
  else
    check(ctsm_spmv_t(ctx(), m.n_rows, m.n_cols, m.rs.p, m.col.p, m.val.p, yd.p, xd.p, nullptr));
  std::vector<double> x(m.n_cols);
  d2h(x.data(), xd.p, x.size());
  return x;
}

double spectral_norm_power(const DeviceSystemMatrix& w, int iters, std::uint64_t seed) {
  const auto& m = w.impl();
  if (m.nnz == 0) throw Error(ErrorCode::ZeroMatrix, "matrix has no entries");
  const std::vector<double> v = normal_samples(m.n_cols, seed);
  DevBuf<double> vd(m.n_cols);
  h2d(vd.p, v.data(), v.size());
  const ctsm_operator op = m.op();
  double out = 0.0;
  check(ctsm_spectral_norm_power(ctx(), &op, iters, vd.p, &out, nullptr));
  return out;
}

SolveResult nag_tikhonov(const DeviceSystemMatrix& w, const std::vector<double>& p,
                         const SolveOptions& opt, bool keep_trace) {
  const auto& m = w.impl();
  if (p.size() != m.n_rows)
    throw Error(ErrorCode::DimensionMismatch, "data size does not match matrix rows");
  if (!(opt.lambda >= 0.0) || !(opt.tol >= 0.0) || opt.max_iter < 0)
    throw Error(ErrorCode::InvalidConfig, "solver options must be nonnegative");
  SolveResult res;
  res.u.assign(m.n_cols, 0.0);
  if (m.nnz == 0) throw Error(ErrorCode::ZeroMatrix, "matrix has no entries");
  DevBuf<double> pd(m.n_rows), ud(m.n_cols);
  h2d(pd.p, p.data(), p.size());
  const ctsm_operator op = m.op();
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

// ---- independent numerical oracles (oracle.hpp:24-45) -------------------------
std::vector<McEstimate> mc_volume_3d(const std::vector<double>& boxes,
                                     const std::vector<double>& phi, double s, double d,
                                     double d_y, double d_z, const std::vector<int>& m_y,
                                     const std::vector<int>& m_z, std::uint64_t n_samples,
                                     std::uint64_t seed) {
  const size_t n = phi.size();
  if (boxes.size() != 6 * n || m_y.size() != n || m_z.size() != n)
    throw Error(ErrorCode::DimensionMismatch, "one box, angle and cell per case is required");
  std::vector<double> v(n), se(n);
  check(ctsm_mc_volume_3d(ctx(), n, boxes.data(), phi.data(), s, d, d_y, d_z, m_y.data(),
                          m_z.data(), n_samples, seed, v.data(), se.data(), nullptr));
  std::vector<McEstimate> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = {v[i], se[i]};
  return out;
}

std::vector<double> multiline_volume_3d(const std::vector<double>& boxes,
                                        const std::vector<double>& phi, double s, double d,
                                        double d_y, double d_z, const std::vector<int>& m_y,
                                        const std::vector<int>& m_z, int k) {
  const size_t n = phi.size();
  if (boxes.size() != 6 * n || m_y.size() != n || m_z.size() != n)
    throw Error(ErrorCode::DimensionMismatch, "one box, angle and cell per case is required");
  std::vector<double> out(n);
  check(ctsm_multiline_volume_3d(ctx(), n, boxes.data(), phi.data(), s, d, d_y, d_z, m_y.data(),
                                 m_z.data(), k, out.data()));
  return out;
}

McEstimate mc_volume_3d(double x0, double x1, double y0, double y1, double zb, double zt,
                        double phi, double s, double d, double d_y, double d_z, int m_y, int m_z,
                        std::uint64_t n_samples, std::uint64_t seed) {
  return mc_volume_3d(std::vector<double>{x0, x1, y0, y1, zb, zt}, std::vector<double>{phi}, s, d,
                      d_y, d_z, std::vector<int>{m_y}, std::vector<int>{m_z}, n_samples, seed)[0];
}

double multiline_volume_3d(double x0, double x1, double y0, double y1, double zb, double zt,
                           double phi, double s, double d, double d_y, double d_z, int m_y,
                           int m_z, int k) {
  return multiline_volume_3d(std::vector<double>{x0, x1, y0, y1, zb, zt}, std::vector<double>{phi},
                             s, d, d_y, d_z, std::vector<int>{m_y}, std::vector<int>{m_z}, k)[0];
}

std::pair<std::vector<double>, std::vector<double>> gauss_legendre(int k) {
  if (k <= 0) throw Error(ErrorCode::InvalidSpec, "k must be > 0");
  std::vector<double> x((size_t)k), w((size_t)k);
  ctsm_gauss_legendre(k, x.data(), w.data());
  return {x, w};
}

// ---- multi-GPU variants -----------------------------------------------------
namespace {
struct Multi {
  ctsm_multi* m = nullptr;
  explicit Multi(const std::vector<int>& devices) {
    check(ctsm_multi_create(devices.data(), (int)devices.size(), &m));
  }
  ~Multi() { ctsm_multi_destroy(m); }
};

void need_consistent(MatrixMode mode) {
  if (mode != MatrixMode::consistent)
    throw Error(ErrorCode::InvalidSpec, "the multi-GPU projectors implement the consistent mode");
}

template <typename T>
std::vector<T> multi_fwd(const ScanGeometry& g, MatrixMode mode, const std::vector<T>& x,
                         const std::vector<int>& devices, int dtype) {
  need_consistent(mode);
  g.validate();
  if (x.size() != g.n_voxels())
    throw Error(ErrorCode::DimensionMismatch, "image size does not match the grid");
  const ctsm_geometry c = to_c(g);
  Multi mm(devices);
  std::vector<T> y(g.n_measurements());
  check(ctsm_multi_forward_project_matrix_free_host(mm.m, &c, dtype, x.data(), y.data()));
  return y;
}

template <typename T>
std::vector<T> multi_bwd(const ScanGeometry& g, MatrixMode mode, const std::vector<T>& y,
                         const std::vector<int>& devices, int dtype) {
  need_consistent(mode);
  g.validate();
  if (y.size() != g.n_measurements())
    throw Error(ErrorCode::DimensionMismatch, "sinogram size does not match the scan");
  const ctsm_geometry c = to_c(g);
  Multi mm(devices);
  std::vector<T> x(g.n_voxels());
  check(ctsm_multi_back_project_matrix_free_host(mm.m, &c, dtype, y.data(), x.data()));
  return x;
}

template <typename T>
std::vector<T> multi_sirt(const ScanGeometry& g, const std::vector<T>& y, const std::vector<T>& x0,
                          int iters, const std::vector<int>& devices, int dtype) {
  g.validate();
  if (y.size() != g.n_measurements() || x0.size() != g.n_voxels())
    throw Error(ErrorCode::DimensionMismatch, "operand sizes do not match the scan");
  const ctsm_geometry c = to_c(g);
  Multi mm(devices);
  std::vector<T> x = x0;
  check(ctsm_multi_sirt_host(mm.m, &c, dtype, y.data(), x.data(), iters));
  return x;
}
}  // namespace

std::vector<double> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                                const std::vector<double>& x,
                                                const std::vector<int>& devices) {
  (void)k;
  return multi_fwd<double>(g, mode, x, devices, CTSM_F64);
}
std::vector<double> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                             const std::vector<double>& y,
                                             const std::vector<int>& devices) {
  (void)k;
  return multi_bwd<double>(g, mode, y, devices, CTSM_F64);
}
std::vector<float> forward_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                               const std::vector<float>& x,
                                               const std::vector<int>& devices) {
  (void)k;
  return multi_fwd<float>(g, mode, x, devices, CTSM_F32);
}
std::vector<float> back_project_matrix_free(const ScanGeometry& g, MatrixMode mode, int k,
                                            const std::vector<float>& y,
                                            const std::vector<int>& devices) {
  (void)k;
  return multi_bwd<float>(g, mode, y, devices, CTSM_F32);
}
std::vector<double> sirt(const ScanGeometry& g, const std::vector<double>& y,
                         const std::vector<double>& x0, int iters,
                         const std::vector<int>& devices) {
  return multi_sirt<double>(g, y, x0, iters, devices, CTSM_F64);
}
std::vector<float> sirt(const ScanGeometry& g, const std::vector<float>& y,
                        const std::vector<float>& x0, int iters, const std::vector<int>& devices) {
  return multi_sirt<float>(g, y, x0, iters, devices, CTSM_F32);
}

}  // namespace ctsm

extern "C" void ctsm_normal_samples(uint64_t n, uint64_t seed, double* out) {
  const std::vector<double> v = ctsm::normal_samples((std::size_t)n, seed);
  std::copy(v.begin(), v.end(), out);
}
