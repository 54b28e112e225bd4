// C++ drop-in check: the reference's projector-level contracts
// (test_projector.cpp:42-155 ideas) exercised through include/ctsm_b200/ctsm.hpp.
// Built and run by tests/test_gpu_cpp_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <random>

#include "ctsm_b200/ctsm.hpp"

using namespace ctsm;

static int failures = 0;
#define EXPECT(cond)                                              \
  do {                                                            \
    if (!(cond)) {                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                 \
    }                                                             \
  } while (0)

template <typename Fn>
static int code_of(Fn&& fn) {
  try {
    fn();
  } catch (const Error& e) {
    return static_cast<int>(e.code());
  }
  return -1;
}

static ScanGeometry small_scan(bool three_d) {
  ScanGeometry g;
  g.s = 250;
  g.d = 250;
  g.d_y = 1.5;
  g.n_det_y = 44;
  g.n_angles = 6;
  g.a = g.b = 1.5;
  g.n_x = g.n_y = 12;
  if (three_d) {
    g.d_z = 1.5;
    g.n_det_z = 12;
    g.c = 1.5;
    g.n_z = 12;
  }
  g.validate();
  return g;
}

static std::vector<double> randn(std::size_t n, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> d;
  std::vector<double> v(n);
  for (auto& x : v) x = d(rng);
  return v;
}

static double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

int main() {
  int k = 0;
  EXPECT(parse_matrix_mode("consistent", &k) == MatrixMode::consistent);
  EXPECT(parse_matrix_mode("multiline:8", &k) == MatrixMode::multiline && k == 8);
  EXPECT(code_of([&] { parse_matrix_mode("area", &k); }) == (int)ErrorCode::InvalidConfig);

  for (bool three_d : {false, true}) {
    const ScanGeometry g = small_scan(three_d);
    const SparseSystemMatrix w = build_system_matrix(g, MatrixMode::consistent);
    EXPECT(w.n_rows == g.n_measurements());
    EXPECT(w.n_cols == g.n_voxels());
    EXPECT(w.row_start.front() == 0 && w.row_start.back() == w.nnz());
    for (std::uint64_t r = 0; r < w.n_rows; ++r)
      for (std::uint64_t j = w.row_start[r] + 1; j < w.row_start[r + 1]; ++j)
        EXPECT(w.col[j - 1] < w.col[j]);
    EXPECT(w.meta.find("mode=consistent") != std::string::npos);
    // adjoint
    const auto x = randn(w.n_cols, 31), y = randn(w.n_rows, 32);
    const double lhs = dot(forward_project(w, x), y), rhs = dot(x, back_project(w, y));
    EXPECT(std::abs(lhs - rhs) <= 1e-12 * std::abs(lhs));
    // matrix-free == stored matrix
    const auto y0 = forward_project(w, x);
    const auto y1 = forward_project_matrix_free(g, MatrixMode::consistent, 1, x, 2);
    double md = 0, mv = 0;
    for (std::size_t i = 0; i < y0.size(); ++i) {
      md = std::max(md, std::abs(y0[i] - y1[i]));
      mv = std::max(mv, std::abs(y0[i]));
    }
    EXPECT(md <= 1e-10 * std::max(1.0, mv));  // fast path vs exact CSR: fp64 parity bar
    // matrix-free adjoint == stored transpose
    const auto x0 = back_project(w, y);
    const auto x1 = back_project_matrix_free(g, MatrixMode::consistent, 1, y, 2);
    md = 0, mv = 0;
    for (std::size_t i = 0; i < x0.size(); ++i) {
      md = std::max(md, std::abs(x0[i] - x1[i]));
      mv = std::max(mv, std::abs(x0[i]));
    }
    EXPECT(md <= 1e-10 * std::max(1.0, mv));  // fast path vs exact CSR: fp64 parity bar
    EXPECT(code_of([&] { forward_project(w, std::vector<double>(w.n_cols + 1)); }) ==
           (int)ErrorCode::DimensionMismatch);
  }
  // per-angle column sums never exceed one pixel (test_projector.cpp:121-132)
  {
    const ScanGeometry g = small_scan(false);
    const auto sums = angle_column_sums(g, MatrixMode::consistent, 1, 2);
    double mx = 0, mn = 2;
    for (double s : sums) {
      mx = std::max(mx, s);
      mn = std::min(mn, s);
    }
    EXPECT(mx <= 1.0 + 1e-9);
    EXPECT(mn >= 0.99);
  }
  // spectral norm: scaling by 1/norm gives norm 1
  {
    const ScanGeometry g = small_scan(false);
    SparseSystemMatrix w = build_system_matrix(g, MatrixMode::consistent);
    const double nrm = spectral_norm_power(w, 150, 7);
    scale_values(&w, 1.0 / nrm);
    EXPECT(std::abs(spectral_norm_power(w, 150, 7) - 1.0) <= 1e-8);
  }
  // NAG-Tikhonov (solver.cpp:17-75): converges on the normalised matrix and
  // decreases the objective; option validation
  {
    const ScanGeometry g = small_scan(false);
    SparseSystemMatrix w = build_system_matrix(g, MatrixMode::consistent);
    scale_values(&w, 1.0 / spectral_norm_power(w, 100, 7));
    std::vector<double> u0(w.n_cols, 0.01);
    const std::vector<double> p = forward_project(w, u0);
    SolveOptions opt;
    opt.lambda = 1e-2;
    opt.max_iter = 400;
    opt.tol = 1e-8;
    const SolveResult r = nag_tikhonov(w, p, opt, true);
    EXPECT(r.converged && r.iterations < 400 && (int)r.trace.size() == r.iterations);
    EXPECT(r.trace.back().objective < r.trace.front().objective);
    SolveOptions bad;
    bad.lambda = -1.0;
    EXPECT(code_of([&] { nag_tikhonov(w, p, bad); }) == (int)ErrorCode::InvalidConfig);
    // CSM1 round trip (io.cpp:153-227) and CTT1
    write_matrix("/tmp/ctsm_cpp_api_test.csm", w);
    const SparseSystemMatrix r2 = read_matrix("/tmp/ctsm_cpp_api_test.csm");
    EXPECT(r2.row_start == w.row_start && r2.col == w.col && r2.val == w.val &&
           r2.meta == w.meta && r2.n_cols == w.n_cols);
    write_tensor("/tmp/ctsm_cpp_api_test.ctt", {2, 3}, {1, 2, 3, 4, 5, 6});
    std::vector<std::uint64_t> dims;
    const auto t = read_tensor("/tmp/ctsm_cpp_api_test.ctt", &dims);
    EXPECT(dims.size() == 2 && dims[1] == 3 && t.size() == 6 && t[5] == 6.0);
    EXPECT(code_of([&] { read_matrix("/tmp/ctsm_no_such_file.csm"); }) ==
           (int)ErrorCode::IoFailure);
  }
  // memory budget and size limits (test_projector.cpp:144-155)
  {
    const ScanGeometry g = small_scan(true);
    EXPECT(code_of([&] { build_system_matrix(g, MatrixMode::consistent, 1, 1, 1024); }) ==
           (int)ErrorCode::OutOfMemory);
    ScanGeometry huge = small_scan(true);
    huge.n_x = huge.n_y = huge.n_z = 2048;
    huge.a = huge.b = huge.c = 0.01;
    EXPECT(code_of([&] { build_system_matrix(huge, MatrixMode::consistent); }) ==
           (int)ErrorCode::TooLarge);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
