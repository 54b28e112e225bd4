// C++ drop-in check: the reference's projector-level contracts
// (test_projector.cpp:42-155 ideas) exercised through include/ctsm_b200/ctsm.hpp.
// Built and run by tests/test_gpu_cpp_api.py on a GPU box.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>

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
  // ---- the reference's weight API (weights2d.hpp:31-32, weights3d.hpp:90-91,
  // projector.hpp:72-78) against the unmodified reference compiled with the
  // correctly rounded libm (oracle/_ref/libctsm_ref_cr.so, test infrastructure;
  // its path comes from CTSM_TEST_ORACLE_LIB): same entries, same order, same bits
  {
    struct RefGeom {  // == ctsm_geometry
      double s, d, d_y, d_z;
      int32_t n_det_y, n_det_z, n_angles, pad0;
      double angle_start, angle_end, a, b, c;
      int32_t n_x, n_y, n_z, pad1;
    };
    auto to_ref = [](const ScanGeometry& g) {
      RefGeom r{};
      r.s = g.s; r.d = g.d; r.d_y = g.d_y; r.d_z = g.d_z;
      r.n_det_y = g.n_det_y; r.n_det_z = g.n_det_z; r.n_angles = g.n_angles;
      r.angle_start = g.angle_start; r.angle_end = g.angle_end;
      r.a = g.a; r.b = g.b; r.c = g.c; r.n_x = g.n_x; r.n_y = g.n_y; r.n_z = g.n_z;
      return r;
    };
    const char* lib = std::getenv("CTSM_TEST_ORACLE_LIB");
    void* h = lib ? dlopen(lib, RTLD_NOW) : nullptr;
    using paf_t = long (*)(const RefGeom*, int, int, double, int32_t*, double*, long);
    using vvf_t = long (*)(const RefGeom*, int, int, int, double, int32_t*, int32_t*, double*, long);
    using abe_t = long (*)(const RefGeom*, int, uint32_t*, uint32_t*, double*, long);
    paf_t ref_paf = h ? (paf_t)dlsym(h, "ref_pixel_area_factors") : nullptr;
    vvf_t ref_vvf = h ? (vvf_t)dlsym(h, "ref_voxel_volume_factors") : nullptr;
    abe_t ref_abe = h ? (abe_t)dlsym(h, "ref_angle_block_entries") : nullptr;
    if (lib) EXPECT(ref_paf && ref_vvf && ref_abe);
    for (bool three_d : {false, true}) {
      const ScanGeometry g = small_scan(three_d);
      const RefGeom rg = to_ref(g);
      // every voxel of the two central slices (whose shadows the small detector
      // covers fully) at a scan angle and at an off-grid angle
      std::vector<VoxelIndex> idx;
      std::vector<double> phi;
      for (int iz : {g.n_z / 2 - 1, g.n_z / 2})
        for (int iy = 0; iy < g.n_y; ++iy)
          for (int ix = 0; ix < g.n_x; ++ix) {
            idx.push_back({ix, iy, three_d ? iz : 0});
            phi.push_back(idx.size() % 2 ? g.angle(1) : 0.777);
          }
      if (!three_d) {
        const auto all = pixel_area_factors(idx, phi, g);
        for (std::size_t q = 0; q < idx.size(); ++q) {
          double sum = 0;
          for (const CellWeight& cw : all[q]) sum += cw.w;
          EXPECT(std::abs(sum - 1.0) <= 1e-10);  // partition (test_weights2d.cpp:51-78)
          if (ref_paf) {
            int32_t my[64];
            double w[64];
            const long n = ref_paf(&rg, idx[q].ix, idx[q].iy, phi[q], my, w, 64);
            EXPECT(n == (long)all[q].size());
            for (long i = 0; i < n && i < (long)all[q].size(); ++i)
              EXPECT(my[i] == all[q][i].m_y && std::memcmp(&w[i], &all[q][i].w, 8) == 0);
          }
        }
        const auto one = pixel_area_factors(idx[5], phi[5], g);
        EXPECT(one.size() == all[5].size());
      } else {
        const auto all = voxel_volume_factors(idx, phi, g);
        for (std::size_t q = 0; q < idx.size(); ++q) {
          double sum = 0;
          for (const VoxelWeight& vw : all[q]) sum += vw.w;
          EXPECT(std::abs(sum - 1.0) <= 1e-9);  // partition (test_weights3d.cpp:59-74)
          if (ref_vvf) {
            int32_t my[256], mz[256];
            double w[256];
            const long n = ref_vvf(&rg, idx[q].ix, idx[q].iy, idx[q].iz, phi[q], my, mz, w, 256);
            EXPECT(n == (long)all[q].size());
            for (long i = 0; i < n && i < (long)all[q].size(); ++i)
              EXPECT(my[i] == all[q][i].m_y && mz[i] == all[q][i].m_z &&
                     std::memcmp(&w[i], &all[q][i].w, 8) == 0);
          }
        }
        EXPECT(code_of([&] { voxel_volume_factors(idx[0], 0.1, small_scan(false)); }) ==
               (int)ErrorCode::InvalidSpec);
      }
      // angle_block_entries: the emission stream rebuilds A x of that angle
      // (projector.cpp:235-252) and equals the reference's stream
      const int ip = 2;
      std::vector<std::uint32_t> er, ec;
      std::vector<double> ew;
      detail::angle_block_entries(g, MatrixMode::consistent, 1, ip,
                                  [&](std::uint32_t r, std::uint32_t c, double w) {
                                    er.push_back(r);
                                    ec.push_back(c);
                                    ew.push_back(w);
                                  });
      const auto x = randn(g.n_voxels(), 77);
      std::vector<double> blk((std::size_t)g.n_det_y * g.n_det_z, 0.0);
      for (std::size_t i = 0; i < er.size(); ++i) blk[er[i]] += ew[i] * x[ec[i]];
      const auto yfull = forward_project_matrix_free(g, MatrixMode::consistent, 1, x);
      double md = 0;
      for (std::size_t i = 0; i < blk.size(); ++i)
        md = std::max(md, std::abs(blk[i] - yfull[(std::size_t)ip * blk.size() + i]));
      EXPECT(md <= 1e-10);
      if (ref_abe) {
        const long n = ref_abe(&rg, ip, nullptr, nullptr, nullptr, 0);
        EXPECT(n == (long)er.size());
        std::vector<std::uint32_t> rr(n), rc(n);
        std::vector<double> rw(n);
        ref_abe(&rg, ip, rr.data(), rc.data(), rw.data(), n);
        EXPECT(rr == er && rc == ec);
        EXPECT(n == (long)ew.size() && std::memcmp(rw.data(), ew.data(), 8 * (std::size_t)n) == 0);
      }
      // line mode streams row by row
      std::uint64_t nline = 0;
      std::uint32_t last_row = 0;
      bool ordered = true;
      detail::angle_block_entries(g, MatrixMode::line, 1, ip,
                                  [&](std::uint32_t r, std::uint32_t, double) {
                                    if (r < last_row) ordered = false;
                                    last_row = r;
                                    ++nline;
                                  });
      EXPECT(nline > 0 && ordered);
    }
  }
  // ---- device-resident matrix: uploaded / built once, applied many times ----
  {
    const ScanGeometry g = small_scan(true);
    const SparseSystemMatrix w = build_system_matrix(g, MatrixMode::consistent);
    DeviceSystemMatrix dm(w);
    DeviceSystemMatrix db(g, MatrixMode::consistent);
    EXPECT(db.nnz() == w.nnz() && dm.nnz() == w.nnz() && db.n_rows() == w.n_rows);
    const SparseSystemMatrix back = db.download();
    EXPECT(back.row_start == w.row_start && back.col == w.col && back.val == w.val &&
           back.meta == w.meta);
    const auto x = randn(w.n_cols, 5), y = randn(w.n_rows, 6);
    EXPECT(forward_project(dm, x) == forward_project(w, x));
    EXPECT(back_project(db, y) == back_project(w, y));
    // K4 as a gather over the CSC transpose: the same bits as the scatter
    db.build_transpose();
    EXPECT(db.has_transpose());
    EXPECT(back_project(db, y) == back_project(w, y));
    EXPECT(spectral_norm_power(dm, 30, 7) == spectral_norm_power(w, 30, 7));
    const double nrm = spectral_norm_power(dm, 100, 7);
    dm.build_transpose();
    dm.scale_values(1.0 / nrm);
    EXPECT(!dm.has_transpose());  // the transpose held the old values
    EXPECT(std::abs(spectral_norm_power(dm, 100, 7) - 1.0) <= 1e-8);
    SolveOptions opt;
    opt.lambda = 1e-2;
    opt.max_iter = 50;
    const auto p = forward_project(dm, std::vector<double>(w.n_cols, 0.01));
    SparseSystemMatrix ws = w;
    scale_values(&ws, 1.0 / nrm);
    EXPECT(nag_tikhonov(dm, p, opt).u == nag_tikhonov(ws, p, opt).u);
  }
  // ---- fp32 operands and the device-list variants (one device here) ---------
  {
    const ScanGeometry g = small_scan(true);
    const auto xd = randn(g.n_voxels(), 9), yd = randn(g.n_measurements(), 10);
    std::vector<float> xf(xd.begin(), xd.end()), yf(yd.begin(), yd.end());
    const auto y64 = forward_project_matrix_free(g, MatrixMode::consistent, 1, xd);
    const auto y32 = forward_project_matrix_free(g, MatrixMode::consistent, 1, xf);
    const auto x64 = back_project_matrix_free(g, MatrixMode::consistent, 1, yd);
    const auto x32 = back_project_matrix_free(g, MatrixMode::consistent, 1, yf);
    double my = 0, mx = 0, sy = 0, sx = 0;
    for (std::size_t i = 0; i < y64.size(); ++i) {
      my = std::max(my, std::abs(y64[i] - y32[i]));
      sy = std::max(sy, std::abs(y64[i]));
    }
    for (std::size_t i = 0; i < x64.size(); ++i) {
      mx = std::max(mx, std::abs(x64[i] - x32[i]));
      sx = std::max(sx, std::abs(x64[i]));
    }
    EXPECT(my <= 1e-5 * std::max(1.0, sy) && mx <= 1e-5 * std::max(1.0, sx));
    const std::vector<int> devs{0};
    EXPECT(forward_project_matrix_free(g, MatrixMode::consistent, 1, xd, devs) == y64);
    EXPECT(back_project_matrix_free(g, MatrixMode::consistent, 1, yd, devs) == x64);
    const std::vector<double> z(g.n_voxels(), 0.0);
    const auto s1 = sirt(g, yd, z, 2), sm = sirt(g, yd, z, 2, devs);
    double ms = 0;
    for (std::size_t i = 0; i < s1.size(); ++i) ms = std::max(ms, std::abs(s1[i] - sm[i]));
    EXPECT(ms <= 1e-10);
    EXPECT(code_of([&] { forward_project_matrix_free(g, MatrixMode::consistent, 1, xd,
                                                     std::vector<int>{0, 0}); }) ==
           (int)ErrorCode::InvalidSpec);
  }
  // ---- device MC / Gauss-Legendre oracles (oracle.hpp:24-45) ----------------
  {
    const ScanGeometry g = small_scan(true);
    const VoxelIndex n{4, 7, 6};
    const double phi = 0.7;
    const auto ws = voxel_volume_factors(n, phi, g);
    EXPECT(!ws.empty());
    const VoxelWeight* best = &ws[0];
    for (const auto& vw : ws)
      if (vw.w > best->w) best = &vw;
    const McEstimate mc =
        mc_volume_3d(g.face_x(n.ix), g.face_x(n.ix + 1), g.face_y(n.iy), g.face_y(n.iy + 1),
                     g.face_z(n.iz), g.face_z(n.iz + 1), phi, g.s, g.d, g.d_y, g.d_z, best->m_y,
                     best->m_z, 400000, 99);
    EXPECT(std::abs(best->w - mc.value) < 4 * mc.std_err + 1e-6);  // test_weights3d.cpp:198-212
    const double gl = multiline_volume_3d(g.face_x(n.ix), g.face_x(n.ix + 1), g.face_y(n.iy),
                                          g.face_y(n.iy + 1), g.face_z(n.iz), g.face_z(n.iz + 1),
                                          phi, g.s, g.d, g.d_y, g.d_z, best->m_y, best->m_z, 100);
    EXPECT(std::abs(gl - best->w) < 2e-5);  // k = 100 quadrature of a kinked integrand
    const auto glw = gauss_legendre(16);
    double sw = 0;
    for (double v : glw.second) sw += v;
    EXPECT(std::abs(sw - 2.0) < 1e-13);
  }
  // ---- re-entrancy: concurrent calls from several host threads (each thread
  // gets its own context) give the single-thread result ----------------------
  {
    const ScanGeometry g = small_scan(true);
    const auto x = randn(g.n_voxels(), 3);
    const auto ref = forward_project_matrix_free(g, MatrixMode::consistent, 1, x);
    std::vector<std::vector<double>> out(4);
    std::vector<std::thread> th;
    for (int t = 0; t < 4; ++t)
      th.emplace_back([&, t] {
        for (int r = 0; r < 3; ++r)
          out[t] = forward_project_matrix_free(g, MatrixMode::consistent, 1, x);
      });
    for (auto& t : th) t.join();
    for (int t = 0; t < 4; ++t) EXPECT(out[t] == ref);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
