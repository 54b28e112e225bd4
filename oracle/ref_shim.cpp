// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" adapter over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled where they lie by oracle/Makefile)
// so the Python tests and bench.py's reference arm can drive the reference's
// own public API: pixel_area_factors (weights2d.hpp:31), voxel_volume_factors
// (weights3d.hpp:90), detail::angle_block_entries (projector.hpp:76),
// build_system_matrix / forward_project / back_project /
// forward_project_matrix_free (projector.hpp:41-59).
//
// Two restatements the reference lacks are composed here from its own calls,
// exactly as SURVEY.md §8(a) a16 prescribes:
//  * matrix-free A^T y: x[c] += w * y[r] through detail::angle_block_entries,
//    per-angle partial volumes summed in ascending angle order (deterministic
//    for any thread count, like ordered_parallel_for, projector.cpp:114-140);
//  * SIRT: x <- x + C .* A^T (R .* (y - A x)), R = 1/(A 1), C = 1/(A^T 1),
//    zero sums -> 0 (BASELINE.json configs[4]).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "ctsm/baseline.hpp"
#include "ctsm/geometry.hpp"
#include "ctsm/io.hpp"
#include "ctsm/phantoms.hpp"
#include "ctsm/projector.hpp"
#include "ctsm/solver.hpp"
#include "ctsm/weights2d.hpp"
#include "ctsm/weights3d.hpp"

namespace {

struct RefGeom {  // layout == ctsm_geometry in include/ctsm_b200.h
  double s, d, d_y, d_z;
  int32_t n_det_y, n_det_z, n_angles, pad0;
  double angle_start, angle_end;
  double a, b, c;
  int32_t n_x, n_y, n_z, pad1;
};

ctsm::ScanGeometry to_g(const RefGeom* r) {
  ctsm::ScanGeometry g;
  g.s = r->s;
  g.d = r->d;
  g.d_y = r->d_y;
  g.d_z = r->d_z;
  g.n_det_y = r->n_det_y;
  g.n_det_z = r->n_det_z;
  g.n_angles = r->n_angles;
  g.angle_start = r->angle_start;
  g.angle_end = r->angle_end;
  g.a = r->a;
  g.b = r->b;
  g.c = r->c;
  g.n_x = r->n_x;
  g.n_y = r->n_y;
  g.n_z = r->n_z;
  return g;
}

thread_local std::string g_err;

int fail_code(const ctsm::Error& e) {
  g_err = e.what();
  return -(static_cast<int>(e.code()) + 1);
}

#define REF_GUARD(...)                           \
  try {                                          \
    __VA_ARGS__                                  \
  } catch (const ctsm::Error& e) {               \
    return fail_code(e);                         \
  } catch (const std::exception& e) {            \
    g_err = e.what();                            \
    return -100;                                 \
  }

// Runs fn(i) for i in [0,count) on up to `threads` workers, each worker taking
// a contiguous index range; rethrows the first error.
template <typename Fn>
void parallel_range(int count, int threads, Fn fn) {
  threads = std::max(1, std::min(threads, count));
  if (threads == 1) {
    for (int i = 0; i < count; ++i) fn(i);
    return;
  }
  std::vector<std::exception_ptr> errs(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      const int lo = (int)((int64_t)count * t / threads);
      const int hi = (int)((int64_t)count * (t + 1) / threads);
      try {
        for (int i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate(const RefGeom* rg) {
  REF_GUARD(to_g(rg).validate(); return 0;)
}

double ref_angle(const RefGeom* rg, int i) { return to_g(rg).angle(i); }

// pixel_area_factors (weights2d.cpp:105-129). Returns the count (<= cap written).
long ref_pixel_area_factors(const RefGeom* rg, int ix, int iy, double phi, int32_t* my,
                            double* w, long cap) {
  REF_GUARD(const auto ws = ctsm::pixel_area_factors(ctsm::VoxelIndex{ix, iy, 0}, phi,
                                                     to_g(rg));
            for (long i = 0; i < (long)ws.size() && i < cap; ++i) {
              my[i] = ws[i].m_y;
              w[i] = ws[i].w;
            } return (long)ws.size();)
}

// voxel_volume_factors (weights3d.cpp:354-462).
long ref_voxel_volume_factors(const RefGeom* rg, int ix, int iy, int iz, double phi,
                              int32_t* my, int32_t* mz, double* w, long cap) {
  REF_GUARD(const auto ws = ctsm::voxel_volume_factors(ctsm::VoxelIndex{ix, iy, iz}, phi,
                                                       to_g(rg));
            for (long i = 0; i < (long)ws.size() && i < cap; ++i) {
              my[i] = ws[i].m_y;
              mz[i] = ws[i].m_z;
              w[i] = ws[i].w;
            } return (long)ws.size();)
}

// detail::angle_block_entries (projector.cpp:44-84), consistent mode. Entries
// in emission order; returns the total count (only the first cap are stored).
long ref_angle_block_entries(const RefGeom* rg, int ip, uint32_t* row, uint32_t* col,
                             double* w, long cap) {
  REF_GUARD(long n = 0; ctsm::detail::angle_block_entries(
                to_g(rg), ctsm::MatrixMode::consistent, 1, ip,
                [&](uint32_t r, uint32_t c, double v) {
                  if (n < cap) {
                    row[n] = r;
                    col[n] = c;
                    w[n] = v;
                  }
                  ++n;
                });
            return n;)
}

// detail::angle_block_entries (projector.cpp:44-84, consistent mode) with the
// z slabs (2D: pixel rows) spread over `threads` workers: each slab calls the
// reference's public voxel_volume_factors / pixel_area_factors for its voxels
// in the reference's z -> y -> x order with the reference's raster and column
// maps, and the slabs are concatenated in slab order, so the entries (and
// their order) are identical to ref_angle_block_entries. Used by the flip
// tests against the reference as shipped (glibc libm) at BASELINE size.
long ref_angle_block_entries_par(const RefGeom* rg, int ip, uint32_t* row, uint32_t* col,
                                 double* w, long cap, int threads) {
  REF_GUARD(
      const ctsm::ScanGeometry g = to_g(rg); g.validate(); const double phi = g.angle(ip);
      const bool two_d = g.is_2d(); const int n_slab = two_d ? g.n_y : g.n_z;
      struct Ent { uint32_t r, c; double w; };
      std::vector<std::vector<Ent>> slabs(n_slab);
      const auto raster = [&](int m_y, int m_z) {
        return (uint32_t)((m_z + g.n_det_z / 2) * g.n_det_y + (m_y + g.n_det_y / 2));
      };
      parallel_range(n_slab, threads, [&](int sl) {
        auto& out = slabs[sl];
        if (two_d) {
          for (int ix = 0; ix < g.n_x; ++ix) {
            const ctsm::VoxelIndex n{ix, sl, 0};
            const uint32_t c = (uint32_t)ctsm::voxel_column(g, n);
            for (const auto& cw : ctsm::pixel_area_factors(n, phi, g))
              out.push_back({raster(cw.m_y, 0), c, cw.w});
          }
          return;
        }
        for (int iy = 0; iy < g.n_y; ++iy)
          for (int ix = 0; ix < g.n_x; ++ix) {
            const ctsm::VoxelIndex n{ix, iy, sl};
            const uint32_t c = (uint32_t)ctsm::voxel_column(g, n);
            for (const auto& vw : ctsm::voxel_volume_factors(n, phi, g))
              out.push_back({raster(vw.m_y, vw.m_z), c, vw.w});
          }
      });
      long n = 0;
      for (const auto& sv : slabs) for (const Ent& e : sv) {
        if (n < cap) {
          row[n] = e.r;
          col[n] = e.c;
          w[n] = e.w;
        }
        ++n;
      }
      return n;)
}

// build_system_matrix (projector.cpp:144-201) -> opaque handle.
void* ref_build_system_matrix(const RefGeom* rg, int threads, uint64_t budget, int* status) {
  try {
    auto* m = new ctsm::SparseSystemMatrix(
        ctsm::build_system_matrix(to_g(rg), ctsm::MatrixMode::consistent, 1, threads, budget));
    *status = 0;
    return m;
  } catch (const ctsm::Error& e) {
    *status = fail_code(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    *status = -100;
  }
  return nullptr;
}

uint64_t ref_csr_nnz(void* h) { return static_cast<ctsm::SparseSystemMatrix*>(h)->nnz(); }
uint64_t ref_csr_rows(void* h) { return static_cast<ctsm::SparseSystemMatrix*>(h)->n_rows; }

void ref_csr_copy(void* h, uint64_t* row_start, uint32_t* col, double* val) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  std::memcpy(row_start, m->row_start.data(), m->row_start.size() * sizeof(uint64_t));
  std::memcpy(col, m->col.data(), m->col.size() * sizeof(uint32_t));
  std::memcpy(val, m->val.data(), m->val.size() * sizeof(double));
}

void ref_csr_free(void* h) { delete static_cast<ctsm::SparseSystemMatrix*>(h); }

// forward_project / back_project (projector.cpp:203-233).
int ref_forward_project(void* h, const double* x, double* y) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  REF_GUARD(const std::vector<double> xv(x, x + m->n_cols);
            const auto yv = ctsm::forward_project(*m, xv);
            std::copy(yv.begin(), yv.end(), y); return 0;)
}

int ref_back_project(void* h, const double* y, double* x) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  REF_GUARD(const std::vector<double> yv(y, y + m->n_rows);
            const auto xv = ctsm::back_project(*m, yv);
            std::copy(xv.begin(), xv.end(), x); return 0;)
}

// forward_project_matrix_free (projector.cpp:235-260), all angles.
int ref_forward_project_matrix_free(const RefGeom* rg, const double* x, double* y,
                                    int threads) {
  REF_GUARD(const ctsm::ScanGeometry g = to_g(rg);
            const std::vector<double> xv(x, x + g.n_voxels());
            const auto yv = ctsm::forward_project_matrix_free(
                g, ctsm::MatrixMode::consistent, 1, xv, threads);
            std::copy(yv.begin(), yv.end(), y); return 0;)
}

// A x restricted to a list of angles (sampled timing / parity at C3/C4):
// y_sel[k * rows_per_angle + r] = (A x)[angles[k] * rows_per_angle + r].
// Same per-angle accumulation as forward_project_matrix_free (249-252).
int ref_forward_mf_angles(const RefGeom* rg, const int32_t* angles, int n_sel,
                          const double* x, double* y_sel, int threads) {
  REF_GUARD(const ctsm::ScanGeometry g = to_g(rg); g.validate();
            const uint64_t rpa = (uint64_t)g.n_det_y * g.n_det_z;
            parallel_range(n_sel, threads, [&](int k) {
              double* block = y_sel + (uint64_t)k * rpa;
              std::fill(block, block + rpa, 0.0);
              ctsm::detail::angle_block_entries(
                  g, ctsm::MatrixMode::consistent, 1, angles[k],
                  [&](uint32_t r, uint32_t c, double wv) { block[r] += wv * x[c]; });
            });
            return 0;)
}

// Matrix-free A^T y over a list of angles (restatement):
// x = sum over listed angles (in list order) of the per-angle partial volume.
// y is indexed like the full sinogram: y[angles[k] * rows_per_angle + r].
int ref_back_mf_angles(const RefGeom* rg, const int32_t* angles, int n_sel, const double* y,
                       double* x, int threads) {
  REF_GUARD(const ctsm::ScanGeometry g = to_g(rg); g.validate();
            const uint64_t rpa = (uint64_t)g.n_det_y * g.n_det_z;
            const uint64_t nv = g.n_voxels(); std::fill(x, x + nv, 0.0);
            const int chunk = std::max(1, threads);
            std::vector<std::vector<double>> part(chunk);
            for (int k0 = 0; k0 < n_sel; k0 += chunk) {
              const int n = std::min(chunk, n_sel - k0);
              parallel_range(n, threads, [&](int t) {
                auto& p = part[t];
                p.assign(nv, 0.0);
                const double* yb = y + (uint64_t)angles[k0 + t] * rpa;
                ctsm::detail::angle_block_entries(
                    g, ctsm::MatrixMode::consistent, 1, angles[k0 + t],
                    [&](uint32_t r, uint32_t c, double wv) { p[c] += wv * yb[r]; });
              });
              for (int t = 0; t < n; ++t)
                for (uint64_t i = 0; i < nv; ++i) x[i] += part[t][i];
            } return 0;)
}

// Bounded sample of one A x + A^T y step for bench.py's reference arm and
// cpu_baseline. The reference's API cannot bound an angle block, so the work
// items here are (listed angle, listed slab) pairs spread over `threads`
// workers: a slab is one z plane of voxels (3D) or one pixel row (2D). Each
// item walks its voxels in projector.cpp:53-69's order with the reference's
// own voxel_volume_factors / pixel_area_factors (weights3d.hpp:90,
// weights2d.hpp:31) TWICE, as a reference user would for the two products:
// pass 1 is forward_project_matrix_free's accumulation y[r] += w x[c] into the
// item's angle block (projector.cpp:249-252), pass 2 the a16 adjoint
// x_out[c] += w y[r], re-evaluating the weights. Slabs are disjoint, so the
// reference's per-angle parallelism (ordered_parallel_for,
// projector.cpp:114-140) is kept while a few angles still use every core.
// *updates = weights applied (one per weight and direction).
int ref_mf_pair_sample(const RefGeom* rg, const int32_t* angles, int n_sel,
                       const int32_t* slabs, int n_slabs, const double* x, const double* y,
                       double* checksum, uint64_t* updates, int threads) {
  REF_GUARD(
      const ctsm::ScanGeometry g = to_g(rg); g.validate();
      const bool two_d = g.is_2d();
      const uint64_t rpa = (uint64_t)g.n_det_y * g.n_det_z;
      const int items = n_sel * n_slabs;
      std::vector<double> sums(items, 0.0);
      std::vector<uint64_t> counts(items, 0);
      const auto raster = [&](int m_y, int m_z) {
        return (uint32_t)((m_z + g.n_det_z / 2) * g.n_det_y + (m_y + g.n_det_y / 2));
      };
      parallel_range(items, threads, [&](int it) {
        const int k = it % n_sel, sl = slabs[it / n_sel];  // angles interleaved over workers
        const double phi = g.angle(angles[k]);
        const double* yb = y + (uint64_t)angles[k] * rpa;
        const uint64_t plane = two_d ? (uint64_t)g.n_x : (uint64_t)g.n_x * g.n_y;
        const uint64_t base = (uint64_t)sl * plane;
        std::vector<double> block(rpa, 0.0);   // the angle's sinogram block (pass 1)
        std::vector<double> xp(plane, 0.0);    // the angle's partial volume slab (pass 2)
        uint64_t n = 0;
        for (int pass = 0; pass < 2; ++pass) {
          const auto apply = [&](uint32_t r, uint32_t c, double w) {
            if (pass == 0) block[r] += w * x[c]; else xp[c - base] += w * yb[r];
            ++n;
          };
          if (two_d) {
            for (int ix = 0; ix < g.n_x; ++ix) {
              const ctsm::VoxelIndex v{ix, sl, 0};
              const uint32_t c = (uint32_t)ctsm::voxel_column(g, v);
              for (const auto& cw : ctsm::pixel_area_factors(v, phi, g))
                apply(raster(cw.m_y, 0), c, cw.w);
            }
            continue;
          }
          for (int iy = 0; iy < g.n_y; ++iy)
            for (int ix = 0; ix < g.n_x; ++ix) {
              const ctsm::VoxelIndex v{ix, iy, sl};
              const uint32_t c = (uint32_t)ctsm::voxel_column(g, v);
              for (const auto& vw : ctsm::voxel_volume_factors(v, phi, g))
                apply(raster(vw.m_y, vw.m_z), c, vw.w);
            }
        }
        double bs = 0.0;
        for (double v : block) bs += v;
        for (double v : xp) bs += v;
        sums[it] = bs;
        counts[it] = n;
      });
      double cs = 0.0; uint64_t nu = 0;
      for (int i = 0; i < items; ++i) { cs += sums[i]; nu += counts[i]; }
      *checksum = cs; *updates = nu; return 0;)
}

// Bounded sample of build_system_matrix for bench.py's CSR cpu_baseline (C2's
// 55 GB matrix does not fit a bounded run): the listed angles' blocks, one
// angle per worker as ordered_parallel_for does (projector.cpp:114-140), each
// built as build_angle_block does (projector.cpp:92-104): per-row entry
// vectors filled through detail::angle_block_entries, then a stable sort by
// column. *nnz = entries of the listed angle blocks.
int ref_csr_angle_sample(const RefGeom* rg, const int32_t* angles, int n_sel, uint64_t* nnz,
                         int threads) {
  REF_GUARD(
      const ctsm::ScanGeometry g = to_g(rg); g.validate();
      const uint64_t rpa = (uint64_t)g.n_det_y * g.n_det_z;
      std::vector<uint64_t> counts(n_sel, 0);
      parallel_range(n_sel, threads, [&](int k) {
        std::vector<std::vector<std::pair<uint32_t, double>>> rows(rpa);
        ctsm::detail::angle_block_entries(
            g, ctsm::MatrixMode::consistent, 1, angles[k],
            [&](uint32_t r, uint32_t c, double w) { rows[r].emplace_back(c, w); });
        uint64_t n = 0;
        for (auto& row : rows) {
          std::stable_sort(row.begin(), row.end(),
                           [](const auto& a, const auto& b) { return a.first < b.first; });
          n += row.size();
        }
        counts[k] = n;
      });
      uint64_t total = 0;
      for (uint64_t c : counts) total += c;
      *nnz = total; return 0;)
}

int ref_back_project_matrix_free(const RefGeom* rg, const double* y, double* x, int threads) {
  std::vector<int32_t> all(rg->n_angles);
  for (int i = 0; i < rg->n_angles; ++i) all[i] = i;
  return ref_back_mf_angles(rg, all.data(), rg->n_angles, y, x, threads);
}

// SIRT (BASELINE.json configs[4]) composed from the reference's projector:
// R = 1/(A 1), C = 1/(A^T 1) (zero sums -> 0); iters x (x += C (A^T (R (y - A x)))).
int ref_sirt(const RefGeom* rg, const double* y, double* x, int iters, int threads) {
  const uint64_t nv = (uint64_t)rg->n_x * rg->n_y * rg->n_z;
  const uint64_t nm = (uint64_t)rg->n_angles * rg->n_det_y * rg->n_det_z;
  std::vector<double> ones_v(nv, 1.0), ones_m(nm, 1.0), R(nm), C(nv), ax(nm), r(nm), bp(nv);
  int st = ref_forward_project_matrix_free(rg, ones_v.data(), R.data(), threads);
  if (st) return st;
  st = ref_back_project_matrix_free(rg, ones_m.data(), C.data(), threads);
  if (st) return st;
  for (auto& v : R) v = v != 0.0 ? 1.0 / v : 0.0;
  for (auto& v : C) v = v != 0.0 ? 1.0 / v : 0.0;
  for (int it = 0; it < iters; ++it) {
    st = ref_forward_project_matrix_free(rg, x, ax.data(), threads);
    if (st) return st;
    for (uint64_t i = 0; i < nm; ++i) r[i] = R[i] * (y[i] - ax[i]);
    st = ref_back_project_matrix_free(rg, r.data(), bp.data(), threads);
    if (st) return st;
    for (uint64_t i = 0; i < nv; ++i) x[i] += C[i] * bp[i];
  }
  return 0;
}

// spectral_norm_power (projector.cpp:262-280) and nag_tikhonov (solver.cpp:17-75)
// on a reference CSR handle; scale_values (282-286).
int ref_spectral_norm_power(void* h, int iters, uint64_t seed, double* out) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  REF_GUARD(*out = ctsm::spectral_norm_power(*m, iters, seed); return 0;)
}

int ref_scale_values(void* h, double factor) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  REF_GUARD(ctsm::scale_values(m, factor); return 0;)
}

// trace (optional): 3 doubles per iteration {iter, objective, grad_norm_sq}
int ref_nag_tikhonov(void* h, const double* p, double lambda, int max_iter, double tol,
                     double* u, int* iterations, int* converged, double* trace) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  REF_GUARD(const std::vector<double> pv(p, p + m->n_rows);
            ctsm::SolveOptions opt;
            opt.lambda = lambda; opt.max_iter = max_iter; opt.tol = tol;
            const auto r = ctsm::nag_tikhonov(*m, pv, opt, trace != nullptr);
            std::copy(r.u.begin(), r.u.end(), u);
            *iterations = r.iterations; *converged = r.converged ? 1 : 0;
            if (trace) for (std::size_t i = 0; i < r.trace.size(); ++i) {
              trace[3 * i] = r.trace[i].iter;
              trace[3 * i + 1] = r.trace[i].objective;
              trace[3 * i + 2] = r.trace[i].grad_norm_sq;
            }
            return 0;)
}

// normal_samples (phantoms.cpp:78-87).
void ref_normal_samples(uint64_t n, uint64_t seed, double* out) {
  const auto v = ctsm::normal_samples(n, seed);
  std::copy(v.begin(), v.end(), out);
}

// CSM1 / CTT1 writers and readers (io.cpp:153-270).
int ref_write_matrix(void* h, const char* path) {
  auto* m = static_cast<ctsm::SparseSystemMatrix*>(h);
  REF_GUARD(ctsm::write_matrix(path, *m); return 0;)
}

void* ref_read_matrix(const char* path, int* status) {
  try {
    auto* m = new ctsm::SparseSystemMatrix(ctsm::read_matrix(path));
    *status = 0;
    return m;
  } catch (const ctsm::Error& e) {
    *status = fail_code(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    *status = -100;
  }
  return nullptr;
}

uint64_t ref_csr_cols(void* h) { return static_cast<ctsm::SparseSystemMatrix*>(h)->n_cols; }

// meta string (size query with buf == NULL)
uint64_t ref_csr_meta(void* h, char* buf, uint64_t cap) {
  const std::string& s = static_cast<ctsm::SparseSystemMatrix*>(h)->meta;
  if (buf) std::memcpy(buf, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

int ref_write_tensor(const char* path, const uint64_t* dims, int rank, const double* data) {
  REF_GUARD(const std::vector<uint64_t> d(dims, dims + rank);
            uint64_t n = 1; for (auto v : d) n *= v;
            ctsm::write_tensor(path, d, std::vector<double>(data, data + n)); return 0;)
}

// angle_column_sums (projector.cpp:288-295).
int ref_angle_column_sums(const RefGeom* rg, int ip, double* sums) {
  REF_GUARD(const auto v = ctsm::angle_column_sums(to_g(rg), ctsm::MatrixMode::consistent, 1, ip);
            std::copy(v.begin(), v.end(), sums); return 0;)
}

// ---- line / multiline modes ------------------------
// mode: 0 consistent, 1 line, 2 multiline (MatrixMode order, projector.hpp:12-16).
static ctsm::MatrixMode to_mode(int m) {
  return m == 1 ? ctsm::MatrixMode::line
                : (m == 2 ? ctsm::MatrixMode::multiline : ctsm::MatrixMode::consistent);
}

// line_weights / multiline_weights (baseline.cpp:99-128): hits of one
// detector cell in the reference's order; returns the count (<= cap stored).
long ref_line_weights(const RefGeom* rg, int mode, int k, int m_y, int m_z, int ip, uint32_t* col,
                      double* len, long cap) {
  REF_GUARD(const ctsm::ScanGeometry g = to_g(rg);
            const auto hits = mode == 1 ? ctsm::line_weights(m_y, m_z, ip, g)
                                        : ctsm::multiline_weights(m_y, m_z, ip, g, k);
            for (long i = 0; i < (long)hits.size() && i < cap; ++i) {
              col[i] = hits[i].col;
              len[i] = hits[i].len;
            } return (long)hits.size();)
}

// detail::angle_block_entries (projector.cpp:44-84) for any mode.
long ref_angle_block_entries_mode(const RefGeom* rg, int mode, int k, int ip, uint32_t* row,
                                  uint32_t* col, double* w, long cap) {
  REF_GUARD(long n = 0; ctsm::detail::angle_block_entries(
                to_g(rg), to_mode(mode), k, ip,
                [&](uint32_t r, uint32_t c, double v) {
                  if (n < cap) {
                    row[n] = r;
                    col[n] = c;
                    w[n] = v;
                  }
                  ++n;
                });
            return n;)
}

void* ref_build_system_matrix_mode(const RefGeom* rg, int mode, int k, int threads,
                                   uint64_t budget, int* status) {
  try {
    auto* m = new ctsm::SparseSystemMatrix(
        ctsm::build_system_matrix(to_g(rg), to_mode(mode), k, threads, budget));
    *status = 0;
    return m;
  } catch (const ctsm::Error& e) {
    *status = fail_code(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    *status = -100;
  }
  return nullptr;
}

int ref_forward_mf_mode(const RefGeom* rg, int mode, int k, const double* x, double* y,
                        int threads) {
  REF_GUARD(const ctsm::ScanGeometry g = to_g(rg);
            const std::vector<double> xv(x, x + g.n_voxels());
            const auto yv = ctsm::forward_project_matrix_free(g, to_mode(mode), k, xv, threads);
            std::copy(yv.begin(), yv.end(), y); return 0;)
}

// matrix-free A^T y for any mode: the a16 restatement through
// detail::angle_block_entries(mode, k), per-angle partials summed in angle order.
int ref_back_mf_mode(const RefGeom* rg, int mode, int k, const double* y, double* x,
                     int threads) {
  REF_GUARD(const ctsm::ScanGeometry g = to_g(rg); g.validate();
            const uint64_t rpa = (uint64_t)g.n_det_y * g.n_det_z;
            const uint64_t nv = g.n_voxels(); std::fill(x, x + nv, 0.0);
            const int chunk = std::max(1, threads);
            std::vector<std::vector<double>> part(chunk);
            for (int k0 = 0; k0 < g.n_angles; k0 += chunk) {
              const int n = std::min(chunk, g.n_angles - k0);
              parallel_range(n, threads, [&](int t) {
                auto& p = part[t];
                p.assign(nv, 0.0);
                const double* yb = y + (uint64_t)(k0 + t) * rpa;
                ctsm::detail::angle_block_entries(
                    g, to_mode(mode), k, k0 + t,
                    [&](uint32_t r, uint32_t c, double wv) { p[c] += wv * yb[r]; });
              });
              for (int t = 0; t < n; ++t)
                for (uint64_t i = 0; i < nv; ++i) x[i] += part[t][i];
            } return 0;)
}

}  // extern "C"

