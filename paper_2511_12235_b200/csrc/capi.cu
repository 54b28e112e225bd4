// capi.cu -- the extern "C" boundary (include/ctsm_b200.h): context, geometry
// validation, buffer management and the orchestration of the kernels in
// csr.cu / mf.cu. Host code only.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"

namespace ctsmb {

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

namespace {

thread_local std::string g_err;

const char* kCodeNames[] = {"Ok",          "DegenerateGeometry", "RayParallelToFace",
                            "SingularPhi", "CentralRow",         "ZRestrictionViolation",
                            "DimensionMismatch", "NonFinite",    "ZeroMatrix",
                            "TooLarge",    "InvalidSpec",        "OutOfMemory",
                            "InvalidConfig", "IoFailure"};

int fail(int code, const std::string& msg) {
  const char* name = (code >= 0 && code <= 13) ? kCodeNames[code] : "CudaError";
  g_err = std::string(name) + ": " + msg;
  return code;
}

#define CT_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      if (e_ == cudaErrorMemoryAllocation) {                                       \
        cudaGetLastError();                                                        \
        return fail(CTSM_ERR_OUT_OF_MEMORY, std::string("device allocation: ") +   \
                                                cudaGetErrorString(e_));           \
      }                                                                            \
      return fail(CTSM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    }                                                                              \
  } while (0)

#define CT_TRY(expr)          \
  do {                        \
    const int s_ = (expr);    \
    if (s_ != 0) return s_;   \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t n = 0;
};

}  // namespace
}  // namespace ctsmb

using namespace ctsmb;

struct ctsm_ctx {
  int device = 0;
  int* status = nullptr;        // device status word
  double* dred = nullptr;       // device reduction scratch (4 doubles)
  int* h_status = nullptr;      // pinned
  unsigned long long* n_upd = nullptr;    // device: voxel-ray updates of the last forward call
  unsigned long long* h_upd = nullptr;    // pinned mirror
  uint64_t last_updates = 0;
  // kernel family of the last matrix-free call (ctsm_last_kernel_path):
  // CTSM_PATH_* bits, so tests can assert which production kernel ran
  int last_path = 0;
  double* h_red = nullptr;      // pinned
  Buf angles, edges, cs, counts, scan, longrows, acc, part, base, alist, sv_up, sv_h, sv_hp,
      sv_q, sv_v, sv_part, sv_scal, tmp_a, tmp_b, tmp_c, tmp_d,
      tmp_e, tmp_f, lraw_start, lraw_col, lraw_val, lacc, bwd_t, vol_t, plans, rec, grp,
      cursor, plans2, rec2, grp2, angles2, counts2, longrows2, mfplans;
  // key of the base-angle tables currently in `base` / `cs` (upload_base)
  bool base_valid = false;
  std::vector<int> base_cached;
  int base_n_angles = 0;
  double base_a0 = 0.0, base_a1 = 0.0;
  // second stream + events of the pipelined CSR build (ctsm_csr_build)
  cudaStream_t side = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // stream of the host-buffer calls: created non-blocking on first use, so
  // the calls of two contexts (two host threads) overlap their copies with
  // each other's kernels instead of serialising on the legacy stream
  cudaStream_t hstream = nullptr;
};

namespace {

int ensure(ctsm_ctx* ctx, Buf& b, size_t bytes) {
  if (b.n >= bytes && b.p) return 0;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
  if (bytes == 0) return 0;
  CT_CUDA(cudaMalloc(&b.p, bytes));
  b.n = bytes;
  (void)ctx;
  return 0;
}

int set_device(ctsm_ctx* ctx) {
  if (!ctx) return fail(CTSM_ERR_INVALID_SPEC, "null context");
  CT_CUDA(cudaSetDevice(ctx->device));
  return 0;
}

// Synchronises the stream and converts a raised device guard into its code.
int host_stream(ctsm_ctx* ctx, cudaStream_t* st) {
  if (!ctx->hstream) CT_CUDA(cudaStreamCreateWithFlags(&ctx->hstream, cudaStreamNonBlocking));
  *st = ctx->hstream;
  return 0;
}

int check_status(ctsm_ctx* ctx, cudaStream_t st, const char* what) {
  CT_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  const int code = *ctx->h_status;
  if (code != 0) {
    CT_CUDA(cudaMemsetAsync(ctx->status, 0, sizeof(int), st));
    CT_CUDA(cudaStreamSynchronize(st));
    const char* msg = "device guard raised";
    switch (code) {
      case CTSM_ERR_DEGENERATE_GEOMETRY: msg = "point on or behind the source plane / no canonical quadrant"; break;
      case CTSM_ERR_NON_FINITE: msg = "negative weight beyond FP tolerance or non-finite result"; break;
      case CTSM_ERR_TOO_LARGE: msg = "sweep exceeds the device breakpoint capacity"; break;
      case CTSM_ERR_RAY_PARALLEL_TO_FACE: msg = "band ray parallel to x-faces"; break;
      default: break;
    }
    return fail(code, std::string(what) + ": " + msg);
  }
  return 0;
}

// ScanGeometry::validate (geometry.cpp:27-54).
int validate(const ctsm_geometry* g) {
  if (!g) return fail(CTSM_ERR_INVALID_SPEC, "null geometry");
  if (!(g->s > 0.0)) return fail(CTSM_ERR_INVALID_SPEC, "source distance s must be > 0");
  if (!(g->d >= 0.0)) return fail(CTSM_ERR_INVALID_SPEC, "detector distance d must be >= 0");
  if (!(g->d_y > 0.0) || !(g->d_z > 0.0))
    return fail(CTSM_ERR_INVALID_SPEC, "detector pitches must be > 0");
  if (g->n_det_y <= 0 || g->n_det_z <= 0 || g->n_angles <= 0)
    return fail(CTSM_ERR_INVALID_SPEC, "detector and angle counts must be > 0");
  if (g->n_det_y % 2 != 0)
    return fail(CTSM_ERR_INVALID_SPEC, "n_det_y must be even (centered detector)");
  if (g->n_det_z != 1 && g->n_det_z % 2 != 0)
    return fail(CTSM_ERR_INVALID_SPEC, "n_det_z must be 1 (2D) or even (centered detector)");
  if (!(g->a > 0.0) || !(g->b > 0.0) || !(g->c > 0.0))
    return fail(CTSM_ERR_INVALID_SPEC, "voxel sizes must be > 0");
  if (g->n_x <= 0 || g->n_y <= 0 || g->n_z <= 0)
    return fail(CTSM_ERR_INVALID_SPEC, "grid dimensions must be > 0");
  if (g->n_det_z == 1 && g->n_z > 1)
    return fail(CTSM_ERR_INVALID_SPEC, "volume grid requires n_det_z > 1");
  if (!(g->angle_end > g->angle_start))
    return fail(CTSM_ERR_INVALID_SPEC, "angle_end must exceed angle_start");
  if (!std::isfinite(g->s) || !std::isfinite(g->d) || !std::isfinite(g->d_y) ||
      !std::isfinite(g->d_z) || !std::isfinite(g->a) || !std::isfinite(g->b) ||
      !std::isfinite(g->c) || !std::isfinite(g->angle_start) || !std::isfinite(g->angle_end))
    return fail(CTSM_ERR_NON_FINITE, "geometry parameters must be finite");
  const double rx = g->n_x * g->a / 2.0, ry = g->n_y * g->b / 2.0;
  if (g->s <= std::hypot(rx, ry))
    return fail(CTSM_ERR_DEGENERATE_GEOMETRY, "source circle intersects the grid");
  return 0;
}

// Upper bound of the detector cells one pixel's shadow spans: u = sdd L / D
// (L lateral, D depth) moves by at most sdd / D * sqrt(1 + (L / D)^2) per
// unit of displacement, D >= s - R, |L / D| <= R / (s - R), R the grid
// half-diagonal.
double shadow_cells_bound(const ctsm_geometry* g) {
  const double R = std::hypot(g->n_x * g->a / 2.0, g->n_y * g->b / 2.0);
  const double t = R / (g->s - R);
  return std::hypot(g->a, g->b) * (g->s + g->d) / ((g->s - R) * g->d_y) * std::sqrt(1.0 + t * t);
}

// Device capacity of the exact sweep (common.cuh kMaxBrk breakpoints: the 4
// corners and the detector edges inside the shadow). The reference has no
// such limit (its sweep is a std::vector); a geometry beyond it is rejected
// here, by name, instead of failing inside a kernel.
int check_sweep_capacity(const ctsm_geometry* g) {
  const double w = shadow_cells_bound(g);
  if (!(std::floor(w) + 1.0 + 4.0 <= (double)kMaxBrk)) {
    char msg[200];
    snprintf(msg, sizeof msg,
             "a pixel's shadow can span %.0f detector cells; the device sweep holds %d "
             "(detector pitch too fine for the pixel size and magnification)",
             std::floor(w) + 1.0, kMaxBrk - 5);
    return fail(CTSM_ERR_TOO_LARGE, msg);
  }
  return 0;
}

// The 3D matrix-free kernels plan at most mf3d_max_pieces() pieces per column
// sweep (cells of the shadow + 2 zone boundaries).
int check_mf3d_capacity(const ctsm_geometry* g) {
  if (g->n_z == 1 && g->n_det_z == 1) return 0;
  const double w = shadow_cells_bound(g);
  if (!(std::floor(w) + 2.0 + 2.0 <= (double)mf3d_max_pieces())) {
    char msg[200];
    snprintf(msg, sizeof msg,
             "a voxel's shadow can span %.0f detector columns; the 3D matrix-free kernels hold "
             "%d (build the CSR matrix instead, or coarsen the detector)",
             std::floor(w) + 2.0, mf3d_max_pieces() - 2);
    return fail(CTSM_ERR_TOO_LARGE, msg);
  }
  return 0;
}

// Derived device geometry incl. the edge-table extent: every fan angle of the
// grid satisfies |tan| <= R / (s - R), R the grid half-diagonal.
int dev_geom(const ctsm_geometry* g, DevGeom* out) {
  CT_TRY(validate(g));
  DevGeom d = make_dev_geom(*g);
  const double R = std::hypot(g->n_x * g->a / 2.0, g->n_y * g->b / 2.0);
  const double umax = R / (g->s - R) * (g->s + g->d) / g->d_y;
  if (!(umax < (double)(1 << 22)))
    return fail(CTSM_ERR_TOO_LARGE, "fan spans too many detector edges for the edge table");
  const int E = (int)std::ceil(umax) + 3;
  d.edge_lo = -E;
  d.n_edges = 2 * E + 1;
  *out = d;
  return 0;
}

// Upper bound of any row sum of A (sum of voxel fractions in one detector
// cell's ray wedge): the wedge's area / volume inside the depth slab
// |depth - s| <= R divided by the pixel area / voxel volume.
double row_sum_bound(const ctsm_geometry* g) {
  const double R2 = std::hypot(g->n_x * g->a / 2.0, g->n_y * g->b / 2.0);
  const double dt = g->d_y / (g->s + g->d);
  const bool two_d = (g->n_z == 1 && g->n_det_z == 1);
  if (two_d) return 2.0 * g->s * R2 * dt / (g->a * g->b);
  const double da = g->d_z / (g->s + g->d);
  const double hi = g->s + R2, lo = g->s - R2;
  return dt * da * (hi * hi * hi - lo * lo * lo) / 3.0 / (g->a * g->b * g->c);
}

int n_in_shard(int begin, int end, int step) {
  if (step <= 0 || end <= begin) return 0;
  return (end - begin + step - 1) / step;
}

int check_shard(const ctsm_geometry* g, int begin, int end, int step) {
  if (begin < 0 || end > g->n_angles || begin > end || step <= 0)
    return fail(CTSM_ERR_INVALID_SPEC, "angle shard out of range");
  return 0;
}

size_t dtype_size(int dtype) { return dtype == CTSM_F64 ? 8 : 4; }

int check_dtype(int dtype) {
  if (dtype != CTSM_F64 && dtype != CTSM_F32) return fail(CTSM_ERR_INVALID_SPEC, "unknown dtype");
  return 0;
}

int fetch_max_abs(ctsm_ctx* ctx, int dtype, uint64_t n, const void* v, cudaStream_t st,
                  double* out) {
  CT_CUDA(max_abs(dtype, n, v, ctx->dred, st));
  CT_CUDA(cudaMemcpyAsync(ctx->h_red, ctx->dred, sizeof(double), cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  *out = *ctx->h_red;
  return 0;
}

}  // namespace

int ctsmb::set_error(int code, const char* msg) { return fail(code, msg); }
int ctsmb::select_device(ctsm_ctx* ctx) { return ctx ? set_device(ctx) : 0; }

extern "C" {

int ctsm_create(int device, ctsm_ctx** out) {
  if (!out) return fail(CTSM_ERR_INVALID_SPEC, "null output pointer");
  int n = 0;
  CT_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(CTSM_ERR_INVALID_SPEC, "no such CUDA device");
  CT_CUDA(cudaSetDevice(device));
  ctsm_ctx* c = new ctsm_ctx();
  c->device = device;
  CT_CUDA(cudaMalloc(&c->status, sizeof(int)));
  CT_CUDA(cudaMemset(c->status, 0, sizeof(int)));
  CT_CUDA(cudaMalloc(&c->dred, 4 * sizeof(double)));
  CT_CUDA(cudaMallocHost(&c->h_status, sizeof(int)));
  CT_CUDA(cudaMallocHost(&c->h_red, 4 * sizeof(double)));
  CT_CUDA(cudaMalloc(&c->n_upd, sizeof(unsigned long long)));
  CT_CUDA(cudaMallocHost(&c->h_upd, sizeof(unsigned long long)));
  *out = c;
  return 0;
}

int ctsm_destroy(ctsm_ctx* ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->device);
  Buf* bufs[] = {&ctx->angles, &ctx->edges, &ctx->cs,    &ctx->counts, &ctx->scan,
                 &ctx->longrows, &ctx->acc, &ctx->part, &ctx->base, &ctx->alist, &ctx->sv_up, &ctx->sv_h, &ctx->sv_hp, &ctx->sv_q,
                 &ctx->sv_v, &ctx->sv_part, &ctx->sv_scal, &ctx->tmp_a, &ctx->tmp_b,  &ctx->tmp_c,
                 &ctx->tmp_d, &ctx->tmp_e, &ctx->tmp_f, &ctx->lraw_start, &ctx->lraw_col,
                 &ctx->lraw_val, &ctx->lacc, &ctx->bwd_t, &ctx->vol_t, &ctx->plans, &ctx->rec,
                 &ctx->grp, &ctx->cursor, &ctx->plans2, &ctx->rec2, &ctx->grp2, &ctx->angles2,
                 &ctx->counts2, &ctx->longrows2, &ctx->mfplans};
  if (ctx->side) cudaStreamDestroy(ctx->side);
  for (cudaEvent_t e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (Buf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (ctx->hstream) cudaStreamDestroy(ctx->hstream);
  cudaFree(ctx->status);
  cudaFree(ctx->dred);
  cudaFreeHost(ctx->h_status);
  cudaFreeHost(ctx->h_red);
  cudaFree(ctx->n_upd);
  cudaFreeHost(ctx->h_upd);
  delete ctx;
  return 0;
}

const char* ctsm_last_error(void) { return g_err.c_str(); }
const char* ctsm_version(void) { return "ctsm-b200 0.1 (sm_100a)"; }
uint64_t ctsm_launch_count(void) { return g_launches.load(); }

int ctsm_validate_geometry(const ctsm_geometry* g) {
  DevGeom d;
  return dev_geom(g, &d);
}

// ---- K1/K2 ----------------------------------------------------------------
static int prepare_exact(ctsm_ctx* ctx, const DevGeom& d, int angle_begin, int n_sel,
                         cudaStream_t st) {
  CT_TRY(ensure(ctx, ctx->angles, (size_t)(n_sel > 0 ? n_sel : 1) * exact_angle_bytes()));
  CT_TRY(ensure(ctx, ctx->edges, (size_t)d.n_edges * edge_angle_bytes()));
  CT_CUDA(build_exact_tables(d, angle_begin, n_sel, ctx->angles.p, ctx->edges.p, st));
  return 0;
}

// Angles per emission chunk: bounds the per-chunk scratch (plans, records,
// row-grouped arrays) and keeps chunk-local rows and entries below 2^31.
static int csr_chunk_angles(const DevGeom& d, int n_sel, uint64_t per_angle_entries) {
  static const uint64_t rec_budget = [] {  // experiment knob: CTSM_CSR_REC_MB
    const char* e = getenv("CTSM_CSR_REC_MB");
    return (uint64_t)(e ? atoll(e) : 2048) << 20;
  }();
  const uint64_t plan_budget = 1ull << 30;
  uint64_t a = rec_budget / (16ull * (per_angle_entries + 1));
  const size_t plan1 = csr_plan_bytes(d, 1);
  if (plan1) a = std::min<uint64_t>(a, plan_budget / plan1);
  a = std::min<uint64_t>(a, (1ull << 31) / (uint64_t)d.rows_per_angle);
  a = std::min<uint64_t>(a, (uint64_t)n_sel);
  return (int)std::max<uint64_t>(a, 1);
}

// Angle-0 entry count (the reference's budget estimate, projector.cpp:155-169).
static int csr_angle_count(ctsm_ctx* ctx, const DevGeom& d, int angle, uint64_t* nnz,
                           cudaStream_t st) {
  const uint64_t rpa = (uint64_t)d.rows_per_angle;
  CT_TRY(ensure(ctx, ctx->counts, rpa * sizeof(unsigned)));
  CT_TRY(ensure(ctx, ctx->tmp_a, (rpa + 1) * sizeof(uint64_t)));
  CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes(rpa)));
  CT_TRY(ensure(ctx, ctx->plans, csr_plan_bytes(d, 1)));
  CT_TRY(prepare_exact(ctx, d, angle, 1, st));
  CT_CUDA(cudaMemsetAsync(ctx->counts.p, 0, rpa * sizeof(unsigned), st));
  CsrSink sk{0, (unsigned*)ctx->counts.p, nullptr, nullptr, nullptr, nullptr, 0, 0};
  CT_CUDA(csr_emit(d, ctx->angles.p, ctx->edges.p, 1, sk, ctx->plans.p, ctx->status, st));
  CT_CUDA(exclusive_scan_u32_u64((const unsigned*)ctx->counts.p, rpa, (uint64_t*)ctx->tmp_a.p,
                                 ctx->scan.p, st));
  CT_CUDA(cudaMemcpyAsync(nnz, (uint64_t*)ctx->tmp_a.p + rpa, sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, st));
  return check_status(ctx, st, "build_system_matrix");
}

static int csr_budget_check(const ctsm_geometry* g, const DevGeom& d, uint64_t nnz0,
                            uint64_t memory_budget_bytes) {
  const uint64_t n_meas = (uint64_t)d.rows_per_angle * (uint64_t)g->n_angles;
  const uint64_t est_nnz = nnz0 * (uint64_t)g->n_angles;
  const uint64_t est_bytes =
      est_nnz * (sizeof(uint32_t) + sizeof(double)) + (n_meas + 1) * sizeof(uint64_t);
  if (est_bytes > memory_budget_bytes) {
    char msg[256];
    snprintf(msg, sizeof msg, "estimated %llu entries (%llu MiB) exceed the budget of %llu MiB",
             (unsigned long long)est_nnz, (unsigned long long)(est_bytes >> 20),
             (unsigned long long)(memory_budget_bytes >> 20));
    return fail(CTSM_ERR_OUT_OF_MEMORY, msg);
  }
  return 0;
}

static int csr_prologue(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                        DevGeom* d) {
  CT_TRY(dev_geom(g, d));
  CT_TRY(check_sweep_capacity(g));  // before any device work: testable without a GPU
  CT_TRY(set_device(ctx));
  if ((uint64_t)g->n_x * g->n_y * g->n_z > 0xffffffffull)
    return fail(CTSM_ERR_TOO_LARGE, "grid exceeds 2^32 voxel columns");
  return check_shard(g, angle_begin, angle_end, 1);
}

int ctsm_csr_angle_nnz(ctsm_ctx* ctx, const ctsm_geometry* g, int angle, uint64_t* nnz_out,
                       void* stream) {
  DevGeom d;
  CT_TRY(csr_prologue(ctx, g, angle, angle + 1, &d));
  return csr_angle_count(ctx, d, angle, nnz_out, (cudaStream_t)stream);
}

// Two-evaluation protocol: count (this call), the caller allocates, fill.
int ctsm_csr_count(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                   uint64_t memory_budget_bytes, uint64_t* row_start_dev, uint64_t* nnz_out,
                   void* stream) {
  DevGeom d;
  CT_TRY(csr_prologue(ctx, g, angle_begin, angle_end, &d));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = angle_end - angle_begin;
  const uint64_t n_rows = (uint64_t)d.rows_per_angle * n_sel;
  uint64_t nnz0 = 0;
  CT_TRY(csr_angle_count(ctx, d, 0, &nnz0, st));
  CT_TRY(csr_budget_check(g, d, nnz0, memory_budget_bytes));
  const int A = csr_chunk_angles(d, n_sel, nnz0);
  CT_TRY(ensure(ctx, ctx->plans, csr_plan_bytes(d, A)));
  CT_TRY(ensure(ctx, ctx->counts, n_rows * sizeof(unsigned)));
  CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes(n_rows)));
  CT_CUDA(cudaMemsetAsync(ctx->counts.p, 0, n_rows * sizeof(unsigned), st));
  for (int c0 = 0; c0 < n_sel; c0 += A) {
    const int na = std::min(A, n_sel - c0);
    CT_TRY(prepare_exact(ctx, d, angle_begin + c0, na, st));
    CsrSink sk{0, (unsigned*)ctx->counts.p + (uint64_t)c0 * d.rows_per_angle, nullptr, nullptr,
               nullptr, nullptr, 0, 0};
    CT_CUDA(csr_emit(d, ctx->angles.p, ctx->edges.p, na, sk, ctx->plans.p, ctx->status, st));
  }
  CT_CUDA(exclusive_scan_u32_u64((const unsigned*)ctx->counts.p, n_rows, row_start_dev,
                                 ctx->scan.p, st));
  uint64_t nnz = 0;
  CT_CUDA(cudaMemcpyAsync(&nnz, row_start_dev + n_rows, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                          st));
  CT_TRY(check_status(ctx, st, "build_system_matrix"));
  if (angle_begin == 0 && angle_end == g->n_angles && nnz == 0)
    return fail(CTSM_ERR_ZERO_MATRIX, "system matrix has no entries");
  *nnz_out = nnz;
  return 0;
}

// Fill: each chunk is emitted into row-grouped scratch (slots from per-row
// cursors), then radix-sorted by column into the caller's arrays.
int ctsm_csr_fill(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                  const uint64_t* row_start_dev, uint32_t* col_dev, double* val_dev,
                  void* stream) {
  DevGeom d;
  CT_TRY(csr_prologue(ctx, g, angle_begin, angle_end, &d));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = angle_end - angle_begin;
  const uint64_t rpa = (uint64_t)d.rows_per_angle;
  // chunk bounds from the row offsets: two D2H reads per chunk boundary
  uint64_t total = 0;
  CT_CUDA(cudaMemcpyAsync(&total, row_start_dev + rpa * n_sel, sizeof total,
                          cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  const int A = csr_chunk_angles(d, n_sel, n_sel ? total / n_sel + 1 : 1);
  const int n_chunks = (n_sel + A - 1) / A;
  std::vector<uint64_t> bounds((size_t)n_chunks + 1, 0);
  for (int i = 0; i < n_chunks; ++i)
    CT_CUDA(cudaMemcpyAsync(&bounds[i], row_start_dev + rpa * (uint64_t)(i * A), sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  bounds[n_chunks] = total;
  CT_TRY(ensure(ctx, ctx->plans, csr_plan_bytes(d, A)));
  CT_TRY(ensure(ctx, ctx->counts, (size_t)A * rpa * sizeof(unsigned)));
  CT_TRY(ensure(ctx, ctx->longrows, ((size_t)A * rpa + 2) * sizeof(unsigned)));
  size_t ci = 0;
  for (int c0 = 0; c0 < n_sel; c0 += A, ++ci) {
    const int na = std::min(A, n_sel - c0);
    const uint64_t nr = (uint64_t)na * rpa, row_off = (uint64_t)c0 * rpa;
    const uint64_t base = bounds[ci], nnz_c = bounds[ci + 1] - bounds[ci];
    if (nnz_c == 0) continue;
    CT_TRY(ensure(ctx, ctx->grp, nnz_c * 16));
    CT_TRY(prepare_exact(ctx, d, angle_begin + c0, na, st));
    CT_CUDA(cudaMemsetAsync(ctx->counts.p, 0, nr * sizeof(unsigned), st));
    CsrSink sk{1, (unsigned*)ctx->counts.p, row_start_dev + row_off, ctx->grp.p, nullptr, nullptr,
               0, base};
    CT_CUDA(csr_emit(d, ctx->angles.p, ctx->edges.p, na, sk, ctx->plans.p, ctx->status, st));
    unsigned* lr = (unsigned*)ctx->longrows.p;
    CT_CUDA(csr_sort_rows_radix(nr, row_start_dev + row_off, ctx->grp.p, col_dev, val_dev, ~0ull,
                                nnz_c, lr, lr + nr + 1, st, (uint64_t)d.n_vox));
  }
  return check_status(ctx, st, "build_system_matrix");
}

// Single-evaluation build: every weight is evaluated once. Per angle chunk:
// mode-2 emission (row counts + 16-byte records) and the row scan on the
// caller's stream; on a second stream the records are scattered into
// row-grouped scratch and each row is radix-sorted by column into the
// caller's arrays, overlapping the next chunk's (FP64-bound) emission with
// this chunk's (HBM-bound) grouping. Nothing in the loop waits for the
// device: record counts and row offsets are read by the kernels from device
// memory, the per-chunk scratch is double-buffered, and the host checks the
// counts once at the end (dropped records -> the build is redone with a
// larger record buffer). col_dev / val_dev hold `capacity` entries;
// *nnz_out receives the shard's entry count and the arrays are complete only
// if it is <= capacity (rows beyond are skipped: call again with arrays of
// *nnz_out entries).
int ctsm_csr_build(ctsm_ctx* ctx, const ctsm_geometry* g, int angle_begin, int angle_end,
                   uint64_t memory_budget_bytes, uint64_t* row_start_dev, uint32_t* col_dev,
                   double* val_dev, uint64_t capacity, uint64_t* nnz_out, void* stream) {
  DevGeom d;
  CT_TRY(csr_prologue(ctx, g, angle_begin, angle_end, &d));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = angle_end - angle_begin;
  const uint64_t rpa = (uint64_t)d.rows_per_angle;
  uint64_t nnz0 = 0;
  CT_TRY(csr_angle_count(ctx, d, 0, &nnz0, st));
  CT_TRY(csr_budget_check(g, d, nnz0, memory_budget_bytes));
  if (!ctx->side) CT_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  for (int i = 0; i < 4; ++i)
    if (!ctx->ev[i]) CT_CUDA(cudaEventCreateWithFlags(&ctx->ev[i], cudaEventDisableTiming));
  static const bool one_stream = getenv("CTSM_CSR_ONE_STREAM") != nullptr;  // experiment knob
  cudaStream_t sb = one_stream ? st : ctx->side;
  uint64_t per_angle = nnz0 + nnz0 / 2 + 4096;  // angle 0 is a flat (sparser) angle
  const unsigned long long seg_slack = 148ull * 8 * 4 * 256;
  for (int attempt = 0;; ++attempt) {
    // (the scratch is double-buffered: ~4 x the record budget in total)
    const int A = csr_chunk_angles(d, n_sel, per_angle);
    const unsigned long long cap = (unsigned long long)A * per_angle + seg_slack;
    const int n_chunks = (n_sel + A - 1) / A;
    // double-buffered per-chunk scratch
    Buf* plans[2] = {&ctx->plans, &ctx->plans2};
    Buf* angles[2] = {&ctx->angles, &ctx->angles2};
    Buf* counts[2] = {&ctx->counts, &ctx->counts2};
    Buf* rec[2] = {&ctx->rec, &ctx->rec2};
    Buf* grp[2] = {&ctx->grp, &ctx->grp2};
    Buf* lrow[2] = {&ctx->longrows, &ctx->longrows2};
    for (int p = 0; p < 2; ++p) {
      CT_TRY(ensure(ctx, *plans[p], csr_plan_bytes(d, A)));
      CT_TRY(ensure(ctx, *angles[p], (size_t)A * exact_angle_bytes()));
      CT_TRY(ensure(ctx, *counts[p], (size_t)A * rpa * sizeof(unsigned)));
      CT_TRY(ensure(ctx, *rec[p], (size_t)cap * 16));
      CT_TRY(ensure(ctx, *grp[p], (size_t)cap * 16));
      CT_TRY(ensure(ctx, *lrow[p], ((size_t)A * rpa + 2) * sizeof(unsigned)));
    }
    CT_TRY(ensure(ctx, ctx->edges, (size_t)d.n_edges * edge_angle_bytes()));
    CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes((uint64_t)A * rpa)));
    CT_TRY(ensure(ctx, ctx->cursor, ((size_t)n_chunks + 2) * sizeof(unsigned long long)));
    unsigned long long* cursors = (unsigned long long*)ctx->cursor.p;  // [n_chunks], then base
    uint64_t* base_slot = (uint64_t*)(cursors + n_chunks);
    CT_CUDA(cudaMemsetAsync(cursors, 0, ((size_t)n_chunks + 2) * sizeof(unsigned long long), st));
    CT_CUDA(cudaMemsetAsync(row_start_dev, 0, sizeof(uint64_t), st));
    for (int c = 0; c < n_chunks; ++c) {
      const int p = c & 1, c0 = c * A;
      const int na = std::min(A, n_sel - c0);
      const uint64_t nr = (uint64_t)na * rpa, row_off = (uint64_t)c0 * rpa;
      // the grouping of chunk c - 2 must be done with this parity's scratch
      if (c >= 2) CT_CUDA(cudaStreamWaitEvent(st, ctx->ev[2 + p], 0));
      CT_CUDA(build_exact_tables(d, angle_begin + c0, na, angles[p]->p, ctx->edges.p, st));
      CT_CUDA(cudaMemsetAsync(counts[p]->p, 0, nr * sizeof(unsigned), st));
      CsrSink sk{2, (unsigned*)counts[p]->p, nullptr, nullptr, rec[p]->p, cursors + c, cap, 0};
      CT_CUDA(csr_emit(d, angles[p]->p, ctx->edges.p, na, sk, plans[p]->p, ctx->status, st));
      CT_CUDA(cudaMemcpyAsync(base_slot, row_start_dev + row_off, sizeof(uint64_t),
                              cudaMemcpyDeviceToDevice, st));
      CT_CUDA(exclusive_scan_u32_u64((const unsigned*)counts[p]->p, nr, row_start_dev + row_off,
                                     ctx->scan.p, st, 0, base_slot, (unsigned*)counts[p]->p));
      CT_CUDA(cudaEventRecord(ctx->ev[p], st));
      // second stream: group by row (the counts now hold the rows' local
      // offsets and serve as cursors), sort by column
      CT_CUDA(cudaStreamWaitEvent(sb, ctx->ev[p], 0));
      CT_CUDA(csr_scatter_records(rec[p]->p, cursors + c, cap, (unsigned*)counts[p]->p, grp[p]->p,
                                  cap, sb));
      unsigned* lr = (unsigned*)lrow[p]->p;
      CT_CUDA(csr_sort_rows_radix(nr, row_start_dev + row_off, grp[p]->p, col_dev, val_dev,
                                  capacity, cap, lr, lr + nr + 1, sb, (uint64_t)d.n_vox));
      CT_CUDA(cudaEventRecord(ctx->ev[2 + p], sb));
    }
    // join, then look at the counts
    for (int p = 0; p < 2 && p < n_chunks; ++p) CT_CUDA(cudaStreamWaitEvent(st, ctx->ev[2 + p], 0));
    std::vector<unsigned long long> cur_h((size_t)n_chunks);
    uint64_t total = 0;
    CT_CUDA(cudaMemcpyAsync(cur_h.data(), cursors, (size_t)n_chunks * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    CT_CUDA(cudaMemcpyAsync(&total, row_start_dev + rpa * n_sel, sizeof total,
                            cudaMemcpyDeviceToHost, st));
    CT_TRY(check_status(ctx, st, "build_system_matrix"));
    unsigned long long worst = 0;
    for (unsigned long long v : cur_h) worst = std::max(worst, v);
    if (worst <= cap) {
      if (angle_begin == 0 && angle_end == g->n_angles && total == 0)
        return fail(CTSM_ERR_ZERO_MATRIX, "system matrix has no entries");
      *nnz_out = total;
      return 0;
    }
    if (attempt >= 3) return fail(CTSM_ERR_OUT_OF_MEMORY, "record buffer keeps overflowing");
    per_angle = (worst + worst / 4) / (unsigned long long)A + 4096;  // records were dropped
  }
}

// ---- the reference's weight API (weights2d.hpp:31-32, weights3d.hpp:90-91,
// projector.hpp:72-78) ---------------------------------------------------------
int ctsm_weights_batch(ctsm_ctx* ctx, const ctsm_geometry* g, uint64_t n, const int32_t* ix,
                       const int32_t* iy, const int32_t* iz, const double* phi, int cap,
                       int32_t* count, int32_t* m_y, int32_t* m_z, double* w) {
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_sweep_capacity(g));
  CT_TRY(set_device(ctx));
  if (cap <= 0) return fail(CTSM_ERR_INVALID_SPEC, "slab capacity must be > 0");
  if (n == 0) return 0;
  for (uint64_t q = 0; q < n; ++q) {
    // VoxelIndex outside the grid is the caller's error in the reference
    // (faces are computed for any index); keep the indices as given
    (void)q;
  }
  cudaStream_t st = nullptr;
  CT_TRY(ensure(ctx, ctx->edges, (size_t)d.n_edges * edge_angle_bytes()));
  CT_CUDA(build_exact_tables(d, 0, 0, nullptr, ctx->edges.p, st));
  const size_t ni = n * sizeof(int), nd = n * sizeof(double);
  const size_t slab = (size_t)n * cap;
  CT_TRY(ensure(ctx, ctx->tmp_a, 4 * ni + nd));
  CT_TRY(ensure(ctx, ctx->tmp_b, slab * (2 * sizeof(int) + sizeof(double))));
  int* dix = (int*)ctx->tmp_a.p;
  int* diy = dix + n;
  int* diz = diy + n;
  int* dcount = diz + n;
  double* dphi = (double*)((char*)ctx->tmp_a.p + 4 * ni);
  double* dw = (double*)ctx->tmp_b.p;
  int* dmy = (int*)(dw + slab);
  int* dmz = dmy + slab;
  CT_CUDA(cudaMemcpyAsync(dix, ix, ni, cudaMemcpyHostToDevice, st));
  CT_CUDA(cudaMemcpyAsync(diy, iy, ni, cudaMemcpyHostToDevice, st));
  if (iz) CT_CUDA(cudaMemcpyAsync(diz, iz, ni, cudaMemcpyHostToDevice, st));
  else CT_CUDA(cudaMemsetAsync(diz, 0, ni, st));
  CT_CUDA(cudaMemcpyAsync(dphi, phi, nd, cudaMemcpyHostToDevice, st));
  CT_CUDA(weights_batch(d, ctx->edges.p, (long long)n, dix, diy, diz, dphi, cap, dcount, dmy, dmz,
                        dw, ctx->status, st));
  CT_CUDA(cudaMemcpyAsync(count, dcount, ni, cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaMemcpyAsync(m_y, dmy, slab * sizeof(int), cudaMemcpyDeviceToHost, st));
  if (m_z) CT_CUDA(cudaMemcpyAsync(m_z, dmz, slab * sizeof(int), cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaMemcpyAsync(w, dw, slab * sizeof(double), cudaMemcpyDeviceToHost, st));
  CT_TRY(check_status(ctx, st, "weights"));
  for (uint64_t q = 0; q < n; ++q)
    if (count[q] > cap) return fail(CTSM_ERR_TOO_LARGE, "a query has more weights than the slab holds");
  return 0;
}

int ctsm_angle_block_entries(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int angle,
                             uint64_t capacity, uint32_t* raster_dev, uint32_t* col_dev,
                             double* w_dev, uint64_t* n_out, void* stream) {
  DevGeom d;
  CT_TRY(csr_prologue(ctx, g, angle, angle + 1, &d));
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t rpa = (uint64_t)d.rows_per_angle;
  if (mode != CTSM_MODE_CONSISTENT) {
    // ray modes emit row by row (projector.cpp:72-83): the block's CSR order
    CT_TRY(ensure(ctx, ctx->tmp_c, (rpa + 1) * sizeof(uint64_t)));
    uint64_t nnz = 0;
    CT_TRY(ctsm_csr_count_mode(ctx, g, mode, k, angle, angle + 1, ~0ull, (uint64_t*)ctx->tmp_c.p,
                               &nnz, stream));
    *n_out = nnz;
    if (nnz > capacity) return 0;
    CT_TRY(ctsm_csr_fill_mode(ctx, g, mode, k, angle, angle + 1, (const uint64_t*)ctx->tmp_c.p,
                              col_dev, w_dev, stream));
    CT_CUDA(expand_row_index(rpa, (const uint64_t*)ctx->tmp_c.p, raster_dev, st));
    CT_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
  const uint64_t n_cols = (uint64_t)d.n_vox;
  const unsigned long long cap = capacity + 148ull * 8 * 4 * 256;
  CT_TRY(ensure(ctx, ctx->plans, csr_plan_bytes(d, 1)));
  CT_TRY(ensure(ctx, ctx->counts, std::max(rpa, n_cols) * sizeof(unsigned)));
  CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes(std::max(rpa, n_cols))));
  CT_TRY(ensure(ctx, ctx->tmp_c, (std::max(rpa, n_cols) + 1) * sizeof(uint64_t)));
  CT_TRY(ensure(ctx, ctx->cursor, 2 * sizeof(unsigned long long)));
  CT_TRY(ensure(ctx, ctx->rec, (size_t)cap * 16));
  CT_TRY(ensure(ctx, ctx->grp, (size_t)cap * 16));
  CT_TRY(prepare_exact(ctx, d, angle, 1, st));
  CT_CUDA(cudaMemsetAsync(ctx->counts.p, 0, rpa * sizeof(unsigned), st));
  CT_CUDA(cudaMemsetAsync(ctx->cursor.p, 0, sizeof(unsigned long long), st));
  CsrSink sk{2, (unsigned*)ctx->counts.p, nullptr, nullptr, ctx->rec.p,
             (unsigned long long*)ctx->cursor.p, cap, 0};
  CT_CUDA(csr_emit(d, ctx->angles.p, ctx->edges.p, 1, sk, ctx->plans.p, ctx->status, st));
  // the entry count is the sum of the row counts
  CT_CUDA(exclusive_scan_u32_u64((const unsigned*)ctx->counts.p, rpa, (uint64_t*)ctx->tmp_c.p,
                                 ctx->scan.p, st));
  uint64_t nnz = 0;
  unsigned long long cur = 0;
  CT_CUDA(cudaMemcpyAsync(&nnz, (uint64_t*)ctx->tmp_c.p + rpa, sizeof nnz, cudaMemcpyDeviceToHost,
                          st));
  CT_CUDA(cudaMemcpyAsync(&cur, ctx->cursor.p, sizeof cur, cudaMemcpyDeviceToHost, st));
  CT_TRY(check_status(ctx, st, "angle_block_entries"));
  *n_out = nnz;
  if (nnz > capacity || cur > cap) return 0;  // the caller retries with arrays of *n_out
  CT_CUDA(records_to_emission_order(ctx->rec.p, (unsigned long long*)ctx->cursor.p, cap, n_cols,
                                    (unsigned*)ctx->counts.p, (uint64_t*)ctx->tmp_c.p,
                                    ctx->scan.p, ctx->grp.p, g->n_det_y, g->n_det_z, raster_dev,
                                    col_dev, w_dev, st));
  CT_CUDA(cudaStreamSynchronize(st));
  return 0;
}

// ---- independent numerical oracles (oracle.cpp:70-196) -----------------------
static int oracle_upload(ctsm_ctx* ctx, uint64_t n, const double* boxes, const double* phi,
                         const int32_t* m_y, const int32_t* m_z, double** dbox, double** dphi,
                         int** dmy, int** dmz, cudaStream_t st) {
  CT_TRY(ensure(ctx, ctx->tmp_a, n * (7 * sizeof(double) + 2 * sizeof(int))));
  *dbox = (double*)ctx->tmp_a.p;
  *dphi = *dbox + 6 * n;
  *dmy = (int*)(*dphi + n);
  *dmz = *dmy + n;
  CT_CUDA(cudaMemcpyAsync(*dbox, boxes, 6 * n * sizeof(double), cudaMemcpyHostToDevice, st));
  CT_CUDA(cudaMemcpyAsync(*dphi, phi, n * sizeof(double), cudaMemcpyHostToDevice, st));
  CT_CUDA(cudaMemcpyAsync(*dmy, m_y, n * sizeof(int), cudaMemcpyHostToDevice, st));
  CT_CUDA(cudaMemcpyAsync(*dmz, m_z, n * sizeof(int), cudaMemcpyHostToDevice, st));
  return 0;
}

int ctsm_mc_volume_3d(ctsm_ctx* ctx, uint64_t n, const double* boxes, const double* phi, double s,
                      double d, double d_y, double d_z, const int32_t* m_y, const int32_t* m_z,
                      uint64_t n_samples, uint64_t seed, double* value, double* std_err,
                      uint64_t* hits) {
  CT_TRY(set_device(ctx));
  if (n_samples == 0) return fail(CTSM_ERR_INVALID_SPEC, "n_samples must be > 0");
  if (n == 0) return 0;
  cudaStream_t st = nullptr;
  double *dbox, *dphi;
  int *dmy, *dmz;
  CT_TRY(oracle_upload(ctx, n, boxes, phi, m_y, m_z, &dbox, &dphi, &dmy, &dmz, st));
  CT_TRY(ensure(ctx, ctx->tmp_b, n * sizeof(unsigned long long)));
  CT_CUDA(cudaMemsetAsync(ctx->tmp_b.p, 0, n * sizeof(unsigned long long), st));
  CT_CUDA(mc_volume_batch((long long)n, dbox, dphi, s, d, d_y, d_z, dmy, dmz, n_samples, seed,
                          (unsigned long long*)ctx->tmp_b.p, st));
  std::vector<unsigned long long> h(n);
  CT_CUDA(cudaMemcpyAsync(h.data(), ctx->tmp_b.p, n * sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  for (uint64_t i = 0; i < n; ++i) {
    // oracle.cpp:92-97: binomial standard error, floored at one count's worth
    const double p = (double)h[i] / (double)n_samples;
    const double var = std::max(p * (1.0 - p), 1.0 / (double)n_samples);
    if (value) value[i] = p;
    if (std_err) std_err[i] = std::sqrt(var / (double)n_samples);
    if (hits) hits[i] = h[i];
  }
  return 0;
}

int ctsm_multiline_volume_3d(ctsm_ctx* ctx, uint64_t n, const double* boxes, const double* phi,
                             double s, double d, double d_y, double d_z, const int32_t* m_y,
                             const int32_t* m_z, int k, double* out) {
  CT_TRY(set_device(ctx));
  if (k <= 0) return fail(CTSM_ERR_INVALID_SPEC, "ray grid size k must be > 0");
  if (n == 0) return 0;
  cudaStream_t st = nullptr;
  double *dbox, *dphi;
  int *dmy, *dmz;
  CT_TRY(oracle_upload(ctx, n, boxes, phi, m_y, m_z, &dbox, &dphi, &dmy, &dmz, st));
  std::vector<double> nodes((size_t)2 * k);
  gauss_legendre_host(k, nodes.data(), nodes.data() + k);
  CT_TRY(ensure(ctx, ctx->tmp_b, (n + 2 * (size_t)k) * sizeof(double)));
  double* dout = (double*)ctx->tmp_b.p;
  double* dnodes = dout + n;
  CT_CUDA(cudaMemcpyAsync(dnodes, nodes.data(), 2 * (size_t)k * sizeof(double),
                          cudaMemcpyHostToDevice, st));
  CT_CUDA(multiline_volume_batch((long long)n, dbox, dphi, s, d, d_y, d_z, dmy, dmz, k, dnodes,
                                 dnodes + k, dout, st));
  CT_CUDA(cudaMemcpyAsync(out, dout, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  return 0;
}

void ctsm_gauss_legendre(int k, double* x, double* w) {
  if (k > 0) gauss_legendre_host(k, x, w);
}

int ctsm_selftest_division(ctsm_ctx* ctx, uint64_t n, uint64_t seed, uint64_t* mismatches) {
  CT_TRY(set_device(ctx));
  CT_TRY(ensure(ctx, ctx->cursor, 2 * sizeof(unsigned long long)));
  CT_CUDA(cudaMemset(ctx->cursor.p, 0, sizeof(unsigned long long)));
  CT_CUDA(selftest_division(n, seed, (unsigned long long*)ctx->cursor.p, nullptr));
  unsigned long long h = 0;
  CT_CUDA(cudaMemcpy(&h, ctx->cursor.p, sizeof h, cudaMemcpyDeviceToHost));
  *mismatches = h;
  return 0;
}

// ---- K3/K4 ----------------------------------------------------------------
int ctsm_spmv(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols, const uint64_t* row_start_dev,
              const uint32_t* col_dev, const double* val_dev, const double* x_dev,
              double* y_dev, void* stream) {
  CT_TRY(set_device(ctx));
  (void)n_cols;
  cudaStream_t st = (cudaStream_t)stream;
  CT_CUDA(spmv_csr(n_rows, row_start_dev, col_dev, val_dev, x_dev, y_dev, ctx->status, st));
  const int s = check_status(ctx, st, "forward projection");
  if (s == CTSM_ERR_NON_FINITE) return fail(s, "forward projection not finite");
  return s;
}

int ctsm_csr_colsum_max(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                        const uint64_t* row_start_dev, const uint32_t* col_dev,
                        const double* val_dev, double* colsum_max, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  CT_TRY(ensure(ctx, ctx->tmp_a, n_cols * sizeof(double)));
  CT_CUDA(cudaMemsetAsync(ctx->tmp_a.p, 0, n_cols * sizeof(double), st));
  CT_CUDA(colsum_abs(n_rows, row_start_dev, col_dev, val_dev, (double*)ctx->tmp_a.p, st));
  double mcol = 0.0;
  CT_TRY(fetch_max_abs(ctx, CTSM_F64, n_cols, ctx->tmp_a.p, st, &mcol));
  if (!std::isfinite(mcol)) return fail(CTSM_ERR_NON_FINITE, "matrix not finite");
  *colsum_max = mcol;
  return 0;
}

// Fixed-point scale of the CSR scatter: 2^61 / B with B >= max|x_c| rounded
// up to a power of two, so that last-bit differences of the (atomically
// summed) column bound never change the result bits.
static double csr_fixed_scale(double mcol, double my) {
  const double B = mcol * my * (1.0 + 1e-6);
  if (!(B > 0.0)) return 0.0;
  int ex = 0;
  (void)std::frexp(B, &ex);  // B <= 2^ex
  return std::ldexp(1.0, 61 - ex);
}

int ctsm_spmv_t_bound(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                      const uint64_t* row_start_dev, const uint32_t* col_dev,
                      const double* val_dev, double colsum_max, const double* y_dev,
                      double* x_dev, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  if (!std::isfinite(colsum_max) || colsum_max < 0.0)
    return fail(CTSM_ERR_NON_FINITE, "column-sum bound not finite");
  // fixed-point bound: |x_c| <= max|y| * max_c sum_r |A_rc|
  double my = 0.0;
  CT_TRY(fetch_max_abs(ctx, CTSM_F64, n_rows, y_dev, st, &my));
  if (!std::isfinite(my)) return fail(CTSM_ERR_NON_FINITE, "back projection not finite");
  const double scale = csr_fixed_scale(colsum_max, my);
  if (!(scale > 0.0)) {
    CT_CUDA(cudaMemsetAsync(x_dev, 0, n_cols * sizeof(double), st));
    CT_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
  CT_TRY(ensure(ctx, ctx->tmp_b, n_cols * sizeof(unsigned long long)));
  CT_CUDA(cudaMemsetAsync(ctx->tmp_b.p, 0, n_cols * sizeof(unsigned long long), st));
  CT_CUDA(spmvt_csr_fixed(n_rows, row_start_dev, col_dev, val_dev, y_dev,
                          (unsigned long long*)ctx->tmp_b.p, scale, st));
  CT_CUDA(fixed_to_double(n_cols, (const unsigned long long*)ctx->tmp_b.p, scale, x_dev, st));
  return check_status(ctx, st, "back projection");
}

int ctsm_csc_build(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                   const uint64_t* row_start_dev, const uint32_t* col_dev, const double* val_dev,
                   uint64_t* col_start_dev, uint32_t* row_dev, double* valt_dev, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows >= (1ull << 32)) return fail(CTSM_ERR_TOO_LARGE, "CSC row indices are 32-bit");
  uint64_t nnz = 0;
  CT_CUDA(cudaMemcpyAsync(&nnz, row_start_dev + n_rows, sizeof nnz, cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  // counts and cursors (u32 per column), scan scratch
  CT_TRY(ensure(ctx, ctx->tmp_a, n_cols * sizeof(unsigned)));
  CT_TRY(ensure(ctx, ctx->tmp_b, n_cols * sizeof(unsigned long long)));
  CT_TRY(ensure(ctx, ctx->tmp_c, scan_scratch_bytes(n_cols)));
  unsigned* counts = (unsigned*)ctx->tmp_a.p;
  unsigned* cursor = (unsigned*)ctx->tmp_b.p;
  CT_CUDA(cudaMemsetAsync(counts, 0, n_cols * sizeof(unsigned), st));
  CT_CUDA(cudaMemsetAsync(cursor, 0, n_cols * sizeof(unsigned), st));
  CT_CUDA(csc_count(nnz, col_dev, counts, st));
  CT_CUDA(exclusive_scan_u32_u64(counts, n_cols, col_start_dev, ctx->tmp_c.p, st));
  CT_CUDA(csc_scatter(n_rows, row_start_dev, col_dev, val_dev, col_start_dev, cursor, row_dev,
                      valt_dev, st));
  CT_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int ctsm_spmv_t_csc(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols,
                    const uint64_t* col_start_dev, const uint32_t* row_dev,
                    const double* valt_dev, double colsum_max, const double* y_dev,
                    double* x_dev, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  if (!std::isfinite(colsum_max) || colsum_max < 0.0)
    return fail(CTSM_ERR_NON_FINITE, "column-sum bound not finite");
  double my = 0.0;
  CT_TRY(fetch_max_abs(ctx, CTSM_F64, n_rows, y_dev, st, &my));
  if (!std::isfinite(my)) return fail(CTSM_ERR_NON_FINITE, "back projection not finite");
  const double scale = csr_fixed_scale(colsum_max, my);  // the scatter's scale: same integers
  if (!(scale > 0.0)) {
    CT_CUDA(cudaMemsetAsync(x_dev, 0, n_cols * sizeof(double), st));
    CT_CUDA(cudaStreamSynchronize(st));
    return 0;
  }
  CT_TRY(ensure(ctx, ctx->tmp_b, n_cols * sizeof(unsigned long long)));
  CT_CUDA(spmvt_csc_fixed(n_cols, col_start_dev, row_dev, valt_dev, y_dev,
                          (unsigned long long*)ctx->tmp_b.p, scale, st));
  CT_CUDA(fixed_to_double(n_cols, (const unsigned long long*)ctx->tmp_b.p, scale, x_dev, st));
  return check_status(ctx, st, "back projection");
}

int ctsm_spmv_t(ctsm_ctx* ctx, uint64_t n_rows, uint64_t n_cols, const uint64_t* row_start_dev,
                const uint32_t* col_dev, const double* val_dev, const double* y_dev,
                double* x_dev, void* stream) {
  double mcol = 0.0;
  CT_TRY(ctsm_csr_colsum_max(ctx, n_rows, n_cols, row_start_dev, col_dev, val_dev, &mcol, stream));
  return ctsm_spmv_t_bound(ctx, n_rows, n_cols, row_start_dev, col_dev, val_dev, mcol, y_dev,
                           x_dev, stream);
}

// ---- K5/K6 ----------------------------------------------------------------
static int prepare_cs(ctsm_ctx* ctx, const DevGeom& d, int begin, int step, int n_sel,
                      cudaStream_t st) {
  ctx->base_valid = false;  // cs is shared with the symmetric kernels' base tables
  CT_TRY(ensure(ctx, ctx->cs, (size_t)(n_sel > 0 ? n_sel : 1) * sizeof(AngleCS)));
  CT_CUDA(build_angle_cs(d, begin, step, n_sel, (AngleCS*)ctx->cs.p, st));
  return 0;
}

// Quarter-turn symmetry of the scan (see mf.cu): square grid with an even
// side, a == b, n_angles % 4 == 0 and angles covering exactly one full turn.
static bool symmetry_disabled() {
  const char* e = std::getenv("CTSM_NO_SYMMETRY");
  return e && e[0] && e[0] != '0';
}
static bool quarter_symmetric(const ctsm_geometry* g) {
  if (symmetry_disabled()) return false;
  if (g->n_x != g->n_y || g->n_x % 2 != 0 || g->a != g->b || g->n_angles % 4 != 0) return false;
  const double span = g->angle_end - g->angle_start;
  return std::fabs(span - 2.0 * 3.14159265358979323846) <= 1e-12 * span;
}
// Dihedral (8-fold) symmetry: additionally angle_start == 0 and
// n_angles % 8 == 0, so the angle set is closed under reflection phi -> -phi
// (the grid and the detector are centred). CTSM_NO_DIHEDRAL=1 caps the order at 4.
static bool dihedral_disabled() {
  const char* e = std::getenv("CTSM_NO_DIHEDRAL");
  return e && e[0] && e[0] != '0';
}
static int symmetry_order(const ctsm_geometry* g) {
  if (!quarter_symmetric(g)) return 1;
  if (!dihedral_disabled() && g->angle_start == 0.0 && g->n_angles % 8 == 0)
    return 8;
  return 4;
}
// CTSM_PATH_* bits of a symmetric call (include/ctsm_b200.h).
static int sym_path_bits(const ctsm_geometry* g) {
  const bool two_d = (g->n_z == 1 && g->n_det_z == 1);
  int p = symmetry_order(g) == 8 ? CTSM_PATH_DIHEDRAL : CTSM_PATH_QUARTER;
#ifndef CTSM_NO_ZMIRROR
  if (!two_d && g->n_z % 2 == 0) p |= CTSM_PATH_ZMIRROR;
#endif
  return p;
}
// Base angle set of a symmetry order: [0, n/4) for 4, [0, n/8] for 8.
static int base_limit(const ctsm_geometry* g, int order) {
  return order == 8 ? g->n_angles / 8 + 1 : g->n_angles / 4;
}
// All angles of the orbits of `base` (ascending) -- the sinogram rows written.
static std::vector<int> orbit_angles(const ctsm_geometry* g, int order,
                                     const std::vector<int>& base) {
  const int n = g->n_angles, q = n / 4;
  std::vector<char> hit(n, 0);
  for (int i : base)
    for (int k = 0; k < 4; ++k) {
      hit[(i + k * q) % n] = 1;
      if (order == 8) hit[((n - i) % n + k * q) % n] = 1;
    }
  std::vector<int> out;
  for (int a = 0; a < n; ++a)
    if (hit[a]) out.push_back(a);
  return out;
}
// Base angles (< n/4) of a shard closed under +n/4: (begin, end, step) with
// end == n, begin < step and step dividing n/4. Returns false otherwise.
static bool sym_base_of_shard(const ctsm_geometry* g, int begin, int end, int step,
                              std::vector<int>* base) {
  if (symmetry_order(g) == 8) {  // only the full range is closed under reflection
    if (begin != 0 || end != g->n_angles || step != 1) return false;
    base->clear();
    for (int i = 0; i < base_limit(g, 8); ++i) base->push_back(i);
    return true;
  }
  const int q = g->n_angles / 4;
  if (end != g->n_angles || step <= 0 || begin >= step || q % step != 0) return false;
  base->clear();
  for (int i = begin; i < q; i += step) base->push_back(i);
  return true;
}
static int upload_base(ctsm_ctx* ctx, const DevGeom& d, const std::vector<int>& base,
                       cudaStream_t st) {
  const size_t n = base.size();
  // the base list and its (cos, sin) table depend only on the scan's angles:
  // repeated projections of one scan (the common case) skip the upload, the
  // table kernel and the host synchronisation
  if (ctx->base_valid && ctx->base_cached == base && ctx->base_n_angles == d.n_angles &&
      ctx->base_a0 == d.angle_start && ctx->base_a1 == d.angle_end && ctx->base.p && ctx->cs.p)
    return 0;
  ctx->base_valid = false;
  CT_TRY(ensure(ctx, ctx->base, (n ? n : 1) * sizeof(int)));
  if (n)
    CT_CUDA(cudaMemcpyAsync(ctx->base.p, base.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
  CT_TRY(ensure(ctx, ctx->cs, (n ? n : 1) * sizeof(AngleCS)));
  CT_CUDA(build_angle_cs_list(d, (const int*)ctx->base.p, (int)n, (AngleCS*)ctx->cs.p, st));
  CT_CUDA(cudaStreamSynchronize(st));  // base is pageable host memory
  ctx->base_cached = base;
  ctx->base_n_angles = d.n_angles;
  ctx->base_a0 = d.angle_start;
  ctx->base_a1 = d.angle_end;
  ctx->base_valid = true;
  return 0;
}

// Dihedral forward: base angles in [0, n/8], rows of all their D4 images.
static int fwd_d8_impl(ctsm_ctx* ctx, const ctsm_geometry* g, const DevGeom& d, int dtype,
                       const std::vector<int>& base, double mx, const void* x, void* y,
                       cudaStream_t st) {
  const uint64_t n_meas = (uint64_t)d.rows_per_angle * g->n_angles;
  const int nb = (int)base.size();
  if (nb == 0) return 0;
  const bool two_d = (g->n_z == 1 && g->n_det_z == 1);
  const size_t nf = (!two_d && dtype == CTSM_F32) ? fwd3d_f32_scratch_elems(d, 8) : 0;
  if (nf) {  // fp32 3D: vector float reductions, no fixed-point rows
    ctx->last_path |= CTSM_PATH_F32_VECRED;
    CT_TRY(upload_base(ctx, d, base, st));
    CT_TRY(ensure(ctx, ctx->bwd_t, nf * sizeof(float)));
    CT_TRY(ensure(ctx, ctx->vol_t, (size_t)d.n_vox * sizeof(float)));
    CT_CUDA(cudaMemsetAsync(ctx->n_upd, 0, sizeof(unsigned long long), st));
    CT_TRY(ensure(ctx, ctx->mfplans, mf3d_plan_bytes(d, 8)));
    CT_CUDA(fwd3d_mf_d8_f32(d, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb,
                            (const float*)x, (float*)y, ctx->n_upd, ctx->status, st, ctx->vol_t.p,
                            (float*)ctx->bwd_t.p, ctx->mfplans.p));
    CT_CUDA(cudaMemcpyAsync(ctx->h_upd, ctx->n_upd, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    return 0;
  }
  const std::vector<int> rows = orbit_angles(g, 8, base);
  CT_TRY(ensure(ctx, ctx->alist, rows.size() * sizeof(int)));
  CT_CUDA(cudaMemcpyAsync(ctx->alist.p, rows.data(), rows.size() * sizeof(int),
                          cudaMemcpyHostToDevice, st));
  CT_TRY(upload_base(ctx, d, base, st));  // synchronizes: rows may go out of scope
  CT_TRY(ensure(ctx, ctx->acc, n_meas * sizeof(unsigned long long)));
  unsigned long long* acc = (unsigned long long*)ctx->acc.p;
  const int* al = (const int*)ctx->alist.p;
  const int nl = (int)rows.size();
  CT_CUDA(rows_list(d, dtype, al, nl, acc, 1.0, nullptr, 0, st));
  const double B = mx * row_sum_bound(g) * 1.05;
  double scale = B > 0.0 ? std::ldexp(1.0, 61) / B : 1.0;
  // the kernel's shared-memory limbs need every contribution |w x| scale
  // below 2^47 (f64) / 2^23 (f32); weights are area fractions <= 1
  if (two_d && mx > 0.0)
    scale = std::min(scale, std::ldexp(1.0, dtype == CTSM_F64 ? 47 : 23) / (mx * 1.001));
  CT_CUDA(cudaMemsetAsync(ctx->n_upd, 0, sizeof(unsigned long long), st));
  if (two_d) {
    CT_CUDA(fwd_mf_d8(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, x, acc,
                      scale, ctx->n_upd, ctx->status, st));
  } else {
    CT_TRY(ensure(ctx, ctx->vol_t, (size_t)d.n_vox * (dtype == CTSM_F64 ? 8 : 4)));
    CT_TRY(ensure(ctx, ctx->mfplans, mf3d_plan_bytes(d, 8)));
    CT_CUDA(fwd3d_mf_sym(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, x,
                         acc, scale, ctx->n_upd, ctx->status, st, 8, ctx->vol_t.p,
                         ctx->mfplans.p));
  }
  CT_CUDA(rows_list(d, dtype, al, nl, acc, scale, y, 1, st));
  CT_CUDA(cudaMemcpyAsync(ctx->h_upd, ctx->n_upd, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  return 0;
}

// Symmetric forward over the orbit shard of `base` (rows of angles b + k n/4).
static int fwd_sym_impl(ctsm_ctx* ctx, const ctsm_geometry* g, const DevGeom& d, int dtype,
                        const std::vector<int>& base, int base_step, const void* x, void* y,
                        cudaStream_t st) {
  const uint64_t n_meas = (uint64_t)d.rows_per_angle * g->n_angles;
  double mx = 0.0;
  CT_TRY(fetch_max_abs(ctx, dtype, (uint64_t)d.n_vox, x, st, &mx));
  if (!std::isfinite(mx)) return fail(CTSM_ERR_NON_FINITE, "image not finite");
  ctx->last_path = sym_path_bits(g);
  if (symmetry_order(g) == 8) return fwd_d8_impl(ctx, g, d, dtype, base, mx, x, y, st);
  CT_TRY(upload_base(ctx, d, base, st));
  CT_TRY(ensure(ctx, ctx->acc, n_meas * sizeof(unsigned long long)));
  unsigned long long* acc = (unsigned long long*)ctx->acc.p;
  const int q = g->n_angles / 4, nb = (int)base.size();
  if (nb == 0) return 0;
  for (int k = 0; k < 4; ++k) CT_CUDA(zero_rows_u64(d, base[0] + k * q, base_step, nb, acc, st));
  const double B = mx * row_sum_bound(g) * 1.05;
  const double scale = B > 0.0 ? std::ldexp(1.0, 61) / B : 1.0;
  CT_CUDA(cudaMemsetAsync(ctx->n_upd, 0, sizeof(unsigned long long), st));
  const bool two_d = (g->n_z == 1 && g->n_det_z == 1);
  if (two_d) {
    CT_CUDA(fwd_mf_sym(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, x, acc,
                       scale, ctx->n_upd, ctx->status, st));
  } else {
    CT_TRY(ensure(ctx, ctx->vol_t, (size_t)d.n_vox * (dtype == CTSM_F64 ? 8 : 4)));
    CT_TRY(ensure(ctx, ctx->mfplans, mf3d_plan_bytes(d, 4)));
    CT_CUDA(fwd3d_mf_sym(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, x,
                         acc, scale, ctx->n_upd, ctx->status, st, 4, ctx->vol_t.p,
                         ctx->mfplans.p));
  }
  for (int k = 0; k < 4; ++k)
    CT_CUDA(fixed_to_float_rows(d, dtype, base[0] + k * q, base_step, nb, acc, scale, y, st));
  CT_CUDA(cudaMemcpyAsync(ctx->h_upd, ctx->n_upd, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  return 0;
}

static int bwd_sym_impl(ctsm_ctx* ctx, const ctsm_geometry* g, const DevGeom& d, int dtype,
                        const std::vector<int>& base, const void* y, void* x, cudaStream_t st) {
  ctx->last_path = sym_path_bits(g);
  CT_TRY(upload_base(ctx, d, base, st));
  const int nb = (int)base.size();
  const bool two_d = (g->n_z == 1 && g->n_det_z == 1);
  if (!two_d) {
    const size_t ne = bwd3d_scratch_elems(d, symmetry_order(g), dtype);
    if (!ne) ctx->last_path &= ~CTSM_PATH_ZMIRROR;  // the plain-gather variant has no mirror
    if (ne) CT_TRY(ensure(ctx, ctx->bwd_t, ne * (dtype == CTSM_F64 ? 8 : 4)));
    // two partial volumes (the split symmetric back-projection, mf.cu)
    CT_TRY(ensure(ctx, ctx->vol_t, 2 * (size_t)d.n_vox * (dtype == CTSM_F64 ? 8 : 4)));
    CT_TRY(ensure(ctx, ctx->mfplans, mf3d_plan_bytes(d, symmetry_order(g))));
    CT_CUDA(bwd3d_mf_sym(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, y, x,
                         ctx->status, st, symmetry_order(g), ne ? ctx->bwd_t.p : nullptr,
                         ctx->vol_t.p, ctx->mfplans.p));
  } else if (symmetry_order(g) == 8) {
    const int nc = bwd_d8_chunks(d, nb);
    if (nc > 1) CT_TRY(ensure(ctx, ctx->part, (size_t)nc * g->n_x * g->n_y * sizeof(double)));
    const size_t ne = bwd_d8_scratch_elems(d, nb, dtype);
    if (ne) CT_TRY(ensure(ctx, ctx->bwd_t, ne * (dtype == CTSM_F64 ? 8 : 4)));
    CT_CUDA(bwd_mf_d8(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, y, x,
                      (double*)ctx->part.p, nc, ctx->status, st, ne ? ctx->bwd_t.p : nullptr));
  } else {
    const int nc = bwd_sym_chunks(d, nb);
    if (nc > 1) CT_TRY(ensure(ctx, ctx->part, (size_t)nc * g->n_x * g->n_y * sizeof(double)));
    CT_CUDA(bwd_mf_sym(d, dtype, (const AngleCS*)ctx->cs.p, (const int*)ctx->base.p, nb, y, x,
                       (double*)ctx->part.p, nc, ctx->status, st));
  }
  return 0;
}

static int fwd_impl(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int begin, int end,
                    int step, const void* x, void* y, cudaStream_t st) {
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_mf3d_capacity(g));
  CT_TRY(check_dtype(dtype));
  CT_TRY(check_shard(g, begin, end, step));
  const int n_sel = n_in_shard(begin, end, step);
  if (n_sel == 0) return 0;
  std::vector<int> base;
  if (quarter_symmetric(g) && sym_base_of_shard(g, begin, end, step, &base))
    return fwd_sym_impl(ctx, g, d, dtype, base, step, x, y, st);
  const uint64_t n_meas = (uint64_t)d.rows_per_angle * g->n_angles;
  double mx = 0.0;
  CT_TRY(fetch_max_abs(ctx, dtype, (uint64_t)d.n_vox, x, st, &mx));
  if (!std::isfinite(mx)) return fail(CTSM_ERR_NON_FINITE, "image not finite");
  ctx->last_path = CTSM_PATH_GENERAL;
  CT_TRY(prepare_cs(ctx, d, begin, step, n_sel, st));
  CT_TRY(ensure(ctx, ctx->acc, n_meas * sizeof(unsigned long long)));
  unsigned long long* acc = (unsigned long long*)ctx->acc.p;
  CT_CUDA(zero_rows_u64(d, begin, step, n_sel, acc, st));
  const double B = mx * row_sum_bound(g) * 1.05;
  const double scale = B > 0.0 ? std::ldexp(1.0, 61) / B : 1.0;
  CT_CUDA(cudaMemsetAsync(ctx->n_upd, 0, sizeof(unsigned long long), st));
  CT_TRY(ensure(ctx, ctx->mfplans, mf3d_plan_bytes_general(d)));
  CT_CUDA(fwd_mf(d, dtype, (const AngleCS*)ctx->cs.p, begin, step, n_sel, x, acc, scale,
                 ctx->n_upd, ctx->status, st, ctx->mfplans.p));
  CT_CUDA(fixed_to_float_rows(d, dtype, begin, step, n_sel, acc, scale, y, st));
  CT_CUDA(cudaMemcpyAsync(ctx->h_upd, ctx->n_upd, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  return 0;
}

static int bwd_impl(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int begin, int end,
                    int step, const void* y, void* x, cudaStream_t st) {
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_mf3d_capacity(g));
  CT_TRY(check_dtype(dtype));
  CT_TRY(check_shard(g, begin, end, step));
  const int n_sel = n_in_shard(begin, end, step);
  std::vector<int> base;
  if (n_sel > 0 && quarter_symmetric(g) && sym_base_of_shard(g, begin, end, step, &base))
    return bwd_sym_impl(ctx, g, d, dtype, base, y, x, st);
  ctx->last_path = CTSM_PATH_GENERAL;
  CT_TRY(prepare_cs(ctx, d, begin, step, n_sel, st));
  const int nc = bwd_chunks(d, n_sel);
  if (nc > 1) CT_TRY(ensure(ctx, ctx->part, (size_t)nc * g->n_x * g->n_y * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->mfplans, mf3d_plan_bytes_general(d)));
  CT_CUDA(bwd_mf(d, dtype, (const AngleCS*)ctx->cs.p, begin, step, n_sel, y, x,
                 (double*)ctx->part.p, nc, ctx->status, st, ctx->mfplans.p));
  return 0;
}

int ctsm_fwd_mf(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int angle_begin,
                int angle_end, int angle_step, const void* x_dev, void* y_dev, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  CT_TRY(fwd_impl(ctx, g, dtype, angle_begin, angle_end, angle_step, x_dev, y_dev, st));
  CT_TRY(check_status(ctx, st, "forward_project_matrix_free"));
  ctx->last_updates = *ctx->h_upd;
  return 0;
}

uint64_t ctsm_last_update_count(ctsm_ctx* ctx) { return ctx ? ctx->last_updates : 0; }

int ctsm_last_kernel_path(ctsm_ctx* ctx) { return ctx ? ctx->last_path : 0; }

int ctsm_quarter_symmetric(const ctsm_geometry* g) {
  DevGeom d;
  if (dev_geom(g, &d) != 0) return 0;
  return quarter_symmetric(g) ? 1 : 0;
}

int ctsm_symmetry_order(const ctsm_geometry* g) {
  DevGeom d;
  if (dev_geom(g, &d) != 0) return 1;
  return symmetry_order(g);
}

int ctsm_shard_angles(const ctsm_geometry* g, int rank, int world, int* angles_out, int* n_out,
                      int* orbits_out) {
  CT_TRY(validate(g));
  if (world <= 0 || rank < 0 || rank >= world)
    return fail(CTSM_ERR_INVALID_SPEC, "rank / world out of range");
  const int order = symmetry_order(g);
  std::vector<int> a;
  if (order >= 4) {
    std::vector<int> base;
    for (int i = rank; i < base_limit(g, order); i += world) base.push_back(i);
    a = orbit_angles(g, order, base);
  } else {
    for (int i = rank; i < g->n_angles; i += world) a.push_back(i);
  }
  if (angles_out) std::copy(a.begin(), a.end(), angles_out);
  if (n_out) *n_out = (int)a.size();
  if (orbits_out) *orbits_out = order >= 4 ? 1 : 0;
  return 0;
}

static int orbit_base(const ctsm_geometry* g, int base_begin, int base_step,
                      std::vector<int>* base) {
  if (!quarter_symmetric(g))
    return fail(CTSM_ERR_INVALID_SPEC, "orbit shards need a quarter-turn symmetric scan");
  const int lim = base_limit(g, symmetry_order(g));
  if (base_begin < 0 || base_step <= 0) return fail(CTSM_ERR_INVALID_SPEC, "bad orbit shard");
  base->clear();
  for (int i = base_begin; i < lim; i += base_step) base->push_back(i);
  return 0;
}

int ctsm_fwd_mf_orbits(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int base_begin,
                       int base_step, const void* x_dev, void* y_dev, void* stream) {
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_mf3d_capacity(g));
  CT_TRY(check_dtype(dtype));
  std::vector<int> base;
  CT_TRY(orbit_base(g, base_begin, base_step, &base));
  cudaStream_t st = (cudaStream_t)stream;
  if (base.empty()) return 0;
  CT_TRY(fwd_sym_impl(ctx, g, d, dtype, base, base_step, x_dev, y_dev, st));
  CT_TRY(check_status(ctx, st, "forward_project_matrix_free"));
  ctx->last_updates = *ctx->h_upd;
  return 0;
}

int ctsm_bwd_mf_orbits(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int base_begin,
                       int base_step, const void* y_dev, void* x_dev, void* stream) {
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_mf3d_capacity(g));
  CT_TRY(check_dtype(dtype));
  std::vector<int> base;
  CT_TRY(orbit_base(g, base_begin, base_step, &base));
  cudaStream_t st = (cudaStream_t)stream;
  if (base.empty()) {
    CT_CUDA(cudaMemsetAsync(x_dev, 0, (size_t)d.n_vox * (dtype == CTSM_F64 ? 8 : 4), st));
    return check_status(ctx, st, "back_project_matrix_free");
  }
  CT_TRY(bwd_sym_impl(ctx, g, d, dtype, base, y_dev, x_dev, st));
  return check_status(ctx, st, "back_project_matrix_free");
}

int ctsm_bwd_mf(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int angle_begin,
                int angle_end, int angle_step, const void* y_dev, void* x_dev, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  CT_TRY(bwd_impl(ctx, g, dtype, angle_begin, angle_end, angle_step, y_dev, x_dev, st));
  return check_status(ctx, st, "back_project_matrix_free");
}

// ---- line / multiline modes (baseline.cpp:13-128) ----
static int check_mode(int mode, int k) {
  if (mode != CTSM_MODE_CONSISTENT && mode != CTSM_MODE_LINE && mode != CTSM_MODE_MULTILINE)
    return fail(CTSM_ERR_INVALID_SPEC, "unknown matrix mode");
  if (mode == CTSM_MODE_MULTILINE && k <= 0)
    return fail(CTSM_ERR_INVALID_SPEC, "multiline ray count must be > 0");
  return 0;
}

// Final (merged) entry counts of the ray-mode rows of angles [angle_begin,
// angle_begin + n_sel) into ctx->counts. Multiline rows are traced into
// ctx->lraw_* (offsets ctx->lraw_start) and merged there in place
// (merge_hits, baseline.cpp:81-94); line rows have distinct columns already.
static int ray_rows(ctsm_ctx* ctx, const DevGeom& d, int mode, int k, int angle_begin, int n_sel,
                    cudaStream_t st) {
  const uint64_t n_rows = (uint64_t)d.rows_per_angle * n_sel;
  CT_TRY(ensure(ctx, ctx->angles, (size_t)(n_sel > 0 ? n_sel : 1) * ray_angle_bytes()));
  CT_CUDA(ray_angle_table(d, angle_begin, 1, n_sel, ctx->angles.p, st));
  CT_TRY(ensure(ctx, ctx->counts, (n_rows ? n_rows : 1) * sizeof(unsigned)));
  CT_CUDA(ray_count(d, ctx->angles.p, mode, k, n_rows, (unsigned*)ctx->counts.p, st));
  if (mode == CTSM_MODE_LINE || k == 1) return 0;
  CT_TRY(ensure(ctx, ctx->lraw_start, (n_rows + 1) * sizeof(uint64_t)));
  CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes(n_rows)));
  CT_CUDA(exclusive_scan_u32_u64((const unsigned*)ctx->counts.p, n_rows,
                                 (uint64_t*)ctx->lraw_start.p, ctx->scan.p, st));
  uint64_t raw = 0;
  CT_CUDA(cudaMemcpyAsync(&raw, (uint64_t*)ctx->lraw_start.p + n_rows, sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  CT_TRY(ensure(ctx, ctx->lraw_col, (raw ? raw : 1) * sizeof(uint32_t)));
  CT_TRY(ensure(ctx, ctx->lraw_val, (raw ? raw : 1) * sizeof(double)));
  CT_CUDA(ray_fill(d, ctx->angles.p, mode, k, n_rows, (const uint64_t*)ctx->lraw_start.p,
                   (uint32_t*)ctx->lraw_col.p, (double*)ctx->lraw_val.p, st));
  CT_TRY(ensure(ctx, ctx->longrows, (n_rows + 1) * sizeof(unsigned)));
  CT_CUDA(ray_sort_merge(n_rows, (const uint64_t*)ctx->lraw_start.p, (unsigned*)ctx->counts.p,
                         (uint32_t*)ctx->lraw_col.p, (double*)ctx->lraw_val.p,
                         (unsigned*)ctx->longrows.p, (unsigned*)ctx->longrows.p + n_rows,
                         ctx->status, st));
  return 0;
}

// Bound on any column sum of a line / multiline matrix over one angle: the
// (sub-)rays through a voxel land in its detector footprint, whose width is
// at most W = diag * sdd / D (1 + U / D) per axis (D >= s - R_xy the least
// depth, U the largest lateral offset); at most k W / pitch + 1 sub-rays of
// weight <= diag / k (k^2 W_y W_z / pitch^2 .. in 3D) cross it.
static double ray_colsum_bound(const ctsm_geometry* g) {
  const bool two_d = g->n_z == 1 && g->n_det_z == 1;
  const double rxy = std::hypot(g->n_x * g->a / 2.0, g->n_y * g->b / 2.0);
  const double zmax = g->n_z * g->c / 2.0;
  const double diag = two_d ? std::hypot(g->a, g->b)
                            : std::sqrt(g->a * g->a + g->b * g->b + g->c * g->c);
  const double dmin = g->s - rxy, sdd = g->s + g->d;
  const double wy = diag * sdd / dmin * (1.0 + rxy / dmin);
  double b = diag * (wy / g->d_y + 2.0);
  if (!two_d) b *= diag * sdd / dmin * (1.0 + zmax / dmin) / g->d_z + 2.0;
  return 2.0 * b;
}

int ctsm_csr_count_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int angle_begin,
                        int angle_end, uint64_t memory_budget_bytes, uint64_t* row_start_dev,
                        uint64_t* nnz_out, void* stream) {
  CT_TRY(check_mode(mode, k));
  if (mode == CTSM_MODE_CONSISTENT)
    return ctsm_csr_count(ctx, g, angle_begin, angle_end, memory_budget_bytes, row_start_dev,
                          nnz_out, stream);
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  if ((uint64_t)g->n_x * g->n_y * g->n_z > 0xffffffffull)
    return fail(CTSM_ERR_TOO_LARGE, "grid exceeds 2^32 voxel columns");
  CT_TRY(check_shard(g, angle_begin, angle_end, 1));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = angle_end - angle_begin;
  const uint64_t rpa = (uint64_t)d.rows_per_angle;
  const uint64_t n_rows = rpa * n_sel;
  const uint64_t n_meas = rpa * (uint64_t)g->n_angles;
  {  // budget estimate from angle 0 (projector.cpp:155-169)
    CT_TRY(ray_rows(ctx, d, mode, k, 0, 1, st));
    CT_TRY(ensure(ctx, ctx->tmp_a, (rpa + 1) * sizeof(uint64_t)));
    CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes(rpa)));
    CT_CUDA(exclusive_scan_u32_u64((const unsigned*)ctx->counts.p, rpa, (uint64_t*)ctx->tmp_a.p,
                                   ctx->scan.p, st));
    uint64_t nnz0 = 0;
    CT_CUDA(cudaMemcpyAsync(&nnz0, (uint64_t*)ctx->tmp_a.p + rpa, sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, st));
    CT_TRY(check_status(ctx, st, "build_system_matrix"));
    const uint64_t est_nnz = nnz0 * (uint64_t)g->n_angles;
    const uint64_t est_bytes = est_nnz * (sizeof(uint32_t) + sizeof(double)) +
                               (n_meas + 1) * sizeof(uint64_t);
    if (est_bytes > memory_budget_bytes) {
      char msg[256];
      snprintf(msg, sizeof msg, "estimated %llu entries (%llu MiB) exceed the budget of %llu MiB",
               (unsigned long long)est_nnz, (unsigned long long)(est_bytes >> 20),
               (unsigned long long)(memory_budget_bytes >> 20));
      return fail(CTSM_ERR_OUT_OF_MEMORY, msg);
    }
  }
  CT_TRY(ray_rows(ctx, d, mode, k, angle_begin, n_sel, st));
  CT_TRY(ensure(ctx, ctx->scan, scan_scratch_bytes(n_rows)));
  CT_CUDA(exclusive_scan_u32_u64((const unsigned*)ctx->counts.p, n_rows, row_start_dev,
                                 ctx->scan.p, st));
  uint64_t nnz = 0;
  CT_CUDA(cudaMemcpyAsync(&nnz, row_start_dev + n_rows, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                          st));
  CT_TRY(check_status(ctx, st, "build_system_matrix"));
  if (angle_begin == 0 && angle_end == g->n_angles && nnz == 0)
    return fail(CTSM_ERR_ZERO_MATRIX, "system matrix has no entries");
  *nnz_out = nnz;
  return 0;
}

int ctsm_csr_fill_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int angle_begin,
                       int angle_end, const uint64_t* row_start_dev, uint32_t* col_dev,
                       double* val_dev, void* stream) {
  CT_TRY(check_mode(mode, k));
  if (mode == CTSM_MODE_CONSISTENT)
    return ctsm_csr_fill(ctx, g, angle_begin, angle_end, row_start_dev, col_dev, val_dev, stream);
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_shard(g, angle_begin, angle_end, 1));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = angle_end - angle_begin;
  const uint64_t n_rows = (uint64_t)d.rows_per_angle * n_sel;
  if (mode == CTSM_MODE_LINE || k == 1) {
    // rays traced straight into the caller's rows, then the stable column sort
    CT_TRY(ensure(ctx, ctx->angles, (size_t)(n_sel > 0 ? n_sel : 1) * ray_angle_bytes()));
    CT_CUDA(ray_angle_table(d, angle_begin, 1, n_sel, ctx->angles.p, st));
    CT_CUDA(ray_fill(d, ctx->angles.p, mode, k, n_rows, row_start_dev, col_dev, val_dev, st));
    CT_TRY(ensure(ctx, ctx->counts, (n_rows ? n_rows : 1) * sizeof(unsigned)));
    CT_TRY(ensure(ctx, ctx->longrows, (n_rows + 1) * sizeof(unsigned)));
    CT_CUDA(ray_sort_merge(n_rows, row_start_dev, (unsigned*)ctx->counts.p, col_dev, val_dev,
                           (unsigned*)ctx->longrows.p, (unsigned*)ctx->longrows.p + n_rows,
                           ctx->status, st));
  } else {
    CT_TRY(ray_rows(ctx, d, mode, k, angle_begin, n_sel, st));
    CT_CUDA(ray_compact(n_rows, (const uint64_t*)ctx->lraw_start.p, row_start_dev,
                        (const uint32_t*)ctx->lraw_col.p, (const double*)ctx->lraw_val.p, col_dev,
                        val_dev, st));
  }
  return check_status(ctx, st, "build_system_matrix");
}

int ctsm_fwd_mf_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int dtype,
                     int angle_begin, int angle_end, int angle_step, const void* x_dev,
                     void* y_dev, void* stream) {
  CT_TRY(check_mode(mode, k));
  if (mode == CTSM_MODE_CONSISTENT)
    return ctsm_fwd_mf(ctx, g, dtype, angle_begin, angle_end, angle_step, x_dev, y_dev, stream);
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_dtype(dtype));
  CT_TRY(check_shard(g, angle_begin, angle_end, angle_step));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = n_in_shard(angle_begin, angle_end, angle_step);
  CT_TRY(ensure(ctx, ctx->angles, (size_t)(n_sel > 0 ? n_sel : 1) * ray_angle_bytes()));
  CT_CUDA(ray_angle_table(d, angle_begin, angle_step, n_sel, ctx->angles.p, st));
  CT_CUDA(cudaMemsetAsync(ctx->n_upd, 0, sizeof(unsigned long long), st));
  CT_CUDA(ray_fwd_mf(d, dtype, ctx->angles.p, mode, k, angle_begin, angle_step, n_sel, x_dev,
                     y_dev, ctx->n_upd, ctx->status, st));
  CT_CUDA(cudaMemcpyAsync(ctx->h_upd, ctx->n_upd, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, st));
  CT_TRY(check_status(ctx, st, "forward_project_matrix_free"));
  ctx->last_updates = *ctx->h_upd;
  return 0;
}

int ctsm_bwd_mf_mode(ctsm_ctx* ctx, const ctsm_geometry* g, int mode, int k, int dtype,
                     int angle_begin, int angle_end, int angle_step, const void* y_dev,
                     void* x_dev, void* stream) {
  CT_TRY(check_mode(mode, k));
  if (mode == CTSM_MODE_CONSISTENT)
    return ctsm_bwd_mf(ctx, g, dtype, angle_begin, angle_end, angle_step, y_dev, x_dev, stream);
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_dtype(dtype));
  CT_TRY(check_shard(g, angle_begin, angle_end, angle_step));
  cudaStream_t st = (cudaStream_t)stream;
  const int n_sel = n_in_shard(angle_begin, angle_end, angle_step);
  const uint64_t n_meas = (uint64_t)d.rows_per_angle * g->n_angles;
  double my = 0.0;
  CT_TRY(fetch_max_abs(ctx, dtype, n_meas, y_dev, st, &my));
  if (!std::isfinite(my)) return fail(CTSM_ERR_NON_FINITE, "sinogram not finite");
  // fixed-point scale: a power of two with max |x_c| * scale < 2^61
  const double B = my * (double)n_sel * ray_colsum_bound(g);
  int e = 0;
  std::frexp(B, &e);
  const double scale = B > 0.0 ? std::ldexp(1.0, 61 - e) : 1.0;
  CT_TRY(ensure(ctx, ctx->angles, (size_t)(n_sel > 0 ? n_sel : 1) * ray_angle_bytes()));
  CT_CUDA(ray_angle_table(d, angle_begin, angle_step, n_sel, ctx->angles.p, st));
  CT_TRY(ensure(ctx, ctx->lacc, (size_t)d.n_vox * sizeof(unsigned long long)));
  CT_CUDA(ray_bwd_mf(d, dtype, ctx->angles.p, mode, k, angle_begin, angle_step, n_sel, y_dev,
                     (unsigned long long*)ctx->lacc.p, scale, x_dev, st));
  return check_status(ctx, st, "back_project_matrix_free");
}

// ---- K7/K8 ----------------------------------------------------------------
int ctsm_invert_nonzero(ctsm_ctx* ctx, int dtype, uint64_t n, void* v_dev, void* stream) {
  CT_TRY(set_device(ctx));
  CT_TRY(check_dtype(dtype));
  CT_CUDA(invert_nonzero(dtype, n, v_dev, (cudaStream_t)stream));
  return 0;
}

int ctsm_sirt_residual(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, int angle_begin,
                       int angle_end, int angle_step, const void* y_dev, const void* rinv_dev,
                       void* ax_inout_dev, void* stream) {
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_dtype(dtype));
  CT_TRY(check_shard(g, angle_begin, angle_end, angle_step));
  CT_CUDA(sirt_residual(d, dtype, angle_begin, angle_step,
                        n_in_shard(angle_begin, angle_end, angle_step), y_dev, rinv_dev,
                        ax_inout_dev, (cudaStream_t)stream));
  return 0;
}

int ctsm_sirt_update(ctsm_ctx* ctx, int dtype, uint64_t n, const void* cinv_dev,
                     const void* bp_dev, void* x_inout_dev, void* stream) {
  CT_TRY(set_device(ctx));
  CT_TRY(check_dtype(dtype));
  CT_CUDA(sirt_update(dtype, n, cinv_dev, bp_dev, x_inout_dev, (cudaStream_t)stream));
  return 0;
}

int ctsm_sirt(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, const void* y_dev,
              void* x_inout_dev, int iters, void* stream) {
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  CT_TRY(check_dtype(dtype));
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t nv = (uint64_t)d.n_vox;
  const uint64_t nm = (uint64_t)d.rows_per_angle * g->n_angles;
  const size_t es = dtype_size(dtype);
  CT_TRY(ensure(ctx, ctx->tmp_c, nm * es));  // R (inverse row sums)
  CT_TRY(ensure(ctx, ctx->tmp_d, nv * es));  // C (inverse column sums)
  CT_TRY(ensure(ctx, ctx->tmp_e, nm * es));  // A x / residual
  CT_TRY(ensure(ctx, ctx->tmp_f, nv * es));  // A^T r / ones
  const int n = g->n_angles;
  // R = 1 / (A 1)
  CT_CUDA(fill_value(dtype, nv, 1.0, ctx->tmp_f.p, st));
  CT_TRY(fwd_impl(ctx, g, dtype, 0, n, 1, ctx->tmp_f.p, ctx->tmp_c.p, st));
  CT_CUDA(invert_nonzero(dtype, nm, ctx->tmp_c.p, st));
  // C = 1 / (A^T 1)
  CT_CUDA(fill_value(dtype, nm, 1.0, ctx->tmp_e.p, st));
  CT_TRY(bwd_impl(ctx, g, dtype, 0, n, 1, ctx->tmp_e.p, ctx->tmp_d.p, st));
  CT_CUDA(invert_nonzero(dtype, nv, ctx->tmp_d.p, st));
  CT_TRY(check_status(ctx, st, "sirt"));
  for (int it = 0; it < iters; ++it) {
    CT_TRY(fwd_impl(ctx, g, dtype, 0, n, 1, x_inout_dev, ctx->tmp_e.p, st));
    CT_CUDA(sirt_residual(d, dtype, 0, 1, n, y_dev, ctx->tmp_c.p, ctx->tmp_e.p, st));
    CT_TRY(bwd_impl(ctx, g, dtype, 0, n, 1, ctx->tmp_e.p, ctx->tmp_f.p, st));
    CT_CUDA(sirt_update(dtype, nv, ctx->tmp_d.p, ctx->tmp_f.p, x_inout_dev, st));
  }
  return check_status(ctx, st, "sirt");
}

// ---- solvers ------------------------------------------
namespace {

struct OpRun {
  const ctsm_operator* op;
  uint64_t n_rows = 0, n_cols = 0;
  double mcol = 0.0;  // CSR: max column |sum| (fixed-point bound of W^T)
  double s = 1.0;     // operator scale
};

int op_prepare(ctsm_ctx* ctx, const ctsm_operator* op, cudaStream_t st, OpRun* r) {
  if (!op) return fail(CTSM_ERR_INVALID_SPEC, "null operator");
  r->op = op;
  if (op->kind == CTSM_OP_CSR) {
    if (op->scale != 1.0)
      return fail(CTSM_ERR_INVALID_SPEC, "CSR operators are scaled with ctsm_scale_values");
    r->n_rows = op->n_rows;
    r->n_cols = op->n_cols;
    uint64_t nnz = 0;
    if (r->n_rows > 0)
      CT_CUDA(cudaMemcpy(&nnz, op->row_start + r->n_rows, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (nnz == 0) return fail(CTSM_ERR_ZERO_MATRIX, "matrix has no entries");
    CT_TRY(ensure(ctx, ctx->tmp_a, r->n_cols * sizeof(double)));
    CT_CUDA(cudaMemsetAsync(ctx->tmp_a.p, 0, r->n_cols * sizeof(double), st));
    CT_CUDA(colsum_abs(r->n_rows, op->row_start, op->col, op->val, (double*)ctx->tmp_a.p, st));
    CT_TRY(fetch_max_abs(ctx, CTSM_F64, r->n_cols, ctx->tmp_a.p, st, &r->mcol));
    if (!std::isfinite(r->mcol)) return fail(CTSM_ERR_NON_FINITE, "matrix not finite");
  } else if (op->kind == CTSM_OP_MATRIX_FREE) {
    DevGeom d;
    CT_TRY(dev_geom(op->geom, &d));
    r->n_rows = (uint64_t)d.rows_per_angle * op->geom->n_angles;
    r->n_cols = (uint64_t)d.n_vox;
    r->s = op->scale;
    if (!std::isfinite(r->s)) return fail(CTSM_ERR_NON_FINITE, "operator scale must be finite");
  } else {
    return fail(CTSM_ERR_INVALID_SPEC, "unknown operator kind");
  }
  return 0;
}

// y = A x (unscaled)
int op_fwd(ctsm_ctx* ctx, const OpRun& r, const double* x, double* y, cudaStream_t st) {
  const ctsm_operator* op = r.op;
  if (op->kind == CTSM_OP_CSR) {
    CT_CUDA(spmv_csr(r.n_rows, op->row_start, op->col, op->val, x, y, ctx->status, st));
    return 0;
  }
  return fwd_impl(ctx, op->geom, CTSM_F64, 0, op->geom->n_angles, 1, x, y, st);
}

// x = A^T y (unscaled), deterministic
int op_bwd(ctsm_ctx* ctx, const OpRun& r, const double* y, double* x, cudaStream_t st) {
  const ctsm_operator* op = r.op;
  if (op->kind == CTSM_OP_CSR) {
    double my = 0.0;
    CT_TRY(fetch_max_abs(ctx, CTSM_F64, r.n_rows, y, st, &my));
    if (!std::isfinite(my)) return fail(CTSM_ERR_NON_FINITE, "back projection not finite");
    const double scale = csr_fixed_scale(r.mcol, my);
    if (!(scale > 0.0)) {
      CT_CUDA(cudaMemsetAsync(x, 0, r.n_cols * sizeof(double), st));
      return 0;
    }
    CT_TRY(ensure(ctx, ctx->tmp_b, r.n_cols * sizeof(unsigned long long)));
    if (op->col_start && op->trow && op->tval) {
      // the caller keeps a CSC transpose: gather (same integers, same bits)
      CT_CUDA(spmvt_csc_fixed(r.n_cols, op->col_start, op->trow, op->tval, y,
                              (unsigned long long*)ctx->tmp_b.p, scale, st));
    } else {
      CT_CUDA(cudaMemsetAsync(ctx->tmp_b.p, 0, r.n_cols * sizeof(unsigned long long), st));
      CT_CUDA(spmvt_csr_fixed(r.n_rows, op->row_start, op->col, op->val, y,
                              (unsigned long long*)ctx->tmp_b.p, scale, st));
    }
    CT_CUDA(fixed_to_double(r.n_cols, (const unsigned long long*)ctx->tmp_b.p, scale, x, st));
    return 0;
  }
  return bwd_impl(ctx, op->geom, CTSM_F64, 0, op->geom->n_angles, 1, y, x, st);
}

int read_scalars(ctsm_ctx* ctx, int n, double* out, cudaStream_t st) {
  CT_CUDA(cudaMemcpyAsync(out, ctx->sv_scal.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CT_CUDA(cudaStreamSynchronize(st));
  return 0;
}

}  // namespace

int ctsm_scale_values(ctsm_ctx* ctx, uint64_t nnz, double* val_dev, double factor, void* stream) {
  CT_TRY(set_device(ctx));
  if (!std::isfinite(factor)) return fail(CTSM_ERR_NON_FINITE, "scale factor must be finite");
  CT_CUDA(scale_in_place(nnz, val_dev, factor, (cudaStream_t)stream));
  return 0;
}

int ctsm_spectral_norm_power(ctsm_ctx* ctx, const ctsm_operator* op, int iters,
                             double* v_dev, double* norm_out, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  OpRun r;
  CT_TRY(op_prepare(ctx, op, st, &r));
  CT_TRY(ensure(ctx, ctx->sv_v, r.n_rows * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_h, r.n_cols * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_part, solver_partial_doubles() * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_scal, 4 * sizeof(double)));
  double* u = (double*)ctx->sv_h.p;
  double* y = (double*)ctx->sv_v.p;
  double* part = (double*)ctx->sv_part.p;
  double* lam = (double*)ctx->sv_scal.p;
  // v /= ||v|| (projector.cpp:268-271)
  CT_CUDA(norm2(r.n_cols, v_dev, 1.0, part, lam, st));
  CT_CUDA(normalize_by(r.n_cols, v_dev, 1.0, lam, v_dev, ctx->status, st));
  const double s2 = r.s * r.s;
  for (int it = 0; it < iters; ++it) {
    CT_TRY(op_fwd(ctx, r, v_dev, y, st));
    CT_TRY(op_bwd(ctx, r, y, u, st));
    // lam = ||W^T W v|| = s^2 ||A^T A v||; v = W^T W v / lam
    CT_CUDA(norm2(r.n_cols, u, s2, part, lam, st));
    CT_CUDA(normalize_by(r.n_cols, u, s2, lam, v_dev, ctx->status, st));
  }
  double h = 0.0;
  CT_TRY(read_scalars(ctx, 1, &h, st));
  const int s = check_status(ctx, st, "spectral_norm_power");
  if (s == CTSM_ERR_ZERO_MATRIX) return fail(s, "power iteration collapsed");
  if (s) return s;
  *norm_out = iters > 0 ? std::sqrt(h) : 0.0;
  return 0;
}

int ctsm_nag_tikhonov(ctsm_ctx* ctx, const ctsm_operator* op, const double* p_dev,
                      double lambda, int max_iter, double tol, double* u_dev,
                      double* trace_host, int* iterations, int* converged, void* stream) {
  CT_TRY(set_device(ctx));
  cudaStream_t st = (cudaStream_t)stream;
  if (!(lambda >= 0.0) || !(tol >= 0.0) || max_iter < 0)
    return fail(CTSM_ERR_INVALID_CONFIG, "solver options must be nonnegative");
  OpRun r;
  CT_TRY(op_prepare(ctx, op, st, &r));
  const uint64_t n = r.n_cols, nr = r.n_rows;
  CT_TRY(ensure(ctx, ctx->sv_up, n * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_h, n * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_hp, n * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_q, n * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_v, nr * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_part, solver_partial_doubles() * sizeof(double)));
  CT_TRY(ensure(ctx, ctx->sv_scal, 4 * sizeof(double)));
  double* up = (double*)ctx->sv_up.p;
  double* h = (double*)ctx->sv_h.p;
  double* hp = (double*)ctx->sv_hp.p;
  double* q = (double*)ctx->sv_q.p;
  double* v = (double*)ctx->sv_v.p;
  double* part = (double*)ctx->sv_part.p;
  double* scal = (double*)ctx->sv_scal.p;
  const double lam = lambda, L = 1.0 + lam, s = r.s, s2 = s * s;
  // q = W^T p (solver.cpp:28)
  CT_TRY(op_bwd(ctx, r, p_dev, q, st));
  if (s != 1.0) CT_CUDA(scale_in_place(n, q, s, st));
  CT_CUDA(cudaMemsetAsync(u_dev, 0, n * sizeof(double), st));
  CT_CUDA(cudaMemsetAsync(up, 0, n * sizeof(double), st));
  CT_CUDA(cudaMemsetAsync(h, 0, n * sizeof(double), st));
  CT_CUDA(cudaMemsetAsync(hp, 0, n * sizeof(double), st));
  double t = 1.0;
  int iters = 0, conv = 0;
  for (int it = 0; it < max_iter; ++it) {
    const double t_next = (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0;
    const double m = (t - 1.0) / t_next;
    CT_CUDA(nag_step(n, m, lam, L, u_dev, up, h, hp, q, st));
    t = t_next;
    // v = W u, h = W^T v (solver.cpp:52-53)
    CT_TRY(op_fwd(ctx, r, u_dev, v, st));
    CT_TRY(op_bwd(ctx, r, v, h, st));
    CT_CUDA(nag_grad_sq(n, s2, lam, h, u_dev, q, part, scal, st));
    double vals[3] = {0.0, 0.0, 0.0};
    if (trace_host) {
      CT_CUDA(nag_trace_sums(nr, n, s, v, p_dev, u_dev, part, scal + 1, st));
      CT_TRY(read_scalars(ctx, 3, vals, st));
    } else {
      CT_TRY(read_scalars(ctx, 1, vals, st));
    }
    CT_TRY(check_status(ctx, st, "nag_tikhonov"));
    const double grad_sq = vals[0];
    iters = it + 1;
    if (trace_host) {
      trace_host[3 * it] = (double)(it + 1);
      trace_host[3 * it + 1] = 0.5 * vals[1] + 0.5 * lam * vals[2];
      trace_host[3 * it + 2] = grad_sq;
    }
    if (!std::isfinite(grad_sq)) {
      if (iterations) *iterations = iters;
      return fail(CTSM_ERR_NON_FINITE, "solver iterate diverged");
    }
    if (grad_sq < tol) {
      conv = 1;
      break;
    }
  }
  if (iterations) *iterations = iters;
  if (converged) *converged = conv;
  return 0;
}

// ---- host-buffer entry points ------------------------------------------------
// The reference's value-semantics calls (projector.hpp:56-59 and the a16
// adjoint): host x / y in, host y / x out, copies and kernels on the
// context's own non-blocking stream. f64, and the fp32 overloads (SURVEY.md
// §8(b) "fp32 overloads") whose weights are still evaluated in FP64.
static int fwd_host(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, const void* x_host,
                    void* y_host) {
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  const size_t es = dtype == CTSM_F64 ? 8 : 4;
  const uint64_t nv = (uint64_t)d.n_vox, nm = (uint64_t)d.rows_per_angle * g->n_angles;
  CT_TRY(ensure(ctx, ctx->tmp_a, nv * es));
  CT_TRY(ensure(ctx, ctx->tmp_b, nm * es));
  cudaStream_t st;
  CT_TRY(host_stream(ctx, &st));
  CT_CUDA(cudaMemcpyAsync(ctx->tmp_a.p, x_host, nv * es, cudaMemcpyHostToDevice, st));
  CT_TRY(fwd_impl(ctx, g, dtype, 0, g->n_angles, 1, ctx->tmp_a.p, ctx->tmp_b.p, st));
  CT_CUDA(cudaMemcpyAsync(y_host, ctx->tmp_b.p, nm * es, cudaMemcpyDeviceToHost, st));
  CT_TRY(check_status(ctx, st, "forward_project_matrix_free"));
  ctx->last_updates = *ctx->h_upd;
  return 0;
}

static int bwd_host(ctsm_ctx* ctx, const ctsm_geometry* g, int dtype, const void* y_host,
                    void* x_host) {
  CT_TRY(set_device(ctx));
  DevGeom d;
  CT_TRY(dev_geom(g, &d));
  const size_t es = dtype == CTSM_F64 ? 8 : 4;
  const uint64_t nv = (uint64_t)d.n_vox, nm = (uint64_t)d.rows_per_angle * g->n_angles;
  CT_TRY(ensure(ctx, ctx->tmp_a, nv * es));
  CT_TRY(ensure(ctx, ctx->tmp_b, nm * es));
  cudaStream_t st;
  CT_TRY(host_stream(ctx, &st));
  CT_CUDA(cudaMemcpyAsync(ctx->tmp_b.p, y_host, nm * es, cudaMemcpyHostToDevice, st));
  CT_TRY(bwd_impl(ctx, g, dtype, 0, g->n_angles, 1, ctx->tmp_b.p, ctx->tmp_a.p, st));
  CT_CUDA(cudaMemcpyAsync(x_host, ctx->tmp_a.p, nv * es, cudaMemcpyDeviceToHost, st));
  return check_status(ctx, st, "back_project_matrix_free");
}

int ctsm_forward_project_matrix_free_host(ctsm_ctx* ctx, const ctsm_geometry* g,
                                          const double* x_host, double* y_host) {
  return fwd_host(ctx, g, CTSM_F64, x_host, y_host);
}

int ctsm_back_project_matrix_free_host(ctsm_ctx* ctx, const ctsm_geometry* g,
                                       const double* y_host, double* x_host) {
  return bwd_host(ctx, g, CTSM_F64, y_host, x_host);
}

int ctsm_forward_project_matrix_free_host_f32(ctsm_ctx* ctx, const ctsm_geometry* g,
                                              const float* x_host, float* y_host) {
  return fwd_host(ctx, g, CTSM_F32, x_host, y_host);
}

int ctsm_back_project_matrix_free_host_f32(ctsm_ctx* ctx, const ctsm_geometry* g,
                                           const float* y_host, float* x_host) {
  return bwd_host(ctx, g, CTSM_F32, y_host, x_host);
}

}  // extern "C"

extern "C" double ctsm_bench_dfma(int device) { return ctsmb::bench_dfma_tflops(device); }
