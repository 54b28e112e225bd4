// multi.cu -- multi-GPU context of the C-ABI: one
// process drives n devices, each with its own ctsm_ctx and stream. Angles are
// sharded by orbits (symmetric scans) or strided; A x needs no communication,
// A^T y and SIRT sum the partial volumes with ncclAllReduce over the devices'
// communicators (NVLink / NVSwitch). NCCL is bound at run time (dlopen of
// libnccl.so.2: the copy torch has already loaded, or the system one), so the
// library loads on machines without NCCL and single-device use never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ctsm_b200.h"
#include "kernels.h"

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  bool load(std::string* why) {
    if (lib) return true;
    lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      *why = std::string("libnccl.so.2 not found: ") + dlerror();
      return false;
    }
#define BIND(field, sym)                                                       \
  field = reinterpret_cast<decltype(field)>(dlsym(lib, sym));                   \
  if (!field) {                                                                \
    *why = std::string("NCCL symbol missing: ") + sym;                         \
    return false;                                                              \
  }
    BIND(CommInitAll, "ncclCommInitAll")
    BIND(CommDestroy, "ncclCommDestroy")
    BIND(AllReduce, "ncclAllReduce")
    BIND(GroupStart, "ncclGroupStart")
    BIND(GroupEnd, "ncclGroupEnd")
    BIND(GetErrorString, "ncclGetErrorString")
    BIND(GetVersion, "ncclGetVersion")
#undef BIND
    return true;
  }
};

struct DevSlot {
  int device = 0;
  ctsm_ctx* ctx = nullptr;
  cudaStream_t st = nullptr;
  ncclComm_t comm = nullptr;
  void* x = nullptr;   // volume
  void* y = nullptr;   // sinogram
  void* r = nullptr;   // SIRT: R (rows), then residual input
  void* c = nullptr;   // SIRT: C (volume)
  void* bp = nullptr;  // partial / summed back-projection
  size_t xn = 0, yn = 0, rn = 0, cn = 0, bpn = 0;
  std::vector<int> angles;  // the shard's angles (ascending)
  int orbits = 0;
  int status = 0;
  std::string err;
};

int grow(void** p, size_t* have, size_t bytes) {
  if (*have >= bytes && *p) return 0;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  if (cudaMalloc(p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return ctsmb::set_error(CTSM_ERR_OUT_OF_MEMORY, "device allocation failed");
  }
  *have = bytes;
  return 0;
}

}  // namespace

struct ctsm_multi {
  std::vector<DevSlot> dev;
  NcclApi nccl;
  bool have_comms = false;
};

namespace {

size_t esize(int dtype) { return dtype == CTSM_F64 ? 8 : 4; }

// Runs fn(slot index) on one host thread per device and returns the first
// failure (the messages are thread-local in the C-ABI, so they are carried).
template <class F>
int on_all(ctsm_multi* m, F fn) {
  const int n = (int)m->dev.size();
  std::vector<std::thread> th;
  for (int i = 0; i < n; ++i)
    th.emplace_back([m, i, &fn] {
      DevSlot& d = m->dev[i];
      cudaSetDevice(d.device);
      d.status = fn(i);
      if (d.status) d.err = ctsm_last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < n; ++i)
    if (m->dev[i].status) {
      const std::string& e = m->dev[i].err;
      const size_t pos = e.find(": ");
      return ctsmb::set_error(m->dev[i].status, pos == std::string::npos ? e : e.substr(pos + 2));
    }
  return 0;
}

int shard(ctsm_multi* m, const ctsm_geometry* g) {
  const int n = (int)m->dev.size();
  for (int i = 0; i < n; ++i) {
    DevSlot& d = m->dev[i];
    d.angles.assign((size_t)g->n_angles, 0);
    int cnt = 0;
    const int s = ctsm_shard_angles(g, i, n, d.angles.data(), &cnt, &d.orbits);
    if (s) return s;
    d.angles.resize((size_t)cnt);
  }
  return 0;
}

// Local forward / backward of slot i on its shard (device-resident operands).
int fwd_local(ctsm_multi* m, int i, const ctsm_geometry* g, int dtype, const void* x, void* y) {
  DevSlot& d = m->dev[i];
  const int n = (int)m->dev.size();
  if (d.orbits) return ctsm_fwd_mf_orbits(d.ctx, g, dtype, i, n, x, y, d.st);
  return ctsm_fwd_mf(d.ctx, g, dtype, i, g->n_angles, n, x, y, d.st);
}
int bwd_local(ctsm_multi* m, int i, const ctsm_geometry* g, int dtype, const void* y, void* x) {
  DevSlot& d = m->dev[i];
  const int n = (int)m->dev.size();
  if (d.orbits) return ctsm_bwd_mf_orbits(d.ctx, g, dtype, i, n, y, x, d.st);
  return ctsm_bwd_mf(d.ctx, g, dtype, i, g->n_angles, n, y, x, d.st);
}

// Sum of the devices' buffers (count elements each), in place on every device.
int all_reduce(ctsm_multi* m, int dtype, size_t count, void* DevSlot::*buf) {
  const int n = (int)m->dev.size();
  if (n == 1 && !m->have_comms) return 0;
  const ncclDataType_t ty = dtype == CTSM_F64 ? ncclDouble : ncclFloat;
  ncclResult_t r = m->nccl.GroupStart();
  for (int i = 0; i < n && r == ncclSuccess; ++i) {
    DevSlot& d = m->dev[i];
    r = m->nccl.AllReduce(d.*buf, d.*buf, count, ty, ncclSum, d.comm, d.st);
  }
  const ncclResult_t r2 = m->nccl.GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess)
    return ctsmb::set_error(CTSM_ERR_CUDA, std::string("ncclAllReduce: ") + m->nccl.GetErrorString(r));
  for (int i = 0; i < n; ++i) {
    cudaSetDevice(m->dev[i].device);
    if (cudaStreamSynchronize(m->dev[i].st) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "stream synchronisation after the all-reduce failed");
  }
  return 0;
}

int check_geometry(const ctsm_geometry* g, int dtype) {
  const int s = ctsm_validate_geometry(g);
  if (s) return s;
  if (dtype != CTSM_F64 && dtype != CTSM_F32)
    return ctsmb::set_error(CTSM_ERR_INVALID_SPEC, "unknown dtype");
  return 0;
}

}  // namespace

extern "C" {

int ctsm_multi_create(const int* devices, int n, ctsm_multi** out) {
  if (!out || !devices || n <= 0)
    return ctsmb::set_error(CTSM_ERR_INVALID_SPEC, "device list must hold at least one device");
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j])
        return ctsmb::set_error(CTSM_ERR_INVALID_SPEC, "a device is listed twice");
  ctsm_multi* m = new ctsm_multi();
  m->dev.resize((size_t)n);
  for (int i = 0; i < n; ++i) {
    DevSlot& d = m->dev[i];
    d.device = devices[i];
    const int s = ctsm_create(devices[i], &d.ctx);
    if (s) {
      ctsm_multi_destroy(m);
      return s;
    }
    cudaSetDevice(d.device);
    if (cudaStreamCreateWithFlags(&d.st, cudaStreamNonBlocking) != cudaSuccess) {
      ctsm_multi_destroy(m);
      return ctsmb::set_error(CTSM_ERR_CUDA, "stream creation failed");
    }
  }
  if (n > 1 || getenv("CTSM_MULTI_FORCE_NCCL")) {
    std::string why;
    if (!m->nccl.load(&why)) {
      ctsm_multi_destroy(m);
      return ctsmb::set_error(CTSM_ERR_CUDA, why);
    }
    std::vector<ncclComm_t> comms((size_t)n);
    const ncclResult_t r = m->nccl.CommInitAll(comms.data(), n, devices);
    if (r != ncclSuccess) {
      ctsm_multi_destroy(m);
      return ctsmb::set_error(CTSM_ERR_CUDA,
                              std::string("ncclCommInitAll: ") + m->nccl.GetErrorString(r));
    }
    for (int i = 0; i < n; ++i) m->dev[i].comm = comms[i];
    m->have_comms = true;
  }
  *out = m;
  return 0;
}

int ctsm_multi_destroy(ctsm_multi* m) {
  if (!m) return 0;
  for (DevSlot& d : m->dev) {
    if (!d.ctx) continue;  // slot never came up (e.g. no such device): nothing to release
    cudaSetDevice(d.device);
    if (d.comm && m->nccl.CommDestroy) m->nccl.CommDestroy(d.comm);
    void* bufs[] = {d.x, d.y, d.r, d.c, d.bp};
    for (void* b : bufs)
      if (b) cudaFree(b);
    if (d.st) cudaStreamDestroy(d.st);
    if (d.ctx) ctsm_destroy(d.ctx);
  }
  delete m;
  return 0;
}

int ctsm_multi_size(const ctsm_multi* m) { return m ? (int)m->dev.size() : 0; }

int ctsm_multi_nccl_version(const ctsm_multi* m) {
  int v = 0;
  if (m && m->have_comms && m->nccl.GetVersion) m->nccl.GetVersion(&v);
  return v;
}

// A x over all angles: every device projects its shard from its copy of x and
// its rows go straight to the host sinogram. No communication.
int ctsm_multi_forward_project_matrix_free_host(ctsm_multi* m, const ctsm_geometry* g, int dtype,
                                                const void* x_host, void* y_host) {
  if (!m) return ctsmb::set_error(CTSM_ERR_INVALID_SPEC, "null context");
  int s = check_geometry(g, dtype);
  if (s) return s;
  if ((s = shard(m, g))) return s;
  const size_t es = esize(dtype);
  const size_t nv = (size_t)g->n_x * g->n_y * g->n_z;
  const size_t rpa = (size_t)g->n_det_y * g->n_det_z;
  const size_t nm = rpa * (size_t)g->n_angles;
  return on_all(m, [&](int i) -> int {
    DevSlot& d = m->dev[i];
    int e;
    if ((e = grow(&d.x, &d.xn, nv * es))) return e;
    if ((e = grow(&d.y, &d.yn, nm * es))) return e;
    if (cudaMemcpyAsync(d.x, x_host, nv * es, cudaMemcpyHostToDevice, d.st) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "host to device copy failed");
    if ((e = fwd_local(m, i, g, dtype, d.x, d.y))) return e;
    for (int a : d.angles)
      if (cudaMemcpyAsync((char*)y_host + (size_t)a * rpa * es, (char*)d.y + (size_t)a * rpa * es,
                          rpa * es, cudaMemcpyDeviceToHost, d.st) != cudaSuccess)
        return ctsmb::set_error(CTSM_ERR_CUDA, "device to host copy failed");
    if (cudaStreamSynchronize(d.st) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "stream synchronisation failed");
    return 0;
  });
}

// A^T y: local back-projections of the shards, one all-reduce, result from
// device 0.
int ctsm_multi_back_project_matrix_free_host(ctsm_multi* m, const ctsm_geometry* g, int dtype,
                                             const void* y_host, void* x_host) {
  if (!m) return ctsmb::set_error(CTSM_ERR_INVALID_SPEC, "null context");
  int s = check_geometry(g, dtype);
  if (s) return s;
  if ((s = shard(m, g))) return s;
  const size_t es = esize(dtype);
  const size_t nv = (size_t)g->n_x * g->n_y * g->n_z;
  const size_t rpa = (size_t)g->n_det_y * g->n_det_z;
  const size_t nm = rpa * (size_t)g->n_angles;
  s = on_all(m, [&](int i) -> int {
    DevSlot& d = m->dev[i];
    int e;
    if ((e = grow(&d.y, &d.yn, nm * es))) return e;
    if ((e = grow(&d.bp, &d.bpn, nv * es))) return e;
    for (int a : d.angles)  // only the shard's rows are read
      if (cudaMemcpyAsync((char*)d.y + (size_t)a * rpa * es, (const char*)y_host + (size_t)a * rpa * es,
                          rpa * es, cudaMemcpyHostToDevice, d.st) != cudaSuccess)
        return ctsmb::set_error(CTSM_ERR_CUDA, "host to device copy failed");
    return bwd_local(m, i, g, dtype, d.y, d.bp);
  });
  if (s) return s;
  if ((s = all_reduce(m, dtype, nv, &DevSlot::bp))) return s;
  cudaSetDevice(m->dev[0].device);
  if (cudaMemcpy(x_host, m->dev[0].bp, nv * es, cudaMemcpyDeviceToHost) != cudaSuccess)
    return ctsmb::set_error(CTSM_ERR_CUDA, "device to host copy failed");
  return 0;
}

// SIRT (BASELINE.json configs[4]): x replicated, rows sharded; one all-reduce
// for C = 1 / (A^T 1) and one per iteration.
int ctsm_multi_sirt_host(ctsm_multi* m, const ctsm_geometry* g, int dtype, const void* y_host,
                         void* x_inout_host, int iters) {
  if (!m) return ctsmb::set_error(CTSM_ERR_INVALID_SPEC, "null context");
  int s = check_geometry(g, dtype);
  if (s) return s;
  if (iters < 0) return ctsmb::set_error(CTSM_ERR_INVALID_CONFIG, "iters must be >= 0");
  if ((s = shard(m, g))) return s;
  const size_t es = esize(dtype);
  const size_t nv = (size_t)g->n_x * g->n_y * g->n_z;
  const size_t rpa = (size_t)g->n_det_y * g->n_det_z;
  const size_t nm = rpa * (size_t)g->n_angles;
  // setup: x, y rows, R = 1 / (A 1) on the shard's rows (0 elsewhere), A^T 1
  s = on_all(m, [&](int i) -> int {
    DevSlot& d = m->dev[i];
    int e;
    if ((e = grow(&d.x, &d.xn, nv * es))) return e;
    if ((e = grow(&d.y, &d.yn, nm * es))) return e;
    if ((e = grow(&d.r, &d.rn, 2 * nm * es))) return e;  // R, then the A x / residual rows
    if ((e = grow(&d.c, &d.cn, nv * es))) return e;
    if ((e = grow(&d.bp, &d.bpn, nv * es))) return e;
    char* R = (char*)d.r;
    char* ax = R + nm * es;
    if (cudaMemsetAsync(d.y, 0, nm * es, d.st) != cudaSuccess ||
        cudaMemsetAsync(R, 0, 2 * nm * es, d.st) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "memset failed");
    for (int a : d.angles)
      if (cudaMemcpyAsync((char*)d.y + (size_t)a * rpa * es, (const char*)y_host + (size_t)a * rpa * es,
                          rpa * es, cudaMemcpyHostToDevice, d.st) != cudaSuccess)
        return ctsmb::set_error(CTSM_ERR_CUDA, "host to device copy failed");
    if ((e = ctsmb::fill_value(dtype, nv, 1.0, d.x, d.st)) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "fill failed");
    if ((e = fwd_local(m, i, g, dtype, d.x, R))) return e;
    if ((e = ctsm_invert_nonzero(d.ctx, dtype, nm, R, d.st))) return e;
    // A^T 1 over the shard: ones on the shard's rows only matter
    if ((e = ctsmb::fill_value(dtype, nm, 1.0, ax, d.st)) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "fill failed");
    if ((e = bwd_local(m, i, g, dtype, ax, d.c))) return e;
    if (cudaMemsetAsync(ax, 0, nm * es, d.st) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "memset failed");
    if (cudaMemcpyAsync(d.x, x_inout_host, nv * es, cudaMemcpyHostToDevice, d.st) != cudaSuccess)
      return ctsmb::set_error(CTSM_ERR_CUDA, "host to device copy failed");
    return cudaStreamSynchronize(d.st) == cudaSuccess
               ? 0
               : ctsmb::set_error(CTSM_ERR_CUDA, "stream synchronisation failed");
  });
  if (s) return s;
  if ((s = all_reduce(m, dtype, nv, &DevSlot::c))) return s;
  s = on_all(m, [&](int i) -> int {
    DevSlot& d = m->dev[i];
    return ctsm_invert_nonzero(d.ctx, dtype, nv, d.c, d.st);
  });
  if (s) return s;
  for (int it = 0; it < iters; ++it) {
    s = on_all(m, [&](int i) -> int {
      DevSlot& d = m->dev[i];
      char* R = (char*)d.r;
      char* ax = R + nm * es;
      int e;
      if ((e = fwd_local(m, i, g, dtype, d.x, ax))) return e;
      // ax <- R (y - A x): rows of other shards stay 0 (R is 0 there)
      if ((e = ctsm_sirt_residual(d.ctx, g, dtype, 0, g->n_angles, 1, d.y, R, ax, d.st))) return e;
      return bwd_local(m, i, g, dtype, ax, d.bp);
    });
    if (s) return s;
    if ((s = all_reduce(m, dtype, nv, &DevSlot::bp))) return s;
    s = on_all(m, [&](int i) -> int {
      DevSlot& d = m->dev[i];
      const int e = ctsm_sirt_update(d.ctx, dtype, nv, d.c, d.bp, d.x, d.st);
      if (e) return e;
      return cudaStreamSynchronize(d.st) == cudaSuccess
                 ? 0
                 : ctsmb::set_error(CTSM_ERR_CUDA, "stream synchronisation failed");
    });
    if (s) return s;
  }
  cudaSetDevice(m->dev[0].device);
  if (cudaMemcpy(x_inout_host, m->dev[0].x, nv * es, cudaMemcpyDeviceToHost) != cudaSuccess)
    return ctsmb::set_error(CTSM_ERR_CUDA, "device to host copy failed");
  return 0;
}

}  // extern "C"
