// io.cu -- CSM1 / CTT1 containers for device-resident data (SURVEY.md §8(f)
// row 2; reference io.hpp:31-48, io.cpp:153-270).
//
// CSM1: "CSM1", u64 n_rows, n_cols, nnz, meta_len (little endian), the meta
// bytes, row_start[n_rows+1] u64, col[nnz] u64 (u32 in memory), val[nnz] f64.
// CTT1: "CTT1", u32 rank, u64 dims[rank], f64 payload.
//
// The writer streams a device CSR through two pinned staging buffers: while
// chunk i is written to the file, chunk i+1 is widened (u32 -> u64 columns,
// on the device) and copied down, so a C2-sized matrix (4.6e9 entries, a
// 74 GB file) never needs a host copy of the matrix. The reader validates
// exactly what the reference's read_matrix validates (magic, TooLarge column
// count, row offsets start at 0 / end at nnz / never decrease, columns in
// range) and streams the arrays up the same way (column range checked and
// narrowed on the device).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ctsm_b200.h"
#include "kernels.h"

namespace ctsmb {
namespace {

constexpr size_t kChunkBytes = 64u << 20;  // per staging buffer

__global__ void widen_kernel(uint64_t n, const uint32_t* in, uint64_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void narrow_kernel(uint64_t n, const uint64_t* in, uint64_t n_cols, uint32_t* out,
                              int* bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = in[i];
    if (c >= n_cols) atomicExch(bad, 1);
    out[i] = (uint32_t)c;
  }
}

unsigned io_grid(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return (unsigned)(b == 0 ? 1 : (b < 148ull * 16 ? b : 148ull * 16));
}

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool ok = false;
  Pinned() {
    ok = cudaMallocHost(&p[0], kChunkBytes) == cudaSuccess &&
         cudaMallocHost(&p[1], kChunkBytes) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) == cudaSuccess;
  }
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (p[i]) cudaFreeHost(p[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
};

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

int io_fail(const std::string& msg) { return set_error(CTSM_ERR_IO_FAILURE, msg); }

// Streams n elements of `elem` bytes from device memory to the file, through
// the two pinned buffers. If widen32 is set, `dev` holds u32 values written
// as u64 (widened on the device into `scratch`, kChunkBytes).
int stream_down(FILE* f, const std::string& path, const void* dev, uint64_t n, size_t elem,
                bool widen32, void* scratch, Pinned& pin, cudaStream_t st) {
  const size_t out_elem = widen32 ? 8 : elem;
  const uint64_t per = kChunkBytes / out_elem;
  const uint64_t n_chunks = (n + per - 1) / per;
  auto issue = [&](uint64_t c) -> cudaError_t {
    const uint64_t i0 = c * per, m = (n - i0) < per ? (n - i0) : per;
    const int b = (int)(c & 1);
    const void* src = (const char*)dev + i0 * elem;
    if (widen32) {
      widen_kernel<<<io_grid(m), 256, 0, st>>>(m, (const uint32_t*)src, (uint64_t*)scratch);
      count_launch();
      src = scratch;
    }
    cudaError_t e = cudaMemcpyAsync(pin.p[b], src, m * out_elem, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaEventRecord(pin.ev[b], st);
    return e;
  };
  if (n_chunks == 0) return 0;
  if (issue(0) != cudaSuccess) return set_error(CTSM_ERR_CUDA, "device to host copy failed");
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const int b = (int)(c & 1);
    if (cudaEventSynchronize(pin.ev[b]) != cudaSuccess)
      return set_error(CTSM_ERR_CUDA, "device to host copy failed");
    // the scratch buffer is free once chunk c has landed: start chunk c+1
    if (c + 1 < n_chunks && issue(c + 1) != cudaSuccess)
      return set_error(CTSM_ERR_CUDA, "device to host copy failed");
    const uint64_t i0 = c * per, m = (n - i0) < per ? (n - i0) : per;
    if (std::fwrite(pin.p[b], out_elem, m, f) != m) return io_fail("write failed for " + path);
  }
  return 0;
}

// Streams n elements from the file up to device memory. narrow: the file holds
// u64 columns checked against n_cols and stored as u32.
int stream_up(FILE* f, const std::string& path, void* dev, uint64_t n, size_t elem, bool narrow,
              uint64_t n_cols, void* scratch, int* bad_dev, Pinned& pin, cudaStream_t st) {
  const size_t in_elem = narrow ? 8 : elem;
  const uint64_t per = kChunkBytes / in_elem;
  for (uint64_t i0 = 0, c = 0; i0 < n; i0 += per, ++c) {
    const uint64_t m = (n - i0) < per ? (n - i0) : per;
    const int b = (int)(c & 1);
    // buffer b was last read by the copy of chunk c-2: wait for it
    if (c >= 2 && cudaEventSynchronize(pin.ev[b]) != cudaSuccess)
      return set_error(CTSM_ERR_CUDA, "host to device copy failed");
    if (std::fread(pin.p[b], in_elem, m, f) != m) return io_fail("read failed for " + path);
    void* dst = narrow ? scratch : (char*)dev + i0 * elem;
    cudaError_t e = cudaMemcpyAsync(dst, pin.p[b], m * in_elem, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && narrow) {
      narrow_kernel<<<io_grid(m), 256, 0, st>>>(m, (const uint64_t*)scratch, n_cols,
                                                (uint32_t*)dev + i0, bad_dev);
      count_launch();
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(pin.ev[b], st);
    if (e != cudaSuccess) return set_error(CTSM_ERR_CUDA, "host to device copy failed");
    // narrow reuses one scratch buffer: finish this chunk before the next one
    if (narrow && cudaEventSynchronize(pin.ev[b]) != cudaSuccess)
      return set_error(CTSM_ERR_CUDA, "host to device copy failed");
  }
  if (cudaStreamSynchronize(st) != cudaSuccess)
    return set_error(CTSM_ERR_CUDA, "host to device copy failed");
  return 0;
}

}  // namespace
}  // namespace ctsmb

using namespace ctsmb;

extern "C" {

int ctsm_write_csm1_device(ctsm_ctx* ctx, const char* path, uint64_t n_rows, uint64_t n_cols,
                           const uint64_t* row_start_dev, const uint32_t* col_dev,
                           const double* val_dev, const char* meta, uint64_t meta_len,
                           void* stream) {
  if (int e = select_device(ctx)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t nnz = 0;
  if (cudaMemcpy(&nnz, row_start_dev + n_rows, sizeof(uint64_t), cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return set_error(CTSM_ERR_CUDA, "cannot read the row offsets");
  File out(path, "wb");
  if (!out.f) return io_fail(std::string("cannot open ") + path + " for writing");
  const uint64_t hdr[4] = {n_rows, n_cols, nnz, meta_len};
  if (std::fwrite("CSM1", 1, 4, out.f) != 4 || std::fwrite(hdr, 8, 4, out.f) != 4 ||
      (meta_len && std::fwrite(meta, 1, meta_len, out.f) != meta_len))
    return io_fail(std::string("write failed for ") + path);
  Pinned pin;
  if (!pin.ok) return set_error(CTSM_ERR_OUT_OF_MEMORY, "pinned staging allocation failed");
  void* scratch = nullptr;
  if (cudaMalloc(&scratch, kChunkBytes) != cudaSuccess)
    return set_error(CTSM_ERR_OUT_OF_MEMORY, "device staging allocation failed");
  int s = stream_down(out.f, path, row_start_dev, n_rows + 1, 8, false, nullptr, pin, st);
  if (!s) s = stream_down(out.f, path, col_dev, nnz, 4, true, scratch, pin, st);
  if (!s) s = stream_down(out.f, path, val_dev, nnz, 8, false, nullptr, pin, st);
  cudaStreamSynchronize(st);
  cudaFree(scratch);
  if (s) return s;
  if (std::fflush(out.f) != 0) return io_fail(std::string("write failed for ") + path);
  return 0;
}

int ctsm_csm1_header(const char* path, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz,
                     uint64_t* meta_len) {
  File in(path, "rb");
  if (!in.f) return io_fail(std::string("cannot open ") + path);
  char magic[4] = {};
  if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, "CSM1", 4) != 0)
    return io_fail(std::string(path) + " is not a CSM1 matrix file");
  uint64_t hdr[4];
  if (std::fread(hdr, 8, 4, in.f) != 4) return io_fail(std::string("read failed for ") + path);
  if (hdr[1] > 0xffffffffull)
    return set_error(CTSM_ERR_TOO_LARGE, "matrix has too many columns for this build");
  *n_rows = hdr[0];
  *n_cols = hdr[1];
  *nnz = hdr[2];
  *meta_len = hdr[3];
  return 0;
}

int ctsm_read_csm1_device(ctsm_ctx* ctx, const char* path, uint64_t* row_start_dev,
                          uint32_t* col_dev, double* val_dev, char* meta_out, void* stream) {
  if (int e = select_device(ctx)) return e;
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t n_rows = 0, n_cols = 0, nnz = 0, meta_len = 0;
  int s = ctsm_csm1_header(path, &n_rows, &n_cols, &nnz, &meta_len);
  if (s) return s;
  File in(path, "rb");
  if (!in.f || std::fseek(in.f, 36, SEEK_SET) != 0)
    return io_fail(std::string("cannot open ") + path);
  std::string meta(meta_len, '\0');
  if (meta_len && std::fread(&meta[0], 1, meta_len, in.f) != meta_len)
    return io_fail(std::string("read failed for ") + path);
  if (meta_out && meta_len) std::memcpy(meta_out, meta.data(), meta_len);
  // row offsets: validated on the host (they pass through the staging buffers)
  std::vector<uint64_t> rs(n_rows + 1);
  if (std::fread(rs.data(), 8, n_rows + 1, in.f) != n_rows + 1)
    return io_fail(std::string("read failed for ") + path);
  if (rs[0] != 0 || rs[n_rows] != nnz)
    return io_fail(std::string(path) + " has inconsistent row offsets");
  for (uint64_t r = 0; r < n_rows; ++r)
    if (rs[r + 1] < rs[r]) return io_fail(std::string(path) + " has decreasing row offsets");
  if (cudaMemcpyAsync(row_start_dev, rs.data(), (n_rows + 1) * 8, cudaMemcpyHostToDevice, st) !=
      cudaSuccess)
    return set_error(CTSM_ERR_CUDA, "host to device copy failed");
  Pinned pin;
  if (!pin.ok) return set_error(CTSM_ERR_OUT_OF_MEMORY, "pinned staging allocation failed");
  void* scratch = nullptr;
  int* bad = nullptr;
  if (cudaMalloc(&scratch, kChunkBytes) != cudaSuccess || cudaMalloc(&bad, sizeof(int)) != cudaSuccess) {
    if (scratch) cudaFree(scratch);
    return set_error(CTSM_ERR_OUT_OF_MEMORY, "device staging allocation failed");
  }
  cudaMemsetAsync(bad, 0, sizeof(int), st);
  s = stream_up(in.f, path, col_dev, nnz, 4, true, n_cols, scratch, bad, pin, st);
  if (!s) s = stream_up(in.f, path, val_dev, nnz, 8, false, 0, nullptr, nullptr, pin, st);
  int h_bad = 0;
  cudaStreamSynchronize(st);
  cudaMemcpy(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(scratch);
  cudaFree(bad);
  if (s) return s;
  if (h_bad) return io_fail(std::string(path) + " has a column index out of range");
  return 0;
}

int ctsm_write_ctt1(const char* path, const uint64_t* dims, int rank, const double* data_host) {
  if (rank < 1 || rank > 8)
    return set_error(CTSM_ERR_INVALID_SPEC, "tensor rank must be between 1 and 8");
  uint64_t count = 1;
  for (int i = 0; i < rank; ++i) count *= dims[i];
  File out(path, "wb");
  if (!out.f) return io_fail(std::string("cannot open ") + path + " for writing");
  const uint32_t r = (uint32_t)rank;
  if (std::fwrite("CTT1", 1, 4, out.f) != 4 || std::fwrite(&r, 4, 1, out.f) != 1 ||
      std::fwrite(dims, 8, (size_t)rank, out.f) != (size_t)rank ||
      std::fwrite(data_host, 8, count, out.f) != count)
    return io_fail(std::string("write failed for ") + path);
  return 0;
}

int ctsm_ctt1_header(const char* path, uint64_t* dims_out, int* rank_out) {
  File in(path, "rb");
  if (!in.f) return io_fail(std::string("cannot open ") + path);
  char magic[4] = {};
  if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, "CTT1", 4) != 0)
    return io_fail(std::string(path) + " is not a CTT1 tensor file");
  uint32_t rank = 0;
  if (std::fread(&rank, 4, 1, in.f) != 1) return io_fail(std::string("read failed for ") + path);
  if (rank == 0 || rank > 8) return io_fail(std::string(path) + " has an unreasonable tensor rank");
  uint64_t count = 1;
  for (uint32_t i = 0; i < rank; ++i) {
    if (std::fread(&dims_out[i], 8, 1, in.f) != 1)
      return io_fail(std::string("read failed for ") + path);
    count *= dims_out[i];
  }
  if (count > (1ull << 33)) return set_error(CTSM_ERR_TOO_LARGE, std::string(path) + " tensor is too large to load");
  *rank_out = (int)rank;
  return 0;
}

int ctsm_read_ctt1(const char* path, double* data_host, uint64_t count) {
  uint64_t dims[8];
  int rank = 0;
  int s = ctsm_ctt1_header(path, dims, &rank);
  if (s) return s;
  uint64_t n = 1;
  for (int i = 0; i < rank; ++i) n *= dims[i];
  if (n != count) return set_error(CTSM_ERR_DIMENSION_MISMATCH, "tensor size does not match the buffer");
  File in(path, "rb");
  if (!in.f || std::fseek(in.f, 8 + 8L * rank, SEEK_SET) != 0)
    return io_fail(std::string("cannot open ") + path);
  if (std::fread(data_host, 8, n, in.f) != n) return io_fail(std::string("read failed for ") + path);
  return 0;
}

}  // extern "C"
