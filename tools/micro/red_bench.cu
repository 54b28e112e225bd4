// Microbenchmark: fp32 reductions of 32-byte (8-float) segments into a large
// L2-resident / HBM array from every lane, as the fp32 3D forward does.
//  A: two red.global.add.v4.f32 per segment (what fwd3d_sym_kernel issues)
//  B: one cp.reduce.async.bulk (TMA bulk reduction, 32 bytes) per segment from
//     a per-lane shared-memory slot
//  C: one red.global.add.v4.f32 per segment (half the data: lane-op rate)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a red_bench.cu -o red_bench
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(128) k(float* __restrict__ y, unsigned nseg, int iters, int stride_rows) {
  __shared__ __align__(128) float stage[2][128][8];
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  // a lane walks consecutive segments (rows) like a voxel chunk; lanes of a
  // warp are stride_rows apart; the start is pseudo-random per warp and trip
  unsigned seg = 0;
  float v = 1.0f + (float)(tid & 7);
  for (int i = 0; i < iters; ++i) {
    if ((i & 7) == 0) seg = (hash((tid >> 5) * 977u + (unsigned)i) + (threadIdx.x & 31) * stride_rows) % (nseg - 16);
    float* dst = y + (size_t)(seg + (i & 7)) * 8;
    if (MODE == 3 || MODE == 4) {
      // the forward's flush: two segments per lane and trip (a row and its z
      // mirror), far apart (3: rows r and N-1-r) or adjacent (4: a paired layout)
      float* d2 = MODE == 3 ? y + (size_t)(nseg - 1 - (seg + (i & 7))) * 8
                            : y + (size_t)((seg + (i & 7)) ^ 1u) * 8;
      float* d1 = MODE == 3 ? dst : y + (size_t)((seg + (i & 7)) & ~1u) * 8;
      if (MODE == 4) d2 = d1 + 8;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d1), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d1 + 4), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d2), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d2 + 4), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
    } else if (MODE == 0 || MODE == 2) {
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      if (MODE == 0)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
    } else {
      float* s = stage[i & 1][threadIdx.x];
      // the slot's previous bulk reduction (two trips ago) has been read
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      reinterpret_cast<float4*>(s)[0] = make_float4(v, v, v, v);
      reinterpret_cast<float4*>(s)[1] = make_float4(v, v, v, v);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 32;" ::"l"(dst), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    v += 0.5f;
  }
  if (MODE == 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  // 32-byte segments: 2^24 = 512 MB (default; mostly L2 misses), 2^21 = 64 MB (L2-resident)
  const unsigned nseg = 1u << (argc > 2 ? atoi(argv[2]) : 24);
  const int iters = argc > 1 ? atoi(argv[1]) : 4096;
  float* y;
  cudaMalloc(&y, (size_t)nseg * 32);
  cudaMemset(y, 0, (size_t)nseg * 32);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 4;
  for (int stride = 1; stride <= 5; stride += 4)
    for (int mode = 0; mode < 5; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<blocks, 128>>>(y, nseg, iters, stride);
        if (mode == 1) k<1><<<blocks, 128>>>(y, nseg, iters, stride);
        if (mode == 2) k<2><<<blocks, 128>>>(y, nseg, iters, stride);
        if (mode == 3) k<3><<<blocks, 128>>>(y, nseg, iters, 2 * stride);
        if (mode == 4) k<4><<<blocks, 128>>>(y, nseg, iters, 2 * stride);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 1) {
          const double segs = (double)blocks * 128 * iters * (mode >= 3 ? 2 : 1);
          printf("mode %d (%s) lane stride %d rows: %.3f ms, %.2f G segments/s, %.3f segments/clk/SM @1.9GHz  err=%s\n",
                 mode, mode == 0 ? "2 x red.v4" : mode == 1 ? "1 x bulk reduce 32 B" : mode == 2 ? "1 x red.v4 (half)" : mode == 3 ? "row + far mirror row (2 segments per trip)" : "row + adjacent mirror row (2 segments per trip)",
                 stride, ms, segs / ms * 1e-6, segs / (ms * 1e-3) / 148 / 1.9e9,
                 cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
  return 0;
}
