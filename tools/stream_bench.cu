// stream_bench.cu -- read-bandwidth calibration for the GQSA access pattern.
//
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
// Run:    tools/stream_bench            (prints one line per variant)
//
// Variants (all read every byte once, ~26 MB per launch like 14336x4096
// W4S50, rotating over copies > 2x L2):
//   ldg<D>:       each warp streams a contiguous range of 1824-B tiles with
//                 128-bit L1::no_allocate loads, D tiles in flight.
//   ldg<D>+pf:    same, plus one cp.async.bulk.prefetch.L2 of the range.
//   flat<U>:      grid-stride uint4 loads, U per thread in flight (classic).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg128(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

constexpr int kTile = 1824;

template <int D, bool PF>
__global__ void __launch_bounds__(256) tiles_kernel(const uint8_t* base, int num_tiles, int warps, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (gw >= warps) return;
  const int q = num_tiles / warps, r = num_tiles % warps;
  const int tb = gw * q + min(gw, r), te = tb + q + (gw < r);
  if (PF && lane == 0 && te > tb) {
    const uint8_t* a = base + (int64_t)tb * kTile;
    uint32_t left = (uint32_t)(te - tb) * kTile;
    while (left) {
      uint32_t n = min(left, 65536u);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
      a += n; left -= n;
    }
  }
  uint32_t acc = 0;
  uint4 buf[D][4];
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (tb + i < te) {
      const uint8_t* t = base + (int64_t)(tb + i) * kTile;
      buf[i][0] = ldg128(t + 32 + lane * 16);
      buf[i][1] = ldg128(t + 32 + 512 + lane * 16);
      buf[i][2] = ldg128(t + 1056 + lane * 16);
      buf[i][3] = ldg128(t);
    }
  for (int t0 = tb; t0 < te; t0 += D) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int t = t0 + i;
      if (t < te) {
#pragma unroll
        for (int k = 0; k < 4; ++k) acc ^= buf[i][k].x ^ buf[i][k].y ^ buf[i][k].z ^ buf[i][k].w;
        if (t + D < te) {
          const uint8_t* p = base + (int64_t)(t + D) * kTile;
          buf[i][0] = ldg128(p + 32 + lane * 16);
          buf[i][1] = ldg128(p + 32 + 512 + lane * 16);
          buf[i][2] = ldg128(p + 1056 + lane * 16);
          buf[i][3] = ldg128(p);
        }
      }
    }
  }
  if (acc == 0x12345678u) out[gw] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) flat_kernel(const uint4* base, int64_t n16, uint32_t* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (i + u * stride < n16) ? ldg128(base + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
float time_rot(F launch, int reps, int R) {
  // capture R launches (one per buffer copy) in a CUDA graph: no host launch gaps
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < R; ++i) launch(i, st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(a, st);
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(st);
  return ms * 1e3f / (reps * R);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tiles = 14336;  // ~26 MB
  const int64_t bytes = (int64_t)tiles * kTile;
  const int R = 12;
  uint8_t* buf;
  CK(cudaMalloc(&buf, bytes * R));
  CK(cudaMemset(buf, 1, bytes * R));
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int reps = 240;
  for (int ctas : {1, 2, 3, 4}) {
    const int grid = sms * ctas, warps = grid * 8;
#define RUN(D, PF)                                                                                 \
  {                                                                                                \
    float us = time_rot([&](int r, cudaStream_t st) { tiles_kernel<D, PF><<<grid, 256, 0, st>>>(buf + r * bytes, tiles, warps, out); }, 20, R); \
    printf("tiles ctas/SM=%d D=%d pf=%d: %.3f us  %.1f GB/s\n", ctas, D, (int)PF, us, bytes / us / 1e3); \
  }
    RUN(1, false) RUN(2, false) RUN(3, false) RUN(4, false) RUN(2, true) RUN(4, true)
  }
  for (int ctas : {2, 4, 8}) {
    const int grid = sms * ctas;
#define RUNF(U)                                                                                     \
  {                                                                                                 \
    float us = time_rot([&](int r, cudaStream_t st) { flat_kernel<U><<<grid, 256, 0, st>>>((const uint4*)(buf + r * bytes), bytes / 16, out); }, 20, R); \
    printf("flat ctas/SM=%d U=%d: %.3f us  %.1f GB/s\n", ctas, U, us, bytes / us / 1e3);          \
  }
    RUNF(2) RUNF(4) RUNF(8)
  }
  // big single stream for the asymptotic number
  for (int ctas : {2, 4, 8}) {
    const int64_t big = bytes * R;
    for (int U : {4, 8, 16}) {
      float us = 0;
      if (U == 4) us = time_rot([&](int, cudaStream_t st) { flat_kernel<4><<<sms * ctas, 256, 0, st>>>((const uint4*)buf, big / 16, out); }, 10, 1);
      if (U == 8) us = time_rot([&](int, cudaStream_t st) { flat_kernel<8><<<sms * ctas, 256, 0, st>>>((const uint4*)buf, big / 16, out); }, 10, 1);
      if (U == 16) us = time_rot([&](int, cudaStream_t st) { flat_kernel<16><<<sms * ctas, 256, 0, st>>>((const uint4*)buf, big / 16, out); }, 10, 1);
      printf("flat big %.0f MB ctas/SM=%d U=%d: %.1f us  %.1f GB/s\n", big / 1e6, ctas, U, us, big / us / 1e3);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
