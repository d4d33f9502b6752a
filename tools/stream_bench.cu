// stream_bench.cu -- read-only bandwidth calibration for the GQSA access pattern
// (the third roofline denominator of SURVEY §8(d): what a kernel that only
// READS the blob's bytes, with the same per-warp tile streams, reaches).
//
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu
// Run:    tools/stream_bench > profiles/<round>_stream_bench.jsonl   (one JSON line per variant)
//
// Variants (every byte read once per launch, rotating over copies > 2x L2,
// back-to-back launches in a CUDA graph):
//   tiles W=<warps/CTA> D=<tiles in flight>: one CTA per SM, each warp streams
//       a contiguous range of 1792-B LAYOUT v3 tiles (3 x 512-B + 256-B
//       no-allocate loads per tile, like the GEMV kernel), D tiles in flight.
//   flat U=<loads in flight>: grid-stride uint4 loads (classic STREAM read).
// Sizes: the bench layers (7.4 / 26 MB), the bench step (59 MB), and 300 MB.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                       \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ uint4 ldg128(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ldg64(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void ldg256(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

constexpr int kTile = 1792;

// Per-lane contiguous 32-B code chunk: one 256-bit load for the codes (1 KB
// per warp request), then s/z (128-bit) and columns (64-bit): 3 loads per tile.
template <int D, int W>
__global__ void __launch_bounds__(32 * W, 1) tiles256_kernel(const uint8_t* base, int num_tiles, int warps, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * W + (threadIdx.x >> 5);
  if (gw >= warps) return;
  const int q = num_tiles / warps, r = num_tiles % warps;
  const int tb = gw * q + min(gw, r), te = tb + q + (gw < r);
  uint32_t acc = 0;
  uint4 buf[D][3];
  uint2 col[D];
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (tb + i < te) {
      const uint8_t* t = base + (int64_t)(tb + i) * kTile;
      ldg256(t + lane * 32, buf[i][0], buf[i][1]);
      buf[i][2] = ldg128(t + 1024 + lane * 16);
      col[i] = ldg64(t + 1536 + lane * 8);
    }
  for (int t0 = tb; t0 < te; t0 += D) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int t = t0 + i;
      if (t < te) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc ^= buf[i][k].x ^ buf[i][k].y ^ buf[i][k].z ^ buf[i][k].w;
        acc ^= col[i].x ^ col[i].y;
        if (t + D < te) {
          const uint8_t* p = base + (int64_t)(t + D) * kTile;
          ldg256(p + lane * 32, buf[i][0], buf[i][1]);
          buf[i][2] = ldg128(p + 1024 + lane * 16);
          col[i] = ldg64(p + 1536 + lane * 8);
        }
      }
    }
  }
  if (acc == 0x12345678u) out[gw] = acc;
}

template <int D, int W>
__global__ void __launch_bounds__(32 * W, 1) tiles_kernel(const uint8_t* base, int num_tiles, int warps, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * W + (threadIdx.x >> 5);
  if (gw >= warps) return;
  const int q = num_tiles / warps, r = num_tiles % warps;
  const int tb = gw * q + min(gw, r), te = tb + q + (gw < r);
  uint32_t acc = 0;
  uint4 buf[D][3];
  uint2 col[D];
#pragma unroll
  for (int i = 0; i < D; ++i)
    if (tb + i < te) {
      const uint8_t* t = base + (int64_t)(tb + i) * kTile;
      buf[i][0] = ldg128(t + lane * 16);
      buf[i][1] = ldg128(t + 512 + lane * 16);
      buf[i][2] = ldg128(t + 1024 + lane * 16);
      col[i] = ldg64(t + 1536 + lane * 8);
    }
  for (int t0 = tb; t0 < te; t0 += D) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int t = t0 + i;
      if (t < te) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc ^= buf[i][k].x ^ buf[i][k].y ^ buf[i][k].z ^ buf[i][k].w;
        acc ^= col[i].x ^ col[i].y;
        if (t + D < te) {
          const uint8_t* p = base + (int64_t)(t + D) * kTile;
          buf[i][0] = ldg128(p + lane * 16);
          buf[i][1] = ldg128(p + 512 + lane * 16);
          buf[i][2] = ldg128(p + 1024 + lane * 16);
          col[i] = ldg64(p + 1536 + lane * 8);
        }
      }
    }
  }
  if (acc == 0x12345678u) out[gw] = acc;
}

// Same tiles, but each warp walks TWO halves of its range in alternation
// (two independent streams per warp: the memory parallelism of 2W warps).
template <int D, int W>
__global__ void __launch_bounds__(32 * W, 1) tiles2_kernel(const uint8_t* base, int num_tiles, int warps, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * W + (threadIdx.x >> 5);
  if (gw >= warps) return;
  const int q = num_tiles / warps, r = num_tiles % warps;
  const int tb = gw * q + min(gw, r), te = tb + q + (gw < r);
  const int h = (te - tb + 1) / 2;
  uint32_t acc = 0;
  uint4 buf[2][D][3];
  uint2 col[2][D];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int t = tb + s * h + i;
      if (t < (s ? te : tb + h)) {
        const uint8_t* p = base + (int64_t)t * kTile;
        buf[s][i][0] = ldg128(p + lane * 16);
        buf[s][i][1] = ldg128(p + 512 + lane * 16);
        buf[s][i][2] = ldg128(p + 1024 + lane * 16);
        col[s][i] = ldg64(p + 1536 + lane * 8);
      }
    }
  for (int k0 = 0; k0 < h; k0 += D) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int t = tb + s * h + k0 + i, end = s ? te : tb + h;
        if (t < end) {
#pragma unroll
          for (int k = 0; k < 3; ++k) acc ^= buf[s][i][k].x ^ buf[s][i][k].y ^ buf[s][i][k].z ^ buf[s][i][k].w;
          acc ^= col[s][i].x ^ col[s][i].y;
          if (t + D < end) {
            const uint8_t* p = base + (int64_t)(t + D) * kTile;
            buf[s][i][0] = ldg128(p + lane * 16);
            buf[s][i][1] = ldg128(p + 512 + lane * 16);
            buf[s][i][2] = ldg128(p + 1024 + lane * 16);
            col[s][i] = ldg64(p + 1536 + lane * 8);
          }
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
  // R launches (one per buffer copy) in a CUDA graph: no host launch gaps
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < R; ++i) launch(i, st);
  cudaStreamEndCapture(st, &g);
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess || cudaGetLastError() != cudaSuccess) return -1.f;
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
  const int64_t pool = 640ll << 20;
  uint8_t* buf;
  CK(cudaMalloc(&buf, pool));
  CK(cudaMemset(buf, 1, pool));
  uint32_t* out;
  CK(cudaMalloc(&out, 1 << 20));
  for (int tiles : {4118, 14400, 32900, 167000}) {  // ~7.4 MB, 26 MB, 59 MB, 300 MB
    const int64_t bytes = (int64_t)tiles * kTile;
    const int R = (int)(pool / bytes) < 12 ? (int)(pool / bytes) : 12;
#define RUN(D, W)                                                                                         \
  {                                                                                                       \
    const int warps = sms * W < tiles ? sms * W : tiles;                                                  \
    float us = time_rot([&](int r, cudaStream_t st) {                                                     \
      tiles_kernel<D, W><<<sms, 32 * W, 0, st>>>(buf + r * bytes, tiles, warps, out); }, 20, R);         \
    fflush(stdout); printf("{\"variant\": \"tiles\", \"bytes\": %lld, \"warps_per_cta\": %d, \"tiles_in_flight\": %d, "  \
           "\"us\": %.3f, \"gbs\": %.1f}\n", (long long)bytes, W, D, us, bytes / us / 1e3);               \
  }
    RUN(2, 8) RUN(4, 8) RUN(6, 8) RUN(2, 16) RUN(3, 16) RUN(4, 16) RUN(2, 24) RUN(3, 24) RUN(2, 32) RUN(3, 32)
#define RUN2(D, W)                                                                                        \
  {                                                                                                       \
    const int warps = sms * W < tiles ? sms * W : tiles;                                                  \
    float us = time_rot([&](int r, cudaStream_t st) {                                                     \
      tiles2_kernel<D, W><<<sms, 32 * W, 0, st>>>(buf + r * bytes, tiles, warps, out); }, 20, R);        \
    fflush(stdout); printf("{\"variant\": \"tiles_2streams\", \"bytes\": %lld, \"warps_per_cta\": %d, "        \
           "\"tiles_in_flight_per_stream\": %d, \"us\": %.3f, \"gbs\": %.1f}\n", (long long)bytes, W, D, us,     \
           bytes / us / 1e3);                                                                             \
  }
    RUN2(1, 16) RUN2(2, 16)
#define RUN3(D, W)                                                                                        \
  {                                                                                                       \
    const int warps = sms * W < tiles ? sms * W : tiles;                                                  \
    float us = time_rot([&](int r, cudaStream_t st) {                                                     \
      tiles256_kernel<D, W><<<sms, 32 * W, 0, st>>>(buf + r * bytes, tiles, warps, out); }, 20, R);      \
    fflush(stdout); printf("{\"variant\": \"tiles_ldg256\", \"bytes\": %lld, \"warps_per_cta\": %d, "          \
           "\"tiles_in_flight\": %d, \"us\": %.3f, \"gbs\": %.1f}\n", (long long)bytes, W, D, us, bytes / us / 1e3); \
  }
    RUN3(2, 8) RUN3(4, 8) RUN3(2, 16) RUN3(3, 16) RUN3(2, 32)
    for (int U : {4, 8}) {
      float us = 0;
      if (U == 4) us = time_rot([&](int r, cudaStream_t st) { flat_kernel<4><<<sms * 4, 256, 0, st>>>((const uint4*)(buf + r * bytes), bytes / 16, out); }, 20, R);
      if (U == 8) us = time_rot([&](int r, cudaStream_t st) { flat_kernel<8><<<sms * 4, 256, 0, st>>>((const uint4*)(buf + r * bytes), bytes / 16, out); }, 20, R);
      printf("{\"variant\": \"flat\", \"bytes\": %lld, \"loads_in_flight\": %d, \"us\": %.3f, \"gbs\": %.1f}\n",
             (long long)bytes, U, us, bytes / us / 1e3);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
