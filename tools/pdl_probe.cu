// pdl_probe.cu -- does Programmatic Dependent Launch overlap two kernels here?
// Kernel A (1 CTA/SM, small) triggers launch_dependents at entry then spins
// ~20 us; kernel B records when its CTAs start.  Prints B's first start
// relative to A's start, for plain stream launches and for a captured graph.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void kA(uint64_t* ts, int spin_ns, int trigger) {
  if (threadIdx.x == 0) ts[blockIdx.x] = gtime();
  if (trigger) asm volatile("griddepcontrol.launch_dependents;");
  const uint64_t t0 = gtime();
  while (gtime() - t0 < (uint64_t)spin_ns) {
  }
  if (threadIdx.x == 0) ts[1024 + blockIdx.x] = gtime();
}

__global__ void kB(uint64_t* ts) {
  if (threadIdx.x == 0) ts[2048 + blockIdx.x] = gtime();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) ts[3072 + blockIdx.x] = gtime();
}

static void launch(cudaStream_t s, uint64_t* ts, int sms, bool pdl, int trigger) {
  kA<<<sms, 128, 0, s>>>(ts, 20000, trigger);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kB, ts);
}

static void report(const char* what, uint64_t* d, int sms) {
  static uint64_t h[4096];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  uint64_t a0 = ~0ull, aend = 0, b0 = ~0ull, bw = ~0ull;
  for (int i = 0; i < sms; ++i) {
    a0 = h[i] < a0 ? h[i] : a0;
    aend = h[1024 + i] > aend ? h[1024 + i] : aend;
    b0 = h[2048 + i] < b0 ? h[2048 + i] : b0;
    bw = h[3072 + i] < bw ? h[3072 + i] : bw;
  }
  printf("%-28s A runs %.2f us; B first start at %+.2f us, first release at %+.2f us (rel. A start)\n", what,
         (aend - a0) / 1e3, ((double)b0 - (double)a0) / 1e3, ((double)bw - (double)a0) / 1e3);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* ts;
  cudaMalloc(&ts, 4096 * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int trig = 0; trig < 2; ++trig) {
      launch(s, ts, sms, pdl, trig);
      cudaStreamSynchronize(s);
      launch(s, ts, sms, pdl, trig);
      cudaStreamSynchronize(s);
      char name[64];
      snprintf(name, sizeof(name), "stream pdl=%d trigger=%d", pdl, trig);
      report(name, ts, sms);
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      launch(s, ts, sms, pdl, trig);
      cudaStreamEndCapture(s, &g);
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
        printf("graph instantiate failed\n");
        continue;
      }
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      snprintf(name, sizeof(name), "graph  pdl=%d trigger=%d", pdl, trig);
      report(name, ts, sms);
    }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
