// gqsa_kernels.h -- launch parameters shared by the C-ABI shim and the kernels.
#pragma once
#include <stdint.h>

namespace gqsa {

constexpr int kMaxWarps = 32;           // warps per CTA: a launch-time choice <= 32
constexpr int kMaxThreads = 32 * kMaxWarps;
constexpr int kMaxStages = 8;            // tiles in flight per warp (shared-memory TMA ring)
constexpr int kMinStages = 2;
constexpr int kSmemPerSm = 228 * 1024;   // shared memory per SM (incl. 1 KB reserved per CTA)
constexpr int kMaxBatch = 8;
constexpr int kMaxPeers = 8;            // ranks of a fused all-gather (one NVLink domain)
constexpr int kMaxCtasPerSm = 1;         // default residency: one CTA of up to 16 warps per SM
constexpr int kCoResidentKernels = 2;    // leave room for the next PDL-launched GEMV
// Register budget: 4 resident CTAs (64 regs/thread) at batch 1 -- the HBM
// stream wants many warps with loads in flight; bigger batches need more
// accumulators and are ALU / smem-bound anyway.
// Launch bounds: batch <= 2 launches up to 32 warps per CTA at <= 64
// registers; larger batches (more accumulators) use 8 warps.
// Launch bounds: 16+ warps at batch <= 2 (64 registers), 8 warps above.  W8
// holds 64 code bytes per lane per tile: 8 warps, <= 128 registers (two CTAs
// per SM, so the next PDL launch can be resident).
#ifndef GQSA_B12_THREADS
#define GQSA_B12_THREADS kMaxThreads
#define GQSA_B12_MINB 1
#endif
// FEW: 12 warps per CTA with up to 85 registers (two CTAs per SM for PDL
// co-residency), for batch 1 on layers with few tiles per warp (e.g.
// 4096x4096 at S50: 5.13 -> 4.47 us; 14336x4096 / 4096x14336 unchanged, they
// keep 16 warps) and for every batch-2 layer (-13..14 %).
constexpr int kFewWarps = 12;
constexpr int kFewTiles = 148 * 16 * 4;  // below ~4 tiles per warp of a 16-warp grid
constexpr int max_threads_for(int bits, int B, bool few = false) {
  return few ? 32 * kFewWarps : bits == 8 ? 256 : (B <= 2 ? GQSA_B12_THREADS : 256);
}
constexpr int min_blocks_for(int bits, int B, bool few = false) {
  return few ? 2 : (bits == 8 || B > 2) ? 2 : GQSA_B12_MINB;
}
constexpr int kMaxWarpsBound = 8192;     // workspace records (>= any grid we launch)
constexpr int kWsSlotBytes = 8;          // fix-up slot {partial, flag} per (warp, batch, lane)
constexpr int kSmemBudget = 200 * 1024;  // above this, x is gathered from L1/L2

struct KParams {
  const uint8_t* tiles;   // blob + off_tiles
  const int32_t* perm;    // blob + off_nzrow: row of each (slice, lane), -1 = unused
  const int32_t* empty;   // blob + off_empty
  const uint16_t* X;      // [B][ldx] fp16
  void* Y;                // [B][ldy] fp32 (or fp16 when out_f16)
  const float* bias;      // [rows] or null
  uint32_t* ws;           // [active_warps][B][32] 8-B slots, zero between calls
  int64_t ldx, ldy;
  int32_t rows, cols, num_tiles, n_empty, active_warps, lanes_per_row;
  int32_t part_q, part_r;  // num_tiles = part_q * active_warps + part_r
  int32_t stages;          // ring depth NS (tiles) per warp
  int32_t ring_offset;     // shared-memory offset of the TMA ring (after x and the column sums)
  uint64_t* trace;         // optional [active_warps][8] %globaltimer stamps (debug)
  int32_t slice_k;         // 1: data-centric partition (whole slices per warp, no fix-up)
  int32_t out_f16;         // 1: Y is fp16 (RNE of the fp32 result)
  int32_t fix_offset;      // shared-memory offset of the intra-CTA fix-up records (0: all global)
  // Fused all-gather epilogue (gqsa_gemm_allgather): when n_peers > 0 every
  // output element is stored into each peer's full-length Y (peer pointers,
  // e.g. NVLink P2P / symmetric memory) at global row row_offset + row,
  // instead of into Y.
  int32_t n_peers;
  int32_t row_offset;
  uint64_t peer_y[kMaxPeers];
};

// Persistent chain kernel (gqsa_chain.cu): one launch runs up to kMaxChain
// GEMVs in order, one CTA of kChainThreads per SM (cooperative launch).
constexpr int kMaxChain = 16;
constexpr int kChainThreads = 512;
struct ChainParams {
  KParams item[kMaxChain];        // per item: exactly the per-GEMV kernel's parameters
  int32_t wait_prev[kMaxChain];   // 1: item j reads X only after items < j completed
  int32_t reuse_x[kMaxChain];     // 1: item j has item j-1's X (and no wait): skip restaging
  int32_t n;                      // items
  int32_t stages;                 // ring depth NS (tiles) per warp
  int32_t ring_offset;            // shared-memory offset of the TMA ring
  int32_t fix_offset;             // shared-memory offset of intra-CTA fix-up records (0: none)
  int32_t total_warps;            // grid * warps per CTA (every warp arrives once per item)
  uint32_t* counter;              // workspace: CTA arrivals (returned to 0 by the launch's last arrival)
  uint64_t* trace;                // optional [total_warps][n][4] %globaltimer stamps (debug)
};
static_assert(sizeof(ChainParams) <= 4096, "kernel parameter space");

const void* select_kernel(int bits, int G, int B, bool few);
const void* select_chain_kernel(int bits, int B);
// Bytes of the column-sum table per batch row (see gqsa_gemv.cu pq_per_group).
inline size_t pq_bytes_per_row(int B, int cols, int G = 16) {
  return (size_t)cols / G * ((G == 16 && B <= 2) ? 2 : 1) * 8;
}

}  // namespace gqsa
