// gqsa_kernels.h -- launch parameters shared by the C-ABI shim and the kernels.
#pragma once
#include <stdint.h>

namespace gqsa {

constexpr int kThreads = 256;            // 8 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kDepth = 2;                // tiles in flight per warp (register ring)
constexpr int kMaxBatch = 8;
constexpr int kMaxCtasPerSm = 2;
constexpr int kMaxWarpsBound = 4096;     // workspace records (>= any grid we launch)
constexpr int kWsWords = 16;             // 64-B fix-up record per warp
constexpr int kWsFlag = 15;              // word holding the record's flag
constexpr uint32_t kFlagClosed = 1u;     // published row segment ends in that warp
constexpr uint32_t kFlagOpen = 2u;       // ... continues into the next warp
constexpr int kSmemBudget = 200 * 1024;  // above this, x is gathered from L1/L2

struct KParams {
  const uint8_t* tiles;   // blob + off_tiles
  const int32_t* nzrow;   // blob + off_nzrow: row of each non-empty-row ordinal
  const int32_t* empty;   // blob + off_empty
  const uint16_t* X;      // [B][ldx] fp16
  float* Y;               // [B][ldy] fp32
  const float* bias;      // [rows] or null
  uint32_t* ws;           // [active_warps][kWsWords], zero between calls
  int64_t ldx, ldy;
  int32_t rows, cols, num_tiles, n_empty, active_warps;
};

const void* select_kernel(int bits, int B, bool xsmem);

}  // namespace gqsa
