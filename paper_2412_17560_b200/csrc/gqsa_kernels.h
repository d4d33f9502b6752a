// gqsa_kernels.h -- launch parameters shared by the C-ABI shim (gqsa_capi.cu)
// and the Stream-K kernel (gqsa_stream.cu).
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#endif

namespace gqsa {

constexpr int kMaxItems = 8;            // independent GEMVs per launch (gqsa_gemm_grouped)
constexpr int kMaxBatch = 8;
constexpr int kMaxPeers = 8;            // ranks of a fused all-gather (one NVLink domain)
constexpr int kSmemPerSm = 228 * 1024;  // shared memory per SM
constexpr int kMaxDynSmem = 225 * 1024; // opt-in dynamic shared memory per CTA (227 KB - the static item table)
// Tile register buffers per warp (HBM -> registers, no shared-memory
// staging): one at B <= 2, where more warps (fewer registers each) plus L2
// prefetching keep more bytes in flight than a second register buffer does
// (bench step 11.8 vs 12.6 us); two above.
#ifndef GQSA_BUFS_SMALL
#define GQSA_BUFS_SMALL 1
#endif
#ifndef GQSA_BUFS_LARGE
#define GQSA_BUFS_LARGE 2
#endif
#ifndef GQSA_BUFS_B2
#define GQSA_BUFS_B2 GQSA_BUFS_SMALL
#endif
__host__ __device__ constexpr int bufs_for(int B) { return B == 1 ? GQSA_BUFS_SMALL : B == 2 ? GQSA_BUFS_B2 : GQSA_BUFS_LARGE; }
// L2 prefetch distance in tiles (<= the register buffers: off): lane 0 issues
// cp.async.bulk.prefetch.L2 for tile t + d as it requests tile t into
// registers, so each warp keeps d tiles moving from HBM while only the
// register buffers hold data (bench step, measured: d = 2..4 within 1 %;
// no prefetch with two register buffers: 15.1 us).
#ifndef GQSA_L2PF_SMALL
#define GQSA_L2PF_SMALL 2
#endif
#ifndef GQSA_L2PF_LARGE
#define GQSA_L2PF_LARGE 3
#endif
__host__ __device__ constexpr int l2pf_for(int B) { return B <= 2 ? GQSA_L2PF_SMALL : GQSA_L2PF_LARGE; }
// 1: the in-loop prefetch is one prefetch.global.L2 per lane (a 128-B line
// each); 0: one cp.async.bulk.prefetch.L2 of the whole tile from lane 0.
#ifndef GQSA_LANE_PF
#define GQSA_LANE_PF 1
#endif
// Warps per CTA (one CTA per SM): more warps keep more weight loads in
// flight (a read-only stream of the same tiles reaches 4.9 / 5.3 / 5.5 TB/s
// with 16 / 24 / 32 warps per SM on the 59 MB bench step,
// profiles/r02_stream_bench.jsonl); the register budget (<= 65536 / 32W per
// thread, no spills) sets the count: 20 at batch 1, 16 above (batch 8 on
// 14336x4096: 8 warps 46 us, 16 warps 39 us).
#ifndef GQSA_WARPS_SMALL
#define GQSA_WARPS_SMALL 20
#endif
#ifndef GQSA_WARPS_LARGE
#define GQSA_WARPS_LARGE 16
#endif
__host__ __device__ constexpr int warps_for(int B) { return B == 1 ? GQSA_WARPS_SMALL : B == 2 ? 16 : GQSA_WARPS_LARGE; }
// Resident CTAs per SM the kernel is compiled for (launch bounds): 2 lets the
// next launch on the stream be resident during this one's tail (PDL).
#ifndef GQSA_MINB
#define GQSA_MINB 1
#endif
__host__ __device__ constexpr int min_blocks_for(int B) { return B <= 2 ? GQSA_MINB : 1; }
// CTAs per SM of a whole-SM launch at B = 1 (the grid is this many x #SMs).
#ifndef GQSA_FULL_CTAS
#define GQSA_FULL_CTAS 1
#endif
__host__ __device__ constexpr int full_ctas_for(int B) { return B == 1 ? GQSA_FULL_CTAS : 1; }
// Pipelined mode (x_ready, B <= 2): the launch takes HALF of
// every SM (one CTA of half the warps, compiled for 2 resident CTAs), so the
// next independent launch on the stream runs its prologue, activation staging
// and tile loop on the other half while this one drains; every global write
// of the loop is deferred until after griddepcontrol.wait.
#ifndef GQSA_WARPS_HALF
#define GQSA_WARPS_HALF 6
#endif
#ifndef GQSA_PIPE_CTAS
#define GQSA_PIPE_CTAS 4
#endif
// Resident CTAs per SM the pipelined kernel is compiled for: four launches
// in flight at B = 1 (6 warps each, <= 80 registers; bench step: 2 x 12 warps
// 11.8 us, 3 x 8 11.1, 4 x 6 10.9 -- the fourth needs the one-entry-per-group
// column-sum table and 4 deferred-store slots to fit 55 KB of shared memory);
// two at B = 2 (its accumulators need the registers).
__host__ __device__ constexpr int pipe_ctas_for(int B) { return B == 1 ? GQSA_PIPE_CTAS : 2; }
__host__ __device__ constexpr int warps_half(int B) { return B == 1 ? GQSA_WARPS_HALF : 8; }
__host__ __device__ constexpr int warps_of(int B, int half) { return half ? warps_half(B) : warps_for(B); }
// Deferred row stores buffered per warp in shared memory before the wait
// (more closed slices than this in one range: the warp waits and stores).
#ifndef GQSA_DEFER_SLOTS
#define GQSA_DEFER_SLOTS 4
#endif
constexpr int kDeferSlots = GQSA_DEFER_SLOTS;
__host__ __device__ constexpr int defer_bytes_per_warp(int B) { return kDeferSlots * 32 * 4 * (B + 1); }
// dynamic shared memory per CTA of a pipelined launch (pipe_ctas_for(B) CTAs per SM)
__host__ __device__ constexpr int half_smem_limit(int B) {
  return (kSmemPerSm - pipe_ctas_for(B) * 2048) / pipe_ctas_for(B);
}
// Small launches use fewer warps per CTA so that each warp streams at least
// this many tiles (4096^2 dependent launch: 20 warps / 1.4 tiles each 6.10 us,
// 10 warps / 2.8 tiles 5.59 us; LLaMA-3-8B stack 1188 -> 1155 us per token;
// larger layers and the bench step have more tiles per warp and are unchanged;
// batch 1 only: at batch 8 4096^2 measured 16.3 -> 16.8 us).
#ifndef GQSA_MIN_TPW
#define GQSA_MIN_TPW 3
#endif
constexpr int kMinTilesPerWarp = GQSA_MIN_TPW;  // see min_tiles_per_warp() in gqsa_capi.cu
constexpr int kMaxWarpsBound = 148 * 32;  // fix-up records the workspace holds per launch (any B200 grid)

// One GEMV of a launch.  Its tiles occupy global tile indices
// [tile_begin, tile_end) of the launch's concatenated tile stream.
struct Item {
  const uint8_t* tiles;        // blob + off_tiles
  const int32_t* perm;         // [num_slices][32] row of each (slice, lane), -1 = unused lane
  const int32_t* slice_tile0;  // [num_slices + 1] first tile of each slice
  const int32_t* tile_slice;   // [num_tiles] slice of each tile
  const int32_t* empty;        // [n_empty] empty rows
  const uint16_t* X;           // [B][ldx] fp16
  void* Y;                     // [B][ldy] fp32 (fp16 when out_f16)
  const float* bias;           // [rows] or null
  int64_t ldx, ldy;
  int32_t rows, cols, n_empty, lanes_per_row, num_slices;
  int32_t tile_begin, tile_end;
  int32_t xrow;       // shared-memory bytes per staged activation row (2K + zero block)
  int32_t pqrow;      // shared-memory bytes per row of the (-P, -Q) column-sum table
  int32_t smem_bytes; // B * (xrow + pqrow), rounded to 128
  int32_t n_peers;    // fused all-gather: store every element into each peer_y (global row row_offset + r)
  int32_t row_offset;
  int32_t peer_mc;    // 1: peer_y[0] is an NVLS multicast address, stored with multimem.st (one store
                      //    reaches every rank bound to the multicast object)
  int32_t pad_;
  uint64_t peer_y[kMaxPeers];
};

struct Params {
  Item item[kMaxItems];
  int32_t n_items, total_tiles, active_warps, part_q, part_r;  // total_tiles = part_q * active_warps + part_r
  int32_t slice_k;   // 1: data-centric partition (whole slices per warp, no fix-up)
  int32_t out_f16;   // 1: Y is fp16 (RNE of the fp32 result)
  int32_t x_ready;   // 1: X is not written by the previous kernel on the stream: stage it before the PDL wait
  int32_t stage_tab_offset;  // shared offset of the staging table (after the largest staged footprint)
  int32_t defer_offset;      // pipelined mode: shared offset of the per-warp deferred-store buffers
  int32_t cta_fix;           // whole-SM Stream-K: reduce split slices inside the CTA through shared
                             // memory; only CTA-level partials take the global fix-up
  int32_t wait_first;        // experiments: griddepcontrol.wait before the first weight loads (x_ready = 0)
  int32_t cta_slicek;        // slice-aligned CTA ranges, Stream-K among the CTA's warps (one item, cta_fix)
  uint32_t* cnt;                 // unused by the stream kernel since the look-back fix-up (kept zero)
  unsigned long long* rec;       // [active_warps][2][B][32] fix-up records {partial, flag}
  uint64_t* trace;               // optional [active_warps][8] %globaltimer stamps (debug)
};
static_assert(sizeof(Params) <= 4096, "kernel parameter space");

// Shared-memory layout of one staged item (per batch row b):
//   x  : [B][xrow]  fp16 activations, then kXPadBytes of zeros (padding entries read them)
//   pq : [B][pqrow] float2 (-P, -Q) per chunk index f (G = 16, B <= 2) or per column group
// One (-P, -Q) entry per column group (default), or, with GQSA_PQ_PER_GROUP=0
// at G = 16, B <= 2, one per 16-B x chunk (the pair duplicated: the lookup
// offset is the column field >> 1, one instruction fewer per group, but twice
// the table: 2.5 % faster at 3 CTAs per SM, too big for 4).
#ifndef GQSA_PQ_PER_GROUP
#define GQSA_PQ_PER_GROUP 1
#endif
__host__ __device__ constexpr bool pq_per_chunk(int B, int G) { return G == 16 && B <= 2 && !GQSA_PQ_PER_GROUP; }
__host__ __device__ constexpr int pq_entries(int B, int G, int cols) {
  return pq_per_chunk(B, G) ? 2 * (cols / G) : cols / G;
}
__host__ __device__ constexpr int pq_row_bytes(int B, int G, int cols) {
  return ((pq_entries(B, G, cols) + 2) * 8 + 15) / 16 * 16;  // + zero entries for padding
}

const void* select_kernel(int bits, int G, int B, int half = 0);

// LAYOUT-TC kernel (gqsa_tc.cu): one GEMM over 16-row blocks on mma.sync.
constexpr int kTcWarps = 16;
// LAYOUT-TC tiles are 768 B (vs 1792 B for the stream layout): more of them in
// flight per warp to keep the same bytes in flight per SM.
#ifndef GQSA_TC_BUFS
#define GQSA_TC_BUFS 4
#endif
constexpr int kTcBufs = GQSA_TC_BUFS;
struct TcParams {
  const uint8_t* tiles;         // blob + off_tiles (768-B tiles of 4 items)
  const uint16_t* tile_cols;    // [num_tiles][4] item columns
  const int32_t* block_tile0;   // [nb + 1]
  const int32_t* tile_block;    // [num_tiles]
  const uint16_t* X;            // [B][ldx] fp16
  void* Y;                      // [B][ldy] fp32 (fp16 when out_f16)
  const float* bias;            // [rows] or null
  int64_t ldx, ldy;
  int32_t rows, cols, num_tiles, nb;
  int32_t active_warps, part_q, part_r;
  int32_t slice_k, out_f16, x_ready;
  int32_t xrow;                 // shared bytes per staged x row (2K + 32: zero chunk for padding items)
  int32_t cta_fix;              // reduce split blocks inside the CTA first
  uint32_t* cnt;                // [active_warps] fix-up arrival counters (zero between launches)
  unsigned long long* rec;      // [active_warps][2][4][32] fix-up records
  uint64_t* trace;
};
const void* select_tc_kernel(int B, bool xq_mma);

}  // namespace gqsa
