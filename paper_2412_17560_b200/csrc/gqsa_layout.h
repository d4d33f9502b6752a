// gqsa_layout.h -- LAYOUT v2 of the packed GQSA blob (product-internal).
//
// The blob is the paper's BSR (rowIndex / groups / values +
// per-group scale and zero) re-laid out offline for the B200
// kernel as a sliced-ELL stream of 128-group tiles (4 slots x 32 lanes, one
// lane per row): every warp-level load is a fully-coalesced 512-B (codes,
// s/z) or 256-B (columns) request, and a lane accumulates its row without
// cross-lane reductions.  Full description: DESIGN.md §5.
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

constexpr uint32_t kMagic = 0x41535147u;  // "GQSA"
constexpr int kVersion = 2;
constexpr int kGroup = 16;          // G (v1/v2)
constexpr int kTileGroups = 128;    // groups (incl. padding) per tile record
constexpr int kLanes = 32;          // one warp consumes one tile, one lane per row
constexpr int kPerLane = kTileGroups / kLanes;  // 4 slots per lane per tile
constexpr int kHeaderBytes = 256;
constexpr int kTileHeaderBytes = 32;  // u32 (slice<<2 | FIRST | LAST), tiles_to_slice_end, slice_first_tile; 0[5]
constexpr int kSectionAlign = 256;
constexpr uint32_t kFlagTargetDeal = 4u;     // bank-aware dealing: lane l reads chunk f = 2c+swap,
                                             // f mod 16 == l mod 16 whenever the row allows
constexpr int kFlagLanesPerRowShift = 8;     // flags bits 8..15: lanes per row S
constexpr int kMaxCols = 32768;              // column field = byte offset (2c+swap)*16 < 65536
constexpr uint32_t kTileFirst = 1u;          // tile header flags
constexpr uint32_t kTileLast = 2u;

// Group sizes: G = 16 for every bit width (the paper's default);
// G = 8 and G = 32 for W4 (the group-size sweep).
__host__ __device__ constexpr bool group_supported(int bits, int G) {
  return G == kGroup ? (bits == 2 || bits == 4 || bits == 8) : (bits == 4 && (G == 8 || G == 32));
}
// Bytes of one group's codes (G*n/8).
__host__ __device__ constexpr int group_code_bytes(int bits, int G = kGroup) { return G * bits / 8; }
// Codes plane: each lane owns 16 B per plane -> 16/cb groups per plane (cb <= 16).
__host__ __device__ constexpr int groups_per_plane(int bits, int G = kGroup) { return 16 / group_code_bytes(bits, G); }
__host__ __device__ constexpr int codes_bytes(int bits, int G = kGroup) { return kTileGroups * group_code_bytes(bits, G); }
__host__ __device__ constexpr int off_sz(int bits, int G = kGroup) { return kTileHeaderBytes + codes_bytes(bits, G); }
__host__ __device__ constexpr int off_cols(int bits, int G = kGroup) { return off_sz(bits, G) + kTileGroups * 4; }
__host__ __device__ constexpr int tile_bytes(int bits, int G = kGroup) { return off_cols(bits, G) + kTileGroups * 2; }

// Offset (within a tile) of the code bytes of the group in lane l, slot u.
__host__ __device__ constexpr int off_codes_g(int bits, int G, int lane, int u) {
  return kTileHeaderBytes + (u / groups_per_plane(bits, G)) * 512 + lane * 16 +
         (u % groups_per_plane(bits, G)) * group_code_bytes(bits, G);
}
__host__ __device__ constexpr int off_codes(int bits, int lane, int u) { return off_codes_g(bits, kGroup, lane, u); }

// Column field of a kept group at group column c: the byte offset of the
// first 16-B activation chunk the lane reads.  G = 16: chunk 2c + swap
// (swap = lane parity); G = 8: chunk c; G = 32: chunk
// 4c + rot, rot = lane mod 4 -- the lane reads the group's four chunks
// rot, rot+1, .. (mod 4) and its code words are stored in that order, so the
// lanes of a quarter-warp spread over the bank quads.
__host__ __device__ constexpr uint32_t col_field(int G, uint32_t c, uint32_t rot) {
  return G == 16 ? (((c << 1) | rot) << 4) : G == 8 ? (c << 4) : (((c << 2) | rot) << 4);
}
// Rotation (G = 32) / swap (G = 16) of lane l; 0 for G = 8.
__host__ __device__ constexpr uint32_t lane_rot(int G, int lane) {
  return G == 16 ? (uint32_t)(lane & 1) : G == 32 ? (uint32_t)(lane & 3) : 0u;
}

constexpr int kTargetSlots = 64;  // slots per lane of the longest slice (16 tiles)

// Target slots per lane for a layer of nnzg kept groups: short slices when the
// layer has few tiles per warp of a B200 grid (148 SMs x 16 warps), so a
// slice spans few warps and the fix-up chain stays short; long slices (less
// tile padding) otherwise.  Measured (W4S50, B = 1): 1024x4096 4.28 -> 2.92 us
// (16), 4096x4096 4.49 -> 4.13 us (32), 14336x4096 best at 64.
inline int target_slots_for(int64_t nnzg) {
  const double tiles_per_warp = (double)nnzg / kTileGroups / (148.0 * 16.0);
  return tiles_per_warp < 1.6 ? 16 : tiles_per_warp < 4.0 ? 32 : kTargetSlots;
}

// Lanes per row S (a power of two <= 32): large enough that the longest row
// needs at most kTargetSlots slots per lane (short slices -> few warps per
// slice -> short fix-up chains), and large enough that a layer with fewer
// than 32 non-empty rows still fills the 32 lanes.
inline int lanes_per_row_for(int n_nz, int64_t max_len, int target_slots = kTargetSlots) {
  if (n_nz <= 0) return 1;
  int s = 1;
  while (s < kLanes && (max_len + s - 1) / s > target_slots) s <<= 1;
  int p = 1;
  while (p < n_nz && p < kLanes) p <<= 1;
  const int s_small = kLanes / p;
  return s > s_small ? s : s_small;
}

// Offset (within a tile) of the column field of lane l, slot u.
__host__ __device__ constexpr int off_cols_g(int bits, int G, int lane, int u) {
  return off_cols(bits, G) + lane * 8 + u * 2;
}

// On-blob header; the first 104 bytes mirror gqsa_desc_t field-for-field.
struct BlobHeader {
  uint32_t magic, version;
  int32_t rows, cols, group_size, bits;
  int64_t nnzg;
  int32_t tile_groups, num_tiles;
  int32_t n_nzrows, n_empty;
  int32_t tile_bytes, flags;
  int32_t row_begin, row_end;
  uint64_t off_row_index, off_nzrow, off_empty, off_tiles, blob_bytes;
  uint8_t reserved[kHeaderBytes - 104];
};
static_assert(sizeof(BlobHeader) == kHeaderBytes, "header size");

}  // namespace gqsa
