// gqsa_layout.h -- LAYOUT v3 of the packed GQSA blob (product-internal).
//
// The blob is the paper's BSR (rowIndex / groups / values +
// per-group scale and zero) re-laid out offline for the B200
// kernel as a sliced-ELL stream of 128-group tiles (4 slots x 32 lanes, one
// lane per row): every warp-level load of a tile is a fully coalesced,
// 128-B-aligned 512-B (codes, s/z) or 256-B (columns) request straight into
// registers, and a lane accumulates its row without cross-lane reductions.
// Slice boundaries live in two small side tables instead of per-tile headers,
// so a tile is an exact multiple of 128 B.  Full description: DESIGN.md §5.
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
constexpr int kVersion = 3;
constexpr int kGroup = 16;          // G (the paper's default)
constexpr int kTileGroups = 128;    // groups (incl. padding) per tile record
constexpr int kLanes = 32;          // one warp consumes one tile, one lane per row
constexpr int kPerLane = kTileGroups / kLanes;  // 4 slots per lane per tile
constexpr int kHeaderBytes = 256;
constexpr int kSectionAlign = 256;
constexpr uint32_t kFlagTargetDeal = 4u;     // bank-aware dealing (G = 16)
constexpr int kFlagLanesPerRowShift = 8;     // flags bits 8..15: lanes per row S
// The column field is the byte offset of a 16-B activation chunk in a u16;
// padding entries point at a 64-B zero block right after the K activations
// of each batch row (offset 2K), so 2K + 64 <= 65536.
constexpr int kMaxCols = 32736;
// Bytes of zero padding after each staged activation row (>= one G = 32 group).
constexpr int kXPadBytes = 64;

// Group sizes: G = 16 for every bit width; G = 8 and G = 32 for W4 (the
// group-size sweep).
__host__ __device__ constexpr bool group_supported(int bits, int G) {
  return G == kGroup ? (bits == 2 || bits == 4 || bits == 8) : (bits == 4 && (G == 8 || G == 32));
}
// Bytes of one group's codes (G*n/8).
__host__ __device__ constexpr int group_code_bytes(int bits, int G = kGroup) { return G * bits / 8; }
// Codes plane: each lane owns 16 B per plane -> 16/cb groups per plane (cb <= 16).
__host__ __device__ constexpr int groups_per_plane(int bits, int G = kGroup) { return 16 / group_code_bytes(bits, G); }
__host__ __device__ constexpr int code_planes(int bits, int G = kGroup) { return G * bits / 32; }
__host__ __device__ constexpr int codes_bytes(int bits, int G = kGroup) { return kTileGroups * group_code_bytes(bits, G); }
__host__ __device__ constexpr int off_sz(int bits, int G = kGroup) { return codes_bytes(bits, G); }
__host__ __device__ constexpr int off_cols(int bits, int G = kGroup) { return off_sz(bits, G) + kTileGroups * 4; }
__host__ __device__ constexpr int tile_bytes(int bits, int G = kGroup) { return off_cols(bits, G) + kTileGroups * 2; }
static_assert(tile_bytes(4) % 128 == 0 && tile_bytes(2) % 128 == 0 && tile_bytes(8) % 128 == 0 &&
                  tile_bytes(4, 8) % 128 == 0 && tile_bytes(4, 32) % 128 == 0,
              "tiles are whole 128-B lines");

// Offset (within a tile) of the code bytes of the group in lane l, slot u.
__host__ __device__ constexpr int off_codes_g(int bits, int G, int lane, int u) {
  return (u / groups_per_plane(bits, G)) * 512 + lane * 16 + (u % groups_per_plane(bits, G)) * group_code_bytes(bits, G);
}
// Offset (within a tile) of the (s, z) pair of lane l, slot u.
__host__ __device__ constexpr int off_sz_g(int bits, int G, int lane, int u) { return off_sz(bits, G) + lane * 16 + u * 4; }
// Offset (within a tile) of the column field of lane l, slot u.
__host__ __device__ constexpr int off_cols_g(int bits, int G, int lane, int u) {
  return off_cols(bits, G) + lane * 8 + u * 2;
}

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
// Column field of a padding entry: the zero block after the activations.
__host__ __device__ constexpr uint32_t pad_field(int cols) { return 2u * (uint32_t)cols; }

// LAYOUT-TC (the small-batch tensor-core layout, W4 G16):
// rows in blocks of 16 (the mma M dimension); a block's ITEMS are the group
// columns kept by any of its rows, ascending, each the 16 x 16 code matrix of
// the block at that column (zeros and s = 0 for rows that do not keep it) in
// mma.m16n8k16 A-fragment order, so a lane loads its fragment with one 32-bit
// word; tiles of 4 items: codes [lane][item] 4 B (512 B) + (s, z) [row pair
// g, g+8][item] 8 B (256 B).  Item columns live in a side array (u16 [tile][4]).
constexpr uint32_t kFlagTC = 2u;   // flags bit 1: the blob is LAYOUT-TC
constexpr int kTcRows = 16;        // rows per block
constexpr int kTcItems = 4;        // items per tile
constexpr int kTcTileBytes = 768;  // 4 x 32 lanes x 4 B codes + 8 row pairs x 4 items x 8 B (s, z)
// Nibble j (bits 4j..4j+3) of lane L's word for one item holds A[row][k],
// row = (L >> 2) + 8 * (j & 1), k = 2 (L & 3) + ((j >> 1) & 1) * 8 + (j >> 2):
// LOP3(w >> 4m, 0x000F000F) for m = 0..3 gives the fragment registers
// a_m = half2(1024 + A[row_m][k_m], 1024 + A[row_m][k_m + 1]).
__host__ __device__ constexpr int tc_nib_row(int lane, int j) { return (lane >> 2) + 8 * (j & 1); }
__host__ __device__ constexpr int tc_nib_k(int lane, int j) { return 2 * (lane & 3) + ((j >> 1) & 1) * 8 + (j >> 2); }

constexpr int kTargetSlots = 256;  // slots per lane of the longest slice (64 tiles)

// Target slots per lane for a layer of nnzg kept groups: short slices when the
// layer has few tiles per warp of a B200 grid (148 SMs x 16 warps), so a
// slice spans few warps and the fix-up chain stays short; long slices
// otherwise -- a slice's slot count is padded to whole tiles (4 slots), so
// long slices pad less (LLaMA-3-8B W4S50: 4096^2 11.9 % -> 1.6 %; bench step
// 13.7 -> 12.6 us).
inline int target_slots_for(int64_t nnzg) {
  const double tiles_per_warp = (double)nnzg / kTileGroups / (148.0 * 16.0);
  return tiles_per_warp < 1.6 ? 16 : tiles_per_warp < 4.0 ? 128 : kTargetSlots;
}

// Lanes per row S (a power of two <= 32): large enough that the longest row
// needs at most target_slots slots per lane, and large enough that a layer
// with fewer than 32 non-empty rows still fills the 32 lanes.
inline int lanes_per_row_for(int n_nz, int64_t max_len, int target_slots = kTargetSlots) {
  if (n_nz <= 0) return 1;
  int s = 1;
  while (s < kLanes && (max_len + s - 1) / s > target_slots) s <<= 1;
  int p = 1;
  while (p < n_nz && p < kLanes) p <<= 1;
  const int s_small = kLanes / p;
  return s > s_small ? s : s_small;
}

// On-blob header; the first 128 bytes mirror gqsa_desc_t field-for-field.
struct BlobHeader {
  uint32_t magic, version;
  int32_t rows, cols, group_size, bits;
  int64_t nnzg;
  int32_t tile_groups, num_tiles;
  int32_t n_nzrows, n_empty;
  int32_t tile_bytes, flags;
  int32_t row_begin, row_end;
  int32_t num_slices, reserved0;
  uint64_t off_row_index, off_perm, off_empty, off_slice_tile0, off_tile_slice, off_tiles, blob_bytes;
  uint8_t reserved[kHeaderBytes - 128];
};
static_assert(sizeof(BlobHeader) == kHeaderBytes, "header size");

}  // namespace gqsa
