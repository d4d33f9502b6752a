// gqsa_layout.h -- LAYOUT v1 of the packed GQSA blob (product-internal).
//
// The blob is the paper's BSR (rowIndex / groups / values +
// per-group scale and zero) re-laid out offline for the B200
// kernel: 128-kept-group tile records whose per-lane payloads are 16-B
// vectors, so that every warp-level load is a fully-coalesced 512-B (codes,
// s/z) or 256-B (columns) request.  Full description: DESIGN.md §5.
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
constexpr int kVersion = 1;
constexpr int kGroup = 16;          // G (v1)
constexpr int kTileGroups = 128;    // kept groups per tile record
constexpr int kLanes = 32;          // one warp consumes one tile
constexpr int kPerLane = kTileGroups / kLanes;  // 4 groups per lane per tile
constexpr int kHeaderBytes = 256;
constexpr int kTileHeaderBytes = 32;  // u32 segmask[4]; i32 m0; u32 reserved[3]
constexpr int kSectionAlign = 256;
constexpr uint32_t kFlagLaneParitySwap = 1u;  // swap bit of a group = lane & 1

// Bytes of one group's codes (G*n/8).
__host__ __device__ constexpr int group_code_bytes(int bits) { return kGroup * bits / 8; }
// Codes plane: each lane owns 16 B per plane -> 16/cb groups per plane.
__host__ __device__ constexpr int groups_per_plane(int bits) { return 16 / group_code_bytes(bits); }
__host__ __device__ constexpr int codes_bytes(int bits) { return kTileGroups * group_code_bytes(bits); }
__host__ __device__ constexpr int off_sz(int bits) { return kTileHeaderBytes + codes_bytes(bits); }
__host__ __device__ constexpr int off_cols(int bits) { return off_sz(bits) + kTileGroups * 4; }
__host__ __device__ constexpr int tile_bytes(int bits) { return off_cols(bits) + kTileGroups * 2; }

// Offset (within a tile) of the code bytes of the group in lane l, slot u.
__host__ __device__ constexpr int off_codes(int bits, int lane, int u) {
  return kTileHeaderBytes + (u / groups_per_plane(bits)) * 512 + lane * 16 +
         (u % groups_per_plane(bits)) * group_code_bytes(bits);
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
