// gqsa_pack.cpp -- host packer, unpacker and validator for LAYOUT v3.
//
// Offline pre-processing ("quantized weights are grouped by size
// G and saved ... along with scaling factors and zero points"): the plain BSR
// is validated and re-laid out for the
// B200 kernel:
//   * non-empty rows are ordered by kept-group count (descending, ties by row)
//     and cut into SLICES of 32 lanes; a row occupies S = lanes_per_row
//     consecutive lanes (S = 1 unless the layer has fewer than 32 non-empty
//     rows), the rest of the slice's lanes are padding;
//   * each lane's groups are dealt into SLOTS: a row's kept groups, starting at
//     a hashed rotation, go round-robin over its S lanes;
//   * a slice's slots are cut into 128-group TILES (4 slots x 32 lanes) whose
//     per-lane payloads are 16-B vectors (codes, s/z) and 8-B vectors (columns);
//     slice boundaries are kept in side tables (slice_tile0, tile_slice);
//   * padding entries (s = z = 0, codes 0) point at the zero block after the
//     staged activations, so they contribute exactly 0 for any input x;
//   * per (slot, quarter-warp) the swap bit of each group picks which 16-B half
//     of its activation slice is read first, balancing shared-memory bank quads.
// gqsa_unpack is the exact inverse (it re-sorts each row by column).
#include <algorithm>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <vector>

#include "../../include/gqsa.h"
#include "gqsa_layout.h"
#include "gqsa_pack_internal.h"

using namespace gqsa;

namespace {

inline uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

inline bool f16_finite(uint16_t h) { return ((h >> 10) & 0x1f) != 0x1f; }
inline bool f16_positive(uint16_t h) { return !(h & 0x8000) && (h & 0x7fff) != 0; }

int check_bsr_header(const gqsa_bsr_t* b) {
  if (!b) return GQSA_ERR_BUFFER;
  if (b->rows < 0 || b->cols <= 0 || b->group_size <= 0 || b->nnzg < 0) return GQSA_ERR_SHAPE;
  if (!group_supported(b->bits, b->group_size)) return GQSA_ERR_UNSUPPORTED;
  if (b->cols % b->group_size) return GQSA_ERR_SHAPE;
  if (b->cols > kMaxCols) return GQSA_ERR_UNSUPPORTED;  // col field = byte offset in u16 (+ zero block)
  if (!b->row_index) return GQSA_ERR_BUFFER;
  if (b->nnzg > 0 && (!b->group_cols || !b->codes || !b->scales_f16 || !b->zeros_f16))
    return GQSA_ERR_BUFFER;
  return GQSA_OK;
}

// Validate the whole row_index and the groups of rows [r0, r1).
int validate(const gqsa_bsr_t* b, int32_t r0, int32_t r1) {
  const int32_t* ri = b->row_index;
  if (ri[0] != 0) return GQSA_ERR_VALIDATION;
  for (int32_t r = 0; r < b->rows; ++r)
    if (ri[r + 1] < ri[r]) return GQSA_ERR_VALIDATION;
  if ((int64_t)ri[b->rows] != b->nnzg) return GQSA_ERR_VALIDATION;
  const int32_t gpr = b->cols / b->group_size;
  for (int32_t r = r0; r < r1; ++r) {
    for (int64_t g = ri[r]; g < ri[r + 1]; ++g) {
      if ((int32_t)b->group_cols[g] >= gpr) return GQSA_ERR_VALIDATION;
      if (g > ri[r] && b->group_cols[g] <= b->group_cols[g - 1]) return GQSA_ERR_VALIDATION;
      if (!f16_finite(b->scales_f16[g]) || !f16_positive(b->scales_f16[g])) return GQSA_ERR_VALIDATION;
      if (!f16_finite(b->zeros_f16[g])) return GQSA_ERR_VALIDATION;
    }
  }
  return GQSA_OK;
}

// Slice structure of rows [r0, r1) (local row ids 0..rows-1).
struct Slices {
  int32_t rows = 0, n_nz = 0, n_empty = 0, lanes_per_row = 1, rows_per_slice = 32, num_slices = 0;
  int32_t num_tiles = 0;
  std::vector<int32_t> order;       // non-empty local rows, sorted (count desc, row asc)
  std::vector<int32_t> empty;       // empty local rows, ascending
  std::vector<int64_t> count;       // kept groups per local row
  std::vector<int32_t> tile0;       // first tile of each slice (+ sentinel)
};

Slices make_slices(const gqsa_bsr_t* b, int32_t r0, int32_t r1) {
  Slices s;
  s.rows = r1 - r0;
  s.count.resize(s.rows);
  for (int32_t r = 0; r < s.rows; ++r) {
    s.count[r] = (int64_t)b->row_index[r0 + r + 1] - b->row_index[r0 + r];
    if (s.count[r] > 0) s.order.push_back(r);
    else s.empty.push_back(r);
  }
  std::stable_sort(s.order.begin(), s.order.end(),
                   [&](int32_t a, int32_t c) { return s.count[a] > s.count[c]; });
  s.n_nz = (int32_t)s.order.size();
  s.n_empty = (int32_t)s.empty.size();
  static const int target_env = [] {
    const char* e = std::getenv("GQSA_TARGET_SLOTS");  // experiment knob (overrides the rule)
    return e && std::atoi(e) >= 4 ? std::atoi(e) : 0;
  }();
  int64_t nnz_range = 0;
  for (int32_t r : s.order) nnz_range += s.count[r];
  const int target = target_env ? target_env : target_slots_for(nnz_range);
  s.lanes_per_row = lanes_per_row_for(s.n_nz, s.n_nz ? s.count[s.order[0]] : 0, target);
  s.rows_per_slice = kLanes / s.lanes_per_row;
  s.num_slices = (s.n_nz + s.rows_per_slice - 1) / s.rows_per_slice;
  s.tile0.resize(s.num_slices + 1);
  int64_t t = 0;
  for (int32_t sl = 0; sl < s.num_slices; ++sl) {
    s.tile0[sl] = (int32_t)t;
    const int64_t longest = s.count[s.order[(size_t)sl * s.rows_per_slice]];
    const int64_t slots = (longest + s.lanes_per_row - 1) / s.lanes_per_row;
    t += (slots + kPerLane - 1) / kPerLane;
  }
  s.tile0[s.num_slices] = (int32_t)t;
  s.num_tiles = (int32_t)t;
  return s;
}

struct Offsets {
  uint64_t ri, perm, empty, st0, ts, tiles, total;
};

Offsets offsets(const Slices& s, int bits, int G) {
  Offsets o;
  o.ri = kHeaderBytes;
  o.perm = align_up(o.ri + 4ull * (s.rows + 1), kSectionAlign);
  o.empty = align_up(o.perm + 4ull * kLanes * s.num_slices, kSectionAlign);
  o.st0 = align_up(o.empty + 4ull * s.n_empty, kSectionAlign);
  o.ts = align_up(o.st0 + 4ull * (s.num_slices + 1), kSectionAlign);
  o.tiles = align_up(o.ts + 4ull * s.num_tiles, kSectionAlign);
  o.total = align_up(o.tiles + (uint64_t)s.num_tiles * tile_bytes(bits, G), kSectionAlign);
  return o;
}

void fill_desc(const BlobHeader& h, gqsa_desc_t* d) {
  static_assert(offsetof(gqsa_desc_t, blob_bytes) == offsetof(BlobHeader, blob_bytes), "desc mirror");
  static_assert(sizeof(gqsa_desc_t) == 128, "desc size");
  std::memcpy(d, &h, sizeof(gqsa_desc_t));
}

}  // namespace

extern "C" int gqsa_pack_size_ex(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, int32_t layout,
                                 size_t* blob_bytes) {
  int st = check_bsr_header(bsr);
  if (st) return st;
  if (!blob_bytes) return GQSA_ERR_BUFFER;
  if (row_begin < 0 || row_end < row_begin || row_end > bsr->rows) return GQSA_ERR_SHAPE;
  if (layout != GQSA_LAYOUT_STREAM && layout != GQSA_LAYOUT_TC) return GQSA_ERR_SHAPE;
  if ((st = validate(bsr, row_begin, row_end))) return st;
  if (layout == GQSA_LAYOUT_TC) return pack_tc_size(bsr, row_begin, row_end, blob_bytes);
  *blob_bytes = (size_t)offsets(make_slices(bsr, row_begin, row_end), bsr->bits, bsr->group_size).total;
  return GQSA_OK;
}

extern "C" int gqsa_pack_size(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, size_t* blob_bytes) {
  return gqsa_pack_size_ex(bsr, row_begin, row_end, GQSA_LAYOUT_STREAM, blob_bytes);
}

extern "C" int gqsa_pack(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, void* blob,
                         size_t blob_bytes, gqsa_desc_t* desc) {
  return gqsa_pack_ex(bsr, row_begin, row_end, GQSA_LAYOUT_STREAM, blob, blob_bytes, desc);
}

extern "C" int gqsa_pack_ex(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, int32_t layout, void* blob,
                            size_t blob_bytes, gqsa_desc_t* desc) {
  int st = check_bsr_header(bsr);
  if (st) return st;
  if (!blob) return GQSA_ERR_BUFFER;
  if (row_begin < 0 || row_end < row_begin || row_end > bsr->rows) return GQSA_ERR_SHAPE;
  if (layout != GQSA_LAYOUT_STREAM && layout != GQSA_LAYOUT_TC) return GQSA_ERR_SHAPE;
  if ((st = validate(bsr, row_begin, row_end))) return st;
  if (layout == GQSA_LAYOUT_TC) return pack_tc(bsr, row_begin, row_end, blob, blob_bytes, desc);
  const Slices s = make_slices(bsr, row_begin, row_end);
  const Offsets o = offsets(s, bsr->bits, bsr->group_size);
  if (blob_bytes < o.total) return GQSA_ERR_BUFFER;
  uint8_t* out = static_cast<uint8_t*>(blob);
  std::memset(out, 0, o.total);
  const int64_t g_begin = bsr->row_index[row_begin];
  const int bits = bsr->bits, G = bsr->group_size, cb = group_code_bytes(bits, G), S = s.lanes_per_row;
  const int tb = tile_bytes(bits, G);

  BlobHeader h{};
  h.magic = kMagic;
  h.version = kVersion;
  h.rows = s.rows;
  h.cols = bsr->cols;
  h.group_size = G;
  h.bits = bits;
  h.nnzg = (int64_t)bsr->row_index[row_end] - g_begin;
  h.tile_groups = kTileGroups;
  h.num_tiles = s.num_tiles;
  h.n_nzrows = s.n_nz;
  h.n_empty = s.n_empty;
  h.tile_bytes = tb;
  h.flags = (int32_t)((G == kGroup ? kFlagTargetDeal : 0u) | ((uint32_t)S << kFlagLanesPerRowShift));
  h.row_begin = row_begin;
  h.row_end = row_end;
  h.num_slices = s.num_slices;
  h.off_row_index = o.ri;
  h.off_perm = o.perm;
  h.off_empty = o.empty;
  h.off_slice_tile0 = o.st0;
  h.off_tile_slice = o.ts;
  h.off_tiles = o.tiles;
  h.blob_bytes = o.total;
  std::memcpy(out, &h, sizeof(h));

  int32_t* ri = reinterpret_cast<int32_t*>(out + o.ri);
  for (int32_t r = 0; r <= s.rows; ++r) ri[r] = (int32_t)(bsr->row_index[row_begin + r] - g_begin);
  int32_t* perm = reinterpret_cast<int32_t*>(out + o.perm);
  for (int64_t i = 0; i < (int64_t)kLanes * s.num_slices; ++i) perm[i] = -1;
  int32_t* em = reinterpret_cast<int32_t*>(out + o.empty);
  for (int32_t i = 0; i < s.n_empty; ++i) em[i] = s.empty[i];
  int32_t* st0 = reinterpret_cast<int32_t*>(out + o.st0);
  int32_t* ts = reinterpret_cast<int32_t*>(out + o.ts);
  for (int32_t sl = 0; sl <= s.num_slices; ++sl) st0[sl] = s.tile0[sl];
  for (int32_t sl = 0; sl < s.num_slices; ++sl)
    for (int32_t t = s.tile0[sl]; t < s.tile0[sl + 1]; ++t) ts[t] = sl;

  const uint16_t padf = (uint16_t)pad_field(bsr->cols);  // the zero block after x
  std::vector<int64_t> deal;          // [lane][slot] source group, -1 = padding
  for (int32_t sl = 0; sl < s.num_slices; ++sl) {
    int32_t row_of_lane[kLanes];
    for (int l = 0; l < kLanes; ++l) {
      const int64_t k = (int64_t)sl * s.rows_per_slice + l / S;
      row_of_lane[l] = k < s.n_nz ? s.order[k] : -1;
      perm[(int64_t)sl * kLanes + l] = row_of_lane[l];
    }
    const int32_t nt = s.tile0[sl + 1] - s.tile0[sl];
    const int64_t L = (int64_t)nt * kPerLane;  // slots per lane
    deal.assign((size_t)kLanes * L, -1);
    // Bank-aware dealing (kFlagTargetDeal): at slot j lane l wants a group
    // whose column c has c mod 8 == want8(l, j) = (((l mod 8) / 2 + j) mod 4)
    // + 4 * ((l / 8) mod 2), read with swap = l mod 2.  The chunk index
    // f = 2c + swap then covers the 8 bank quads of every quarter-warp once
    // (conflict-free LDS.128) and 16 distinct f mod 16 per half-warp
    // (conflict-free LDS.64 of the column sums); the residue a lane wants
    // rotates with j, so a row's buckets drain evenly.
    for (int l0 = 0; l0 < kLanes; l0 += S) {
      const int32_t row = row_of_lane[l0];
      if (row < 0) continue;
      const int64_t g0 = bsr->row_index[row_begin + row], n = s.count[row];
      if (G != kGroup) {  // G = 8 / 32: CSR order, round robin over the row's lanes
        for (int64_t p = 0; p < n; ++p) deal[(size_t)(l0 + p % S) * L + p / S] = g0 + p;
        continue;
      }
      std::vector<int64_t> bucket[8];
      size_t head[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int64_t g = g0; g < g0 + n; ++g) bucket[bsr->group_cols[g] & 7].push_back(g);
      int64_t left = n;
      for (int64_t j = 0; j < L && left > 0; ++j) {
        for (int k = 0; k < S && left > 0; ++k) {
          const int l = l0 + k;
          const int want = (int)((((l & 7) >> 1) + j) & 3) + 4 * ((l >> 3) & 1);
          int b = want;
          if (head[b] == bucket[b].size()) b = want ^ 4;
          if (head[b] == bucket[b].size()) {  // most populated remaining bucket
            b = 0;
            for (int c = 1; c < 8; ++c)
              if (bucket[c].size() - head[c] > bucket[b].size() - head[b]) b = c;
          }
          deal[(size_t)l * L + j] = bucket[b][head[b]++];
          --left;
        }
      }
    }
    for (int32_t tau = 0; tau < nt; ++tau) {
      const int32_t t = s.tile0[sl] + tau;
      uint8_t* tile = out + o.tiles + (uint64_t)t * tb;
      for (int u = 0; u < kPerLane; ++u) {
        for (int l = 0; l < kLanes; ++l) {
          const int64_t g = deal[(size_t)l * L + (int64_t)tau * kPerLane + u];
          uint16_t* col = reinterpret_cast<uint16_t*>(tile + off_cols_g(bits, G, l, u));
          if (g < 0) {  // padding: codes, s, z zero; reads the zero block (contributes exactly 0)
            *col = padf;
            continue;
          }
          const uint32_t swap = lane_rot(G, l);
          const uint8_t* src = bsr->codes + g * cb;
          uint8_t* dst = tile + off_codes_g(bits, G, l, u);
          if (G == 32) {  // code word k <- the group's word (k + rot) mod 4 (chunk read order)
            for (int k = 0; k < 4; ++k) std::memcpy(dst + 4 * k, src + 4 * ((k + swap) & 3), 4);
          } else if (swap) {
            std::memcpy(dst, src + cb / 2, cb / 2);
            std::memcpy(dst + cb / 2, src, cb / 2);
          } else {
            std::memcpy(dst, src, cb);
          }
          uint16_t* sz = reinterpret_cast<uint16_t*>(tile + off_sz_g(bits, G, l, u));
          sz[0] = bsr->scales_f16[g];
          sz[1] = bsr->zeros_f16[g];
          *col = (uint16_t)col_field(G, bsr->group_cols[g], swap);  // byte offset of the first x chunk
        }
      }
    }
  }
  if (desc) fill_desc(h, desc);
  return GQSA_OK;
}

extern "C" int gqsa_read_desc(const void* blob, size_t blob_bytes, gqsa_desc_t* desc) {
  if (!blob || !desc) return GQSA_ERR_BUFFER;
  if (blob_bytes < (size_t)kHeaderBytes) return GQSA_ERR_BUFFER;
  BlobHeader h;
  std::memcpy(&h, blob, sizeof(h));
  if (h.magic != kMagic || h.version != (uint32_t)kVersion) return GQSA_ERR_VALIDATION;
  if (!group_supported(h.bits, h.group_size)) return GQSA_ERR_UNSUPPORTED;
  if (h.rows < 0 || h.cols <= 0 || h.cols % h.group_size || h.cols > kMaxCols || h.nnzg < 0 || h.num_tiles < 0)
    return GQSA_ERR_VALIDATION;
  if ((uint32_t)h.flags & kFlagTC) {  // LAYOUT-TC (the small-batch tensor-core layout)
    if (h.blob_bytes > blob_bytes) return GQSA_ERR_BUFFER;
    const int st = read_desc_tc(h, static_cast<const uint8_t*>(blob));
    if (st) return st;
    fill_desc(h, desc);
    return GQSA_OK;
  }
  if (h.tile_groups != kTileGroups || h.tile_bytes != tile_bytes(h.bits, h.group_size)) return GQSA_ERR_VALIDATION;
  if (h.rows < 0 || h.cols <= 0 || h.cols % h.group_size || h.cols > kMaxCols || h.nnzg < 0)
    return GQSA_ERR_VALIDATION;
  if (h.n_nzrows < 0 || h.n_empty < 0 || h.n_nzrows + h.n_empty != h.rows) return GQSA_ERR_VALIDATION;
  if (h.nnzg < h.n_nzrows || h.num_tiles < 0) return GQSA_ERR_VALIDATION;
  const int S = (int)((uint32_t)h.flags >> kFlagLanesPerRowShift) & 0xff;
  if (S < 1 || S > kLanes || (S & (S - 1))) return GQSA_ERR_VALIDATION;
  const int64_t slices = (h.n_nzrows + kLanes / S - 1) / (kLanes / S);
  if (h.num_slices != slices || h.num_tiles < slices) return GQSA_ERR_VALIDATION;
  if (h.off_row_index < (uint64_t)kHeaderBytes || h.off_perm < h.off_row_index + 4ull * (h.rows + 1) ||
      h.off_empty < h.off_perm + 4ull * kLanes * slices || h.off_slice_tile0 < h.off_empty + 4ull * h.n_empty ||
      h.off_tile_slice < h.off_slice_tile0 + 4ull * (slices + 1) ||
      h.off_tiles < h.off_tile_slice + 4ull * h.num_tiles || h.off_tiles % kSectionAlign ||
      h.blob_bytes < h.off_tiles + (uint64_t)h.num_tiles * h.tile_bytes)
    return GQSA_ERR_VALIDATION;
  if (h.blob_bytes > blob_bytes) return GQSA_ERR_BUFFER;
  // slice tables: slice_tile0 is a strictly increasing cover of [0, num_tiles)
  // and tile_slice its inverse (the kernel trusts both)
  const uint8_t* b = static_cast<const uint8_t*>(blob);
  const int32_t* st0 = reinterpret_cast<const int32_t*>(b + h.off_slice_tile0);
  const int32_t* ts = reinterpret_cast<const int32_t*>(b + h.off_tile_slice);
  if (st0[0] != 0 || st0[slices] != h.num_tiles) return GQSA_ERR_VALIDATION;
  for (int64_t sl = 0; sl < slices; ++sl) {
    if (st0[sl + 1] <= st0[sl]) return GQSA_ERR_VALIDATION;
    for (int32_t t = st0[sl]; t < st0[sl + 1]; ++t)
      if (ts[t] != (int32_t)sl) return GQSA_ERR_VALIDATION;
  }
  fill_desc(h, desc);
  return GQSA_OK;
}

extern "C" int gqsa_unpack(const void* blob, size_t blob_bytes, gqsa_bsr_t* out) {
  gqsa_desc_t d;
  int st = gqsa_read_desc(blob, blob_bytes, &d);
  if (st) return st;
  if (!out) return GQSA_ERR_BUFFER;
  int32_t* o_ri = const_cast<int32_t*>(out->row_index);
  uint16_t* o_gc = const_cast<uint16_t*>(out->group_cols);
  uint8_t* o_codes = const_cast<uint8_t*>(out->codes);
  uint16_t* o_s = const_cast<uint16_t*>(out->scales_f16);
  uint16_t* o_z = const_cast<uint16_t*>(out->zeros_f16);
  if (!o_ri || (d.nnzg > 0 && (!o_gc || !o_codes || !o_s || !o_z))) return GQSA_ERR_BUFFER;
  if ((uint32_t)d.flags & kFlagTC) {
    st = unpack_tc(d, static_cast<const uint8_t*>(blob), out);
    return st ? st : validate(out, 0, d.rows);
  }

  const uint8_t* b = static_cast<const uint8_t*>(blob);
  const int32_t* ri = reinterpret_cast<const int32_t*>(b + d.off_row_index);
  const int32_t* perm = reinterpret_cast<const int32_t*>(b + d.off_perm);
  const int32_t* em = reinterpret_cast<const int32_t*>(b + d.off_empty);
  const int32_t* ts = reinterpret_cast<const int32_t*>(b + d.off_tile_slice);
  const int bits = d.bits, GS = d.group_size, cb = group_code_bytes(bits, GS);
  const uint16_t padf = (uint16_t)pad_field(d.cols);

  struct G {
    uint16_t col, s, z;
    const uint8_t* codes;
    bool swap;     // G = 16: halves exchanged
    uint32_t rot;  // G = 32: code words rotated
  };
  std::vector<std::vector<G>> rows(d.rows);
  for (int32_t t = 0; t < d.num_tiles; ++t) {
    const uint8_t* tile = b + d.off_tiles + (uint64_t)t * d.tile_bytes;
    const int32_t slice = ts[t];
    for (int u = 0; u < kPerLane; ++u) {
      for (int l = 0; l < kLanes; ++l) {
        const int32_t row = perm[(int64_t)slice * kLanes + l];
        const uint16_t* sz = reinterpret_cast<const uint16_t*>(tile + off_sz_g(bits, GS, l, u));
        const uint16_t col = *reinterpret_cast<const uint16_t*>(tile + off_cols_g(bits, GS, l, u));
        const uint8_t* src = tile + off_codes_g(bits, GS, l, u);
        if (sz[0] == 0) {  // padding (a kept group always has s > 0)
          if (sz[1] || col != padf) return GQSA_ERR_VALIDATION;
          for (int i = 0; i < cb; ++i)
            if (src[i]) return GQSA_ERR_VALIDATION;
          continue;
        }
        if (row < 0 || row >= d.rows) return GQSA_ERR_VALIDATION;
        if ((col & 15u) || col >= 2u * (uint32_t)d.cols) return GQSA_ERR_VALIDATION;
        if (GS == kGroup) {
          rows[row].push_back(G{(uint16_t)(col >> 5), sz[0], sz[1], src, ((col >> 4) & 1u) != 0, 0});
        } else if (GS == 8) {
          rows[row].push_back(G{(uint16_t)(col >> 4), sz[0], sz[1], src, false, 0});
        } else {
          if (((col >> 4) & 3u) != lane_rot(GS, l)) return GQSA_ERR_VALIDATION;
          rows[row].push_back(G{(uint16_t)(col >> 6), sz[0], sz[1], src, false, (col >> 4) & 3u});
        }
      }
    }
  }
  // row order inside the stream is a rotation; CSR order is ascending column
  int64_t acc = 0;
  int32_t iem = 0, n_nz = 0;
  for (int32_t r = 0; r < d.rows; ++r) {
    if (ri[r] != acc) return GQSA_ERR_VALIDATION;
    o_ri[r] = (int32_t)acc;
    auto& v = rows[r];
    std::sort(v.begin(), v.end(), [](const G& a, const G& c) { return a.col < c.col; });
    if (v.empty()) {
      if (iem >= d.n_empty || em[iem++] != r) return GQSA_ERR_VALIDATION;
    } else {
      ++n_nz;
    }
    for (const G& g : v) {
      if (acc >= d.nnzg) return GQSA_ERR_VALIDATION;
      o_gc[acc] = g.col;
      o_s[acc] = g.s;
      o_z[acc] = g.z;
      uint8_t* dst = o_codes + acc * cb;
      if (GS == 32) {  // stored word k is the group's word (k + rot) mod 4
        for (int k = 0; k < 4; ++k) std::memcpy(dst + 4 * ((k + g.rot) & 3), g.codes + 4 * k, 4);
      } else if (g.swap) {
        std::memcpy(dst, g.codes + cb / 2, cb / 2);
        std::memcpy(dst + cb / 2, g.codes, cb / 2);
      } else {
        std::memcpy(dst, g.codes, cb);
      }
      ++acc;
    }
  }
  if (acc != d.nnzg || ri[d.rows] != acc || n_nz != d.n_nzrows) return GQSA_ERR_VALIDATION;
  o_ri[d.rows] = (int32_t)acc;
  out->rows = d.rows;
  out->cols = d.cols;
  out->group_size = d.group_size;
  out->bits = d.bits;
  out->nnzg = d.nnzg;
  return validate(out, 0, d.rows);
}

extern "C" const char* gqsa_status_string(int status) {
  switch (status) {
    case GQSA_OK: return "ok";
    case GQSA_ERR_SHAPE: return "shape error";
    case GQSA_ERR_VALIDATION: return "validation error";
    case GQSA_ERR_UNSUPPORTED: return "unsupported configuration";
    case GQSA_ERR_BUFFER: return "buffer error";
    case GQSA_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

extern "C" int gqsa_version(void) { return GQSA_VERSION; }
