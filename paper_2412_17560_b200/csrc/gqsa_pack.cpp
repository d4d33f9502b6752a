// gqsa_pack.cpp -- host packer, unpacker and validator for LAYOUT v1.
//
// Offline pre-processing ("quantized weights are grouped by size
// G and saved ... along with scaling factors and zero points"): the plain BSR
// is validated and rewritten as a blob of
// 128-group tile records in CSR stream order.  gqsa_unpack is
// its exact inverse.  No device code here.
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/gqsa.h"
#include "gqsa_layout.h"

using namespace gqsa;

namespace {

inline uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

inline bool f16_finite(uint16_t h) { return ((h >> 10) & 0x1f) != 0x1f; }
inline bool f16_positive(uint16_t h) { return !(h & 0x8000) && (h & 0x7fff) != 0; }

struct Plan {
  int32_t rows, cols, bits;
  int64_t g_begin, nnzg;
  int32_t num_tiles, n_nz, n_empty;
  uint64_t off_ri, off_nz, off_empty, off_tiles, total;
};

int check_bsr_header(const gqsa_bsr_t* b) {
  if (!b) return GQSA_ERR_BUFFER;
  if (b->rows < 0 || b->cols <= 0 || b->group_size <= 0 || b->nnzg < 0) return GQSA_ERR_SHAPE;
  if (b->group_size != kGroup || (b->bits != 4 && b->bits != 2)) return GQSA_ERR_UNSUPPORTED;
  if (b->cols % b->group_size) return GQSA_ERR_SHAPE;
  if (b->cols / kGroup > 32767) return GQSA_ERR_UNSUPPORTED;  // col field = 2c+swap in u16
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

Plan make_plan(const gqsa_bsr_t* b, int32_t r0, int32_t r1) {
  Plan p{};
  p.rows = r1 - r0;
  p.cols = b->cols;
  p.bits = b->bits;
  p.g_begin = b->row_index[r0];
  p.nnzg = (int64_t)b->row_index[r1] - p.g_begin;
  p.num_tiles = (int32_t)((p.nnzg + kTileGroups - 1) / kTileGroups);
  p.n_nz = 0;
  for (int32_t r = r0; r < r1; ++r) p.n_nz += (b->row_index[r + 1] > b->row_index[r]);
  p.n_empty = p.rows - p.n_nz;
  p.off_ri = kHeaderBytes;
  p.off_nz = align_up(p.off_ri + 4ull * (p.rows + 1), kSectionAlign);
  p.off_empty = align_up(p.off_nz + 4ull * p.n_nz, kSectionAlign);
  p.off_tiles = align_up(p.off_empty + 4ull * p.n_empty, kSectionAlign);
  p.total = align_up(p.off_tiles + (uint64_t)p.num_tiles * tile_bytes(p.bits), kSectionAlign);
  return p;
}

void fill_desc(const BlobHeader& h, gqsa_desc_t* d) {
  static_assert(offsetof(gqsa_desc_t, blob_bytes) == offsetof(BlobHeader, blob_bytes), "desc mirror");
  static_assert(sizeof(gqsa_desc_t) == 104, "desc size");
  std::memcpy(d, &h, sizeof(gqsa_desc_t));
}

}  // namespace

extern "C" int gqsa_pack_size(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end,
                              size_t* blob_bytes) {
  int st = check_bsr_header(bsr);
  if (st) return st;
  if (!blob_bytes) return GQSA_ERR_BUFFER;
  if (row_begin < 0 || row_end < row_begin || row_end > bsr->rows) return GQSA_ERR_SHAPE;
  if ((st = validate(bsr, row_begin, row_end))) return st;
  *blob_bytes = (size_t)make_plan(bsr, row_begin, row_end).total;
  return GQSA_OK;
}

extern "C" int gqsa_pack(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, void* blob,
                         size_t blob_bytes, gqsa_desc_t* desc) {
  int st = check_bsr_header(bsr);
  if (st) return st;
  if (!blob) return GQSA_ERR_BUFFER;
  if (row_begin < 0 || row_end < row_begin || row_end > bsr->rows) return GQSA_ERR_SHAPE;
  if ((st = validate(bsr, row_begin, row_end))) return st;
  const Plan p = make_plan(bsr, row_begin, row_end);
  if (blob_bytes < p.total) return GQSA_ERR_BUFFER;
  uint8_t* out = static_cast<uint8_t*>(blob);
  std::memset(out, 0, p.total);

  BlobHeader h{};
  h.magic = kMagic;
  h.version = kVersion;
  h.rows = p.rows;
  h.cols = p.cols;
  h.group_size = kGroup;
  h.bits = p.bits;
  h.nnzg = p.nnzg;
  h.tile_groups = kTileGroups;
  h.num_tiles = p.num_tiles;
  h.n_nzrows = p.n_nz;
  h.n_empty = p.n_empty;
  h.tile_bytes = tile_bytes(p.bits);
  h.flags = kFlagLaneParitySwap;
  h.row_begin = row_begin;
  h.row_end = row_end;
  h.off_row_index = p.off_ri;
  h.off_nzrow = p.off_nz;
  h.off_empty = p.off_empty;
  h.off_tiles = p.off_tiles;
  h.blob_bytes = p.total;
  std::memcpy(out, &h, sizeof(h));

  // Row sections (rebased to the shard).
  int32_t* ri = reinterpret_cast<int32_t*>(out + p.off_ri);
  int32_t* nz = reinterpret_cast<int32_t*>(out + p.off_nz);
  int32_t* em = reinterpret_cast<int32_t*>(out + p.off_empty);
  std::vector<int32_t> row_of(p.nnzg);      // local row of each stream position
  std::vector<int32_t> ord_of_row(p.rows);  // ordinal among non-empty rows
  int32_t inz = 0, iem = 0;
  for (int32_t r = 0; r < p.rows; ++r) {
    const int64_t a = bsr->row_index[row_begin + r] - p.g_begin;
    const int64_t e = bsr->row_index[row_begin + r + 1] - p.g_begin;
    ri[r] = (int32_t)a;
    if (e > a) {
      ord_of_row[r] = inz;
      nz[inz++] = r;
    } else {
      ord_of_row[r] = -1;
      em[iem++] = r;
    }
    for (int64_t g = a; g < e; ++g) row_of[g] = r;
  }
  ri[p.rows] = (int32_t)p.nnzg;

  // Tile records.
  const int bits = p.bits;
  const int cb = group_code_bytes(bits);
  for (int32_t t = 0; t < p.num_tiles; ++t) {
    uint8_t* tile = out + p.off_tiles + (uint64_t)t * tile_bytes(bits);
    uint32_t segmask[kPerLane] = {0, 0, 0, 0};
    const int64_t p0 = (int64_t)t * kTileGroups;
    const int32_t m0 = ord_of_row[row_of[p0]];
    for (int u = 0; u < kPerLane; ++u) {
      for (int l = 0; l < kLanes; ++l) {
        const int64_t pos = p0 + u * kLanes + l;
        if (pos >= p.nnzg) continue;  // padding group: all zero
        const int64_t g = p.g_begin + pos;  // index into the source BSR
        if (pos == 0 || row_of[pos] != row_of[pos - 1]) segmask[u] |= 1u << l;
        const uint32_t swap = (uint32_t)(l & 1);  // kFlagLaneParitySwap
        // codes: the group's G*n/8 bytes, halves exchanged when swap = 1
        const uint8_t* src = bsr->codes + g * cb;
        uint8_t* dst = tile + off_codes(bits, l, u);
        if (swap) {
          std::memcpy(dst, src + cb / 2, cb / 2);
          std::memcpy(dst + cb / 2, src, cb / 2);
        } else {
          std::memcpy(dst, src, cb);
        }
        uint16_t* sz = reinterpret_cast<uint16_t*>(tile + off_sz(bits) + l * 16 + u * 4);
        sz[0] = bsr->scales_f16[g];
        sz[1] = bsr->zeros_f16[g];
        uint16_t* col = reinterpret_cast<uint16_t*>(tile + off_cols(bits) + l * 8 + u * 2);
        *col = (uint16_t)((bsr->group_cols[g] << 1) | swap);
      }
    }
    std::memcpy(tile, segmask, sizeof(segmask));
    std::memcpy(tile + 16, &m0, 4);
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
  if (h.group_size != kGroup || (h.bits != 4 && h.bits != 2)) return GQSA_ERR_UNSUPPORTED;
  if (h.tile_groups != kTileGroups || h.tile_bytes != tile_bytes(h.bits)) return GQSA_ERR_VALIDATION;
  if (h.rows < 0 || h.cols <= 0 || h.cols % kGroup || h.nnzg < 0) return GQSA_ERR_VALIDATION;
  if ((int64_t)h.num_tiles != (h.nnzg + kTileGroups - 1) / kTileGroups) return GQSA_ERR_VALIDATION;
  if (h.n_nzrows < 0 || h.n_empty < 0 || h.n_nzrows + h.n_empty != h.rows) return GQSA_ERR_VALIDATION;
  if (h.nnzg < h.n_nzrows) return GQSA_ERR_VALIDATION;
  if (h.off_row_index < (uint64_t)kHeaderBytes || h.off_nzrow < h.off_row_index + 4ull * (h.rows + 1) ||
      h.off_empty < h.off_nzrow + 4ull * h.n_nzrows || h.off_tiles < h.off_empty + 4ull * h.n_empty ||
      h.off_tiles % kSectionAlign ||
      h.blob_bytes < h.off_tiles + (uint64_t)h.num_tiles * h.tile_bytes)
    return GQSA_ERR_VALIDATION;
  if (h.blob_bytes > blob_bytes) return GQSA_ERR_BUFFER;
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

  const uint8_t* b = static_cast<const uint8_t*>(blob);
  const int32_t* ri = reinterpret_cast<const int32_t*>(b + d.off_row_index);
  const int32_t* nz = reinterpret_cast<const int32_t*>(b + d.off_nzrow);
  const int32_t* em = reinterpret_cast<const int32_t*>(b + d.off_empty);
  const int bits = d.bits, cb = group_code_bytes(bits);

  // Rebuild per-row counts from the tile stream alone.
  std::vector<int64_t> count(d.rows, 0);
  int64_t m = -1;  // current row ordinal
  for (int32_t t = 0; t < d.num_tiles; ++t) {
    const uint8_t* tile = b + d.off_tiles + (uint64_t)t * d.tile_bytes;
    uint32_t segmask[kPerLane];
    int32_t m0;
    std::memcpy(segmask, tile, sizeof(segmask));
    std::memcpy(&m0, tile + 16, 4);
    const int64_t p0 = (int64_t)t * kTileGroups;
    for (int u = 0; u < kPerLane; ++u) {
      for (int l = 0; l < kLanes; ++l) {
        const int64_t pos = p0 + u * kLanes + l;
        const bool start = (segmask[u] >> l) & 1u;
        const uint16_t* sz = reinterpret_cast<const uint16_t*>(tile + off_sz(bits) + l * 16 + u * 4);
        const uint16_t col = *reinterpret_cast<const uint16_t*>(tile + off_cols(bits) + l * 8 + u * 2);
        const uint8_t* src = tile + off_codes(bits, l, u);
        if (pos >= d.nnzg) {  // padding must be all zero
          if (start || sz[0] || sz[1] || col) return GQSA_ERR_VALIDATION;
          for (int i = 0; i < cb; ++i)
            if (src[i]) return GQSA_ERR_VALIDATION;
          continue;
        }
        if (pos == 0 && !start) return GQSA_ERR_VALIDATION;
        if (start) ++m;
        if (u == 0 && l == 0 && m0 != m) return GQSA_ERR_VALIDATION;
        if (m < 0 || m >= d.n_nzrows) return GQSA_ERR_VALIDATION;
        const int32_t row = nz[m];
        if (row < 0 || row >= d.rows) return GQSA_ERR_VALIDATION;
        count[row]++;
        const uint32_t swap = col & 1u;
        o_gc[pos] = (uint16_t)(col >> 1);
        o_s[pos] = sz[0];
        o_z[pos] = sz[1];
        uint8_t* dst = o_codes + pos * cb;
        if (swap) {
          std::memcpy(dst, src + cb / 2, cb / 2);
          std::memcpy(dst + cb / 2, src, cb / 2);
        } else {
          std::memcpy(dst, src, cb);
        }
      }
    }
  }
  if (m + 1 != d.n_nzrows) return GQSA_ERR_VALIDATION;
  // Offsets from counts; must equal the stored row_index; nzrow / empty lists
  // must agree with the counts.
  int64_t acc = 0;
  int32_t inz = 0, iem = 0;
  for (int32_t r = 0; r < d.rows; ++r) {
    if (ri[r] != acc) return GQSA_ERR_VALIDATION;
    o_ri[r] = (int32_t)acc;
    if (count[r] > 0) {
      if (inz >= d.n_nzrows || nz[inz++] != r) return GQSA_ERR_VALIDATION;
    } else {
      if (iem >= d.n_empty || em[iem++] != r) return GQSA_ERR_VALIDATION;
    }
    acc += count[r];
  }
  if (acc != d.nnzg || ri[d.rows] != acc) return GQSA_ERR_VALIDATION;
  o_ri[d.rows] = (int32_t)acc;
  // Validate rows of the rebuilt BSR (strictly increasing columns, finite s/z).
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
