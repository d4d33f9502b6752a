// gqsa_pack_tc.cpp -- host packer / unpacker / validator of LAYOUT-TC, the
// small-batch tensor-core layout (W4, G = 16).
//
// Offline pre-processing of the paper's BSR ("grouped by
// size G and saved ... along with scaling factors and zero points") for the
// batch 2-8 GEMM ("TensorCores (MMA) or CudaCores (FMA)"): rows
// are taken in blocks of 16 (the mma M dimension); the ITEMS of a block are
// the group columns kept by any of its rows, in ascending column order, each
// stored as the block's 16 x 16 code matrix at that column (rows that do not
// keep the column: codes 0, s = z = 0) in mma.m16n8k16 A-fragment order.  The
// kernel then multiplies one item by the 16 x B activation slice of its
// column on the tensor cores.  A block without any kept group gets one
// padding item so that its rows are written.  Padding items point at column
// cols / 16 (the zero block after the staged activations).
#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/gqsa.h"
#include "gqsa_layout.h"
#include "gqsa_pack_internal.h"

using namespace gqsa;

namespace {

inline uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

struct TcPlan {
  int32_t rows = 0, nb = 0, num_tiles = 0, n_empty = 0;
  std::vector<std::vector<uint16_t>> cols;  // per block: item columns (ascending)
  std::vector<int32_t> tile0;               // first tile of each block (+ sentinel)
  std::vector<int32_t> empty;               // empty rows
};

TcPlan plan_tc(const gqsa_bsr_t* b, int32_t r0, int32_t r1) {
  TcPlan t;
  t.rows = r1 - r0;
  t.nb = (t.rows + kTcRows - 1) / kTcRows;
  t.cols.resize(t.nb);
  t.tile0.resize(t.nb + 1);
  const uint16_t pad_col = (uint16_t)(b->cols / b->group_size);
  int64_t tiles = 0;
  for (int32_t blk = 0; blk < t.nb; ++blk) {
    std::vector<uint16_t>& c = t.cols[blk];
    for (int32_t r = blk * kTcRows; r < std::min(t.rows, (blk + 1) * kTcRows); ++r) {
      const int64_t g0 = b->row_index[r0 + r], g1 = b->row_index[r0 + r + 1];
      if (g1 == g0) t.empty.push_back(r);
      for (int64_t g = g0; g < g1; ++g) c.push_back(b->group_cols[g]);
    }
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    if (c.empty()) c.push_back(pad_col);  // a padding item: the block's rows are still written
    t.tile0[blk] = (int32_t)tiles;
    tiles += (int64_t)(c.size() + kTcItems - 1) / kTcItems;
  }
  t.tile0[t.nb] = (int32_t)tiles;
  t.num_tiles = (int32_t)tiles;
  t.n_empty = (int32_t)t.empty.size();
  return t;
}

struct TcOffsets {
  uint64_t ri, tcols, empty, bt0, tb, tiles, total;
};

TcOffsets tc_offsets(const TcPlan& t) {
  TcOffsets o;
  o.ri = kHeaderBytes;
  o.tcols = align_up(o.ri + 4ull * (t.rows + 1), kSectionAlign);
  o.empty = align_up(o.tcols + 2ull * kTcItems * t.num_tiles, kSectionAlign);
  o.bt0 = align_up(o.empty + 4ull * t.n_empty, kSectionAlign);
  o.tb = align_up(o.bt0 + 4ull * (t.nb + 1), kSectionAlign);
  o.tiles = align_up(o.tb + 4ull * t.num_tiles, kSectionAlign);
  o.total = align_up(o.tiles + (uint64_t)t.num_tiles * kTcTileBytes, kSectionAlign);
  return o;
}

int check_tc(const gqsa_bsr_t* b) {
  if (b->bits != 4 || b->group_size != kGroup) return GQSA_ERR_UNSUPPORTED;
  return GQSA_OK;
}

}  // namespace

namespace gqsa {

int pack_tc_size(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, size_t* blob_bytes) {
  const int st = check_tc(bsr);
  if (st) return st;
  *blob_bytes = (size_t)tc_offsets(plan_tc(bsr, row_begin, row_end)).total;
  return GQSA_OK;
}

int pack_tc(const gqsa_bsr_t* bsr, int32_t row_begin, int32_t row_end, void* blob, size_t blob_bytes,
            gqsa_desc_t* desc) {
  int st = check_tc(bsr);
  if (st) return st;
  const TcPlan t = plan_tc(bsr, row_begin, row_end);
  const TcOffsets o = tc_offsets(t);
  if (blob_bytes < o.total) return GQSA_ERR_BUFFER;
  uint8_t* out = static_cast<uint8_t*>(blob);
  std::memset(out, 0, o.total);
  const int64_t g_begin = bsr->row_index[row_begin];

  BlobHeader h{};
  h.magic = kMagic;
  h.version = kVersion;
  h.rows = t.rows;
  h.cols = bsr->cols;
  h.group_size = kGroup;
  h.bits = 4;
  h.nnzg = (int64_t)bsr->row_index[row_end] - g_begin;
  h.tile_groups = kTcItems * kTcRows;
  h.num_tiles = t.num_tiles;
  h.n_nzrows = t.rows - t.n_empty;
  h.n_empty = t.n_empty;
  h.tile_bytes = kTcTileBytes;
  h.flags = (int32_t)(kFlagTC | (1u << kFlagLanesPerRowShift));
  h.row_begin = row_begin;
  h.row_end = row_end;
  h.num_slices = t.nb;  // blocks play the role of slices
  h.off_row_index = o.ri;
  h.off_perm = o.tcols;  // LAYOUT-TC: the item columns u16 [tile][4]
  h.off_empty = o.empty;
  h.off_slice_tile0 = o.bt0;
  h.off_tile_slice = o.tb;
  h.off_tiles = o.tiles;
  h.blob_bytes = o.total;
  std::memcpy(out, &h, sizeof(h));

  int32_t* ri = reinterpret_cast<int32_t*>(out + o.ri);
  for (int32_t r = 0; r <= t.rows; ++r) ri[r] = (int32_t)(bsr->row_index[row_begin + r] - g_begin);
  int32_t* em = reinterpret_cast<int32_t*>(out + o.empty);
  for (int32_t i = 0; i < t.n_empty; ++i) em[i] = t.empty[i];
  int32_t* bt0 = reinterpret_cast<int32_t*>(out + o.bt0);
  int32_t* tb = reinterpret_cast<int32_t*>(out + o.tb);
  for (int32_t blk = 0; blk <= t.nb; ++blk) bt0[blk] = t.tile0[blk];
  for (int32_t blk = 0; blk < t.nb; ++blk)
    for (int32_t tt = t.tile0[blk]; tt < t.tile0[blk + 1]; ++tt) tb[tt] = blk;
  uint16_t* tcols = reinterpret_cast<uint16_t*>(out + o.tcols);
  const uint16_t pad_col = (uint16_t)(bsr->cols / kGroup);

  for (int32_t blk = 0; blk < t.nb; ++blk) {
    const std::vector<uint16_t>& cols = t.cols[blk];
    // group index of (block row rr, item) or -1
    const int nrows = std::min(kTcRows, t.rows - blk * kTcRows);
    std::vector<int64_t> gidx((size_t)kTcRows * cols.size(), -1);
    for (int rr = 0; rr < nrows; ++rr) {
      const int32_t r = row_begin + blk * kTcRows + rr;
      size_t it = 0;
      for (int64_t g = bsr->row_index[r]; g < bsr->row_index[r + 1]; ++g) {
        while (cols[it] != bsr->group_cols[g]) ++it;
        gidx[(size_t)rr * cols.size() + it] = g;
      }
    }
    const int32_t ntile = t.tile0[blk + 1] - t.tile0[blk];
    for (int32_t k = 0; k < ntile; ++k) {
      const int32_t tile_i = t.tile0[blk] + k;
      uint8_t* tile = out + o.tiles + (uint64_t)tile_i * kTcTileBytes;
      for (int u = 0; u < kTcItems; ++u) {
        const size_t item = (size_t)k * kTcItems + u;
        tcols[(size_t)tile_i * kTcItems + u] = item < cols.size() ? cols[item] : pad_col;
        if (item >= cols.size()) continue;  // padding item: all zero
        for (int lane = 0; lane < kLanes; ++lane) {
          uint32_t w = 0;
          for (int j = 0; j < 8; ++j) {
            const int rr = tc_nib_row(lane, j), kk = tc_nib_k(lane, j);
            const int64_t g = gidx[(size_t)rr * cols.size() + item];
            if (g < 0) continue;
            const uint32_t q = (bsr->codes[(g * kGroup + kk) / 2] >> (4 * ((g * kGroup + kk) & 1))) & 0xFu;
            w |= q << (4 * j);
          }
          std::memcpy(tile + lane * 16 + u * 4, &w, 4);
        }
        for (int pr = 0; pr < 8; ++pr) {  // (s, z) of rows pr and pr + 8
          uint16_t sz[4] = {0, 0, 0, 0};
          for (int h2 = 0; h2 < 2; ++h2) {
            const int64_t g = gidx[(size_t)(pr + 8 * h2) * cols.size() + item];
            if (g < 0) continue;
            sz[2 * h2] = bsr->scales_f16[g];
            sz[2 * h2 + 1] = bsr->zeros_f16[g];
          }
          std::memcpy(tile + 512 + pr * 32 + u * 8, sz, 8);
        }
      }
    }
  }
  if (desc) std::memcpy(desc, &h, sizeof(gqsa_desc_t));
  return GQSA_OK;
}

int read_desc_tc(const BlobHeader& h, const uint8_t* b) {
  if (h.bits != 4 || h.group_size != kGroup || h.tile_groups != kTcItems * kTcRows || h.tile_bytes != kTcTileBytes)
    return GQSA_ERR_VALIDATION;
  const int64_t nb = (h.rows + kTcRows - 1) / kTcRows;
  if (h.num_slices != nb || h.num_tiles < nb || h.n_empty < 0 || h.n_empty > h.rows ||
      h.n_nzrows + h.n_empty != h.rows)
    return GQSA_ERR_VALIDATION;
  if (h.off_row_index < (uint64_t)kHeaderBytes || h.off_perm < h.off_row_index + 4ull * (h.rows + 1) ||
      h.off_empty < h.off_perm + 2ull * kTcItems * h.num_tiles ||
      h.off_slice_tile0 < h.off_empty + 4ull * h.n_empty || h.off_tile_slice < h.off_slice_tile0 + 4ull * (nb + 1) ||
      h.off_tiles < h.off_tile_slice + 4ull * h.num_tiles || h.off_tiles % kSectionAlign ||
      h.blob_bytes < h.off_tiles + (uint64_t)h.num_tiles * kTcTileBytes)
    return GQSA_ERR_VALIDATION;
  const int32_t* bt0 = reinterpret_cast<const int32_t*>(b + h.off_slice_tile0);
  const int32_t* tb = reinterpret_cast<const int32_t*>(b + h.off_tile_slice);
  const uint16_t* tcols = reinterpret_cast<const uint16_t*>(b + h.off_perm);
  if (bt0[0] != 0 || bt0[nb] != h.num_tiles) return GQSA_ERR_VALIDATION;
  for (int64_t blk = 0; blk < nb; ++blk) {
    if (bt0[blk + 1] <= bt0[blk]) return GQSA_ERR_VALIDATION;
    for (int32_t t = bt0[blk]; t < bt0[blk + 1]; ++t)
      if (tb[t] != (int32_t)blk) return GQSA_ERR_VALIDATION;
  }
  for (int64_t i = 0; i < (int64_t)kTcItems * h.num_tiles; ++i)
    if ((int32_t)tcols[i] > h.cols / kGroup) return GQSA_ERR_VALIDATION;  // the kernel gathers x with it
  return GQSA_OK;
}

int unpack_tc(const gqsa_desc_t& d, const uint8_t* b, gqsa_bsr_t* out) {
  int32_t* o_ri = const_cast<int32_t*>(out->row_index);
  uint16_t* o_gc = const_cast<uint16_t*>(out->group_cols);
  uint8_t* o_codes = const_cast<uint8_t*>(out->codes);
  uint16_t* o_s = const_cast<uint16_t*>(out->scales_f16);
  uint16_t* o_z = const_cast<uint16_t*>(out->zeros_f16);
  const int32_t* ri = reinterpret_cast<const int32_t*>(b + d.off_row_index);
  const uint16_t* tcols = reinterpret_cast<const uint16_t*>(b + d.off_perm);
  const int32_t* bt0 = reinterpret_cast<const int32_t*>(b + d.off_slice_tile0);
  struct Grp {
    uint16_t col, s, z;
    uint8_t q[kGroup];
  };
  std::vector<std::vector<Grp>> rows(d.rows);
  const int nb = d.num_slices;
  for (int blk = 0; blk < nb; ++blk) {
    int last_col = -1;
    for (int32_t tt = bt0[blk]; tt < bt0[blk + 1]; ++tt) {
      const uint8_t* tile = b + d.off_tiles + (uint64_t)tt * kTcTileBytes;
      for (int u = 0; u < kTcItems; ++u) {
        const int col = tcols[(size_t)tt * kTcItems + u];
        bool any = false;
        for (int rr = 0; rr < kTcRows; ++rr) {
          uint16_t sz[2];
          std::memcpy(sz, tile + 512 + (rr & 7) * 32 + u * 8 + (rr >> 3) * 4, 4);
          if (sz[0] == 0) {  // not kept: zero scale, zero zero point and codes
            if (sz[1]) return GQSA_ERR_VALIDATION;
            continue;
          }
          const int row = blk * kTcRows + rr;
          if (row >= d.rows || col >= d.cols / kGroup) return GQSA_ERR_VALIDATION;
          Grp g{(uint16_t)col, sz[0], sz[1], {}};
          rows[row].push_back(g);
          any = true;
        }
        // codes: nibble j of lane L's word
        for (int lane = 0; lane < kLanes; ++lane) {
          uint32_t w;
          std::memcpy(&w, tile + lane * 16 + u * 4, 4);
          for (int j = 0; j < 8; ++j) {
            const int rr = tc_nib_row(lane, j), kk = tc_nib_k(lane, j);
            const uint8_t q = (w >> (4 * j)) & 0xF;
            const int row = blk * kTcRows + rr;
            if (row < d.rows && !rows[row].empty() && rows[row].back().col == col && rows[row].back().s != 0)
              rows[row].back().q[kk] = q;
            else if (q)
              return GQSA_ERR_VALIDATION;  // codes of a row that does not keep the column
          }
        }
        if (any) {
          if (col <= last_col) return GQSA_ERR_VALIDATION;  // items ascend by column
          last_col = col;
        }
      }
    }
  }
  int64_t acc = 0;
  int32_t n_empty = 0;
  for (int32_t r = 0; r < d.rows; ++r) {
    if (ri[r] != acc) return GQSA_ERR_VALIDATION;
    o_ri[r] = (int32_t)acc;
    if (rows[r].empty()) ++n_empty;
    for (const Grp& g : rows[r]) {
      if (acc >= d.nnzg) return GQSA_ERR_VALIDATION;
      o_gc[acc] = g.col;
      o_s[acc] = g.s;
      o_z[acc] = g.z;
      for (int k = 0; k < kGroup; k += 2) o_codes[(acc * kGroup + k) / 2] = (uint8_t)(g.q[k] | (g.q[k + 1] << 4));
      ++acc;
    }
  }
  if (acc != d.nnzg || ri[d.rows] != acc || n_empty != d.n_empty) return GQSA_ERR_VALIDATION;
  o_ri[d.rows] = (int32_t)acc;
  out->rows = d.rows;
  out->cols = d.cols;
  out->group_size = d.group_size;
  out->bits = d.bits;
  out->nnzg = d.nnzg;
  return GQSA_OK;
}

}  // namespace gqsa
