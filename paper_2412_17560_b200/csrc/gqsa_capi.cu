// gqsa_capi.cu -- extern "C" entry points that validate arguments, plan the
// Stream-K grid and launch the sm_100a kernel (see include/gqsa.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <vector>

#include "../../include/gqsa.h"
#include "gqsa_kernels.h"
#include "gqsa_layout.h"

using namespace gqsa;

static_assert(GQSA_MAX_ITEMS == kMaxItems, "item limit");
static_assert(GQSA_MAX_COLS == kMaxCols, "column limit");

namespace {

std::atomic<uint64_t> g_launches{0};
uint64_t* g_trace = nullptr;  // gqsa_debug_trace buffer (device), or null
size_t g_trace_bytes = 0;
std::mutex g_mu;
int g_sms[64] = {};
std::set<std::pair<int, const void*>> g_attr_set;  // (device, kernel) with the smem attribute set

int device_sms(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return 0;
  if (!g_sms[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    g_sms[dev] = v;
  }
  return g_sms[dev];
}
int current_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return device_sms(dev);
}

// Pipelined launches: GQSA_PIPELINE=0 off, 1 (default) for
// x_ready calls, 2 for every call at B <= 2 (A/B experiments).
int pipeline_mode() {
  static const int mode = [] {
    const char* e = std::getenv("GQSA_PIPELINE");
    return e && (e[0] == '0' || e[0] == '2') ? e[0] - '0' : 1;
  }();
  return mode;
}

// CTA-level fix-up of whole-SM Stream-K launches:
// GQSA_CTA_FIX=0 turns it off (the warp-level protocol; A/B experiments).
int cta_fix_mode() {
  static const int mode = [] {
    const char* e = std::getenv("GQSA_CTA_FIX");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return mode;
}

// Experiments (dependent launches, x_ready = 0): GQSA_DEP_PDL=0 launches them
// without programmatic dependent launch; GQSA_DEP_WAIT_FIRST=1 makes them wait
// for the previous kernel before their first weight loads.
int env_flag(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && e[0] ? (e[0] != '0') : dflt;
}
int dep_pdl() {
  static const int v = env_flag("GQSA_DEP_PDL", 1);
  return v;
}
// Slice-aligned CTA ranges for single-item whole-SM launches (no cross-CTA
// fix-up): by default at batch >= 2 (B = 1 measured neutral:
// the range lookups delay the first weight loads); GQSA_CTA_SLICEK=1 at every
// batch, 0 off.
bool cta_slicek_for(int Bc) {
  static const int v = [] {
    const char* e = std::getenv("GQSA_CTA_SLICEK");
    return e && e[0] ? (e[0] != '0' ? 1 : 0) : 2;
  }();
  return v == 1 || (v == 2 && Bc >= 2);
}
int dep_wait_first() {
  static const int v = env_flag("GQSA_DEP_WAIT_FIRST", 0);
  return v;
}

// Minimum tiles per warp when sizing a launch's warps per CTA (0 = off); A/B knob GQSA_MIN_TPW.
int min_tiles_per_warp() {
  static const int v = [] {
    const char* e = std::getenv("GQSA_MIN_TPW");
    return e ? std::atoi(e) : kMinTilesPerWarp;
  }();
  return v;
}

bool lanes_per_row_ok(uint32_t s) { return s >= 1 && s <= 32 && (s & (s - 1)) == 0; }

bool is_tc(const gqsa_desc_t* d) { return ((uint32_t)d->flags & kFlagTC) != 0; }

bool desc_ok(const gqsa_desc_t* d) {
  if (d && is_tc(d))
    return d->magic == kMagic && d->version == (uint32_t)kVersion && d->bits == 4 && d->group_size == kGroup &&
           d->tile_bytes == kTcTileBytes && d->rows >= 0 && d->cols > 0 && d->cols % kGroup == 0 &&
           d->cols <= kMaxCols && d->num_tiles >= 0 && d->num_slices == (d->rows + kTcRows - 1) / kTcRows;
  return d && d->magic == kMagic && d->version == (uint32_t)kVersion && group_supported(d->bits, d->group_size) &&
         d->tile_groups == kTileGroups && d->rows >= 0 && d->cols > 0 && d->cols % d->group_size == 0 &&
         d->cols <= kMaxCols && d->num_tiles >= 0 && d->num_slices >= 0 &&
         d->tile_bytes == tile_bytes(d->bits, d->group_size) &&
         lanes_per_row_ok(((uint32_t)d->flags >> kFlagLanesPerRowShift) & 0xff);
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Shared-memory bytes one item needs in a CTA for Bc batch columns.
int item_smem(const gqsa_desc_t* d, int Bc) {
  const int xrow = 2 * d->cols + kXPadBytes;
  const int pqrow = pq_row_bytes(Bc, d->group_size, d->cols);
  return (Bc * (xrow + pqrow) + 127) / 128 * 128;
}

// Workspace: [256 B reserved][cnt: kMaxWarpsBound u32][rec: kMaxWarpsBound x 2 x B x 32 u64]
size_t ws_bytes_for(int B) {
  return 256 + (size_t)kMaxWarpsBound * 4 + (size_t)kMaxWarpsBound * 2 * B * kLanes * 8;
}

struct Launch {
  int grid = 0, W = 0, active = 0, total_tiles = 0, part_q = 0, part_r = 0;
  int half = 0;  // pipelined mode: half of every SM, deferred writes
  size_t smem = 0, tab_offset = 0, defer_offset = 0;
};
// shared bytes of the per-CTA staging table (gqsa_device.cuh StageEntry x kMaxItems + 16)
constexpr size_t kStageTab = kMaxItems * 40 + 16;

// Stream-K grid over the concatenated tiles of `n` items at batch Bc, and the
// largest shared-memory footprint of any CTA (the items its range touches).
int plan_launch(const gqsa_desc_t* const* d, int n, int Bc, Launch* L, int half = 0) {
  const int sms = current_sms();
  if (sms <= 0) return GQSA_ERR_CUDA;
  L->half = half;
  L->W = warps_of(Bc, half);
  int64_t total = 0, n_empty = 0;
  for (int j = 0; j < n; ++j) {
    total += d[j]->num_tiles;
    n_empty += d[j]->n_empty;
  }
  if (total > INT32_MAX / 2) return GQSA_ERR_SHAPE;
  L->total_tiles = (int)total;
  // small launches: fewer warps per CTA (on every SM), so each warp streams
  // at least min_tiles_per_warp() tiles -- shorter fix-up chains, less
  // per-warp start-up, and CTAs small enough for the next launch to be
  // resident beside them
  const int mt = Bc == 1 ? min_tiles_per_warp() : 0;  // measured neutral-to-worse at batch 8
  if (mt > 0) L->W = (int)std::max<int64_t>(1, std::min<int64_t>(L->W, (total + (int64_t)sms * mt - 1) / ((int64_t)sms * mt)));
  const int warps = std::min(sms * L->W * (half ? 1 : full_ctas_for(Bc)), kMaxWarpsBound);
  L->active = (int)std::min<int64_t>(total, warps);
  L->part_q = L->active ? L->total_tiles / L->active : 0;
  L->part_r = L->active ? L->total_tiles % L->active : 0;
  L->grid = (L->active + L->W - 1) / L->W;
  if (L->grid == 0) {  // nnzg == 0 everywhere: only empty rows to write
    L->grid = (int)std::min<int64_t>(std::max<int64_t>(1, (n_empty + 32 * L->W - 1) / (32 * L->W)), sms);
  }
  // per-CTA footprint: packed touched items (mirrors item_smem_off on the device)
  size_t worst = 0;
  std::vector<int> tb(n), te(n);
  int acc = 0;
  for (int j = 0; j < n; ++j) {
    tb[j] = acc;
    acc += d[j]->num_tiles;
    te[j] = acc;
  }
  for (int c = 0; c * L->W < L->active; ++c) {
    const int w0 = c * L->W, w1 = std::min(w0 + L->W, L->active) - 1;
    const int t0 = w0 * L->part_q + std::min(w0, L->part_r);
    const int t1 = w1 * L->part_q + std::min(w1, L->part_r) + L->part_q + (w1 < L->part_r ? 1 : 0);
    size_t s = 0;
    for (int j = 0; j < n; ++j)
      if (tb[j] < t1 && te[j] > t0 && te[j] > tb[j]) s += (size_t)item_smem(d[j], Bc);
    worst = std::max(worst, s);
  }
  L->smem = worst + kStageTab;  // + the staging table
  L->tab_offset = worst;
  L->defer_offset = 0;
  if (!half && cta_fix_mode())  // the CTA-level fix-up reuses the staging area: [W][2][Bc][32] f32 + [W] i32
    L->smem = std::max(L->smem, (size_t)L->W * 2 * Bc * kLanes * 4 + (size_t)L->W * 4);
  if (half) {  // + the per-warp deferred-store buffers (16-B aligned)
    L->defer_offset = (L->smem + 15) / 16 * 16;
    L->smem = L->defer_offset + (size_t)L->W * defer_bytes_per_warp(Bc);
  }
  return GQSA_OK;
}

// The launch of n items at batch Bc under options o: the pipelined mode
// (half of every SM, deferred writes) when X is declared ready -- the launch
// may then overlap the previous one on the stream -- and its footprint fits
// pipe_ctas_for(Bc) times per SM; else the whole-SM launch.
int choose_launch(const gqsa_desc_t* const* d, int n, int Bc, const gqsa_options_t& o, Launch* L) {
  int st = GQSA_OK;
  const int mode = pipeline_mode();
  if (Bc <= 2 && (mode == 2 || (mode == 1 && o.x_ready))) {
    if ((st = plan_launch(d, n, Bc, L, 1))) return st;
    if (L->smem <= (size_t)half_smem_limit(Bc)) return GQSA_OK;
  }
  return plan_launch(d, n, Bc, L);
}

// Largest batch chunk whose footprint fits; the batch runs as ceil(B / Bc)
// balanced launches (each re-streams the weights: DESIGN.md §10).
int batch_chunk(const gqsa_desc_t* const* d, int n, int B, int* Bc_out, Launch* L) {
  for (int Bc = B; Bc >= 1; --Bc) {
    const int launches = (B + Bc - 1) / Bc;
    const int Bb = (B + launches - 1) / launches;  // balanced
    const int st = plan_launch(d, n, Bb, L);
    if (st) return st;
    if (L->smem <= (size_t)kMaxDynSmem) {
      *Bc_out = Bb;
      return GQSA_OK;
    }
  }
  return GQSA_ERR_UNSUPPORTED;
}

int set_attrs(const void* fn) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GQSA_ERR_CUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_attr_set.count({dev, fn})) return GQSA_OK;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem) != cudaSuccess ||
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared) !=
          cudaSuccess)
    return GQSA_ERR_CUDA;
  g_attr_set.insert({dev, fn});
  return GQSA_OK;
}

// Fused all-gather destinations of one item (n == 0: plain Y).
struct Peers {
  int n = 0;
  int mc = 0;  // y[0] is a multicast address
  int32_t row_offset = 0;
  void* y[kMaxPeers] = {};
};

// One launch over `n` items at batch Bc (x of every CTA's items fits).
// X/Y of item j start at batch column b0 (already folded into the pointers).
int launch_items(const gqsa_gemm_item_t* items, int n, int Bc, const gqsa_options_t& o, void* d_ws, void* stream,
                 const Peers* peers) {
  std::vector<const gqsa_desc_t*> d(n);
  for (int j = 0; j < n; ++j) d[j] = items[j].desc;
  Launch L;
  int st = choose_launch(d.data(), n, Bc, o, &L);
  if (st) return st;
  if (L.smem > (size_t)kMaxDynSmem) return GQSA_ERR_UNSUPPORTED;
  const int bits = d[0]->bits, G = d[0]->group_size;
  const void* fn = select_kernel(bits, G, Bc, L.half);
  if (!fn) return GQSA_ERR_UNSUPPORTED;
  if ((st = set_attrs(fn))) return st;

  Params p;
  std::memset(&p, 0, sizeof(p));
  int tile0 = 0, rows = 0;
  for (int j = 0; j < n; ++j) {
    const gqsa_desc_t* desc = d[j];
    const uint8_t* blob = static_cast<const uint8_t*>(items[j].d_blob);
    Item& it = p.item[j];
    it.tiles = blob + desc->off_tiles;
    it.perm = reinterpret_cast<const int32_t*>(blob + desc->off_perm);
    it.slice_tile0 = reinterpret_cast<const int32_t*>(blob + desc->off_slice_tile0);
    it.tile_slice = reinterpret_cast<const int32_t*>(blob + desc->off_tile_slice);
    it.empty = reinterpret_cast<const int32_t*>(blob + desc->off_empty);
    it.X = items[j].d_X;
    it.Y = items[j].d_Y;
    it.bias = items[j].d_bias;
    it.ldx = items[j].ldx;
    it.ldy = items[j].ldy;
    it.rows = desc->rows;
    it.cols = desc->cols;
    it.n_empty = desc->n_empty;
    it.lanes_per_row = ((uint32_t)desc->flags >> kFlagLanesPerRowShift) & 0xff;
    it.num_slices = desc->num_slices;
    it.tile_begin = tile0;
    tile0 += desc->num_tiles;
    it.tile_end = tile0;
    it.xrow = 2 * desc->cols + kXPadBytes;
    it.pqrow = pq_row_bytes(Bc, G, desc->cols);
    it.smem_bytes = item_smem(desc, Bc);
    rows += desc->rows;
    if (peers && peers->n) {
      it.n_peers = peers->n;
      it.peer_mc = peers->mc;
      it.row_offset = peers->row_offset;
      for (int k = 0; k < peers->n; ++k)  // batch chunk offset is folded into d_Y relative to peer 0
        it.peer_y[k] = reinterpret_cast<uint64_t>(peers->y[k]) +
                       (reinterpret_cast<uintptr_t>(items[j].d_Y) - reinterpret_cast<uintptr_t>(peers->y[0]));
    }
  }
  p.n_items = n;
  p.total_tiles = L.total_tiles;
  p.active_warps = L.active;
  p.part_q = L.part_q;
  p.part_r = L.part_r;
  p.slice_k = o.partition == GQSA_PARTITION_SLICE_K ? 1 : 0;
  p.out_f16 = o.out_f16;
  p.x_ready = o.x_ready;
  p.stage_tab_offset = (int32_t)L.tab_offset;
  p.defer_offset = (int32_t)L.defer_offset;
  p.cta_fix = (!L.half && !p.slice_k && cta_fix_mode()) ? 1 : 0;
  p.wait_first = (!o.x_ready && dep_wait_first()) ? 1 : 0;
  p.cta_slicek = (p.cta_fix && n == 1 && cta_slicek_for(Bc)) ? 1 : 0;
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  p.cnt = reinterpret_cast<uint32_t*>(ws + 256);
  p.rec = reinterpret_cast<unsigned long long*>(ws + 256 + (size_t)kMaxWarpsBound * 4);
  p.trace = (g_trace && g_trace_bytes >= (size_t)L.active * 64) ? g_trace : nullptr;
  if (rows == 0) return GQSA_OK;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(32 * L.W);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (o.x_ready || dep_pdl()) ? 1 : 0;
  void* args[] = {&p};
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) return GQSA_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return GQSA_OK;
}

int check_options(const gqsa_options_t& o) {
  if (o.partition != GQSA_PARTITION_STREAM_K && o.partition != GQSA_PARTITION_SLICE_K) return GQSA_ERR_SHAPE;
  if ((o.out_f16 != 0 && o.out_f16 != 1) || (o.x_ready != 0 && o.x_ready != 1) || o.reserved != 0)
    return GQSA_ERR_SHAPE;
  return GQSA_OK;
}

int check_item(const gqsa_gemm_item_t& it, int B, int out_f16, bool check_y = true) {
  if (!it.desc || !it.d_blob || !it.d_X || (check_y && !it.d_Y)) return GQSA_ERR_BUFFER;
  if (!desc_ok(it.desc)) return GQSA_ERR_VALIDATION;
  if (B < 1 || B > kMaxBatch) return GQSA_ERR_SHAPE;
  if (it.ldx < it.desc->cols || it.ldx % 8 || it.ldy < it.desc->rows) return GQSA_ERR_SHAPE;
  if (!aligned(it.d_blob, 256) || !aligned(it.d_X, 16) || (it.d_bias && !aligned(it.d_bias, 4)) ||
      (check_y && !aligned(it.d_Y, out_f16 ? 2 : 4)))
    return GQSA_ERR_BUFFER;
  return GQSA_OK;
}

// n items (same bits / G), all batch columns: batch chunks x item groups.
int run_grouped(const gqsa_gemm_item_t* items, int n, int B, const gqsa_options_t& o, void* d_ws, size_t ws_bytes,
                void* stream, const Peers* peers = nullptr) {
  if (!d_ws || !aligned(d_ws, 256)) return GQSA_ERR_BUFFER;
  if (ws_bytes < ws_bytes_for(B)) return GQSA_ERR_BUFFER;
  std::vector<const gqsa_desc_t*> d(n);
  for (int j = 0; j < n; ++j) d[j] = items[j].desc;
  Launch L;
  int Bc = B;
  int st = batch_chunk(d.data(), n, B, &Bc, &L);
  if (st == GQSA_ERR_UNSUPPORTED && n > 1) {  // too many activations for one CTA: split the items
    const int h = n / 2;
    if ((st = run_grouped(items, h, B, o, d_ws, ws_bytes, stream, peers))) return st;
    return run_grouped(items + h, n - h, B, o, d_ws, ws_bytes, stream, peers);
  }
  if (st) return st;
  const size_t es = o.out_f16 ? 2 : 4;
  std::vector<gqsa_gemm_item_t> chunk(items, items + n);
  for (int b0 = 0; b0 < B; b0 += Bc) {
    const int nb = std::min(Bc, B - b0);
    for (int j = 0; j < n; ++j) {
      chunk[j].d_X = items[j].d_X + (int64_t)b0 * items[j].ldx;
      chunk[j].d_Y = static_cast<uint8_t*>(items[j].d_Y) + (size_t)b0 * items[j].ldy * es;
    }
    if ((st = launch_items(chunk.data(), n, nb, o, d_ws, stream, peers))) return st;
  }
  return GQSA_OK;
}

// ---- LAYOUT-TC (small-batch tensor-core GEMM, gqsa_tc.cu)
// Shared memory of one LAYOUT-TC launch over Bc batch rows: x (+ a zero chunk
// per row) and, unless the column sums come from the mma (xq_mma), the X_c table.
size_t tc_smem(const gqsa_desc_t* d, int Bc, bool xq_mma) {
  const size_t xrow = 2 * (size_t)d->cols + 32;
  const size_t s = (size_t)Bc * xrow + (xq_mma ? 0 : ((size_t)d->cols / kGroup + 1) * 32);
  // the CTA-level fix-up reuses the staging area: [warps][2][4][32] f32 + [warps] i32
  return cta_fix_mode() ? std::max(s, (size_t)kTcWarps * 2 * 4 * kLanes * 4 + (size_t)kTcWarps * 4) : s;
}

// Batch chunking of a LAYOUT-TC GEMM: the largest balanced chunk whose x fits,
// preferring the X_c table; each extra launch re-streams the weights.
bool tc_chunking(const gqsa_desc_t* d, int B, int* Bc_out, int* launches_out, bool* xq_mma_out) {
  for (int Bc = B; Bc >= 1; --Bc) {
    const int launches = (B + Bc - 1) / Bc, Bb = (B + launches - 1) / launches;
    for (int xm = 0; xm < 2; ++xm) {
      if (tc_smem(d, Bb, xm != 0) <= (size_t)kMaxDynSmem) {
        *Bc_out = Bb;
        *launches_out = launches;
        *xq_mma_out = xm != 0;
        return true;
      }
    }
  }
  return false;
}

int run_tc(const gqsa_desc_t* d, const void* d_blob, const uint16_t* d_X, int B, int64_t ldx, void* d_Y, int64_t ldy,
           const float* d_bias, const gqsa_options_t& o, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_ws || !aligned(d_ws, 256)) return GQSA_ERR_BUFFER;
  if (ws_bytes < ws_bytes_for(std::max(B, 4))) return GQSA_ERR_BUFFER;
  const int sms = current_sms();
  if (sms <= 0) return GQSA_ERR_CUDA;
  int Bc = 0, launches = 0;
  bool xm = false;
  if (!tc_chunking(d, B, &Bc, &launches, &xm)) return GQSA_ERR_UNSUPPORTED;
  const size_t es = o.out_f16 ? 2 : 4;
  const uint8_t* blob = static_cast<const uint8_t*>(d_blob);
  for (int b0 = 0; b0 < B; b0 += Bc) {
    const int nb = std::min(Bc, B - b0);
    const void* fn = select_tc_kernel(nb, xm);
    if (!fn) return GQSA_ERR_UNSUPPORTED;
    int st = set_attrs(fn);
    if (st) return st;
    TcParams p;
    std::memset(&p, 0, sizeof(p));
    p.tiles = blob + d->off_tiles;
    p.tile_cols = reinterpret_cast<const uint16_t*>(blob + d->off_perm);
    p.block_tile0 = reinterpret_cast<const int32_t*>(blob + d->off_slice_tile0);
    p.tile_block = reinterpret_cast<const int32_t*>(blob + d->off_tile_slice);
    p.X = d_X + (int64_t)b0 * ldx;
    p.Y = static_cast<uint8_t*>(d_Y) + (size_t)b0 * ldy * es;
    p.bias = d_bias;
    p.ldx = ldx;
    p.ldy = ldy;
    p.rows = d->rows;
    p.cols = d->cols;
    p.num_tiles = d->num_tiles;
    p.nb = d->num_slices;
    const int warps = std::min(sms * kTcWarps, kMaxWarpsBound);
    p.active_warps = std::min(d->num_tiles, warps);
    p.part_q = p.active_warps ? d->num_tiles / p.active_warps : 0;
    p.part_r = p.active_warps ? d->num_tiles % p.active_warps : 0;
    p.slice_k = o.partition == GQSA_PARTITION_SLICE_K ? 1 : 0;
    p.out_f16 = o.out_f16;
    p.x_ready = o.x_ready;
    p.xrow = 2 * d->cols + 32;
    p.cta_fix = (!p.slice_k && cta_fix_mode()) ? 1 : 0;
    uint8_t* ws = static_cast<uint8_t*>(d_ws);
    p.cnt = reinterpret_cast<uint32_t*>(ws + 256);
    p.rec = reinterpret_cast<unsigned long long*>(ws + 256 + (size_t)kMaxWarpsBound * 4);
    p.trace = (g_trace && g_trace_bytes >= (size_t)p.active_warps * 64) ? g_trace : nullptr;
    if (d->rows == 0 || p.active_warps == 0) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((p.active_warps + kTcWarps - 1) / kTcWarps);
    cfg.blockDim = dim3(32 * kTcWarps);
    cfg.dynamicSmemBytes = tc_smem(d, nb, xm);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&p};
    if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) return GQSA_ERR_CUDA;
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return GQSA_OK;
}

}  // namespace

extern "C" int gqsa_workspace_size(const gqsa_desc_t* desc, int32_t batch, size_t* bytes) {
  if (!desc || !bytes) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (batch < 1 || batch > kMaxBatch) return GQSA_ERR_SHAPE;
  *bytes = ws_bytes_for(is_tc(desc) ? std::max(batch, 4) : batch);  // LAYOUT-TC: 4 values per lane
  return GQSA_OK;
}

extern "C" int gqsa_launch_plan(const gqsa_desc_t* desc, int32_t B, gqsa_plan_t* plan) {
  return gqsa_launch_plan_ex(desc, B, nullptr, plan);
}

extern "C" int gqsa_launch_plan_ex(const gqsa_desc_t* desc, int32_t B, const gqsa_options_t* opts,
                                   gqsa_plan_t* plan) {
  if (!desc || !plan) return GQSA_ERR_BUFFER;
  const gqsa_options_t o = opts ? *opts : gqsa_options_t{GQSA_PARTITION_STREAM_K, 0, 0, 0};
  if (check_options(o)) return GQSA_ERR_SHAPE;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (B < 1 || B > kMaxBatch) return GQSA_ERR_SHAPE;
  if (is_tc(desc)) {  // LAYOUT-TC: 16 warps per CTA, one CTA per SM, x of the batch chunk in shared memory
    const int sms = current_sms();
    if (sms <= 0) return GQSA_ERR_CUDA;
    int Bc = 0, launches = 0;
    bool xm = false;
    if (!tc_chunking(desc, B, &Bc, &launches, &xm)) return GQSA_ERR_UNSUPPORTED;
    std::memset(plan, 0, sizeof(*plan));
    plan->warps_per_cta = kTcWarps;
    plan->active_warps = std::min(desc->num_tiles, std::min(sms * kTcWarps, kMaxWarpsBound));
    plan->grid = (plan->active_warps + kTcWarps - 1) / kTcWarps;
    plan->num_tiles = desc->num_tiles;
    plan->smem_bytes = (int32_t)tc_smem(desc, Bc, xm);
    plan->x_in_smem = 1;
    plan->stages = kTcBufs;
    plan->ctas_per_sm = 1;
    plan->batch_per_launch = Bc;
    plan->launches = launches;
    return GQSA_OK;
  }
  Launch L;
  int Bc = B;
  int st = batch_chunk(&desc, 1, B, &Bc, &L);
  if (st) return st;
  if ((st = choose_launch(&desc, 1, Bc, o, &L))) return st;
  std::memset(plan, 0, sizeof(*plan));
  plan->grid = L.grid;
  plan->warps_per_cta = L.W;
  plan->active_warps = L.active;
  plan->num_tiles = L.total_tiles;
  plan->smem_bytes = (int32_t)L.smem;
  plan->x_in_smem = 1;
  plan->stages = bufs_for(Bc);
  plan->ctas_per_sm = L.half ? pipe_ctas_for(Bc) : 1;
  plan->ring_bytes = 0;
  plan->batch_per_launch = Bc;
  plan->launches = (B + Bc - 1) / Bc;
  plan->coresident = L.half;
  return GQSA_OK;
}

extern "C" int gqsa_gemm_grouped(const gqsa_gemm_item_t* items, int32_t n, int32_t B, const gqsa_options_t* opts,
                                 void* d_ws, size_t ws_bytes, void* stream) {
  const gqsa_options_t o = opts ? *opts : gqsa_options_t{GQSA_PARTITION_STREAM_K, 0, 0, 0};
  int st = check_options(o);
  if (st) return st;
  if (!items) return GQSA_ERR_BUFFER;
  if (n < 1 || n > kMaxItems) return GQSA_ERR_SHAPE;
  for (int j = 0; j < n; ++j) {
    if ((st = check_item(items[j], B, o.out_f16))) return st;
    if (items[j].desc->bits != items[0].desc->bits || items[j].desc->group_size != items[0].desc->group_size ||
        is_tc(items[j].desc))  // LAYOUT-TC blobs run through gqsa_gemm_ex / gqsa_gemm_smallbatch
      return GQSA_ERR_UNSUPPORTED;
  }
  return run_grouped(items, n, B, o, d_ws, ws_bytes, stream);
}

extern "C" int gqsa_gemm_ex(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B,
                            int64_t ldx, void* d_Y, int64_t ldy, const float* d_bias, void* d_ws,
                            size_t ws_bytes, const gqsa_options_t* opts, void* stream) {
  const gqsa_options_t o = opts ? *opts : gqsa_options_t{GQSA_PARTITION_STREAM_K, 0, 0, 0};
  int st = check_options(o);
  if (st) return st;
  const gqsa_gemm_item_t it{desc, d_blob, d_X, ldx, d_Y, ldy, d_bias};
  if ((st = check_item(it, B, o.out_f16))) return st;
  if (is_tc(desc)) return run_tc(desc, d_blob, d_X, B, ldx, d_Y, ldy, d_bias, o, d_ws, ws_bytes, stream);
  return run_grouped(&it, 1, B, o, d_ws, ws_bytes, stream);
}

extern "C" int gqsa_gemm_allgather(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B,
                                   int64_t ldx, void* const* d_peer_Y, int32_t n_peers, int64_t ldy,
                                   int32_t row_offset, int32_t out_f16, const float* d_bias, void* d_ws,
                                   size_t ws_bytes, void* stream) {
  if (!desc || !d_blob || !d_X || !d_peer_Y || !d_ws) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (is_tc(desc)) return GQSA_ERR_UNSUPPORTED;  // the fused epilogue is the CUDA-core kernel's
  if (n_peers < 1 || n_peers > kMaxPeers || B < 1 || B > kMaxBatch || (out_f16 != 0 && out_f16 != 1))
    return GQSA_ERR_SHAPE;
  if (row_offset < 0 || ldy < (int64_t)row_offset + desc->rows || ldx < desc->cols || ldx % 8) return GQSA_ERR_SHAPE;
  for (int k = 0; k < n_peers; ++k)
    if (!d_peer_Y[k] || !aligned(d_peer_Y[k], out_f16 ? 2 : 4)) return GQSA_ERR_BUFFER;
  if (!aligned(d_blob, 256) || !aligned(d_X, 16) || (d_bias && !aligned(d_bias, 4))) return GQSA_ERR_BUFFER;
  const gqsa_options_t o{GQSA_PARTITION_STREAM_K, out_f16, 0, 0};
  Peers peers;
  peers.n = n_peers;
  peers.row_offset = row_offset;
  for (int k = 0; k < n_peers; ++k) peers.y[k] = d_peer_Y[k];
  const gqsa_gemm_item_t it{desc, d_blob, d_X, ldx, d_peer_Y[0], ldy, d_bias};
  return run_grouped(&it, 1, B, o, d_ws, ws_bytes, stream, &peers);
}

extern "C" int gqsa_gemm_allgather_multicast(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X,
                                             int32_t B, int64_t ldx, void* d_mc_Y, int64_t ldy, int32_t row_offset,
                                             int32_t out_f16, const float* d_bias, void* d_ws, size_t ws_bytes,
                                             void* stream) {
  if (!desc || !d_blob || !d_X || !d_mc_Y || !d_ws) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (is_tc(desc)) return GQSA_ERR_UNSUPPORTED;
  if (B < 1 || B > kMaxBatch || (out_f16 != 0 && out_f16 != 1)) return GQSA_ERR_SHAPE;
  if (out_f16) return GQSA_ERR_UNSUPPORTED;  // multimem.st has no 16-bit scalar form
  if (row_offset < 0 || ldy < (int64_t)row_offset + desc->rows || ldx < desc->cols || ldx % 8) return GQSA_ERR_SHAPE;
  if (!aligned(d_mc_Y, 4) || !aligned(d_blob, 256) || !aligned(d_X, 16) ||
      (d_bias && !aligned(d_bias, 4)))
    return GQSA_ERR_BUFFER;
  const gqsa_options_t o{GQSA_PARTITION_STREAM_K, out_f16, 0, 0};
  Peers peers;
  peers.n = 1;
  peers.mc = 1;
  peers.row_offset = row_offset;
  peers.y[0] = d_mc_Y;
  const gqsa_gemm_item_t it{desc, d_blob, d_X, ldx, d_mc_Y, ldy, d_bias};
  return run_grouped(&it, 1, B, o, d_ws, ws_bytes, stream, &peers);
}

extern "C" int gqsa_gemm_smallbatch(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X,
                                    int32_t B, int64_t ldx, float* d_Y, int64_t ldy,
                                    const float* d_bias, void* d_ws, size_t ws_bytes, void* stream) {
  return gqsa_gemm_ex(desc, d_blob, d_X, B, ldx, d_Y, ldy, d_bias, d_ws, ws_bytes, nullptr, stream);
}

extern "C" int gqsa_gemv(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_x, float* d_y,
                         const float* d_bias, void* d_ws, size_t ws_bytes, void* stream) {
  if (!desc) return GQSA_ERR_BUFFER;
  return gqsa_gemm_smallbatch(desc, d_blob, d_x, 1, desc->cols, d_y, desc->rows, d_bias, d_ws,
                              ws_bytes, stream);
}

extern "C" int gqsa_hostio_stage_size(const gqsa_desc_t* desc, int32_t B, size_t* bytes) {
  if (!desc || !bytes) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (B < 1 || B > kMaxBatch) return GQSA_ERR_SHAPE;
  const size_t xb = ((size_t)B * desc->cols * 2 + 255) / 256 * 256;
  *bytes = xb + (size_t)B * desc->rows * 4;
  return GQSA_OK;
}

extern "C" int gqsa_gemm_hostio(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* h_X,
                                int32_t B, float* h_Y, const float* d_bias, void* d_stage,
                                size_t stage_bytes, void* d_ws, size_t ws_bytes, void* stream) {
  if (!desc || !h_X || !h_Y || !d_stage) return GQSA_ERR_BUFFER;
  size_t need = 0;
  int st = gqsa_hostio_stage_size(desc, B, &need);
  if (st) return st;
  if (stage_bytes < need || !aligned(d_stage, 256)) return GQSA_ERR_BUFFER;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* stage = static_cast<uint8_t*>(d_stage);
  const size_t xb = ((size_t)B * desc->cols * 2 + 255) / 256 * 256;
  uint16_t* dX = reinterpret_cast<uint16_t*>(stage);
  float* dY = reinterpret_cast<float*>(stage + xb);
  if (cudaMemcpyAsync(dX, h_X, (size_t)B * desc->cols * 2, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return GQSA_ERR_CUDA;
  st = gqsa_gemm_smallbatch(desc, d_blob, dX, B, desc->cols, dY, desc->rows, d_bias, d_ws, ws_bytes,
                            stream);
  if (st) return st;
  if (cudaMemcpyAsync(h_Y, dY, (size_t)B * desc->rows * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return GQSA_ERR_CUDA;
  return GQSA_OK;
}

// Stage layout: [x_0 .. x_{n-1}: B*cols_j fp16 each][y_0 .. y_{n-1}: B*rows_j fp32]
namespace {
int multi_layout(const gqsa_desc_t* const* descs, int n, int B, size_t* x_off, size_t* y_off,
                 size_t* x_bytes_total, size_t* y_bytes_total) {
  if (!descs) return GQSA_ERR_BUFFER;
  if (n < 1 || B < 1 || B > kMaxBatch) return GQSA_ERR_SHAPE;
  size_t xo = 0;
  for (int j = 0; j < n; ++j) {
    if (!descs[j]) return GQSA_ERR_BUFFER;
    if (!desc_ok(descs[j])) return GQSA_ERR_VALIDATION;
    if (x_off) x_off[j] = xo;
    // cols % 8 == 0 (G >= 8): every segment starts 16-B aligned, as the kernel's X needs
    xo += (size_t)B * descs[j]->cols * 2;
  }
  const size_t y0 = (xo + 255) / 256 * 256;
  size_t yo = y0;
  for (int j = 0; j < n; ++j) {
    if (y_off) y_off[j] = yo;
    yo += (size_t)B * descs[j]->rows * 4;
  }
  if (x_bytes_total) *x_bytes_total = xo;
  if (y_bytes_total) *y_bytes_total = yo - y0;
  return GQSA_OK;
}
}  // namespace

extern "C" int gqsa_multi_hostio_stage_size(const gqsa_desc_t* const* descs, int32_t n, int32_t B, size_t* bytes) {
  if (!bytes) return GQSA_ERR_BUFFER;
  size_t xt = 0, yt = 0;
  const int st = multi_layout(descs, n, B, nullptr, nullptr, &xt, &yt);
  if (st) return st;
  *bytes = (xt + 255) / 256 * 256 + yt;
  return GQSA_OK;
}

extern "C" int gqsa_gemm_multi_hostio(const gqsa_desc_t* const* descs, const void* const* d_blobs, int32_t n,
                                      int32_t B, const uint16_t* h_X, float* h_Y, void* d_stage,
                                      size_t stage_bytes, void* const* d_ws, const size_t* ws_bytes,
                                      void* stream) {
  if (!d_blobs || !h_X || !h_Y || !d_stage || !d_ws || !ws_bytes) return GQSA_ERR_BUFFER;
  if (n > 4096) return GQSA_ERR_SHAPE;
  std::vector<size_t> xo((size_t)(n > 0 ? n : 1)), yo((size_t)(n > 0 ? n : 1));
  size_t xt = 0, yt = 0;
  int st = multi_layout(descs, n, B, xo.data(), yo.data(), &xt, &yt);
  if (st) return st;
  if (stage_bytes < (xt + 255) / 256 * 256 + yt || !aligned(d_stage, 256)) return GQSA_ERR_BUFFER;
  for (int j = 1; j < n; ++j)
    if (descs[j]->bits != descs[0]->bits || descs[j]->group_size != descs[0]->group_size)
      return GQSA_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* stage = static_cast<uint8_t*>(d_stage);
  if (cudaMemcpyAsync(stage, h_X, xt, cudaMemcpyHostToDevice, s) != cudaSuccess) return GQSA_ERR_CUDA;
  std::vector<gqsa_gemm_item_t> items((size_t)n);
  for (int j = 0; j < n; ++j) {
    const gqsa_desc_t* d = descs[j];
    items[j] = gqsa_gemm_item_t{d, d_blobs[j], reinterpret_cast<const uint16_t*>(stage + xo[j]), d->cols,
                                reinterpret_cast<float*>(stage + yo[j]), d->rows, nullptr};
    if ((st = check_item(items[j], B, 0))) return st;
  }
  const gqsa_options_t o{GQSA_PARTITION_STREAM_K, 0, 0, 0};
  for (int j0 = 0; j0 < n; j0 += kMaxItems) {
    const int nj = std::min(kMaxItems, n - j0);
    if ((st = run_grouped(items.data() + j0, nj, B, o, d_ws[0], ws_bytes[0], stream))) return st;
  }
  if (cudaMemcpyAsync(h_Y, stage + yo[0], yt, cudaMemcpyDeviceToHost, s) != cudaSuccess) return GQSA_ERR_CUDA;
  return GQSA_OK;
}

extern "C" uint64_t gqsa_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int gqsa_debug_trace(void* d_buf, size_t bytes) {
  g_trace = static_cast<uint64_t*>(d_buf);
  g_trace_bytes = d_buf ? bytes : 0;
  return GQSA_OK;
}
