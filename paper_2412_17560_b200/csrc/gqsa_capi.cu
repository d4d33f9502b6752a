// gqsa_capi.cu -- extern "C" entry points that validate arguments, plan the
// Stream-K grid and launch the sm_100a kernels (see include/gqsa.h).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/gqsa.h"
#include "gqsa_kernels.h"
#include "gqsa_layout.h"

using namespace gqsa;

namespace {

std::atomic<uint64_t> g_launches{0};
uint64_t* g_trace = nullptr;  // gqsa_debug_trace buffer (device), or null
size_t g_trace_bytes = 0;

struct DevInfo {
  int sms = 0;
  bool attr_set[27][2 * (kMaxBatch + 1)] = {};  // [bits + 9 * (G = 8: 1, 32: 2)][batch (+ FEW)]
  bool chain_attr_set[9][3] = {};
};
std::mutex g_mu;
DevInfo g_dev[64];

int device_sms(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return 0;
  if (!g_dev[dev].sms) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    g_dev[dev].sms = v;
  }
  return g_dev[dev].sms;
}

bool lanes_per_row_ok(uint32_t s) { return s >= 1 && s <= 32 && (s & (s - 1)) == 0; }

bool desc_ok(const gqsa_desc_t* d) {
  return d && d->magic == kMagic && d->version == (uint32_t)kVersion && group_supported(d->bits, d->group_size) &&
         d->tile_groups == kTileGroups && d->rows >= 0 && d->cols > 0 && d->cols % d->group_size == 0 &&
         d->num_tiles >= 0 &&
         lanes_per_row_ok(((uint32_t)d->flags >> kFlagLanesPerRowShift) & 0xff);
}

// Tuning knobs (environment, read once): resident CTAs per SM and ring depth.
int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : dflt;
  return v >= lo && v <= hi ? v : dflt;
}
int ctas_per_sm_cap() {
  static int cap = env_int("GQSA_CTAS_PER_SM", kMaxCtasPerSm, 1, 8);
  return cap;
}
int stages_cap() {
  static int cap = env_int("GQSA_STAGES", kMaxStages, kMinStages, kMaxStages);
  return cap;
}

// The FEW kernel variant (12 warps, <= 85 registers) for layers with few
// tiles per warp; GQSA_FEW=0 disables it (experiments).
bool few_for(const gqsa_desc_t* d, int B) {
  static int on = env_int("GQSA_FEW", 1, 0, 2);  // 2: every layer (experiments)
  // batch 2 always (twice the accumulators: 80 registers and NS = 4 beat 16
  // warps at 64 registers by 13-14 % on 14336x4096 / 4096x14336); batch 1
  // only for small layers
  if (d->group_size == 32) return B <= 2;  // four code planes per tile: needs the FEW register budget
  return on && d->group_size == kGroup && B <= 2 && (d->bits == 4 || d->bits == 2) &&
         (on == 2 || B == 2 || d->num_tiles < kFewTiles);
}
int warps_per_cta(const gqsa_desc_t* d, int B) {
  static int w1 = env_int("GQSA_WARPS", 16, 1, kMaxWarps);
  if (few_for(d, B)) return kFewWarps;
  return d->bits == 8 ? 8 : (B <= 2 ? w1 : 8);  // <= max_threads_for(bits, B) / 32
}

// Shared-memory plan per CTA of W warps: [x: B*K fp16][(P, Q) column sums]
// [TMA ring: W x NS tiles][ring mbarriers].  Preferred: one CTA per SM using
// at most half of the SM's shared memory, so the next GEMV on the stream (PDL)
// is resident at the same time and streams its first tiles during this one's
// tail.  If x does not leave room for that, the CTA takes the whole SM; if x
// does not fit at all, the batch is split into launches of `batch` columns.
struct SmemPlan {
  bool coresident;
  int stages, warps, batch, launches;
  size_t ring, total, fix;
};
// x and its column sums, rounded up to 128 B: the fix-up records and the
// TMA ring that follow must stay 16-B aligned (bulk-copy destinations; e.g.
// B = 3, K = 208 gives 1560 B unrounded).
size_t x_bytes(int B, int cols, int G = kGroup) {
  const size_t v = (size_t)B * cols * 2 + (size_t)B * pq_bytes_per_row(B, cols, G);
  return (v + 127) / 128 * 128;
}
size_t ring_bytes_for(const gqsa_desc_t* d, int W, int ns) {  // ring + its mbarriers
  return (size_t)W * ns * tile_bytes(d->bits, d->group_size) + (size_t)W * kMaxStages * 8;
}
// intra-CTA fix-up records (batch <= 2; larger batches use the global workspace)
size_t fix_bytes(int W, int B) { return B <= 2 ? (size_t)W * B * kLanes * kWsSlotBytes : 0; }
constexpr size_t kMaxDynSmem = kSmemPerSm - 2048;  // per-CTA limit we request (227 KB - reserve)

SmemPlan smem_plan(const gqsa_desc_t* d, int B) {
  SmemPlan sp{};
  // largest batch chunk whose x fits next to a minimal ring (default warps,
  // else 8 warps); cols <= kMaxCols makes Bc = 1 always fit
  int Bc = B, W = warps_per_cta(d, B);
  for (;; --Bc) {
    W = warps_per_cta(d, Bc);
    if (x_bytes(Bc, d->cols, d->group_size) + ring_bytes_for(d, W, kMinStages) <= kMaxDynSmem) break;
    if (W > 8 && x_bytes(Bc, d->cols, d->group_size) + ring_bytes_for(d, 8, kMinStages) <= kMaxDynSmem) {
      W = 8;
      break;
    }
    if (Bc == 1) break;
  }
  sp.launches = (B + Bc - 1) / Bc;
  const int Bb = (B + sp.launches - 1) / sp.launches;  // balanced chunks (<= Bc: fits)
  if (Bb != Bc) W = warps_per_cta(d, Bb) > W ? W : warps_per_cta(d, Bb);
  Bc = Bb;
  sp.batch = Bc;
  const size_t tb = (size_t)tile_bytes(d->bits, d->group_size);
  // intra-CTA fix-up records, if they fit next to x and a minimal ring
  size_t fb = fix_bytes(W, Bc);
  if (x_bytes(Bc, d->cols, d->group_size) + fb + ring_bytes_for(d, W, kMinStages) > kMaxDynSmem) fb = 0;
  const size_t xb = x_bytes(Bc, d->cols, d->group_size) + fb;  // x, column sums, fix-up records
  static const int cores = env_int("GQSA_CORESIDENT", kCoResidentKernels, 1, 4);  // experiments
  const size_t share = (size_t)kSmemPerSm / (ctas_per_sm_cap() * cores);
  const size_t budget = share > 2048 ? share - 2048 : 0;  // reserved + static smem
  int ns = kMinStages;
  sp.coresident = xb + ring_bytes_for(d, W, kMinStages) <= budget;
  if (sp.coresident) {
    ns = (int)((budget - xb - (size_t)W * kMaxStages * 8) / ((size_t)W * tb));
    if (ns > stages_cap()) ns = stages_cap();
    ns &= ~1;  // the ring holds tile pairs (one bulk copy + mbarrier per pair)
    if (ns < kMinStages) ns = kMinStages;
  }
  sp.warps = W;
  sp.stages = ns;
  sp.ring = (size_t)W * ns * tb;
  sp.total = xb + ring_bytes_for(d, W, ns);
  sp.fix = fb;
  return sp;
}

// Resident CTAs per SM for (kernel, block, dynamic smem), memoised: the
// occupancy query costs microseconds of host time per launch otherwise.
bool cached_occupancy(int dev, const void* fn, int threads, size_t smem, int* occ) {
  struct Key {
    int dev;
    const void* fn;
    int threads;
    size_t smem;
  };
  static std::vector<std::pair<Key, int>> cache;
  std::lock_guard<std::mutex> lk(g_mu);
  for (const auto& e : cache)
    if (e.first.dev == dev && e.first.fn == fn && e.first.threads == threads && e.first.smem == smem) {
      *occ = e.second;
      return true;
    }
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem) != cudaSuccess) return false;
  if (cache.size() < 4096) cache.push_back({Key{dev, fn, threads, smem}, v});
  *occ = v;
  return true;
}

// Fill the launch plan of the first (or only) batch chunk; returns a status.
int make_plan(const gqsa_desc_t* d, int B, gqsa_plan_t* pl, const void** kfn) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GQSA_ERR_CUDA;
  const int sms = device_sms(dev);
  if (sms <= 0) return GQSA_ERR_CUDA;
  const SmemPlan sp = smem_plan(d, B);
  const size_t smem = sp.total;
  const void* fn = select_kernel(d->bits, d->group_size, sp.batch, few_for(d, sp.batch));
  if (!fn) return GQSA_ERR_UNSUPPORTED;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    bool& set = g_dev[dev].attr_set[d->bits + (d->group_size == 8 ? 9 : d->group_size == 32 ? 18 : 0)]
                                   [sp.batch + (few_for(d, sp.batch) ? kMaxBatch + 1 : 0)];
    if (!set) {
      // maximum shared-memory carveout: two kernels' CTAs (this launch and
      // the next, PDL) must fit on one SM at the same time
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem) !=
              cudaSuccess ||
          cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared) != cudaSuccess)
        return GQSA_ERR_CUDA;
      set = true;
    }
  }
  const int W = sp.warps, threads = 32 * sp.warps;
  int occ = 0;
  if (!cached_occupancy(dev, fn, threads, smem, &occ)) return GQSA_ERR_CUDA;
  if (occ < 1) return GQSA_ERR_UNSUPPORTED;
  // the next launch on the stream (same configuration) can be resident
  // during this one's tail only if two CTAs fit (shared memory AND registers)
  const bool coresident = occ >= ctas_per_sm_cap() + 1;
  if (occ > ctas_per_sm_cap()) occ = ctas_per_sm_cap();
  int warps = sms * occ * W;
  if (warps > kMaxWarpsBound) warps = kMaxWarpsBound;
  const int active = d->num_tiles < warps ? d->num_tiles : warps;
  int grid = (active + W - 1) / W;
  if (grid == 0) {  // nnzg == 0: only empty rows to write
    grid = (d->n_empty + threads - 1) / threads;
    if (grid > sms) grid = sms;
    if (grid < 1) grid = 1;
  }
  pl->grid = grid;
  pl->warps_per_cta = W;
  pl->active_warps = active;
  pl->num_tiles = d->num_tiles;
  pl->smem_bytes = (int32_t)smem;
  pl->x_in_smem = 1;
  pl->stages = sp.stages;
  pl->ctas_per_sm = occ;
  pl->ring_bytes = (int32_t)sp.ring;
  pl->batch_per_launch = sp.batch;
  pl->launches = sp.launches;
  pl->coresident = coresident ? 1 : 0;
  if (kfn) *kfn = fn;
  return GQSA_OK;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace

namespace {
// One launch over Bc batch columns (x of Bc columns fits in shared memory).
// Fused all-gather destinations of one launch (n == 0: plain Y).
struct Peers {
  int n = 0;
  int32_t row_offset = 0;
  void* y[kMaxPeers] = {};
};

// `plan0`/`fn0`: the caller's plan when it was made for exactly Bc columns.
int launch_chunk(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int Bc, int64_t ldx,
                 void* d_Y, int64_t ldy, const float* d_bias, void* d_ws, const gqsa_options_t& o,
                 void* stream, const gqsa_plan_t* plan0 = nullptr, const void* fn0 = nullptr,
                 const Peers* peers = nullptr) {
  gqsa_plan_t pl;
  const void* fn = nullptr;
  if (plan0 && fn0 && plan0->launches == 1 && plan0->batch_per_launch == Bc) {
    pl = *plan0;
    fn = fn0;
  } else {
    int st = make_plan(desc, Bc, &pl, &fn);
    if (st) return st;
  }
  if (pl.batch_per_launch != Bc) return GQSA_ERR_UNSUPPORTED;  // unreachable: chunks always fit
  const uint8_t* blob = static_cast<const uint8_t*>(d_blob);
  KParams p{};
  p.tiles = blob + desc->off_tiles;
  p.perm = reinterpret_cast<const int32_t*>(blob + desc->off_nzrow);
  p.empty = reinterpret_cast<const int32_t*>(blob + desc->off_empty);
  p.X = d_X;
  p.Y = d_Y;
  p.bias = d_bias;
  p.ws = static_cast<uint32_t*>(d_ws);
  p.ldx = ldx;
  p.ldy = ldy;
  p.rows = desc->rows;
  p.cols = desc->cols;
  p.num_tiles = desc->num_tiles;
  p.n_empty = desc->n_empty;
  p.active_warps = pl.active_warps;
  p.lanes_per_row = ((uint32_t)desc->flags >> kFlagLanesPerRowShift) & 0xff;
  p.part_q = pl.active_warps ? desc->num_tiles / pl.active_warps : 0;
  p.part_r = pl.active_warps ? desc->num_tiles % pl.active_warps : 0;
  p.stages = pl.stages;
  p.ring_offset = pl.smem_bytes - pl.ring_bytes - pl.warps_per_cta * kMaxStages * 8;
  {
    static const int fix_local = env_int("GQSA_FIX_LOCAL", 1, 0, 1);
    const size_t fb = smem_plan(desc, Bc).fix;
    p.fix_offset = (fb && fix_local) ? p.ring_offset - (int32_t)fb : 0;  // records sit before the ring
  }
  p.trace = (g_trace && g_trace_bytes >= (size_t)pl.active_warps * 64) ? g_trace : nullptr;
  p.slice_k = o.partition == GQSA_PARTITION_SLICE_K ? 1 : 0;
  p.out_f16 = o.out_f16;
  if (peers && peers->n) {
    p.n_peers = peers->n;
    p.row_offset = peers->row_offset;
    for (int k = 0; k < peers->n; ++k)  // chunk b0 is folded into d_Y's offset from peer 0
      p.peer_y[k] = reinterpret_cast<uint64_t>(peers->y[k]) +
                    (reinterpret_cast<uintptr_t>(d_Y) - reinterpret_cast<uintptr_t>(peers->y[0]));
  }
  if (desc->rows == 0) return GQSA_OK;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(32 * pl.warps_per_cta);
  cfg.dynamicSmemBytes = pl.smem_bytes;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&p};
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) return GQSA_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return GQSA_OK;
}
}  // namespace

extern "C" int gqsa_workspace_size(const gqsa_desc_t* desc, int32_t batch, size_t* bytes) {
  if (!desc || !bytes) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (batch < 1 || batch > kMaxBatch) return GQSA_ERR_SHAPE;
  const int64_t recs = desc->num_tiles < kMaxWarpsBound ? desc->num_tiles : kMaxWarpsBound;
  *bytes = (size_t)(recs > 0 ? recs : 1) * batch * kLanes * kWsSlotBytes;
  return GQSA_OK;
}

extern "C" int gqsa_launch_plan(const gqsa_desc_t* desc, int32_t B, gqsa_plan_t* plan) {
  if (!desc || !plan) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (B < 1 || B > kMaxBatch) return GQSA_ERR_SHAPE;
  return make_plan(desc, B, plan, nullptr);
}

extern "C" int gqsa_gemm_ex(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B,
                            int64_t ldx, void* d_Y, int64_t ldy, const float* d_bias, void* d_ws,
                            size_t ws_bytes, const gqsa_options_t* opts, void* stream) {
  const gqsa_options_t o = opts ? *opts : gqsa_options_t{GQSA_PARTITION_STREAM_K, 0};
  if (o.partition != GQSA_PARTITION_STREAM_K && o.partition != GQSA_PARTITION_SLICE_K) return GQSA_ERR_SHAPE;
  if (o.out_f16 != 0 && o.out_f16 != 1) return GQSA_ERR_SHAPE;
  if (!desc || !d_blob || !d_X || !d_Y || !d_ws) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (B < 1 || B > kMaxBatch) return GQSA_ERR_SHAPE;
  if (ldx < desc->cols || ldx % 8 || ldy < desc->rows) return GQSA_ERR_SHAPE;
  if (!aligned(d_blob, 256) || !aligned(d_X, 16) || !aligned(d_ws, 16) ||
      (d_bias && !aligned(d_bias, 4)) || !aligned(d_Y, o.out_f16 ? 2 : 4))
    return GQSA_ERR_BUFFER;
  size_t need = 0;
  gqsa_workspace_size(desc, B, &need);
  if (ws_bytes < need) return GQSA_ERR_BUFFER;

  gqsa_plan_t pl0;
  const void* fn0 = nullptr;
  int st = make_plan(desc, B, &pl0, &fn0);
  if (st) return st;
  for (int b0 = 0; b0 < B; b0 += pl0.batch_per_launch) {  // batch chunks whose x fits in smem
    const int Bc = B - b0 < pl0.batch_per_launch ? B - b0 : pl0.batch_per_launch;
    void* y0 = static_cast<uint8_t*>(d_Y) + (size_t)b0 * ldy * (o.out_f16 ? 2 : 4);
    st = launch_chunk(desc, d_blob, d_X + (int64_t)b0 * ldx, Bc, ldx, y0, ldy, d_bias, d_ws, o, stream, &pl0,
                      fn0);
    if (st) return st;
  }
  return GQSA_OK;
}

extern "C" int gqsa_gemm_allgather(const gqsa_desc_t* desc, const void* d_blob, const uint16_t* d_X, int32_t B,
                                   int64_t ldx, void* const* d_peer_Y, int32_t n_peers, int64_t ldy,
                                   int32_t row_offset, int32_t out_f16, const float* d_bias, void* d_ws,
                                   size_t ws_bytes, void* stream) {
  if (!desc || !d_blob || !d_X || !d_peer_Y || !d_ws) return GQSA_ERR_BUFFER;
  if (!desc_ok(desc)) return GQSA_ERR_VALIDATION;
  if (n_peers < 1 || n_peers > kMaxPeers || B < 1 || B > kMaxBatch || (out_f16 != 0 && out_f16 != 1))
    return GQSA_ERR_SHAPE;
  if (row_offset < 0 || ldy < (int64_t)row_offset + desc->rows || ldx < desc->cols || ldx % 8) return GQSA_ERR_SHAPE;
  for (int k = 0; k < n_peers; ++k)
    if (!d_peer_Y[k] || !aligned(d_peer_Y[k], out_f16 ? 2 : 4)) return GQSA_ERR_BUFFER;
  if (!aligned(d_blob, 256) || !aligned(d_X, 16) || !aligned(d_ws, 16) || (d_bias && !aligned(d_bias, 4)))
    return GQSA_ERR_BUFFER;
  size_t need = 0;
  gqsa_workspace_size(desc, B, &need);
  if (ws_bytes < need) return GQSA_ERR_BUFFER;
  const gqsa_options_t o{GQSA_PARTITION_STREAM_K, out_f16};
  gqsa_plan_t pl0;
  const void* fn0 = nullptr;
  int st = make_plan(desc, B, &pl0, &fn0);
  if (st) return st;
  Peers peers;
  peers.n = n_peers;
  peers.row_offset = row_offset;
  for (int k = 0; k < n_peers; ++k) peers.y[k] = d_peer_Y[k];
  const size_t es = out_f16 ? 2 : 4;
  for (int b0 = 0; b0 < B; b0 += pl0.batch_per_launch) {
    const int Bc = B - b0 < pl0.batch_per_launch ? B - b0 : pl0.batch_per_launch;
    void* y0 = static_cast<uint8_t*>(d_peer_Y[0]) + (size_t)b0 * ldy * es;
    st = launch_chunk(desc, d_blob, d_X + (int64_t)b0 * ldx, Bc, ldx, y0, ldy, d_bias, d_ws, o, stream, &pl0, fn0,
                      &peers);
    if (st) return st;
  }
  return GQSA_OK;
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

// ---------------------------------------------------------------- chain
namespace {
struct ChainPlan {
  int grid, warps, stages, total_warps;
  size_t smem, ring_offset, fix_offset, rec_bytes;  // rec_bytes: global fix-up records per item
};

int chain_check(const gqsa_chain_item_t* items, int n, int B) {
  if (!items) return GQSA_ERR_BUFFER;
  if (n < 1 || n > kMaxChain || B < 1 || B > 2) return GQSA_ERR_SHAPE;
  for (int j = 0; j < n; ++j) {
    const gqsa_desc_t* d = items[j].desc;
    if (!d) return GQSA_ERR_BUFFER;
    if (!desc_ok(d)) return GQSA_ERR_VALIDATION;
    if (d->bits != items[0].desc->bits || d->group_size != kGroup) return GQSA_ERR_UNSUPPORTED;
  }
  if (items[0].desc->bits == 8) return GQSA_ERR_UNSUPPORTED;
  return GQSA_OK;
}

int chain_plan(const gqsa_chain_item_t* items, int n, int B, ChainPlan* cpl) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GQSA_ERR_CUDA;
  const int sms = device_sms(dev);
  if (sms <= 0) return GQSA_ERR_CUDA;
  static const int W = env_int("GQSA_CHAIN_WARPS", 16, 4, kChainThreads / 32);
  // half = leave half the SM to the next launch (PDL overlap across launches)
  static const int half = env_int("GQSA_CHAIN_HALF", 0, 0, 1);
  const int bits = items[0].desc->bits;
  size_t xb = 0;
  for (int j = 0; j < n; ++j) {
    const size_t v = x_bytes(B, items[j].desc->cols);
    if (v > xb) xb = v;
  }
  xb = (xb + 127) / 128 * 128;
  const size_t fb = fix_bytes(W, B);
  const size_t budget = half ? (size_t)kSmemPerSm / 2 - 2048 : kMaxDynSmem;
  const size_t bars = (size_t)W * kMaxStages * 8;
  const size_t tb = (size_t)tile_bytes(bits);
  if (xb + fb + bars + (size_t)W * kMinStages * tb > budget) return GQSA_ERR_UNSUPPORTED;
  int ns = (int)((budget - xb - fb - bars) / ((size_t)W * tb));
  if (ns > stages_cap()) ns = stages_cap();
  ns &= ~1;
  cpl->grid = sms;
  cpl->warps = W;
  cpl->stages = ns;
  cpl->total_warps = sms * W;
  cpl->fix_offset = xb;
  cpl->ring_offset = xb + fb;
  cpl->smem = xb + fb + (size_t)W * ns * tb + bars;
  cpl->rec_bytes = ((size_t)cpl->total_warps * B * kLanes * kWsSlotBytes + 255) / 256 * 256;
  return GQSA_OK;
}
}  // namespace

extern "C" int gqsa_chain_workspace_size(const gqsa_chain_item_t* items, int32_t n, int32_t B,
                                         size_t* bytes) {
  if (!bytes) return GQSA_ERR_BUFFER;
  int st = chain_check(items, n, B);
  if (st) return st;
  ChainPlan cpl;
  st = chain_plan(items, n, B, &cpl);
  if (st) return st;
  *bytes = 256 + (size_t)n * cpl.rec_bytes;
  return GQSA_OK;
}

extern "C" int gqsa_gemm_chain(const gqsa_chain_item_t* items, int32_t n, int32_t B, void* d_ws,
                               size_t ws_bytes, void* stream) {
  int st = chain_check(items, n, B);
  if (st) return st;
  if (!d_ws || !aligned(d_ws, 256)) return GQSA_ERR_BUFFER;
  for (int j = 0; j < n; ++j) {
    const gqsa_chain_item_t& it = items[j];
    if (!it.d_blob || !it.d_X || !it.d_Y) return GQSA_ERR_BUFFER;
    if (it.ldx < it.desc->cols || it.ldx % 8 || it.ldy < it.desc->rows) return GQSA_ERR_SHAPE;
    if (it.wait_prev != 0 && it.wait_prev != 1) return GQSA_ERR_SHAPE;
    if (it.out_f16 != 0 && it.out_f16 != 1) return GQSA_ERR_SHAPE;
    if (!aligned(it.d_blob, 256) || !aligned(it.d_X, 16) || !aligned(it.d_Y, it.out_f16 ? 2 : 4) ||
        (it.d_bias && !aligned(it.d_bias, 4)))
      return GQSA_ERR_BUFFER;
  }
  ChainPlan cpl;
  st = chain_plan(items, n, B, &cpl);
  if (st) return st;
  if (ws_bytes < 256 + (size_t)n * cpl.rec_bytes) return GQSA_ERR_BUFFER;
  const void* fn = select_chain_kernel(items[0].desc->bits, B);
  if (!fn) return GQSA_ERR_UNSUPPORTED;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return GQSA_ERR_CUDA;
    std::lock_guard<std::mutex> lk(g_mu);
    bool& s = g_dev[dev].chain_attr_set[items[0].desc->bits][B];
    if (!s) {
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem) != cudaSuccess ||
          cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared) != cudaSuccess)
        return GQSA_ERR_CUDA;
      s = true;
    }
  }
  ChainParams cp;
  std::memset(&cp, 0, sizeof(cp));
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  cp.counter = reinterpret_cast<uint32_t*>(ws);
  for (int j = 0; j < n; ++j) {
    const gqsa_chain_item_t& it = items[j];
    const gqsa_desc_t* desc = it.desc;
    const uint8_t* blob = static_cast<const uint8_t*>(it.d_blob);
    KParams& p = cp.item[j];
    p.tiles = blob + desc->off_tiles;
    p.perm = reinterpret_cast<const int32_t*>(blob + desc->off_nzrow);
    p.empty = reinterpret_cast<const int32_t*>(blob + desc->off_empty);
    p.X = it.d_X;
    p.Y = it.d_Y;
    p.bias = it.d_bias;
    p.ws = reinterpret_cast<uint32_t*>(ws + 256 + (size_t)j * cpl.rec_bytes);
    p.ldx = it.ldx;
    p.ldy = it.ldy;
    p.rows = desc->rows;
    p.cols = desc->cols;
    p.num_tiles = desc->num_tiles;
    p.n_empty = desc->n_empty;
    p.active_warps = desc->num_tiles < cpl.total_warps ? desc->num_tiles : cpl.total_warps;
    p.lanes_per_row = ((uint32_t)desc->flags >> kFlagLanesPerRowShift) & 0xff;
    p.part_q = p.active_warps ? desc->num_tiles / p.active_warps : 0;
    p.part_r = p.active_warps ? desc->num_tiles % p.active_warps : 0;
    p.out_f16 = it.out_f16;
    cp.wait_prev[j] = j == 0 ? 0 : it.wait_prev;
    cp.reuse_x[j] = (j > 0 && !cp.wait_prev[j] && it.d_X == items[j - 1].d_X && it.ldx == items[j - 1].ldx &&
                     it.desc->cols == items[j - 1].desc->cols)
                        ? 1
                        : 0;
  }
  cp.n = n;
  cp.stages = cpl.stages;
  cp.ring_offset = (int32_t)cpl.ring_offset;
  cp.fix_offset = (int32_t)cpl.fix_offset;
  cp.total_warps = cpl.total_warps;
  cp.trace = (g_trace && g_trace_bytes >= (size_t)cpl.total_warps * n * 32) ? g_trace : nullptr;

  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * cpl.warps, cpl.smem) != cudaSuccess)
    return GQSA_ERR_CUDA;
  if (occ < 1) return GQSA_ERR_UNSUPPORTED;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cpl.grid);
  cfg.blockDim = dim3(32 * cpl.warps);
  cfg.dynamicSmemBytes = cpl.smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  static const int coop = env_int("GQSA_CHAIN_COOP", 1, 0, 1);
  cfg.numAttrs = coop ? 2 : 1;
  void* args[] = {&cp};
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) return GQSA_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return GQSA_OK;
}

// Stage layout: [x_0 .. x_{n-1}: B*cols_j fp16 each, 16-B aligned][y_0 .. y_{n-1}: B*rows_j fp32]
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
    xo += (size_t)B * descs[j]->cols * 2;  // cols % 16 == 0: segments stay 32-B aligned
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
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* stage = static_cast<uint8_t*>(d_stage);
  if (cudaMemcpyAsync(stage, h_X, xt, cudaMemcpyHostToDevice, s) != cudaSuccess) return GQSA_ERR_CUDA;
  for (int j = 0; j < n; ++j) {
    const gqsa_desc_t* d = descs[j];
    st = gqsa_gemm_smallbatch(d, d_blobs[j], reinterpret_cast<const uint16_t*>(stage + xo[j]), B, d->cols,
                              reinterpret_cast<float*>(stage + yo[j]), d->rows, nullptr, d_ws[j], ws_bytes[j],
                              stream);
    if (st) return st;
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
