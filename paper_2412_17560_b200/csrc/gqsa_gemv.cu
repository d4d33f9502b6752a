// gqsa_gemv.cu -- sm_100a Stream-K group-sparse W2/W4/W8 GEMV / small-batch GEMM.
//
// Computes, for every batch column b < B and output row r (PAPER.md:64-69
// [Eq. 3], 95-101 [§3.2 BSR], 134 [§3.5]):
//
//   y[b][r] = sum_{g in row r} s_g * ( sum_t q_{g,t} x[b][c_g*G+t] - z_g * X_{b,c_g} ),
//   X_{b,c} = sum_t x[b][c*G+t]       (Eq. 3 applied per group, z folded once)
//
// Design:
//  * Layout: rows are sorted by kept-group count and cut into
//    32-row slices (sliced ELL); a lane owns a row and walks its groups slot
//    by slot, so the hot loop has no cross-lane reduction at all.
//  * Task-centric partition (PAPER.md:161 Stream-K, App. J): the
//    tile stream (128 groups per tile) is cut into contiguous, equal (+-1
//    tile) ranges, one per WARP, regardless of row or slice boundaries.
//  * Weights stream HBM -> shared memory through a per-warp ring of 1-D TMA
//    bulk copies (tile pairs, one mbarrier per pair, evict-first L2 policy);
//    the first pairs are requested BEFORE griddepcontrol.wait so they overlap
//    the previous kernel (PDL; this CTA uses at most half an SM so the next
//    launch is resident during its tail).
//  * Activations are staged in shared memory once per CTA, together with the
//    per-column-group sums (P, Q) the offset-folded dequantization needs.
//  * Dequantization: LOP3 magic (0x6400 = fp16 1024) turns code fields into
//    exact fp16 (1024 + 2^k q); FHFMA (fma.rn.f32.f16) multiplies them by fp16
//    x with exact products and fp32 accumulation; the offsets are removed once
//    per group with (P, Q).  No tensor cores: the rows of a warp hold groups
//    at unrelated columns, and batch 1 is bandwidth-bound
//    (PAPER.md:9, 134).
//  * Fix-up: a slice split across warps is finished by the warp that owns its
//    first tile, which adds the per-lane partials its successors publish
//    (64-bit {value, flag} slots, no fences), in warp order: deterministic.
#include "gqsa_device.cuh"

namespace gqsa {

template <int BITS, int B, bool FEW, int G = kGroup>
__global__ void __launch_bounds__(max_threads_for(BITS, B, FEW), min_blocks_for(BITS, B, FEW))
    gqsa_streamk_kernel(KParams p) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nthreads = blockDim.x;
  const int gw = blockIdx.x * (nthreads >> 5) + warp;

  // ---- task-centric partition: contiguous tile range per warp (+-1 tile)
  int t_begin = 0, t_end = 0;
  if (gw < p.active_warps) {  // q = num_tiles / warps, r = num_tiles % warps (host)
    t_begin = gw * p.part_q + min(gw, p.part_r);
    t_end = t_begin + p.part_q + (gw < p.part_r ? 1 : 0);
  }
  const uint8_t* tiles = p.tiles;
  const int tb = tile_bytes(BITS, G);
  const int NS = p.stages;
  if (p.slice_k && t_end > t_begin) {
    // data-centric partition (Slice-K): the warp owns the slices whose FIRST
    // tile lies in its Stream-K range, each in full (tile header word 1 =
    // tiles from this tile to its slice's last tile)
    const uint2 hb = __ldg(reinterpret_cast<const uint2*>(tiles + (int64_t)t_begin * tb));
    const uint2 he = __ldg(reinterpret_cast<const uint2*>(tiles + (int64_t)(t_end - 1) * tb));
    const int b = (hb.x & kTileFirst) ? t_begin : t_begin + (int)hb.y + 1;
    const int e = t_end + (int)he.y;
    t_begin = b;
    t_end = b < t_end ? e : b;
  }

  // ---- weights never depend on the previous kernel: each warp's first NS
  //      tiles are requested (1-D TMA bulk copies into its shared-memory
  //      ring) BEFORE the PDL wait, so they overlap the previous kernel
  // shared memory: [x: B*K fp16][(P,Q): B*K/16*pq_per_group float2][TMA ring: W x NS tiles]
  uint8_t* ring = smem + p.ring_offset + (size_t)warp * NS * tb;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  // the ring's mbarriers follow the ring: [W][kMaxStages] u64
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(
      smem + p.ring_offset + (size_t)(nthreads >> 5) * NS * tb + (size_t)warp * kMaxStages * 8);
  const uint64_t pol = evict_first_policy();
  // The ring is NP = NS/2 slots of two consecutive tiles: one bulk copy and
  // one mbarrier per tile pair (the host keeps NS even).
  const int NP = NS >> 1;
  auto fill_slot = [&](int slot, int t_first) {  // lane 0 only
    const int n = min(2, t_end - t_first);
    if (n > 0) {
      mbar_expect_tx(bar0 + 8 * slot, n * tb);
      bulk_g2s(ring_s + slot * 2 * tb, tiles + (int64_t)t_first * tb, n * tb, bar0 + 8 * slot, pol);
    }
  };
  if (lane == 0) {
    for (int s = 0; s < NP; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NP; ++s) fill_slot(s, t_begin + 2 * s);
  }
  __syncwarp();
  int row = -1;  // this lane's row in the first slice (the perm table is part of the blob)
  uint32_t hdr0 = 0, first0 = 0;
  if (t_end > t_begin) {
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(tiles + (int64_t)t_begin * tb));
    hdr0 = h.x;
    first0 = h.z;  // first tile of the slice the range starts in
    row = __ldg(p.perm + (int64_t)(hdr0 >> 2) * kLanes + lane);
  }
  // fix-up records of warps of the same CTA go through shared memory
  const int W = nthreads >> 5;
  const int cta_w0 = blockIdx.x * W;
  const int cta_t0 = cta_w0 * p.part_q + min(cta_w0, p.part_r);  // the CTA's first tile
  const uint32_t fx = p.fix_offset ? (uint32_t)__cvta_generic_to_shared(smem + p.fix_offset) : 0u;
  if (fx) {
    for (int i = threadIdx.x; i < W * B * kLanes; i += nthreads)
      asm volatile("st.shared.b64 [%0], %1;" ::"r"(fx + 8u * i), "l"(0ull) : "memory");
  }
  trace_point(p, gw, lane, 0);
  // let the next launch on the stream become resident now (it needs half an
  // SM: measured best; later triggers delay its weight prefetch)
  pdl_launch_dependents();
  pdl_wait();  // x, y, bias and the workspace may belong to the previous kernel
  trace_point(p, gw, lane, 1);

  // ---- stage activations in shared memory with plain 128-bit loads (not
  //      through the TMA unit, whose queue holds the weight ring fills) and
  //      compute the per-column-group sums X_{b,c} (fp32, fixed t order) from
  //      the same registers: one pass, one barrier.
  const int KG = p.cols / G;
  uint8_t* xs = smem;
  uint8_t* pq = xs + (size_t)B * p.cols * 2;  // [B][K/16 * pq_per_group] float2 (P, Q)
  stage_activations<BITS, B, false, G>(p, xs, pq, KG, nthreads);
  trace_point(p, gw, lane, 6);
  __syncthreads();

  // ---- empty rows get bias (or 0): grid-stride over the empty-row list
  for (int i = blockIdx.x * nthreads + threadIdx.x; i < p.n_empty; i += gridDim.x * nthreads) {
    const int erow = __ldg(p.empty + i);
    const float bias = p.bias ? __ldg(p.bias + erow) : 0.f;
#pragma unroll
    for (int b = 0; b < B; ++b) store_y(p, (int64_t)b * p.ldy + erow, bias);
  }
  trace_point(p, gw, lane, 2);
  if (t_end <= t_begin) {
    if (p.n_peers) __threadfence_system();
    return;
  }

  // ---- stream the warp's tile range; lane = one row of the current slice
  float acc[kMaxBatch];
#pragma unroll
  for (int b = 0; b < kMaxBatch; ++b) acc[b] = 0.f;
  bool foreign = !(hdr0 & kTileFirst);  // slice opened by an earlier warp
  uint32_t last_hdr = 0;
  int w_last = gw;
  unsigned long long pre[kPre][kMaxBatch];
  int s = 0;
  uint32_t phase = 0;
  trace_point(p, gw, lane, 3);

  // Per-tile work once its registers are loaded: accumulate the lane's four
  // groups, close the slice at its LAST tile, and (at the warp's final tile,
  // when it owns a slice continuing downstream) request the fix-up records.
  const bool local_owner = fx && (int)first0 >= cta_t0;  // owner of the opening slice is in this CTA
  int wg0 = gw + 1;  // first successor with a global record
  auto consume = [&](const TileRegs<BITS, G>& tr, int t) {
    if (t == t_end - 1 && !(tr.hdr & kTileLast) && !foreign) {
      w_last = warp_of_tile(p, t_end - 1 + (int)tr.rem);
      wg0 = fx ? max(gw + 1, min(w_last + 1, cta_w0 + W)) : gw + 1;
#pragma unroll
      for (int k = 0; k < kPre; ++k)
#pragma unroll
        for (int b = 0; b < B; ++b)
          pre[k][b] = (wg0 + k <= w_last) ? ld_slot(ws_slot<B>(p, wg0 + k, b, lane)) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kPerLane; ++u) group_accumulate<BITS, B, G>(p, tr, u, acc);
    last_hdr = tr.hdr;
    if (tr.hdr & kTileLast) {  // the slice ends in this tile: its rows are complete
      if (foreign) publish<B>(p, gw, acc, lane, local_owner, fx, gw - cta_w0);
      else store_rows<B>(p, acc, row, lane);
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = 0.f;
      foreign = false;
      if (t + 1 < t_end) row = __ldg(p.perm + (int64_t)((tr.hdr >> 2) + 1) * kLanes + lane);
    }
  };
  // two tiles per iteration: one ring handshake (wait, copy) per pair, and
  // the x gathers of both tiles can be in flight together
  int t = t_begin;
  for (; t + 1 < t_end; t += 2) {
    mbar_wait(bar0 + 8 * s, phase);
    const uint8_t* slot = ring + (size_t)s * 2 * tb;
    TileRegs<BITS, G> tr0, tr1;
    read_tile<BITS, G>(tr0, slot, lane);
    read_tile<BITS, G>(tr1, slot + tb, lane);
    __syncwarp();  // every lane has read the pair: refill its slot
    if (lane == 0) {
      // Generic-proxy reads of the slot, then an async-proxy (TMA) write to
      // it.  By default no fence.proxy.async (its MEMBAR cost 2 % per step):
      // the reads return within tens of cycles, the copy's first write lands
      // a global round trip (>= 0.5 us) later.  That is a timing argument,
      // not a memory-model guarantee; -DGQSA_PROXY_FENCE restores the fence.
#ifdef GQSA_PROXY_FENCE
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
      fill_slot(s, t + NS);
    }
    if (++s == NP) { s = 0; phase ^= 1u; }
    consume(tr0, t);
    consume(tr1, t + 1);
  }
  if (t < t_end) {  // odd count: the last slot holds one tile
    mbar_wait(bar0 + 8 * s, phase);
    TileRegs<BITS, G> tr;
    read_tile<BITS, G>(tr, ring + (size_t)s * 2 * tb, lane);
    consume(tr, t);
  }

  trace_point(p, gw, lane, 4);
  // ---- a slice left open at the end of the range continues downstream
  if (!(last_hdr & kTileLast)) {
    if (foreign) {  // the whole range lies inside a slice owned upstream
      publish<B>(p, gw, acc, lane, local_owner, fx, gw - cta_w0);
      if (p.trace && lane == 0) p.trace[(int64_t)gw * 8 + 7] = 1;
    } else {  // owner: add the successors' partials, then store
      collect<B>(p, gw, w_last, acc, lane, pre, wg0, fx, cta_w0);
      store_rows<B>(p, acc, row, lane);
      if (p.trace && lane == 0) p.trace[(int64_t)gw * 8 + 7] = 100 + w_last - gw;
    }
  } else if (p.trace && lane == 0) {
    p.trace[(int64_t)gw * 8 + 7] = 0;
  }
  trace_point(p, gw, lane, 5);
  if (p.n_peers) __threadfence_system();  // peer stores visible before the launch completes
}

// ---------------------------------------------------------------- launchers
template <int BITS, int B, bool FEW = false, int G = kGroup>
const void* kernel_ptr() {
  return reinterpret_cast<const void*>(&gqsa_streamk_kernel<BITS, B, FEW, G>);
}

#define GQSA_KSEL(BITS)                         \
  switch (B) {                                  \
    case 1: return kernel_ptr<BITS, 1>();       \
    case 2: return kernel_ptr<BITS, 2>();       \
    case 3: return kernel_ptr<BITS, 3>();       \
    case 4: return kernel_ptr<BITS, 4>();       \
    case 5: return kernel_ptr<BITS, 5>();       \
    case 6: return kernel_ptr<BITS, 6>();       \
    case 7: return kernel_ptr<BITS, 7>();       \
    case 8: return kernel_ptr<BITS, 8>();       \
    default: return nullptr;                    \
  }

#define GQSA_KSEL_G(G)                                  \
  switch (B) {                                          \
    case 1: return kernel_ptr<4, 1, false, G>();        \
    case 2: return kernel_ptr<4, 2, false, G>();        \
    case 3: return kernel_ptr<4, 3, false, G>();        \
    case 4: return kernel_ptr<4, 4, false, G>();        \
    case 5: return kernel_ptr<4, 5, false, G>();        \
    case 6: return kernel_ptr<4, 6, false, G>();        \
    case 7: return kernel_ptr<4, 7, false, G>();        \
    case 8: return kernel_ptr<4, 8, false, G>();        \
    default: return nullptr;                            \
  }

const void* select_kernel(int bits, int G, int B, bool few) {
  if (G != kGroup) {  // W4 at G = 8 / 32 (group-size sweep)
    if (bits != 4) return nullptr;
    if (G == 32 && few && B <= 2) return B == 1 ? kernel_ptr<4, 1, true, 32>() : kernel_ptr<4, 2, true, 32>();
    if (G == 8) { GQSA_KSEL_G(8) }
    if (G == 32) { GQSA_KSEL_G(32) }
    return nullptr;
  }
  if (few && B <= 2 && (bits == 4 || bits == 2)) {
    if (bits == 4) return B == 1 ? kernel_ptr<4, 1, true>() : kernel_ptr<4, 2, true>();
    return B == 1 ? kernel_ptr<2, 1, true>() : kernel_ptr<2, 2, true>();
  }
  if (bits == 4) { GQSA_KSEL(4) }
  if (bits == 2) { GQSA_KSEL(2) }
  if (bits == 8) { GQSA_KSEL(8) }
  return nullptr;
}

}  // namespace gqsa
