// gqsa_stream.cu -- sm_100a Stream-K group-sparse W2/W4/W8 GEMV / small-batch
// GEMM over LAYOUT v3, for one or several independent GEMVs per launch.
//
// Computes, for every item (GEMV) of the launch, every batch column b < B and
// output row r (PAPER.md:64-69 [Eq. 3], 95-101 [§3.2 BSR], 134 [§3.5]):
//
//   y[b][r] = sum_{g in row r} s_g * ( sum_t q_{g,t} x[b][c_g*G+t] - z_g * X_{b,c_g} ),
//   X_{b,c} = sum_t x[b][c*G+t]       (Eq. 3 applied per group, z folded once)
//
// Design:
//  * Layout: rows sorted by kept-group count, cut into 32-lane
//    slices (sliced ELL); a lane owns a row and walks its groups slot by slot,
//    so the hot loop has no cross-lane reduction at all.
//  * Task-centric partition (PAPER.md:161 Stream-K, App. J): the
//    launch's concatenated tile stream (all items, 128 groups per tile) is cut
//    into contiguous, equal (+-1 tile) ranges, one per WARP, regardless of
//    row, slice or item boundaries.
//  * Weights stream HBM -> registers (128-bit no-allocate loads, evict-first
//    L2 policy) plus an L2 prefetch of the tile two ahead, the first ones
//    requested BEFORE griddepcontrol.wait (they never depend on the previous
//    kernel).  No shared-memory staging of weights: shared memory serves only
//    the activation gathers.
//  * Pipelined launches (HALF = 1; x_ready, B <= 2): the grid
//    takes part of every SM so the next launches run beside it, and every
//    global write (rows, fix-up records) is deferred until after
//    griddepcontrol.wait -- closed slices' rows wait in shared memory.
//  * The loop is issue-bound at 6 TB/s: keep per-tile instructions out of it
//    (DESIGN.md §11).
//  * Activations are staged in shared memory once per CTA (the items its
//    range touches), with the negated column-group sums (-P, -Q) the
//    offset-folded dequantization needs and a zero block for padding slots.
//  * Dequantization: LOP3 magic (0x6400 = fp16 1024) turns code fields into
//    exact fp16 (1024 + 2^k q); FHFMA (fma.rn.f32.f16) multiplies them by fp16
//    x with exact products into an fp32 chain that STARTS at -P - z Q, so the
//    offsets and z leave with one FFMA and s is applied with one more.  No
//    tensor cores: the rows of a warp hold groups at unrelated columns
//    (DESIGN.md §10), and batch 1 is bandwidth-bound.
//  * Fix-up (slices split across warps), look-back: every participant but the
//    last publishes its per-lane partials as 64-bit {value, flag} records; the
//    participant holding the slice's last tile adds them in order
//    (deterministic), then its own, stores the rows and resets the flags.  It
//    waits only for lower-indexed participants, which never wait for a higher
//    one.  Whole-SM launches first reduce the pieces inside each CTA through
//    shared memory, so only CTA-level partials cross CTAs.
#include "gqsa_device.cuh"

namespace gqsa {

namespace {

__device__ __forceinline__ void range_of(const Params& p, int w, int& b, int& e) {
  b = w * p.part_q + min(w, p.part_r);
  e = b + p.part_q + (w < p.part_r ? 1 : 0);
}
// Warp that owns global tile t under the +-1 partition.
__device__ __forceinline__ int warp_of_tile(const Params& p, int t) {
  const int big = p.part_r * (p.part_q + 1);
  return t < big ? t / (p.part_q + 1) : p.part_r + (t - big) / p.part_q;
}
__device__ __forceinline__ int item_of(const Params& p, int t) {
  int i = 0;
  while (i + 1 < p.n_items && t >= p.item[i].tile_end) ++i;
  return i;
}
// First tile of CTA c under slice-aligned CTA ranges (Params::cta_slicek, one
// item): the slice boundary nearest to the even split c * total / grid.
// Monotone in c; two CTAs may share a boundary (an empty CTA).
__device__ __forceinline__ int cta_boundary(const Params& p, int c) {
  if (c <= 0) return 0;
  if (c >= (int)gridDim.x) return p.total_tiles;
  const int ideal = (int)((int64_t)c * p.total_tiles / gridDim.x);
  const Item& it = p.item[0];
  const int s = __ldg(it.tile_slice + ideal);
  const int b0 = __ldg(it.slice_tile0 + s);
  if (b0 == ideal) return ideal;
  const int b1 = __ldg(it.slice_tile0 + s + 1);
  return ideal - b0 <= b1 - ideal ? b0 : b1;
}
// Shared-memory offset of item i's staged activations in a CTA whose tile
// range is [t0, t1): the touched items are packed in item order.
__device__ __forceinline__ uint32_t item_smem_off(const Item* items, int i, int t0, int t1) {
  uint32_t off = 0;
  for (int j = 0; j < i; ++j)
    if (item_touched(items[j], t0, t1)) off += (uint32_t)items[j].smem_bytes;
  return off;
}

// y element i of item `it`: fp32, or fp16 rounded to nearest even (PAPER.md:134 step 5).
__device__ __forceinline__ void store_y(const Item& it, int out_f16, int64_t i, float v) {
  if (it.peer_mc) {  // fused all-gather over NVLink SHARP: one multicast store reaches every rank (fp32 only)
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(reinterpret_cast<float*>(it.peer_y[0]) + i +
                                                                      it.row_offset),
                 "f"(v)
                 : "memory");
    return;
  }
  if (it.n_peers) {  // fused all-gather: this shard's rows land in every rank's full y
#pragma unroll 1
    for (int k = 0; k < it.n_peers; ++k) {
      if (out_f16) reinterpret_cast<__half*>(it.peer_y[k])[i + it.row_offset] = __float2half_rn(v);
      else reinterpret_cast<float*>(it.peer_y[k])[i + it.row_offset] = v;
    }
    return;
  }
  if (out_f16) reinterpret_cast<__half*>(it.Y)[i] = __float2half_rn(v);
  else reinterpret_cast<float*>(it.Y)[i] = v;
}

// Sum over the S lanes of a row (S = lanes per row, a power of two) and store.
template <int B>
__device__ __forceinline__ void store_rows(const Params& p, const Item& it, float (&v)[B], int row, int lane) {
  const int S = it.lanes_per_row;
  for (int d = 1; d < S; d <<= 1) {
#pragma unroll
    for (int b = 0; b < B; ++b) v[b] += __shfl_xor_sync(0xffffffffu, v[b], d);
  }
  if (row >= 0 && (lane & (S - 1)) == 0) {
    const float bias = it.bias ? __ldg(it.bias + row) : 0.f;
#pragma unroll
    for (int b = 0; b < B; ++b) store_y(it, p.out_f16, (int64_t)b * it.ldy + row, v[b] + bias);
  }
}

// Pipelined mode: reduce over the row's S lanes as store_rows does, but keep
// the result in the warp's shared-memory buffer slot k (the lane that would
// store it records row | item << 28, the others -1).
template <int B>
__device__ __forceinline__ void defer_rows(const Item& it, float (&v)[B], int row, int item, int lane, uint32_t* buf,
                                           int k) {
  const int S = it.lanes_per_row;
  for (int d = 1; d < S; d <<= 1) {
#pragma unroll
    for (int b = 0; b < B; ++b) v[b] += __shfl_xor_sync(0xffffffffu, v[b], d);
  }
  uint32_t* e = buf + k * 32 * (B + 1);
  e[lane] = (row >= 0 && (lane & (S - 1)) == 0) ? ((uint32_t)row | ((uint32_t)item << 28)) : 0xffffffffu;
#pragma unroll
  for (int b = 0; b < B; ++b) e[(b + 1) * 32 + lane] = __float_as_uint(v[b]);
}
template <int B>
__device__ __forceinline__ void flush_deferred(const Params& p, const Item* items, const uint32_t* buf, int k,
                                               int lane) {
  const uint32_t* e = buf + k * 32 * (B + 1);
  const uint32_t ri = e[lane];
  if (ri == 0xffffffffu) return;
  const int row = (int)(ri & 0x0fffffffu);
  const Item& it = items[ri >> 28];
  const float bias = it.bias ? __ldg(it.bias + row) : 0.f;
#pragma unroll
  for (int b = 0; b < B; ++b) store_y(it, p.out_f16, (int64_t)b * it.ldy + row, __uint_as_float(e[(b + 1) * 32 + lane]) + bias);
}

// ---------------------------------------------------------------- fix-up
// Record of warp w for its head (which = 0) or tail (which = 1) slice:
// [B][32 lanes] 8-byte words {partial, flag}; each is ONE 64-bit store, so a
// reader that sees the flag sees the value (single-copy atomicity).
template <int B>
__device__ __forceinline__ unsigned long long* rec_ptr(const Params& p, int w, int which, int b, int lane) {
  return p.rec + (((int64_t)w * 2 + which) * B + b) * kLanes + lane;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* a, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
template <int B>
__device__ __forceinline__ void publish(const Params& p, int w, int which, const float (&v)[B], int lane) {
#pragma unroll
  for (int b = 0; b < B; ++b)
    st_relaxed64(rec_ptr<B>(p, w, which, b, lane), (1ull << 32) | __float_as_uint(v[b]));
}
// Records loaded per round trip by a collector.
#ifndef GQSA_KREC
#define GQSA_KREC 8
#endif
constexpr int kRec = GQSA_KREC;
// A record whose flag was not yet visible: poll it (rare; kept out of line so
// that the collect loop stays small -- the fix-up runs once per launch and
// its code is cold in the instruction cache).
__device__ __noinline__ unsigned long long wait_record(const unsigned long long* a) {
  unsigned long long v = ld_relaxed64(a);
  unsigned int spins = 0;
  while ((v >> 32) == 0ull) {
    if (++spins > (1u << 26)) __trap();  // a lost record: fail loudly, never hang
    __nanosleep(32);
    v = ld_relaxed64(a);
  }
  return v;
}
// Look-back fix-up.  A slice split over participants c0..c1 (CTAs in the
// CTA-level fix-up of whole-SM launches, Params::cta_fix; warps otherwise) is
// finished by c1, the participant holding its last tile: c0..c1-1 publish
// their partial as a record (c0: tail record, the others: head records) and
// move on; c1 adds the records in participant order, then its own partial,
// and stores the rows.  c1 waits only for LOWER-indexed participants, which
// never wait for a higher one -- the forward-progress assumption of decoupled
// look-back (CTAs are dispatched in index order; the warps of a CTA are
// co-resident) -- so there is no arrival counter and no atomic round trip.
template <int B>
__device__ __noinline__ void collect_lower(const Params& p, const Item* items, int c0, int c1, const float (&own)[B],
                                           int item, int row, int lane) {
  float v[B];
#pragma unroll
  for (int b = 0; b < B; ++b) v[b] = 0.f;
#pragma unroll 1
  for (int cb = c0; cb < c1; cb += kRec) {
    unsigned long long r[kRec][B];
#pragma unroll
    for (int k = 0; k < kRec; ++k)
#pragma unroll
      for (int b = 0; b < B; ++b)
        r[k][b] = cb + k < c1 ? ld_relaxed64(rec_ptr<B>(p, cb + k, cb + k == c0 ? 1 : 0, b, lane)) : (1ull << 32);
#pragma unroll
    for (int k = 0; k < kRec; ++k) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (cb + k >= c1) continue;
        unsigned long long* a = rec_ptr<B>(p, cb + k, cb + k == c0 ? 1 : 0, b, lane);
        if ((r[k][b] >> 32) == 0ull) r[k][b] = wait_record(a);
        v[b] = (cb + k == c0) ? __uint_as_float((uint32_t)r[k][b]) : v[b] + __uint_as_float((uint32_t)r[k][b]);
        st_relaxed64(a, 0ull);
      }
    }
  }
#pragma unroll
  for (int b = 0; b < B; ++b) v[b] += own[b];
  store_rows<B>(p, items[item], v, row, lane);
}
template <int B>
__device__ __forceinline__ void cta_finish(const Params& p, const Item* items, const float (&v)[B], int c0, int c,
                                           int c1, int item, int row, int lane) {
  if (c < c1) publish<B>(p, c, c == c0 ? 1 : 0, v, lane);
  else collect_lower<B>(p, items, c0, c1, v, item, row, lane);
}

// Empty rows get bias (or 0): grid-stride over every item's empty-row list.
template <int B>
__device__ __forceinline__ void store_empty_rows(const Params& p, const Item* items) {
  for (int i = 0; i < p.n_items; ++i) {
    const Item& it = items[i];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < it.n_empty; k += gridDim.x * blockDim.x) {
      const int erow = __ldg(it.empty + k);
      const float bias = it.bias ? __ldg(it.bias + erow) : 0.f;
#pragma unroll
      for (int b = 0; b < B; ++b) store_y(it, p.out_f16, (int64_t)b * it.ldy + erow, bias);
    }
  }
}

// Optional timeline instrumentation (gqsa_debug_trace): lane 0 of each warp
// stamps %globaltimer at fixed points; off (one predicated branch) by default.
__device__ __forceinline__ void trace_point(const Params& p, int gw, int lane, int k) {
  if (p.trace && lane == 0 && gw < p.active_warps) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(int64_t)gw * 8 + k] = t;
  }
}

}  // namespace

template <int BITS, int B, int G, int HALF>
__global__ void __launch_bounds__(32 * warps_of(B, HALF), HALF ? pipe_ctas_for(B) : min_blocks_for(B))
    gqsa_stream_kernel(const __grid_constant__ Params p) {
  const int W = blockDim.x >> 5;  // warps per CTA (<= warps_of(B, HALF); fewer for small launches)
  constexpr int TB = tile_bytes(BITS, G);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * W + warp;
  trace_point(p, gw, lane, 0);
  // per-item parameters, copied to shared memory: the loop indexes them by
  // a runtime item number (indexed parameter-space loads can miss the
  // constant cache); visible after the staging barrier
  __shared__ Item s_item[kMaxItems];
  static_assert(sizeof(Item) % 8 == 0, "item copy");
  for (int i = threadIdx.x; i < p.n_items * (int)(sizeof(Item) / 8); i += blockDim.x)
    reinterpret_cast<uint64_t*>(s_item)[i] = reinterpret_cast<const uint64_t*>(p.item)[i];
  const Item* its = p.item;  // -> s_item after the barrier

  // ---- task-centric partition: contiguous tile range per warp (+-1 tile)
  int t_begin = 0, t_end = 0;
  // the CTA's range (its warps' ranges are consecutive): which items it stages
  int cta_t0 = 0, cta_t1 = 0;
  int nbusy = 0;  // warps of this CTA with tiles (the trailing ones may be idle)
  if (p.cta_slicek) {
    // slice-aligned CTA ranges (single-item whole-SM launches): every CTA
    // starts and ends on a slice boundary, its warps split its range +-1 tile,
    // so every split slice is finished inside the CTA (CTA-level fix-up)
    cta_t0 = cta_boundary(p, blockIdx.x);
    cta_t1 = cta_boundary(p, blockIdx.x + 1);
    const int n = cta_t1 - cta_t0, q = n / W, r = n % W;
    t_begin = cta_t0 + warp * q + min(warp, r);
    t_end = t_begin + q + (warp < r ? 1 : 0);
    nbusy = min(W, n);
  } else {
    if (gw < p.active_warps) range_of(p, gw, t_begin, t_end);
    const int w0 = blockIdx.x * W, w1 = min(w0 + W, p.active_warps) - 1;
    if (w0 < p.active_warps) {
      int e;
      range_of(p, w0, cta_t0, e);
      range_of(p, w1, e, cta_t1);
    }
    nbusy = min(W, p.active_warps - blockIdx.x * W);
  }
  if (p.slice_k && t_end > t_begin) {
    // data-centric partition (Slice-K): the warp owns the slices whose FIRST
    // tile lies in its Stream-K range, each in full
    const int ib = item_of(p, t_begin);
    const Item& a = p.item[ib];
    const int sb = __ldg(a.tile_slice + (t_begin - a.tile_begin));
    const int st = a.tile_begin + __ldg(a.slice_tile0 + sb);
    const int b = st == t_begin ? t_begin : a.tile_begin + __ldg(a.slice_tile0 + sb + 1);
    const int ie = item_of(p, t_end - 1);
    const Item& c = p.item[ie];
    const int se = __ldg(c.tile_slice + (t_end - 1 - c.tile_begin));
    const int e = c.tile_begin + __ldg(c.slice_tile0 + se + 1);
    t_begin = b;
    t_end = b < t_end ? e : b;
  }

  if (p.wait_first) pdl_wait();  // experiments: no weight loads before the previous kernel completes
  // ---- the first tiles: requested before anything else (weights never
  //      depend on the previous kernel on the stream)
  const uint64_t pol = evict_first_policy();
  constexpr int kBufs = bufs_for(B), kL2Pf = l2pf_for(B);
  TileRegs<BITS, G> buf[kBufs];
  int li = 0, lend = 0;  // load cursor: item, end of its tiles
  const uint8_t* lptr = nullptr;
  if (t_end > t_begin) {
    li = item_of(p, t_begin);
    lptr = p.item[li].tiles + (size_t)(t_begin - p.item[li].tile_begin) * TB;
    lend = p.item[li].tile_end;
  }
  auto issue = [&](TileRegs<BITS, G>& r, int t) {  // t: the next tile of the load cursor
    if (t == lend) {
      do { ++li; } while (its[li].tile_end == its[li].tile_begin);
      lptr = its[li].tiles;
      lend = its[li].tile_end;
    }
    load_tile<BITS, G>(r, lptr, lane, pol);
#if GQSA_LANE_PF
    // per-lane L2 prefetch of the tile kL2Pf ahead: lane l fetches its 128-B line
    // (cheaper to issue than one bulk prefetch from lane 0 with uniform operands)
    if (kL2Pf > kBufs && lane < TB / 128 && t + kL2Pf < min(t_end, lend))
      prefetch_line_l2(lptr + (size_t)kL2Pf * TB + lane * 128);
#else
    if (kL2Pf > kBufs && lane == 0 && t + kL2Pf < min(t_end, lend)) prefetch_l2(lptr + (size_t)kL2Pf * TB, TB);
#endif
    lptr += TB;
  };
  if (kL2Pf > kBufs && lane == 0 && t_end > t_begin) {
    // the tiles between the register buffers and the prefetch distance, as
    // ONE bulk prefetch (contiguous within the item; later tiles: issue());
    // prefetching further ahead here measured slower
    const int n = min(t_begin + kL2Pf, min(t_end, lend)) - (t_begin + kBufs);
    if (n > 0) prefetch_l2(lptr + (size_t)kBufs * TB, (uint32_t)(n * TB));
  }
#pragma unroll
  for (int k = 0; k < kBufs; ++k)
    if (t_begin + k < t_end) issue(buf[k], t_begin + k);

  // ---- slice cursor: current slice (item ci, slice cs, global first / end
  //      tile cst0 / cend, this lane's row crow) and the next one, prefetched.
  //      Only the first lookup is issued before the PDL trigger; everything
  //      that depends on it is consumed after the activations are staged.
  int ci = 0, cs = 0, cst0 = 0, cend = 0, crow = -1;
  int ni = 0, ns = 0, nend = 0, nrow = -1;
  auto prefetch_next = [&]() {  // successor of (ci, cs), if the range continues past cend
    if (cend >= t_end) return;
    ni = ci;
    ns = cs + 1;
    if (ns == its[ci].num_slices) {
      do { ++ni; } while (its[ni].tile_end == its[ni].tile_begin);
      ns = 0;
    }
    const Item& it = its[ni];
    nend = it.tile_begin + __ldg(it.slice_tile0 + ns + 1);
    nrow = __ldg(it.perm + (int64_t)ns * kLanes + lane);
  };
  if (t_end > t_begin) {
    ci = item_of(p, t_begin);
    cs = __ldg(p.item[ci].tile_slice + (t_begin - p.item[ci].tile_begin));
  }

  // let the next launch on the stream start its prologue (its weight loads);
  // triggering later (e.g. half-way through the range) measured slower
  pdl_launch_dependents();
  // the first slice's bounds and rows and the staging table: immutable blob
  // and parameters only, so they are fetched before the PDL wait
  if (t_end > t_begin) {
    const Item& it = p.item[ci];
    cst0 = it.tile_begin + __ldg(it.slice_tile0 + cs);
    cend = it.tile_begin + __ldg(it.slice_tile0 + cs + 1);
    crow = __ldg(it.perm + (int64_t)cs * kLanes + lane);
  }
  StageEntry* const stab = reinterpret_cast<StageEntry*>(smem + p.stage_tab_offset);
  stage_table<B, G>(p, cta_t0, cta_t1, stab);
  // x may be the previous kernel's output; with x_ready the wait is deferred
  // to just before this launch's first global write (y, fix-up records)
  bool waited = !p.x_ready;
  if (waited) pdl_wait();
  trace_point(p, gw, lane, 1);

  // ---- stage the activations of every item this CTA's range touches
  stage_all<BITS, B, G>(p, smem, stab);
  __syncthreads();
  its = s_item;
  trace_point(p, gw, lane, 2);
  auto ensure_wait = [&]() {
    if (!waited) {
      pdl_wait();
      waited = true;
    }
  };
  if (t_end <= t_begin) {
    ensure_wait();
    store_empty_rows<B>(p, its);
    if (p.item[0].n_peers) __threadfence_system();
    return;
  }
  bool foreign = cst0 < t_begin;  // the current slice began in an earlier warp's range
  int cw0 = foreign ? warp_of_tile(p, cst0) : gw;  // warp owning the current slice's first tile
  prefetch_next();

  // ---- stream the warp's tile range; lane = one row of the current slice
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  XView xv;
  auto set_item = [&]() {
    const Item& it = its[ci];
    xv.xs = sbase + item_smem_off(its, ci, cta_t0, cta_t1);
    xv.xrow = (uint32_t)it.xrow;
    xv.pq = xv.xs + (uint32_t)B * xv.xrow;
    xv.pqrow = (uint32_t)it.pqrow;
  };
  set_item();
  float acc[B];
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.f;
  // head slice (began upstream, closed in this range): this warp holds its last
  // tile, so it collects it after the loop (look-back)
  int h_w0 = 0, h_item = 0, h_row = -1;
  // pipelined mode: rows of slices closed before the PDL wait, buffered per
  // lane in shared memory ([slot][lane] row | item << 28, then [slot][b][lane]
  // values), and the head slice's partial (published after the wait)
  uint32_t* dbuf = HALF ? reinterpret_cast<uint32_t*>(smem + p.defer_offset + warp * defer_bytes_per_warp(B)) : nullptr;
  int n_def = 0;
  // CTA-level fix-up (whole-SM launches): split slices are reduced in shared
  // memory after the loop; the head slice's partial waits in hacc
  const bool cfix = !HALF && p.cta_fix && !p.slice_k;
  bool h_defer = false;
  float hacc[B];
  trace_point(p, gw, lane, 3);

  auto consume = [&](const TileRegs<BITS, G>& tr, int t) {
#pragma unroll
    for (int u = 0; u < kPerLane; ++u) group_accumulate<BITS, B, G>(tr, u, acc, xv);
#ifdef GQSA_TRACE_TILE0  // debug builds: a per-tile check is too costly in the hot loop
    if (p.trace && t == t_begin) trace_point(p, gw, lane, 6);  // first tile landed and consumed
#endif
    if (t + 1 == cend) {  // the slice ends with this tile: its rows are complete here
      if (!HALF) ensure_wait();
      if (foreign) {  // ... but began upstream: finished after the loop (look-back / CTA reduction)
        h_w0 = cw0;
        h_item = ci;
        h_row = crow;
        h_defer = true;
#pragma unroll
        for (int b = 0; b < B; ++b) hacc[b] = acc[b];
      } else if (HALF && !waited && n_def < kDeferSlots) {
        defer_rows<B>(its[ci], acc, crow, ci, lane, dbuf, n_def++);
      } else {
        ensure_wait();
        store_rows<B>(p, its[ci], acc, crow, lane);
      }
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = 0.f;
      foreign = false;
      cw0 = gw;
      if (t + 1 < t_end) {  // advance to the prefetched next slice
        const bool new_item = ni != ci;
        ci = ni;
        cs = ns;
        cend = nend;
        crow = nrow;
        if (new_item) set_item();
        prefetch_next();
      }
    }
  };

  int t = t_begin;
  while (t < t_end) {
#pragma unroll
    for (int k = 0; k < kBufs; ++k) {
      if (t < t_end) {
        consume(buf[k], t);
        if (t + kBufs < t_end) issue(buf[k], t + kBufs);
        ++t;
      }
    }
  }
  trace_point(p, gw, lane, 4);
  ensure_wait();
  if (HALF)  // the row stores deferred during the loop
    for (int k = 0; k < n_def; ++k) flush_deferred<B>(p, its, dbuf, k, lane);

  int fix_path = 0;  // debug trace: 2 published, +10 head collected; CTA level: 4 stored in the CTA, 5 CTA piece
                     // published or collected
  if (cfix) {
    // ---- CTA-level fix-up.  The CTA's warps hold consecutive ranges, so the
    //      pieces of a slice inside the CTA belong to consecutive warps: the
    //      slice's first warp here (its owner, or warp 0 for a slice that
    //      began in an earlier CTA) adds them in warp order from shared
    //      memory (the activation staging is dead once every loop is done).
    //      Only slices crossing a CTA boundary reach the global look-back,
    //      with one record per CTA instead of one per warp.
    const int nw = nbusy;
    asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
    float* P = reinterpret_cast<float*>(smem);  // [W][2: head, tail][B][32]
    int* meta = reinterpret_cast<int*>(smem + (size_t)W * 2 * B * kLanes * 4);
    const bool has_t = cend > t_end;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (h_defer) P[((warp * 2 + 0) * B + b) * kLanes + lane] = hacc[b];
      if (has_t) P[((warp * 2 + 1) * B + b) * kLanes + lane] = acc[b];
    }
    if (lane == 0) meta[warp] = (h_defer ? 1 : 0) | (has_t && foreign ? 2 : 0);
    asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
#ifdef GQSA_TRACE_FIX  // debug builds: the CTA's pieces are in shared memory (trace slot 6)
    trace_point(p, gw, lane, 6);
#endif
    const int c = blockIdx.x;
    if (has_t && (!foreign || warp == 0)) {  // this warp starts the CTA's piece of its open slice
      float v[B];
#pragma unroll
      for (int b = 0; b < B; ++b) v[b] = acc[b];
      bool closed = false;
#pragma unroll 1
      for (int k = warp + 1; k < nw && !closed; ++k) {
        const int m = meta[k];
        closed = !(m & 2);  // warp k is not a middle participant: the slice closes in its range
#pragma unroll
        for (int b = 0; b < B; ++b) v[b] += P[((k * 2 + (closed ? 0 : 1)) * B + b) * kLanes + lane];
      }
      if (closed && !foreign) {
        store_rows<B>(p, its[ci], v, crow, lane);
        fix_path += 4;
      } else {
        cta_finish<B>(p, its, v, foreign ? cw0 / W : c, c, closed ? c : warp_of_tile(p, cend - 1) / W, ci, crow,
                      lane);
        fix_path += 5;
      }
    }
    // after this warp's own piece is out (publish before waiting: no chains of waits across CTAs)
    if (warp == 0 && h_defer) {  // a slice from an earlier CTA closed in warp 0: its only piece here
      cta_finish<B>(p, its, hacc, h_w0 / W, c, c, h_item, h_row, lane);
      fix_path += 10;
    }
  }
  if (!cfix) {
    // ---- warp-level look-back: publish this warp's piece of the slice left
    //      open at the range end (head record if the slice began upstream),
    //      then finish the slice that began upstream and closed here
    if (cend > t_end) {
      publish<B>(p, gw, foreign ? 0 : 1, acc, lane);
      fix_path = 2;
    }
    if (h_defer) {
      collect_lower<B>(p, its, h_w0, gw, hacc, h_item, h_row, lane);
      fix_path += 10;
    }
  }
  if (p.trace && lane == 0 && gw < p.active_warps) p.trace[(int64_t)gw * 8 + 7] = (uint64_t)fix_path;
  store_empty_rows<B>(p, its);
  trace_point(p, gw, lane, 5);
  if (p.item[0].n_peers) __threadfence_system();  // peer stores visible before the launch completes
}

// ---------------------------------------------------------------- selection
template <int BITS, int B, int G = kGroup, int HALF = 0>
const void* kernel_ptr() {
  return reinterpret_cast<const void*>(&gqsa_stream_kernel<BITS, B, G, HALF>);
}

#define GQSA_KSEL(BITS, G)                    \
  switch (B) {                                \
    case 1: return half ? kernel_ptr<BITS, 1, G, 1>() : kernel_ptr<BITS, 1, G>();  \
    case 2: return half ? kernel_ptr<BITS, 2, G, 1>() : kernel_ptr<BITS, 2, G>();  \
    case 3: return kernel_ptr<BITS, 3, G>();  \
    case 4: return kernel_ptr<BITS, 4, G>();  \
    case 5: return kernel_ptr<BITS, 5, G>();  \
    case 6: return kernel_ptr<BITS, 6, G>();  \
    case 7: return kernel_ptr<BITS, 7, G>();  \
    case 8: return kernel_ptr<BITS, 8, G>();  \
    default: return nullptr;                  \
  }

const void* select_kernel(int bits, int G, int B, int half) {
  if (half && B > 2) return nullptr;
#ifdef GQSA_FAST_BUILD  // experiments: W4, G = 16 only
  if (bits == 4 && G == kGroup) { GQSA_KSEL(4, 16) }
  return nullptr;
#endif
  if (G == 8 && bits == 4) { GQSA_KSEL(4, 8) }
  if (G == 32 && bits == 4) { GQSA_KSEL(4, 32) }
  if (G != kGroup) return nullptr;
  if (bits == 4) { GQSA_KSEL(4, 16) }
  if (bits == 2) { GQSA_KSEL(2, 16) }
  if (bits == 8) { GQSA_KSEL(8, 16) }
  return nullptr;
}

}  // namespace gqsa
