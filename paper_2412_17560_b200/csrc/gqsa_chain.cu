// gqsa_chain.cu -- persistent sm_100a kernel that runs a CHAIN of GQSA GEMVs
// (the decode sequence of a model's linear layers) in ONE launch.
//
// Each item j of the chain computes, exactly as one gqsa_gemv call
// (PAPER.md:64-69 [Eq. 3], 95-101 [§3.2 BSR], 134 [§3.5], 161 [Stream-K]):
//
//   Y_j[b][r] = sum_{g in row r} s_g * sum_t (q_{g,t} - z_g) X_j[b][c_g*G+t]  (+ bias_j[r])
//
// and item j reads X_j only after every earlier item has completed when
// wait_prev[j] is set (X_j may be an earlier item's output): a grid-wide
// arrival counter replaces the kernel boundary.  The point
// is that the weight stream never stops at a layer boundary: each warp's TMA
// ring runs ahead across items, so while the slowest warps finish item j
// (and while the barrier and activation staging of item j+1 are pending) the
// ring is already filling with item j+1's tiles, and one launch's CTA owns
// the whole SM, so the ring is ~3x deeper than the per-GEMV kernel's
// (which must leave half the SM to the next PDL launch).
//
// Per item the work is the per-GEMV kernel's: Stream-K over 128-group tiles
// at warp granularity, lane-per-row sliced ELL, offset-folded LOP3/FHFMA
// dequant-dot, deterministic cross-warp fix-up.  Requires all CTAs resident
// (cooperative launch, one CTA per SM).
#include "gqsa_device.cuh"

namespace gqsa {

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_acqrel_add(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int BITS, int B>
__global__ void __launch_bounds__(kChainThreads, 1) gqsa_chain_kernel(const __grid_constant__ ChainParams cp) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nthreads = blockDim.x;
  const int W = nthreads >> 5;
  const int gw = blockIdx.x * W + warp;
  const int tb = tile_bytes(BITS);
  const int NS = cp.stages;
  const int NP = NS >> 1;

  // this warp's Stream-K range of item j (+-1 tile per warp)
  auto range = [&](int j, int& b, int& e) {
    const KParams& p = cp.item[j];
    if (gw < p.active_warps) {
      b = gw * p.part_q + min(gw, p.part_r);
      e = b + p.part_q + (gw < p.part_r ? 1 : 0);
    } else {
      b = e = 0;
    }
  };

  // ---- TMA ring: NP slots of tile pairs per warp, filled in chain order
  //      (item by item, pairs never straddle items) by lane 0
  uint8_t* ring = smem + cp.ring_offset + (size_t)warp * NS * tb;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(
      smem + cp.ring_offset + (size_t)W * NS * tb + (size_t)warp * kMaxStages * 8);
  const uint64_t pol = evict_first_policy();
  int fj = 0, ft = 0, fe = 0;  // filler cursor: item, next tile, end of the warp's range
  range(0, ft, fe);
  auto fill_slot = [&](int slot) {  // lane 0 only
    while (ft >= fe) {
      if (++fj >= cp.n) return;
      range(fj, ft, fe);
    }
    const int n = min(2, fe - ft);
    mbar_expect_tx(bar0 + 8 * slot, n * tb);
    bulk_g2s(ring_s + slot * 2 * tb, cp.item[fj].tiles + (int64_t)ft * tb, n * tb, bar0 + 8 * slot, pol);
    ft += n;
  };
  if (lane == 0) {
    for (int s = 0; s < NP; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NP; ++s) fill_slot(s);
  }
  __syncwarp();
  pdl_launch_dependents();
  pdl_wait();  // the first item's x (and every buffer) may belong to the previous kernel

  const uint32_t fx = cp.fix_offset ? (uint32_t)__cvta_generic_to_shared(smem + cp.fix_offset) : 0u;
  const int cta_w0 = blockIdx.x * W;
  int s = 0;
  uint32_t phase = 0;

  for (int j = 0; j < cp.n; ++j) {
    const KParams& p = cp.item[j];
    int t_begin, t_end;
    range(j, t_begin, t_end);
    // the first tile's header (row of this lane, slice owner): from the blob
    int row = -1;
    uint32_t hdr0 = 0, first0 = 0;
    if (t_end > t_begin) {
      const uint4 h = __ldg(reinterpret_cast<const uint4*>(p.tiles + (int64_t)t_begin * tb));
      hdr0 = h.x;
      first0 = h.z;
      row = __ldg(p.perm + (int64_t)(hdr0 >> 2) * kLanes + lane);
    }
    // ---- item boundary: this CTA is done with item j-1 (x buffer and
    //      fix-up records free); with wait_prev, every warp of the grid is
    if (j > 0) {
      __syncthreads();
      if (cp.wait_prev[j] && threadIdx.x == 0) {
        const uint32_t target = (uint32_t)j * gridDim.x;
        int spins = 0;
        while (ld_acquire(cp.counter) < target) {
          if (++spins > (1 << 26)) __trap();  // a lost arrival: fail loudly, never hang the device
        }
      }
    }
    if (fx) {
      for (int i = threadIdx.x; i < W * B * kLanes; i += nthreads)
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(fx + 8u * i), "l"(0ull) : "memory");
    }
    __syncthreads();
    const int KG = p.cols / kGroup;
    uint8_t* xs = smem;
    uint8_t* pq = xs + (size_t)B * p.cols * 2;
    if (cp.trace && lane == 0) cp.trace[((int64_t)gw * cp.n + j) * 4 + 0] = globaltimer();
    if (!cp.reuse_x[j]) {  // else: same X as item j-1 and no wait: x and (P, Q) are in place
      stage_activations<BITS, B, true>(p, xs, pq, KG, nthreads);
      __syncthreads();
    }
    if (cp.trace && lane == 0) cp.trace[((int64_t)gw * cp.n + j) * 4 + 1] = globaltimer();
    for (int i = blockIdx.x * nthreads + threadIdx.x; i < p.n_empty; i += gridDim.x * nthreads) {
      const int erow = __ldg(p.empty + i);
      const float bias = p.bias ? __ldg(p.bias + erow) : 0.f;
#pragma unroll
      for (int b = 0; b < B; ++b) store_y(p, (int64_t)b * p.ldy + erow, bias);
    }

    if (t_end > t_begin) {
      const int cta_t0 = cta_w0 < p.active_warps ? cta_w0 * p.part_q + min(cta_w0, p.part_r) : p.num_tiles;
      float acc[kMaxBatch];
#pragma unroll
      for (int b = 0; b < kMaxBatch; ++b) acc[b] = 0.f;
      bool foreign = !(hdr0 & kTileFirst);
      uint32_t last_hdr = 0;
      int w_last = gw;
      unsigned long long pre[kPre][kMaxBatch];
      const bool local_owner = fx && (int)first0 >= cta_t0;
      int wg0 = gw + 1;
      auto consume = [&](const TileRegs<BITS>& tr, int t) {
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
        for (int u = 0; u < kPerLane; ++u) group_accumulate<BITS, B>(p, tr, u, acc);
        last_hdr = tr.hdr;
        if (tr.hdr & kTileLast) {
          if (foreign) publish<B>(p, gw, acc, lane, local_owner, fx, gw - cta_w0);
          else store_rows<B>(p, acc, row, lane);
#pragma unroll
          for (int b = 0; b < B; ++b) acc[b] = 0.f;
          foreign = false;
          if (t + 1 < t_end) row = __ldg(p.perm + (int64_t)((tr.hdr >> 2) + 1) * kLanes + lane);
        }
      };
      int t = t_begin;
      for (; t < t_end; t += 2) {
        mbar_wait(bar0 + 8 * s, phase);
        const uint8_t* slot = ring + (size_t)s * 2 * tb;
        const bool two = t + 1 < t_end;
        TileRegs<BITS> tr0, tr1;
        read_tile<BITS>(tr0, slot, lane);
        if (two) read_tile<BITS>(tr1, slot + tb, lane);
        __syncwarp();  // every lane has read the slot: refill it (possibly with the next item's tiles)
        if (lane == 0) {
      // Generic-proxy reads of the slot, then an async-proxy (TMA) write to
      // it.  By default no fence.proxy.async (its MEMBAR cost 2 % per step):
      // the reads return within tens of cycles, the copy's first write lands
      // a global round trip (>= 0.5 us) later.  That is a timing argument,
      // not a memory-model guarantee; -DGQSA_PROXY_FENCE restores the fence.
#ifdef GQSA_PROXY_FENCE
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
          fill_slot(s);
        }
        if (++s == NP) { s = 0; phase ^= 1u; }
        consume(tr0, t);
        if (two) consume(tr1, t + 1);
      }
      if (!(last_hdr & kTileLast)) {
        if (foreign) {
          publish<B>(p, gw, acc, lane, local_owner, fx, gw - cta_w0);
        } else {
          collect<B>(p, gw, w_last, acc, lane, pre, wg0, fx, cta_w0);
          store_rows<B>(p, acc, row, lane);
        }
      }
    }
    if (cp.trace && lane == 0) cp.trace[((int64_t)gw * cp.n + j) * 4 + 2] = globaltimer();
    // ---- arrive: ONE arrival per CTA once all its warps are done with item
    //      j (outputs and fix-up records written): 148 atomics per barrier on
    //      the counter's L2 slice instead of one per warp
    __syncthreads();
    if (threadIdx.x == 0) {
      // release at gpu scope; bar.sync above orders the CTA's other warps'
      // writes before it (cumulativity)
      if (j + 1 < cp.n) {
        red_release_add(cp.counter, 1u);
      } else {
        // the last arrival of the launch resets the counter for the next one
        // (read only after that launch's PDL wait)
        const uint32_t total = (uint32_t)cp.n * gridDim.x;
        if (atom_acqrel_add(cp.counter, 1u) == total - 1u) atomicExch(cp.counter, 0u);
      }
    }
  }
}

template <int BITS, int B>
const void* chain_kernel_ptr() {
  return reinterpret_cast<const void*>(&gqsa_chain_kernel<BITS, B>);
}

const void* select_chain_kernel(int bits, int B) {
  if (bits == 4) return B == 1 ? chain_kernel_ptr<4, 1>() : B == 2 ? chain_kernel_ptr<4, 2>() : nullptr;
  if (bits == 2) return B == 1 ? chain_kernel_ptr<2, 1>() : B == 2 ? chain_kernel_ptr<2, 2>() : nullptr;
  return nullptr;
}

}  // namespace gqsa
