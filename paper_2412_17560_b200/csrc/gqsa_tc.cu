// gqsa_tc.cu -- sm_100a small-batch (B = 2..8) group-sparse W4 GEMM over
// LAYOUT-TC on the tensor cores (mma.sync.m16n8k16, fp16 x fp16 -> fp32).
//
// Computes, for every batch column b < B and output row r (PAPER.md:64-69
// [Eq. 3], 95-101 [§3.2 BSR], 134 [§3.5 "TensorCores (MMA) or CudaCores"]):
//
//   y[b][r] = sum_{g in row r} s_g * ( sum_t q_{g,t} x[b][c_g*G+t] - z_g * X_{b,c_g} )
//
// Design:
//  * LAYOUT-TC: rows in blocks of 16; a block's ITEMS are the
//    group columns any of its rows keeps; an item is the 16 x 16 code matrix
//    of the block at that column (absent rows: zero codes, s = z = 0) stored
//    in A-fragment order -- one 32-bit word per lane.
//  * Per item one mma: A = 1024 + q (exact fp16 from the LOP3 magic, no
//    subtraction), B = the 16 x 8 activation slice x[b][16c .. 16c+15]
//    (batch columns >= B read as zero), D = 16 rows x 8 batch columns of raw
//    dots in fp32 (exact products); the epilogue removes the offset and z and
//    applies s per (row, item): acc += s (D - (1024 + z) X_c), X_c the staged
//    column sums.  Accumulators (2 rows x 2 batch columns per lane) live in
//    registers for the whole block.
//  * Weights stream HBM -> registers (768-B tiles of 4 items, 128-bit
//    no-allocate loads, four tiles in flight per warp), Stream-K over tiles;
//    blocks split across warps are reduced inside the CTA through shared
//    memory, and across CTAs by the wait-free last-arriver fix-up (4 values
//    per lane, one record per CTA), deterministic.
#include <cuda_fp16.h>

#include "gqsa_device.cuh"

namespace gqsa {

namespace {

constexpr int kNV = 4;  // accumulators per lane: rows g, g+8 x batch 2t, 2t+1
constexpr uint32_t kOnes = 0x3C003C00u;  // fp16 (1, 1)

// Record k of lane `lane` of warp w's head (which = 0) / tail (1) partial sum:
// a lane's kNV records are contiguous (two 128-bit accesses).
__device__ __forceinline__ unsigned long long* tc_rec(const TcParams& p, int w, int which, int v, int lane) {
  return p.rec + (((int64_t)w * 2 + which) * kLanes + lane) * kNV + v;
}
__device__ __forceinline__ void st_rel64(unsigned long long* a, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rel64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel64x2(unsigned long long* a, unsigned long long v0, unsigned long long v1) {
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(a), "l"(v0), "l"(v1) : "memory");
}
__device__ __forceinline__ void ld_rel64x2(const unsigned long long* a, unsigned long long& v0, unsigned long long& v1) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(v0), "=l"(v1) : "l"(a) : "memory");
}
__device__ __forceinline__ void tc_publish(const TcParams& p, int w, int which, const float (&v)[kNV], int lane) {
  unsigned long long* a = tc_rec(p, w, which, 0, lane);
  st_rel64x2(a, (1ull << 32) | __float_as_uint(v[0]), (1ull << 32) | __float_as_uint(v[1]));
  st_rel64x2(a + 2, (1ull << 32) | __float_as_uint(v[2]), (1ull << 32) | __float_as_uint(v[3]));
}
__device__ __forceinline__ int tc_arrive(const TcParams& p, int w0, int lane) {
  __syncwarp();
  int old = 0;
  if (lane == 0) old = (int)atomicAdd(p.cnt + w0, 1u);
  return __shfl_sync(0xffffffffu, old, 0);
}
__device__ __forceinline__ int tc_warp_of_tile(const TcParams& p, int t) {
  const int big = p.part_r * (p.part_q + 1);
  return t < big ? t / (p.part_q + 1) : p.part_r + (t - big) / p.part_q;
}

// y of block rows g, g+8 and batch columns 2t, 2t+1 (+ bias).
template <int B>
__device__ __forceinline__ void tc_store(const TcParams& p, int blk, const float (&v)[kNV], int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int k = 0; k < kNV; ++k) {
    const int row = blk * kTcRows + g + 8 * (k >> 1), b = 2 * t + (k & 1);
    if (b < B && row < p.rows) {
      const float val = v[k] + (p.bias ? __ldg(p.bias + row) : 0.f);
      const int64_t i = (int64_t)b * p.ldy + row;
      if (p.out_f16) reinterpret_cast<__half*>(p.Y)[i] = __float2half_rn(val);
      else reinterpret_cast<float*>(p.Y)[i] = val;
    }
  }
}

// The last arriver of a block split over warps w0..w1 adds every record in
// warp order (w0's tail record, then head records), resets them and the
// counter, and stores.  Only waits for records already issued.
template <int B>
__device__ __forceinline__ void tc_collect(const TcParams& p, int w0, int w1, int blk, int lane) {
  // A block spans up to ~12 warps.  The records of kChunk warps are requested
  // at once, and the code is kept compact (rolled loops, one re-read loop for
  // the rare not-yet-visible record): this tail code runs once per block on a
  // cold instruction cache, and an unrolled version cost several microseconds
  // of instruction fetch.
  constexpr int kChunk = 8;
  unsigned int total_spins = 0;
  float v[kNV];
#pragma unroll
  for (int k = 0; k < kNV; ++k) v[k] = 0.f;
#pragma unroll 1
  for (int wb = w0; wb <= w1; wb += kChunk) {
    unsigned long long r[kChunk][kNV];
#pragma unroll 1
    for (unsigned int spins = 0;; ++spins) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        if (wb + j <= w1) {
          const unsigned long long* a = tc_rec(p, wb + j, wb + j == w0 ? 1 : 0, 0, lane);
          ld_rel64x2(a, r[j][0], r[j][1]);
          ld_rel64x2(a + 2, r[j][2], r[j][3]);
        } else {
#pragma unroll
          for (int k = 0; k < kNV; ++k) r[j][k] = 1ull << 32;
        }
      }
#pragma unroll
      for (int j = 0; j < kChunk; ++j)
#pragma unroll
        for (int k = 0; k < kNV; ++k) ok = ok && (r[j][k] >> 32) != 0ull;
      if (ok) break;
      total_spins++;
      if (spins > (1u << 26)) __trap();
    }
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      if (wb + j <= w1)
#pragma unroll
        for (int k = 0; k < kNV; ++k)
          v[k] = (wb + j == w0) ? __uint_as_float((uint32_t)r[j][k]) : v[k] + __uint_as_float((uint32_t)r[j][k]);
#pragma unroll
    for (int j = 0; j < kChunk; ++j)
      if (wb + j <= w1) {
        unsigned long long* a = tc_rec(p, wb + j, wb + j == w0 ? 1 : 0, 0, lane);
        st_rel64x2(a, 0ull, 0ull);
        st_rel64x2(a + 2, 0ull, 0ull);
      }
  }
  if (lane == 0) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p.cnt + w0), "r"(0u) : "memory");
  tc_store<B>(p, blk, v, lane);
#ifdef GQSA_TC_SPINTRACE
  if (p.trace && lane == 0) p.trace[(int64_t)(blockIdx.x * kTcWarps + (threadIdx.x >> 5)) * 8 + 7] = 1000000ull * (w1 - w0 + 1) + total_spins;
#endif
}

// CTA-level fix-up: CTA c's (already reduced) piece of a block split over
// CTAs c0..c1 takes the last-arriver protocol with CTAs as participants.
template <int B>
__device__ __forceinline__ void tc_cta_finish(const TcParams& p, const float (&v)[kNV], int c0, int c, int c1,
                                              int blk, int lane) {
  tc_publish(p, c, c == c0 ? 1 : 0, v, lane);
  if (tc_arrive(p, c0, lane) == c1 - c0) tc_collect<B>(p, c0, c1, blk, lane);
}

struct TcTile {
  uint4 codes;  // items 0..3: this lane's A-fragment word
  uint4 sz0;    // items 0, 1: (s, z) of rows g, g+8
  uint4 sz1;    // items 2, 3
  uint2 cols;   // 4 x u16 item columns (uniform)
};

__device__ __forceinline__ void tc_load(TcTile& r, const TcParams& p, int t, int lane, uint64_t pol) {
  const uint8_t* tile = p.tiles + (size_t)t * kTcTileBytes;
  r.codes = ldg_stream128(tile + lane * 16, pol);
  r.sz0 = ldg_stream128(tile + 512 + (lane >> 2) * 32, pol);
  r.sz1 = ldg_stream128(tile + 512 + (lane >> 2) * 32 + 16, pol);
  r.cols = __ldg(reinterpret_cast<const uint2*>(p.tile_cols) + t);
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f), "f"(0.f), "f"(0.f), "f"(0.f));
}

__device__ __forceinline__ void trace_tc(const TcParams& p, int gw, int lane, int k) {
  if (p.trace && lane == 0 && gw < p.active_warps) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(int64_t)gw * 8 + k] = t;
  }
}

}  // namespace

// XM: the column sums X_c come from a second mma against an all-ones A
// (every row of D' is X_c) instead of a staged table -- the shared memory then
// holds x alone, which is what lets B = 8 at K = 14336 run as one launch.
template <int B, bool XM>
__global__ void __launch_bounds__(32 * kTcWarps, 1) gqsa_tc_kernel(const __grid_constant__ TcParams p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * kTcWarps + warp;
  const int g = lane >> 2, tq = lane & 3;
  trace_tc(p, gw, lane, 0);
  int t_begin = 0, t_end = 0;
  if (gw < p.active_warps) {
    t_begin = gw * p.part_q + min(gw, p.part_r);
    t_end = t_begin + p.part_q + (gw < p.part_r ? 1 : 0);
  }
  if (p.slice_k && t_end > t_begin) {  // data-centric: whole blocks whose first tile lies in the range
    const int bb = __ldg(p.tile_block + t_begin);
    const int b = __ldg(p.block_tile0 + bb) == t_begin ? t_begin : __ldg(p.block_tile0 + bb + 1);
    const int e = __ldg(p.block_tile0 + __ldg(p.tile_block + t_end - 1) + 1);
    t_begin = b;
    t_end = b < t_end ? e : b;
  }
  const uint64_t pol = evict_first_policy();
  TcTile buf[kTcBufs];
#pragma unroll
  for (int k = 0; k < kTcBufs; ++k)
    if (t_begin + k < t_end) tc_load(buf[k], p, t_begin + k, lane, pol);
  int blk = 0, bend = 0, bst = 0, bnext = 0;
  if (t_end > t_begin) blk = __ldg(p.tile_block + t_begin);
  pdl_launch_dependents();
  bool waited = !p.x_ready;
  if (waited) pdl_wait();
  if (t_end > t_begin) {
    bst = __ldg(p.block_tile0 + blk);
    bend = __ldg(p.block_tile0 + blk + 1);
    if (blk + 1 < p.nb) bnext = __ldg(p.block_tile0 + blk + 2);
  }

  // ---- stage x [B][K] (+ a zero chunk per row for padding items) and the
  //      column sums X[c][8] (fp32, t ascending; zero for c = K/16, b >= B)
  const int KG = p.cols / kGroup;
  uint8_t* xs = smem;
  float* xq = reinterpret_cast<float*>(smem + (size_t)B * p.xrow);
  constexpr int kSt = 4;  // column groups per thread in flight
  for (int i0 = threadIdx.x; i0 < B * KG; i0 += kSt * blockDim.x) {
    uint4 v[kSt][2];
#pragma unroll
    for (int j = 0; j < kSt; ++j) {
      const int i = i0 + j * blockDim.x;
      if (i < B * KG) {
        const int b = i / KG, c = i - b * KG;
        const uint4* src = reinterpret_cast<const uint4*>(p.X + (int64_t)b * p.ldx) + 2 * c;
        v[j][0] = __ldg(src);
        v[j][1] = __ldg(src + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < kSt; ++j) {
      const int i = i0 + j * blockDim.x;
      if (i < B * KG) {
        const int b = i / KG, c = i - b * KG;
        uint4* dst = reinterpret_cast<uint4*>(xs + (size_t)b * p.xrow) + 2 * c;
        dst[0] = v[j][0];
        dst[1] = v[j][1];
        if (XM) continue;
        const uint32_t w[8] = {v[j][0].x, v[j][0].y, v[j][0].z, v[j][0].w,
                               v[j][1].x, v[j][1].y, v[j][1].z, v[j][1].w};
        const uint32_t one = 0x3C003C00u;
        float ae = 0.f, ao = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          ae = fhfma<0, 0>(w[e], one, ae);
          ao = fhfma<1, 0>(w[e], one, ao);
        }
        xq[c * 8 + b] = ae + ao;
      }
    }
  }
  if (!XM)
    for (int i = threadIdx.x; i < (KG + 1) * 8; i += blockDim.x) {
      const int c = i >> 3, b = i & 7;
      if (c == KG || b >= B) xq[i] = 0.f;
    }
  for (int i = threadIdx.x; i < B * 2; i += blockDim.x)
    reinterpret_cast<uint4*>(xs + (size_t)(i >> 1) * p.xrow + 2 * p.cols)[i & 1] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  trace_tc(p, gw, lane, 2);
  auto ensure_wait = [&]() {
    if (!waited) {
      pdl_wait();
      waited = true;
    }
  };
  if (t_end <= t_begin) {
    ensure_wait();
    return;
  }
  bool foreign = bst < t_begin;
  int cw0 = foreign ? tc_warp_of_tile(p, bst) : gw;
  bool h_pending = false;
  int h_old = 0, h_w0 = 0, h_blk = 0;
  // CTA-level fix-up: the head block's partial waits in hacc for the reduction after the loop
  const bool cfix = p.cta_fix && !p.slice_k;
  bool h_defer = false;
  float hacc[kNV];
  float acc[kNV] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(xs);
  const uint32_t xq_s = (uint32_t)__cvta_generic_to_shared(xq);
  const uint32_t xrow_g = xs_s + (uint32_t)(g < B ? g : 0) * (uint32_t)p.xrow + 4u * tq;  // this lane's batch row
  trace_tc(p, gw, lane, 3);

  auto consume = [&](const TcTile& tr, int t) {
#pragma unroll
    for (int u = 0; u < kTcItems; ++u) {
      const uint32_t w = u == 0 ? tr.codes.x : u == 1 ? tr.codes.y : u == 2 ? tr.codes.z : tr.codes.w;
      const uint32_t a0 = lop3_and_or(w, 0x000F000Fu, kMagic1024);        // (row g,   k 2t, 2t+1)
      const uint32_t a1 = lop3_and_or(w >> 4, 0x000F000Fu, kMagic1024);   // (row g+8, k 2t, 2t+1)
      const uint32_t a2 = lop3_and_or(w >> 8, 0x000F000Fu, kMagic1024);   // (row g,   k 2t+8, 2t+9)
      const uint32_t a3 = lop3_and_or(w >> 12, 0x000F000Fu, kMagic1024);  // (row g+8, k 2t+8, 2t+9)
      const uint32_t cw = u < 2 ? tr.cols.x : tr.cols.y;
      const uint32_t c = (u & 1) ? (cw >> 16) : (cw & 0xffffu);
      uint32_t b0 = 0u, b1 = 0u;  // x[g][16c + 2t .. +1], x[g][16c + 2t + 8 .. +9]
      if (g < B) {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(b0) : "r"(xrow_g + c * 32u));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(b1) : "r"(xrow_g + c * 32u + 16u));
      }
      float d[4];
      mma16816(d, a0, a1, a2, a3, b0, b1);
      float2 X;  // column sums of batch 2t, 2t+1
      if (XM) {
        float dx[4];
        mma16816(dx, kOnes, kOnes, kOnes, kOnes, b0, b1);
        X = make_float2(dx[0], dx[1]);
      } else {
        X = lds64f(xq_s + c * 32u + 8u * tq);
      }
      const uint4& szv = u < 2 ? tr.sz0 : tr.sz1;
      const uint32_t slo = (u & 1) ? szv.z : szv.x, shi = (u & 1) ? szv.w : szv.y;
      const __half2 hlo = *reinterpret_cast<const __half2*>(&slo), hhi = *reinterpret_cast<const __half2*>(&shi);
      const float s_lo = __low2float(hlo), z_lo = __high2float(hlo) + 1024.f;
      const float s_hi = __low2float(hhi), z_hi = __high2float(hhi) + 1024.f;
      acc[0] = fmaf(s_lo, fmaf(-z_lo, X.x, d[0]), acc[0]);
      acc[1] = fmaf(s_lo, fmaf(-z_lo, X.y, d[1]), acc[1]);
      acc[2] = fmaf(s_hi, fmaf(-z_hi, X.x, d[2]), acc[2]);
      acc[3] = fmaf(s_hi, fmaf(-z_hi, X.y, d[3]), acc[3]);
    }
    if (t + 1 == bend) {  // the block ends with this tile
      ensure_wait();
      if (foreign && cfix) {
        h_defer = true;
        h_w0 = cw0;
        h_blk = blk;
#pragma unroll
        for (int k = 0; k < kNV; ++k) hacc[k] = acc[k];
      } else if (foreign) {
        tc_publish(p, gw, 0, acc, lane);
        __syncwarp();
        if (lane == 0) h_old = (int)atomicAdd(p.cnt + cw0, 1u);
        h_pending = true;
        h_w0 = cw0;
        h_blk = blk;
      } else {
        tc_store<B>(p, blk, acc, lane);
      }
#pragma unroll
      for (int k = 0; k < kNV; ++k) acc[k] = 0.f;
      foreign = false;
      cw0 = gw;
      if (t + 1 < t_end) {
        ++blk;
        bend = bnext;  // loaded one block ahead: no load latency on the next compare
        if (blk + 1 < p.nb) bnext = __ldg(p.block_tile0 + blk + 2);
      }
    }
  };

  int t = t_begin;
  while (t < t_end) {
#pragma unroll
    for (int k = 0; k < kTcBufs; ++k) {
      if (t < t_end) {
        consume(buf[k], t);
        if (t + kTcBufs < t_end) tc_load(buf[k], p, t + kTcBufs, lane, pol);
        ++t;
      }
    }
  }
  trace_tc(p, gw, lane, 4);
  ensure_wait();
  if (cfix) {
    // ---- CTA-level fix-up (as in the stream kernel): the
    //      pieces of a block inside the CTA belong to consecutive warps; the
    //      block's first warp here adds them from shared memory (the staging
    //      is dead once every loop is done); only blocks crossing a CTA
    //      boundary take the global protocol, one record per CTA.
    const int nw = min(kTcWarps, p.active_warps - (int)blockIdx.x * kTcWarps);
    asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
    float* P = reinterpret_cast<float*>(smem);  // [warps][2: head, tail][kNV][32]
    int* meta = reinterpret_cast<int*>(smem + (size_t)kTcWarps * 2 * kNV * kLanes * 4);
    const bool has_t = bend > t_end;
#pragma unroll
    for (int k = 0; k < kNV; ++k) {
      if (h_defer) P[((warp * 2 + 0) * kNV + k) * kLanes + lane] = hacc[k];
      if (has_t) P[((warp * 2 + 1) * kNV + k) * kLanes + lane] = acc[k];
    }
    if (lane == 0) meta[warp] = (h_defer ? 1 : 0) | (has_t && foreign ? 2 : 0);
    asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
    const int c = blockIdx.x;
    if (has_t && (!foreign || warp == 0)) {  // this warp starts the CTA's piece of its open block
      float v[kNV];
#pragma unroll
      for (int k = 0; k < kNV; ++k) v[k] = acc[k];
      bool closed = false;
#pragma unroll 1
      for (int w = warp + 1; w < nw && !closed; ++w) {
        closed = !(meta[w] & 2);  // warp w is not a middle participant: the block closes in its range
#pragma unroll
        for (int k = 0; k < kNV; ++k) v[k] += P[((w * 2 + (closed ? 0 : 1)) * kNV + k) * kLanes + lane];
      }
      if (closed && !foreign) tc_store<B>(p, blk, v, lane);
      else
        tc_cta_finish<B>(p, v, foreign ? cw0 / kTcWarps : c, c,
                         closed ? c : tc_warp_of_tile(p, bend - 1) / kTcWarps, blk, lane);
    }
    if (warp == 0 && h_defer) tc_cta_finish<B>(p, hacc, h_w0 / kTcWarps, c, c, h_blk, lane);
    trace_tc(p, gw, lane, 6);
    trace_tc(p, gw, lane, 5);
    return;
  }
  // Up to two collections (the block continuing downstream, the head block
  // that ended in this range), run through one call site of the collect code.
  int a_w0 = 0, a_w1 = 0, a_blk = 0, b_w0 = 0, b_w1 = 0, b_blk = 0, nc = 0;
  if (bend > t_end) {  // the block continues downstream
    const int w1 = tc_warp_of_tile(p, bend - 1);
    tc_publish(p, gw, foreign ? 0 : 1, acc, lane);
    const int old = tc_arrive(p, cw0, lane);
    trace_tc(p, gw, lane, 1);
    if (old == w1 - cw0) {
      a_w0 = cw0, a_w1 = w1, a_blk = blk;
      nc = 1;
    }
  }
  if (h_pending) {
    const int old = __shfl_sync(0xffffffffu, h_old, 0);
    if (old == gw - h_w0) {
      if (nc == 0) a_w0 = h_w0, a_w1 = gw, a_blk = h_blk;
      else b_w0 = h_w0, b_w1 = gw, b_blk = h_blk;
      ++nc;
    }
  }
#pragma unroll 1
  for (int i = 0; i < nc; ++i) tc_collect<B>(p, i ? b_w0 : a_w0, i ? b_w1 : a_w1, i ? b_blk : a_blk, lane);
  trace_tc(p, gw, lane, 6);
  trace_tc(p, gw, lane, 5);
}

template <int B>
const void* tc_ptr(bool xm) {
  return xm ? reinterpret_cast<const void*>(&gqsa_tc_kernel<B, true>)
            : reinterpret_cast<const void*>(&gqsa_tc_kernel<B, false>);
}

const void* select_tc_kernel(int B, bool xq_mma) {
  switch (B) {
    case 1: return tc_ptr<1>(xq_mma);
    case 2: return tc_ptr<2>(xq_mma);
    case 3: return tc_ptr<3>(xq_mma);
    case 4: return tc_ptr<4>(xq_mma);
    case 5: return tc_ptr<5>(xq_mma);
    case 6: return tc_ptr<6>(xq_mma);
    case 7: return tc_ptr<7>(xq_mma);
    case 8: return tc_ptr<8>(xq_mma);
    default: return nullptr;
  }
}

}  // namespace gqsa
