// gqsa_device.cuh -- device helpers of the Stream-K kernel (gqsa_stream.cu):
// PTX wrappers, streaming tile loads, LOP3/FHFMA dequant-dot, per-group
// accumulation (Eq. 3), activation staging.  See DESIGN.md §6.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gqsa_kernels.h"
#include "gqsa_layout.h"

namespace gqsa {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// fp32 += fp16 * fp16 with the exact product (FHFMA).  `a`/`b` are half2
// registers; HA/HB pick the half (folded into the SASS operand selector).
template <int HA, int HB>
__device__ __forceinline__ float fhfma(uint32_t a, uint32_t b, float c) {
  const unsigned short ah = HA ? (unsigned short)(a >> 16) : (unsigned short)(a & 0xffffu);
  const unsigned short bh = HB ? (unsigned short)(b >> 16) : (unsigned short)(b & 0xffffu);
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(ah), "h"(bh), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t magic) {
  uint32_t d;  // (a & mask) | magic
  asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(d) : "r"(a), "r"(mask), "r"(magic));
  return d;
}
constexpr uint32_t kMagic1024 = 0x64006400u;  // half2(1024, 1024)

// Weight tiles are read exactly once per call: streamed HBM -> registers,
// no L1 allocation, evict-first in L2 (they must not push the activations,
// column sums and outputs -- small, reused -- out of L2).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ldg_stream128(const void* ptr, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ uint2 ldg_stream64(const void* ptr, uint64_t pol) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_line_l2(const void* ptr) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64f(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

extern __shared__ __align__(128) uint8_t smem[];

// ---------------------------------------------------------------- dequant-dot
// Raw (offset-carrying) dot of one word of eight 4-bit codes with x[0..7]:
// de += sum_{j even} (1024 + e_j) x_j,  dd += sum_{j odd} (1024 + 16 e_j) x_j.
// Each LOP3 makes two exact fp16 values; each product is exact in fp32.
__device__ __forceinline__ void dot8_w4_raw(uint32_t w, uint32_t x01, uint32_t x23, uint32_t x45,
                                            uint32_t x67, float& de, float& dd) {
  const uint32_t w8 = w >> 8;
  const uint32_t e04 = lop3_and_or(w, 0x000F000Fu, kMagic1024);   // (1024+e0, 1024+e4)
  const uint32_t e15 = lop3_and_or(w, 0x00F000F0u, kMagic1024);   // (1024+16e1, 1024+16e5)
  const uint32_t e26 = lop3_and_or(w8, 0x000F000Fu, kMagic1024);  // (1024+e2, 1024+e6)
  const uint32_t e37 = lop3_and_or(w8, 0x00F000F0u, kMagic1024);  // (1024+16e3, 1024+16e7)
  de = fhfma<0, 0>(e04, x01, de);
  dd = fhfma<0, 1>(e15, x01, dd);
  de = fhfma<0, 0>(e26, x23, de);
  dd = fhfma<0, 1>(e37, x23, dd);
  de = fhfma<1, 0>(e04, x45, de);
  dd = fhfma<1, 1>(e15, x45, dd);
  de = fhfma<1, 0>(e26, x67, de);
  dd = fhfma<1, 1>(e37, x67, dd);
}

// Raw dot of one word of four 8-bit codes (element j in byte j) with
// x[0..3] = (x0, x1) (x2, x3): acc += sum_j (1024 + q_j) x_j, products exact.
__device__ __forceinline__ void dot4_w8_raw(uint32_t w, uint32_t x01, uint32_t x23, float& acc) {
  const uint32_t e02 = lop3_and_or(w, 0x00FF00FFu, kMagic1024);       // (1024+q0, 1024+q2)
  const uint32_t e13 = lop3_and_or(w >> 8, 0x00FF00FFu, kMagic1024);  // (1024+q1, 1024+q3)
  acc = fhfma<0, 0>(e02, x01, acc);
  acc = fhfma<0, 1>(e13, x01, acc);
  acc = fhfma<1, 0>(e02, x23, acc);
  acc = fhfma<1, 1>(e13, x23, acc);
}

// Raw dot of one word of sixteen 2-bit codes with x[0..15] (low 16-bit half
// <-> chunk xa, high half <-> xb): element e lands in set j = e mod 4 as the
// exact fp16 1024 + 4^j q_e (one LOP3 per pair), d[j] += sum (1024 + 4^j q_e) x_e.
__device__ __forceinline__ void dot16_w2_raw(uint32_t w, const uint4& xa, const uint4& xb, float& d0,
                                             float& d1, float& d2, float& d3) {
  const uint32_t w8 = w >> 8;
  const uint32_t r0 = lop3_and_or(w, 0x00030003u, kMagic1024);   // (e0, e8)   x1
  const uint32_t r1 = lop3_and_or(w, 0x000C000Cu, kMagic1024);   // (e1, e9)   x4
  const uint32_t r2 = lop3_and_or(w, 0x00300030u, kMagic1024);   // (e2, e10)  x16
  const uint32_t r3 = lop3_and_or(w, 0x00C000C0u, kMagic1024);   // (e3, e11)  x64
  const uint32_t q0 = lop3_and_or(w8, 0x00030003u, kMagic1024);  // (e4, e12)
  const uint32_t q1 = lop3_and_or(w8, 0x000C000Cu, kMagic1024);  // (e5, e13)
  const uint32_t q2 = lop3_and_or(w8, 0x00300030u, kMagic1024);  // (e6, e14)
  const uint32_t q3 = lop3_and_or(w8, 0x00C000C0u, kMagic1024);  // (e7, e15)
  d0 = fhfma<0, 0>(r0, xa.x, d0);
  d1 = fhfma<0, 1>(r1, xa.x, d1);
  d2 = fhfma<0, 0>(r2, xa.y, d2);
  d3 = fhfma<0, 1>(r3, xa.y, d3);
  d0 = fhfma<0, 0>(q0, xa.z, d0);
  d1 = fhfma<0, 1>(q1, xa.z, d1);
  d2 = fhfma<0, 0>(q2, xa.w, d2);
  d3 = fhfma<0, 1>(q3, xa.w, d3);
  d0 = fhfma<1, 0>(r0, xb.x, d0);
  d1 = fhfma<1, 1>(r1, xb.x, d1);
  d2 = fhfma<1, 0>(r2, xb.y, d2);
  d3 = fhfma<1, 1>(r3, xb.y, d3);
  d0 = fhfma<1, 0>(q0, xb.z, d0);
  d1 = fhfma<1, 1>(q1, xb.z, d1);
  d2 = fhfma<1, 0>(q2, xb.w, d2);
  d3 = fhfma<1, 1>(q3, xb.w, d3);
}

// Column-group sums of one group's activations w[0..G/2-1] = (x0,x1), (x2,x3), ..
// (t ascending within each sum), returned NEGATED as (-P, -Q): Q = sum_t x_t and
// P the offset the raw dot products carry -- W4: 1024 X_even + 64 X_odd;
// W8: 1024 Q; W2: 1024 X_0 + 256 X_1 + 64 X_2 + 16 X_3 (X_j = sum_{t = j mod 4} x_t).
template <int BITS, int G>
__device__ __forceinline__ float2 neg_column_sums(const uint32_t* w) {
  const uint32_t one = 0x3C003C00u;  // half2(1, 1): x * 1 is exact, one FHFMA per element
  if (BITS == 2) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a0 = fhfma<0, 0>(w[2 * i], one, a0);
      a1 = fhfma<1, 0>(w[2 * i], one, a1);
      a2 = fhfma<0, 0>(w[2 * i + 1], one, a2);
      a3 = fhfma<1, 0>(w[2 * i + 1], one, a3);
    }
    return make_float2(-fmaf(1024.f, a0, fmaf(256.f, a1, fmaf(64.f, a2, 16.f * a3))), -((a0 + a1) + (a2 + a3)));
  } else {
    float ae = 0.f, ao = 0.f;
#pragma unroll
    for (int e = 0; e < G / 2; ++e) {  // even t = 0, 2, .. and odd t = 1, 3, .., in order
      ae = fhfma<0, 0>(w[e], one, ae);
      ao = fhfma<1, 0>(w[e], one, ao);
    }
    const float q = ae + ao;
    return make_float2(BITS == 8 ? -1024.f * q : -fmaf(1024.f, ae, 64.f * ao), -q);
  }
}

// ---------------------------------------------------------------- tile regs
template <int BITS, int G>
struct TileRegs {
  uint4 codes[code_planes(BITS, G)];  // the lane's 4 slots
  uint4 sz;                           // 4 x (s, z) half pairs
  uint2 cols;                         // 4 x u16 column fields
};

template <int BITS, int G>
__device__ __forceinline__ void load_tile(TileRegs<BITS, G>& r, const uint8_t* tile, int lane, uint64_t pol) {
#pragma unroll
  for (int pl = 0; pl < code_planes(BITS, G); ++pl) r.codes[pl] = ldg_stream128(tile + pl * 512 + lane * 16, pol);
  r.sz = ldg_stream128(tile + off_sz(BITS, G) + lane * 16, pol);
  r.cols = ldg_stream64(tile + off_cols(BITS, G) + lane * 8, pol);
}

// Where a lane's staged activations live for the current item.
struct XView {
  uint32_t xs;     // shared address of x row 0
  uint32_t pq;     // shared address of (-P, -Q) row 0
  uint32_t xrow;   // bytes per x row
  uint32_t pqrow;  // bytes per (-P, -Q) row
};

// acc[b] += s * sum_t (q_t - z) x[b][c*G + t] for the lane's group in slot u
// (Eq. 3 applied per group, z folded once through the column sums): the raw
// dot starts from -P - z Q, so the offsets of the LOP3 magic and z leave in
// one FFMA, and one more FFMA applies s.
template <int BITS, int B, int G>
__device__ __forceinline__ void group_accumulate(const TileRegs<BITS, G>& tr, int u, float (&acc)[B],
                                                 const XView& xv) {
  const uint32_t colw = (u < 2) ? tr.cols.x : tr.cols.y;
  const uint32_t f0 = (u & 1) ? (colw >> 16) : (colw & 0xffffu);  // byte offset of the first x chunk
  // (-P, -Q) entry: G = 16, B <= 2: per chunk index f (f * 8 = f0 / 2); else
  // per column group c (c * 8 = f0 / 4 at G = 16, f0 / 2 at G = 8, f0 / 8 at G = 32)
  constexpr bool kPerChunk = pq_per_chunk(B, G);  // see pq_entries()
  const uint32_t pqoff = G == 8 ? f0 >> 1 : G == 32 ? (f0 >> 3) & ~7u : kPerChunk ? f0 >> 1 : (f0 >> 2) & ~7u;
  const uint32_t szw = u == 0 ? tr.sz.x : u == 1 ? tr.sz.y : u == 2 ? tr.sz.z : tr.sz.w;
  const __half2 sz = *reinterpret_cast<const __half2*>(&szw);
  const float s = __low2float(sz), z = __high2float(sz);
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint32_t xrow = xv.xs + b * xv.xrow;
    const float2 X = lds64f(xv.pq + b * xv.pqrow + pqoff);
    const float u0 = fmaf(z, X.y, X.x);  // -P - z Q
    if (BITS == 4 && G == 8) {
      const uint4 xa = lds128(xrow + f0);
      float de = u0, dd = 0.f;
      const uint32_t w = u == 0 ? tr.codes[0].x : u == 1 ? tr.codes[0].y : u == 2 ? tr.codes[0].z : tr.codes[0].w;
      dot8_w4_raw(w, xa.x, xa.y, xa.z, xa.w, de, dd);
      acc[b] = fmaf(s, fmaf(dd, 0.0625f, de), acc[b]);
    } else if (BITS == 4 && G == 32) {  // four chunks from the lane's rotation: (f0 + 16k) mod 64 in the group
      const uint4 c = tr.codes[u];
      const uint32_t gb = xrow + (f0 & ~63u);
      const uint4 x0 = lds128(gb + (f0 & 63u)), x1 = lds128(gb + ((f0 + 16u) & 63u));
      const uint4 x2 = lds128(gb + ((f0 + 32u) & 63u)), x3 = lds128(gb + ((f0 + 48u) & 63u));
      float de = u0, dd = 0.f;
      dot8_w4_raw(c.x, x0.x, x0.y, x0.z, x0.w, de, dd);
      dot8_w4_raw(c.y, x1.x, x1.y, x1.z, x1.w, de, dd);
      dot8_w4_raw(c.z, x2.x, x2.y, x2.z, x2.w, de, dd);
      dot8_w4_raw(c.w, x3.x, x3.y, x3.z, x3.w, de, dd);
      acc[b] = fmaf(s, fmaf(dd, 0.0625f, de), acc[b]);
    } else {
      const uint4 xa = lds128(xrow + f0);
      const uint4 xb = lds128((xrow + f0) ^ 16u);  // x rows are 32-B aligned at G = 16
      if (BITS == 8) {  // every element carries +1024: sum (q - z) x = sum (1024 + q) x - 1024 Q - z Q
        const uint4 c = tr.codes[u];
        float d0 = u0, d1 = 0.f;
        dot4_w8_raw(c.x, xa.x, xa.y, d0);  // elements 0..3 <-> first x chunk
        dot4_w8_raw(c.y, xa.z, xa.w, d1);  // 4..7
        dot4_w8_raw(c.z, xb.x, xb.y, d0);  // 8..11 <-> second x chunk
        dot4_w8_raw(c.w, xb.z, xb.w, d1);  // 12..15
        acc[b] = fmaf(s, d0 + d1, acc[b]);
      } else if (BITS == 4) {
        // sum (q - z) x = D_even + D_odd / 16 - (1024 X_even + 64 X_odd) - z Q
        const uint4& c = tr.codes[u >> 1];
        const uint32_t w0 = (u & 1) ? c.z : c.x, w1 = (u & 1) ? c.w : c.y;
        float de = u0, dd = 0.f;
        dot8_w4_raw(w0, xa.x, xa.y, xa.z, xa.w, de, dd);  // word 0 <-> first x chunk
        dot8_w4_raw(w1, xb.x, xb.y, xb.z, xb.w, de, dd);  // word 1 <-> second x chunk
        acc[b] = fmaf(s, fmaf(dd, 0.0625f, de), acc[b]);
      } else {
        // W2: sum (q - z) x = D0 + D1/4 + D2/16 + D3/64 - (1024 X0 + 256 X1 + 64 X2 + 16 X3) - z Q
        const uint32_t w = u == 0 ? tr.codes[0].x : u == 1 ? tr.codes[0].y : u == 2 ? tr.codes[0].z : tr.codes[0].w;
        float d0 = u0, d1 = 0.f, d2 = 0.f, d3 = 0.f;
        dot16_w2_raw(w, xa, xb, d0, d1, d2, d3);
        const float dsum = fmaf(d3, 0.015625f, fmaf(d2, 0.0625f, fmaf(d1, 0.25f, d0)));
        acc[b] = fmaf(s, dsum, acc[b]);
      }
    }
  }
}

// Stage the activations of every item a CTA's tile range [t0, t1) touches,
// in one round of loads for the common sizes: the column groups of all
// touched items form one index space (a small table of the touched items is
// built in shared memory first, so the lookups stay on chip), each thread
// loads U of them (all loads in flight together), then writes x rows (of
// xrow bytes, followed by a zero block) and the negated column-group sums
// (-P, -Q) (fp32, fixed t order) computed from the same registers, plus zero
// entries for padding.  Items are packed in item order from shared offset 0
// (mirrors the host's plan).  `tab` is kStageTabBytes of shared memory after
// the staging area (kMaxItems entries, then the count and total).  Caller
// synchronises.
__device__ __forceinline__ bool item_touched(const Item& it, int t0, int t1) {
  return it.tile_begin < t1 && it.tile_end > t0 && it.tile_end > it.tile_begin;
}
struct StageEntry {
  const uint16_t* X;
  int64_t ldx;
  int32_t first;   // first global column-group index of this item
  int32_t kg;      // column groups per batch row
  int32_t cols, xrow, pqrow;
  uint32_t off;    // shared offset of the item's x rows
};
constexpr int kStageTabBytes = kMaxItems * (int)sizeof(StageEntry) + 16;
static_assert(sizeof(StageEntry) == 40, "gqsa_capi.cu kStageTab");
// The staging table (thread 0; parameters only, so it may run before the PDL wait).
template <int B, int G>
__device__ __forceinline__ void stage_table(const Params& p, int t0, int t1, StageEntry* tab) {
  if (threadIdx.x == 0) {
    int first = 0, n = 0;
    uint32_t off = 0;
    for (int i = 0; i < p.n_items; ++i) {
      const Item& it = p.item[i];
      if (!item_touched(it, t0, t1)) continue;
      tab[n] = StageEntry{it.X, it.ldx, first, it.cols / G, it.cols, it.xrow, it.pqrow, off};
      first += B * (it.cols / G);
      off += (uint32_t)it.smem_bytes;
      ++n;
    }
    reinterpret_cast<volatile int*>(tab + kMaxItems)[0] = n;
    reinterpret_cast<volatile int*>(tab + kMaxItems)[1] = first;
  }
}
// Loads and sums (all threads; after stage_table and, unless x_ready, the PDL wait).
template <int BITS, int B, int G>
__device__ __forceinline__ void stage_all(const Params& p, uint8_t* sm, StageEntry* tab) {
  constexpr int NC = G / 8;            // 16-B chunks per column group
#ifndef GQSA_STAGE_U
#define GQSA_STAGE_U 4
#endif
  constexpr int U = NC >= 4 ? 2 : GQSA_STAGE_U;  // column groups per thread in flight per round
  constexpr int PG = pq_per_chunk(B, G) ? 2 : 1;  // (-P, -Q) entries per column group (one per chunk order)
  const int nthreads = blockDim.x;
  __syncthreads();  // the table
  const int n_t = reinterpret_cast<const int*>(tab + kMaxItems)[0];
  const int total = reinterpret_cast<const int*>(tab + kMaxItems)[1];
  auto locate = [&](int gi) {  // entry of global column-group index gi
    int k = 0;
    while (k + 1 < n_t && gi >= tab[k + 1].first) ++k;
    return k;
  };
  for (int base = threadIdx.x; base < total; base += U * nthreads) {
    uint4 v[U][NC];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int gi = base + k * nthreads;
      if (gi < total) {
        const StageEntry& e = tab[locate(gi)];
        const int l = gi - e.first, b = B == 1 ? 0 : l / e.kg, c = l - b * e.kg;
        const uint4* src = reinterpret_cast<const uint4*>(e.X + (int64_t)b * e.ldx) + NC * c;
#pragma unroll
        for (int h = 0; h < NC; ++h) v[k][h] = __ldg(src + h);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int gi = base + k * nthreads;
      if (gi < total) {
        const StageEntry& e = tab[locate(gi)];
        const int l = gi - e.first, b = B == 1 ? 0 : l / e.kg, c = l - b * e.kg;
        uint8_t* xs = sm + e.off;
        uint4* dst = reinterpret_cast<uint4*>(xs + (size_t)b * e.xrow) + NC * c;
        uint32_t w[4 * NC];
#pragma unroll
        for (int h = 0; h < NC; ++h) {
          dst[h] = v[k][h];
          w[4 * h] = v[k][h].x;
          w[4 * h + 1] = v[k][h].y;
          w[4 * h + 2] = v[k][h].z;
          w[4 * h + 3] = v[k][h].w;
        }
        const float2 v2 = neg_column_sums<BITS, G>(w);
        float2* pdst = reinterpret_cast<float2*>(xs + (size_t)B * e.xrow + (size_t)b * e.pqrow) + (size_t)c * PG;
        pdst[0] = v2;
        if (PG == 2) pdst[1] = v2;
      }
    }
  }
  // zero block after each x row and the padding entries of the column-sum tables
  for (int k = 0; k < n_t; ++k) {
    const StageEntry& e = tab[k];
    uint8_t* xs = sm + e.off;
    for (int j = threadIdx.x; j < B * (kXPadBytes / 16); j += nthreads) {
      const int b = j / (kXPadBytes / 16), q = j % (kXPadBytes / 16);
      reinterpret_cast<uint4*>(xs + (size_t)b * e.xrow + 2 * e.cols)[q] = make_uint4(0, 0, 0, 0);
    }
    const int ne = pq_entries(B, G, e.cols);
    for (int j = threadIdx.x; j < B * 2; j += nthreads)
      reinterpret_cast<float2*>(xs + (size_t)B * e.xrow + (size_t)(j >> 1) * e.pqrow)[ne + (j & 1)] =
          make_float2(0.f, 0.f);
  }
}

}  // namespace gqsa
