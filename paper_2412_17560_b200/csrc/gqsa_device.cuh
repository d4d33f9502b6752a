// gqsa_device.cuh -- device helpers shared by the per-GEMV Stream-K kernel
// (gqsa_gemv.cu) and the persistent chain kernel (gqsa_chain.cu): PTX
// wrappers, LOP3/FHFMA dequant-dot, per-group accumulation (Eq. 3), the
// cross-warp fix-up records and the activation staging.  See DESIGN.md §6.
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
// registers; H0/H1 pick the half (folded into the SASS operand selector).
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
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

constexpr uint32_t kMagic1024 = 0x64006400u;   // half2(1024, 1024)
constexpr uint32_t kNeg1024 = 0xE400E400u;     // half2(-1024, -1024)

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

// Raw (offset-carrying) dot of one word of sixteen 2-bit codes with x[0..15]
// (low 16-bit half <-> x chunk xa, high half <-> xb): element e lands in set
// j = e mod 4 as the exact fp16 1024 + 4^j q_e (one LOP3 per pair, no
// HADD2/HFMA2), and d[j] += sum_{e in set j} (1024 + 4^j q_e) x_e with exact
// products.  The offsets are removed once per group with the set sums.
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

// Column-group sums of one group's 16 activations w[0..7] = (x0,x1) .. (x14,x15)
// (t ascending within each sum): (P, Q) with Q = sum_t x_t and P the offset
// the raw dot products carry: W4 / W8 P = 1024 X_even + 64 X_odd (W8 uses
// only Q and the plain 1024 X = 1024 Q - ... see group_accumulate), W2
// P = 1024 X_0 + 256 X_1 + 64 X_2 + 16 X_3 with X_j = sum_{t = j mod 4} x_t.
template <int BITS, int G = kGroup>
__device__ __forceinline__ float2 column_sums(const uint32_t* w) {
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
    return make_float2(fmaf(1024.f, a0, fmaf(256.f, a1, fmaf(64.f, a2, 16.f * a3))), (a0 + a1) + (a2 + a3));
  } else {
    float ae = 0.f, ao = 0.f;
#pragma unroll
    for (int e = 0; e < G / 2; ++e) {  // even t = 0, 2, .. and odd t = 1, 3, .., in order
      ae = fhfma<0, 0>(w[e], one, ae);
      ao = fhfma<1, 0>(w[e], one, ao);
    }
    return make_float2(fmaf(1024.f, ae, 64.f * ao), ae + ao);
  }
}

// ---------------------------------------------------------------- tile regs
// 16-B code planes per lane per tile: 4 slots x G*n/8 bytes (W2: 1, W4: 2,
// W8: 4 at G = 16; W4: 1 at G = 8, 4 at G = 32).
template <int BITS, int G = kGroup>
constexpr int code_planes() { return G * BITS / 32; }

template <int BITS, int G = kGroup>
struct TileRegs {
  uint4 codes[code_planes<BITS, G>()];  // the lane's 4 slots
  uint4 sz;                        // 4 x (s, z) half pairs
  uint2 cols;                      // 4 x u16 (2c + swap)
  uint32_t hdr;                    // slice << 2 | FIRST | LAST
  uint32_t rem;                    // tiles from this one to its slice's last tile
};


// Group code word(s) of slot u from the lane's codes.
template <int BITS, int G = kGroup>
__device__ __forceinline__ uint2 group_words(const TileRegs<BITS, G>& r, int u) {
  if (G == 8 || G == 32) {  // W4: G = 8 one word per slot; G = 32 reads the whole plane (codes[u])
    const uint4& c = r.codes[0];
    return G == 8 ? make_uint2(u == 0 ? c.x : u == 1 ? c.y : u == 2 ? c.z : c.w, 0u) : make_uint2(0u, 0u);
  } else if (BITS == 8) {
    return make_uint2(0u, 0u);  // W8 reads the whole 16-B slot (tr.codes[u])
  } else if (BITS == 4) {
    const uint4& c = r.codes[u >> 1];
    return (u & 1) ? make_uint2(c.z, c.w) : make_uint2(c.x, c.y);
  } else {
    const uint4& c = r.codes[0];
    const uint32_t w = u == 0 ? c.x : u == 1 ? c.y : u == 2 ? c.z : c.w;
    return make_uint2(w, 0u);
  }
}

// acc[b] += s * sum_t (q_t - z) x_t for the lane's group in slot u (Eq. 3
// per group, z applied once through the column-group sums).
//   xs : activations [B][K] fp16 in shared memory
//   pq : float2 (P, Q) per column group c (B >= 3) or per 16-B chunk index
//        f = 2c + swap (B <= 2: duplicated, saves one instruction per group), with
//        P = 1024 X_even + 64 X_odd and Q = X_even + X_odd of column group c
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64f(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

extern __shared__ __align__(128) uint8_t smem[];

// Column-sum table entries per column group: 2 (indexed by f = 2c + swap) at
// batch <= 2, else 1 (indexed by c; halves the table so that larger batches
// keep x resident in shared memory).
template <int B, int G = kGroup>
constexpr int pq_per_group() { return (G == kGroup && B <= 2) ? 2 : 1; }

template <int BITS, int B, int G = kGroup>
__device__ __forceinline__ void group_accumulate(const KParams& p, const TileRegs<BITS, G>& tr, int u,
                                                 float (&acc)[kMaxBatch]) {
  // shared-window offsets recomputed here so that they stay in uniform
  // registers ([R + UR] addressing on every LDS)
  const uint32_t xs = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t pq = xs + (uint32_t)B * 2u * (uint32_t)p.cols;
  const uint32_t pq_row = (uint32_t)p.cols / G * pq_per_group<B, G>() * 8u;  // bytes per batch row
  const uint32_t colw = (u < 2) ? tr.cols.x : tr.cols.y;
  const uint32_t xoff0 = (u & 1) ? (colw >> 16) : (colw & 0xffffu);  // byte offset of the first x chunk
  const uint32_t xoff1 = xoff0 ^ 16u;                                  // the other chunk (G = 16)
  // (P, Q) entry: G = 16, B <= 2: per chunk index f (f * 8 = xoff0 / 2); else
  // per column group c (c * 8 = xoff0 / 4 at G = 16, xoff0 / 2 at G = 8, xoff0 / 8 at G = 32)
  const uint32_t pqoff = G == 8 ? xoff0 >> 1
                         : G == 32 ? (xoff0 >> 3) & ~7u
                                   : (pq_per_group<B, G>() == 2 ? xoff0 >> 1 : (xoff0 >> 2) & ~7u);
  const uint2 w = group_words<BITS, G>(tr, u);
  const uint32_t szw = u == 0 ? tr.sz.x : u == 1 ? tr.sz.y : u == 2 ? tr.sz.z : tr.sz.w;
  const __half2 sz = *reinterpret_cast<const __half2*>(&szw);
  const float s = __low2float(sz), z = __high2float(sz);
#pragma unroll
  for (int b = 0; b < B; ++b) {
    // x of batch row b at shared offset b * 2K (x is at the start of smem)
    const uint32_t xrow = xs + b * 2u * (uint32_t)p.cols;
    const float2 X = lds64f(pq + b * pq_row + pqoff);
    if (G == 8) {  // W4, one chunk: sum_t (q_t - z) x_t = D_even + D_odd/16 - P - z Q
      const uint4 xa = lds128(xrow + xoff0);
      float de = 0.f, dd = 0.f;
      dot8_w4_raw(w.x, xa.x, xa.y, xa.z, xa.w, de, dd);
      acc[b] = fmaf(s, fmaf(-z, X.y, fmaf(dd, 0.0625f, de) - X.x), acc[b]);
      continue;
    }
    if (G == 32) {  // W4, four chunks from the lane's rotation: (xoff0 + 16k) mod 64 within the group
      const uint4 c = tr.codes[u];
      const uint32_t gb = xrow + (xoff0 & ~63u);
      const uint4 x0 = lds128(gb + (xoff0 & 63u)), x1 = lds128(gb + ((xoff0 + 16u) & 63u));
      const uint4 x2 = lds128(gb + ((xoff0 + 32u) & 63u)), x3 = lds128(gb + ((xoff0 + 48u) & 63u));
      float de = 0.f, dd = 0.f;
      dot8_w4_raw(c.x, x0.x, x0.y, x0.z, x0.w, de, dd);
      dot8_w4_raw(c.y, x1.x, x1.y, x1.z, x1.w, de, dd);
      dot8_w4_raw(c.z, x2.x, x2.y, x2.z, x2.w, de, dd);
      dot8_w4_raw(c.w, x3.x, x3.y, x3.z, x3.w, de, dd);
      acc[b] = fmaf(s, fmaf(-z, X.y, fmaf(dd, 0.0625f, de) - X.x), acc[b]);
      continue;
    }
    const uint4 xa = lds128(xrow + xoff0);
    const uint4 xb = lds128(xrow + xoff1);
    if (BITS == 8) {
      // Every element carries the +1024 offset of the LOP3 magic:
      //   sum_t (q_t - z) x_t = sum_t (1024 + q_t) x_t - (1024 + z) X.
      const uint4 c = tr.codes[u];
      float d0 = 0.f, d1 = 0.f;
      dot4_w8_raw(c.x, xa.x, xa.y, d0);  // elements 0..3 <-> first x chunk
      dot4_w8_raw(c.y, xa.z, xa.w, d1);  // 4..7
      dot4_w8_raw(c.z, xb.x, xb.y, d0);  // 8..11 <-> second x chunk
      dot4_w8_raw(c.w, xb.z, xb.w, d1);  // 12..15
      const float t = fmaf(-z, X.y, fmaf(-1024.f, X.y, d0 + d1));
      acc[b] = fmaf(s, t, acc[b]);
    } else if (BITS == 4) {
      // Offset-folded dequantization: the LOP3 magic leaves
      // 1024 + q (even elements) and 1024 + 16 q (odd elements) as exact fp16;
      // their products with x are exact in fp32, and the offsets are removed
      // once per group with the column sums: sum_t (q_t - z) x_t =
      //   D_even + D_odd/16 - (1024 X_even + 64 X_odd) - z (X_even + X_odd).
      float de = 0.f, dd = 0.f;
      dot8_w4_raw(w.x, xa.x, xa.y, xa.z, xa.w, de, dd);  // word 0 <-> first x chunk
      dot8_w4_raw(w.y, xb.x, xb.y, xb.z, xb.w, de, dd);  // word 1 <-> second x chunk
      const float t = fmaf(-z, X.y, fmaf(dd, 0.0625f, de) - X.x);
      acc[b] = fmaf(s, t, acc[b]);
    } else {
      // Offset-folded W2 (as W4): sum_t (q_t - z) x_t =
      //   D0 + D1/4 + D2/16 + D3/64 - (1024 X_0 + 256 X_1 + 64 X_2 + 16 X_3) - z X
      float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
      dot16_w2_raw(w.x, xa, xb, d0, d1, d2, d3);
      const float dsum = fmaf(d3, 0.015625f, fmaf(d2, 0.0625f, fmaf(d1, 0.25f, d0)));
      const float t = fmaf(-z, X.y, dsum - X.x);
      acc[b] = fmaf(s, t, acc[b]);
    }
  }
}

// ---------------------------------------------------------------- fix-up
// Record of warp w: [B][32 lanes] 8-byte slots {partial, flag}; each slot is
// written with ONE 64-bit store, so a reader that sees the flag sees the
// value (single-copy atomicity): no fence needed.
template <int B>
__device__ __forceinline__ unsigned long long* ws_slot(const KParams& p, int w, int b, int lane) {
  return reinterpret_cast<unsigned long long*>(p.ws) + ((int64_t)w * B + b) * kLanes + lane;
}

// Intra-CTA records live in shared memory: [W][B][32 lanes] 8-B slots at
// `fx` (zeroed in the prologue), indexed by the warp's index in its CTA.
__device__ __forceinline__ uint32_t fx_slot(uint32_t fx, int wl, int B, int b, int lane) {
  return fx + (uint32_t)(((wl * B + b) * kLanes + lane) * 8);
}

// local: the owner of the slice is a warp of this CTA (shared-memory record)
template <int B>
__device__ __forceinline__ void publish(const KParams& p, int gw, const float (&v)[kMaxBatch], int lane,
                                        bool local, uint32_t fx, int wl) {
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const unsigned long long w = (1ull << 32) | __float_as_uint(v[b]);
    if (local)
      asm volatile("st.volatile.shared.b64 [%0], %1;" ::"r"(fx_slot(fx, wl, B, b, lane)), "l"(w) : "memory");
    else
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(ws_slot<B>(p, gw, b, lane)), "l"(w) : "memory");
  }
}

// Add the partials of warps gw+1 .. w_last (in warp order) and reset them.
__device__ __forceinline__ unsigned long long ld_slot(const unsigned long long* slot) {
  unsigned long long s;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(s) : "l"(slot) : "memory");
  return s;
}

constexpr int kPre = 2;  // successor records an owner requests before its last tile

template <int B>
__device__ __forceinline__ void collect(const KParams& p, int gw, int w_last, float (&v)[kMaxBatch],
                                        int lane, unsigned long long (&pre)[kPre][kMaxBatch], int wg0,
                                        uint32_t fx, int cta_w0) {
  // successors in this CTA (warps gw+1 .. wg0-1): shared-memory records
  for (int w = gw + 1; w < wg0; ++w) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint32_t a = fx_slot(fx, w - cta_w0, B, b, lane);
      unsigned long long s;
      do {
        asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(s) : "r"(a) : "memory");
      } while ((s >> 32) == 0ull);
      v[b] += __uint_as_float((uint32_t)s);
    }
  }
  gw = wg0 - 1;  // the remaining successors (other CTAs) use global records
  // records requested early (during the owner's last tile): usually ready
#pragma unroll
  for (int k = 0; k < kPre; ++k) {
    const int w = gw + 1 + k;
    if (w > w_last) break;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      unsigned long long* slot = ws_slot<B>(p, w, b, lane);
      unsigned long long s = pre[k][b];
      int spins = 0;
      while ((s >> 32) == 0ull) {
        if (++spins > 2) __nanosleep(64);
        s = ld_slot(slot);
      }
      v[b] += __uint_as_float((uint32_t)s);
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(slot), "l"(0ull) : "memory");
    }
  }
  constexpr int kBatch = 8;  // further records polled per round trip
  for (int w0 = gw + 1 + kPre; w0 <= w_last; w0 += kBatch) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      unsigned long long s[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k)  // independent loads: one L2 round trip
        s[k] = (w0 + k <= w_last) ? ld_slot(ws_slot<B>(p, w0 + k, b, lane)) : (1ull << 32);
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {  // add in warp order (deterministic)
        if (w0 + k > w_last) break;
        unsigned long long* slot = ws_slot<B>(p, w0 + k, b, lane);
        int spins = 0;
        while ((s[k] >> 32) == 0ull) {
          if (++spins > 2) __nanosleep(64);
          s[k] = ld_slot(slot);
        }
        v[b] += __uint_as_float((uint32_t)s[k]);
        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(slot), "l"(0ull) : "memory");
      }
    }
  }
}

// y element i: fp32, or fp16 rounded to nearest even (PAPER.md:134 step 5).
__device__ __forceinline__ void store_y(const KParams& p, int64_t i, float v) {
  if (p.n_peers) {  // fused all-gather: this shard's rows land in every rank's full y
#pragma unroll 1
    for (int k = 0; k < p.n_peers; ++k) {
      if (p.out_f16) reinterpret_cast<__half*>(p.peer_y[k])[i + p.row_offset] = __float2half_rn(v);
      else reinterpret_cast<float*>(p.peer_y[k])[i + p.row_offset] = v;
    }
    return;
  }
  if (p.out_f16) reinterpret_cast<__half*>(p.Y)[i] = __float2half_rn(v);
  else reinterpret_cast<float*>(p.Y)[i] = v;
}

// Sum over the S lanes of a row (S = lanes per row, a power of two) and store.
template <int B>
__device__ __forceinline__ void store_rows(const KParams& p, float (&v)[kMaxBatch], int row, int lane) {
  for (int d = 1; d < p.lanes_per_row; d <<= 1) {
#pragma unroll
    for (int b = 0; b < B; ++b) v[b] += __shfl_xor_sync(0xffffffffu, v[b], d);
  }
  if (row >= 0 && (lane & (p.lanes_per_row - 1)) == 0) {
    const float bias = p.bias ? __ldg(p.bias + row) : 0.f;
#pragma unroll
    for (int b = 0; b < B; ++b) store_y(p, (int64_t)b * p.ldy + row, v[b] + bias);
  }
}

// Warp that owns tile t under the +-1 partition of num_tiles over active_warps.
__device__ __forceinline__ int warp_of_tile(const KParams& p, int t) {
  const int big = p.part_r * (p.part_q + 1);
  return t < big ? t / (p.part_q + 1) : p.part_r + (t - big) / p.part_q;
}

// ---------------------------------------------------------------- kernel
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Weight tiles are read exactly once per call: stream them with an
// evict-first L2 policy so they do not push activations, column sums and
// outputs (reused, small) out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

// Optional timeline instrumentation (gqsa_debug_trace): lane 0 of each warp
// stamps %globaltimer at fixed points; off (one predicated branch) by default.
__device__ __forceinline__ void trace_point(const KParams& p, int gw, int lane, int k) {
  if (p.trace && lane == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(int64_t)gw * 8 + k] = t;
  }
}

// One lane's view of a tile that has landed in shared memory.
template <int BITS, int G = kGroup>
__device__ __forceinline__ void read_tile(TileRegs<BITS, G>& r, const uint8_t* tile, int lane) {
#pragma unroll
  for (int pl = 0; pl < code_planes<BITS, G>(); ++pl)
    r.codes[pl] = *reinterpret_cast<const uint4*>(tile + kTileHeaderBytes + pl * 512 + lane * 16);
  r.sz = *reinterpret_cast<const uint4*>(tile + off_sz(BITS, G) + lane * 16);
  r.cols = *reinterpret_cast<const uint2*>(tile + off_cols(BITS, G) + lane * 8);
  const uint2 h = *reinterpret_cast<const uint2*>(tile);  // broadcast
  r.hdr = h.x;
  r.rem = h.y;
}


// Stage x (B rows of `cols` fp16, row stride ldx) into shared memory at xs
// and compute the per-column-group sums (P, Q) into pq, with plain 128-bit
// loads (two column groups per thread in flight).  Caller synchronises.
// COHERENT: x may have been written earlier in the SAME launch (chain
// kernel), so it is read through L2 only (ld.global.cg), never through the
// non-coherent L1/texture path.
template <int BITS, int B, bool COHERENT = false, int G = kGroup>
__device__ __forceinline__ void stage_activations(const KParams& p, uint8_t* xs, uint8_t* pq, int KG,
                                                  int nthreads) {
  constexpr int NC = G / 8;  // 16-B chunks per column group
  constexpr int U = NC >= 4 ? 1 : 2;  // column groups per thread per round in flight
  for (int i0 = threadIdx.x; i0 < B * KG; i0 += U * nthreads) {
    uint4 v[U][NC];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = i0 + k * nthreads;
      if (i < B * KG) {
        const int b = i / KG, c = i - b * KG;
        const uint4* src = reinterpret_cast<const uint4*>(p.X + (int64_t)b * p.ldx) + NC * c;
#pragma unroll
        for (int h = 0; h < NC; ++h) v[k][h] = COHERENT ? __ldcg(src + h) : __ldg(src + h);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int i = i0 + k * nthreads;
      if (i < B * KG) {
        const int b = i / KG, c = i - b * KG;
        uint4* dst = reinterpret_cast<uint4*>(xs + (size_t)b * p.cols * 2) + NC * c;
        uint32_t w[4 * NC];
#pragma unroll
        for (int h = 0; h < NC; ++h) {
          dst[h] = v[k][h];
          w[4 * h] = v[k][h].x;
          w[4 * h + 1] = v[k][h].y;
          w[4 * h + 2] = v[k][h].z;
          w[4 * h + 3] = v[k][h].w;
        }
        // (P, Q) of column group c, stored for both chunk orders (swap = 0, 1) at G = 16, B <= 2
        const float2 v2 = column_sums<BITS, G>(w);
        constexpr int PG = pq_per_group<B, G>();
        float2* pdst = reinterpret_cast<float2*>(pq) + ((size_t)b * KG + c) * PG;
        pdst[0] = v2;
        if (PG == 2) pdst[1] = v2;
      }
    }
  }
}

}  // namespace gqsa
