// quant_dev.cuh -- the per-block NVFP4 stage of ARC quantization (oracle STAGE,
// DESIGN.md Q7 op order) shared by the standalone quantization kernel (quant.cu)
// and the fused decode linear's producer phase (decode.cu): FMUL2 products,
// cvt.rn.satfinite.e2m1x2 encoding, the exact residual e = t - v(q1),
// the ceil-rounded E4M3 block scale (Q2) and the physical block map (App.D).
#pragma once
#include "arc_device.cuh"

#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace arc {

// Two fp32 products z*k with one FMUL2 (mul.rn.f32x2: two IEEE RN multiplies).
ARC_DEV float2 mul2(float a, float b, float k) {
  unsigned long long x, y, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a), "f"(b));
  asm("mov.b64 %0, {%1, %1};" : "=l"(y) : "f"(k));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}

// One NVFP4 stage on 16 values (oracle C4) given the block's multiplier k:
// t = z*k (mul.rn.f32x2), q = rne_e2m1(t) (cvt.rn.satfinite.e2m1x2), packed with
// element 2i in the low nibble of byte i (bytes assembled by the PTX byte-vector mov).
ARC_DEV uint2 encode16(const float (&z)[16], float k) {
  float t[16];
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const float2 p = mul2(z[i], z[i + 1], k);
    t[i] = p.x;
    t[i + 1] = p.y;
  }
  uint32_t w0, w1;
  asm("{\n\t.reg .b8 b<8>;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %3, %2;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %5, %4;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %7, %6;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %9, %8;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b4, %11, %10;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b5, %13, %12;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b6, %15, %14;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b7, %17, %16;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t"
      "mov.b32 %1, {b4, b5, b6, b7};\n\t}"
      : "=r"(w0), "=r"(w1)
      : "f"(t[0]), "f"(t[1]), "f"(t[2]), "f"(t[3]), "f"(t[4]), "f"(t[5]), "f"(t[6]), "f"(t[7]), "f"(t[8]),
        "f"(t[9]), "f"(t[10]), "f"(t[11]), "f"(t[12]), "f"(t[13]), "f"(t[14]), "f"(t[15]));
#if ARC_E2M1_SIGN_FIXUP
  uint32_t s0 = 0, s1 = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s0 |= (__float_as_uint(t[i]) >> 31) << (4 * i + 3);
    s1 |= (__float_as_uint(t[i + 8]) >> 31) << (4 * i + 3);
  }
  w0 = (w0 & 0x77777777u) | s0;
  w1 = (w1 & 0x77777777u) | s1;
#endif
  return make_uint2(w0, w1);
}

ARC_DEV uint2 encode16(const float (&z)[16], float k, float (&t)[16]) {
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const float2 p = mul2(z[i], z[i + 1], k);
    t[i] = p.x;
    t[i + 1] = p.y;
  }
  uint32_t w0, w1;
  asm("{\n\t.reg .b8 b<8>;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %3, %2;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %5, %4;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %7, %6;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %9, %8;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b4, %11, %10;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b5, %13, %12;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b6, %15, %14;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b7, %17, %16;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t"
      "mov.b32 %1, {b4, b5, b6, b7};\n\t}"
      : "=r"(w0), "=r"(w1)
      : "f"(t[0]), "f"(t[1]), "f"(t[2]), "f"(t[3]), "f"(t[4]), "f"(t[5]), "f"(t[6]), "f"(t[7]), "f"(t[8]),
        "f"(t[9]), "f"(t[10]), "f"(t[11]), "f"(t[12]), "f"(t[13]), "f"(t[14]), "f"(t[15]));
  return make_uint2(w0, w1);
}

// e = t - v(q) for 16 codes (exact: t and v(q) are multiples of ulp(t)).  The
// E2M1 values come from the hardware decoder cvt.rn.f16x2.e2m1x2 (exact in f16).
ARC_DEV void residual16(const float (&t)[16], uint2 packed, float (&e)[16]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? packed.x : packed.y;
    const uint32_t byte = (w >> (8 * (i & 3))) & 0xFFu;
    uint32_t h2;
    asm("{\n\t.reg .b8 b;\n\t.reg .b16 lo, hi;\n\t"
        "cvt.u8.u32 b, %1;\n\t"
        "cvt.rn.f16x2.e2m1x2 %0, b;\n\t}"
        : "=r"(h2)
        : "r"(byte));
    const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&h2));
    e[2 * i] = __fsub_rn(t[2 * i], v.x);
    e[2 * i + 1] = __fsub_rn(t[2 * i + 1], v.y);
  }
}

// k2 = RN(d1 / d2) for scale codes c1, c2 (oracle STAGE's k with base d1).  For two
// normal E4M3 values the quotient is 2^(e1-e2) * (8+m1)/(8+m2), so RN commutes with
// the power of two: k2 = RN((8+m1)/(8+m2)) scaled by 2^(e1-e2) (exact exponent add).
// Subnormal codes take the IEEE division.
ARC_DEV float ratio_k(uint32_t c1, uint32_t c2, const float* rat) {
  if (c2 == 0u) return 0.0f;
  if (c1 < 8u || c2 < 8u) return __fdiv_rn(e4m3_value(c1), e4m3_value(c2));
  const float r = rat[((c1 & 7u) << 3) | (c2 & 7u)];
  return __uint_as_float(__float_as_uint(r) + ((int)(c1 >> 3) - (int)(c2 >> 3)) * (1 << 23));
}

// max |z| over 16 values as a shallow tree (exact; order-independent)
ARC_DEV float absmax16(const float (&z)[16]) {
  float m[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m[i] = fmaxf(fabsf(z[2 * i]), fabsf(z[2 * i + 1]));
#pragma unroll
  for (int i = 0; i < 4; ++i) m[i] = fmaxf(m[i], m[i + 4]);
  return fmaxf(fmaxf(m[0], m[2]), fmaxf(m[1], m[3]));
}

// Branch-free smallest E4M3 code >= v (v >= 0), saturating at 0x7E (Q2); same
// result as arc::e4m3_ceil (probe-tested).
ARC_DEV uint32_t e4m3_ceil_nb(float v) {
  const uint32_t b = __float_as_uint(v);
  const uint32_t cn = min((b >> 20) - 960u + ((b & 0xFFFFFu) != 0u), 126u);  // normal grid, saturated
  const uint32_t cs = (uint32_t)ceilf(__fmul_rn(v, 512.0f));                 // subnormal grid (v < 2^-6)
  return v < 0.015625f ? cs : cn;
}

// physical block of logical block l (App.D P:591-597 interleaved, or the
// logical concatenation of P:138): primaries l < K/16, residual j = K/16 + j
ARC_DEV int phys_block(int l, int nb, int ns, int layout) {
  if (layout != 0) return l;
  if (l < ns) return 2 * l;
  if (l < nb) return l + ns;
  return 2 * (l - nb) + 1;
}

// ------------------------------------------------------------------ RMSNorm (reading Q23)
// 1/sqrt(ss/K + eps) of one bf16 row (generic pointer: shared or global), computed by one warp
// in the oracle's pinned order (reading Q23): per 16-channel block a sequential fma over its 16
// squares; block b goes to lane b mod 32 (so a warp's loads at each step are 1 KB contiguous:
// no shared-memory bank conflicts), each lane reduces its BPL blocks as a pairwise tree in
// increasing b, and the 32 lane partials as a pairwise tree over the lanes (xor shuffles).
template <int BPL>
ARC_DEV float rms_scale_warp(const uint8_t* row, int K, float eps, int lane) {
  const int nb = K >> 4;
  // local pairwise tree over this lane's BPL leaves as a binary counter: lv[l] holds the
  // pending left subtree of size 2^l; indices are compile-time (unrolled), so registers only
  float lv[7];
  float c = 0.0f;
#pragma unroll
  for (int j = 0; j < BPL; ++j) {
    const int b = j * 32 + lane;
    float acc = 0.0f;
    if (b < nb) {
      const uint4 w0 = *reinterpret_cast<const uint4*>(row + b * 32);
      const uint4 w1 = *reinterpret_cast<const uint4*>(row + b * 32 + 16);
      const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xFFFF0000u);
        acc = __fmaf_rn(lo, lo, acc);
        acc = __fmaf_rn(hi, hi, acc);
      }
    }
    c = acc;
#pragma unroll
    for (int l = 0; (1 << l) < BPL; ++l) {
      if (j & (1 << l)) {
        c = __fadd_rn(lv[l], c);  // left + right
      } else {
        lv[l] = c;
        break;
      }
    }
  }
  float ss = c;  // the root of the lane's subtree (BPL a power of two)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  const float mean = __fdiv_rn(ss, (float)K);
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(mean, eps)));
}

// MAXNB: an upper bound on K/16 known at compile time (the kernel's row-slot size), so only the tree
// depths that can occur are instantiated (each deeper one is a fully unrolled loop of 2x the code)
template <int MAXNB = 2048>
ARC_DEV float rms_scale_any(const uint8_t* row, int K, float eps, int lane) {
  const int nb = K >> 4;
  if (MAXNB <= 32 || nb <= 32) return rms_scale_warp<1>(row, K, eps, lane);
  if (MAXNB <= 64 || nb <= 64) return rms_scale_warp<2>(row, K, eps, lane);
  if (MAXNB <= 128 || nb <= 128) return rms_scale_warp<4>(row, K, eps, lane);
  if (MAXNB <= 256 || nb <= 256) return rms_scale_warp<8>(row, K, eps, lane);
  if (MAXNB <= 512 || nb <= 512) return rms_scale_warp<16>(row, K, eps, lane);
  if (MAXNB <= 1024 || nb <= 1024) return rms_scale_warp<32>(row, K, eps, lane);
  return rms_scale_warp<64>(row, K, eps, lane);
}

// y_j = bf16(g_j * bf16(x_j * r)) for 8 channels (one 16-byte word of x and of gamma)
ARC_DEV uint4 rms_apply8(uint4 x, uint4 g, float r) {
  const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, gw[4] = {g.x, g.y, g.z, g.w};
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(xw[i] << 16), r),
                                                   __fmul_rn(__uint_as_float(xw[i] & 0xFFFF0000u), r));
    const uint32_t tw = *reinterpret_cast<const uint32_t*>(&t);
    const __nv_bfloat162 y = __floats2bfloat162_rn(
        __fmul_rn(__uint_as_float(gw[i] << 16), __uint_as_float(tw << 16)),
        __fmul_rn(__uint_as_float(gw[i] & 0xFFFF0000u), __uint_as_float(tw & 0xFFFF0000u)));
    o[i] = *reinterpret_cast<const uint32_t*>(&y);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// ------------------------------------------------------------------ SiLU-mul (Fig.5, reading Q24)
// fp32 SiLU of a bf16 gate value as the pinned sequence of IEEE RN ops of reading Q24
// (DESIGN.md): Cody-Waite reduction of e^-|g|, degree-7 Taylor in Horner form (one fma per
// step), exact power-of-two scaling in two halves, then sigma = 1/(1+E) or E/(1+E).
ARC_DEV float exp2i(int n) { return __int_as_float((n + 127) << 23); }  // 2^n, -126 <= n <= 127

ARC_DEV float silu_f32(float g) {
  const float a = fmaxf(-fabsf(g), -104.0f);
  const float n = rintf(__fmul_rn(a, 0x1.715476p+0f));
  float r = __fmaf_rn(n, -0x1.62e4p-1f, a);
  r = __fmaf_rn(n, -0x1.7f7d1cp-20f, r);
  float p = 0x1.a01a02p-13f;
  p = __fmaf_rn(p, r, 0x1.6c16c2p-10f);
  p = __fmaf_rn(p, r, 0x1.111112p-7f);
  p = __fmaf_rn(p, r, 0x1.555556p-5f);
  p = __fmaf_rn(p, r, 0x1.555556p-3f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  const int ni = (int)n, n1 = ni / 2, n2 = ni - n1;
  const float E = __fmul_rn(__fmul_rn(p, exp2i(n1)), exp2i(n2));
  const float rc = __frcp_rn(__fadd_rn(1.0f, E));
  const float q = g >= 0.0f ? g : __fmul_rn(g, E);
  return __fmul_rn(q, rc);
}

// h = bf16(bf16(SiLU(g)) * u) of one gate/up pair, as fp32 (exact: h is a bf16 value)
ARC_DEV float silu_mul1(float g, float u) {
  const float s = __bfloat162float(__float2bfloat16_rn(silu_f32(g)));
  return __bfloat162float(__float2bfloat16_rn(__fmul_rn(s, u)));
}

// 8 channels: one 16-byte word of gate and of up -> one 16-byte word of h (bf16)
ARC_DEV uint4 silu_mul8(uint4 g, uint4 u) {
  const uint32_t gw[4] = {g.x, g.y, g.z, g.w}, uw[4] = {u.x, u.y, u.z, u.w};
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(
        silu_mul1(__uint_as_float(gw[i] << 16), __uint_as_float(uw[i] << 16)),
        silu_mul1(__uint_as_float(gw[i] & 0xFFFF0000u), __uint_as_float(uw[i] & 0xFFFF0000u)));
    o[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// SiLU (reading Q24) of a bf16 gate pattern gb -> bf16 pattern of bf16(SiLU(g)).  Patterns with
// |g| in [2^-9, 128) -- magnitude bits [SILU_LO, SILU_LO + SILU_N) -- read a per-CTA table at
// index (mag - SILU_LO) | (sign << 11), built with silu_f32 itself; the rest follow from the
// pinned sequence in closed form (checked against the oracle over all 2^16 patterns):
//   |g| < 2^-125 (exponent field 0 or 1): E = 1, d = 2, s = g/2 exactly, bf16 ties to even;
//   2^-125 <= |g| < 2^-9: bf16(SiLU(g)) = g/2 (exponent - 1);
//   g >= 128: g;  g <= -128: -0.
constexpr uint32_t SILU_LO = 0x3B00u, SILU_N = 0x800u;
constexpr int SILU_TAB = 4096;

ARC_DEV uint32_t silu_bf16_bits(uint32_t gb, const uint16_t* tab) {
  const uint32_t mag = gb & 0x7FFFu;
  const uint32_t t = mag - SILU_LO;
  if (t < SILU_N) return tab[t | ((gb >> 4) & 0x800u)];
  const uint32_t neg = gb & 0x8000u;
  if (mag < 0x100u) return ((mag + ((mag >> 1) & 1u)) >> 1) | neg;
  if (mag < SILU_LO) return (mag - 0x80u) | neg;
  return neg ? 0x8000u : mag;
}

ARC_DEV void build_silu_table(uint16_t* tab, int tid, int nthreads) {
  for (int c = tid; c < SILU_TAB; c += nthreads) {
    const uint32_t gb = (((uint32_t)c & 2047u) + SILU_LO) | (((uint32_t)c & 2048u) << 4);
    tab[c] = __bfloat16_as_ushort(__float2bfloat16_rn(silu_f32(__uint_as_float(gb << 16))));
  }
}

}  // namespace arc
