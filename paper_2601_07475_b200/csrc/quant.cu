// quant.cu -- the fused ARC reorder + NVFP4 primary quantize + residual quantize
// kernel ("Online Activation Quantization", "Fused
// Quantization Kernel"), its weight-preparation mode, and the two
// reduction kernels of the offline path (calibration abs-max; tensor
// scale, P:118 / P:453).
//
// HBM-bound.  Per token row: read K bf16 (2K B), write Kp/2 code bytes + Kp/16
// scale bytes.  Rows are staged in shared memory with cp.async.bulk (one bulk
// copy per row, double-buffered across row tiles, mbarrier completion); the
// calibrated permutation lives in shared memory as uint16.  One thread owns one
// 16-element physical block: it gathers its 16 channels from the staged row,
// computes the block max, the ceil-rounded E4M3 scale, the E2M1 codes
// (cvt.rn.satfinite.e2m1x2) and, for residual blocks, the second stage on the
// exact residual e = t - v(q1); it writes its 8 code bytes (a warp writes 256
// contiguous bytes) and the 4 scale bytes of each 4-block unit are gathered with
// two shuffles into one 32-bit store in the 128x4 tile layout.
//
// Bit-exactness: every fp32 op is one IEEE RN op in the order of the oracle's
// STAGE (Q7): c6 = base/6, v = a*c6, sf = ceil_e4m3(v), d = e4m3(sf),
// k = base/d, t = z*k, q = rne_e2m1(t); residual e = t - v(q) (exact),
// stage 2 with base = d1.
#include "arc_device.cuh"
#include "arc_internal.h"
#include "quant_dev.cuh"
#include "arc_probe.h"

#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace arc {

ARC_DEV int64_t dmin64(int64_t a, int64_t b) { return a < b ? a : b; }
static inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
static inline int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

struct QuantArgs {
  const uint16_t* x;   // bf16 bits [rows][ld]
  int64_t rows;
  int32_t K;
  int64_t ld;
  const int32_t* perm;
  int32_t S;
  const float* gs;
  int32_t layout;      // 0 interleaved, 1 contiguous
  int32_t weight_mode; // 1: augmented blocks duplicate the primary block
  uint8_t* codes;
  uint8_t* sf;
  int32_t Kp;
  int32_t rows_per_tile;
  int32_t stages;
  int32_t npw;     // primary warps
  int32_t nrw;     // residual warps
  int32_t bulk;    // producer uses one cp.async.bulk per row (else 16-byte cp.async per lane)
  int32_t debug;   // perf experiments only (env ARC_QUANT_DEBUG): 1 = skip compute, 2 = skip loads, 5 = SiLU mode
                   // without table lookups, 6 = SiLU mode without the up gather,
                   // 3 = quantizing warps do not wait for the norm warps, 4 = norm warps skip the RMS
  const uint16_t* gamma;  // RMSNorm weight bf16[K] (norm mode)
  float eps;
  int32_t norm;    // 1: RMSNorm the staged rows in place before quantizing (R norm warps)
  int64_t up_off;  // SiLU-mul mode (Fig.5, reading Q24): x holds gate, x + up_off holds up
  unsigned long long* trace;  // timing experiments only (ARC_TRACE): [cta][8] globaltimer stamps
  int32_t consts_ready;       // perm may be read before griddepcontrol.wait (arc_linear)
  int32_t f16;                // the 16-bit rows are IEEE fp16 (ARC_FP16), else bf16
  int32_t stage_rows;         // arc_quant_small_kernel: copy the CTA's x rows to shared memory with 16-byte
                              // coalesced loads, then gather from there (else 16 2-byte gathers from L2)
};

ARC_DEV void qtrace(const QuantArgs& a, int i) {
  if (a.trace && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(size_t)blockIdx.x * 8 + i] = t;
  }
}

ARC_DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async copies completed
ARC_DEV void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// a 16-bit input element (bf16, or IEEE fp16 for F16 = true: arc_dtype_t ARC_FP16) as fp32 (exact)
template <bool F16>
ARC_DEV float in16_to_f32(uint32_t h) {
  if (F16) return __half2float(__ushort_as_half((unsigned short)h));
  return bf16_bits_to_f32(h);
}
// gather 16 channels of one staged row (byte offsets into smem) as fp32 (exact)
template <bool F16 = false>
ARC_DEV void gather16(const uint8_t* base, const uint32_t (&off)[16], float (&z)[16]) {
#pragma unroll
  for (int q = 0; q < 16; ++q) z[q] = in16_to_f32<F16>(*reinterpret_cast<const uint16_t*>(base + off[q]));
}

// RMSNorm of the 16 gathered channels of logical block l (reading Q23): z = bf16(g * bf16(z * r)).
// gperm holds gamma in reordered order (gperm[16 l + q] = gamma[perm[16 l + q]], staged once per
// CTA), so a lane's 16 gains are two conflict-free 16-byte loads at gperm + 32 l.  Pairs:
// mul.rn.f32x2, one cvt.rn.bf16x2.f32, one bf16x2 multiply (the product of two bf16 is exact in
// fp32, so its single rounding equals the oracle's).
ARC_DEV void norm16w(float (&z)[16], const uint32_t (&gw)[8], float r) {
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const float2 p = mul2(z[i], z[i + 1], r);
    const __nv_bfloat162 t = __floats2bfloat162_rn(p.x, p.y);
    const __nv_bfloat162 y = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&gw[i >> 1]), t);
    const uint32_t yw = *reinterpret_cast<const uint32_t*>(&y);
    z[i] = __uint_as_float(yw << 16);
    z[i + 1] = __uint_as_float(yw & 0xFFFF0000u);
  }
}
ARC_DEV void norm16(float (&z)[16], const uint8_t* gblk, float r) {
  const uint4 g0 = *reinterpret_cast<const uint4*>(gblk);
  const uint4 g1 = *reinterpret_cast<const uint4*>(gblk + 16);
  const uint32_t gw[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  norm16w(z, gw, r);
}

// h = bf16(s * u) for two (SiLU bits, up-in-high-half word) pairs: one mul.rn.f32x2 + one
// cvt.rn.bf16x2.f32 (s * u of two bf16 values is exact in fp32 unless it underflows, where the
// fp32 rounding happens exactly as in the oracle's fp32 multiply)
ARC_DEV void silu_prod2(uint32_t s0, uint32_t s1, uint32_t w0, uint32_t w1, float& z0, float& z1) {
  unsigned long long a, b, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(s0 << 16), "r"(s1 << 16));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "r"(w0 & 0xFFFF0000u), "r"(w1 & 0xFFFF0000u));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  float p0, p1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(p0), "=f"(p1) : "l"(r));
  const __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
  const uint32_t hw = *reinterpret_cast<const uint32_t*>(&h);
  z0 = __uint_as_float(hw << 16);
  z1 = __uint_as_float(hw & 0xFFFF0000u);
}

// SiLU-mul of one 16-channel block (reading Q24): z = bf16(bf16(SiLU(g)) * u) for the 16
// gathered (g, u) pairs.  MODE 1: gate row at `row`, up row at row + upb (two LDS.U16 per
// channel); MODE 2: (g, u) adjacent bf16 pairs, one LDS.32 per channel (off = 4 * channel).
// The block's 16 gate patterns are first checked against the table range (one branch per
// block, rarely divergent).
// (Measured alternatives: a MUFU fast path -- ex2.approx + rcp.approx with a
// midpoint-distance check falling back to the table -- is MUFU-bound and 40 % slower; a
// (g, u)-pair layout with one LDS.32 per channel is no faster.)
template <int MODE>
ARC_DEV void silu_mul_block16(float (&z)[16], const uint8_t* row, const uint32_t (&off)[16], int upb,
                              const uint16_t* tab, int dbg = 0) {
#pragma unroll
  for (int hb = 0; hb < 16; hb += 8) {  // two halves of 8 channels: 8 live (g, u) words
    uint32_t w[8];  // gate bits | up bits << 16
    uint32_t tmax = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 2) w[q] = *reinterpret_cast<const uint32_t*>(row + off[hb + q]);
      else if (dbg == 6) w[q] = *reinterpret_cast<const uint16_t*>(row + off[hb + q]) | 0x3F800000u;
      else w[q] = *reinterpret_cast<const uint16_t*>(row + off[hb + q]) |
                  ((uint32_t)*reinterpret_cast<const uint16_t*>(row + upb + off[hb + q]) << 16);
      tmax = max(tmax, (w[q] & 0x7FFFu) - SILU_LO);
    }
    if (dbg == 5) {
#pragma unroll
      for (int q = 0; q < 8; q += 2) silu_prod2(w[q] & 0xFFFFu, w[q + 1] & 0xFFFFu, w[q], w[q + 1], z[hb + q], z[hb + q + 1]);
    } else if (tmax < SILU_N) {
#pragma unroll
      for (int q = 0; q < 8; q += 2)
        silu_prod2(tab[((w[q] & 0x7FFFu) - SILU_LO) | ((w[q] >> 4) & 0x800u)],
                   tab[((w[q + 1] & 0x7FFFu) - SILU_LO) | ((w[q + 1] >> 4) & 0x800u)], w[q], w[q + 1], z[hb + q],
                   z[hb + q + 1]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; q += 2)
        silu_prod2(silu_bf16_bits(w[q] & 0xFFFFu, tab), silu_bf16_bits(w[q + 1] & 0xFFFFu, tab), w[q], w[q + 1],
                   z[hb + q], z[hb + q + 1]);
    }
  }
}

// MX block scale (reading Q25): for block abs-max a > 0, e = ceil(log2(RN(a/6))) (exact from the
// fp32 bits), clamped to [lo, hi] -- the exponents whose 2^(e - c) E4M3 can hold -- so a block far
// below the tensor's range flushes toward 0 and one above it saturates at +-6 with a scale that
// matches its codes (reading Q25b); k = 2^-e (t = z*k exact), code = E4M3 code of 2^(e - c);
// a = 0 -> code 0, k = 1.
ARC_DEV uint32_t mx_pow2_code(int k) {
  if (k >= -6) return (uint32_t)min(k + 7, 15) << 3;
  return 1u << max(k + 9, 0);
}
ARC_DEV int mx_ceil_exp(float a) {  // ceil(log2(RN(a / 6))) for a > 0
  const uint32_t b = __float_as_uint(__fdiv_rn(a, 6.0f));
  const int ex = (int)((b >> 23) & 0xFFu);
  if (ex == 0) {  // subnormal RN(a/6): value = m 2^-149, ceil(log2) = 32 - clz(m - 1) - 149
    const uint32_t m = b & 0x7FFFFFu;
    return (m <= 1u ? 0 : 32 - __clz(m - 1u)) - 149;
  }
  return ex - 127 + ((b & 0x7FFFFFu) != 0u);
}
ARC_DEV float mx_pow2_inv(int e) { return __int_as_float((min(max(127 - e, 1), 254)) << 23); }
ARC_DEV void mx_scale(float a, int c, uint32_t& code, float& k, int& e) {
  if (a == 0.0f) {
    code = 0u;
    k = 1.0f;
    e = 0;
    return;
  }
  e = min(max(mx_ceil_exp(a), c - 9), c + 8);
  code = mx_pow2_code(e - c);
  k = mx_pow2_inv(e);
}

// Rows of a tile.  Tile t of the 128-row group g holds rows base + 32 i, i < R, with
// base = 128 g + 32 R h + r (t = g * 128/R + 32 h + r): the R rows share (m & 31) and
// have consecutive (m >> 5) & 3, so in the 128x4 scale layout the tile's scales of one
// 4-block unit are R * 4 contiguous bytes -- staged in smem and stored as one R*4-byte
// word per unit instead of 4R scattered bytes.
template <int R>
ARC_DEV int tile_base(int t) {
  constexpr int TPG = 128 / R;
  const int g = t / TPG, tin = t - g * TPG;
  return g * 128 + (tin >> 5) * (R * 32) + (tin & 31);
}
template <int R>
ARC_DEV int tile_rows(int base, int64_t rows) {  // valid rows base + 32 i < rows
  const int64_t left = rows - base;
  return left <= 0 ? 0 : (int)dmin64(R, (left + 31) / 32);
}

// The quantization kernel.  Warp roles (no intra-warp divergence in steady state):
//  * primary warps: lane t owns logical primary block t (or a zero pad block) for
//    every row; its 16 gather offsets (byte offsets of the calibrated channels in
//    a staged row, P:136's reorder) live in registers; per row: 16 LDS, block
//    max, ceil-rounded E4M3 scale, 16 products and E2M1 codes (stage 1 of Eq.1).
//  * residual warps: lane i owns (row i / ns, outlier block i % ns) of each tile
//    and runs stage 1 + the residual stage 2 -- or, for weights, writes
//    the bitwise duplicate.  Gathering the outlier blocks of all R rows
//    of a tile into one warp keeps the heavier dual-stage work from serializing
//    a warp of primaries.
//  * producer warp: streams rows HBM -> smem (one cp.async.bulk per row) into an
//    ST-deep ring of R-row tiles (full[s] completes on the bytes); compute warps
//    release a slot by arriving on empty[s] (no CTA-wide barrier).  Before it
//    refills a slot the producer writes the slot's staged scale bytes out
//    (R*4-byte words, one per 4-block unit).
// Rows sit at a fixed ROWP stride (ROWB + 16: rows of one tile fall in different
// banks for the residual warp's cross-row gathers) and the tile loop is unrolled
// over the ring so the gathers are `LDS [off + const]`.
//
// SILU mode (the down-proj input site; ROWB then holds 4K bytes): SILU = 1, a staged row is the
// gate row [0, 2K) bytes followed by the up row [2K, 4K); SILU = 2, the row holds (g_j, u_j)
// bf16 pairs (an interleaved gate_up output).  The quantizing warps gather each of their 16
// channels' (g, u) and quantize h = bf16(bf16(SiLU(g)) * u) (silu_mul_block16, reading Q24).
//
// MX mode (reading Q25): MXFP4-ARC -- 32-channel blocks (the 16-blocks of lanes 2j, 2j+1,
// max combined with one shuffle), power-of-two scales 2^e = E8M0_up(amax/6), t = z * 2^-e, written in
// the NVFP4 physical format with the E4M3 code of 2^(e - c) (gs = 2^-c), so arc_gemm consumes it.
#ifndef ARC_QUANT_ROLL_ALL
#define ARC_QUANT_ROLL_ALL 0
#endif
constexpr bool kRollAll = ARC_QUANT_ROLL_ALL != 0;  // experiment: roll the plain kernels' loops too
template <int IPT, int R, int ROWB, int ST, bool NORM, int SILU, bool MX, bool F16 = false>
__global__ void __launch_bounds__(1024) arc_quant_kernel(QuantArgs p) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int ROWP = ROWB + 16;
  constexpr int SLOT = R * ROWP;
  constexpr int UB = R * 4;  // staged scale bytes per 4-block unit per tile
  // The fused producers' per-block bodies (RMSNorm / SiLU-mul + quantize) are large: unrolling them over
  // the ring's stages and the tile's rows made 250-370 KB kernels that stall on instruction fetch, so those
  // instantiations keep the stage and row loops rolled (the slot / row offsets become uniform registers).
  constexpr int UNR_S = (NORM || SILU || kRollAll) ? 1 : ST;
  constexpr int UNR_R = (NORM || SILU || kRollAll) ? 1 : R;
  const int K = p.K;
  const int npw = p.npw, nrw = p.nrw;
  constexpr uint32_t OSC = SILU == 2 ? 4u : 2u;  // staged bytes per channel index
  const int NU = p.Kp >> 6;  // 4-block units per row
  uint8_t* sfst = smem + ST * SLOT;  // [ST][NU][UB]
  // tables and mbarriers start 16-byte aligned: ST * NU * UB is only a multiple of 4 when Kp/64 is odd
  float* k1tab = reinterpret_cast<float*>(smem + ((ST * SLOT + ST * NU * UB + 15) & ~15));
  float* c6tab = k1tab + 128;  // RN(e4m3(c) / 6): the residual stage's c6 for base d1 = e4m3(c)
  float* rat = c6tab + 128;    // RN((8+m1)/(8+m2)): mantissa ratio of two normal E4M3 scales
  uint64_t* full = reinterpret_cast<uint64_t*>(rat + 64);
  uint64_t* empty = full + ST;
  uint64_t* normed = empty + ST;  // norm mode: the RMS scales of slot s's rows are ready
  float* rscale = reinterpret_cast<float*>(normed + ST);  // [ST][R] 1/rms of each staged row
  // gam: addressed from `smem` (an integer offset) so every access stays an LDS/STS, not a generic access
  uint8_t* gam = smem + ((reinterpret_cast<uint8_t*>(rscale + ST * R) - smem + 15) & ~15);
  // SiLU table at the same place, addressed from `smem` so loads stay in the shared window
  const uint16_t* stab = reinterpret_cast<const uint16_t*>(gam);
  // gam: gamma in reordered channel order, bf16[K], staged once per CTA (norm mode)

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int ntile = (int)((p.rows + 127) / 128) * (128 / R);
  const int my_tiles = ntile > (int)blockIdx.x ? (ntile - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int sf_rb_stride = (p.Kp >> 6) * 512;
  const int code_row = p.Kp >> 1;
  // (PDL) wait first, then let the next kernel launch: a dependent launched from here on knows every
  // kernel before this one has completed (the decode GEMM streams weights before its own wait).
  // Weight preparation never lets dependents launch early: a kernel that follows it may then
  // assume the weights are complete (the invariant the decode GEMM's early weight stream uses).
  if (threadIdx.x == 0) qtrace(p, 0);
  pdl_wait();  // the previous kernel's writes are visible from here on
  if (!p.weight_mode) pdl_launch_dependents();
  if (threadIdx.x == 0) qtrace(p, 1);
  const float gs = __ldg(p.gs);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], p.bulk ? 1 : 32);
      mbar_init(&empty[s], npw + nrw);
      mbar_init(&normed[s], R);
    }
    fence_mbar_init();
  }
  // k1 = RN(gs / e4m3(c)) for every scale code: the primary stage's multiplier
  // depends only on the code, so the IEEE division is done once per CTA.
  for (int c = tid; c < 128; c += blockDim.x) {
    k1tab[c] = (c == 0 || c == 127) ? 0.0f : __fdiv_rn(gs, e4m3_value((uint32_t)c));
    c6tab[c] = __fdiv_rn(e4m3_value((uint32_t)c), 6.0f);
    if (c < 64) rat[c] = __fdiv_rn((float)(8 + (c >> 3)), (float)(8 + (c & 7)));
  }
  if (SILU) build_silu_table(reinterpret_cast<uint16_t*>(gam), tid, blockDim.x);
  if (NORM) {
    // gamma in reordered channel order: 8 channels per thread, the 8 perm words and then the 8 gamma
    // gathers issued back to back (independent loads), one 16-byte shared store
    const unsigned short* g16 = reinterpret_cast<const unsigned short*>(p.gamma);
    for (int c8 = tid * 8; c8 < K; c8 += blockDim.x * 8) {
      const int4 a = __ldg(reinterpret_cast<const int4*>(p.perm + c8));
      const int4 b = __ldg(reinterpret_cast<const int4*>(p.perm + c8 + 4));
      const uint32_t v0 = __ldg(g16 + a.x), v1 = __ldg(g16 + a.y), v2 = __ldg(g16 + a.z), v3 = __ldg(g16 + a.w);
      const uint32_t v4 = __ldg(g16 + b.x), v5 = __ldg(g16 + b.y), v6 = __ldg(g16 + b.z), v7 = __ldg(g16 + b.w);
      *reinterpret_cast<uint4*>(gam + 2 * c8) = make_uint4(v0 | (v1 << 16), v2 | (v3 << 16), v4 | (v5 << 16), v6 | (v7 << 16));
    }
  }

  __syncthreads();

  if (warp == npw + nrw) {
    // ---------------------------------------------------------------- producer warp
    const uint32_t ring = smem_u32(smem) + (uint32_t)lane * 16u;
    const int kc = K >> 3;  // 16-byte chunks per row
    const uint32_t rowbytes = (uint32_t)K * (SILU ? 4u : 2u);
    // X is read once: evict-first at streaming sizes; a decode-size activation (<= 64 rows) keeps the
    // normal priority so it stays in L2 while the next GEMM streams its weights with evict-first
    const uint64_t x_policy = p.rows <= 64 ? policy_evict_normal() : policy_evict_first();
    // scales staged for tile jt (slot s) -> global, one UB-byte word per unit
    auto flush_sf = [&](int s, int jt) {
      const int base = tile_base<R>((int)blockIdx.x + jt * (int)gridDim.x);
      uint8_t* dst = p.sf + (int64_t)(base >> 7) * sf_rb_stride + (base & 31) * 16 + ((base >> 5) & 3) * 4;
      const uint8_t* src = sfst + s * NU * UB;
      for (int u = lane; u < NU; u += 32) {
        if (UB == 16) *reinterpret_cast<uint4*>(dst + u * 512) = *reinterpret_cast<const uint4*>(src + u * 16);
        else if (UB == 8) *reinterpret_cast<uint2*>(dst + u * 512) = *reinterpret_cast<const uint2*>(src + u * 8);
        else *reinterpret_cast<uint32_t*>(dst + u * 512) = *reinterpret_cast<const uint32_t*>(src + u * 4);
      }
    };
    for (int j0 = 0; j0 < my_tiles; j0 += ST) {
#pragma unroll
      for (int s = 0; s < ST; ++s) {
        const int j = j0 + s;
        if (j < my_tiles) {
          if (j >= ST) {
            mbar_wait(&empty[s], ((j / ST) - 1) & 1);
            fence_proxy_async();  // order the consumers' generic-proxy reads before the async refill
            flush_sf(s, j - ST);
          }
          const int base = tile_base<R>((int)blockIdx.x + j * (int)gridDim.x);
          const int nr = tile_rows<R>(base, p.rows);
          if (p.bulk) {
            // one cp.async.bulk per row (TMA engine, no LSU/MIO traffic); lane 0 only
            if (lane == 0) {
              mbar_expect_tx(&full[s], (uint32_t)nr * rowbytes);
              if (p.debug != 2)
                for (int r = 0; r < nr; ++r) {  // X is read once: evict-first
                  bulk_load_hint(smem + s * SLOT + r * ROWP, p.x + (int64_t)(base + 32 * r) * p.ld,
                                 (uint32_t)K * (SILU == 2 ? 4 : 2), &full[s], x_policy);
                  if (SILU == 1)
                    bulk_load_hint(smem + s * SLOT + r * ROWP + K * 2, p.x + (int64_t)(base + 32 * r) * p.ld + p.up_off,
                                   (uint32_t)K * 2, &full[s], x_policy);
                }
              else
                mbar_complete_tx_self(&full[s], (uint32_t)nr * rowbytes);
            }
          } else {
            if (p.debug != 2) {
#pragma unroll
              for (int r = 0; r < R; ++r)
                if (r < nr) {
                  const uint16_t* src = p.x + (int64_t)(base + 32 * r) * p.ld + lane * 8;
                  for (int c = 0; c < kc - lane; c += 32)
                    cp_async16(ring + (uint32_t)(s * SLOT + r * ROWP + c * 16), src + c * 8);
                }
            }
            cp_async_arrive(&full[s]);
          }
        }
      }
    }
    for (int jt = my_tiles > ST ? my_tiles - ST : 0; jt < my_tiles; ++jt) {
      const int s = jt % ST;
      mbar_wait(&empty[s], (jt / ST) & 1);
      flush_sf(s, jt);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (lane == 0) qtrace(p, 2);
    return;
  }

  if (NORM && warp > npw + nrw) {
    // ---------------------------------------------------------------- norm warps (RMSNorm)
    // norm warp r owns row r of every tile: its RMS scale 1/sqrt(mean(x^2)+eps) in the pinned
    // order (Q23), published in smem; the quantizing warps apply y = bf16(g * bf16(x * r)) to
    // the 16 channels they gather (norm16)
    const int r = warp - (npw + nrw + 1);
    for (int j0 = 0; j0 < my_tiles; j0 += ST) {
#pragma unroll 1
      for (int s = 0; s < ST; ++s) {
        const int j = j0 + s;
        if (j < my_tiles) {
          mbar_wait(&full[s], (j / ST) & 1);
          const int base = tile_base<R>((int)blockIdx.x + j * (int)gridDim.x);
          if (r < tile_rows<R>(base, p.rows) && p.debug != 1 && p.debug != 4) {
            const float sc = rms_scale_any<ROWB / 32>(smem + s * SLOT + r * ROWP, K, p.eps, lane);
            if (lane == 0) rscale[s * R + r] = sc;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&normed[s]);
        }
      }
    }
    return;
  }

  const int nb = K >> 4, ns = p.S >> 4;
  const int ka16 = nb + ns, NB = p.Kp >> 4;
  uint64_t* ready = (NORM && p.debug != 3) ? normed : full;  // what the quantizing warps wait for
  const float c6g = __fdiv_rn(gs, 6.0f);
  const int mx_c = 127 - (int)((__float_as_uint(gs) >> 23) & 0xFFu);  // MX: gs = 2^-c

  if (warp < npw) {
    // ---------------------------------------------------------------- primary warps
    uint32_t off[IPT][16];
    uint32_t greg[IPT][8];    // norm mode: the lane's 16 gains (reordered order), kept in registers
    int pbs[IPT], kind[IPT];  // kind: 0 idle, 1 primary, 3 zero pad block
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const int t = tid + i * npw * 32;
      int l = 0, k = 0, pb = 0;
      if (t < nb) { l = t; k = 1; pb = phys_block(t, nb, ns, p.layout); }
      else if (t < nb + (NB - ka16)) { k = 3; pb = ka16 + (t - nb); }
      kind[i] = k;
      pbs[i] = pb;
      if (NORM) {
        const uint4 g0 = *reinterpret_cast<const uint4*>(gam + 32 * l);
        const uint4 g1 = *reinterpret_cast<const uint4*>(gam + 32 * l + 16);
        greg[i][0] = g0.x; greg[i][1] = g0.y; greg[i][2] = g0.z; greg[i][3] = g0.w;
        greg[i][4] = g1.x; greg[i][5] = g1.y; greg[i][6] = g1.z; greg[i][7] = g1.w;
      }
      const int4* pp = reinterpret_cast<const int4*>(p.perm + 16 * l);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 v = __ldg(pp + q);
        off[i][4 * q + 0] = (uint32_t)v.x * OSC;
        off[i][4 * q + 1] = (uint32_t)v.y * OSC;
        off[i][4 * q + 2] = (uint32_t)v.z * OSC;
        off[i][4 * q + 3] = (uint32_t)v.w * OSC;
      }
    }
    for (int j0 = 0; j0 < my_tiles; j0 += ST) {
#pragma unroll UNR_S
      for (int s = 0; s < ST; ++s) {
        const int j = j0 + s;
        if (j < my_tiles) {
          mbar_wait(&ready[s], (j / ST) & 1);
          if (p.debug != 1) {
            const int base = tile_base<R>((int)blockIdx.x + j * (int)gridDim.x);
            const int nr = tile_rows<R>(base, p.rows);
            uint8_t* st = sfst + s * NU * UB;
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
              if (MX) {
                // every lane takes part (the block max is shared by lane pairs); idle lanes store nothing
                const int pb = pbs[i];
                uint8_t* cptr = p.codes + (int64_t)base * code_row + pb * 8;
                uint8_t* sst = st + (pb >> 2) * UB + (pb & 3);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  uint32_t sfb = 0;
                  if (r < nr) {
                    float z[16];
                    if (kind[i] == 1) gather16<F16>(smem + s * SLOT + r * ROWP, off[i], z);
                    else
#pragma unroll
                      for (int q = 0; q < 16; ++q) z[q] = 0.0f;
                    float a = absmax16(z);
                    a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, 1));
                    float k;
                    int e;
                    mx_scale(a, mx_c, sfb, k, e);
                    const uint2 packed = encode16(z, k);
                    if (kind[i] != 0) *reinterpret_cast<uint2*>(cptr + (int64_t)(32 * r) * code_row) = packed;
                    if (kind[i] != 1) sfb = 0;
                  }
                  if (kind[i] != 0) sst[4 * r] = (uint8_t)sfb;
                }
              } else if (kind[i] != 0) {
                const int pb = pbs[i];
                uint8_t* cptr = p.codes + (int64_t)base * code_row + pb * 8;
                uint8_t* sst = st + (pb >> 2) * UB + (pb & 3);
#pragma unroll UNR_R
                for (int r = 0; r < R; ++r) {
                  uint32_t sfb = 0;
                  if (r < nr) {
                    uint2 packed = make_uint2(0u, 0u);
                    if (kind[i] == 1) {
                      float z[16];
                      if (SILU) {
                        silu_mul_block16<SILU>(z, smem + s * SLOT + r * ROWP, off[i], K * 2, stab, p.debug);
                      } else {
                        gather16<F16>(smem + s * SLOT + r * ROWP, off[i], z);
                        if (NORM) norm16w(z, greg[i], rscale[s * R + r]);
                      }
                      // stage 1 (Eq.1 with the NVFP4 two-level scale, Q7 op order)
                      sfb = e4m3_ceil_nb(__fmul_rn(absmax16(z), c6g));
                      packed = encode16(z, k1tab[sfb]);
                    }
                    *reinterpret_cast<uint2*>(cptr + (int64_t)(32 * r) * code_row) = packed;
                  }
                  sst[4 * r] = (uint8_t)sfb;  // rows past M stage a 0 scale (padding rows)
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
      }
    }
    if (warp == 0 && lane == 0) qtrace(p, 3);
    return;
  }

  // ---------------------------------------------------------------- residual warps
  if (MX) {
    // warp-uniform item loop (lane pairs share each 32-block's maxima); items (row, outlier 16-block).
    // The lane's first item's 16 gather offsets are kept in registers (the common case R*ns <= 32*nrw).
    uint32_t moff[16];
    {
      const int it = (warp - npw) * 32 + lane;
      const int jb = it < R * ns ? it % ns : 0, r = it < R * ns ? it / ns : 0;
      const int4* pp = reinterpret_cast<const int4*>(p.perm + 16 * jb);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 v = __ldg(pp + q);
        moff[4 * q + 0] = (uint32_t)v.x * 2u + (uint32_t)(r * ROWP);
        moff[4 * q + 1] = (uint32_t)v.y * 2u + (uint32_t)(r * ROWP);
        moff[4 * q + 2] = (uint32_t)v.z * 2u + (uint32_t)(r * ROWP);
        moff[4 * q + 3] = (uint32_t)v.w * 2u + (uint32_t)(r * ROWP);
      }
    }
    for (int j0 = 0; j0 < my_tiles; j0 += ST) {
#pragma unroll UNR_S
      for (int s = 0; s < ST; ++s) {
        const int j = j0 + s;
        if (j < my_tiles) {
          mbar_wait(&ready[s], (j / ST) & 1);
          const int base = tile_base<R>((int)blockIdx.x + j * (int)gridDim.x);
          const int nr = tile_rows<R>(base, p.rows);
          uint8_t* st = sfst + s * NU * UB;
          for (int it0 = (warp - npw) * 32; it0 < R * ns; it0 += nrw * 32) {
            const int it = it0 + lane;
            const bool has = it < R * ns;
            const int r = has ? it / ns : 0, jb = has ? it - (it / ns) * ns : 0;
            const bool live = has && r < nr;
            float z[16];
            if (live && it0 == (warp - npw) * 32) {
              gather16<F16>(smem + s * SLOT, moff, z);
            } else if (live) {
              const int* pp = p.perm + 16 * jb;
#pragma unroll
              for (int q = 0; q < 16; ++q)
                z[q] = in16_to_f32<F16>(*reinterpret_cast<const uint16_t*>(smem + s * SLOT + r * ROWP + 2 * __ldg(pp + q)));
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q) z[q] = 0.0f;
            }
            float a = absmax16(z);
            a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, 1));
            uint32_t c1;
            float k1;
            int e1;
            mx_scale(a, mx_c, c1, k1, e1);
            float t[16];
            uint2 packed = encode16(z, k1, t);
            uint32_t sfb = c1;
            if (!p.weight_mode) {
              float ee[16];
              residual16(t, packed, ee);
              float a2 = absmax16(ee);
              a2 = fmaxf(a2, __shfl_xor_sync(0xffffffffu, a2, 1));
              // stage 2 in units of 2^e1: absolute exponent e1 + e2 clamped like the primary's
              uint32_t c2 = 0u;
              float k2 = 1.0f;
              if (a != 0.0f && a2 != 0.0f) {
                const int ea = min(max(e1 + mx_ceil_exp(a2), mx_c - 9), mx_c + 8);
                c2 = mx_pow2_code(ea - mx_c);
                k2 = mx_pow2_inv(ea - e1);
              }
              packed = encode16(ee, k2);
              sfb = c2;
            }  // weight mode: bitwise duplicate of the primary block
            const int pb = phys_block(nb + jb, nb, ns, p.layout);
            if (live) *reinterpret_cast<uint2*>(p.codes + (int64_t)(base + 32 * r) * code_row + pb * 8) = packed;
            if (has) st[(pb >> 2) * UB + 4 * r + (pb & 3)] = live ? (uint8_t)sfb : (uint8_t)0;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
      }
    }
    return;
  }
  const int rl = (warp - npw) * 32 + lane;  // residual lane index
  const int nitems = R * ns;                // (row, outlier block) pairs per tile
  // common case (R*ns <= 32*nrw): one fixed item per lane, offsets in registers
  int fr = 0, fjb = 0;
  uint32_t foff[16];
  if (rl < nitems) { fr = rl / ns; fjb = rl - fr * ns; }
  {
    const int4* pp = reinterpret_cast<const int4*>(p.perm + 16 * fjb);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 v = __ldg(pp + q);
      foff[4 * q + 0] = (uint32_t)v.x * OSC + (uint32_t)(fr * ROWP);
      foff[4 * q + 1] = (uint32_t)v.y * OSC + (uint32_t)(fr * ROWP);
      foff[4 * q + 2] = (uint32_t)v.z * OSC + (uint32_t)(fr * ROWP);
      foff[4 * q + 3] = (uint32_t)v.w * OSC + (uint32_t)(fr * ROWP);
    }
  }
  const int fpb = phys_block(nb + fjb, nb, ns, p.layout);
  for (int j0 = 0; j0 < my_tiles; j0 += ST) {
#pragma unroll
    for (int s = 0; s < ST; ++s) {
      const int j = j0 + s;
      if (j < my_tiles) {
        mbar_wait(&ready[s], (j / ST) & 1);
        if (p.debug != 1) {
          const int base = tile_base<R>((int)blockIdx.x + j * (int)gridDim.x);
          const int nr = tile_rows<R>(base, p.rows);
          uint8_t* st = sfst + s * NU * UB;
          for (int it = rl; it < nitems; it += nrw * 32) {
            int r = fr, jb = fjb, pb = fpb;
            uint32_t off[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) off[q] = foff[q];
            if (it != rl) {  // overflow items (very large S): offsets from L1
              r = it / ns;
              jb = it - r * ns;
              pb = phys_block(nb + jb, nb, ns, p.layout);
              const int4* pp = reinterpret_cast<const int4*>(p.perm + 16 * jb);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int4 v = __ldg(pp + q);
                off[4 * q + 0] = (uint32_t)v.x * OSC + (uint32_t)(r * ROWP);
                off[4 * q + 1] = (uint32_t)v.y * OSC + (uint32_t)(r * ROWP);
                off[4 * q + 2] = (uint32_t)v.z * OSC + (uint32_t)(r * ROWP);
                off[4 * q + 3] = (uint32_t)v.w * OSC + (uint32_t)(r * ROWP);
              }
            }
            uint32_t sfb = 0;
            if (r < nr) {
              const int m = base + 32 * r;
              float z[16];
              if (SILU) {
                silu_mul_block16<SILU>(z, smem + s * SLOT, off, K * 2, stab, p.debug);
              } else {
                gather16<F16>(smem + s * SLOT, off, z);
                if (NORM) norm16(z, gam + 32 * jb, rscale[s * R + r]);
              }
              const uint32_t sf1 = e4m3_ceil_nb(__fmul_rn(absmax16(z), c6g));
              float t[16];
              uint2 packed = encode16(z, k1tab[sf1], t);
              sfb = sf1;
              if (!p.weight_mode) {
                // residual of the encoded primary in units of d1/gs, exact (Q6): e = t - v(q1);
                // stage 2 with base d1: c6 = RN(d1/6) (table), k2 = RN(d1/d2)
                float e[16];
                residual16(t, packed, e);
                const uint32_t sf2 = e4m3_ceil_nb(__fmul_rn(absmax16(e), c6tab[sf1]));
                packed = encode16(e, ratio_k(sf1, sf2, rat));
                sfb = sf2;
              }  // weight mode: bitwise duplicate of the primary block
              *reinterpret_cast<uint2*>(p.codes + (int64_t)m * code_row + pb * 8) = packed;
            }
            st[(pb >> 2) * UB + 4 * r + (pb & 3)] = (uint8_t)sfb;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
  }
}

// ------------------------------------------------------------------ offline reductions
// Column abs-max over rows (calibration).  |bf16| bit patterns order like
// their values, so the max is taken on integers (exact) and merged with an
// integer atomicMax on the float bits (non-negative floats order as ints).
// f16: the 15-bit magnitudes are IEEE fp16 (they order as integers too) -> converted to float bits at the end
ARC_DEV uint32_t mag16_to_f32_bits(uint32_t m, int f16) {
  return f16 ? __float_as_uint(__half2float(__ushort_as_half((unsigned short)m))) : m << 16;
}
__global__ void arc_calib_absmax_kernel(const uint16_t* x, int64_t rows, int K, int64_t ld, int rows_per_cta,
                                        float* chan_max, int f16) {
  const int c8 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c8 >= K) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t r1 = dmin64(rows, r0 + rows_per_cta);
  uint32_t mx[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t r = r0; r < r1; ++r) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + r * ld + c8));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mx[2 * j] = max(mx[2 * j], w[j] & 0x7FFFu);
      mx[2 * j + 1] = max(mx[2 * j + 1], (w[j] >> 16) & 0x7FFFu);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) atomicMax(reinterpret_cast<unsigned int*>(chan_max + c8 + j), mag16_to_f32_bits(mx[j], f16));
}

// max |x| over a whole matrix into *amax_bits (float bits, caller zeroes it).
__global__ void arc_absmax_all_kernel(const uint16_t* x, int64_t rows, int K, int64_t ld, unsigned int* amax_bits,
                                      int f16) {
  uint32_t mx = 0;
  const int64_t n8 = rows * (K / 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (K / 8);
    const int c = (int)(i - r * (K / 8)) * 8;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + r * ld + c));
    mx = max(mx, max(max(v.x & 0x7FFFu, (v.x >> 16) & 0x7FFFu), max(v.y & 0x7FFFu, (v.y >> 16) & 0x7FFFu)));
    mx = max(mx, max(max(v.z & 0x7FFFu, (v.z >> 16) & 0x7FFFu), max(v.w & 0x7FFFu, (v.w >> 16) & 0x7FFFu)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, mag16_to_f32_bits(mx, f16));
}

// gs = 2688 / amax (reading Q3), in place over the amax bits; amax = 0 -> 1.
__global__ void arc_finalize_scale_kernel(float* gs) {
  const float amax = *gs;
  *gs = amax > 0.0f ? __fdiv_rn(2688.0f, amax) : 1.0f;
}

// MXFP4-ARC tensor offset (reading Q25): gs = 2^-c, c = ceil(log2(RN(amax/6))) - 8, in place over the
// amax bits; amax = 0 -> 1.  Same arithmetic as arc_mx_tensor_scale on the host.
__global__ void arc_finalize_mx_scale_kernel(float* gs) {
  const float amax = *gs;
  int c = 0;
  if (amax > 0.0f) {
    int x;
    const float f = frexpf(__fdiv_rn(amax, 6.0f), &x);
    c = (f == 0.5f ? x - 1 : x) - 8;
  }
  *gs = ldexpf(1.0f, -c);
}

// Native MXFP4-ARC (reading Q25 with UE8M0's own exponent range): one thread per (row,
// physical 32-block) of the native MX format -- the App.D block map at 32-element granularity, packed E2M1
// codes and one UE8M0 byte (e + 127; an all-zero block 0) per block, Kpm = roundup(K+S, 128).  The
// thread gathers its 32 calibrated channels straight from x (L2), runs the primary stage, and for a
// residual block the exact residual stage (activations) or the bitwise duplicate (weights).
__global__ void arc_mx_native_quant_kernel(const uint16_t* __restrict__ x, int64_t rows, int K, int S, int Kpm,
                                           int64_t ldx, const int32_t* __restrict__ perm, int weight, int layout,
                                           uint8_t* __restrict__ codes, uint8_t* __restrict__ sf) {
  pdl_wait();
  if (!weight) pdl_launch_dependents();
  const int np = Kpm >> 5, nb = K >> 5, ns = S >> 5;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * np) return;
  const int64_t m = idx / np;
  const int pb = (int)(idx - m * np);
  int l = -1;
  bool res = false;
  if (layout == 0) {
    if (pb < 2 * ns) { l = pb >> 1; res = (pb & 1) != 0; }
    else if (pb < nb + ns) l = pb - ns;
  } else {
    if (pb < nb) l = pb;
    else if (pb < nb + ns) { l = pb - nb; res = true; }
  }
  uint2 pk[2] = {make_uint2(0u, 0u), make_uint2(0u, 0u)};
  uint32_t byte = 0;
  if (l >= 0) {
    float z[2][16];
    const int4* pp = reinterpret_cast<const int4*>(perm + 32 * l);
    const unsigned short* xr = x + m * ldx;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int4 c = __ldg(pp + q);
      z[q >> 2][4 * (q & 3) + 0] = bf16_bits_to_f32(__ldg(xr + c.x));
      z[q >> 2][4 * (q & 3) + 1] = bf16_bits_to_f32(__ldg(xr + c.y));
      z[q >> 2][4 * (q & 3) + 2] = bf16_bits_to_f32(__ldg(xr + c.z));
      z[q >> 2][4 * (q & 3) + 3] = bf16_bits_to_f32(__ldg(xr + c.w));
    }
    const float a = fmaxf(absmax16(z[0]), absmax16(z[1]));
    int e = 0;
    if (a != 0.0f) e = min(max(mx_ceil_exp(a), -127), 127);
    const float k = ldexpf(1.0f, -e);
    float t[2][16];
    pk[0] = encode16(z[0], k, t[0]);
    pk[1] = encode16(z[1], k, t[1]);
    byte = a != 0.0f ? (uint32_t)(e + 127) : 0u;
    if (res && !weight) {
      float ee[2][16];
      residual16(t[0], pk[0], ee[0]);
      residual16(t[1], pk[1], ee[1]);
      const float a2 = fmaxf(absmax16(ee[0]), absmax16(ee[1]));
      float k2 = 1.0f;
      byte = 0u;
      if (a != 0.0f && a2 != 0.0f) {
        const int ea = min(max(e + mx_ceil_exp(a2), -127), 127);
        k2 = ldexpf(1.0f, e - ea);
        byte = (uint32_t)(ea + 127);
      }
      pk[0] = encode16(ee[0], k2);
      pk[1] = encode16(ee[1], k2);
    }  // weights: the residual block is the bitwise duplicate of the primary
  }
  uint4* dst = reinterpret_cast<uint4*>(codes + m * (Kpm >> 1) + pb * 16);
  *dst = make_uint4(pk[0].x, pk[0].y, pk[1].x, pk[1].y);
  const int64_t rb = m >> 7;
  sf[rb * (int64_t)(np >> 2) * 512 + (pb >> 2) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4 + (pb & 3)] = (uint8_t)byte;
}

// Fig.8a comparator: plain MXFP8 of a bf16 matrix -- Eq.3's single stage per 32-block
// (E8M0 scale = smallest power of two >= RN(amax/448), E4M3 codes RN-even of x / scale), no reordering, no
// residual; K padded to Kp8 = roundup(K, 128) with zero blocks of scale 1.  One thread per (row, 32-block):
// 64 B of x in, 32 code bytes + 1 scale byte (128x4 tile layout, Kp8/32 columns) out.
__global__ void arc_mxfp8_quant_kernel(const uint16_t* __restrict__ x, int64_t rows, int K, int Kp8, int64_t ldx,
                                       uint8_t* __restrict__ codes, uint8_t* __restrict__ sf) {
  pdl_wait();
  pdl_launch_dependents();
  const int nb = Kp8 >> 5;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * nb) return;
  const int64_t m = idx / nb;
  const int b = (int)(idx - m * nb);
  uint4 out[2] = {make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)};
  int e = 0;
  if (b * 32 < K) {
    float z[32];
    const uint4* src = reinterpret_cast<const uint4*>(x + m * ldx + b * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = __ldg(src + q);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        z[8 * q + 2 * h] = __uint_as_float(w[h] << 16);
        z[8 * q + 2 * h + 1] = __uint_as_float(w[h] & 0xFFFF0000u);
      }
    }
    float a = 0.0f;
#pragma unroll
    for (int i = 0; i < 32; ++i) a = fmaxf(a, fabsf(z[i]));
    if (a > 0.0f) {
      int ex;
      const float f = frexpf(__fdiv_rn(a, 448.0f), &ex);  // RN(a/448) = f 2^ex, f in [0.5, 1)
      e = f == 0.5f ? ex - 1 : ex;                        // smallest 2^e >= RN(a/448)
    }
    const float inv = ldexpf(1.0f, -e);                   // x / 2^e is exact
    uint32_t* o = reinterpret_cast<uint32_t*>(out);
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      uint16_t lo, hi;
      asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(__fmul_rn(z[i + 1], inv)), "f"(__fmul_rn(z[i], inv)));
      asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(__fmul_rn(z[i + 3], inv)), "f"(__fmul_rn(z[i + 2], inv)));
      o[i >> 2] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(codes + m * Kp8 + b * 32);
  dst[0] = out[0];
  dst[1] = out[1];
  const int64_t rb = m >> 7;
  sf[rb * (int64_t)(nb >> 2) * 512 + (b >> 2) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4 + (b & 3)] =
      (uint8_t)(e + 127);
}

// ------------------------------------------------------------------ launchers

// Per-(kernel, threads, smem) launch configuration, computed once per process:
// the attribute calls and the occupancy query cost more host time than the
// kernel itself at decode sizes.
template <int IPT, int R, int ROWB, int ST, bool NORM, int SILU = 0, bool MX = false, bool F16 = false>
static cudaError_t launch_quant_cfg(QuantArgs a, int threads, cudaStream_t stream) {
  a.rows_per_tile = R;
  a.stages = ST;
  const size_t smem = (size_t)ST * R * (ROWB + 16) + (size_t)ST * (a.Kp / 64) * (R * 4) + 16 + (128 + 128 + 64) * 4 + 3 * ST * 8 +
                      (size_t)ST * R * 4 + (NORM ? 16 + (size_t)a.K * 2 : 0) + (SILU ? 16 + SILU_TAB * 2 : 0);
  struct Cfg { int dev, threads; size_t smem; int occ; };
  static thread_local Cfg cache[8];
  static thread_local int ncache = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int occ = 0;
  for (int i = 0; i < ncache && i < 8; ++i)
    if (cache[i].dev == dev && cache[i].threads == threads && cache[i].smem == smem) occ = cache[i].occ;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(arc_quant_kernel<IPT, R, ROWB, ST, NORM, SILU, MX, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    // the full shared-memory carveout so several CTAs' rings fit per SM
    e = cudaFuncSetAttribute(arc_quant_kernel<IPT, R, ROWB, ST, NORM, SILU, MX, F16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, arc_quant_kernel<IPT, R, ROWB, ST, NORM, SILU, MX, F16>, threads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    cache[ncache % 8] = Cfg{dev, threads, smem, occ};
    ++ncache;
  }
  const int64_t ntile = (a.rows + 127) / 128 * (128 / R);
  const int64_t grid = imin64(ntile, (int64_t)num_sms() * occ);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_quant_kernel<IPT, R, ROWB, ST, NORM, SILU, MX, F16>, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int SILU>
static cudaError_t launch_silu_cfg(QuantArgs a, int th, int ipt, int64_t rb, cudaStream_t stream) {
  if (ipt == 1) {
    if (rb <= 8192) return launch_quant_cfg<1, 4, 8192, 3, false, SILU>(a, th, stream);
    if (rb <= 16384) return launch_quant_cfg<1, 2, 16384, 3, false, SILU>(a, th, stream);
    if (rb <= 32768) return launch_quant_cfg<1, 2, 32768, 3, false, SILU>(a, th, stream);
    return launch_quant_cfg<1, 1, 65536, 3, false, SILU>(a, th, stream);
  }
  return launch_quant_cfg<2, 1, 65536, 3, false, SILU>(a, th, stream);
}

// Decode-size activations (<= 64 rows): one thread per (row m, physical block pb), gathering the
// block's 16 calibrated channels straight from x (L2) -- no staging ring, no mbarriers, one memory
// round trip between griddepcontrol.wait and the stores.  The STAGE arithmetic of arc_quant_kernel
// (Q7 op order: primary stage, residual stage of P:138 for residual blocks), bit-identical.
__global__ void __launch_bounds__(1024) arc_quant_small_kernel(QuantArgs p) {
  if (threadIdx.x == 0) qtrace(p, 0);
  const int NB = p.Kp >> 4, nb = p.K >> 4, ns = p.S >> 4;
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = it < p.rows * NB;
  const int m = live ? it / NB : 0, pb = live ? it - m * NB : 0;
  int l = -1;
  bool res = false;
  if (p.layout == 0) {  // interleaved P0 R0 P1 R1 ... (App.D)
    if (pb < 2 * ns) { l = pb >> 1; res = (pb & 1) != 0; }
    else if (pb < nb + ns) l = pb - ns;
  } else {              // contiguous [Q_X | Q_Ro]
    if (pb < nb) l = pb;
    else if (pb < nb + ns) { l = pb - nb; res = true; }
  }
  // the block's 16 channel indices: a calibration constant -- loaded before the wait when the caller
  // guarantees it was complete before the preceding kernel started (arc_linear), so only the x gathers
  // sit between griddepcontrol.wait and the stores
  int4 c[4];
  if (p.consts_ready && live && l >= 0) {
    const int4* pp = reinterpret_cast<const int4*>(p.perm + 16 * l);
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = __ldg(pp + q);
  }
  pdl_wait();
  pdl_launch_dependents();  // (after the wait: see arc_quant_kernel)
  if (threadIdx.x == 0) qtrace(p, 1);
  const unsigned short* xs = nullptr;  // this thread's row, staged (stage_rows)
  if (p.stage_rows) {
    extern __shared__ __align__(16) uint8_t qsmall_rows[];
    const int64_t it0 = (int64_t)blockIdx.x * blockDim.x;
    const int m0 = (int)(it0 / NB);
    const int m1 = (int)min(p.rows - 1, (it0 + (int64_t)blockDim.x - 1) / NB);
    const int n16 = p.K >> 3;  // 16-byte pieces per row
    uint4* dst = reinterpret_cast<uint4*>(qsmall_rows);
    for (int i = threadIdx.x; i < (m1 - m0 + 1) * n16; i += blockDim.x) {
      const int r = i / n16, j = i - r * n16;
      dst[i] = __ldg(reinterpret_cast<const uint4*>(p.x + (int64_t)(m0 + r) * p.ld) + j);
    }
    __syncthreads();
    xs = reinterpret_cast<const unsigned short*>(qsmall_rows) + (int64_t)(m - m0) * p.K;
  }
  if (!live) return;
  if (!p.consts_ready && l >= 0) {
    const int4* pp = reinterpret_cast<const int4*>(p.perm + 16 * l);
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = __ldg(pp + q);
  }
  uint2 packed = make_uint2(0u, 0u);
  uint32_t sfb = 0;
  if (l >= 0) {
    const float gs = __ldg(p.gs);
    const unsigned short* xr = reinterpret_cast<const unsigned short*>(p.x) + (int64_t)m * p.ld;
    float z[16];
    if (xs) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        z[4 * q + 0] = p.f16 ? in16_to_f32<true>(xs[c[q].x]) : bf16_bits_to_f32(xs[c[q].x]);
        z[4 * q + 1] = p.f16 ? in16_to_f32<true>(xs[c[q].y]) : bf16_bits_to_f32(xs[c[q].y]);
        z[4 * q + 2] = p.f16 ? in16_to_f32<true>(xs[c[q].z]) : bf16_bits_to_f32(xs[c[q].z]);
        z[4 * q + 3] = p.f16 ? in16_to_f32<true>(xs[c[q].w]) : bf16_bits_to_f32(xs[c[q].w]);
      }
    } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (p.f16) {
        z[4 * q + 0] = in16_to_f32<true>(__ldg(xr + c[q].x));
        z[4 * q + 1] = in16_to_f32<true>(__ldg(xr + c[q].y));
        z[4 * q + 2] = in16_to_f32<true>(__ldg(xr + c[q].z));
        z[4 * q + 3] = in16_to_f32<true>(__ldg(xr + c[q].w));
      } else {
        z[4 * q + 0] = bf16_bits_to_f32(__ldg(xr + c[q].x));
        z[4 * q + 1] = bf16_bits_to_f32(__ldg(xr + c[q].y));
        z[4 * q + 2] = bf16_bits_to_f32(__ldg(xr + c[q].z));
        z[4 * q + 3] = bf16_bits_to_f32(__ldg(xr + c[q].w));
      }
    }
    }
    const uint32_t sf1 = e4m3_ceil_nb(__fmul_rn(absmax16(z), __fdiv_rn(gs, 6.0f)));
    const float d1 = e4m3_value(sf1);
    float t[16];
    packed = encode16(z, sf1 == 0u ? 0.0f : __fdiv_rn(gs, d1), t);
    sfb = sf1;
    if (res) {
      float e[16];
      residual16(t, packed, e);
      const uint32_t sf2 = e4m3_ceil_nb(__fmul_rn(absmax16(e), __fdiv_rn(d1, 6.0f)));
      packed = encode16(e, sf2 == 0u ? 0.0f : __fdiv_rn(d1, e4m3_value(sf2)));
      sfb = sf2;
    }
  }
  *reinterpret_cast<uint2*>(p.codes + (int64_t)m * (p.Kp >> 1) + pb * 8) = packed;
  p.sf[(pb >> 2) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4 + (pb & 3)] = (uint8_t)sfb;
  if (it == 0) qtrace(p, 3);
}

cudaError_t launch_quant(const void* x, int64_t rows, int K, int64_t ld, const int32_t* perm, int S, const float* gs,
                         int layout, int weight_mode, uint8_t* codes, uint8_t* sf, cudaStream_t stream,
                         const void* gamma, float eps, int64_t up_off, int mx, int consts_ready, int f16) {
  QuantArgs a;
  a.stage_rows = 0;
  a.consts_ready = consts_ready;
  a.f16 = f16;
  // fp16 rows (ARC_FP16): the plain quantize / weight kernels; the bf16 model producers do not take them
  if (f16 && (gamma != nullptr || up_off != -1 || mx)) return cudaErrorInvalidValue;
  a.up_off = up_off;
  a.trace = trace_slot();
  a.gamma = static_cast<const uint16_t*>(gamma);
  a.eps = eps;
  a.norm = gamma != nullptr ? 1 : 0;
  a.x = static_cast<const uint16_t*>(x);
  a.rows = rows;
  a.K = K;
  a.ld = ld;
  a.perm = perm;
  a.S = S;
  a.gs = gs;
  a.layout = layout;
  a.weight_mode = weight_mode;
  a.codes = codes;
  a.sf = sf;
  a.Kp = (int)kp_of(K, S);
  static const int dbg = getenv("ARC_QUANT_DEBUG") ? atoi(getenv("ARC_QUANT_DEBUG")) : 0;
  a.debug = dbg;
  static const int bulk_env = getenv("ARC_QUANT_BULK") ? atoi(getenv("ARC_QUANT_BULK")) : -1;
  // whole-row bulk copies need 16-byte aligned rows (ld % 8 == 0 is validated) -- always true here
  a.bulk = bulk_env >= 0 ? bulk_env : 1;
  const int NB = a.Kp / 16, ns = S / 16;
  const int nprim = NB - ns;                 // primary + pad blocks per row
  const int64_t rowb = (int64_t)K * 2;
  // decode-size activations: the direct-gather kernel (ARC_QUANT_SMALL=0 keeps the ring kernel)
  static const int env_small = getenv("ARC_QUANT_SMALL") ? atoi(getenv("ARC_QUANT_SMALL")) : 1;
  if (env_small && rows <= 64 && !weight_mode && !a.norm && up_off == -1 && !mx) {
    static const int env_tpb = getenv("ARC_QSMALL_TPB") ? atoi(getenv("ARC_QSMALL_TPB")) : 0;
    int tpb = (env_tpb == 64 || env_tpb == 128 || env_tpb == 256 || env_tpb == 1024) ? env_tpb : 256;
    // staged rows: a window of tpb consecutive (row, block) items spans at most (tpb - 1) / NB + 2 rows
    // Auto: stage when the gathers are many (>= 32 rows) and the staged rows are at most twice the bytes
    // the CTA's items use (measured, LLaMA-3-8B decode step: M = 32 / 64 faster by 1-2 us, M <= 16 and
    // K = 14336 rows at 256 threads slower -- profiles/r2_decode_cluster.txt); long rows (K = 14336) are
    // staged by 1024-thread CTAs, which cover a whole row (<= 3x the bytes their items use; each 2-byte
    // gather from L2 moves a 32-byte sector).  ARC_QSMALL_STAGE=0 / 1 forces staging on / off,
    // ARC_QSMALL_WIDE=0 keeps 256-thread CTAs for long rows.
    static const int env_stage = getenv("ARC_QSMALL_STAGE") ? atoi(getenv("ARC_QSMALL_STAGE")) : -1;
    static const int env_wide = getenv("ARC_QSMALL_WIDE") ? atoi(getenv("ARC_QSMALL_WIDE")) : 1;
    auto span_bytes = [&](int t) {
      return (size_t)std::min<int64_t>(rows, (t - 1) / NB + 2) * (size_t)K * 2;
    };
    bool auto_stage = rows >= 32 && span_bytes(tpb) <= (size_t)2 * tpb * 32;
    if (rows >= 32 && !auto_stage && env_tpb == 0 && env_wide && span_bytes(1024) <= (size_t)3 * 1024 * 32) {
      tpb = 1024;
      auto_stage = true;
    }
    const size_t stage_bytes = span_bytes(tpb);
    a.stage_rows = (env_stage < 0 ? auto_stage : env_stage != 0) && stage_bytes <= 200 * 1024 ? 1 : 0;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)((rows * NB + tpb - 1) / tpb));
    cfg.blockDim = dim3(tpb);
    if (a.stage_rows) {
      cfg.dynamicSmemBytes = stage_bytes;
      static PerDeviceOnce small_attr;
      const cudaError_t ae = small_attr.run([] {
        return cudaFuncSetAttribute(arc_quant_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      });
      if (ae != cudaSuccess) return ae;
    }
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, arc_quant_small_kernel, a);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  if (up_off >= 0 || up_off == -2) {
    // SiLU-mul mode: a staged row is gate + up (4K bytes); always whole-row bulk copies.
    // up_off == -2: (g, u) pairs (SILU = 2); else up at x + up_off (SILU = 1).
    a.bulk = 1;
    const int64_t rb = 2 * rowb;
    const int R = rb <= 8192 ? 4 : rb <= 32768 ? 2 : 1;
    const int ipt2 = (nprim + 28 * 32 - 1) / (28 * 32);
    a.npw = (nprim + 32 * ipt2 - 1) / (32 * ipt2);
    a.nrw = ns == 0 ? 0 : (int)imin64(2, (R * ns + 31) / 32);
    const int th = (a.npw + a.nrw + 1) * 32;
    if (th > 1024 || rb > 65536) return cudaErrorInvalidValue;
    if (up_off == -2) return launch_silu_cfg<2>(a, th, ipt2, rb, stream);
    return launch_silu_cfg<1>(a, th, ipt2, rb, stream);
  }
  // ring configurations (rows per tile R, row slot bytes, stages), tuned on B200:
  // K <= 4096: R=4 (the residual warp gets a full 32 items per tile), 3 x 32 KB slots
  // -> 2 CTAs/SM; K <= 8192: R=2, 3 x 32 KB; K <= 16384: R=2, 3 x 64 KB (1 CTA/SM).
  // Norm mode adds R norm warps (one per row of a tile).
  int ipt = (nprim + 28 * 32 - 1) / (28 * 32);  // <= 28 primary warps
  if (ipt == 1) {
    const int R = rowb <= 8192 ? 4 : 2;
    a.npw = (nprim + 31) / 32;
    a.nrw = ns == 0 ? 0 : (int)imin64(2, (R * ns + 31) / 32);
    const int th = (a.npw + a.nrw + 1 + (a.norm ? R : 0)) * 32;
    if (th <= 1024) {
      if (a.norm) {  // gamma takes 2K bytes of shared memory: 2-stage rings above K = 8192
        if (rowb <= 8192) return launch_quant_cfg<1, 4, 8192, 3, true>(a, th, stream);
        if (rowb <= 16384) return launch_quant_cfg<1, 2, 16384, 3, true>(a, th, stream);
        return launch_quant_cfg<1, 2, 32768, 2, true>(a, th, stream);
      }
      if (mx) {
        if (rowb <= 8192) return launch_quant_cfg<1, 4, 8192, 3, false, 0, true>(a, th, stream);
        if (rowb <= 16384) return launch_quant_cfg<1, 2, 16384, 3, false, 0, true>(a, th, stream);
        return launch_quant_cfg<1, 2, 32768, 3, false, 0, true>(a, th, stream);
      }
      if (f16) {
        if (rowb <= 8192) return launch_quant_cfg<1, 4, 8192, 3, false, 0, false, true>(a, th, stream);
        if (rowb <= 16384) return launch_quant_cfg<1, 2, 16384, 3, false, 0, false, true>(a, th, stream);
        return launch_quant_cfg<1, 2, 32768, 3, false, 0, false, true>(a, th, stream);
      }
      if (rowb <= 8192) return launch_quant_cfg<1, 4, 8192, 3, false>(a, th, stream);
      if (rowb <= 16384) return launch_quant_cfg<1, 2, 16384, 3, false>(a, th, stream);
      return launch_quant_cfg<1, 2, 32768, 3, false>(a, th, stream);
    }
    ipt = 2;  // norm mode with 28 primary warps: two blocks per primary lane instead
  }
  if (ipt == 2) {
    a.npw = (nprim + 63) / 64;
    a.nrw = ns == 0 ? 0 : (int)imin64(2, (ns + 31) / 32);  // R = 1
    const int threads = (a.npw + a.nrw + 1 + (a.norm ? 1 : 0)) * 32;
    if (threads > 1024) return cudaErrorInvalidValue;
    if (a.norm) return launch_quant_cfg<2, 1, 65536, 2, true>(a, threads, stream);
    if (mx) return launch_quant_cfg<2, 1, 65536, 3, false, 0, true>(a, threads, stream);
    if (f16) return launch_quant_cfg<2, 1, 65536, 3, false, 0, false, true>(a, threads, stream);
    return launch_quant_cfg<2, 1, 65536, 3, false>(a, threads, stream);
  }
  return cudaErrorInvalidValue;  // K + S > 32768 is rejected in api.cu
}

// Standalone RMSNorm (the unfused comparison and the calibration input of a normed site):
// one warp per row, the same device functions (and so the same bits) as the fused kernel.
__global__ void __launch_bounds__(128) arc_rmsnorm_kernel(const uint16_t* x, int64_t rows, int K, int64_t ldx,
                                                          const uint16_t* gamma, float eps, uint16_t* y, int64_t ldy) {
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  for (int64_t m = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5); m < rows; m += (int64_t)gridDim.x * 4) {
    const uint8_t* row = reinterpret_cast<const uint8_t*>(x + m * ldx);
    const float sc = rms_scale_any<>(row, K, eps, lane);
    for (int c0 = lane * 8; c0 < K; c0 += 256) {
      const uint4 g = __ldg(reinterpret_cast<const uint4*>(gamma + c0));
      *reinterpret_cast<uint4*>(y + m * ldy + c0) = rms_apply8(*reinterpret_cast<const uint4*>(row + c0 * 2), g, sc);
    }
  }
}

cudaError_t launch_rmsnorm(const void* x, int64_t rows, int K, int64_t ldx, const void* gamma, float eps, void* y,
                           int64_t ldy, cudaStream_t s) {
  const int64_t grid = imax64(1, imin64((rows + 3) / 4, (int64_t)num_sms() * 16));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_rmsnorm_kernel, static_cast<const uint16_t*>(x), rows, K, ldx,
                                     static_cast<const uint16_t*>(gamma), eps, static_cast<uint16_t*>(y), ldy);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Standalone SiLU-mul (the unfused comparison and the calibration input of the down-proj site):
// 8 channels per thread, the same device function (and so the same bits) as the fused kernel.
__global__ void __launch_bounds__(256) arc_silu_mul_kernel(const uint16_t* gu, int64_t rows, int K, int64_t ld,
                                                           int64_t up_off, uint16_t* h, int64_t ldh) {
  pdl_launch_dependents();
  pdl_wait();
  const int k8 = K >> 3;
  const int64_t n = rows * k8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / k8;
    const int c = (int)(i - m * k8) * 8;
    uint4 g, u;
    if (up_off == -2) {  // (g_j, u_j) pairs: 8 channels = 32 bytes
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(gu + m * ld + 2 * c));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(gu + m * ld + 2 * c + 8));
      g = make_uint4(__byte_perm(a.x, a.y, 0x5410), __byte_perm(a.z, a.w, 0x5410), __byte_perm(b.x, b.y, 0x5410),
                     __byte_perm(b.z, b.w, 0x5410));
      u = make_uint4(__byte_perm(a.x, a.y, 0x7632), __byte_perm(a.z, a.w, 0x7632), __byte_perm(b.x, b.y, 0x7632),
                     __byte_perm(b.z, b.w, 0x7632));
    } else {
      g = __ldg(reinterpret_cast<const uint4*>(gu + m * ld + c));
      u = __ldg(reinterpret_cast<const uint4*>(gu + m * ld + up_off + c));
    }
    *reinterpret_cast<uint4*>(h + m * ldh + c) = silu_mul8(g, u);
  }
}

cudaError_t launch_silu_mul(const void* gu, int64_t rows, int K, int64_t ld, int64_t up_off, void* h, int64_t ldh,
                            cudaStream_t s) {
  const int64_t n = rows * (K / 8);
  const int64_t grid = imax64(1, imin64((n + 255) / 256, (int64_t)num_sms() * 8));
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_silu_mul_kernel, static_cast<const uint16_t*>(gu), rows, K, ld, up_off,
                                     static_cast<uint16_t*>(h), ldh);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_calib_absmax(const void* x, int64_t rows, int K, int64_t ld, float* chan_max, cudaStream_t s,
                                int f16) {
  const int threads = 128;
  const int rows_per_cta = 64;
  dim3 grid((unsigned)((K / 8 + threads - 1) / threads), (unsigned)((rows + rows_per_cta - 1) / rows_per_cta));
  arc_calib_absmax_kernel<<<grid, threads, 0, s>>>(static_cast<const uint16_t*>(x), rows, K, ld, rows_per_cta,
                                                   chan_max, f16);
  return cudaGetLastError();
}

cudaError_t launch_tensor_scale(const void* x, int64_t rows, int K, int64_t ld, float* gs_out, cudaStream_t s,
                                int mx, int f16) {
  cudaError_t e = cudaMemsetAsync(gs_out, 0, sizeof(float), s);
  if (e != cudaSuccess) return e;
  const int64_t n8 = rows * (K / 8);
  const int64_t grid = imax64(1, imin64((n8 + 255) / 256, (int64_t)num_sms() * 8));
  arc_absmax_all_kernel<<<(unsigned)grid, 256, 0, s>>>(static_cast<const uint16_t*>(x), rows, K, ld,
                                                      reinterpret_cast<unsigned int*>(gs_out), f16);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (mx) arc_finalize_mx_scale_kernel<<<1, 1, 0, s>>>(gs_out);
  else arc_finalize_scale_kernel<<<1, 1, 0, s>>>(gs_out);
  return cudaGetLastError();
}

// Probe (include/arc_probe.h): the fused kernel's SiLU stage exactly as the quantizing warps
// run it -- silu_mul_block16 over a staged 16-channel (gate, up = 1.0) row -- so tests can pin
// bf16(SiLU(g)) of the fused path against the oracle for every bf16 pattern.
__global__ void __launch_bounds__(128) probe_silu_block_kernel(const uint16_t* g, int64_t n, uint16_t* out) {
  __shared__ __align__(16) uint16_t tab[SILU_TAB];
  __shared__ __align__(16) uint8_t rows[128 * 64];
  build_silu_table(tab, threadIdx.x, blockDim.x);
  __syncthreads();
  uint8_t* row = rows + threadIdx.x * 64;  // gate bf16[16] | up bf16[16]
  uint32_t off[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) off[q] = 2u * q;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; b < n; b += (int64_t)gridDim.x * blockDim.x * 16) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      reinterpret_cast<uint16_t*>(row)[q] = b + q < n ? g[b + q] : 0;
      reinterpret_cast<uint16_t*>(row)[16 + q] = 0x3F80;  // up = 1.0: h = bf16(SiLU(g))
    }
    float z[16];
    silu_mul_block16<1>(z, row, off, 32, tab);
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (b + q < n) out[b + q] = (uint16_t)(__float_as_uint(z[q]) >> 16);
  }
}

cudaError_t launch_mx_native_quant(const void* x, int64_t rows, int K, int S, int64_t ld, const int32_t* perm,
                                   int weight, int layout, uint8_t* codes, uint8_t* sf, cudaStream_t stream) {
  const int Kpm = (K + S + 127) / 128 * 128;
  const int64_t n = rows * (Kpm / 32);
  if (n == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)((n + 127) / 128));
  cfg.blockDim = dim3(128);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_mx_native_quant_kernel, static_cast<const uint16_t*>(x), rows, K, S,
                                     Kpm, ld, perm, weight, layout, codes, sf);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_mxfp8_quant(const void* x, int64_t rows, int K, int64_t ld, uint8_t* codes, uint8_t* sf,
                               cudaStream_t stream) {
  const int Kp8 = (K + 127) / 128 * 128;
  const int64_t n = rows * (Kp8 / 32);
  if (n == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)((n + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_mxfp8_quant_kernel, static_cast<const uint16_t*>(x), rows, K, Kp8, ld,
                                     codes, sf);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace arc

extern "C" arc_status_t arc_probe_silu(const uint16_t* g, int64_t n, uint16_t* out, void* stream) {
  if (!g || !out) return ARC_ERR_NULL;
  if (n < 0) return ARC_ERR_SHAPE;
  if (!arc_device_supported()) return ARC_ERR_UNSUPPORTED;
  if (n == 0) return ARC_OK;
  const int64_t blocks = std::min<int64_t>((n + 128 * 16 - 1) / (128 * 16), 1024);
  arc::probe_silu_block_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(g, n, out);
  return cudaGetLastError() == cudaSuccess ? ARC_OK : ARC_ERR_CUDA;
}
