// decode.cu -- the fused ARC linear for decode-size M (M <= 128 tokens): ONE kernel per
// linear layer that
//   phase 1  quantizes the activation -- reorder, primary NVFP4 of every block, exact
//            residual of the S outlier channels and its NVFP4 re-quantization (P:138,
//            the "Fused Quantization Kernel" of P:164) -- into the workspace, the work
//            spread over every CTA of the grid;
//   phase 2  runs the augmented NVFP4 GEMM (Eq.2; tcgen05.mma kind::mxf4nvf4
//            block_scale scale_vec::4X, TMEM accumulator) over a stream-K partition of the
//            (256-feature weight tile, 256-element K block) units, so every SM streams an
//            equal share of the weight bytes -- the decode roofline (SURVEY.md §8(d):
//            HBM-bound on weights);
//   phase 3  sums the tiles split across CTAs in a fixed segment order (deterministic)
//            in the last CTA to finish each tile, and stores Y.
// The weights do not depend on the previous kernel: before griddepcontrol.wait the producer
// issues the first pipeline stages of weights and the (still idle) epilogue warps pull the
// rest of the CTA's weight range into L2 (bulk prefetch, one contiguous run per weight row),
// so the weight stream overlaps the previous kernel's tail, the quantize phase and the grid
// barrier that publishes the quantized activation (all CTAs are co-resident: one per SM).
//
// Measured on B200: correct and bit-exact, but SLOWER than the two-launch
// path (quantize kernel, then the split-K GEMM) at every decode size -- the grid barrier
// costs ~3.5 us between the quantize phase and the first MMA, more than a PDL-overlapped
// launch boundary -- so ARC_LINEAR_AUTO does not select it; ARC_LINEAR_FUSED requests it.
//
// Operand roles (measured): a tcgen05.mma costs about the same issue time
// for N = 16 as for N = 256, and each 512-byte scale chunk is one tcgen05.cp, so the weights
// go in the N = 256 slot (the most weight bytes per tensor-core instruction) and the M <= 128
// tokens in the M = 128 slot (rows >= M are TMA zero fill).
//
// Workspace (arc_linear's): [sync words | A codes | A scales | partials | tile counters].  The
// sync words (grid-barrier count and generation, 256 bytes at offset 0 of every arc_linear
// workspace) must be zero before the first use of a workspace; every call leaves the count at
// zero.  The tile counters need no initial value (CTA 0 zeroes them before the grid barrier).
#include "arc_device.cuh"
#include "arc_internal.h"
#include "quant_dev.cuh"
#include "arc_probe.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace arc {
namespace {

constexpr int FBM = 128;                       // MMA M: token rows (rows >= M are TMA zero fill)
constexpr int FBN = 256;                       // MMA N: weight rows (output features) per tile
constexpr int FBK = 256;                       // K elements per unit / pipeline stage
constexpr int FBKB = FBK / 2;                  // bytes per row per stage (one 128B swizzle atom)
constexpr int FST = 4;                         // pipeline stages
constexpr int F_A_BYTES = FBM * FBKB;          // 16 KB
constexpr int F_B_BYTES = FBN * FBKB;          // 32 KB
constexpr int F_SFA_BYTES = 4 * 512;           // 2 KB
constexpr int F_SFB_BYTES = 2 * 4 * 512;       // 4 KB
constexpr int F_STAGE = F_A_BYTES + F_B_BYTES + F_SFA_BYTES + F_SFB_BYTES;  // 54 KB
constexpr int F_THREADS = 192;                 // warp 0 producer, 1 MMA, 2-5 epilogue; 1-5 quantize in phase 1
constexpr int F_NQ = 160;                      // phase-1 quantizer threads per CTA (warps 1..5)
constexpr int F_SFA_COL = 256;                 // TMEM: accumulator [0,256), SFA 16 cols, SFB 32 cols
constexpr int F_SFB_COL = 272;
constexpr int F_SMEM = FST * F_STAGE + 1024 + 256;
constexpr uint32_t kIdescF = (1u << 7) | (1u << 10) | ((uint32_t)(FBN >> 3) << 17) | ((uint32_t)(FBM >> 4) << 24);

struct FArgs {
  const uint16_t* x;   // bf16 [M][ldx]
  int64_t ldx;
  const int32_t* perm;
  const float* gs_x;
  int M, N, K, S, Kp, layout;
  uint8_t* a_codes;    // workspace: quantized activation [M][Kp/2]
  uint8_t* a_sf;       // workspace: its scales, one 128-row tile x Kp/16
  const uint8_t* w_codes;  // weight codes [N][Kp/2] (L2 prefetch; the staged loads use the tensor map)
  const uint8_t* sfb;  // weight scales
  const float* gs_w;
  void* y;
  int64_t ldy;
  int y_fp32;
  unsigned* sync;      // [0] barrier count (zero between calls), [1] barrier generation
  unsigned* tile_cnt;  // [num_n] arrivals at each weight tile (zeroed by CTA 0 before the grid barrier)
  float* part;         // [num_n][maxseg][M][FBN] fp32 partials of split tiles
  int64_t units;       // num_n * nkb
  int maxseg;
  int debug;           // timing experiments only (env ARC_FUSED_DEBUG bits): 1 skip quantize compute,
                       // 2 skip the grid-barrier wait, 4 skip partial stores + reduction, 8 skip MMAs,
                       // 16 no L2 weight prefetch
  unsigned long long* trace;  // timing experiments only (env ARC_FUSED_TRACE): [grid][8] globaltimer stamps
};

ARC_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FTRACE(i) do { if (a.trace) a.trace[(size_t)blockIdx.x * 8 + (i)] = globaltimer(); } while (0)

ARC_DEV uint32_t ld_acquire_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
ARC_DEV uint32_t atom_add_acq_rel(unsigned* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
ARC_DEV void st_relaxed_u32(unsigned* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
ARC_DEV void st_release_u32(unsigned* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// generic-proxy global writes <-> async-proxy (TMA) global reads
ARC_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
ARC_DEV void named_bar(uint32_t id, uint32_t n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// Bulk prefetch of [p, p + bytes) into L2 (bytes a multiple of 16, p 16-byte aligned).
ARC_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// CTA owning stream-K unit u when U units are split evenly over G CTAs
// (CTA g owns [floor(gU/G), floor((g+1)U/G))).
ARC_DEV int owner_of(int64_t u, int64_t U, int G) { return (int)(((u + 1) * (int64_t)G - 1) / U); }

// One (row m, physical block pb) of the augmented activation (oracle C5 / C8):
// primary stage of logical block l, plus the residual stage for residual blocks.
ARC_DEV void quant_block(const FArgs& a, int m, int pb, float gs, float c6g) {
  const int nb = a.K >> 4, ns = a.S >> 4;
  int l = -1;
  bool res = false;
  if (a.layout == 0) {  // interleaved P0 R0 P1 R1 ... (App.D)
    if (pb < 2 * ns) { l = pb >> 1; res = (pb & 1) != 0; }
    else if (pb < nb + ns) l = pb - ns;
  } else {              // contiguous [Q_X | Q_Ro]
    if (pb < nb) l = pb;
    else if (pb < nb + ns) { l = pb - nb; res = true; }
  }
  uint2 packed = make_uint2(0u, 0u);
  uint32_t sfb = 0;
  if (l >= 0) {
    const int4* pp = reinterpret_cast<const int4*>(a.perm + 16 * l);
    const unsigned short* xr = reinterpret_cast<const unsigned short*>(a.x) + (int64_t)m * a.ldx;
    int4 c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = __ldg(pp + q);
    float z[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      z[4 * q + 0] = bf16_bits_to_f32(__ldg(xr + c[q].x));
      z[4 * q + 1] = bf16_bits_to_f32(__ldg(xr + c[q].y));
      z[4 * q + 2] = bf16_bits_to_f32(__ldg(xr + c[q].z));
      z[4 * q + 3] = bf16_bits_to_f32(__ldg(xr + c[q].w));
    }
    // stage 1 (Eq.1 with the NVFP4 two-level scale; Q7 op order)
    const uint32_t sf1 = e4m3_ceil_nb(__fmul_rn(absmax16(z), c6g));
    const float d1 = e4m3_value(sf1);
    float t[16];
    packed = encode16(z, sf1 == 0u ? 0.0f : __fdiv_rn(gs, d1), t);
    sfb = sf1;
    if (res) {
      // exact residual e = t - v(q1) in units of d1/gs, stage 2 with base d1 (Q6)
      float e[16];
      residual16(t, packed, e);
      const uint32_t sf2 = e4m3_ceil_nb(__fmul_rn(absmax16(e), __fdiv_rn(d1, 6.0f)));
      packed = encode16(e, sf2 == 0u ? 0.0f : __fdiv_rn(d1, e4m3_value(sf2)));
      sfb = sf2;
    }
  }
  *reinterpret_cast<uint2*>(a.a_codes + (int64_t)m * (a.Kp >> 1) + pb * 8) = packed;
  a.a_sf[(pb >> 2) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4 + (pb & 3)] = (uint8_t)sfb;
}

// 4 consecutive outputs of row m starting at column n (n % 4 == 0), clipped at N
ARC_DEV void store_y4(const FArgs& a, int m, int n, float4 v) {
  const float vv[4] = {v.x, v.y, v.z, v.w};
  if (a.y_fp32) {
    float* yr = static_cast<float*>(a.y) + (int64_t)m * a.ldy + n;
    if (n + 4 <= a.N) *reinterpret_cast<float4*>(yr) = v;
    else for (int j = 0; j < 4 && n + j < a.N; ++j) yr[j] = vv[j];
  } else {
    __nv_bfloat16* yr = static_cast<__nv_bfloat16*>(a.y) + (int64_t)m * a.ldy + n;
    if (n + 4 <= a.N) {
      __nv_bfloat162 b0 = __floats2bfloat162_rn(v.x, v.y), b1 = __floats2bfloat162_rn(v.z, v.w);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&b0);
      w.y = *reinterpret_cast<uint32_t*>(&b1);
      *reinterpret_cast<uint2*>(yr) = w;
    } else {
      for (int j = 0; j < 4 && n + j < a.N; ++j) yr[j] = __float2bfloat16_rn(vv[j]);
    }
  }
}

__global__ void __launch_bounds__(F_THREADS, 1)
    arc_linear_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            FArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FST * F_STAGE);
  uint64_t* empty = full + FST;
  uint64_t* tfull = empty + FST;
  uint64_t* buf_free = tfull + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(buf_free + 1);
  uint32_t* gen_old = tmem_holder + 1;
  uint32_t* last_flag = gen_old + 1;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = (int)gridDim.x, g = (int)blockIdx.x;
  const int M = a.M, N = a.N, Kp = a.Kp;
  const int nkb = (Kp + FBK - 1) / FBK;
  const int kc_total = Kp / 64;
  const int n_rb = (N + 127) / 128;
  const int64_t U = a.units;
  const int64_t u0 = (int64_t)g * U / G, u1 = (int64_t)(g + 1) * U / G;
  const int nu = (int)(u1 - u0);

  if (tid == 0) FTRACE(0);
  if (tid == 0) {
    for (int s = 0; s < FST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(buf_free, 4);
    fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_holder, 512);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int npre = nu < FST ? nu : FST;

  // (PDL) the weights are static: stream them before waiting on the previous kernel
  const uint64_t w_pol = policy_evict_first();  // weights are read once per call
  auto load_b = [&](int i) {
    const int64_t u = u0 + i;
    const int t = (int)(u / nkb), kb = (int)(u - (int64_t)t * nkb);
    const int nk = min(4, kc_total - kb * 4);
    const int nrb = min(2, n_rb - 2 * t);
    const int s = i % FST;
    uint8_t* sB = smem + s * F_STAGE + F_A_BYTES;
    uint8_t* sSFB = sB + F_B_BYTES + F_SFA_BYTES;
    mbar_expect_tx(&full[s], (uint32_t)(F_A_BYTES + F_B_BYTES + nk * 512 * (1 + nrb)));
    tma_load_2d(sB, &tmB, &full[s], kb * FBKB, t * FBN, w_pol);
    for (int rb = 0; rb < nrb; ++rb)
      bulk_load(sSFB + rb * 2048, a.sfb + ((int64_t)(2 * t + rb) * kc_total + kb * 4) * 512, nk * 512, &full[s]);
  };
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < npre; ++i) load_b(i);
  } else if (warp >= 2 && nu > npre && !(a.debug & 16)) {
    // the epilogue warps (idle until the first tile completes) pull the rest of this CTA's
    // weight range into L2: one contiguous run of (K blocks) x 128 B per weight row (sequential
    // DRAM pages) and the contiguous scale chunks of each 128-row block
    const int pt = tid - 64;  // 0..127
    const int64_t ua = u0 + npre;
    const int ta = (int)(ua / nkb), tb = (int)((u1 - 1) / nkb);
    const int64_t row_bytes = Kp / 2;
    for (int t = ta; t <= tb; ++t) {
      const int ka = t == ta ? (int)(ua - (int64_t)t * nkb) : 0;
      const int kz = t == tb ? (int)(u1 - (int64_t)t * nkb) : nkb;  // exclusive
      const int64_t b0 = (int64_t)ka * FBKB, b1 = std::min<int64_t>((int64_t)kz * FBKB, row_bytes);
      const int rows = min(FBN, N - t * FBN);
      for (int r = pt; r < rows; r += 128)
        prefetch_l2(a.w_codes + (int64_t)(t * FBN + r) * row_bytes + b0, (uint32_t)(b1 - b0));
      if (pt < min(2, n_rb - 2 * t)) {
        const int c0 = ka * 4, c1 = min(kz * 4, kc_total);
        prefetch_l2(a.sfb + ((int64_t)(2 * t + pt) * kc_total + c0) * 512, (uint32_t)(c1 - c0) * 512u);
      }
    }
  }
  if (tid == 0) FTRACE(1);
  pdl_wait();
  if (tid == 0) FTRACE(2);
  if (tid == 0) *gen_old = ld_acquire_u32(&a.sync[1]);  // before any arrival of this CTA
  __syncthreads();

  if (warp >= 1) {
    // ------------------------------------------------------------ phase 1: quantize A
    const float gs = __ldg(a.gs_x);
    const float c6g = __fdiv_rn(gs, 6.0f);
    const int NB = Kp >> 4;
    const int64_t total = (int64_t)M * NB;
    for (int64_t task = (int64_t)g * F_NQ + (tid - 32); task < ((a.debug & 1) ? 0 : total); task += (int64_t)G * F_NQ) {
      const int m = (int)(task / NB);
      quant_block(a, m, (int)(task - (int64_t)m * NB), gs, c6g);
    }
    if (g == 0) {  // the split-tile counters start at zero (ordered before their use by the grid barrier)
      const int num_n = (N + FBN - 1) / FBN;
      for (int t = tid - 32; t < num_n; t += F_NQ) a.tile_cnt[t] = 0u;
    }
    fence_proxy_async_global();  // these generic writes are read by other CTAs' TMA
    __threadfence();
    named_bar(1, F_NQ);
    if (tid == 32) {
      FTRACE(3);
      // grid barrier arrival; the last CTA resets the count and publishes a new generation
      if (atom_add_acq_rel(&a.sync[0], 1u) == (uint32_t)(G - 1)) {
        st_relaxed_u32(&a.sync[0], 0u);
        st_release_u32(&a.sync[1], *gen_old + 1u);
      }
    }
  }

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- producer
      uint32_t spins = 0;
      while (!(a.debug & 2) && ld_acquire_u32(&a.sync[1]) == *gen_old)
        if (++spins > (1u << 24)) __trap();  // a missing CTA would hang the GPU: fail loudly instead
      FTRACE(4);
      fence_proxy_async_global();
      const uint64_t a_pol = policy_evict_last();  // every CTA re-reads the activation
      for (int i = 0; i < nu; ++i) {
        const int s = i % FST;
        const uint32_t ph = (uint32_t)(i / FST) & 1u;
        if (i >= npre) {
          mbar_wait(&empty[s], ph ^ 1u);
          load_b(i);
        }
        const int kb = (int)((u0 + i) % nkb);
        const int nk = min(4, kc_total - kb * 4);
        uint8_t* sA = smem + s * F_STAGE;
        uint8_t* sSFA = sA + F_A_BYTES + F_B_BYTES;
        tma_load_2d(sA, &tmA, &full[s], kb * FBKB, 0, a_pol);
        bulk_load(sSFA, a.a_sf + (int64_t)kb * 4 * 512, nk * 512, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      int seg = 0;
      for (int i = 0; i < nu; ++i) {
        const int s = i % FST;
        const uint32_t ph = (uint32_t)(i / FST) & 1u;
        const int kb = (int)((u0 + i) % nkb);
        const bool first = (i == 0) || (kb == 0);
        const bool last = (i == nu - 1) || (kb == nkb - 1);
        if (first && seg > 0) {
          mbar_wait(buf_free, (uint32_t)(seg - 1) & 1u);  // the epilogue drained the accumulator
          tc_fence_after();
        }
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (i == 0) FTRACE(5);
        const int nk = min(4, kc_total - kb * 4);
        const uint32_t sA = smem_u32(smem + s * F_STAGE);
        const uint32_t sB = sA + F_A_BYTES;
        const uint32_t sSFA = sB + F_B_BYTES;
        const uint32_t sSFB = sSFA + F_SFA_BYTES;
        for (int kk = 0; kk < nk; ++kk) {
          utccp_32x128b_warpx4(tmem + F_SFA_COL + 4 * kk, smem_desc(sSFA + kk * 512, 0, 128, kLayoutSwizzleNone));
          utccp_32x128b_warpx4(tmem + F_SFB_COL + 8 * kk, smem_desc(sSFB + kk * 512, 0, 128, kLayoutSwizzleNone));
          utccp_32x128b_warpx4(tmem + F_SFB_COL + 8 * kk + 4,
                               smem_desc(sSFB + 2048 + kk * 512, 0, 128, kLayoutSwizzleNone));
        }
        for (int kk = 0; kk < ((a.debug & 8) ? 0 : nk); ++kk) {
          const uint64_t ad = smem_desc(sA + kk * 32, 16, 1024, kLayoutSwizzle128B);
          const uint64_t bd = smem_desc(sB + kk * 32, 16, 1024, kLayoutSwizzle128B);
          mma_nvf4(tmem, ad, bd, kIdescF, (first && kk == 0) ? 0u : 1u, tmem + F_SFA_COL + 4 * kk,
                   tmem + F_SFB_COL + 8 * kk);
        }
        tc_commit(&empty[s]);
        if (last) {
          tc_commit(tfull);
          ++seg;
        }
      }
      FTRACE(6);
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const float alpha = __fdiv_rn(1.0f, __fmul_rn(__ldg(a.gs_x), __ldg(a.gs_w)));
    const int q = warp & 3;  // TMEM lane quadrant
    const int m = q * 32 + lane;
    const int et = tid - 64;  // 0..127
    if (nu > 0) {
      const int t0 = (int)(u0 / nkb), t1 = (int)((u1 - 1) / nkb);
      int seg = 0;
      for (int t = t0; t <= t1; ++t, ++seg) {
        const int f = owner_of((int64_t)t * nkb, U, G);
        const int nseg = owner_of((int64_t)(t + 1) * nkb - 1, U, G) - f + 1;
        float* slot = a.part + ((int64_t)t * a.maxseg + (g - f)) * (int64_t)M * FBN;
        mbar_wait(tfull, (uint32_t)seg & 1u);
        tc_fence_after();
        if (q * 32 < M) {
#pragma unroll 1
          for (int cc = 0; cc < FBN / 32; ++cc) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + cc * 32, r);
            tmem_ld_wait();
            const int n0 = t * FBN + cc * 32;
            if (m >= M || n0 >= N || (a.debug & 4)) continue;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 v = make_float4(__fmul_rn(__uint_as_float(r[j]), alpha),
                                           __fmul_rn(__uint_as_float(r[j + 1]), alpha),
                                           __fmul_rn(__uint_as_float(r[j + 2]), alpha),
                                           __fmul_rn(__uint_as_float(r[j + 3]), alpha));
              if (nseg > 1) *reinterpret_cast<float4*>(slot + (int64_t)m * FBN + cc * 32 + j) = v;
              else if (n0 + j < N) store_y4(a, m, n0 + j, v);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(buf_free);  // the MMA may overwrite the accumulator
        if (nseg > 1 && !(a.debug & 4)) {
          // last CTA to finish tile t sums its nseg partials in segment order (deterministic)
          __threadfence();
          named_bar(2, 128);
          if (et == 0) *last_flag = atom_add_acq_rel(&a.tile_cnt[t], 1u) == (uint32_t)(nseg - 1) ? 1u : 0u;
          named_bar(2, 128);
          if (*last_flag) {
            __threadfence();
            const float4* base = reinterpret_cast<const float4*>(a.part + (int64_t)t * a.maxseg * (int64_t)M * FBN);
            const int64_t seg4 = (int64_t)M * FBN / 4;  // float4 per segment
            // 4 float4 per thread per round; each segment's 4 loads are independent of the adds
            for (int64_t e0 = et; e0 < seg4; e0 += 4 * 128) {
              float4 acc[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                acc[j] = e0 + j * 128 < seg4 ? __ldcg(base + e0 + j * 128) : make_float4(0.f, 0.f, 0.f, 0.f);
              for (int sg = 1; sg < nseg; ++sg) {
                float4 p[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  p[j] = e0 + j * 128 < seg4 ? __ldcg(base + sg * seg4 + e0 + j * 128) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  acc[j].x = __fadd_rn(acc[j].x, p[j].x);
                  acc[j].y = __fadd_rn(acc[j].y, p[j].y);
                  acc[j].z = __fadd_rn(acc[j].z, p[j].z);
                  acc[j].w = __fadd_rn(acc[j].w, p[j].w);
                }
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int64_t e = e0 + j * 128;
                if (e < seg4) {
                  const int row = (int)(e * 4 / FBN), col = (int)(e * 4 % FBN);
                  if (t * FBN + col < N) store_y4(a, row, t * FBN + col, acc[j]);
                }
              }
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (tid == 0) FTRACE(7);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// timing experiments only: per-CTA globaltimer stamps of the last fused launch (env ARC_FUSED_TRACE)
unsigned long long* fused_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (getenv("ARC_FUSED_TRACE") && cudaMalloc(&buf, 4096 * 8 * sizeof(unsigned long long)) != cudaSuccess)
      buf = nullptr;
  });
  return buf;
}

}  // namespace

// Copies the stamps of the last traced launch (rows of 8 u64 per CTA); 0 rows when tracing is off.
extern "C" ARC_API int arc_debug_fused_trace(unsigned long long* host, int max_ctas) {
  unsigned long long* b = fused_trace_buffer();
  if (!b) return 0;
  const int n = max_ctas < 4096 ? max_ctas : 4096;
  if (cudaMemcpy(host, b, (size_t)n * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}

FusedPlan plan_fused(int64_t M, int64_t N, int64_t Kp) {
  FusedPlan pl;
  pl.ok = M >= 1 && M <= FBM;
  const int64_t num_n = (N + FBN - 1) / FBN, nkb = (Kp + FBK - 1) / FBK;
  pl.units = num_n * nkb;
  static const int min_units = getenv("ARC_FUSED_MIN_UNITS") ? std::max(1, atoi(getenv("ARC_FUSED_MIN_UNITS"))) : 1;
  int64_t G = std::min<int64_t>((int64_t)num_sms(), pl.units / min_units);
  if (G < 1) G = 1;
  pl.grid = (int)G;
  int maxseg = 1;
  auto owner = [&](int64_t u) { return ((u + 1) * G - 1) / pl.units; };
  for (int64_t t = 0; t < num_n; ++t)
    maxseg = std::max<int>(maxseg, (int)(owner((t + 1) * nkb - 1) - owner(t * nkb) + 1));
  pl.maxseg = maxseg;
  pl.a_code_bytes = (size_t)round_up(M * (Kp / 2), 256);
  pl.a_sf_bytes = (size_t)round_up(128 * (Kp / 16), 256);
  pl.part_bytes = maxseg > 1 ? (size_t)(num_n * maxseg * M * FBN * 4) : 0;
  pl.cnt_bytes = (size_t)round_up(num_n * 4, 256);
  pl.ws_bytes = pl.a_code_bytes + pl.a_sf_bytes + pl.part_bytes + pl.cnt_bytes;
  return pl;
}

cudaError_t launch_linear_fused(const FusedProblem& p, cudaStream_t stream, const char** detail) {
  const FusedPlan pl = plan_fused(p.M, p.N, p.Kp);
  if (!pl.ok || p.ws_bytes < pl.ws_bytes || p.sync == nullptr) {
    if (detail) *detail = "fused linear: M > 128 or workspace too small";
    return cudaErrorInvalidValue;
  }
  uint8_t* ws = static_cast<uint8_t*>(p.ws);
  FArgs a;
  a.x = static_cast<const uint16_t*>(p.x);
  a.ldx = p.ldx;
  a.perm = p.perm;
  a.gs_x = p.gs_x;
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.K = (int)p.K;
  a.S = (int)p.S;
  a.Kp = (int)p.Kp;
  a.layout = p.layout;
  a.sync = p.sync;
  a.a_codes = ws;
  a.a_sf = a.a_codes + pl.a_code_bytes;
  a.part = reinterpret_cast<float*>(a.a_sf + pl.a_sf_bytes);
  a.tile_cnt = reinterpret_cast<unsigned*>(a.a_sf + pl.a_sf_bytes + pl.part_bytes);
  a.w_codes = p.b_codes;
  a.sfb = p.b_sf;
  a.gs_w = p.gs_w;
  a.y = p.y;
  a.ldy = p.ldy;
  a.y_fp32 = p.y_fp32;
  a.units = pl.units;
  a.maxseg = pl.maxseg;
  static const int dbg = getenv("ARC_FUSED_DEBUG") ? atoi(getenv("ARC_FUSED_DEBUG")) : 0;
  a.debug = dbg;
  a.trace = fused_trace_buffer();
  CUtensorMap tmA, tmB;
  if (!make_operand_map(&tmA, a.a_codes, p.M, p.Kp / 2, FBM, FBKB) ||
      !make_operand_map(&tmB, p.b_codes, p.N, p.Kp / 2, FBN, FBKB)) {
    if (detail) *detail = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  static PerDeviceOnce attr_once;
  const cudaError_t attr_err = attr_once.run([] {
    return cudaFuncSetAttribute(arc_linear_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
  });
  if (attr_err != cudaSuccess) return attr_err;
  if (getenv("ARC_FUSED_VERBOSE"))
    fprintf(stderr, "arc_linear fused: M=%lld N=%lld Kp=%lld grid=%d units=%lld maxseg=%d\n", (long long)p.M,
            (long long)p.N, (long long)p.Kp, pl.grid, (long long)pl.units, pl.maxseg);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)pl.grid);
  cfg.blockDim = dim3(F_THREADS);
  cfg.dynamicSmemBytes = F_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_linear_fused_kernel, tmA, tmB, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace arc
