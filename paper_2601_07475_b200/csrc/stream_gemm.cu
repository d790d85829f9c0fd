// stream_gemm.cu -- the ARC linear at decode-size M (<= 64 tokens): a weight-streaming, stream-K
// augmented NVFP4 GEMM (Eq.2), optionally with the activation quantize (P:138,
// the fused kernel of P:164) as its own first phase.
//
// At M <= 64 the layer is bound by reading the quantized weights once (N x Kp x 9/16 bytes) from
// HBM; the FLOPs are negligible.  Design:
//  * persistent grid, one CTA per SM (G = min(units, SMs)); the work is the flat list of units
//    (128 weight rows x 256 K elements = 16 KB codes + 2 KB scales), tile-major; CTA c takes units
//    [c U / G, (c+1) U / G): every SM streams the same number of weight bytes;
//  * shared memory and TMEM are sized for TWO resident CTAs per SM (<= 113 KB, 256 TMEM columns, <= 168
//    registers): the kernel lets its dependents launch at entry, so the next layer's kernel is resident
//    while this one finishes and streams its first weight stages (weights never depend on the previous
//    kernel: every kernel that writes weights launches its dependents only at exit) -- the per-call
//    tail of one linear overlaps the start of the next;
//  * fused mode (arc_linear): after griddepcontrol.wait the epilogue warps of CTA q(kb) quantize the
//    activation blocks of 256-element K block kb (all M rows; the standalone quantize kernel's STAGE
//    arithmetic, bit-identical) into the workspace and publish them with a per-K-block ready word
//    (the launch's epoch); the producer waits only for the K blocks its units need, so no grid-wide
//    barrier sits on the path.  The last CTA to finish advances the epoch;
//  * MMA: tcgen05.mma kind::mxf4nvf4 block_scale scale_vec::4X, M = 128 (activation rows; rows >= Mt
//    hold stale shared memory and are never read back), N = 128 weight rows, K = 64, four per unit,
//    one 128-column TMEM accumulator per K segment of a tile;
//  * a tile whose K range one CTA covers is written directly (alpha * acc -> bf16 / fp32); a split
//    tile: every segment writes its fp32 partial, and the last CTA to arrive (CUTLASS-style semaphore)
//    sums the partials in segment order (deterministic) and writes Y.  Counters return to zero.
#include "arc_device.cuh"
#include "arc_internal.h"
#include "quant_dev.cuh"

#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace arc {
namespace {

constexpr int SBN = 128;                 // weight rows per unit (MMA N)
constexpr int SBK = 256;                 // K elements per unit
constexpr int SBKB = SBK / 2;            // bytes per row per unit (one 128B swizzle atom)
constexpr int SB_BYTES = SBN * SBKB;     // 16 KB
constexpr int SSF_BYTES = 4 * 512;       // 4 scale chunks (128 rows x 64 K each)
constexpr int S_MAX_STAGES = 8;
constexpr int S_SMEM_BUDGET = 113 * 1024;  // two CTAs per SM
constexpr int S_TMEM_COLS = 256;
constexpr int S_SFA_COL = 128;
constexpr int S_SFB_COL = 144;
constexpr int S_THREADS = 192;
// counter region (kGemmCounterBytes = 16 KB of u32, zero before first use): split-tile arrivals,
// quantize-ready epochs per K block, the finished-CTA count and the epoch
constexpr int CNT_TILE0 = 0, CNT_TILES = 2048;
constexpr int CNT_QRDY0 = 2048;
constexpr int CNT_DONE = 3072, CNT_EPOCH = 3073;
// E2M1 x E2M1, UE4M3 scales, K-major A/B, N = 128 at [17,23), M = 128 at [24,29)
constexpr uint32_t kIdescS = (1u << 7) | (1u << 10) | ((uint32_t)(SBN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

struct SArgs {
  int M, N, Kp, a_rows;
  int nkb, units;
  int nst, stage_bytes, a_bytes;
  const uint8_t* sfa;
  const uint8_t* sfb;
  const float* gs_x;
  const float* gs_w;
  void* y;
  int64_t ldy;
  int y_fp32;
  float* part;       // [n_tiles][maxseg][a_rows][128] fp32 partials
  unsigned* cnt;     // the counter region
  int maxseg;
  int w_early;       // stream the first stages' weights before griddepcontrol.wait
  int hold_w;        // fused: start the weight stream only once the CTA's first K block is quantized
  // fused quantize (x != nullptr): x bf16 [M][ldx], perm[K], S, layout -> a_codes / a_sf (= sfa)
  const uint16_t* x;
  int64_t ldx;
  const int32_t* perm;
  int K, S, layout;
  uint8_t* a_codes;
  uint8_t* a_sf;
  unsigned long long* trace;  // timing experiments only (env ARC_STREAM_TRACE): [grid][8] globaltimer stamps
  int debug;         // timing experiments only (ARC_STREAM_DEBUG): 1 = no MMAs
};

__device__ __forceinline__ int unit_begin(int c, const SArgs& a) {
  return (int)(((int64_t)c * a.units) / gridDim.x);
}
__device__ __forceinline__ int unit_owner(int u, const SArgs& a) {  // CTA whose range holds unit u
  return (int)((((int64_t)u + 1) * gridDim.x - 1) / a.units);
}
__device__ __forceinline__ int quant_owner(int kb, const SArgs& a) {  // CTA quantizing K block kb
  return (int)(((int64_t)kb * gridDim.x) / a.nkb);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STRACE(i) do { if (args.trace) args.trace[(size_t)blockIdx.x * 8 + (i)] = globaltimer(); } while (0)

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(unsigned* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// generic-proxy global writes <-> async-proxy (TMA) global reads
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// One (row m, physical block pb) of the augmented activation: the STAGE arithmetic of the standalone
// quantize kernel (Q7 op order; primary stage, plus the residual stage of P:138 for residual
// blocks), gathering the 16 calibrated channels of logical block l straight from x (L2).
__device__ __forceinline__ void quant_block(const SArgs& a, int m, int pb, float gs, float c6g) {
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
    const unsigned short* xr = a.x + (int64_t)m * a.ldx;
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
    const uint32_t sf1 = e4m3_ceil_nb(__fmul_rn(absmax16(z), c6g));
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
  *reinterpret_cast<uint2*>(a.a_codes + (int64_t)m * (a.Kp >> 1) + pb * 8) = packed;
  a.a_sf[(pb >> 2) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4 + (pb & 3)] = (uint8_t)sfb;
}

// Store one 32-column chunk of row m (values v[j] = alpha * acc, columns n0 + j).
__device__ __forceinline__ void store_row_chunk(const SArgs& a, int m, int n0, const float (&v)[32]) {
  if (a.y_fp32) {
    float* yr = static_cast<float*>(a.y) + (int64_t)m * a.ldy + n0;
    if (n0 + 32 <= a.N) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(yr + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < a.N) yr[j] = v[j];
    }
  } else {
    __nv_bfloat16* yr = static_cast<__nv_bfloat16*>(a.y) + (int64_t)m * a.ldy + n0;
    if (n0 + 32 <= a.N) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 w;
        uint32_t* pw = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(v[j + 2 * h], v[j + 2 * h + 1]);
          pw[h] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(yr + j) = w;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < a.N) yr[j] = __float2bfloat16_rn(v[j]);
    }
  }
}

__global__ void __launch_bounds__(S_THREADS, 2)
    arc_stream_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           SArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nst = args.nst, stage_bytes = args.stage_bytes, a_bytes = args.a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
  uint64_t* empty = full + S_MAX_STAGES;
  uint64_t* acc_full = empty + S_MAX_STAGES;
  uint64_t* acc_free = acc_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_free + 1);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_holder + 1);
  volatile uint32_t* epoch_s = reinterpret_cast<volatile uint32_t*>(tmem_holder + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int u0 = unit_begin(cta, args), u1 = unit_begin(cta + 1, args);
  const int nkb = args.nkb;
  const int kc_total = args.Kp / 64;
  const bool fused = args.x != nullptr;

  if (threadIdx.x == 0) {
    STRACE(0);
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_free, 4);  // one arrival per epilogue warp
    fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_holder, S_TMEM_COLS);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------------------------------------------------------- producer
      const uint64_t pol_w = policy_evict_first();  // weights: read once per call
      const uint64_t pol_a = policy_evict_last();   // activation tiles: re-read by every N tile
      const int n_units = u1 - u0;
      const int n_pre = min(nst, n_units);
      auto load_w = [&](int i, int u) {
        const int tile = u / nkb, kb = u - tile * nkb;
        const int nk = min(4, kc_total - kb * 4);
        uint8_t* st = smem + i * stage_bytes;
        mbar_expect_tx(&full[i], (uint32_t)(args.a_rows * SBKB + SB_BYTES + 2 * nk * 512));
        tma_load_2d(st + a_bytes, &tmB, &full[i], kb * SBKB, tile * SBN, pol_w);
        bulk_load_hint(st + a_bytes + SB_BYTES + SSF_BYTES, args.sfb + ((int64_t)tile * kc_total + kb * 4) * 512,
                       nk * 512, &full[i], pol_w);
      };
      uint64_t ready[2] = {0ull, 0ull};  // K blocks whose activation is known to be quantized (fused)
      uint32_t epoch = 0;
      auto load_a = [&](int i, int u) {
        const int kb = u % nkb;
        if (fused && !((ready[kb >> 6] >> (kb & 63)) & 1ull)) {
          // wait for CTA quant_owner(kb) to publish this launch's epoch for K block kb
          while (ld_acquire_u32(args.cnt + CNT_QRDY0 + kb) != epoch + 1u) {
          }
          fence_proxy_async_global();
          ready[kb >> 6] |= 1ull << (kb & 63);
        }
        const int nk = min(4, kc_total - kb * 4);
        uint8_t* st = smem + i * stage_bytes;
        tma_load_2d(st, &tmA, &full[i], kb * SBKB, 0, pol_a);
        bulk_load_hint(st + a_bytes + SB_BYTES, args.sfa + (int64_t)kb * 4 * 512, nk * 512, &full[i], pol_a);
      };
      if (fused && args.hold_w) {
        // hold the weight stream until the first K block this CTA needs is quantized: a full-rate weight
        // stream floods the memory queues and multiplies the latency of the quantize phase's gathers,
        // stores and ready words, which sit on every CTA's critical path
        pdl_wait();
        epoch = ld_acquire_u32(args.cnt + CNT_EPOCH);
        STRACE(1);
        const int kb0 = u0 % nkb;
        while (ld_acquire_u32(args.cnt + CNT_QRDY0 + kb0) != epoch + 1u) {
        }
        STRACE(2);
        for (int i = 0; i < n_pre; ++i) {
          load_w(i, u0 + i);
          load_a(i, u0 + i);
        }
      } else {
        // weights of the first stages: independent of the previous kernel (see the file comment)
        if (!args.w_early) pdl_wait();
        for (int i = 0; i < n_pre; ++i) load_w(i, u0 + i);
        STRACE(1);
        if (args.w_early) pdl_wait();
        if (fused) epoch = ld_acquire_u32(args.cnt + CNT_EPOCH);
        STRACE(2);
        for (int i = 0; i < n_pre; ++i) load_a(i, u0 + i);
      }
      int stage = n_pre % nst;
      uint32_t phase = n_pre == nst ? 1u : 0u;
      for (int i = n_pre; i < n_units; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        load_w(stage, u0 + i);
        load_a(stage, u0 + i);
        if (++stage == nst) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------------------------------------------------------- MMA issuer
      int stage = 0, seg = 0;
      uint32_t phase = 0;
      for (int u = u0; u < u1; ++u) {
        const int kb = u % nkb;
        const bool first = (u == u0) || kb == 0;
        const bool last = (u == u1 - 1) || kb == nkb - 1;
        if (first) {
          if (seg >= 1) mbar_wait(acc_free, (seg - 1) & 1);  // the epilogue drained the accumulator
          tc_fence_after();
        }
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (u == u0) STRACE(3);
        const int nk = min(4, kc_total - kb * 4);
        const uint32_t sA = smem_u32(smem + stage * stage_bytes);
        const uint32_t sB = sA + a_bytes;
        const uint32_t sSFA = sB + SB_BYTES;
        const uint32_t sSFB = sSFA + SSF_BYTES;
        if (args.debug != 1) {
          for (int kk = 0; kk < nk; ++kk) {
            utccp_32x128b_warpx4(tmem + S_SFA_COL + 4 * kk, smem_desc(sSFA + kk * 512, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4(tmem + S_SFB_COL + 4 * kk, smem_desc(sSFB + kk * 512, 0, 128, kLayoutSwizzleNone));
          }
          for (int kk = 0; kk < nk; ++kk) {
            const uint64_t ad = smem_desc(sA + kk * 32, 16, 1024, kLayoutSwizzle128B);
            const uint64_t bd = smem_desc(sB + kk * 32, 16, 1024, kLayoutSwizzle128B);
            mma_nvf4(tmem, ad, bd, kIdescS, (!first) || (kk != 0), tmem + S_SFA_COL + 4 * kk, tmem + S_SFB_COL + 4 * kk);
          }
        }
        tc_commit(&empty[stage]);
        if (last) {
          tc_commit(acc_full);
          ++seg;
        }
        if (++stage == nst) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    pdl_wait();
    const int t128 = threadIdx.x - 64;
    if (fused) {
      // quantize phase: this CTA's K blocks (all M rows), published with the launch's epoch
      if (t128 == 0) *epoch_s = ld_acquire_u32(args.cnt + CNT_EPOCH);
      named_bar_sync(1, 128);
      const uint32_t epoch = *epoch_s;
      const float gs = __ldg(args.gs_x);
      const float c6g = __fdiv_rn(gs, 6.0f);
      const int npb = args.Kp >> 4;
      for (int kb = (int)(((int64_t)cta * nkb + gridDim.x - 1) / gridDim.x); kb < nkb && quant_owner(kb, args) == cta;
           ++kb) {
        const int pb0 = kb * 16, npbk = min(16, npb - pb0);
        for (int it = t128; it < args.M * npbk; it += 128) quant_block(args, it / npbk, pb0 + it % npbk, gs, c6g);
        fence_proxy_async_global();  // generic writes read by other CTAs' TMA
        named_bar_sync(1, 128);
        if (t128 == 0) st_release_u32(args.cnt + CNT_QRDY0 + kb, epoch + 1u);
      }
      if (t128 == 0) STRACE(6);
    }
    const int q = warp & 3;               // TMEM lane quadrant = activation rows [32q, 32q+32)
    const int m = q * 32 + lane;
    const bool has_rows = q * 32 < args.M;
    const float alpha = __fdiv_rn(1.0f, __fmul_rn(__ldg(args.gs_x), __ldg(args.gs_w)));
    int seg = 0;
    for (int u = u0; u < u1; ++seg) {
      const int tile = u / nkb;
      const int u_end = min(u1, (tile + 1) * nkb);
      const int c_first = unit_owner(tile * nkb, args), c_last = unit_owner((tile + 1) * nkb - 1, args);
      const int nseg = c_last - c_first + 1, si = cta - c_first;
      mbar_wait(acc_full, seg & 1);
      tc_fence_after();
      if (warp == 2 && lane == 0 && u_end == u1) STRACE(4);
      const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16);
      const int n_base = tile * SBN;
      if (nseg == 1) {
        if (has_rows) {
#pragma unroll 1
          for (int c = 0; c < SBN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tacc + c * 32, r);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(__uint_as_float(r[j]), alpha);
            if (m < args.M && n_base + c * 32 < args.N) store_row_chunk(args, m, n_base + c * 32, v);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_free);
      } else {
        // split tile: publish this segment's fp32 partial (rows < M, 512 B per row; tcgen05.ld is
        // warp-collective, so the loads run warp-uniformly and only the stores are per row)
        float* slot = args.part + (((int64_t)tile * args.maxseg + si) * args.a_rows) * SBN;
        if (has_rows) {
#pragma unroll 1
          for (int c = 0; c < SBN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tacc + c * 32, r);
            tmem_ld_wait();
            if (m < args.M) {
              float* dst = slot + (int64_t)m * SBN + c * 32;
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                __stcg(reinterpret_cast<float4*>(dst + j), make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                                      __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_free);  // the accumulator is free: the next segment's MMAs may start
        // arrival (CUTLASS-style semaphore): the CTA barrier orders every epilogue thread's partial stores
        // before thread 0's acq_rel atomic at gpu scope; the last arriver's acquire + barrier make every
        // segment's partial visible to all its epilogue threads
        named_bar_sync(1, 128);
        if (t128 == 0) {
          const unsigned old = atom_add_acq_rel(args.cnt + CNT_TILE0 + tile, 1u);
          const int is_last = old == (unsigned)(nseg - 1);
          if (is_last) args.cnt[CNT_TILE0 + tile] = 0u;  // every segment has arrived: reset for the next call
          *last_flag = is_last;
        }
        named_bar_sync(1, 128);
        if (*last_flag) {
          // thread t owns columns 4(t % 32) .. +3 and rows t/32 + 4j; per batch 4 rows x up to 8 segments of
          // float4 partials are in flight, then each element is summed over the segments in order
          const int cg = t128 & 31, r0 = t128 >> 5;
          const float* pb = args.part + (int64_t)tile * args.maxseg * args.a_rows * SBN + 4 * cg;
          const bool col_ok = n_base + 4 * cg < args.N;
#pragma unroll 1
          for (int j0 = 0; 4 * j0 < args.M; j0 += 4) {
            float4 acc[4];
#pragma unroll 1
            for (int s0 = 0; s0 < nseg; s0 += 8) {
              float4 v[4][8];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int mm = r0 + 4 * (j0 + i);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  v[i][k] = (mm < args.M && s0 + k < nseg)
                                ? __ldcg(reinterpret_cast<const float4*>(pb + ((int64_t)(s0 + k) * args.a_rows + mm) * SBN))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  if (s0 + k < nseg) {
                    if (s0 + k == 0) {
                      acc[i] = v[i][k];
                    } else {
                      acc[i].x = __fadd_rn(acc[i].x, v[i][k].x);
                      acc[i].y = __fadd_rn(acc[i].y, v[i][k].y);
                      acc[i].z = __fadd_rn(acc[i].z, v[i][k].z);
                      acc[i].w = __fadd_rn(acc[i].w, v[i][k].w);
                    }
                  }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int mm = r0 + 4 * (j0 + i);
              if (mm < args.M && col_ok) {
                const float o[4] = {__fmul_rn(acc[i].x, alpha), __fmul_rn(acc[i].y, alpha), __fmul_rn(acc[i].z, alpha),
                                    __fmul_rn(acc[i].w, alpha)};
                const int64_t off = (int64_t)mm * args.ldy + n_base + 4 * cg;
                if (n_base + 4 * cg + 4 <= args.N) {
                  if (args.y_fp32) {
                    *reinterpret_cast<float4*>(static_cast<float*>(args.y) + off) = make_float4(o[0], o[1], o[2], o[3]);
                  } else {
                    __nv_bfloat162 lo = __floats2bfloat162_rn(o[0], o[1]), hi = __floats2bfloat162_rn(o[2], o[3]);
                    uint2 w;
                    w.x = *reinterpret_cast<uint32_t*>(&lo);
                    w.y = *reinterpret_cast<uint32_t*>(&hi);
                    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(args.y) + off) = w;
                  }
                } else {
                  for (int e = 0; e < 4 && n_base + 4 * cg + e < args.N; ++e) {
                    if (args.y_fp32) static_cast<float*>(args.y)[off + e] = o[e];
                    else static_cast<__nv_bfloat16*>(args.y)[off + e] = __float2bfloat16_rn(o[e]);
                  }
                }
              }
            }
          }
        }
      }
      u = u_end;
    }
    if (fused) {
      // the last CTA to finish advances the epoch (every CTA read it before this point) and resets the count
      named_bar_sync(1, 128);
      if (t128 == 0) {
        if (atom_add_acq_rel(args.cnt + CNT_DONE, 1u) == gridDim.x - 1) {
          args.cnt[CNT_DONE] = 0u;
          st_release_u32(args.cnt + CNT_EPOCH, *epoch_s + 1u);
        }
      }
    }
    if (t128 == 0) STRACE(5);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, S_TMEM_COLS);
  }
}

unsigned long long* stream_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (getenv("ARC_STREAM_TRACE") && cudaMalloc(&buf, 4096 * 8 * sizeof(unsigned long long)) != cudaSuccess)
      buf = nullptr;
  });
  return buf;
}

}  // namespace

// Probe (include/arc_probe.h): the last traced stream-K launch's per-CTA stamps.
extern "C" __attribute__((visibility("default"))) int arc_debug_stream_trace(unsigned long long* host, int max_ctas) {
  unsigned long long* b = stream_trace_buffer();
  if (!b || !host || max_ctas <= 0) return 0;
  const int n = std::min(max_ctas, 4096);
  if (cudaDeviceSynchronize() != cudaSuccess) return 0;
  if (cudaMemcpy(host, b, (size_t)n * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

StreamPlan plan_stream(int64_t M, int64_t N, int64_t Kp) {
  StreamPlan pl;
  pl.ok = M >= 1 && M <= 64;
  if (!pl.ok) return pl;
  pl.a_rows = M <= 16 ? 16 : M <= 32 ? 32 : 64;
  pl.n_tiles = (N + SBN - 1) / SBN;
  pl.nkb = (Kp + SBK - 1) / SBK;
  pl.units = pl.n_tiles * pl.nkb;
  pl.grid = (int)std::min<int64_t>(pl.units, num_sms());
  pl.maxseg = 1;
  for (int64_t t = 0; t < pl.n_tiles; ++t) {  // segments per tile = owners of its first .. last unit
    const int64_t f = t * pl.nkb, l = (t + 1) * pl.nkb - 1;
    const int64_t cf = ((f + 1) * pl.grid - 1) / pl.units, cl = ((l + 1) * pl.grid - 1) / pl.units;
    pl.maxseg = std::max<int64_t>(pl.maxseg, cl - cf + 1);
  }
  if (pl.n_tiles > CNT_TILES || pl.nkb > 128) {  // counter / ready-mask capacity
    pl.ok = false;
    return pl;
  }
  pl.part_bytes = (size_t)round_up((int64_t)pl.n_tiles * pl.maxseg * pl.a_rows * SBN * 4, 256);
  pl.cnt_bytes = kGemmCounterBytes;
  pl.ws_bytes = pl.cnt_bytes + pl.part_bytes;  // [counters | partials]
  return pl;
}

cudaError_t launch_stream_gemm(const GemmProblem& p, const StreamPlan& pl, cudaStream_t stream, const char** detail,
                               const StreamQuant* fq) {
  if (!pl.ok || p.ws == nullptr || p.cnt == nullptr || p.ws_bytes < pl.part_bytes) {
    if (detail) *detail = "stream-K workspace too small";
    return cudaErrorInvalidValue;
  }
  CUtensorMap tmA, tmB;
  if (!make_operand_map(&tmA, p.a_codes, p.M, p.Kp / 2, pl.a_rows, SBKB) ||
      !make_operand_map(&tmB, p.b_codes, p.N, p.Kp / 2, SBN, SBKB)) {
    if (detail) *detail = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  SArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.Kp = (int)p.Kp;
  a.a_rows = pl.a_rows;
  a.nkb = (int)pl.nkb;
  a.units = (int)pl.units;
  a.a_bytes = pl.a_rows * SBKB;
  a.stage_bytes = a.a_bytes + SB_BYTES + 2 * SSF_BYTES;
  static const int env_st = getenv("ARC_STREAM_STAGES") ? atoi(getenv("ARC_STREAM_STAGES")) : 0;
  a.nst = std::min(S_MAX_STAGES, (S_SMEM_BUDGET - 1024 - 256) / a.stage_bytes);
  if (env_st > 0) a.nst = std::min(a.nst, env_st);
  a.sfa = p.a_sf;
  a.sfb = p.b_sf;
  a.gs_x = p.gs_x;
  a.gs_w = p.gs_w;
  a.y = p.y;
  a.ldy = p.ldy;
  a.y_fp32 = p.y_fp32;
  a.cnt = p.cnt;
  a.part = static_cast<float*>(p.ws);
  a.maxseg = (int)pl.maxseg;
  a.w_early = fq ? 1 : p.weights_ready;
  if (fq) {
    a.x = static_cast<const uint16_t*>(fq->x);
    a.ldx = fq->ldx;
    a.perm = fq->perm;
    a.K = fq->K;
    a.S = fq->S;
    a.layout = fq->layout;
    a.a_codes = const_cast<uint8_t*>(p.a_codes);
    a.a_sf = const_cast<uint8_t*>(p.a_sf);
  }
  static const int env_hold = getenv("ARC_STREAM_HOLD") ? atoi(getenv("ARC_STREAM_HOLD")) : 0;
  a.hold_w = env_hold;
  a.trace = stream_trace_buffer();
  static const int dbg = getenv("ARC_STREAM_DEBUG") ? atoi(getenv("ARC_STREAM_DEBUG")) : 0;
  a.debug = dbg;
  const size_t smem = (size_t)a.nst * a.stage_bytes + 1024 + 256;
  static PerDeviceOnce attr_once;
  const cudaError_t ae = attr_once.run([] {
    return cudaFuncSetAttribute(arc_stream_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM_BUDGET);
  });
  if (ae != cudaSuccess) return ae;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)pl.grid);
  cfg.blockDim = dim3(S_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_stream_gemm_kernel, tmA, tmB, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace arc
