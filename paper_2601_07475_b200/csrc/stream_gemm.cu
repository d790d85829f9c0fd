// stream_gemm.cu -- the augmented NVFP4 GEMM (Eq.2) at decode-size M (<= 64
// tokens): a weight-streaming, stream-K kernel.
//
// At M <= 64 the GEMM is bound by reading the quantized weights once (N x Kp x 9/16 bytes) from
// HBM; the FLOPs are negligible.  Design:
//  * persistent grid, one CTA per SM; the work is the flat list of units (128 weight rows x 256 K
//    elements = 16 KB codes + 2 KB scales), tile-major (all K of a 128-row tile, then the next
//    tile); CTA c takes units [c U / G, (c+1) U / G) -- every SM streams the same number of bytes;
//  * the producer issues the weight loads of the first ring stages BEFORE griddepcontrol.wait: the
//    weights do not depend on the previous kernel (the activation quantize), so the weight stream
//    overlaps that kernel and this kernel's launch; the activation tile (Mt = 16/32/64 rows x 128 B,
//    from L2) and its scales are loaded after the wait;
//  * MMA: tcgen05.mma kind::mxf4nvf4 block_scale scale_vec::4X, M = 128 (activation rows; rows >= Mt
//    hold stale shared memory and are never read back), N = 128 weight rows, K = 64, four per unit;
//    three 128-column TMEM accumulators (one per K segment of a tile);
//  * a tile whose K range one CTA covers is written directly (alpha * acc -> bf16 / fp32); a tile
//    split across CTAs: each writes its fp32 partial, and the last CTA to finish the tile (counter)
//    sums the partials in segment order (deterministic, its own from TMEM) and writes Y.  The
//    counters are left at zero.
#include "arc_device.cuh"
#include "arc_internal.h"

#include <cuda.h>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace arc {
namespace {

constexpr int SBN = 128;                 // weight rows per unit (MMA N)
constexpr int SBK = 256;                 // K elements per unit
constexpr int SBKB = SBK / 2;            // bytes per row per unit (one 128B swizzle atom)
constexpr int S_STAGES = 7;
constexpr int SA_BYTES = 64 * SBKB;      // activation rows (<= 64): 8 KB
constexpr int SB_BYTES = SBN * SBKB;     // 16 KB
constexpr int SSF_BYTES = 4 * 512;       // 4 scale chunks (128 rows x 64 K each)
constexpr int S_STAGE = SA_BYTES + SB_BYTES + 2 * SSF_BYTES;  // 28 KB, multiple of 1024
constexpr int S_NACC = 3;                // 128-column accumulators
constexpr int S_SFA_COL = 384;
constexpr int S_SFB_COL = 400;
constexpr int S_THREADS = 192;
constexpr int S_SMEM = S_STAGES * S_STAGE + 1024 + 256;
// E2M1 x E2M1, UE4M3 scales, K-major A/B, N = 128 at [17,23), M = 128 at [24,29)
constexpr uint32_t kIdescS = (1u << 7) | (1u << 10) | ((uint32_t)(SBN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

struct SArgs {
  int M, N, Kp, a_rows;
  int n_tiles, nkb, units;
  const uint8_t* sfa;
  const uint8_t* sfb;
  const float* gs_x;
  const float* gs_w;
  void* y;
  int64_t ldy;
  int y_fp32;
  float* part;       // [n_tiles][maxseg][a_rows][128] fp32 partials
  unsigned* cnt;     // [n_tiles] arrival counters (zero before, left zero)
  int maxseg;
  int w_early;       // stream the first stages' weights before griddepcontrol.wait (GemmProblem::weights_ready)
  int debug;         // timing experiments only (ARC_STREAM_DEBUG): 1 = no MMAs
};

__device__ __forceinline__ int unit_begin(int c, const SArgs& a) {
  return (int)(((int64_t)c * a.units) / gridDim.x);
}
__device__ __forceinline__ int unit_owner(int u, const SArgs& a) {  // CTA whose range holds unit u
  return (int)((((int64_t)u + 1) * gridDim.x - 1) / a.units);
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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

__global__ void __launch_bounds__(S_THREADS, 1)
    arc_stream_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           SArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_STAGES * S_STAGE);
  uint64_t* empty = full + S_STAGES;
  uint64_t* acc_full = empty + S_STAGES;     // [S_NACC]
  uint64_t* acc_free = acc_full + S_NACC;    // [S_NACC]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_free + S_NACC);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int u0 = unit_begin(cta, args), u1 = unit_begin(cta + 1, args);
  const int nkb = args.nkb;
  const int kc_total = args.Kp / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < S_NACC; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_free[b], 4);  // one arrival per epilogue warp
    }
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

  if (warp == 0) {
    if (elect_one()) {
      // ---------------------------------------------------------------- producer
      const uint64_t pol_w = policy_evict_first();  // weights: read once per call
      const uint64_t pol_a = policy_evict_last();   // activation tiles: re-read by every N tile
      const int n_units = u1 - u0;
      const int n_pre = min(S_STAGES, n_units);
      auto load_w = [&](int i, int u) {
        const int tile = u / nkb, kb = u - tile * nkb;
        const int nk = min(4, kc_total - kb * 4);
        uint8_t* st = smem + i * S_STAGE;
        mbar_expect_tx(&full[i], (uint32_t)(args.a_rows * SBKB + SB_BYTES + 2 * nk * 512));
        tma_load_2d(st + SA_BYTES, &tmB, &full[i], kb * SBKB, tile * SBN, pol_w);
        bulk_load_hint(st + SA_BYTES + SB_BYTES + SSF_BYTES, args.sfb + ((int64_t)tile * kc_total + kb * 4) * 512,
                       nk * 512, &full[i], pol_w);
      };
      auto load_a = [&](int i, int u) {
        const int kb = u % nkb;
        const int nk = min(4, kc_total - kb * 4);
        uint8_t* st = smem + i * S_STAGE;
        tma_load_2d(st, &tmA, &full[i], kb * SBKB, 0, pol_a);
        bulk_load_hint(st + SA_BYTES + SB_BYTES, args.sfa + (int64_t)kb * 4 * 512, nk * 512, &full[i], pol_a);
      };
      // weights of the first stages: independent of the previous kernel when the caller says so
      if (!args.w_early) pdl_wait();
      for (int i = 0; i < n_pre; ++i) load_w(i, u0 + i);
      if (args.w_early) pdl_wait();
      for (int i = 0; i < n_pre; ++i) load_a(i, u0 + i);
      int stage = n_pre % S_STAGES;
      uint32_t phase = n_pre == S_STAGES ? 1u : 0u;
      for (int i = n_pre; i < n_units; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        load_w(stage, u0 + i);
        load_a(stage, u0 + i);
        if (++stage == S_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------------------------------------------------------- MMA issuer
      int stage = 0, seg = 0;
      uint32_t phase = 0;
      int b = 0;
      for (int u = u0; u < u1; ++u) {
        const int kb = u % nkb;
        const bool first = (u == u0) || kb == 0;
        const bool last = (u == u1 - 1) || kb == nkb - 1;
        if (first) {
          b = seg % S_NACC;
          if (seg >= S_NACC) mbar_wait(&acc_free[b], ((seg / S_NACC) - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const int nk = min(4, kc_total - kb * 4);
        const uint32_t sA = smem_u32(smem + stage * S_STAGE);
        const uint32_t sB = sA + SA_BYTES;
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
            mma_nvf4(tmem + b * SBN, ad, bd, kIdescS, (!first) || (kk != 0), tmem + S_SFA_COL + 4 * kk,
                     tmem + S_SFB_COL + 4 * kk);
          }
        }
        tc_commit(&empty[stage]);
        if (last) {
          tc_commit(&acc_full[b]);
          ++seg;
        }
        if (++stage == S_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    pdl_wait();
    const int q = warp & 3;               // TMEM lane quadrant = activation rows [32q, 32q+32)
    const int m = q * 32 + lane;
    const bool has_rows = q * 32 < args.M;
    const float alpha = __fdiv_rn(1.0f, __fmul_rn(__ldg(args.gs_x), __ldg(args.gs_w)));
    int seg = 0;
    for (int u = u0; u < u1; ++seg) {
      const int tile = u / nkb;
      const int u_end = min(u1, (tile + 1) * nkb);
      const int b = seg % S_NACC;
      const int c_first = unit_owner(tile * nkb, args), c_last = unit_owner((tile + 1) * nkb - 1, args);
      const int nseg = c_last - c_first + 1, si = cta - c_first;
      mbar_wait(&acc_full[b], (seg / S_NACC) & 1);
      tc_fence_after();
      const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + b * SBN;
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
      } else {
        // split tile: publish this segment's fp32 partial, the last arriver reduces in segment order
        float* slot = args.part + (((int64_t)tile * args.maxseg + si) * args.a_rows) * SBN;
        // (tcgen05.ld is warp-collective: the loads run warp-uniformly, only the stores are per row)
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
        __threadfence();
        named_bar_sync(1, 128);
        if (warp == 2 && lane == 0) {
          const unsigned old = atomicAdd(&args.cnt[tile], 1u);
          const int is_last = old == (unsigned)(nseg - 1);
          if (is_last) {
            args.cnt[tile] = 0u;  // every segment has arrived: reset for the next call
            __threadfence();
          }
          *last_flag = is_last;
        }
        named_bar_sync(1, 128);
        if (*last_flag && has_rows) {  // warp-uniform (tcgen05.ld); rows >= M compute but never store
          const float* base = args.part + ((int64_t)tile * args.maxseg * args.a_rows + m) * SBN;
#pragma unroll 1
          for (int c = 0; c < SBN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tacc + c * 32, r);
            tmem_ld_wait();
            float acc[32];
            const int mr = min(m, args.M - 1);  // rows >= M read a valid row's partials (result unused)
            for (int s = 0; s < nseg; ++s) {
              if (s == si) {
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = s == 0 ? __uint_as_float(r[j]) : __fadd_rn(acc[j], __uint_as_float(r[j]));
              } else {
                const float* src = base + ((int64_t)s * args.a_rows + (mr - m)) * SBN + c * 32;
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                  const float4 p = __ldcg(reinterpret_cast<const float4*>(src + j));
                  if (s == 0) {
                    acc[j] = p.x; acc[j + 1] = p.y; acc[j + 2] = p.z; acc[j + 3] = p.w;
                  } else {
                    acc[j] = __fadd_rn(acc[j], p.x);
                    acc[j + 1] = __fadd_rn(acc[j + 1], p.y);
                    acc[j + 2] = __fadd_rn(acc[j + 2], p.z);
                    acc[j + 3] = __fadd_rn(acc[j + 3], p.w);
                  }
                }
              }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = __fmul_rn(acc[j], alpha);
            if (m < args.M && n_base + c * 32 < args.N) store_row_chunk(args, m, n_base + c * 32, acc);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_free[b]);
      u = u_end;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

StreamPlan plan_stream(int64_t M, int64_t N, int64_t Kp) {
  StreamPlan pl;
  pl.ok = M >= 1 && M <= 64;
  if (!pl.ok) return pl;
  pl.a_rows = M <= 16 ? 16 : M <= 32 ? 32 : 64;
  pl.n_tiles = (N + SBN - 1) / SBN;
  pl.nkb = (Kp + SBK - 1) / SBK;
  pl.units = pl.n_tiles * pl.nkb;
  pl.grid = (int)std::min<int64_t>(pl.units, num_sms());
  // segments per tile = owners of its first .. last unit
  pl.maxseg = 1;
  for (int64_t t = 0; t < pl.n_tiles; ++t) {
    const int64_t f = t * pl.nkb, l = (t + 1) * pl.nkb - 1;
    const int64_t cf = ((f + 1) * pl.grid - 1) / pl.units, cl = ((l + 1) * pl.grid - 1) / pl.units;
    pl.maxseg = std::max<int64_t>(pl.maxseg, cl - cf + 1);
  }
  if (pl.n_tiles * 4 > (int64_t)kGemmCounterBytes) {  // N > 524288: no counter room
    pl.ok = false;
    return pl;
  }
  pl.part_bytes = (size_t)round_up((int64_t)pl.n_tiles * pl.maxseg * pl.a_rows * SBN * 4, 256);
  pl.cnt_bytes = kGemmCounterBytes;
  pl.ws_bytes = pl.cnt_bytes + pl.part_bytes;  // [counters | partials]
  return pl;
}

cudaError_t launch_stream_gemm(const GemmProblem& p, const StreamPlan& pl, cudaStream_t stream, const char** detail) {
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
  static PerDeviceOnce attr_once;
  const cudaError_t ae = attr_once.run([] {
    return cudaFuncSetAttribute(arc_stream_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, S_SMEM);
  });
  if (ae != cudaSuccess) return ae;
  SArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.Kp = (int)p.Kp;
  a.a_rows = pl.a_rows;
  a.n_tiles = (int)pl.n_tiles;
  a.nkb = (int)pl.nkb;
  a.units = (int)pl.units;
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
  a.w_early = p.weights_ready;
  static const int dbg = getenv("ARC_STREAM_DEBUG") ? atoi(getenv("ARC_STREAM_DEBUG")) : 0;
  a.debug = dbg;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)pl.grid);
  cfg.blockDim = dim3(S_THREADS);
  cfg.dynamicSmemBytes = S_SMEM;
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
