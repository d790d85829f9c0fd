// gemm.cu -- the augmented NVFP4 block-scaled GEMM on sm_100a tensor cores.
//
// Y[m,n] = alpha * sum_{p < Kp} e2m1(A[m,p]) e4m3(SFA[m,p/16]) e2m1(B[n,p]) e4m3(SFB[n,p/16]),
// alpha = 1/(gs_x*gs_w): Eq.2, the GEMM over the extended
// reduction dimension K+S whose FP32 accumulator sums the primary products and
// the residual corrections.
//
// Kernel: persistent, warp-specialized, one CTA per SM (smem-limited), 192
// threads.
//   warp 0 (one lane): producer.  Per K-block of 256 elements: TMA 2D loads of
//     the A tile (128 rows x 128 B) and the B tile (256 rows x 128 B), both
//     128B-swizzled, plus cp.async.bulk of the matching scale-factor chunks
//     (512 B per 128 rows x 64 K, already in the tcgen05 128x4 layout in
//     global memory, so one contiguous 2 KB copy per 128 rows), all completing
//     on the stage's mbarrier.  4-stage ring.
//   warp 1 (one lane): MMA issuer.  tcgen05.cp moves the stage's scales
//     smem -> TMEM (32x128b.warpx4), then 4 x tcgen05.mma.kind::mxf4nvf4
//     .block_scale.scale_vec::4X (M=128, N=256, K=64) accumulate into TMEM;
//     tcgen05.commit releases the smem stage and, after the last K-block,
//     signals the epilogue.
//   warps 2-5: epilogue.  tcgen05.ld 32x32b.x32 (each warp owns its TMEM lane
//     quadrant = 32 output rows), scale by alpha, convert, store.
// TMEM: 512 columns = two overlapping 256-column accumulators ([0,256) and
// [192,448)) + SFA 16 + SFB 32; the epilogue of tile t overlaps the MMAs of t+1.
#include "arc_device.cuh"
#include "arc_internal.h"
#include "quant_dev.cuh"

#include <cuda.h>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

namespace arc {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 256;           // K elements per stage
constexpr int BKB = BK / 2;       // bytes per row per stage (one 128B swizzle atom)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BKB;                // 16 KB
constexpr int B_BYTES = BN * BKB;                // 32 KB
constexpr int SFA_BYTES = (BM / 128) * 4 * 512;  // 2 KB
constexpr int SFB_BYTES = (BN / 128) * 4 * 512;  // 4 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;  // 54 KB (multiple of 1024)
constexpr int TMEM_COLS = 512;
// Two overlapping 256-column accumulators (CUTLASS-style "overlapping accum"):
// buffer 0 = [0, 256), buffer 1 = [192, 448); they share [192, 256), which the
// epilogue drains first so the next tile's MMAs can start while it drains the rest.
constexpr int ACC1_COL = 192;  // buffer b starts at column b * ACC1_COL
constexpr int OVL_CHUNKS = 2;  // 32-column chunks in the shared region
// Scale factors of one stage (4 MMAs x (SFA 4 + SFB 8) columns, 32x128b.warpx4 placement).
// (A per-MMA ring of slots with interleaved copies measured slower: each MMA then waits for
// its own tcgen05.cp; batching the stage's 12 copies ahead of its 4 MMAs exposes one wait.)
constexpr int SFA_COL = 448;
constexpr int SFB_COL = 448 + 16;
constexpr int NUM_THREADS = 192;
constexpr int EPI_STAGE_BYTES = 32 * 64;   // per epilogue warp: 32 rows x 32 bf16 (64B-swizzled)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 4 * EPI_STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
// the 1-SM kernel with ST ring stages and EW chunks (2 KB each) of epilogue staging per warp
constexpr int gemm_smem_bytes(int st, int ew) { return st * STAGE_BYTES + 4 * EPI_STAGE_BYTES * ew + 1024 + 256; }

struct Args {
  int M, N, Kp;
  const uint8_t* sfa;
  const uint8_t* sfb;
  const float* gs_x;
  const float* gs_w;
  void* y;
  int64_t ldy;
  int y_fp32;
  int nsplit;   // split-K factor (decode-size M): > 1 -> fp32 partials into ws[nsplit][M][N]
  int kbs;      // K-blocks per split
  float* ws;
  int a_rows;   // rows of the A (activation) TMA box: BM, or 16/32/64 at decode-size M (rows >= M of the
                // 128-row MMA operand then hold stale shared memory -- harmless: an output row depends
                // only on its own A row, and rows >= M are never stored)
  int swiglu;   // SwiGLU epilogue: y = h [M][N/2] bf16 from 16-row-interleaved gate/up weight rows
  int raster;   // tile order: 0 = M-tile groups fastest (the A panel stays in L2), 1 = N tiles fastest (B stays)
  // Row-parallel reduction fused into the epilogue: 1 = multimem.red.add into the NVLS
  // multicast view red_mc of every rank's fp32 Y (NVSwitch reduces), 2 = red.add into each of the red_np
  // peer-mapped fp32 Y buffers red_peer[] (NVLink P2P); the Y buffers start at zero on every rank
  int red_mode;
  int red_np;
  float* red_mc;
  float* red_peer[8];
  int mode4;   // CL = 2 kernel launched with a preferred cluster of 4 (NVFP4): a CTA in a 4-CTA cluster shares operands
              // across the cluster's two pairs -- 1: B multicast to all 4 (raster 0: the pairs hold M-tiles
              // 2p..2p+3 of one N tile), 2: A halves multicast across the pairs + B within each pair (raster 1: the
              // pairs hold N tiles n, n+1 of the same two M tiles); CTAs in fallback 2-CTA clusters run as pairs
  unsigned long long* trace;  // timing experiments only (ARC_TRACE): [cta][8] = entry, exit, cluster size, tiles
  int tail64;  // NVFP4 1-SM kernel: the last K block holds 64 or 128 K (Kp % 256): it is loaded with the 64-byte-box,
              // 64B-swizzled tail maps instead of a 128-byte box that the TMA zero-fills past Kp
  int debug;  // perf experiments only (env ARC_GEMM_DEBUG): 1 = no epilogue work, 2 = no scale copies, 3 = no stores, 4 = no TMEM loads,
              // 5 = STG stores, 6 = no TMA store, 7 = MMA ignores the accumulator-free barriers,
              // 8 = MMAs issued twice, 9 = one MMA per stage, 10 = 9 without scale copies (pair kernel; timing only)
};

// instruction descriptor: E2M1 x E2M1 (format 1), UE4M3 scales, K-major A/B,
// N>>3 at [17,23), M>>4 at [24,29).
constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
// MXFP8 (Fig.8a comparator): E4M3 x E4M3 (format 0), UE8M0 scales (bit 23), K = 32 per MMA; the SF byte ids
// (bits 29-30 for A, 4-5 for B) are or-ed in per MMA
constexpr uint32_t kIdescF8 = (1u << 23) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
// W4A8: E4M3 A (format 0) x E2M1 B (MXF8F6F4 format 5, unpacked in shared memory), UE8M0 scales
constexpr uint32_t kIdescW4A8 = kIdescF8 | (5u << 10);
// native MXFP4: E2M1 x E2M1 (MXF4 format 1), UE8M0 scales (bit 23), scale_vec::2X (32 elements per scale)
constexpr uint32_t kIdescMX = (1u << 7) | (1u << 10) | (1u << 23) | ((uint32_t)(BN >> 3) << 17) |
                              ((uint32_t)(BM >> 4) << 24);
__device__ __forceinline__ void mma_mxf4_2x(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate, uint32_t sfa_tmem, uint32_t sfb_tmem) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}
__device__ __forceinline__ void mma_mxf8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate, uint32_t sfa_tmem, uint32_t sfb_tmem) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t"
      "}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}

// fp32 reductions of 4 consecutive outputs into other ranks' Y (sys scope: the other GPUs observe them)
__device__ __forceinline__ void red_add_v4_mc(float* mc, float a, float b, float c, float d) {
  asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_1(float* p, float a) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}
// out[off .. off+3] += v (every rank's Y) through the configured reduction
__device__ __forceinline__ void reduce_out4(const Args& args, int64_t off, float a, float b, float c, float d) {
  if (args.red_mode == 1) {
    red_add_v4_mc(args.red_mc + off, a, b, c, d);
  } else {
#pragma unroll
    for (int p = 0; p < 8; ++p)  // compile-time indices: no local-memory copy of the parameter array
      if (p < args.red_np) red_add_v4(args.red_peer[p] + off, a, b, c, d);
  }
}
__device__ __forceinline__ void reduce_out1(const Args& args, int64_t off, float a) {
  if (args.red_mode == 1) {
    asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(args.red_mc + off), "f"(a) : "memory");
  } else {
#pragma unroll
    for (int p = 0; p < 8; ++p)
      if (p < args.red_np) red_add_1(args.red_peer[p] + off, a);
  }
}

// Epilogue of one output tile, run by the 4 epilogue warps: warp q drains TMEM lanes
// [32q, 32q+32) (= 32 output rows of this CTA's 128) x BN columns of accumulator buffer b,
// scales by alpha and stores.  The two chunks buffer b shares with the other buffer are read
// first and released through ovl_free; the whole buffer is released through buf_free.  In the
// 2-SM kernel (PAIR) both barriers live in the pair's leader CTA (cluster-scope remote arrivals).
template <bool PAIR, int EW = 1>
__device__ __forceinline__ void epilogue_tile(const Args& args, const CUtensorMap* tmY, uint32_t tmem, int b, int mb,
                                              int nbk, int ks, float alpha, uint64_t y_policy, uint8_t* st,
                                              uint64_t* ovl_free, uint64_t* buf_free, int warp, int lane,
                                              uint32_t leader = 0, const uint16_t* stab = nullptr) {
  const int q = warp & 3;  // TMEM lane quadrant this warp may access
  const int M = args.M, N = args.N, nsplit = args.nsplit;
  const int m = mb * BM + q * 32 + lane;
  auto release = [&](uint64_t* bar) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (PAIR) mbar_arrive_cluster(mapa_shared(bar, leader));
      else mbar_arrive(bar);
    }
  };
  uint32_t pre[OVL_CHUNKS][32];  // the shared chunks, read before anything is stored
  if (args.debug != 1 && args.debug != 4) {
#pragma unroll
    for (int k = 0; k < OVL_CHUNKS; ++k) {
      const int c = b == 0 ? BN / 32 - OVL_CHUNKS + k : k;
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + b * ACC1_COL + c * 32, pre[k]);
    }
    tmem_ld_wait();
  }
  release(ovl_free);  // next tile's MMAs may overwrite the shared columns now
#pragma unroll 1
  for (int cc = 0; cc < BN / 32; ++cc) {
    // buffer 0 drains its shared chunks (6, 7) first, buffer 1 its (0, 1)
    const int c = b == 0 ? (cc + BN / 32 - OVL_CHUNKS) % (BN / 32) : cc;
    uint32_t r[32];
    if (args.debug == 1) {
      if (cc == BN / 32 - 1) release(buf_free);
      continue;
    }
    if (args.debug == 4) {
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = 0u;
    } else if (cc < OVL_CHUNKS) {
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = cc == 0 ? pre[0][j] : pre[1][j];
    } else {
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + b * ACC1_COL + c * 32, r);
      tmem_ld_wait();
    }
    if (cc == BN / 32 - 1) release(buf_free);
    const int n0 = nbk * BN + c * 32;
    if (args.red_mode && nsplit == 1 && m < M && n0 < N) {
      // row-parallel output: add this rank's partial into every rank's Y (NVLS multicast or P2P)
      const int64_t off = (int64_t)m * args.ldy + n0;
      if (n0 + 32 <= N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          reduce_out4(args, off + j, __fmul_rn(__uint_as_float(r[j]), alpha), __fmul_rn(__uint_as_float(r[j + 1]), alpha),
                      __fmul_rn(__uint_as_float(r[j + 2]), alpha), __fmul_rn(__uint_as_float(r[j + 3]), alpha));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)  // unrolled: r[] stays in registers
          if (n0 + j < N) reduce_out1(args, off + j, __fmul_rn(__uint_as_float(r[j]), alpha));
      }
    } else if ((args.y_fp32 || nsplit > 1) && m < M && n0 < N) {
      // split-K partial rows use the stride round_up(N, 4) so the float4 stores stay 16-byte
      // aligned for any N (plan_gemm sizes the workspace with the same stride)
      float* yr = nsplit > 1 ? args.ws + ((int64_t)ks * M + m) * ((N + 3) & ~3) + n0
                             : static_cast<float*>(args.y) + (int64_t)m * args.ldy + n0;
      if (n0 + 32 <= N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(yr + j) =
              make_float4(__fmul_rn(__uint_as_float(r[j]), alpha), __fmul_rn(__uint_as_float(r[j + 1]), alpha),
                          __fmul_rn(__uint_as_float(r[j + 2]), alpha), __fmul_rn(__uint_as_float(r[j + 3]), alpha));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (n0 + j < N) yr[j] = __fmul_rn(__uint_as_float(r[j]), alpha);
      }
    }
    if (args.swiglu && nsplit == 1 && mb * BM + q * 32 < M && n0 < N) {
      // SwiGLU (Fig.5, reading Q24): chunk c holds gate channels 16(n0/32) + [0,16) in
      // its first 16 columns and the matching up channels in the last 16 (weight rows
      // interleaved offline in groups of 16).  g, u = bf16(alpha * acc) -- exactly the bf16
      // GEMM output -- then h = bf16(bf16(SiLU(g)) * u); 32 rows x 16 h staged (32 B per row)
      // and TMA-stored into h [M][N/2].
      // two 1 KB staging buffers per warp (alternating chunks): only the store issued two chunks
      // ago must have finished reading its buffer
      uint8_t* sth = st + (cc & 1) * 1024;
      if (lane == 0) bulk_wait_read1();
      __syncwarp();
      uint32_t hw[8];
      if (stab) {
        // per-CTA SiLU table (the 2-SM kernel has the shared memory for it): all 16 gate
        // patterns first, one range check, then 16 independent table loads (pipelined)
        uint32_t gw[8], uw[8];
        uint32_t tmax = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const __nv_bfloat162 g2 = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(r[2 * i]), alpha),
                                                          __fmul_rn(__uint_as_float(r[2 * i + 1]), alpha));
          const __nv_bfloat162 u2 = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(r[16 + 2 * i]), alpha),
                                                          __fmul_rn(__uint_as_float(r[16 + 2 * i + 1]), alpha));
          gw[i] = *reinterpret_cast<const uint32_t*>(&g2);
          uw[i] = *reinterpret_cast<const uint32_t*>(&u2);
          tmax = max(tmax, max((gw[i] & 0x7FFFu) - SILU_LO, ((gw[i] >> 16) & 0x7FFFu) - SILU_LO));
        }
        uint32_t sb[16];
        if (tmax < SILU_N) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            sb[2 * i] = stab[((gw[i] & 0x7FFFu) - SILU_LO) | ((gw[i] >> 4) & 0x800u)];
            sb[2 * i + 1] = stab[(((gw[i] >> 16) & 0x7FFFu) - SILU_LO) | ((gw[i] >> 20) & 0x800u)];
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            sb[2 * i] = silu_bf16_bits(gw[i] & 0xFFFFu, stab);
            sb[2 * i + 1] = silu_bf16_bits(gw[i] >> 16, stab);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(
              __fmul_rn(__uint_as_float(sb[2 * i] << 16), __uint_as_float(uw[i] << 16)),
              __fmul_rn(__uint_as_float(sb[2 * i + 1] << 16), __uint_as_float(uw[i] & 0xFFFF0000u)));
          hw[i] = *reinterpret_cast<const uint32_t*>(&h2);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const __nv_bfloat162 g2 = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(r[2 * i]), alpha),
                                                          __fmul_rn(__uint_as_float(r[2 * i + 1]), alpha));
          const __nv_bfloat162 u2 = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(r[16 + 2 * i]), alpha),
                                                          __fmul_rn(__uint_as_float(r[16 + 2 * i + 1]), alpha));
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(silu_mul1(__low2float(g2), __low2float(u2)),
                                                          silu_mul1(__high2float(g2), __high2float(u2)));
          hw[i] = *reinterpret_cast<const uint32_t*>(&h2);
        }
      }
      *reinterpret_cast<uint4*>(sth + lane * 32) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(sth + lane * 32 + 16) = make_uint4(hw[4], hw[5], hw[6], hw[7]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d_hint(tmY, sth, n0 / 2, mb * BM + q * 32, y_policy);
        bulk_commit();
      }
      continue;
    }
    if (EW == 2 && !args.y_fp32 && nsplit == 1 && mb * BM + q * 32 < M && args.debug != 3) {
      // bf16, wide stores: two column-adjacent 32x32 chunks are staged as one 32-row x 64-col tile
      // (128-byte rows, 128B swizzle: 16-byte unit U of row r at U ^ (r & 7)) and written by ONE TMA
      // store -- half the TMA store operations of the 2 KB path, which share the TMA unit with the
      // operand loads.  The drain order pairs adjacent chunks: (6,7),(0,1),(2,3),(4,5) / (0,1),...
      const int half = cc & 1;
      if (half == 0) {
        if (lane == 0) bulk_wait_read0();  // the previous pair's store finished reading the buffer
        __syncwarp();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 v;
        uint32_t* pv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(r[8 * u + 2 * h]), alpha),
                                                    __fmul_rn(__uint_as_float(r[8 * u + 2 * h + 1]), alpha));
          pv[h] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(st + lane * 128 + (((half * 4 + u) ^ (lane & 7)) << 4)) = v;
      }
      if (half == 1) {
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && n0 - 32 < N) {
          tma_store_2d_hint(tmY, st, n0 - 32, mb * BM + q * 32, y_policy);
          bulk_commit();
        }
      }
      continue;
    }
    if (!args.y_fp32 && nsplit == 1 && mb * BM + q * 32 < M && n0 < N && args.debug != 3) {
      // bf16: stage the 32x32 sub-tile in smem (64B swizzle: 16-byte unit u of row
      // r lives at unit u ^ ((r >> 1) & 3), bank-conflict-free) and TMA-store it
      // (coalesced, clipped at the M/N edges by the tensor map).
      if (lane == 0 && args.debug != 5) bulk_wait_read0();  // previous store finished reading the buffer
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 v;
        uint32_t* pv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(r[8 * u + 2 * h]), alpha),
                                                    __fmul_rn(__uint_as_float(r[8 * u + 2 * h + 1]), alpha));
          pv[h] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(st + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4)) = v;
      }
      if (args.debug == 5) {
        // coalesced STG from the staged sub-tile: lane -> (row lane/4 + 8i, 16-byte unit lane%4)
        __syncwarp();
        const int rr = lane >> 2, uu = lane & 3;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = rr + 8 * i;
          const int gm = mb * BM + q * 32 + row;
          const uint4 v = *reinterpret_cast<const uint4*>(st + row * 64 + ((uu ^ ((row >> 1) & 3)) << 4));
          if (gm < M && n0 + uu * 8 < N)
            *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.y) + (int64_t)gm * args.ldy + n0 + uu * 8) = v;
        }
        __syncwarp();
      } else {
        fence_proxy_async();
        __syncwarp();
        if (lane == 0 && args.debug != 6) {
          // Y is written once: evict-first keeps the reused A/B tiles resident in L2
          tma_store_2d_hint(tmY, st, n0, mb * BM + q * 32, y_policy);
          bulk_commit();
        }
      }
    }
  }
}

// CL = CTAs per cluster along M (1 or 2).  With CL = 2 the two CTAs compute the
// tiles (m, n) and (m+1, n): each TMA-loads HALF of the shared B tile (and its
// scale chunk) multicast into both CTAs' smem, halving L2->SM traffic for B --
// at 128x256 tiles the kernel is otherwise bound by L2 bandwidth (~6 KB/clk).
template <int CL, int ST = STAGES, int EW = 1, int FMT = 0>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    arc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmAt,
                    const __grid_constant__ CUtensorMap tmBt, const __grid_constant__ CUtensorMap tmA64,
                    const __grid_constant__ CUtensorMap tmB64, Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + ST * STAGE_BYTES;  // [4 warps][EW x 2 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_stage + 4 * EPI_STAGE_BYTES * EW);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* ovl_free = tfull + 1;
  uint64_t* buf_free = ovl_free + 1;  // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(buf_free + 2);

  unsigned long long t_entry = 0;
  if (args.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = args.M, N = args.N, Kp = args.Kp;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_mp = (num_m + CL - 1) / CL;   // M-tile groups (one per cluster step)
  const int nsplit = args.nsplit;
  const int num_tiles = num_mp * num_n * nsplit;  // cluster work items (split-K innermost)
  // CL = 2 kernel in a (preferred) 4-CTA cluster: crank 0..3, pair pp = crank / 2, rank = the CTA's row in
  // its pair; tiles are still assigned per pair (cid = blockIdx / 2), so 2- and 4-CTA clusters coexist
  const int crank = CL == 1 ? 0 : (int)cluster_ctarank();
  const int nct = CL == 1 ? 1 : (int)cluster_nctarank();
  const int rank = CL == 2 ? (crank & 1) : crank;
  const int pp = CL == 2 ? (crank >> 1) : 0;
  const int mode4 = (FMT == 0 && CL == 2 && nct == 4) ? args.mode4 : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const uint16_t mc_mask = mode4 ? (uint16_t)0xF
                                 : (uint16_t)(((1u << CL) - 1u) << (CL == 2 ? 2 * pp : 0));  // the pair / cluster
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pp));
  const uint16_t amc_mask = (uint16_t)((1u << rank) | (1u << (rank + 2)));  // mode 2: the CTAs sharing this A tile
  // FMT 0: NVFP4 (256 K per stage, 4 scale chunks of 64 K, UE4M3 per 16); FMT 1: MXFP8 (the Fig.8a
  // comparison format: 128 E4M3 K per stage, 1 scale chunk of 128 K, UE8M0 per 32).  Both move 128 B per
  // operand row per stage.
  // FMT 2: native MXFP4 (256 K per stage, 2 scale chunks of 128 K, UE8M0 per 32).
  // FMT 3: W4A8 (Fig.8a comparator): MXFP8 A x MXFP4 B on the MXFP8 instruction, B landing in
  // shared memory as one byte per E2M1 element (TMA 16U4_ALIGN16B), so the stage geometry is FMT 1's.
  constexpr bool F8 = FMT == 1 || FMT == 3;
  constexpr int KST = F8 ? 128 : BK;                // K elements per stage
  constexpr int CPS = FMT == 0 ? 4 : (F8 ? 1 : 2);  // scale chunks per stage
  const int nkb = (Kp + KST - 1) / KST;
  const int kc_total = Kp / (FMT == 0 ? 64 : 128);  // scale chunks per row block
  const int n_rb = (N + 127) / 128;        // 128-row blocks of the B scale buffer

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mode4 ? 4 : CL);  // one MMA commit from every CTA the slot's data came from / went to
    }
    mbar_init(tfull, 1);
    mbar_init(ovl_free, 4);  // one arrival per epilogue warp
    mbar_init(&buf_free[0], 4);
    mbar_init(&buf_free[1], 4);
    fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_holder, TMEM_COLS);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  pdl_wait();  // everything above overlaps the previous kernel's tail (PDL)
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------------------------------------------------------- producer
      const uint64_t pol = args.debug == 11 ? policy_evict_normal() : policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        const int ks = tile % nsplit, rest = tile / nsplit;
        const int mb = (args.raster ? rest / num_n : rest % num_mp) * CL + rank;
        const int nbk = args.raster ? rest % num_n : rest / num_mp;
        const int nrb = min(2, n_rb - 2 * nbk);   // existing 128-row scale blocks of this B tile
        const bool a_ok = mb < num_m;              // (CL = 2, odd num_m: the last rank-1 tile is empty)
        const int kb0 = ks * args.kbs, kb1 = min(nkb, kb0 + args.kbs);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);     // the slot is free in EVERY CTA of the cluster
          const int nk = min(CPS, kc_total - kb * CPS);
          uint8_t* sA = smem + stage * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          uint8_t* sSFA = sB + B_BYTES;
          uint8_t* sSFB = sSFA + SFA_BYTES;
          // FMT 3: a 16U4_ALIGN16B load counts the packed bytes (half of what lands in shared memory:
          // 8 code bytes + 8 untouched pad bytes per 16 elements; measured by arc_probe_u4_unpack)
          constexpr uint32_t B_TX = FMT == 3 ? B_BYTES / 2 : B_BYTES;
          if (FMT == 0 && args.tail64 && kb == nkb - 1) {
            // last K block of 64 / 128 K: 64-byte boxes (64B swizzle), nothing zero-filled past Kp
            mbar_expect_tx(&full[stage], (uint32_t)(args.a_rows * 64 + BN * 64 + nk * 512 * ((a_ok ? 1 : 0) + nrb)));
            tma_load_2d(sA, &tmAt, &full[stage], kb * BKB, mb * BM, pol);
            if (a_ok) bulk_load(sSFA, args.sfa + ((int64_t)mb * kc_total + kb * CPS) * 512, nk * 512, &full[stage]);
            if (CL == 1) {
              tma_load_2d(sB, &tmBt, &full[stage], kb * BKB, nbk * BN, pol);
              for (int rb = 0; rb < nrb; ++rb)
                bulk_load(sSFB + rb * 2048, args.sfb + ((int64_t)(2 * nbk + rb) * kc_total + kb * CPS) * 512, nk * 512,
                          &full[stage]);
            } else {
              tma_load_2d_mc(sB + rank * (BN / CL) * 64, &tmBt, &full[stage], kb * BKB, nbk * BN + rank * (BN / CL),
                             mc_mask, pol);
              if (CL == 2) {
                if (rank < nrb)
                  bulk_load_mc(sSFB + rank * 2048, args.sfb + ((int64_t)(2 * nbk + rank) * kc_total + kb * CPS) * 512,
                               nk * 512, &full[stage], mc_mask);
              } else {
                for (int j = rank; j < 8; j += CL) {
                  const int rb = j >> 2, kk = j & 3;
                  if (rb < nrb && kk < nk)
                    bulk_load_mc(sSFB + rb * 2048 + kk * 512,
                                 args.sfb + ((int64_t)(2 * nbk + rb) * kc_total + kb * 4 + kk) * 512, 512, &full[stage],
                                 mc_mask);
                }
              }
            }
            if (++stage == ST) { stage = 0; phase ^= 1; }
            continue;
          }
          if (FMT == 0 && CL == 2 && mode4) {
            mbar_expect_tx(&full[stage], (uint32_t)(args.a_rows * BKB + B_TX + nk * 512 * ((a_ok ? 1 : 0) + nrb)));
            if (mode4 == 1) {
              // B shared by the 4 CTAs (M tiles 2p..2p+3 of N tile nbk): a quarter each, multicast to all
              tma_load_2d(sA, &tmA, &full[stage], kb * BKB, mb * BM, pol);
              if (a_ok) bulk_load(sSFA, args.sfa + ((int64_t)mb * kc_total + kb * CPS) * 512, nk * 512, &full[stage]);
              tma_load_2d_mc(sB + crank * (B_BYTES / 4), &tmB64, &full[stage], kb * BKB, nbk * BN + crank * (BN / 4),
                             (uint16_t)0xF, pol);
              for (int j = crank; j < 8; j += 4) {  // chunk j = (row block j/4, K chunk j%4)
                const int rb = j >> 2, kk = j & 3;
                if (rb < nrb && kk < nk)
                  bulk_load_mc(sSFB + rb * 2048 + kk * 512,
                               args.sfb + ((int64_t)(2 * nbk + rb) * kc_total + kb * 4 + kk) * 512, 512, &full[stage],
                               (uint16_t)0xF);
              }
            } else {
              // pairs hold N tiles nbk, nbk+1 of the same two M tiles: the A tile (and its scales) is shared with
              // the same-row CTA of the other pair (half each), B within the pair as usual
              tma_load_2d_mc(sA + pp * (A_BYTES / 2), &tmA64, &full[stage], kb * BKB, mb * BM + pp * (BM / 2), amc_mask,
                             pol);
              if (a_ok)
                for (int kk = pp; kk < nk; kk += 2)
                  bulk_load_mc(sSFA + kk * 512, args.sfa + ((int64_t)mb * kc_total + kb * CPS + kk) * 512, 512,
                               &full[stage], amc_mask);
              tma_load_2d_mc(sB + rank * (B_BYTES / 2), &tmB, &full[stage], kb * BKB, nbk * BN + rank * (BN / 2),
                             pair_mask, pol);
              if (rank < nrb)
                bulk_load_mc(sSFB + rank * 2048, args.sfb + ((int64_t)(2 * nbk + rank) * kc_total + kb * CPS) * 512,
                             nk * 512, &full[stage], pair_mask);
            }
            if (++stage == ST) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[stage], (uint32_t)(args.a_rows * BKB + B_TX + nk * 512 * ((a_ok ? 1 : 0) + nrb)));
          tma_load_2d(sA, &tmA, &full[stage], kb * BKB, mb * BM, pol);
          if (a_ok) bulk_load(sSFA, args.sfa + ((int64_t)mb * kc_total + kb * CPS) * 512, nk * 512, &full[stage]);
          if (CL == 1) {
            tma_load_2d(sB, &tmB, &full[stage], kb * BKB, nbk * BN, pol);
            for (int rb = 0; rb < nrb; ++rb)
              bulk_load(sSFB + rb * 2048, args.sfb + ((int64_t)(2 * nbk + rb) * kc_total + kb * CPS) * 512, nk * 512,
                        &full[stage]);
          } else {
            // this CTA's 1/CL of B (BN/CL rows) and its share of the scale chunks, to every CTA of the cluster
            tma_load_2d_mc(sB + rank * (B_BYTES / CL), &tmB, &full[stage], kb * BKB, nbk * BN + rank * (BN / CL),
                           mc_mask, pol);
            if (CL == 2) {
              if (rank < nrb)
                bulk_load_mc(sSFB + rank * 2048, args.sfb + ((int64_t)(2 * nbk + rank) * kc_total + kb * CPS) * 512,
                             nk * 512, &full[stage], mc_mask);
            } else {
              for (int j = rank; j < 8; j += CL) {  // chunk j = (row block j/4, K chunk j%4)
                const int rb = j >> 2, kk = j & 3;
                if (rb < nrb && kk < nk)
                  bulk_load_mc(sSFB + rb * 2048 + kk * 512,
                               args.sfb + ((int64_t)(2 * nbk + rb) * kc_total + kb * 4 + kk) * 512, 512, &full[stage],
                               mc_mask);
              }
            }
          }
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------------------------------------------------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl, ++t) {
        const int b = t & 1;
        const int ks = tile % nsplit;
        const int kb0 = ks * args.kbs, kb1 = min(nkb, kb0 + args.kbs);
        if (t >= 1 && args.debug != 7) mbar_wait(ovl_free, (t - 1) & 1);            // shared columns drained (tile t-1)
        if (t >= 2 && args.debug != 7) mbar_wait(&buf_free[b], ((t - 2) >> 1) & 1);  // own columns drained (tile t-2)
        tc_fence_after();
        const uint32_t acc = tmem + b * ACC1_COL;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const int nk = min(CPS, kc_total - kb * CPS);
          const uint32_t sA = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sB = sA + A_BYTES;
          const uint32_t sSFA = sB + B_BYTES;
          const uint32_t sSFB = sSFA + SFA_BYTES;
          if (FMT == 2) {
            // native MXFP4: two 128-K scale chunks per stage; MMA kk (K = 64) reads bytes 2(kk%2), 2(kk%2)+1 of
            // chunk kk/2's 32-bit TMEM scale words (byte id in bits 30-31 of the address and in the SF ids)
            for (int c = 0; c < nk; ++c) {
              utccp_32x128b_warpx4(tmem + SFA_COL + 4 * c, smem_desc(sSFA + c * 512, 0, 128, kLayoutSwizzleNone));
              utccp_32x128b_warpx4(tmem + SFB_COL + 8 * c, smem_desc(sSFB + c * 512, 0, 128, kLayoutSwizzleNone));
              utccp_32x128b_warpx4(tmem + SFB_COL + 8 * c + 4,
                                   smem_desc(sSFB + 2048 + c * 512, 0, 128, kLayoutSwizzleNone));
            }
            const int nmma = min(4, (Kp - kb * KST) / 64);
            for (int kk = 0; kk < nmma; ++kk) {
              const uint32_t id = 2u * (uint32_t)(kk & 1);
              const uint64_t ad = smem_desc(sA + kk * 32, 16, 1024, kLayoutSwizzle128B);
              const uint64_t bd = smem_desc(sB + kk * 32, 16, 1024, kLayoutSwizzle128B);
              mma_mxf4_2x(acc, ad, bd, kIdescMX | (id << 29) | (id << 4), (kb != kb0) || (kk != 0),
                          (tmem + SFA_COL + 4 * (kk >> 1)) | (id << 30), (tmem + SFB_COL + 8 * (kk >> 1)) | (id << 30));
            }
            if (CL == 1) tc_commit(&empty[stage]);
            else tc_commit_mc(&empty[stage], mc_mask);
            if (++stage == ST) { stage = 0; phase ^= 1; }
            continue;
          }
          if (F8) {
            // one 128-K scale chunk per 128 rows; MMA j (K = 32) reads byte j of each row's 32-bit TMEM scale
            // word: the byte index rides in bits 30-31 of the scale address and in the descriptor's SF ids
            utccp_32x128b_warpx4(tmem + SFA_COL, smem_desc(sSFA, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4(tmem + SFB_COL, smem_desc(sSFB, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4(tmem + SFB_COL + 4, smem_desc(sSFB + 2048, 0, 128, kLayoutSwizzleNone));
            const int nmma = min(4, (Kp - kb * KST) / 32);
            for (int j = 0; j < nmma; ++j) {
              const uint64_t ad = smem_desc(sA + j * 32, 16, 1024, kLayoutSwizzle128B);
              const uint64_t bd = smem_desc(sB + j * 32, 16, 1024, kLayoutSwizzle128B);
              const uint32_t idesc = (FMT == 3 ? kIdescW4A8 : kIdescF8) | ((uint32_t)j << 29) | ((uint32_t)j << 4);
              mma_mxf8(acc, ad, bd, idesc, (kb != kb0) || (j != 0), (tmem + SFA_COL) | ((uint32_t)j << 30),
                       (tmem + SFB_COL) | ((uint32_t)j << 30));
            }
            if (CL == 1) tc_commit(&empty[stage]);
            else tc_commit_mc(&empty[stage], mc_mask);
            if (++stage == ST) { stage = 0; phase ^= 1; }
            continue;
          }
          for (int kk = 0; kk < nk && args.debug != 2; ++kk) {
            utccp_32x128b_warpx4(tmem + SFA_COL + 4 * kk, smem_desc(sSFA + kk * 512, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4(tmem + SFB_COL + 8 * kk, smem_desc(sSFB + kk * 512, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4(tmem + SFB_COL + 8 * kk + 4,
                                 smem_desc(sSFB + 2048 + kk * 512, 0, 128, kLayoutSwizzleNone));
          }
          const bool t64 = FMT == 0 && args.tail64 && kb == nkb - 1;  // 64-byte rows, 64B swizzle (see producer)
          for (int kk = 0; kk < nk; ++kk) {
            const uint64_t ad = t64 ? smem_desc(sA + kk * 32, 16, 512, kLayoutSwizzle64B)
                                    : smem_desc(sA + kk * 32, 16, 1024, kLayoutSwizzle128B);
            const uint64_t bd = t64 ? smem_desc(sB + kk * 32, 16, 512, kLayoutSwizzle64B)
                                    : smem_desc(sB + kk * 32, 16, 1024, kLayoutSwizzle128B);
            mma_nvf4(acc, ad, bd, kIdesc, (kb != kb0) || (kk != 0), tmem + SFA_COL + 4 * kk, tmem + SFB_COL + 8 * kk);
          }
          if (CL == 1) tc_commit(&empty[stage]);
          else tc_commit_mc(&empty[stage], mc_mask);  // frees the slot in both CTAs
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        tc_commit(tfull);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    const float alpha = args.gs_x ? __fdiv_rn(1.0f, __fmul_rn(__ldg(args.gs_x), __ldg(args.gs_w))) : 1.0f;
    const uint64_t y_policy = policy_evict_first();
    int t = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl, ++t) {
      const int ks = tile % nsplit, rest = tile / nsplit;
      const int mb = (args.raster ? rest / num_n : rest % num_mp) * CL + rank;
        const int nbk = args.raster ? rest % num_n : rest / num_mp;
      mbar_wait(tfull, t & 1);
      tc_fence_after();
      epilogue_tile<false, EW>(args, &tmY, tmem, t & 1, mb, nbk, ks, alpha, y_policy,
                               epi_stage + (warp - 2) * EPI_STAGE_BYTES * EW, ovl_free, &buf_free[t & 1], warp, lane);
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (args.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    args.trace[(size_t)blockIdx.x * 8 + 0] = t_entry;
    args.trace[(size_t)blockIdx.x * 8 + 1] = t;
    args.trace[(size_t)blockIdx.x * 8 + 2] = (unsigned long long)nct;
    args.trace[(size_t)blockIdx.x * 8 + 3] = (unsigned long long)cluster_ctarank();
  }
  if (CL > 1) cluster_sync();  // no CTA leaves while its peer may still multicast into it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ 2-SM (cta_group::2) kernel
// A CTA pair computes one 256 x 256 output tile with M = 256 tcgen05 MMAs issued by the
// pair's leader CTA (even rank): CTA r holds A rows [128(r&1), +128) and B rows [128(r&1), +128)
// of the tile in its own smem; the tensor cores of both SMs read both B halves, so each SM
// stages half the B bytes of the 1-SM kernel (38 KB per stage instead of 54 KB, 5 stages) and
// its shared-memory operand reads drop by a third.  Scales: each CTA holds its own 128 rows of
// SFA and all 256 rows of SFB; the leader's tcgen05.cp.cta_group::2 copies each CTA's smem
// into its own TMEM.
// CLP = CTAs per cluster (2: one pair; 4: two pairs along M computing tiles (m, n), (m+1, n)
// that share the B tile: each CTA TMA-loads a quarter of the pair-B operand and multicasts it
// to the CTA holding the same half in the other pair, halving B's L2 -> SM traffic).
// SFB is split across the cluster's CTAs and multicast to all of them.  All copies complete
// on the destination pair's leader barrier (cta_group::2 form, peer bit cleared); the
// leader's MMA commits multicast to every CTA's empty barrier (a slot is refilled only when
// every pair has consumed it) and to its pair's tfull; both CTAs' epilogues release the
// leader's accumulator barriers remotely.
constexpr int P_B_BYTES = (BN / 2) * BKB;                                     // 16 KB
constexpr int P_STAGE_BYTES = A_BYTES + P_B_BYTES + SFA_BYTES + SFB_BYTES;  // 38 KB
constexpr int p_smem_bytes(int stages) { return stages * P_STAGE_BYTES + 4 * EPI_STAGE_BYTES + 1024 + 256; }
constexpr int P_SILU_TAB_BYTES = SILU_TAB * 2;  // SwiGLU epilogue: bf16 SiLU table after the barriers
constexpr uint32_t kIdescPair = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(2 * BM >> 4) << 24);
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // shared::cluster address bit selecting the odd CTA of a pair

template <int CLP, int P_STAGES>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    arc_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB,
                         const __grid_constant__ CUtensorMap tmY, Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + P_STAGES * P_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_stage + 4 * EPI_STAGE_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;
  uint64_t* ovl_free = tfull + 1;
  uint64_t* buf_free = ovl_free + 1;  // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(buf_free + 2);
  uint16_t* stab = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(full) + 256);
  if (args.swiglu) build_silu_table(stab, threadIdx.x, NUM_THREADS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = args.M, N = args.N, Kp = args.Kp;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_mp = (num_m + CLP - 1) / CLP;  // M-tile groups (one per cluster step)
  const int nsplit = args.nsplit;
  const int num_tiles = num_mp * num_n * nsplit;
  const int rank = (int)cluster_ctarank();
  const int half = rank & 1;          // which half of the pair (A rows / B rows) this CTA holds
  const int pr = rank >> 1;           // pair index in the cluster
  const uint32_t leader = rank & ~1;  // the pair's MMA-issuing CTA
  const int cid = blockIdx.x / CLP, ncl = gridDim.x / CLP;
  const int nkb = (Kp + BK - 1) / BK;
  const int kc_total = Kp / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);            // leader: its expect_tx arrival (+ the bytes landing in the pair)
      mbar_init(&empty[s], CLP / 2);     // one MMA commit per pair of the cluster
    }
    mbar_init(tfull, 1);
    mbar_init(ovl_free, 8);  // one arrival per epilogue warp of both CTAs of the pair
    mbar_init(&buf_free[0], 8);
    mbar_init(&buf_free[1], 8);
    fence_mbar_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmSFA);
    prefetch_tmap(&tmSFB);
  }
  if (warp == 1) tmem_alloc_pair(tmem_holder, TMEM_COLS);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------------------------------------------------------- producer (every CTA)
      const uint64_t pol = args.debug == 11 ? policy_evict_normal() : policy_evict_last();
      const uint16_t mask_b = (uint16_t)(CLP == 4 ? (1u << half) | (4u << half) : 0u);
      const uint16_t mask_all = (uint16_t)((1u << CLP) - 1u);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        const int ks = tile % nsplit, rest = tile / nsplit;
        const int mb = (args.raster ? rest / num_n : rest % num_mp) * CLP + rank;
        const int nbk = args.raster ? rest % num_n : rest / num_mp;
        const int kb0 = ks * args.kbs, kb1 = min(nkb, kb0 + args.kbs);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * P_STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          uint8_t* sSFA = sB + P_B_BYTES;
          uint8_t* sSFB = sSFA + SFA_BYTES;
          const uint32_t fb = smem_u32(&full[stage]) & kPeerBitMask;
          if (half == 0) mbar_expect_tx(&full[stage], 2u * P_STAGE_BYTES);
          // full boxes always (out-of-range rows / K chunks are zero-filled and still counted)
          tma_load_2d_pair(sA, &tmA, fb, kb * BKB, mb * BM, pol);
          tma_load_3d_pair(sSFA, &tmSFA, fb, 0, kb * 4, mb, pol);
          if (CLP == 2) {
            tma_load_2d_pair(sB, &tmB, fb, kb * BKB, nbk * BN + half * (BN / 2), pol);
            tma_load_3d_pair_mc(sSFB + half * 2048, &tmSFB, fb, 0, kb * 4, nbk * 2 + half, mask_all, pol);
          } else {
            tma_load_2d_pair_mc(sB + pr * (P_B_BYTES / 2), &tmB, fb, kb * BKB, nbk * BN + half * (BN / 2) + pr * (BN / 4),
                                mask_b, pol);
            tma_load_3d_pair_mc(sSFB + half * 2048 + pr * 1024, &tmSFB, fb, 0, kb * 4 + pr * 2, nbk * 2 + half, mask_all,
                                pol);
          }
          if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (half == 0 && elect_one()) {
      // ---------------------------------------------------------------- MMA issuer (pair leader)
      const uint16_t mask_all = (uint16_t)((1u << CLP) - 1u);
      const uint16_t mask_pair = (uint16_t)(3u << leader);
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl, ++t) {
        const int b = t & 1;
        const int ks = tile % nsplit;
        const int kb0 = ks * args.kbs, kb1 = min(nkb, kb0 + args.kbs);
        if (t >= 1 && args.debug != 7) mbar_wait_cluster(ovl_free, (t - 1) & 1);
        if (t >= 2 && args.debug != 7) mbar_wait_cluster(&buf_free[b], ((t - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + b * ACC1_COL;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const int nk = min(4, kc_total - kb * 4);
          const uint32_t sA = smem_u32(smem + stage * P_STAGE_BYTES);
          const uint32_t sB = sA + A_BYTES;
          const uint32_t sSFA = sB + P_B_BYTES;
          const uint32_t sSFB = sSFA + SFA_BYTES;
          for (int kk = 0; kk < nk && args.debug != 2 && args.debug != 10; ++kk) {
            utccp_32x128b_warpx4_pair(tmem + SFA_COL + 4 * kk, smem_desc(sSFA + kk * 512, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4_pair(tmem + SFB_COL + 8 * kk, smem_desc(sSFB + kk * 512, 0, 128, kLayoutSwizzleNone));
            utccp_32x128b_warpx4_pair(tmem + SFB_COL + 8 * kk + 4,
                                      smem_desc(sSFB + 2048 + kk * 512, 0, 128, kLayoutSwizzleNone));
          }
          const int nk_mma = (args.debug == 9 || args.debug == 10) ? 1 : nk;  // 9/10: feed ceiling (one MMA per stage)
          for (int rep = 0; rep < (args.debug == 8 ? 2 : 1); ++rep)  // 8: MMA-bound check (math doubled)
            for (int kk = 0; kk < nk_mma; ++kk) {
              const uint64_t ad = smem_desc(sA + kk * 32, 16, 1024, kLayoutSwizzle128B);
              const uint64_t bd = smem_desc(sB + kk * 32, 16, 1024, kLayoutSwizzle128B);
              mma_nvf4_pair(acc, ad, bd, kIdescPair, (kb != kb0) || (kk != 0) || rep, tmem + SFA_COL + 4 * kk,
                            tmem + SFB_COL + 8 * kk);
            }
          tc_commit_pair_mc(&empty[stage], mask_all);  // the slot is free in every CTA once every pair used it
          if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair_mc(tfull, mask_pair);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (every CTA)
    const float alpha = __fdiv_rn(1.0f, __fmul_rn(__ldg(args.gs_x), __ldg(args.gs_w)));
    const uint64_t y_policy = policy_evict_first();
    int t = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl, ++t) {
      const int ks = tile % nsplit, rest = tile / nsplit;
      const int mb = (args.raster ? rest / num_n : rest % num_mp) * CLP + rank;
        const int nbk = args.raster ? rest % num_n : rest / num_mp;
      mbar_wait(tfull, t & 1);
      tc_fence_after();
      epilogue_tile<true>(args, &tmY, tmem, t & 1, mb, nbk, ks, alpha, y_policy,
                          epi_stage + (warp - 2) * EPI_STAGE_BYTES, ovl_free, &buf_free[t & 1], warp, lane, leader,
                          args.swiglu ? stab : nullptr);
    }
    if (lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while a peer's loads / MMAs / arrivals may target it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, TMEM_COLS);
  }
}

// Deterministic split-K reduction: y[m][n] = sum_ks ws[ks][m][n] in ks order.
__global__ void arc_splitk_reduce_kernel(const float* __restrict__ ws, int nsplit, int M, int N, void* y,
                                         int64_t ldy, int y_fp32, int swiglu, Args red) {
  pdl_launch_dependents();
  pdl_wait();
  const int ldp = (N + 3) & ~3;  // partial row stride (see epilogue_tile)
  const int64_t total = (int64_t)M * ldp;
  if (swiglu) {  // h[m][j] from gate column 32(j/16) + j%16 and up column +16 (see epilogue_tile)
    const int NH = N / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)M * NH;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t m = i / NH;
      const int j = (int)(i - m * NH);
      const int64_t ig = m * ldp + 32 * (j >> 4) + (j & 15), iu = ig + 16;
      float g = ws[ig], u = ws[iu];
      for (int k = 1; k < nsplit; ++k) {
        g = __fadd_rn(g, ws[(int64_t)k * total + ig]);
        u = __fadd_rn(u, ws[(int64_t)k * total + iu]);
      }
      static_cast<__nv_bfloat16*>(y)[m * ldy + j] = __float2bfloat16_rn(
          silu_mul1(__bfloat162float(__float2bfloat16_rn(g)), __bfloat162float(__float2bfloat16_rn(u))));
    }
    return;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)M * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / N, n = i - m * N, ip = m * ldp + n;
    float acc = ws[ip];
    for (int k = 1; k < nsplit; ++k) acc = __fadd_rn(acc, ws[(int64_t)k * total + ip]);
    if (red.red_mode) {  // row-parallel output: add the rank's partial into every rank's Y
      reduce_out1(red, m * ldy + n, acc);
      continue;
    }
    if (y_fp32) static_cast<float*>(y)[m * ldy + n] = acc;
    else static_cast<__nv_bfloat16*>(y)[m * ldy + n] = __float2bfloat16_rn(acc);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Packed E2M1 rows [rows][k_elems/2] loaded as one byte per element in shared memory (16 elements per
// 16-byte group, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B): the W4A8 B operand of kind::mxf8f6f4.  Box 128
// elements (128 bytes in shared memory) x box_rows, 128B swizzle.
bool make_u4_unpack_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t k_elems, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)k_elems, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(k_elems / 2)};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t row_bytes, int box_rows) {
  return make_operand_map(m, base, rows, row_bytes, box_rows, BKB);
}

// Scale factors as a 3-D u32 tensor [row blocks][Kp/64 chunks][128 words]: one 512-byte
// chunk holds the 128x4 scale tile of 128 rows x 64 K (tcgen05 layout, already in memory);
// a box of box_kc chunks x box_rb row blocks is (part of) one stage's scales (chunks past Kp
// read zeros).
bool make_sf_map(CUtensorMap* m, const uint8_t* sf, int64_t row_blocks, int64_t kc_total, int box_kc, int box_rb) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {128, (cuuint64_t)kc_total, (cuuint64_t)row_blocks};
  cuuint64_t strides[2] = {512, (cuuint64_t)(512 * kc_total)};
  cuuint32_t box[3] = {128, (cuuint32_t)box_kc, (cuuint32_t)box_rb};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint8_t*>(sf), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// box_cols 32: 64B-swizzled 32x32 sub-tiles; 16: the SwiGLU epilogue's unswizzled 32 rows x 16 h
bool make_y_map(CUtensorMap* m, void* y, int64_t rows, int64_t cols, int64_t ldy, int box_cols) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ldy * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : (box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE),
             CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool make_u4_unpack_map_probe(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t k_elems, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)k_elems, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(k_elems / 2)};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


bool make_operand_map_sw(CUtensorMap* m, const void* base, int64_t rows, int64_t row_bytes, int box_rows, int box_bytes,
                         int swizzle_bytes) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_bytes, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_operand_map(CUtensorMap* m, const void* base, int64_t rows, int64_t row_bytes, int box_rows, int box_bytes) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_bytes, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Co-resident clusters of the persistent grid (clusters of 4 may not tile every GPC's SMs).
int64_t max_clusters(int CL, bool pair) {
  if (CL == 1) return num_sms();
  static int cache[PerDeviceOnce::kMaxDev][2][5] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= PerDeviceOnce::kMaxDev) dev = 0;
  int& c = cache[dev][pair ? 1 : 0][CL];
  if (c == 0) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)(num_sms() / CL * CL));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = pair ? p_smem_bytes(5) : SMEM_BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = !pair ? (CL == 2 ? cudaOccupancyMaxActiveClusters(&n, arc_gemm_kernel<2>, &cfg)
                             : CL == 4 ? cudaOccupancyMaxActiveClusters(&n, arc_gemm_kernel<4>, &cfg)
                                       : cudaOccupancyMaxActiveClusters(&n, arc_gemm_kernel<8>, &cfg))
                    : CL == 2 ? cudaOccupancyMaxActiveClusters(&n, arc_gemm_pair_kernel<2, 5>, &cfg)
                              : cudaOccupancyMaxActiveClusters(&n, arc_gemm_pair_kernel<4, 5>, &cfg);
    if (e != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / CL;
    }
    c = n;
    if (getenv("ARC_GEMM_VERBOSE")) fprintf(stderr, "arc_gemm: CL=%d pair=%d max active clusters %d\n", CL, (int)pair, n);
  }
  return c;
}

GemmPlan plan_gemm(int64_t M, int64_t N, int64_t Kp) {
  static const int env_cl = getenv("ARC_GEMM_CL") ? atoi(getenv("ARC_GEMM_CL")) : 2;
  // The 2-SM kernel is kept selectable (ARC_GEMM_PAIR=1): on the LLaMA-3-8B shapes it measured
  // 0-8 % slower than two 1-SM CTAs sharing B by multicast.
  static const int env_pair = getenv("ARC_GEMM_PAIR") ? atoi(getenv("ARC_GEMM_PAIR")) : 0;
  static const int env_clp = getenv("ARC_GEMM_CLP") ? atoi(getenv("ARC_GEMM_CLP")) : 2;
  GemmPlan pl;
  const int64_t num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN, nkb = (Kp + BK - 1) / BK;
  // CTAs per cluster along M sharing the B tile by TMA multicast (ARC_GEMM_CL: 1, 2, 4 or 8)
  pl.CL = 1;
  for (int c = 2; c <= 8; c *= 2)
    if (env_cl >= c && num_m >= c) pl.CL = c;
  pl.pair = pl.CL == 2 && env_pair != 0;
  if (pl.pair && env_clp == 4 && num_m >= 4) pl.CL = 4;
  const int64_t items = ((num_m + pl.CL - 1) / pl.CL) * num_n;  // cluster work items without split
  const int64_t clusters = num_sms() / pl.CL;
  pl.nsplit = 1;
  pl.kbs = (int)nkb;
  if (items < clusters && nkb >= 4) {
    // decode-size M: split K so every SM streams weights.  Cost model per split count s:
    // waves * (K-blocks per item) * t_kb  +  fp32 partial write+read traffic / HBM,
    // t_kb ~ one 48 KB stage at an SM's share of HBM bandwidth.
    const double t_kb = 48e3 / 44e9, hbm = 6.0e12;
    double best = 1e30;
    static const int env_smax = getenv("ARC_GEMM_SPLIT_MAX") ? atoi(getenv("ARC_GEMM_SPLIT_MAX")) : 32;
    for (int64_t s = 1; s <= std::min<int64_t>(nkb / 2, env_smax); ++s) {
      const int64_t kbs = (nkb + s - 1) / s, ns = (nkb + kbs - 1) / kbs;
      const int64_t it = items * ns, waves = (it + clusters - 1) / clusters;
      const double cost = (double)waves * (double)kbs * t_kb + (ns > 1 ? (double)ns * M * N * 8.0 / hbm : 0.0);
      if (cost < best - 1e-12) {
        best = cost;
        pl.kbs = (int)kbs;
        pl.nsplit = (int)ns;
      }
    }
  }
  pl.ws_bytes = pl.nsplit > 1 ? kGemmCounterBytes + (size_t)pl.nsplit * (size_t)M * (size_t)round_up(N, 4) * sizeof(float)
                              : 0;
  // decode-size M: the stream-K kernel (stream_gemm.cu); the split-K path stays for the SwiGLU epilogue
  const StreamPlan sp = plan_stream(M, N, Kp);
  if (sp.ok) pl.ws_bytes = std::max(pl.ws_bytes, sp.ws_bytes);
  return pl;
}

cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t stream, const char** detail) {
  // decode-size M: the split-K kernel + fixed-order reduce kernel by default; the weight-streaming
  // stream-K kernel (stream_gemm.cu) measured slower on the LLaMA-3-8B decode step
  static const int env_stream = getenv("ARC_GEMM_STREAM") ? atoi(getenv("ARC_GEMM_STREAM")) : 0;
  if (env_stream && !p.swiglu && !p.red_mode && !p.fmt) {
    const StreamPlan sp = plan_stream(p.M, p.N, p.Kp);
    if (sp.ok) return launch_stream_gemm(p, sp, stream, detail);
  }
  // decode-size M: cluster split-K with the reduction in distributed shared memory (decode_gemm.cu)
  if (!p.swiglu && !p.red_mode && !p.fmt) {
    const DecodePlan dp = plan_decode(p.M, p.N, p.Kp);
    if (dp.ok) return launch_decode_gemm(p, dp, stream, detail);
  }
  // MXFP8 (p.fmt == 1): 128 K per 128-byte stage -> plan as an NVFP4 problem with twice the K
  GemmPlan pl = plan_gemm(p.M, p.N, (p.fmt == 1 || p.fmt == 3) ? 2 * p.Kp : p.Kp);
  if (p.fmt) {
    pl.pair = 0;
    if (pl.CL > 2) pl.CL = 2;
  }
  // SwiGLU epilogue: the 2-SM kernel leaves shared memory for the SiLU table (the 1-SM kernel's
  // 4 x 54 KB ring does not), so prefill-size SwiGLU GEMMs run as CTA pairs
  static const int env_swp = getenv("ARC_GEMM_SWIGLU_PAIR") ? atoi(getenv("ARC_GEMM_SWIGLU_PAIR")) : 1;
  if (p.swiglu && env_swp && pl.CL == 2 && pl.nsplit == 1) pl.pair = 1;
  const int CL = pl.CL;
  if (pl.nsplit > 1 && (p.ws == nullptr || p.ws_bytes + kGemmCounterBytes < pl.ws_bytes)) {
    if (detail) *detail = "split-K workspace too small";
    return cudaErrorInvalidValue;
  }
  CUtensorMap tmA, tmB, tmY;
  memset(&tmY, 0, sizeof(tmY));
  // wide epilogue stores (two 32-column chunks per TMA store, 3-stage ring): ARC_GEMM_EPI=2
  static const int env_epi = getenv("ARC_GEMM_EPI") ? atoi(getenv("ARC_GEMM_EPI")) : 1;
  const bool wide = env_epi == 2 && !pl.pair && CL == 2 && !p.swiglu && !p.y_fp32 && pl.nsplit == 1 && !p.fmt;
  if (p.swiglu ? !make_y_map(&tmY, p.y, p.M, p.N / 2, p.ldy, 16)
               : (!p.y_fp32 && !make_y_map(&tmY, p.y, p.M, p.N, p.ldy, wide ? 64 : 32))) {
    if (detail) *detail = "cuTensorMapEncodeTiled (Y) failed";
    return cudaErrorInvalidValue;
  }
  CUtensorMap tmSFA, tmSFB;
  // B box rows: the 1-SM kernel loads 256 (CL 1) or 128 (CL 2, multicast halves); the pair
  // kernel 128 (one pair) or 64 (two pairs, multicast quarters).  SFB box: 4 / 2 chunks.
  const int b_rows = pl.pair ? (CL == 2 ? 128 : 64) : BN / CL;
  // decode-size M on the 1-SM kernel: a 16/32/64-row A box instead of 128 rows of TMA zero fill
  static const int env_abox = getenv("ARC_GEMM_ABOX") ? atoi(getenv("ARC_GEMM_ABOX")) : 1;
  const int a_rows = (!pl.pair && CL == 1 && env_abox && p.M <= 64) ? (p.M <= 16 ? 16 : p.M <= 32 ? 32 : 64) : BM;
  const int64_t row_bytes = (p.fmt == 1 || p.fmt == 3) ? p.Kp : p.Kp / 2;
  const bool b_ok = p.fmt == 3 ? make_u4_unpack_map(&tmB, p.b_codes, p.N, p.Kp, b_rows)
                               : make_map(&tmB, p.b_codes, p.N, row_bytes, b_rows);
  // tail maps: 64-byte boxes with 64B swizzle for a last K block of 64 / 128 K (Kp % 256), so the TMA does not
  // zero-fill the second half of a 128-byte box (measured: a half-empty last block cost more than a full one)
  CUtensorMap tmAt, tmBt;
  memset(&tmAt, 0, sizeof(tmAt));
  memset(&tmBt, 0, sizeof(tmBt));
  static const int env_tail = getenv("ARC_GEMM_TAIL64") ? atoi(getenv("ARC_GEMM_TAIL64")) : 1;
  const int tail64 = env_tail && p.fmt == 0 && !pl.pair && (p.Kp % 256 == 64 || p.Kp % 256 == 128) ? 1 : 0;
  if (tail64 && (!make_operand_map_sw(&tmAt, p.a_codes, p.M, row_bytes, a_rows, 64, 64) ||
                 !make_operand_map_sw(&tmBt, p.b_codes, p.N, row_bytes, b_rows, 64, 64))) {
    if (detail) *detail = "cuTensorMapEncodeTiled (tail) failed";
    return cudaErrorInvalidValue;
  }
  // preferred clusters of 4 over the CL = 2 kernel (NVFP4 prefill): operands shared across the two pairs of a
  // 4-CTA cluster where the GPC packs one, plain pairs elsewhere (ARC_GEMM_PREF4=0 disables)
  static const int env_pref4 = getenv("ARC_GEMM_PREF4") ? atoi(getenv("ARC_GEMM_PREF4")) : 1;
  const int64_t num_m_ = (p.M + BM - 1) / BM, num_n_ = (p.N + BN - 1) / BN;
  const int raster_ = getenv("ARC_GEMM_RASTER") ? atoi(getenv("ARC_GEMM_RASTER")) : (p.M > p.N ? 1 : 0);
  const int64_t grid_pre = std::min<int64_t>(((num_m_ + CL - 1) / CL) * num_n_ * pl.nsplit, max_clusters(CL, pl.pair)) * CL;
  // measured (profiles/r2_gemm_variants_same_box.txt): B shared 4 ways (raster 0) 2.6 % faster on gate_up; the
  // A-sharing 2x2 mode (raster 1) made the 4-CTA clusters ~10 % slower per tile than plain pairs -> opt-in only
  // (ARC_GEMM_PREF4=2)
  const bool pref4 = env_pref4 && p.fmt == 0 && CL == 2 && !pl.pair && !wide && pl.nsplit == 1 && a_rows == BM &&
                     grid_pre % 4 == 0 &&
                     (raster_ == 0 ? ((num_m_ + 1) / 2) % 2 == 0 : (env_pref4 == 2 && num_n_ % 2 == 0));
  CUtensorMap tmA64, tmB64;
  memset(&tmA64, 0, sizeof(tmA64));
  memset(&tmB64, 0, sizeof(tmB64));
  if (pref4 && (!make_map(&tmA64, p.a_codes, p.M, row_bytes, BM / 2) || !make_map(&tmB64, p.b_codes, p.N, row_bytes, BN / 4))) {
    if (detail) *detail = "cuTensorMapEncodeTiled (cluster-4 boxes) failed";
    return cudaErrorInvalidValue;
  }
  if (!make_map(&tmA, p.a_codes, p.M, row_bytes, a_rows) || !b_ok ||
      (pl.pair && (!make_sf_map(&tmSFA, p.a_sf, (p.M + 127) / 128, p.Kp / 64, 4, 1) ||
                   !make_sf_map(&tmSFB, p.b_sf, (p.N + 127) / 128, p.Kp / 64, CL == 2 ? 4 : 2, 1)))) {
    if (detail) *detail = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  static PerDeviceOnce attr_once;
  const cudaError_t attr_err = attr_once.run([] {
    cudaError_t attr_err = cudaFuncSetAttribute(arc_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<2, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      gemm_smem_bytes(3, 2));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<1, STAGES, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<2, STAGES, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<1, STAGES, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<1, STAGES, 1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<2, STAGES, 1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<2, STAGES, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_pair_kernel<2, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      p_smem_bytes(5) + P_SILU_TAB_BYTES);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_pair_kernel<4, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_bytes(5));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(arc_gemm_pair_kernel<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, p_smem_bytes(4));
    return attr_err;
  });
  if (attr_err != cudaSuccess) return attr_err;
  Args a;
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.Kp = (int)p.Kp;
  a.sfa = p.a_sf;
  a.sfb = p.b_sf;
  a.gs_x = p.gs_x;
  a.gs_w = p.gs_w;
  a.y = p.y;
  a.ldy = p.ldy;
  a.y_fp32 = p.y_fp32;
  a.swiglu = p.swiglu;
  a.a_rows = a_rows;
  a.tail64 = pref4 ? 0 : tail64;
  a.mode4 = pref4 ? (raster_ == 0 ? 1 : 2) : 0;
  a.trace = (pl.pair || pl.nsplit > 1) ? nullptr : trace_slot();
  static const int dbg = getenv("ARC_GEMM_DEBUG") ? atoi(getenv("ARC_GEMM_DEBUG")) : 0;
  a.debug = dbg;
  // Keep the smaller operand L2-resident: sweep the tiles along it fastest so each wave of
  // clusters streams the larger operand once (e.g. down-proj: B 30 MB resident, A 59 MB streamed).
  static const int env_raster = getenv("ARC_GEMM_RASTER") ? atoi(getenv("ARC_GEMM_RASTER")) : -1;
  a.raster = env_raster >= 0 ? env_raster : (p.M > p.N ? 1 : 0);
  a.nsplit = pl.nsplit;
  a.kbs = pl.kbs;
  a.ws = static_cast<float*>(p.ws);
  a.red_mode = p.red_mode;
  a.red_np = p.red_np;
  a.red_mc = p.red_mc;
  for (int i = 0; i < 8; ++i) a.red_peer[i] = i < p.red_np ? p.red_peer[i] : nullptr;
  const int64_t num_m = (p.M + BM - 1) / BM, num_n = (p.N + BN - 1) / BN;
  const int64_t work = ((num_m + CL - 1) / CL) * num_n * pl.nsplit;  // cluster work items
  const int64_t grid = std::min<int64_t>(work, max_clusters(CL, pl.pair)) * CL;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NUM_THREADS);
  static const int env_st = getenv("ARC_GEMM_STAGES") ? atoi(getenv("ARC_GEMM_STAGES")) : 5;
  const bool st4 = pl.pair && CL == 2 && env_st == 4;  // experiment only
  cfg.dynamicSmemBytes = pl.pair ? p_smem_bytes(st4 ? 4 : 5) + (p.swiglu ? P_SILU_TAB_BYTES : 0)
                                  : (wide ? gemm_smem_bytes(3, 2) : SMEM_BYTES);
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  attr[2].id = cudaLaunchAttributePreferredClusterDimension;
  attr[2].val.preferredClusterDim.x = 4;
  attr[2].val.preferredClusterDim.y = 1;
  attr[2].val.preferredClusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pref4 ? 3 : 2;
  cudaError_t e = pl.pair ? (CL == 2 ? (st4 ? cudaLaunchKernelEx(&cfg, arc_gemm_pair_kernel<2, 4>, tmA, tmB, tmSFA, tmSFB, tmY, a)
                                                : cudaLaunchKernelEx(&cfg, arc_gemm_pair_kernel<2, 5>, tmA, tmB, tmSFA, tmSFB, tmY, a))
                                     : cudaLaunchKernelEx(&cfg, arc_gemm_pair_kernel<4, 5>, tmA, tmB, tmSFA, tmSFB, tmY, a))
                  : (p.fmt == 1 && CL == 1) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<1, STAGES, 1, 1>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : (p.fmt == 1 && CL == 2) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<2, STAGES, 1, 1>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : (p.fmt == 3 && CL == 1) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<1, STAGES, 1, 3>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : (p.fmt == 3 && CL == 2) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<2, STAGES, 1, 3>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : (p.fmt == 2 && CL == 1) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<1, STAGES, 1, 2>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : (p.fmt == 2 && CL == 2) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<2, STAGES, 1, 2>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : CL == 1 ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<1>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : (CL == 2 && wide) ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<2, 3, 2>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : CL == 2 ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<2>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                  : CL == 4 ? cudaLaunchKernelEx(&cfg, arc_gemm_kernel<4>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a)
                            : cudaLaunchKernelEx(&cfg, arc_gemm_kernel<8>, tmA, tmB, tmY, tmAt, tmBt, tmA64, tmB64, a);
  if (e != cudaSuccess) return e;
  if (pl.nsplit > 1) {
    const int64_t total = p.M * p.N;
    const int64_t rg = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    cudaLaunchConfig_t rc;
    memset(&rc, 0, sizeof(rc));
    rc.gridDim = dim3((unsigned)rg);
    rc.blockDim = dim3(256);
    rc.stream = stream;
    cudaLaunchAttribute ra[1];
    ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ra[0].val.programmaticStreamSerializationAllowed = 1;
    rc.attrs = ra;
    rc.numAttrs = 1;
    e = cudaLaunchKernelEx(&rc, arc_splitk_reduce_kernel, static_cast<const float*>(a.ws), (int)pl.nsplit, (int)p.M,
                           (int)p.N, p.y, p.ldy, p.y_fp32, p.swiglu, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace arc
