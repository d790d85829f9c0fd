// decode_gemm.cu -- the augmented NVFP4 GEMM (Eq.2) at decode-size M (<= 64
// tokens), where the layer is bound by reading the quantized weights once (N x Kp x 9/16 bytes).
//
// Cluster split-K with the reduction in distributed shared memory -- no fp32 partials in HBM, no
// counters, no second kernel:
//  * the grid is n_tiles x KS CTAs in clusters of KS along x (n_tiles = ceil(N / 128)); the KS CTAs of a
//    cluster own one tile of 128 weight rows and split its Kp/256 K blocks into KS contiguous ranges;
//  * operands are swapped relative to the prefill kernel: the 128 weight rows are the MMA's A operand
//    (M = 128, TMEM lane = weight row) and the activation tokens its B operand (N = 16 / 32 / 64, the
//    token count rounded up), so no MMA row is wasted on absent tokens and the accumulator is 128 lanes x
//    16..64 columns;
//  * the producer streams the CTA's weight stages (16 KB codes + 2 KB scales per 256-K block) BEFORE
//    griddepcontrol.wait when the caller guarantees the weights were complete before the preceding kernel
//    started (arc_linear: the weights never depend on the activation quantize that precedes the GEMM),
//    and the activation stages after it; ring of up to 8 stages;
//  * epilogue: each thread (one weight row) reads its token columns from TMEM into a [tokens][128] fp32
//    slice of its CTA's shared memory; after one cluster barrier the owner of token m (CTA m % KS) reads the
//    KS slices with ld.shared::cluster (all loads issued before the first add), sums them in rank order
//    (deterministic), scales by alpha = 1/(gs_x gs_w) and stores Y; a final cluster barrier keeps every
//    slice alive until its readers are done.  (ARC_DECODE_PULL=0: the push variant -- each CTA sends each
//    owner its block with one bulk shared::cta -> shared::cluster copy completing on the owner's mbarrier;
//    measured 2-9 % slower.)
#include "arc_device.cuh"
#include "arc_internal.h"

#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

namespace arc {
namespace {

constexpr int DBW = 128;                  // weight rows per tile (MMA M)
constexpr int DBKB = 128;                 // bytes per row per stage (256 E2M1, one 128B swizzle atom)
constexpr int DW_BYTES = DBW * DBKB;      // 16 KB
constexpr int DSF_BYTES = 4 * 512;        // 4 scale chunks (128 rows x 64 K each)
constexpr int D_MAX_STAGES = 8;
constexpr int D_THREADS = 192;
constexpr int D_SFA_COL = 64;             // weight scales (MMA A) in TMEM
constexpr int D_SFB_COL = 80;             // activation scales (MMA B)
constexpr int D_TMEM_COLS = 128;

struct DArgs {
  int M, N, Kp, a_rows, nkb, ks;
  int nst, stage_bytes;
  int tpd;              // tokens per destination CTA: ceil(M / ks)
  int spin;             // mbarrier waits without a suspend-time hint
  int ybulk;            // Y rows written with bulk copies (else per-element stores)
  int pull;             // split-K reduction: owners pull the slices with ld.shared::cluster after a cluster barrier
  const uint8_t* sfx;   // activation scales [roundup(M,128)][Kp/16] (tcgen05 128x4 layout)
  const uint8_t* sfw;   // weight scales [roundup(N,128)][Kp/16]
  const float* gs_x;
  const float* gs_w;
  void* y;
  int64_t ldy;
  int y_fp32;
  int w_early;          // weights may be streamed before griddepcontrol.wait
  unsigned long long* trace;  // timing experiments only (ARC_TRACE): [cta][4] globaltimer stamps
};

__device__ __forceinline__ void dtrace(const DArgs& a, int i) {
  if (a.trace && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(size_t)blockIdx.x * 8 + i] = t;
  }
}

// bulk copy of this CTA's shared memory into another CTA's (cluster addresses of the destination and
// of its mbarrier, which receives the complete_tx)
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src_cta), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
// bulk copy shared::cta -> global (bulk async-group completion)
__device__ __forceinline__ void bulk_store(void* gdst, uint32_t src_cta, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(src_cta), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
// mbarrier waits without a suspend-time hint (the latency-critical decode chain; ARC_DECODE_SPIN=0 restores
// the hinted wait of the throughput kernels for comparison)
__device__ __forceinline__ void dwait(uint64_t* bar, uint32_t parity, int spin) {
  if (!spin) {
    mbar_wait(bar, parity);
    return;
  }
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void dwait_cluster(uint64_t* bar, uint32_t parity, int spin) {
  if (!spin) {
    mbar_wait_cluster(bar, parity);
    return;
  }
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ float4 ld_dsmem_v4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}

// min 4 CTAs per SM: the one-wave planner (plan_decode) co-schedules up to 4 per SM by shared memory,
// so the registers must allow 4 as well (<= 85 per thread)
__global__ void __launch_bounds__(D_THREADS, 4)
    arc_decode_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                           DArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nst = args.nst, stage_bytes = args.stage_bytes;
  const int x_bytes = args.a_rows * DBKB;
  float* recv = reinterpret_cast<float*>(smem + nst * stage_bytes);  // [ks][tpd][128] fp32 partials pushed here
  uint64_t* full = reinterpret_cast<uint64_t*>(recv + (args.ks == 1 ? 0 : args.ks * args.tpd * DBW));
  uint64_t* empty = full + D_MAX_STAGES;
  uint64_t* acc_full = empty + D_MAX_STAGES;
  uint64_t* recv_bar = acc_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(recv_bar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ks = args.ks;
  const int r = (int)(blockIdx.x % ks);  // == %cluster_ctarank (clusters of ks along x)
  const int tile = (int)(blockIdx.x / ks);
  const int kb0 = (int)(((int64_t)r * args.nkb) / ks), kb1 = (int)(((int64_t)(r + 1) * args.nkb) / ks);
  const int nk = kb1 - kb0;
  const int kc_total = args.Kp / 64;

  long long clk0 = clock64();
  if (threadIdx.x == 0) {
    dtrace(args, 0);
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(recv_bar, 1);
    // the owner's share of tokens receives one block from every CTA of the cluster
    if (r < args.M) mbar_expect_tx(recv_bar, (uint32_t)(args.ks * args.tpd * DBW * 4));
    fence_mbar_init();
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
  }
  if (warp == 1) tmem_alloc(tmem_holder, D_TMEM_COLS);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  cluster_arrive_relaxed();  // barrier inits (fenced above) visible cluster-wide before the first remote access
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  long long ck[4] = {0, 0, 0, 0};  // epilogue clock stamps (trace only; written once at the end)
  long long clk2 = 0;
  float alpha_pull = 0.0f;
  if (warp == 0) {
    if (elect_one()) {
      // ---------------------------------------------------------------- producer
      const uint64_t pol_w = policy_evict_first();  // weights: read once per call
      const uint64_t pol_x = policy_evict_last();   // activation blocks: read by every weight tile
      auto load_w = [&](int s, int kb) {
        const int nkc = min(4, kc_total - kb * 4);
        uint8_t* st = smem + s * stage_bytes;
        mbar_expect_tx(&full[s], (uint32_t)(DW_BYTES + x_bytes + 2 * nkc * 512));
        tma_load_2d(st, &tmW, &full[s], kb * DBKB, tile * DBW, pol_w);
        bulk_load_hint(st + DW_BYTES + x_bytes, args.sfw + ((int64_t)tile * kc_total + kb * 4) * 512, nkc * 512,
                       &full[s], pol_w);
      };
      auto load_x = [&](int s, int kb) {
        const int nkc = min(4, kc_total - kb * 4);
        uint8_t* st = smem + s * stage_bytes;
        tma_load_2d(st + DW_BYTES, &tmX, &full[s], kb * DBKB, 0, pol_x);
        bulk_load_hint(st + DW_BYTES + x_bytes + DSF_BYTES, args.sfx + (int64_t)kb * 4 * 512, nkc * 512, &full[s],
                       pol_x);
      };
      const int npre = min(nst, nk);
      if (!args.w_early) pdl_wait();
      for (int i = 0; i < npre; ++i) load_w(i, kb0 + i);
      if (args.w_early) pdl_wait();
      dtrace(args, 1);
      for (int i = 0; i < npre; ++i) load_x(i, kb0 + i);
      int s = npre % nst;
      uint32_t ph = npre == nst ? 1u : 0u;
      for (int i = npre; i < nk; ++i) {
        dwait(&empty[s], ph ^ 1, args.spin);
        load_w(s, kb0 + i);
        load_x(s, kb0 + i);
        if (++s == nst) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(args.a_rows >> 3) << 17) | ((uint32_t)(DBW >> 4) << 24);
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nk; ++i) {
        const int kb = kb0 + i;
        const int nkc = min(4, kc_total - kb * 4);
        dwait(&full[s], ph, args.spin);
        tc_fence_after();
        const uint32_t sW = smem_u32(smem + s * stage_bytes);
        const uint32_t sX = sW + DW_BYTES;
        const uint32_t sSFW = sX + x_bytes;
        const uint32_t sSFX = sSFW + DSF_BYTES;
        for (int kk = 0; kk < nkc; ++kk) {
          utccp_32x128b_warpx4(tmem + D_SFA_COL + 4 * kk, smem_desc(sSFW + kk * 512, 0, 128, kLayoutSwizzleNone));
          utccp_32x128b_warpx4(tmem + D_SFB_COL + 4 * kk, smem_desc(sSFX + kk * 512, 0, 128, kLayoutSwizzleNone));
        }
        for (int kk = 0; kk < nkc; ++kk) {
          const uint64_t ad = smem_desc(sW + kk * 32, 16, 1024, kLayoutSwizzle128B);
          const uint64_t bd = smem_desc(sX + kk * 32, 16, 1024, kLayoutSwizzle128B);
          mma_nvf4(tmem, ad, bd, idesc, (i != 0) || (kk != 0), tmem + D_SFA_COL + 4 * kk, tmem + D_SFB_COL + 4 * kk);
        }
        tc_commit(&empty[s]);
        if (++s == nst) { s = 0; ph ^= 1; }
      }
      tc_commit(acc_full);
    }
  } else {
    // ---------------------------------------------------------------- epilogue: push partials, reduce
    // Token m belongs to CTA d = m % ks of the cluster (slot j = m / ks).  Each CTA stages its fp32
    // partials grouped by owner ([d][j][n], local shared memory) and one thread sends each owner its
    // block with a bulk shared::cta -> shared::cluster copy (the TMA engine, no per-element remote
    // stores) that completes on the owner's receive barrier; the owner waits for all ks blocks and sums
    // them in rank order (deterministic), scales by alpha and stores Y.  A trailing cluster barrier keeps
    // every staging block alive until its copy has landed.
    const int q = warp & 3;       // TMEM lane quadrant = weight rows [32q, 32q + 32)
    const int n = q * 32 + lane;  // weight row within the tile
    const int tpd = args.tpd;
    const uint32_t blk = (uint32_t)tpd * DBW * 4u;  // bytes per (source, owner) block
    float* stg = reinterpret_cast<float*>(smem);    // [ks][tpd][128] staging (reuses the drained ring)
    cluster_wait();  // every CTA's receive barrier is initialised (long before the accumulator is ready)
    pdl_wait();      // gs_x may come from the preceding kernel: read it only after the wait
    const float alpha = __fdiv_rn(1.0f, __fmul_rn(__ldg(args.gs_x), __ldg(args.gs_w)));
    dwait(acc_full, 0, args.spin);
    tc_fence_after();
    if (threadIdx.x == 64) dtrace(args, 2);
    clk2 = clock64();  // stamps 3..6: SM cycles since the accumulator was ready
    alpha_pull = alpha;
    // Y rows of this CTA's tokens, staged as one [tpd][128] tile after the send staging and written with
    // one bulk copy per token row (no per-element global stores on the critical path)
    const int eb = args.y_fp32 ? 4 : 2;
    uint8_t* ytile = ks == 1 ? smem : smem + (size_t)ks * blk;  // (ks = 1: no send staging)
    const int gn = tile * DBW + n;
    auto put = [&](int sl, float acc) {
      const float out = __fmul_rn(acc, alpha);
      if (args.y_fp32) reinterpret_cast<float*>(ytile)[sl * DBW + n] = out;
      else reinterpret_cast<__nv_bfloat16*>(ytile)[sl * DBW + n] = __float2bfloat16_rn(out);
    };
    if (ks == 1) {
      // one CTA per tile: the accumulator is the result
      for (int c = 0; c < args.M; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c + j < args.M) put(c + j, __uint_as_float(v[j]));
      }
      if (threadIdx.x == 64) ck[0] = ck[1] = ck[2] = clock64() - clk2;
    } else if (args.pull) {
      // pull variant: stage [m][n] locally; owners read the ks slices after one cluster barrier (below)
      for (int c = 0; c < args.M; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c + j < args.M) stg[(c + j) * DBW + n] = __uint_as_float(v[j]);
      }
      if (threadIdx.x == 64) ck[0] = ck[1] = clock64() - clk2;
    } else {
      int d = 0, slot = 0;
      for (int c = 0; c < args.M; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (c + j < args.M) {
            stg[(d * tpd + slot) * DBW + n] = __uint_as_float(v[j]);
            if (++d == ks) { d = 0; ++slot; }
          }
        }
      }
      fence_proxy_async();                 // generic staging writes -> the async (bulk copy) proxy
      named_bar_sync(1, 128);              // all four epilogue warps staged
      if (threadIdx.x == 64) {
        ck[0] = clock64() - clk2;
        const int nd = min(ks, args.M);
        for (int dd = 0; dd < nd; ++dd)
          bulk_s2c(mapa_u32(smem_u32(recv) + (uint32_t)r * blk, (uint32_t)dd), smem_u32(stg) + (uint32_t)dd * blk, blk,
                   mapa_u32(smem_u32(recv_bar), (uint32_t)dd));
        ck[1] = clock64() - clk2;
      }
      if (r < args.M) {
        dwait(recv_bar, 0, args.spin);
        if (threadIdx.x == 64) ck[2] = clock64() - clk2;
        for (int sl = 0, m = r; m < args.M; ++sl, m += ks) {
          float p[8];
#pragma unroll
          for (int src = 0; src < 8; ++src) p[src] = src < ks ? recv[(src * tpd + sl) * DBW + n] : 0.0f;
          float acc = p[0];
#pragma unroll
          for (int src = 1; src < 8; ++src)
            if (src < ks) acc = __fadd_rn(acc, p[src]);
          put(sl, acc);
        }
      }
    }
    if (r < args.M && !(args.pull && ks > 1)) {
      const int valid = min(DBW, args.N - tile * DBW);
      const bool bulk_ok = args.ybulk && ((valid * eb) & 15) == 0;
      if (bulk_ok) {
        fence_proxy_async();
        named_bar_sync(1, 128);
        if (threadIdx.x == 64) {
          for (int sl = 0, m = r; m < args.M; ++sl, m += ks)
            bulk_store(static_cast<uint8_t*>(args.y) + ((int64_t)m * args.ldy + tile * DBW) * eb,
                       smem_u32(ytile + (size_t)sl * DBW * eb), (uint32_t)(valid * eb));
          bulk_commit();
          bulk_wait_read0();  // the tile's shared memory is read before the CTA may exit
        }
      } else if (gn < args.N) {
        for (int sl = 0, m = r; m < args.M; ++sl, m += ks) {
          if (args.y_fp32)
            static_cast<float*>(args.y)[(int64_t)m * args.ldy + gn] = reinterpret_cast<float*>(ytile)[sl * DBW + n];
          else
            static_cast<__nv_bfloat16*>(args.y)[(int64_t)m * args.ldy + gn] =
                reinterpret_cast<__nv_bfloat16*>(ytile)[sl * DBW + n];
        }
      }
    }
    if (threadIdx.x == 64) {
      ck[3] = clock64() - clk2;
      if (args.trace && blockIdx.x < 1024) {
        for (int i = 0; i < 4; ++i) args.trace[(size_t)blockIdx.x * 8 + 3 + i] = (unsigned long long)ck[i];
        args.trace[(size_t)blockIdx.x * 8 + 7] = (unsigned long long)(clock64() - clk0);
      }
    }
  }
  if (warp < 2) cluster_wait();  // (pairs with the arrive after initialisation)

  if (args.pull && ks > 1) {
    // every CTA's [m][n] slice is staged: one cluster barrier, then the owner of token m (CTA m % ks) reads
    // the ks slices with ld.shared::cluster (all issued before the first add), sums them in rank order,
    // scales and stores Y
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp >= 2 && r < args.M) {
      // warp w of the epilogue reduces this CTA's tokens i = w, w + 4, ... (token m = r + ks i); each lane
      // owns 4 consecutive weight rows: one 16-byte ld.shared::cluster per (token, source CTA)
      const int w = warp - 2;
      const int n4 = lane * 4;
      const int gn = tile * DBW + n4;
      if (threadIdx.x == 64) ck[2] = clock64() - clk2;
      uint32_t base[8];
#pragma unroll
      for (int src = 0; src < 8; ++src) base[src] = src < ks ? mapa_u32(smem_u32(smem), (uint32_t)src) : 0u;
      for (int m = r + ks * w; m < args.M; m += 4 * ks) {  // one token per round: its ks loads issued first
        const uint32_t off = (uint32_t)(m * DBW + n4) * 4u;
        float4 p[8];
#pragma unroll
        for (int src = 0; src < 8; ++src)
          p[src] = src < ks ? ld_dsmem_v4(base[src] + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 acc = p[0];
#pragma unroll
        for (int src = 1; src < 8; ++src) {
          if (src < ks) {  // rank order: the fixed summation order of every call
            acc.x = __fadd_rn(acc.x, p[src].x);
            acc.y = __fadd_rn(acc.y, p[src].y);
            acc.z = __fadd_rn(acc.z, p[src].z);
            acc.w = __fadd_rn(acc.w, p[src].w);
          }
        }
        const float o[4] = {__fmul_rn(acc.x, alpha_pull), __fmul_rn(acc.y, alpha_pull),
                            __fmul_rn(acc.z, alpha_pull), __fmul_rn(acc.w, alpha_pull)};
        if (gn + 3 < args.N) {
          if (args.y_fp32) {
            *reinterpret_cast<float4*>(static_cast<float*>(args.y) + (int64_t)m * args.ldy + gn) =
                make_float4(o[0], o[1], o[2], o[3]);
          } else {
            __nv_bfloat162 lo = __floats2bfloat162_rn(o[0], o[1]), hi = __floats2bfloat162_rn(o[2], o[3]);
            uint2 v;
            v.x = *reinterpret_cast<uint32_t*>(&lo);
            v.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(args.y) + (int64_t)m * args.ldy + gn) = v;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (gn + k < args.N) {
              if (args.y_fp32) static_cast<float*>(args.y)[(int64_t)m * args.ldy + gn + k] = o[k];
              else static_cast<__nv_bfloat16*>(args.y)[(int64_t)m * args.ldy + gn + k] = __float2bfloat16_rn(o[k]);
            }
          }
        }
      }
      if (threadIdx.x == 64) {
        ck[3] = clock64() - clk2;
        if (args.trace && blockIdx.x < 1024) {
          for (int i = 0; i < 4; ++i) args.trace[(size_t)blockIdx.x * 8 + 3 + i] = (unsigned long long)ck[i];
          args.trace[(size_t)blockIdx.x * 8 + 7] = (unsigned long long)(clock64() - clk0);
        }
      }
    }
  }

  // every CTA's blocks have landed once every owner has passed its receive wait
  cluster_arrive_relaxed();
  cluster_wait();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, D_TMEM_COLS);
  }
}

}  // namespace

// Co-resident clusters of ks CTAs at `smem` bytes each (cached per device / shape): clusters live inside one
// GPC, so the count depends on how the GPCs' SMs pack, not only on CTAs per SM.
static int decode_max_clusters(int ks, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_tuple(dev, ks, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaFuncSetAttribute(arc_decode_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)(ks * 64));
  cfg.blockDim = dim3(D_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, arc_decode_gemm_kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = std::max(1, num_sms() / ks);
  }
  cache[key] = n;
  return n;
}

static size_t decode_smem(const DecodePlan& pl, int64_t M) {
  const int64_t tpd = (M + pl.ks - 1) / pl.ks;
  return (size_t)pl.nst * pl.stage_bytes + (pl.ks == 1 ? 0 : (size_t)pl.ks * tpd * DBW * 4) + 1024 + 256;
}

DecodePlan plan_decode(int64_t M, int64_t N, int64_t Kp) {
  DecodePlan pl;
  static const int env_on = getenv("ARC_GEMM_DECODE") ? atoi(getenv("ARC_GEMM_DECODE")) : 1;
  static const int env_ks = getenv("ARC_DECODE_KS") ? atoi(getenv("ARC_DECODE_KS")) : 0;
  static const int env_nst = getenv("ARC_DECODE_NST") ? atoi(getenv("ARC_DECODE_NST")) : 0;
  pl.ok = env_on && M >= 1 && M <= 64;
  if (!pl.ok) return pl;
  pl.a_rows = M <= 16 ? 16 : M <= 32 ? 32 : 64;
  pl.n_tiles = (N + DBW - 1) / DBW;
  pl.nkb = (Kp + 2 * DBKB - 1) / (2 * DBKB);
  pl.stage_bytes = DW_BYTES + pl.a_rows * DBKB + 2 * DSF_BYTES;
  // Every cluster of the grid should be resident at once (one wave: all SMs stream from the start and
  // no CTA waits for another's exit).  Co-resident clusters = (clusters of ks that tile the GPCs at one
  // CTA per SM, from the occupancy API) x (CTAs per SM the shared memory allows, <= 4 for TMEM).
  // Among the one-wave configurations take the largest grid (most SMs and bytes in flight), then the
  // most ring stages; if none fits in one wave, one CTA per tile.
  // enough tiles to give every SM one: no split (no reduction tail)
  // clusters of at most 6 CTAs at M <= 16, 4 above (measured, profiles/r2_decode_cluster.txt steps 8 and 12:
  // the reduction tail waits for the slowest CTA of the cluster and grows with the tokens each owner sums;
  // 8-CTA clusters lost more there than their extra streaming SMs gained)
  static const int env_ksmax = getenv("ARC_DECODE_KSMAX") ? atoi(getenv("ARC_DECODE_KSMAX")) : 0;
  const int64_t ksmax = env_ksmax > 0 ? env_ksmax : (M <= 16 ? 6 : 4);
  const int64_t ks_hi =
      pl.n_tiles >= num_sms() ? 1 : std::max<int64_t>(1, std::min<int64_t>({ksmax, 8, pl.nkb / 2}));
  int64_t best_grid = -1;
  for (int64_t ks = 1; ks <= ks_hi; ++ks) {
    if (env_ks > 0 && ks != std::min<int64_t>(env_ks, ks_hi)) continue;
    DecodePlan c = pl;
    c.ks = (int)ks;
    c.grid = pl.n_tiles * ks;
    const int64_t kmax = (pl.nkb + ks - 1) / ks;
    const int64_t tpd = (M + ks - 1) / ks;
    const int64_t recv = ks * tpd * DBW * 4;
    int64_t nst_min = 2;
    while (nst_min * pl.stage_bytes < recv + tpd * DBW * 4) ++nst_min;  // the ring also holds the reduction staging
    const int64_t api = decode_max_clusters((int)ks, 64 * 1024);
    for (int64_t nst = std::max<int64_t>(nst_min, std::min<int64_t>(kmax, D_MAX_STAGES)); nst >= nst_min; --nst) {
      if (env_nst > 0 && nst != std::max<int64_t>(nst_min, env_nst)) continue;
      c.nst = (int)nst;
      const size_t smem = decode_smem(c, M);
      const int64_t per_sm = std::min<int64_t>(4, (int64_t)(233472 / (smem + 1024)));
      if (per_sm < 1) continue;
      if (pl.n_tiles <= api * per_sm || (env_ks > 0 && env_nst > 0)) {
        if (c.grid > best_grid) {
          best_grid = c.grid;
          pl.ks = c.ks;
          pl.grid = c.grid;
          pl.nst = c.nst;
        }
        break;  // the most stages that fit in one wave for this ks
      }
    }
  }
  if (best_grid < 0 || (ks_hi == 1 && env_nst == 0)) {  // one CTA per tile, two per SM
    pl.ks = 1;
    pl.grid = pl.n_tiles;
    // as many stages as leave room for two CTAs per SM (the grid then runs in one wave up to 296 tiles)
    const int64_t fit2 = (113 * 1024 - 1024 - 1280) / pl.stage_bytes;
    pl.nst = (int)std::max<int64_t>(2, std::min<int64_t>({pl.nkb, 4, fit2}));
  }
  if (getenv("ARC_DECODE_VERBOSE"))
    fprintf(stderr, "arc_decode: M=%lld N=%lld Kp=%lld tiles=%lld nkb=%lld -> ks=%d grid=%lld nst=%d smem=%zu\n",
            (long long)M, (long long)N, (long long)Kp, (long long)pl.n_tiles, (long long)pl.nkb, pl.ks,
            (long long)pl.grid, pl.nst, decode_smem(pl, M));
  return pl;
}

cudaError_t launch_decode_gemm(const GemmProblem& p, const DecodePlan& pl, cudaStream_t stream, const char** detail) {
  CUtensorMap tmW, tmX;
  if (!make_operand_map(&tmW, p.b_codes, p.N, p.Kp / 2, DBW, DBKB) ||
      !make_operand_map(&tmX, p.a_codes, p.M, p.Kp / 2, pl.a_rows, DBKB)) {
    if (detail) *detail = "cuTensorMapEncodeTiled failed";
    return cudaErrorInvalidValue;
  }
  DArgs a;
  memset(&a, 0, sizeof(a));
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.Kp = (int)p.Kp;
  a.a_rows = pl.a_rows;
  a.nkb = (int)pl.nkb;
  a.ks = pl.ks;
  a.nst = pl.nst;
  a.stage_bytes = pl.stage_bytes;
  a.sfx = p.a_sf;
  a.sfw = p.b_sf;
  a.gs_x = p.gs_x;
  a.gs_w = p.gs_w;
  a.y = p.y;
  a.ldy = p.ldy;
  a.y_fp32 = p.y_fp32;
  static const int env_we = getenv("ARC_DECODE_WEARLY") ? atoi(getenv("ARC_DECODE_WEARLY")) : 1;
  a.w_early = p.weights_ready && env_we;
  a.tpd = (int)((p.M + pl.ks - 1) / pl.ks);
  static const int env_spin = getenv("ARC_DECODE_SPIN") ? atoi(getenv("ARC_DECODE_SPIN")) : 1;
  a.spin = env_spin;
  static const int env_yb = getenv("ARC_DECODE_YBULK") ? atoi(getenv("ARC_DECODE_YBULK")) : 0;
  a.ybulk = env_yb;
  static const int env_pull = getenv("ARC_DECODE_PULL") ? atoi(getenv("ARC_DECODE_PULL")) : 1;
  a.pull = env_pull;
  a.trace = trace_slot();
  const size_t smem = decode_smem(pl, p.M);
  static PerDeviceOnce attr_once;
  const cudaError_t ae = attr_once.run([] {
    return cudaFuncSetAttribute(arc_decode_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (ae != cudaSuccess) return ae;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)pl.grid);
  cfg.blockDim = dim3(D_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_decode_gemm_kernel, tmW, tmX, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace arc
