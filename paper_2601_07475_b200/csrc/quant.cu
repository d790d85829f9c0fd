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
};

// One NVFP4 stage on 16 values (oracle C4).  Writes codes (packed, element 2i in
// the low nibble of byte i) and returns the scale code; d_out / t keep the
// quantities the residual stage needs.
ARC_DEV uint32_t stage16(const float (&z)[16], float base, float c6, float (&t)[16], float& d_out, uint2& packed) {
  float a = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) a = fmaxf(a, fabsf(z[i]));
  const uint32_t sf = e4m3_ceil(__fmul_rn(a, c6));
  const float d = e4m3_value(sf);
  const float k = (d == 0.0f) ? 0.0f : __fdiv_rn(base, d);
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = __fmul_rn(z[i], k);
  uint32_t w[2] = {0u, 0u};
#pragma unroll
  for (int i = 0; i < 16; i += 2) w[i >> 3] |= e2m1x2(t[i], t[i + 1]) << (4 * (i & 7));
  packed = make_uint2(w[0], w[1]);
  d_out = d;
  return sf;
}

__global__ void __launch_bounds__(256) arc_quant_kernel(QuantArgs p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int K = p.K;
  const int R = p.rows_per_tile;
  const int kpad = (K + 7) & ~7;  // perm entries, rounded to 16 bytes
  uint16_t* perm_s = reinterpret_cast<uint16_t*>(smem);
  uint16_t* xs0 = perm_s + kpad;
  uint16_t* xs1 = xs0 + (size_t)R * K;
  uint64_t* bars = reinterpret_cast<uint64_t*>(xs1 + (size_t)R * K);

  const int tid = threadIdx.x;
  const int64_t ntile = (p.rows + R - 1) / R;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < K; i += blockDim.x) perm_s[i] = (uint16_t)__ldg(p.perm + i);
  __syncthreads();

  auto issue = [&](int64_t tile, int buf) {
    const int64_t r0 = tile * R;
    const int nr = (int)dmin64(R, p.rows - r0);
    uint16_t* dst = buf ? xs1 : xs0;
    mbar_expect_tx(&bars[buf], (uint32_t)(nr * K * 2));
    for (int r = 0; r < nr; ++r) bulk_load(dst + (size_t)r * K, p.x + (r0 + r) * p.ld, (uint32_t)K * 2, &bars[buf]);
  };
  if (tid == 0) {
    if (blockIdx.x < ntile) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < ntile) issue(blockIdx.x + gridDim.x, 1);
  }

  const float gs = __ldg(p.gs);
  const float c6g = __fdiv_rn(gs, 6.0f);
  const int nb = K >> 4, ns = p.S >> 4;
  const int NB = p.Kp >> 4;  // physical blocks per row (multiple of 4)
  const int64_t sf_rb_stride = (int64_t)(p.Kp >> 6) * 512;
  const int lane = tid & 31;

  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    mbar_wait(&bars[buf], (it >> 1) & 1);
    const uint16_t* xs = buf ? xs1 : xs0;
    const int64_t r0 = tile * R;
    const int nr = (int)dmin64(R, p.rows - r0);
    const int items = nr * NB;

    for (int base = 0; base < items; base += blockDim.x) {
      const int i = base + tid;
      const bool valid = i < items;
      uint32_t sfb = 0;
      uint2 packed = make_uint2(0u, 0u);
      int r = 0, pb = 0;
      if (valid) {
        r = i / NB;
        pb = i - r * NB;
        // physical block -> (logical primary block l, residual?)  (App.D)
        int l = -1;
        bool resid = false;
        if (p.layout == 0) {
          if (pb < 2 * ns) { l = pb >> 1; resid = pb & 1; }
          else if (pb < nb + ns) l = pb - ns;
        } else {
          if (pb < nb) l = pb;
          else if (pb < nb + ns) { l = pb - nb; resid = true; }
        }
        if (l >= 0) {
          const uint16_t* xr = xs + (size_t)r * K;
          const uint4* pp = reinterpret_cast<const uint4*>(perm_s + 16 * l);
          const uint4 p0 = pp[0], p1 = pp[1];
          const uint32_t pw[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
          float z[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            z[2 * j] = bf16_bits_to_f32(xr[pw[j] & 0xFFFFu]);
            z[2 * j + 1] = bf16_bits_to_f32(xr[pw[j] >> 16]);
          }
          float t[16], d1;
          sfb = stage16(z, gs, c6g, t, d1, packed);
          if (resid && !p.weight_mode) {
            // residual in units of d1/gs, exact (P:138 R_o = X_o - s*Q_Xo; Q6)
            float e[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const uint32_t q = (j < 8 ? packed.x >> (4 * j) : packed.y >> (4 * (j - 8))) & 15u;
              e[j] = __fsub_rn(t[j], e2m1_value(q));
            }
            float t2[16], d2;
            sfb = stage16(e, d1, __fdiv_rn(d1, 6.0f), t2, d2, packed);
          }
        }
        const int64_t m = r0 + r;
        *reinterpret_cast<uint2*>(p.codes + m * (p.Kp >> 1) + (int64_t)pb * 8) = packed;
      }
      // 4 consecutive lanes hold the 4 scale columns of one 128x4 tile row.
      uint32_t w = sfb;
      w |= __shfl_down_sync(0xffffffffu, sfb, 1) << 8;
      w |= __shfl_down_sync(0xffffffffu, sfb, 2) << 16;
      w |= __shfl_down_sync(0xffffffffu, sfb, 3) << 24;
      if (valid && (lane & 3) == 0) {
        const int64_t m = r0 + r;
        const int64_t off = (m >> 7) * sf_rb_stride + (int64_t)(pb >> 2) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4;
        *reinterpret_cast<uint32_t*>(p.sf + off) = w;
      }
    }
    __syncthreads();  // all reads of this buffer done
    if (tid == 0 && tile + 2 * (int64_t)gridDim.x < ntile) {
      fence_proxy_async();  // generic-proxy reads of buf ordered before the async-proxy refill
      issue(tile + 2 * (int64_t)gridDim.x, buf);
    }
  }
}

// ------------------------------------------------------------------ offline reductions
// Column abs-max over rows (calibration).  |bf16| bit patterns order like
// their values, so the max is taken on integers (exact) and merged with an
// integer atomicMax on the float bits (non-negative floats order as ints).
__global__ void arc_calib_absmax_kernel(const uint16_t* x, int64_t rows, int K, int64_t ld, int rows_per_cta,
                                        float* chan_max) {
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
  for (int j = 0; j < 8; ++j) atomicMax(reinterpret_cast<unsigned int*>(chan_max + c8 + j), mx[j] << 16);
}

// max |x| over a whole matrix into *amax_bits (float bits, caller zeroes it).
__global__ void arc_absmax_all_kernel(const uint16_t* x, int64_t rows, int K, int64_t ld, unsigned int* amax_bits) {
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
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, mx << 16);
}

// gs = 2688 / amax (reading Q3), in place over the amax bits; amax = 0 -> 1.
__global__ void arc_finalize_scale_kernel(float* gs) {
  const float amax = *gs;
  *gs = amax > 0.0f ? __fdiv_rn(2688.0f, amax) : 1.0f;
}

// ------------------------------------------------------------------ launchers
int64_t quant_smem_bytes(int K, int R) { return (int64_t)((K + 7) & ~7) * 2 + 2LL * R * K * 2 + 16; }

int quant_rows_per_tile(int K) {
  int R = 16384 / K;  // <= 32 KB of bf16 per stage
  return R < 1 ? 1 : (R > 8 ? 8 : R);
}

cudaError_t launch_quant(const void* x, int64_t rows, int K, int64_t ld, const int32_t* perm, int S, const float* gs,
                         int layout, int weight_mode, uint8_t* codes, uint8_t* sf, cudaStream_t stream) {
  QuantArgs a;
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
  a.rows_per_tile = quant_rows_per_tile(K);
  const int64_t smem = quant_smem_bytes(K, a.rows_per_tile);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(arc_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, arc_quant_kernel, 256, (size_t)smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) occ = 1;
  const int64_t ntile = (rows + a.rows_per_tile - 1) / a.rows_per_tile;
  const int64_t grid = imin64(ntile, (int64_t)num_sms() * occ);
  arc_quant_kernel<<<(unsigned)grid, 256, (size_t)smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_calib_absmax(const void* x, int64_t rows, int K, int64_t ld, float* chan_max, cudaStream_t s) {
  const int threads = 128;
  const int rows_per_cta = 64;
  dim3 grid((unsigned)((K / 8 + threads - 1) / threads), (unsigned)((rows + rows_per_cta - 1) / rows_per_cta));
  arc_calib_absmax_kernel<<<grid, threads, 0, s>>>(static_cast<const uint16_t*>(x), rows, K, ld, rows_per_cta,
                                                   chan_max);
  return cudaGetLastError();
}

cudaError_t launch_tensor_scale(const void* x, int64_t rows, int K, int64_t ld, float* gs_out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(gs_out, 0, sizeof(float), s);
  if (e != cudaSuccess) return e;
  const int64_t n8 = rows * (K / 8);
  const int64_t grid = imax64(1, imin64((n8 + 255) / 256, (int64_t)num_sms() * 8));
  arc_absmax_all_kernel<<<(unsigned)grid, 256, 0, s>>>(static_cast<const uint16_t*>(x), rows, K, ld,
                                                      reinterpret_cast<unsigned int*>(gs_out));
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  arc_finalize_scale_kernel<<<1, 1, 0, s>>>(gs_out);
  return cudaGetLastError();
}

}  // namespace arc
