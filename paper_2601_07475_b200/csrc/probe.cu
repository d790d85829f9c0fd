// probe.cu -- element-wise probes of the quantization kernel's device primitives
// (include/arc_probe.h).  Test infrastructure exported by libarc.so; the probes
// call the very same inline functions as arc_quant_kernel.
#include "arc.h"
#include "arc_probe.h"
#include "arc_device.cuh"
#include "arc_internal.h"

namespace arc {
__global__ void probe_e2m1_kernel(const float* in, uint32_t start, int64_t n, uint8_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in ? in[i] : __uint_as_float(start + (uint32_t)i);
    out[i] = (uint8_t)(e2m1x2(v, 0.0f) & 15u);
  }
}
__global__ void probe_e2m1_raw_kernel(uint32_t start, int64_t n, uint8_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(e2m1x2_raw(__uint_as_float(start + (uint32_t)i), 0.0f) & 15u);
}
__global__ void probe_e4m3_ceil_kernel(const float* in, int64_t n, uint8_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)e4m3_ceil(in[i]);
}
// TMA 16U4_ALIGN16B probe: load a rows x 128-element box of packed E2M1 with two different expected
// transaction counts (packed bytes / shared-memory bytes) on two barriers, bounded waits, dump shared memory.
__global__ void probe_u4_unpack_kernel(const __grid_constant__ CUtensorMap tm, int rows, uint8_t* out, int* status) {
  __shared__ __align__(1024) uint8_t buf[2][8192];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * 8192; ++i) (&buf[0][0])[i] = 0xEE;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    mbar_expect_tx(&bar[0], (uint32_t)(rows * 64));
    mbar_expect_tx(&bar[1], (uint32_t)(rows * 128));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tma_load_2d(buf[0], &tm, &bar[0], 0, 0, policy_evict_normal());
    tma_load_2d(buf[1], &tm, &bar[1], 0, 0, policy_evict_normal());
    for (int b = 0; b < 2; ++b) {
      uint32_t done = 0;
      for (int it = 0; it < 200000 && !done; ++it) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, 1000;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(&bar[b]))
            : "memory");
      }
      status[b] = (int)done;
    }
    const long long t0 = clock64();
    while (clock64() - t0 < 200000) {
    }
    for (int i = 0; i < 2 * 8192; ++i) out[i] = (&buf[0][0])[i];
  }
}
static arc_status_t probe_status(cudaError_t e) { return e == cudaSuccess ? ARC_OK : ARC_ERR_CUDA; }
static unsigned probe_grid(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16); }
}  // namespace arc

using namespace arc;
extern "C" {
arc_status_t arc_probe_e2m1(const float* in, int64_t n, uint8_t* out, void* stream) {
  if (!in || !out) return ARC_ERR_NULL;
  if (n < 0) return ARC_ERR_SHAPE;
  if (!arc_device_supported()) return ARC_ERR_UNSUPPORTED;
  if (n == 0) return ARC_OK;
  probe_e2m1_kernel<<<probe_grid(n), 256, 0, (cudaStream_t)stream>>>(in, 0u, n, out);
  return probe_status(cudaGetLastError());
}
arc_status_t arc_probe_e2m1_bits(uint32_t start_bits, int64_t n, uint8_t* out, void* stream) {
  if (!out) return ARC_ERR_NULL;
  if (n < 0 || n > (int64_t)1 << 32) return ARC_ERR_SHAPE;
  if (!arc_device_supported()) return ARC_ERR_UNSUPPORTED;
  if (n == 0) return ARC_OK;
  probe_e2m1_kernel<<<probe_grid(n), 256, 0, (cudaStream_t)stream>>>(nullptr, start_bits, n, out);
  return probe_status(cudaGetLastError());
}
arc_status_t arc_probe_e2m1_raw_bits(uint32_t start_bits, int64_t n, uint8_t* out, void* stream) {
  if (!out) return ARC_ERR_NULL;
  if (n < 0 || n > (int64_t)1 << 32) return ARC_ERR_SHAPE;
  if (!arc_device_supported()) return ARC_ERR_UNSUPPORTED;
  if (n == 0) return ARC_OK;
  probe_e2m1_raw_kernel<<<probe_grid(n), 256, 0, (cudaStream_t)stream>>>(start_bits, n, out);
  return probe_status(cudaGetLastError());
}
arc_status_t arc_probe_e4m3_ceil(const float* in, int64_t n, uint8_t* out, void* stream) {
  if (!in || !out) return ARC_ERR_NULL;
  if (n < 0) return ARC_ERR_SHAPE;
  if (!arc_device_supported()) return ARC_ERR_UNSUPPORTED;
  if (n == 0) return ARC_OK;
  probe_e4m3_ceil_kernel<<<probe_grid(n), 256, 0, (cudaStream_t)stream>>>(in, n, out);
  return probe_status(cudaGetLastError());
}
arc_status_t arc_probe_u4_unpack(const uint8_t* src, int64_t rows, uint8_t* out, int32_t* status) {
  if (!src || !out || !status) return ARC_ERR_NULL;
  if (rows < 1 || rows > 64) return ARC_ERR_SHAPE;
  if (!arc_device_supported()) return ARC_ERR_UNSUPPORTED;
  CUtensorMap tm;
  if (!make_u4_unpack_map_probe(&tm, src, rows, 128, (int)rows)) return ARC_ERR_CUDA;
  probe_u4_unpack_kernel<<<1, 32>>>(tm, (int)rows, out, status);
  return probe_status(cudaDeviceSynchronize());
}
}
