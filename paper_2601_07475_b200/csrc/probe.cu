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
}
