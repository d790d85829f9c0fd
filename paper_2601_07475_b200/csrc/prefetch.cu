// arc_prefetch_l2: pull a read-only buffer (the next linear's quantized weights) into the 126 MB L2 while
// the current linear's dependent kernels run, so a decode-size layer keeps one HBM weight stream going
// across its linears.
#include <cuda_runtime.h>
#include <string.h>

#include "arc.h"
#include "arc_device.cuh"
#include "arc_internal.h"

namespace arc {
namespace {

// One warp per CTA; each lane issues bulk L2 prefetches over its CTA's contiguous share.  The kernel lets
// its dependents launch at entry (PDL) and waits for its predecessor only before exiting, so it never
// breaks the stream's ordering (the next kernel's griddepcontrol.wait still covers everything before).
__global__ void __launch_bounds__(32) arc_prefetch_l2_kernel(const uint8_t* p, uint64_t bytes, uint64_t share) {
  pdl_launch_dependents();
  const uint64_t b0 = (uint64_t)blockIdx.x * share, b1 = b0 + share < bytes ? b0 + share : bytes;
  constexpr uint64_t CH = 16384;
  for (uint64_t o = b0 + (uint64_t)threadIdx.x * CH; o < b1; o += 32 * CH) {
    const uint32_t n = (uint32_t)(b1 - o < CH ? b1 - o : CH);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(n) : "memory");
  }
  pdl_wait();
}

}  // namespace

cudaError_t launch_prefetch_l2(const void* ptr, size_t bytes, cudaStream_t stream) {
  const int ctas = num_sms();
  const uint64_t share = (((uint64_t)bytes + ctas - 1) / ctas + 15) & ~(uint64_t)15;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)((bytes + share - 1) / share));
  cfg.blockDim = dim3(32);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, arc_prefetch_l2_kernel, static_cast<const uint8_t*>(ptr), (uint64_t)bytes,
                                     share);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace arc
