/*
 * arc_probe.h -- hardware-semantics probes exported by libarc.so for the test
 * suite (not part of the hot path).  They run the exact device primitives the
 * quantization kernel uses, element-wise, so tests can pin them against the
 * oracle exhaustively (E2M1 rounding, E4M3 ceil).
 * Pointers are device pointers; work is enqueued on `stream`; same status codes
 * and validation conventions as arc.h.
 */
#ifndef ARC_PROBE_H_
#define ARC_PROBE_H_
#include "arc.h"
#ifdef __cplusplus
extern "C" {
#endif
/* out[i] = E2M1 code the kernel assigns to in[i] (cvt.rn.satfinite.e2m1x2 +
 * sign fix-up; reading Q1). */
ARC_API arc_status_t arc_probe_e2m1(const float* in, int64_t n, uint8_t* out, void* stream);
/* Same, for the fp32 whose bit pattern is (uint32)(start_bits + i), i < n. */
ARC_API arc_status_t arc_probe_e2m1_bits(uint32_t start_bits, int64_t n, uint8_t* out, void* stream);
/* Raw hardware cvt.rn.satfinite.e2m1x2.f32 nibble (no sign fix-up) for bits start+i. */
ARC_API arc_status_t arc_probe_e2m1_raw_bits(uint32_t start_bits, int64_t n, uint8_t* out, void* stream);
/* out[i] = the kernel's ceil-rounded E4M3 scale code of in[i] >= 0 (reading Q2). */
ARC_API arc_status_t arc_probe_e4m3_ceil(const float* in, int64_t n, uint8_t* out, void* stream);
/* out[i] = the bf16 pattern of bf16(SiLU(g[i])) as the fused SiLU-mul quantize kernel computes
 * it (per-CTA table + closed-form tails, reading Q24), for bf16 patterns g[i]. */
ARC_API arc_status_t arc_probe_silu(const uint16_t* g, int64_t n, uint16_t* out, void* stream);
/* TMA layout probe for the W4A8 comparator (tests only): loads a rows x 128-element box of packed
 * E2M1 codes `src` (device, rows*64 bytes, row-major) through a CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B
 * map into two shared-memory buffers whose mbarriers expect rows*64 and rows*128 transaction bytes;
 * status[0..1] (device int32) = whether each barrier completed within a bounded wait; out (device,
 * 16384 bytes) = both 8 KB buffers (0xEE = untouched). Synchronous; rows in [1, 64]. */
ARC_API arc_status_t arc_probe_u4_unpack(const uint8_t* src, int64_t rows, uint8_t* out, int32_t* status);
/* Timing experiments only: with env ARC_STREAM_TRACE set, the decode-size stream-K GEMM records 8
 * globaltimer stamps per CTA of its last launch (entry, early weight loads issued,
 * griddepcontrol.wait passed, first stage ready, last MMA issued, last segment's accumulator
 * ready, split-tile arrival counted, epilogue done); copies max_ctas rows of 8 uint64 to host
 * memory (synchronous) and returns the row count (0 when tracing is off). */
ARC_API int arc_debug_stream_trace(unsigned long long* host, int max_ctas);
/* Timing experiments only: with env ARC_TRACE set, every quantize and decode-size GEMM launch takes the
 * next of 64 slots of [1024 CTAs][8] uint64 globaltimer stamps (quantize: entry, griddepcontrol.wait
 * passed, producer done, first primary warp done; decode GEMM: entry, griddepcontrol.wait passed,
 * accumulator ready, partials sent, arrivals done, partials received, exit).  Copies the 64 slots to host (synchronous; host holds 64*1024*8 uint64),
 * clears them and restarts at slot 0; returns the number of slots used since the last call (0 when
 * tracing is off). */
ARC_API int arc_debug_trace(unsigned long long* host);
#ifdef __cplusplus
}
#endif
#endif
