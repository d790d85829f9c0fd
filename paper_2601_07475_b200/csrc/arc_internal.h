// arc_internal.h -- host-side declarations shared by the libarc.so translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace arc {

// Runs f() (returning cudaError_t) once per CUDA device and caches its result: function attributes
// such as the dynamic shared-memory limit are per device, so a process-wide once is not enough.
struct PerDeviceOnce {
  static constexpr int kMaxDev = 64;
  std::mutex mu;
  bool done[kMaxDev] = {};
  cudaError_t err[kMaxDev] = {};
  template <class F>
  cudaError_t run(F&& f) {
    int d = 0;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return e;
    if (d < 0 || d >= kMaxDev) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(mu);
    if (!done[d]) {
      err[d] = f();
      done[d] = true;
    }
    return err[d];
  }
};

inline int64_t kp_of(int64_t K, int64_t S) { return (K + S + 63) / 64 * 64; }
inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

int num_sms();  // SM count of the current device (cached per device)

// Timing experiments only (env ARC_TRACE): per-launch slots of [1024 CTAs][4] globaltimer stamps that the
// quantize and decode-GEMM kernels fill; nullptr when tracing is off (the normal case).
unsigned long long* trace_slot();

// gamma != nullptr: RMSNorm (reading Q23) each row in place before quantizing it.
// up_off >= 0: SiLU-mul mode (reading Q24): quantize bf16(bf16(SiLU(x)) * x[up_off..]) per row.
cudaError_t launch_quant(const void* x, int64_t rows, int K, int64_t ld, const int32_t* perm, int S, const float* gs,
                         int layout, int weight_mode, uint8_t* codes, uint8_t* sf, cudaStream_t stream,
                         const void* gamma = nullptr, float eps = 0.0f, int64_t up_off = -1, int mx = 0,
                         int consts_ready = 0, int f16 = 0);
// consts_ready (arc_linear): perm was complete before the preceding kernel started (calibration constants,
// like the prepared weights), so the decode-size quantize may load it before griddepcontrol.wait.
cudaError_t launch_silu_mul(const void* gu, int64_t rows, int K, int64_t ld, int64_t up_off, void* h, int64_t ldh,
                            cudaStream_t s);
cudaError_t launch_rmsnorm(const void* x, int64_t rows, int K, int64_t ldx, const void* gamma, float eps, void* y,
                           int64_t ldy, cudaStream_t s);
// Native MXFP4-ARC (UE8M0 per 32-block, 32-granular block map, Kpm = roundup(K+S, 128)).
cudaError_t launch_mx_native_quant(const void* x, int64_t rows, int K, int S, int64_t ld, const int32_t* perm,
                                   int weight, int layout, uint8_t* codes, uint8_t* sf, cudaStream_t stream);
// Fig.8a comparator: plain MXFP8 (E4M3 codes [rows][roundup(K,128)], E8M0 scales per 32-block).
cudaError_t launch_mxfp8_quant(const void* x, int64_t rows, int K, int64_t ld, uint8_t* codes, uint8_t* sf,
                               cudaStream_t stream);
cudaError_t launch_calib_absmax(const void* x, int64_t rows, int K, int64_t ld, float* chan_max, cudaStream_t s,
                                int f16 = 0);
// mx = 0: gs = 2688/amax (reading Q3); mx = 1: the MXFP4-ARC offset gs = 2^-c (reading Q25).
cudaError_t launch_tensor_scale(const void* x, int64_t rows, int K, int64_t ld, float* gs_out, cudaStream_t s,
                                int mx = 0, int f16 = 0);

struct GemmProblem {
  int64_t M, N, Kp;
  const uint8_t* a_codes;
  const uint8_t* a_sf;
  const uint8_t* b_codes;
  const uint8_t* b_sf;
  const float* gs_x;
  const float* gs_w;
  void* y;
  int64_t ldy;
  int y_fp32;
  int swiglu = 0;    // SwiGLU epilogue (gate/up rows interleaved in groups of 16): y = h [M][N/2] bf16
  unsigned* cnt = nullptr;  // kGemmCounterBytes of per-tile arrival counters (zero; left zero), decode-size M
  void* ws;                 // fp32 partials of the decode-size split paths (may be null when not split)
  size_t ws_bytes;          // bytes at ws
  // The weights were complete before the kernel preceding this GEMM started (arc_linear: that
  // kernel is the activation quantize, which lets dependents launch only after its own
  // griddepcontrol.wait): the decode-size kernel may then stream them before its own wait.
  int weights_ready = 0;
  // fused row-parallel reduction (arc_gemm_reduce): 1 = NVLS multimem.red into red_mc, 2 = red.add into the
  // red_np peer buffers; fp32 output only, the 1-SM kernel and the split-K reduce kernel
  int fmt = 0;       // 0: NVFP4 ARC operands (Kp = K+S padded to 64); 1: plain MXFP8 (Fig.8a comparator, Kp % 128 == 0);
                     // 2: native MXFP4 (UE8M0 per 32, Kp % 128 == 0); 3: W4A8 (MXFP8 A x packed MXFP4 B, Kp % 128 == 0)
  int red_mode = 0;
  int red_np = 0;
  float* red_mc = nullptr;
  float* red_peer[8] = {};
};
// Decode-size M (<= 64): weight-streaming stream-K GEMM (stream_gemm.cu).
struct StreamPlan {
  bool ok = false;
  int a_rows = 0;                 // activation TMA box rows: 16 / 32 / 64
  int64_t n_tiles = 0, nkb = 0, units = 0, maxseg = 0;
  int grid = 0;
  size_t part_bytes = 0, cnt_bytes = 0, ws_bytes = 0;   // workspace: partials + counters (zero before use)
};
StreamPlan plan_stream(int64_t M, int64_t N, int64_t Kp);
// The activation the decode-size kernel quantizes itself (fused arc_linear): bf16 x [M][ldx], the
// profile's perm / S / layout; the codes and scales go to GemmProblem::a_codes / a_sf.
struct StreamQuant {
  const void* x;
  int64_t ldx;
  const int32_t* perm;
  int K, S, layout;
};
cudaError_t launch_stream_gemm(const GemmProblem& p, const StreamPlan& pl, cudaStream_t stream, const char** detail,
                               const StreamQuant* fq = nullptr);
// Decode-size M (<= 64): cluster split-K GEMM with the K reduction in distributed shared memory
// (decode_gemm.cu): n_tiles x ks CTAs, clusters of ks, no workspace.
struct DecodePlan {
  bool ok = false;
  int a_rows = 0;                  // tokens rounded up to the MMA N: 16 / 32 / 64
  int64_t n_tiles = 0, nkb = 0;    // 128-row weight tiles, 256-K blocks
  int ks = 1;                      // CTAs per cluster (K ranges per tile)
  int64_t grid = 0;
  int nst = 2, stage_bytes = 0;
};
DecodePlan plan_decode(int64_t M, int64_t N, int64_t Kp);
cudaError_t launch_decode_gemm(const GemmProblem& p, const DecodePlan& pl, cudaStream_t stream, const char** detail);
struct GemmPlan {
  int CL;            // CTAs per cluster along M
  int pair;          // CL == 2: 1 = 2-SM tcgen05 MMA (cta_group::2), 0 = two 1-SM CTAs sharing B by multicast
  int nsplit, kbs;   // split-K factor and K-blocks per split
  size_t ws_bytes;   // fp32 partials nsplit*M*N
};
GemmPlan plan_gemm(int64_t M, int64_t N, int64_t Kp);
// Returns a CUresult-style error through cudaError_t (cudaErrorUnknown + text) on encode failure.
cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t stream, const char** detail);

// Bytes at offset 0 of every arc_linear workspace: the GEMM's per-tile counters (kGemmCounterBytes).
inline size_t sync_bytes_of(int64_t /*N*/);

// 2-D K-major operand tensor map (uint8 [rows][row_bytes], 128B swizzle, box box_bytes x box_rows).
bool make_operand_map(CUtensorMap* m, const void* base, int64_t rows, int64_t row_bytes, int box_rows, int box_bytes);
// the same with a 32 / 64 / 128-byte swizzle (0: none)
bool make_operand_map_sw(CUtensorMap* m, const void* base, int64_t rows, int64_t row_bytes, int box_rows, int box_bytes,
                         int swizzle_bytes);

// Every arc_gemm workspace starts with this many bytes of per-tile arrival counters (the
// decode-size stream-K kernel's), zero before the first use and left zero by every call; the
// fp32 partials of either split path follow them, so calls of any shape can share one workspace.
constexpr size_t kGemmCounterBytes = 16384;
inline size_t sync_bytes_of(int64_t /*N*/) { return kGemmCounterBytes; }

bool make_u4_unpack_map_probe(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t k_elems, int box_rows);
}  // namespace arc
