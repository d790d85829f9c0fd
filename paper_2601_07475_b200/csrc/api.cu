// api.cu -- the extern "C" boundary of libarc.so (include/arc.h): synchronous
// argument validation, then kernel launches on the caller's stream.  No device
// memory is allocated and the device is never synchronized (except by the
// documented host-IO variant).  There is no fallback path: a non-sm_100 device
// is ARC_ERR_UNSUPPORTED.
#include "arc.h"
#include "arc_internal.h"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace arc {

static thread_local char g_err[512] = "";

static arc_status_t fail(arc_status_t s, const char* what) {
  std::snprintf(g_err, sizeof(g_err), "%s", what);
  return s;
}
static arc_status_t cuda_fail(cudaError_t e, const char* where, const char* detail = nullptr) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s%s%s", where, cudaGetErrorString(e), detail ? " / " : "",
                detail ? detail : "");
  return ARC_ERR_CUDA;
}

namespace {
constexpr int kTraceSlots = 64, kTraceCtas = 1024;
unsigned long long* g_trace = nullptr;
int g_trace_next = 0;
std::once_flag g_trace_once;
}  // namespace

unsigned long long* trace_slot() {
  std::call_once(g_trace_once, [] {
    if (getenv("ARC_TRACE") &&
        cudaMalloc(&g_trace, (size_t)kTraceSlots * kTraceCtas * 8 * sizeof(unsigned long long)) != cudaSuccess)
      g_trace = nullptr;
    if (g_trace) cudaMemset(g_trace, 0, (size_t)kTraceSlots * kTraceCtas * 8 * sizeof(unsigned long long));
  });
  if (!g_trace) return nullptr;
  return g_trace + (size_t)(g_trace_next++ % kTraceSlots) * kTraceCtas * 8;
}

}  // namespace arc

extern "C" ARC_API int arc_debug_trace(unsigned long long* host) {
  using namespace arc;
  if (!g_trace || !host) return 0;
  const size_t bytes = (size_t)kTraceSlots * kTraceCtas * 8 * sizeof(unsigned long long);
  if (cudaDeviceSynchronize() != cudaSuccess) return 0;
  if (cudaMemcpy(host, g_trace, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  cudaMemset(g_trace, 0, bytes);
  const int n = g_trace_next;
  g_trace_next = 0;
  return n;
}

namespace arc {
int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

static bool device_ok() {
  static int cache[64] = {0};  // 0 unknown, 1 ok, 2 not ok
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  if (cache[dev] == 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cache[dev] = (major == 10 && minor == 0) ? 1 : 2;
  }
  return cache[dev] == 1;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static arc_status_t check_ks(int64_t K, int64_t S) {
  if (K <= 0 || K % 16) return fail(ARC_ERR_SHAPE, "K must be a positive multiple of 16");
  if (S < 0 || S % 16 || S > K) return fail(ARC_ERR_SHAPE, "S must be a multiple of 16 with 0 <= S <= K");
  if (kp_of(K, S) > 32768) return fail(ARC_ERR_SHAPE, "K + S must be <= 32768");
  return ARC_OK;
}

static arc_status_t check_device() {
  if (!device_ok()) return fail(ARC_ERR_UNSUPPORTED, "current CUDA device is not sm_100 (B200); no fallback");
  return ARC_OK;
}

static arc_status_t check_profile(const arc_profile_t* prof) {
  if (!prof || !prof->perm || !prof->gs) return fail(ARC_ERR_NULL, "null profile / perm / gs");
  arc_status_t s = check_ks(prof->K, prof->S);
  if (s != ARC_OK) return s;
  if (prof->layout != ARC_LAYOUT_INTERLEAVED && prof->layout != ARC_LAYOUT_CONTIGUOUS)
    return fail(ARC_ERR_SHAPE, "bad layout");
  return ARC_OK;
}

static arc_status_t check_qweight(const arc_qweight_t* qw) {
  if (!qw || !qw->codes || !qw->sf || !qw->gs) return fail(ARC_ERR_NULL, "null qweight / codes / sf / gs");
  arc_status_t s = check_ks(qw->K, qw->S);
  if (s != ARC_OK) return s;
  if (qw->N <= 0 || qw->N > (1 << 30)) return fail(ARC_ERR_SHAPE, "N must be positive");
  if (qw->Kp != kp_of(qw->K, qw->S)) return fail(ARC_ERR_SHAPE, "qweight Kp != roundup(K+S, 64)");
  if (qw->layout != ARC_LAYOUT_INTERLEAVED && qw->layout != ARC_LAYOUT_CONTIGUOUS)
    return fail(ARC_ERR_SHAPE, "bad layout");
  if (!aligned16(qw->codes) || !aligned16(qw->sf)) return fail(ARC_ERR_ALIGN, "qweight buffers not 16B aligned");
  return ARC_OK;
}

}  // namespace arc

using namespace arc;

extern "C" {

const char* arc_status_string(arc_status_t s) {
  switch (s) {
    case ARC_OK: return "ARC_OK";
    case ARC_ERR_NULL: return "ARC_ERR_NULL";
    case ARC_ERR_SHAPE: return "ARC_ERR_SHAPE";
    case ARC_ERR_ALIGN: return "ARC_ERR_ALIGN";
    case ARC_ERR_UNSUPPORTED: return "ARC_ERR_UNSUPPORTED";
    case ARC_ERR_WORKSPACE: return "ARC_ERR_WORKSPACE";
    case ARC_ERR_CUDA: return "ARC_ERR_CUDA";
    case ARC_ERR_NONFINITE: return "ARC_ERR_NONFINITE";
  }
  return "ARC_ERR_?";
}

const char* arc_last_error(void) { return g_err; }

int arc_device_supported(void) { return device_ok() ? 1 : 0; }

arc_status_t arc_buffer_sizes(int64_t rows, int64_t K, int32_t S, int64_t* Kp, size_t* code_bytes, size_t* sf_bytes) {
  arc_status_t s = check_ks(K, S);
  if (s != ARC_OK) return s;
  if (rows < 0) return fail(ARC_ERR_SHAPE, "rows < 0");
  const int64_t kp = kp_of(K, S);
  if (Kp) *Kp = kp;
  if (code_bytes) *code_bytes = (size_t)(rows * (kp / 2));
  if (sf_bytes) *sf_bytes = (size_t)(round_up(rows, 128) * (kp / 16));
  return ARC_OK;
}

static size_t act_ws_bytes(int64_t M, int64_t K, int32_t S) {
  const int64_t kp = kp_of(K, S);
  return (size_t)round_up(M * (kp / 2), 256) + (size_t)round_up(round_up(M, 128) * (kp / 16), 256);
}

arc_status_t arc_gemm_workspace_size(int64_t M, const arc_qweight_t* qw, size_t* bytes) {
  arc_status_t s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (!bytes) return fail(ARC_ERR_NULL, "null bytes");
  if (M < 0) return fail(ARC_ERR_SHAPE, "M < 0");
  *bytes = M == 0 ? 0 : plan_gemm(M, qw->N, qw->Kp).ws_bytes;
  return ARC_OK;
}

// arc_linear workspace: [GEMM tile counters (kGemmCounterBytes, fixed at offset 0 so calls of any
// shape can share the workspace) | quantized A | GEMM fp32 partials].
static size_t linear_rest_bytes(int64_t M, const arc_qweight_t* qw, int /*flags*/) {
  const size_t g = plan_gemm(M, qw->N, qw->Kp).ws_bytes;
  return act_ws_bytes(M, qw->K, qw->S) + (g ? (size_t)round_up((int64_t)(g - kGemmCounterBytes), 256) : 0);
}

arc_status_t arc_linear_workspace_size(int64_t M, const arc_qweight_t* qw, size_t* bytes) {
  arc_status_t s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (!bytes) return fail(ARC_ERR_NULL, "null bytes");
  if (M < 0) return fail(ARC_ERR_SHAPE, "M < 0");
  *bytes = sync_bytes_of(qw->N) + (M == 0 ? 0 : linear_rest_bytes(M, qw, ARC_LINEAR_AUTO));
  return ARC_OK;
}

static int in16_dtype(arc_dtype_t t) { return t == ARC_FP16 ? 1 : (t == ARC_BF16 ? 0 : -1); }

arc_status_t arc_calib_absmax(const void* x, int64_t rows, int64_t K, int64_t ldx, float* chan_max, void* stream) {
  return arc_calib_absmax_ex(x, ARC_BF16, rows, K, ldx, chan_max, stream);
}
arc_status_t arc_calib_absmax_ex(const void* x, arc_dtype_t x_dtype, int64_t rows, int64_t K, int64_t ldx,
                                 float* chan_max, void* stream) {
  const int f16 = in16_dtype(x_dtype);
  if (f16 < 0) return fail(ARC_ERR_SHAPE, "x_dtype must be ARC_BF16 or ARC_FP16");
  if (!x || !chan_max) return fail(ARC_ERR_NULL, "null x / chan_max");
  if (K <= 0 || K % 16 || rows < 0 || ldx < K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad rows/K/ldx");
  if (!aligned16(x)) return fail(ARC_ERR_ALIGN, "x not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  if (rows == 0) return ARC_OK;
  cudaError_t e = launch_calib_absmax(x, rows, (int)K, ldx, chan_max, (cudaStream_t)stream, f16);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_calib_absmax");
}

arc_status_t arc_select_outliers(const float* chan_max_host, int64_t K, int32_t s_override, int32_t* perm_host,
                                 int32_t* S, int32_t* S_raw, float* M, float* tau, float* gs) {
  if (!chan_max_host || !perm_host || !S || !S_raw || !M || !tau || !gs) return fail(ARC_ERR_NULL, "null argument");
  if (K <= 0 || K % 16) return fail(ARC_ERR_SHAPE, "K must be a positive multiple of 16");
  if (s_override > K || (s_override >= 0 && s_override % 16)) return fail(ARC_ERR_SHAPE, "bad s_override");
  float mx = 0.0f;
  for (int64_t j = 0; j < K; ++j) {
    const float v = chan_max_host[j];
    if (!(v >= 0.0f) || v > 3.4028234663852886e38f) return fail(ARC_ERR_NONFINITE, "non-finite or negative chan_max");
    mx = std::max(mx, v);
  }
  std::vector<int32_t> idx((size_t)K);
  for (int64_t j = 0; j < K; ++j) idx[(size_t)j] = (int32_t)j;
  // descending abs-max, ties to the lower channel index (reading Q9): a total order.
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int32_t a, int32_t b) { return chan_max_host[a] > chan_max_host[b]; });
  std::memcpy(perm_host, idx.data(), sizeof(int32_t) * (size_t)K);
  const float t = mx * 0.125f;  // tau = 2^-3 M, exact
  int64_t sr = 0;
  for (int64_t j = 0; j < K; ++j) sr += chan_max_host[j] > t;
  const int64_t sa = std::min<int64_t>(K, (sr + 15) / 16 * 16);
  *S_raw = (int32_t)sr;
  *S = s_override >= 0 ? s_override : (int32_t)sa;
  *M = mx;
  *tau = t;
  volatile float num = 2688.0f;  // one IEEE fp32 division
  *gs = mx > 0.0f ? num / mx : 1.0f;
  return ARC_OK;
}

// Bank-conflict-aware channel order inside each 16-channel block (see arc.h).
// Warp lanes <-> 32 consecutive blocks; at gather step q every lane reads its
// block's q-th channel from a staged bf16 row: bank = (channel >> 1) & 31, two
// channels in the same 32-bit word are one access.  A step costs the largest
// number of distinct words any bank receives; a seeded local search over
// in-block swaps minimizes the sum over the 16 steps for each 32-block chunk.
static int gather_step_cost(const int32_t* col[32], int n, int shift) {
  int words[32][32];
  int cnt[32] = {0};
  int worst = 0;
  for (int i = 0; i < n; ++i) {
    const int w = *col[i] >> shift, b = w & 31;
    bool dup = false;
    for (int k = 0; k < cnt[b]; ++k) dup |= words[b][k] == w;
    if (!dup) {
      words[b][cnt[b]++] = w;
      worst = std::max(worst, cnt[b]);
    }
  }
  return worst;
}

arc_status_t arc_gather_order(const int32_t* perm_host, int64_t K, int32_t* perm_out_host) {
  return arc_gather_order_ex(perm_host, K, 2, perm_out_host);
}

arc_status_t arc_gather_order_ex(const int32_t* perm_host, int64_t K, int elem_bytes, int32_t* perm_out_host) {
  if (!perm_host || !perm_out_host) return fail(ARC_ERR_NULL, "null perm");
  if (elem_bytes != 2 && elem_bytes != 4) return fail(ARC_ERR_SHAPE, "elem_bytes must be 2 or 4");
  const int shift = elem_bytes == 2 ? 1 : 0;  // channel -> 4-byte shared-memory word
  if (K <= 0 || K % 16) return fail(ARC_ERR_SHAPE, "K must be a positive multiple of 16");
  std::vector<char> seen((size_t)K, 0);
  for (int64_t j = 0; j < K; ++j) {
    const int32_t c = perm_host[j];
    if (c < 0 || c >= K || seen[(size_t)c]) return fail(ARC_ERR_SHAPE, "perm_host is not a permutation");
    seen[(size_t)c] = 1;
  }
  std::vector<int32_t> out(perm_host, perm_host + K);
  const int64_t nblk = K / 16, nchunk = (nblk + 31) / 32;
  // Chunks are independent: each has its own seed (the result does not depend on the thread count) and
  // stops early once every step costs one word per bank (the minimum).
  auto search = [&](int64_t ch) {
    const int64_t c0 = ch * 32;
    const int n = (int)std::min<int64_t>(32, nblk - c0);
    int32_t* B = out.data() + c0 * 16;  // B[i*16 + q]
    const int32_t* col[32];
    int cost[16], total = 0;
    for (int q = 0; q < 16; ++q) {
      for (int i = 0; i < n; ++i) col[i] = &B[i * 16 + q];
      cost[q] = gather_step_cost(col, n, shift);
      total += cost[q];
    }
    uint64_t rng = 0x9E3779B97F4A7C15ull ^ (0xD1B54A32D192ED03ull * (uint64_t)(ch + 1));
    for (int it = 0; it < 4000 && total > 16; ++it) {
      rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
      const int i = (int)(rng % (uint64_t)n), a = (int)((rng >> 16) & 15), b = (int)((rng >> 24) & 15);
      if (a == b) continue;
      std::swap(B[i * 16 + a], B[i * 16 + b]);
      for (int k = 0; k < n; ++k) col[k] = &B[k * 16 + a];
      const int ca = gather_step_cost(col, n, shift);
      for (int k = 0; k < n; ++k) col[k] = &B[k * 16 + b];
      const int cb = gather_step_cost(col, n, shift);
      if (ca + cb <= cost[a] + cost[b]) {
        total += ca + cb - cost[a] - cost[b];
        cost[a] = ca;
        cost[b] = cb;
      } else {
        std::swap(B[i * 16 + a], B[i * 16 + b]);
      }
    }
  };
  const int nth = (int)std::min<int64_t>(nchunk, std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  std::atomic<int64_t> next{0};
  auto worker = [&] {
    for (int64_t ch; (ch = next.fetch_add(1)) < nchunk;) search(ch);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nth; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  std::memcpy(perm_out_host, out.data(), sizeof(int32_t) * (size_t)K);
  return ARC_OK;
}

arc_status_t arc_tensor_scale(const void* x, int64_t rows, int64_t K, int64_t ldx, float* gs_out, void* stream) {
  return arc_tensor_scale_ex(x, ARC_BF16, rows, K, ldx, gs_out, stream);
}
arc_status_t arc_tensor_scale_ex(const void* x, arc_dtype_t x_dtype, int64_t rows, int64_t K, int64_t ldx,
                                 float* gs_out, void* stream) {
  const int f16 = in16_dtype(x_dtype);
  if (f16 < 0) return fail(ARC_ERR_SHAPE, "x_dtype must be ARC_BF16 or ARC_FP16");
  if (!x || !gs_out) return fail(ARC_ERR_NULL, "null x / gs_out");
  if (K <= 0 || K % 16 || rows < 0 || ldx < K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad rows/K/ldx");
  if (!aligned16(x)) return fail(ARC_ERR_ALIGN, "x not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_tensor_scale(x, rows, (int)K, ldx, gs_out, (cudaStream_t)stream, 0, f16);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_tensor_scale");
}

arc_status_t arc_quantize_weight(const void* w, int64_t N, int64_t K, int64_t ldw, const int32_t* perm, int32_t S,
                                 const float* gs_w, arc_layout_t layout, uint8_t* codes, uint8_t* sf, void* stream) {
  return arc_quantize_weight_ex(w, ARC_BF16, N, K, ldw, perm, S, gs_w, layout, codes, sf, stream);
}
arc_status_t arc_quantize_weight_ex(const void* w, arc_dtype_t w_dtype, int64_t N, int64_t K, int64_t ldw,
                                    const int32_t* perm, int32_t S, const float* gs_w, arc_layout_t layout,
                                    uint8_t* codes, uint8_t* sf, void* stream) {
  const int f16 = in16_dtype(w_dtype);
  if (f16 < 0) return fail(ARC_ERR_SHAPE, "w_dtype must be ARC_BF16 or ARC_FP16");
  if (!w || !perm || !gs_w || !codes || !sf) return fail(ARC_ERR_NULL, "null argument");
  arc_status_t s = check_ks(K, S);
  if (s != ARC_OK) return s;
  if (N < 0 || ldw < K || ldw % 8) return fail(ARC_ERR_SHAPE, "bad N/ldw");
  if (layout != ARC_LAYOUT_INTERLEAVED && layout != ARC_LAYOUT_CONTIGUOUS) return fail(ARC_ERR_SHAPE, "bad layout");
  if (!aligned16(w) || !aligned16(codes) || !aligned16(sf)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  if (N == 0) return ARC_OK;
  cudaError_t e = launch_quant(w, N, (int)K, ldw, perm, S, gs_w, (int)layout, 1, codes, sf, (cudaStream_t)stream,
                               nullptr, 0.0f, -1, 0, 0, f16);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_quantize_weight");
}

static arc_status_t quantize_activation_impl(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                            uint8_t* codes, uint8_t* sf, void* stream, int consts_ready, int f16 = 0);
arc_status_t arc_quantize_activation(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                     uint8_t* codes, uint8_t* sf, void* stream) {
  return quantize_activation_impl(x, M, ldx, prof, codes, sf, stream, 0);
}
arc_status_t arc_quantize_activation_ex(const void* x, arc_dtype_t x_dtype, int64_t M, int64_t ldx,
                                        const arc_profile_t* prof, uint8_t* codes, uint8_t* sf, void* stream) {
  const int f16 = in16_dtype(x_dtype);
  if (f16 < 0) return fail(ARC_ERR_SHAPE, "x_dtype must be ARC_BF16 or ARC_FP16");
  return quantize_activation_impl(x, M, ldx, prof, codes, sf, stream, 0, f16);
}
// consts_ready: arc_linear's promise that perm (like the weights) was complete before the preceding kernel
static arc_status_t quantize_activation_impl(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                            uint8_t* codes, uint8_t* sf, void* stream, int consts_ready, int f16) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  if (M < 0 || ldx < prof->K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad M/ldx");
  if (M == 0) return ARC_OK;
  if (!x || !codes || !sf) return fail(ARC_ERR_NULL, "null x / codes / sf");
  if (!aligned16(x) || !aligned16(codes) || !aligned16(sf)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  if (M == 0) return ARC_OK;
  cudaError_t e = launch_quant(x, M, (int)prof->K, ldx, prof->perm, prof->S, prof->gs, (int)prof->layout, 0, codes,
                               sf, (cudaStream_t)stream, nullptr, 0.0f, -1, 0, consts_ready, f16);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_quantize_activation");
}

arc_status_t arc_rmsnorm(const void* x, int64_t M, int64_t K, int64_t ldx, const void* gamma, float eps, void* y,
                         int64_t ldy, void* stream) {
  if (K <= 0 || K % 16 || K > 32768 || M < 0 || ldx < K || ldx % 8 || ldy < K || ldy % 8)
    return fail(ARC_ERR_SHAPE, "bad M/K/ldx/ldy");
  if (!(eps >= 0.0f) || eps > 3.4e38f) return fail(ARC_ERR_SHAPE, "eps must be finite and >= 0");
  if (M == 0) return ARC_OK;
  if (!x || !gamma || !y) return fail(ARC_ERR_NULL, "null x / gamma / y");
  if (!aligned16(x) || !aligned16(gamma) || !aligned16(y)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_rmsnorm(x, M, (int)K, ldx, gamma, eps, y, ldy, (cudaStream_t)stream);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_rmsnorm");
}

arc_status_t arc_rmsnorm_quantize_activation(const void* x, int64_t M, int64_t ldx, const void* gamma, float eps,
                                             const arc_profile_t* prof, uint8_t* codes, uint8_t* sf, void* stream) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  if (M < 0 || ldx < prof->K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad M/ldx");
  if (!(eps >= 0.0f) || eps > 3.4e38f) return fail(ARC_ERR_SHAPE, "eps must be finite and >= 0");
  if (M == 0) return ARC_OK;
  if (!x || !gamma || !codes || !sf) return fail(ARC_ERR_NULL, "null x / gamma / codes / sf");
  if (!aligned16(x) || !aligned16(gamma) || !aligned16(codes) || !aligned16(sf))
    return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_quant(x, M, (int)prof->K, ldx, prof->perm, prof->S, prof->gs, (int)prof->layout, 0, codes,
                               sf, (cudaStream_t)stream, gamma, eps);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_rmsnorm_quantize_activation");
}

// ---------------------------------------------------------------- MXFP4-ARC (f3, reading Q25)
arc_status_t arc_mx_tensor_scale(float amax, float* gs) {
  if (!gs) return fail(ARC_ERR_NULL, "null gs");
  if (!(amax >= 0.0f) || amax > 3.4e38f) return fail(ARC_ERR_NONFINITE, "amax must be finite and >= 0");
  int c = 0;
  if (amax > 0.0f) {
    const float raw = amax / 6.0f;
    int x;
    const float f = frexpf(raw, &x);
    c = (f == 0.5f ? x - 1 : x) - 8;
  }
  *gs = ldexpf(1.0f, -c);
  return ARC_OK;
}

arc_status_t arc_mx_tensor_scale_device(const void* x, int64_t rows, int64_t K, int64_t ldx, float* gs_out,
                                        void* stream) {
  if (!x || !gs_out) return fail(ARC_ERR_NULL, "null x / gs_out");
  if (K <= 0 || K % 16 || rows < 0 || ldx < K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad rows/K/ldx");
  if (!aligned16(x)) return fail(ARC_ERR_ALIGN, "x not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_tensor_scale(x, rows, (int)K, ldx, gs_out, (cudaStream_t)stream, 1);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_mx_tensor_scale_device");
}

static arc_status_t check_mx(int64_t K, int32_t S, const float* gs_host_or_null) {
  if (K % 32 || S % 32) return fail(ARC_ERR_ALIGN, "MXFP4-ARC needs K and S multiples of 32");
  (void)gs_host_or_null;
  return ARC_OK;
}

arc_status_t arc_quantize_activation_mx(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                        uint8_t* codes, uint8_t* sf, void* stream) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  s = check_mx(prof->K, prof->S, nullptr);
  if (s != ARC_OK) return s;
  if (M < 0 || ldx < prof->K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad M/ldx");
  if (M == 0) return ARC_OK;
  if (!x || !codes || !sf) return fail(ARC_ERR_NULL, "null x / codes / sf");
  if (!aligned16(x) || !aligned16(codes) || !aligned16(sf)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_quant(x, M, (int)prof->K, ldx, prof->perm, prof->S, prof->gs, (int)prof->layout, 0, codes,
                               sf, (cudaStream_t)stream, nullptr, 0.0f, -1, 1);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_quantize_activation_mx");
}

arc_status_t arc_quantize_weight_mx(const void* w, int64_t N, int64_t K, int64_t ldw, const int32_t* perm, int32_t S,
                                    const float* gs_w, arc_layout_t layout, uint8_t* codes, uint8_t* sf,
                                    void* stream) {
  if (!w || !perm || !gs_w || !codes || !sf) return fail(ARC_ERR_NULL, "null argument");
  arc_status_t s = check_ks(K, S);
  if (s != ARC_OK) return s;
  s = check_mx(K, S, nullptr);
  if (s != ARC_OK) return s;
  if (N < 0 || ldw < K || ldw % 8) return fail(ARC_ERR_SHAPE, "bad N/ldw");
  if (layout != ARC_LAYOUT_INTERLEAVED && layout != ARC_LAYOUT_CONTIGUOUS) return fail(ARC_ERR_SHAPE, "bad layout");
  if (!aligned16(w) || !aligned16(codes) || !aligned16(sf)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  if (N == 0) return ARC_OK;
  cudaError_t e = launch_quant(w, N, (int)K, ldw, perm, S, gs_w, (int)layout, 1, codes, sf, (cudaStream_t)stream,
                               nullptr, 0.0f, -1, 1);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_quantize_weight_mx");
}

static void split_gemm_ws(void* ws, size_t ws_bytes, void** cnt, void** part, size_t* part_bytes);

arc_status_t arc_mx_native_buffer_sizes(int64_t rows, int64_t K, int32_t S, int64_t* Kpm, size_t* code_bytes,
                                        size_t* sf_bytes) {
  if (rows < 0 || K <= 0 || K % 32 || S < 0 || S % 32 || S > K) return fail(ARC_ERR_SHAPE, "bad rows/K/S");
  const int64_t km = round_up(K + S, 128);
  if (Kpm) *Kpm = km;
  if (code_bytes) *code_bytes = (size_t)(rows * (km / 2));
  if (sf_bytes) *sf_bytes = (size_t)(round_up(rows, 128) * (km / 32));
  return ARC_OK;
}

arc_status_t arc_quantize_mx_native(const void* x, int64_t rows, int64_t K, int64_t ldx, const int32_t* perm, int32_t S,
                                    int32_t weight, arc_layout_t layout, uint8_t* codes, uint8_t* sf, void* stream) {
  if (K <= 0 || K % 32 || K > (1 << 20) || S < 0 || S % 32 || S > K || rows < 0 || ldx < K || ldx % 8)
    return fail(ARC_ERR_SHAPE, "bad rows/K/S/ldx");
  if (layout != ARC_LAYOUT_INTERLEAVED && layout != ARC_LAYOUT_CONTIGUOUS) return fail(ARC_ERR_SHAPE, "bad layout");
  if (rows == 0) return ARC_OK;
  if (!x || !perm || !codes || !sf) return fail(ARC_ERR_NULL, "null x / perm / codes / sf");
  if (!aligned16(x) || !aligned16(perm) || !aligned16(codes)) return fail(ARC_ERR_ALIGN, "x / perm / codes not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_mx_native_quant(x, rows, (int)K, (int)S, ldx, perm, weight ? 1 : 0, (int)layout, codes, sf,
                                         (cudaStream_t)stream);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_quantize_mx_native");
}

arc_status_t arc_gemm_mx_native_workspace_size(int64_t M, int64_t N, int64_t Kpm, size_t* bytes) {
  if (!bytes) return fail(ARC_ERR_NULL, "null bytes");
  if (M < 0 || N <= 0 || Kpm <= 0 || Kpm % 128) return fail(ARC_ERR_SHAPE, "bad M/N/Kpm");
  *bytes = M == 0 ? 0 : plan_gemm(M, N, Kpm).ws_bytes;
  return ARC_OK;
}

arc_status_t arc_gemm_mx_native(const uint8_t* a_codes, const uint8_t* a_sf, int64_t M, const uint8_t* b_codes,
                                const uint8_t* b_sf, int64_t N, int64_t Kpm, void* y, arc_dtype_t y_dtype, int64_t ldy,
                                void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || M > (1 << 30) || N <= 0 || N > (1 << 30) || Kpm <= 0 || Kpm % 128) return fail(ARC_ERR_SHAPE, "bad M/N/Kpm");
  if (M == 0) return ARC_OK;
  if (!a_codes || !a_sf || !b_codes || !b_sf || !y) return fail(ARC_ERR_NULL, "null operand / y");
  if (y_dtype != ARC_BF16 && y_dtype != ARC_FP32) return fail(ARC_ERR_SHAPE, "y_dtype must be ARC_BF16 or ARC_FP32");
  if (ldy < N || ldy % (y_dtype == ARC_FP32 ? 4 : 8)) return fail(ARC_ERR_SHAPE, "ldy must be >= N and a multiple of 16 bytes");
  if (!aligned16(a_codes) || !aligned16(a_sf) || !aligned16(b_codes) || !aligned16(b_sf) || !aligned16(y))
    return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  const GemmPlan pl = plan_gemm(M, N, Kpm);
  if (pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes)) return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  void *cnt, *part;
  size_t part_bytes;
  split_gemm_ws(ws, ws_bytes, &cnt, &part, &part_bytes);
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.Kp = Kpm;
  p.a_codes = a_codes;
  p.a_sf = a_sf;
  p.b_codes = b_codes;
  p.b_sf = b_sf;
  p.gs_x = nullptr;
  p.gs_w = nullptr;
  p.y = y;
  p.ldy = ldy;
  p.y_fp32 = y_dtype == ARC_FP32;
  p.cnt = static_cast<unsigned*>(cnt);
  p.ws = part;
  p.ws_bytes = part_bytes;
  p.fmt = 2;
  const char* detail = nullptr;
  cudaError_t e = launch_gemm(p, (cudaStream_t)stream, &detail);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_gemm_mx_native", detail);
}

arc_status_t arc_gemm_w4a8(const uint8_t* a_codes, const uint8_t* a_sf, int64_t M, const uint8_t* b_codes,
                           const uint8_t* b_sf, int64_t N, int64_t K, void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws,
                           size_t ws_bytes, void* stream) {
  if (M < 0 || M > (1 << 30) || N <= 0 || N > (1 << 30) || K <= 0 || K % 32) return fail(ARC_ERR_SHAPE, "bad M/N/K");
  if (M == 0) return ARC_OK;
  if (!a_codes || !a_sf || !b_codes || !b_sf || !y) return fail(ARC_ERR_NULL, "null operand / y");
  if (y_dtype != ARC_BF16 && y_dtype != ARC_FP32) return fail(ARC_ERR_SHAPE, "y_dtype must be ARC_BF16 or ARC_FP32");
  if (ldy < N || ldy % (y_dtype == ARC_FP32 ? 4 : 8)) return fail(ARC_ERR_SHAPE, "ldy must be >= N and a multiple of 16 bytes");
  if (!aligned16(a_codes) || !aligned16(a_sf) || !aligned16(b_codes) || !aligned16(b_sf) || !aligned16(y))
    return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  const int64_t k8 = round_up(K, 128);
  const GemmPlan pl = plan_gemm(M, N, 2 * k8);
  if (pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes)) return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  void *cnt, *part;
  size_t part_bytes;
  split_gemm_ws(ws, ws_bytes, &cnt, &part, &part_bytes);
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.Kp = k8;
  p.a_codes = a_codes;
  p.a_sf = a_sf;
  p.b_codes = b_codes;
  p.b_sf = b_sf;
  p.gs_x = nullptr;
  p.gs_w = nullptr;
  p.y = y;
  p.ldy = ldy;
  p.y_fp32 = y_dtype == ARC_FP32;
  p.cnt = static_cast<unsigned*>(cnt);
  p.ws = part;
  p.ws_bytes = part_bytes;
  p.fmt = 3;
  const char* detail = nullptr;
  cudaError_t e = launch_gemm(p, (cudaStream_t)stream, &detail);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_gemm_w4a8", detail);
}

arc_status_t arc_mxfp8_buffer_sizes(int64_t rows, int64_t K, int64_t* Kp8, size_t* code_bytes, size_t* sf_bytes) {
  if (rows < 0 || K <= 0 || K % 32) return fail(ARC_ERR_SHAPE, "rows >= 0, K > 0, K % 32 == 0 required");
  const int64_t k8 = round_up(K, 128);
  if (Kp8) *Kp8 = k8;
  if (code_bytes) *code_bytes = (size_t)(rows * k8);
  if (sf_bytes) *sf_bytes = (size_t)(round_up(rows, 128) * (k8 / 32));
  return ARC_OK;
}

arc_status_t arc_quantize_mxfp8(const void* x, int64_t rows, int64_t K, int64_t ldx, uint8_t* codes, uint8_t* sf,
                                void* stream) {
  if (K <= 0 || K % 32 || K > (1 << 20) || rows < 0 || ldx < K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad rows/K/ldx");
  if (rows == 0) return ARC_OK;
  if (!x || !codes || !sf) return fail(ARC_ERR_NULL, "null x / codes / sf");
  if (!aligned16(x) || !aligned16(codes)) return fail(ARC_ERR_ALIGN, "x / codes not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_mxfp8_quant(x, rows, (int)K, ldx, codes, sf, (cudaStream_t)stream);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_quantize_mxfp8");
}

arc_status_t arc_gemm_mxfp8_workspace_size(int64_t M, int64_t N, int64_t K, size_t* bytes) {
  if (!bytes) return fail(ARC_ERR_NULL, "null bytes");
  if (M < 0 || N <= 0 || K <= 0 || K % 32) return fail(ARC_ERR_SHAPE, "bad M/N/K");
  *bytes = M == 0 ? 0 : plan_gemm(M, N, 2 * round_up(K, 128)).ws_bytes;
  return ARC_OK;
}

arc_status_t arc_gemm_mxfp8(const uint8_t* a_codes, const uint8_t* a_sf, int64_t M, const uint8_t* b_codes,
                            const uint8_t* b_sf, int64_t N, int64_t K, void* y, arc_dtype_t y_dtype, int64_t ldy,
                            void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || M > (1 << 30) || N <= 0 || N > (1 << 30) || K <= 0 || K % 32) return fail(ARC_ERR_SHAPE, "bad M/N/K");
  if (M == 0) return ARC_OK;
  if (!a_codes || !a_sf || !b_codes || !b_sf || !y) return fail(ARC_ERR_NULL, "null operand / y");
  if (y_dtype != ARC_BF16 && y_dtype != ARC_FP32) return fail(ARC_ERR_SHAPE, "y_dtype must be ARC_BF16 or ARC_FP32");
  if (ldy < N || ldy % (y_dtype == ARC_FP32 ? 4 : 8)) return fail(ARC_ERR_SHAPE, "ldy must be >= N and a multiple of 16 bytes");
  if (!aligned16(a_codes) || !aligned16(a_sf) || !aligned16(b_codes) || !aligned16(b_sf) || !aligned16(y))
    return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  const int64_t k8 = round_up(K, 128);
  const GemmPlan pl = plan_gemm(M, N, 2 * k8);
  if (pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes)) return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  void *cnt, *part;
  size_t part_bytes;
  split_gemm_ws(ws, ws_bytes, &cnt, &part, &part_bytes);
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.Kp = k8;
  p.a_codes = a_codes;
  p.a_sf = a_sf;
  p.b_codes = b_codes;
  p.b_sf = b_sf;
  p.gs_x = nullptr;  // MX formats carry no tensor scale: alpha = 1
  p.gs_w = nullptr;
  p.y = y;
  p.ldy = ldy;
  p.y_fp32 = y_dtype == ARC_FP32;
  p.cnt = static_cast<unsigned*>(cnt);
  p.ws = part;
  p.ws_bytes = part_bytes;
  p.fmt = 1;
  const char* detail = nullptr;
  cudaError_t e = launch_gemm(p, (cudaStream_t)stream, &detail);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_gemm_mxfp8", detail);
}

arc_status_t arc_silu_mul(const void* gu, int64_t M, int64_t K, int64_t ld, int64_t up_off, void* h, int64_t ldh,
                          void* stream) {
  const bool pairs = up_off == ARC_GU_PAIRS;
  if (K <= 0 || K % 16 || K > 32768 || M < 0 || (!pairs && (up_off < K || up_off % 8)) ||
      ld < (pairs ? 2 * K : up_off + K) || ld % 8 || ldh < K || ldh % 8)
    return fail(ARC_ERR_SHAPE, "bad M/K/ld/up_off/ldh");
  if (M == 0) return ARC_OK;
  if (!gu || !h) return fail(ARC_ERR_NULL, "null gu / h");
  if (!aligned16(gu) || !aligned16(h)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  arc_status_t s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_silu_mul(gu, M, (int)K, ld, pairs ? -2 : up_off, h, ldh, (cudaStream_t)stream);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_silu_mul");
}

arc_status_t arc_silu_mul_quantize_activation(const void* gu, int64_t M, int64_t ld, int64_t up_off,
                                              const arc_profile_t* prof, uint8_t* codes, uint8_t* sf, void* stream) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  const int64_t K = prof->K;
  if (K > 16384) return fail(ARC_ERR_UNSUPPORTED, "SiLU-mul quantize supports K <= 16384");
  const bool pairs = up_off == ARC_GU_PAIRS;
  if (M < 0 || (!pairs && (up_off < K || up_off % 8)) || ld < (pairs ? 2 * K : up_off + K) || ld % 8)
    return fail(ARC_ERR_SHAPE, "bad M/ld/up_off");
  if (M == 0) return ARC_OK;
  if (!gu || !codes || !sf) return fail(ARC_ERR_NULL, "null gu / codes / sf");
  if (!aligned16(gu) || !aligned16(codes) || !aligned16(sf)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = launch_quant(gu, M, (int)K, ld, prof->perm, prof->S, prof->gs, (int)prof->layout, 0, codes, sf,
                               (cudaStream_t)stream, nullptr, 0.0f, pairs ? -2 : up_off);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_silu_mul_quantize_activation");
}

static arc_status_t gemm_impl(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                              const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* cnt,
                              void* part, size_t part_bytes, void* stream, int weights_ready);

// A public GEMM workspace is [kGemmCounterBytes of tile counters | fp32 partials].
static void split_gemm_ws(void* ws, size_t ws_bytes, void** cnt, void** part, size_t* part_bytes) {
  *cnt = ws;
  *part = ws && ws_bytes >= kGemmCounterBytes ? static_cast<uint8_t*>(ws) + kGemmCounterBytes : nullptr;
  *part_bytes = ws_bytes >= kGemmCounterBytes ? ws_bytes - kGemmCounterBytes : 0;
}

arc_status_t arc_gemm(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                      const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws, size_t ws_bytes,
                      void* stream) {
  const GemmPlan pl = M > 0 && check_qweight(qw) == ARC_OK ? plan_gemm(M, qw->N, qw->Kp) : GemmPlan{};
  if (M > 0 && pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes))
    return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  void *cnt, *part;
  size_t part_bytes;
  split_gemm_ws(ws, ws_bytes, &cnt, &part, &part_bytes);
  return gemm_impl(a_codes, a_sf, gs_x, M, qw, y, y_dtype, ldy, cnt, part, part_bytes, stream, 0);
}

// weights_ready: the caller knows the weights were complete before the kernel preceding this GEMM
// started (arc_linear*: that kernel is its own activation quantize), so the decode-size kernel may
// stream them before griddepcontrol.wait.
static arc_status_t gemm_impl(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                              const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* cnt,
                              void* part, size_t part_bytes, void* stream, int weights_ready) {
  arc_status_t s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (M < 0 || M > (1 << 30)) return fail(ARC_ERR_SHAPE, "bad M");
  if (M == 0) return ARC_OK;
  if (!a_codes || !a_sf || !gs_x || !y) return fail(ARC_ERR_NULL, "null a_codes / a_sf / gs_x / y");
  if (y_dtype != ARC_BF16 && y_dtype != ARC_FP32) return fail(ARC_ERR_SHAPE, "y_dtype must be ARC_BF16 or ARC_FP32");
  if (ldy < qw->N || ldy % (y_dtype == ARC_FP32 ? 4 : 8))
    return fail(ARC_ERR_SHAPE, "ldy must be >= N and a multiple of 16 bytes");
  if (!aligned16(a_codes) || !aligned16(a_sf) || !aligned16(y)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  const GemmPlan pl = plan_gemm(M, qw->N, qw->Kp);
  if (pl.ws_bytes > 0 && (!cnt || !part || part_bytes + kGemmCounterBytes < pl.ws_bytes))
    return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  if ((cnt && !aligned16(cnt)) || (part && !aligned16(part))) return fail(ARC_ERR_ALIGN, "ws not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  GemmProblem p;
  p.M = M;
  p.N = qw->N;
  p.Kp = qw->Kp;
  p.a_codes = a_codes;
  p.a_sf = a_sf;
  p.b_codes = qw->codes;
  p.b_sf = qw->sf;
  p.gs_x = gs_x;
  p.gs_w = qw->gs;
  p.y = y;
  p.ldy = ldy;
  p.y_fp32 = y_dtype == ARC_FP32;
  p.cnt = static_cast<unsigned*>(cnt);
  p.ws = part;
  p.ws_bytes = part_bytes;
  p.weights_ready = weights_ready;
  const char* detail = nullptr;
  cudaError_t e = launch_gemm(p, (cudaStream_t)stream, &detail);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_gemm", detail);
}

arc_status_t arc_gemm_reduce(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                             const arc_qweight_t* qw, const arc_reduce_t* red, int64_t ldy, void* ws, size_t ws_bytes,
                             void* stream) {
  arc_status_t s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (!red) return fail(ARC_ERR_NULL, "null red");
  if (M < 0 || M > (1 << 30)) return fail(ARC_ERR_SHAPE, "bad M");
  if (M == 0) return ARC_OK;
  if (!a_codes || !a_sf || !gs_x) return fail(ARC_ERR_NULL, "null a_codes / a_sf / gs_x");
  if (ldy < qw->N || ldy % 4) return fail(ARC_ERR_SHAPE, "ldy must be >= N and a multiple of 4");
  if (red->mode == ARC_REDUCE_MULTIMEM) {
    if (!red->mc) return fail(ARC_ERR_NULL, "null multicast address");
    if (!aligned16(red->mc)) return fail(ARC_ERR_ALIGN, "multicast address not 16B aligned");
  } else if (red->mode == ARC_REDUCE_PEERS) {
    if (red->npeers < 1 || red->npeers > 8) return fail(ARC_ERR_SHAPE, "npeers must be 1..8");
    for (int i = 0; i < red->npeers; ++i) {
      if (!red->peers[i]) return fail(ARC_ERR_NULL, "null peer buffer");
      if (!aligned16(red->peers[i])) return fail(ARC_ERR_ALIGN, "peer buffer not 16B aligned");
    }
  } else {
    return fail(ARC_ERR_SHAPE, "bad reduce mode");
  }
  if (!aligned16(a_codes) || !aligned16(a_sf)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  const GemmPlan pl = plan_gemm(M, qw->N, qw->Kp);
  if (pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes)) return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  if (ws && !aligned16(ws)) return fail(ARC_ERR_ALIGN, "ws not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  void *cnt, *part;
  size_t part_bytes;
  split_gemm_ws(ws, ws_bytes, &cnt, &part, &part_bytes);
  GemmProblem p;
  p.M = M;
  p.N = qw->N;
  p.Kp = qw->Kp;
  p.a_codes = a_codes;
  p.a_sf = a_sf;
  p.b_codes = qw->codes;
  p.b_sf = qw->sf;
  p.gs_x = gs_x;
  p.gs_w = qw->gs;
  p.y = red->mode == ARC_REDUCE_MULTIMEM ? (void*)red->mc : (void*)red->peers[0];
  p.ldy = ldy;
  p.y_fp32 = 1;
  p.cnt = static_cast<unsigned*>(cnt);
  p.ws = part;
  p.ws_bytes = part_bytes;
  p.red_mode = red->mode;
  p.red_np = red->mode == ARC_REDUCE_PEERS ? red->npeers : 0;
  p.red_mc = red->mc;
  for (int i = 0; i < p.red_np; ++i) p.red_peer[i] = red->peers[i];
  const char* detail = nullptr;
  cudaError_t e = launch_gemm(p, (cudaStream_t)stream, &detail);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_gemm_reduce", detail);
}

arc_status_t arc_gemm_swiglu(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                             const arc_qweight_t* qw, void* h, int64_t ldh, void* ws, size_t ws_bytes, void* stream) {
  arc_status_t s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (M < 0 || M > (1 << 30)) return fail(ARC_ERR_SHAPE, "bad M");
  if (qw->N % 32) return fail(ARC_ERR_SHAPE, "SwiGLU weight N must be a multiple of 32 (16-row gate/up groups)");
  if (ldh < qw->N / 2 || ldh % 8) return fail(ARC_ERR_SHAPE, "ldh must be >= N/2 and a multiple of 8");
  if (M == 0) return ARC_OK;
  if (!a_codes || !a_sf || !gs_x || !h) return fail(ARC_ERR_NULL, "null a_codes / a_sf / gs_x / h");
  if (!aligned16(a_codes) || !aligned16(a_sf) || !aligned16(h)) return fail(ARC_ERR_ALIGN, "buffer not 16B aligned");
  const GemmPlan pl = plan_gemm(M, qw->N, qw->Kp);
  if (pl.ws_bytes > 0 && (!ws || ws_bytes < pl.ws_bytes)) return fail(ARC_ERR_WORKSPACE, "split-K workspace too small");
  if (ws && !aligned16(ws)) return fail(ARC_ERR_ALIGN, "ws not 16B aligned");
  s = check_device();
  if (s != ARC_OK) return s;
  void *cnt, *part;
  size_t part_bytes;
  split_gemm_ws(ws, ws_bytes, &cnt, &part, &part_bytes);
  GemmProblem p;
  p.M = M;
  p.N = qw->N;
  p.Kp = qw->Kp;
  p.a_codes = a_codes;
  p.a_sf = a_sf;
  p.b_codes = qw->codes;
  p.b_sf = qw->sf;
  p.gs_x = gs_x;
  p.gs_w = qw->gs;
  p.y = h;
  p.ldy = ldh;
  p.y_fp32 = 0;
  p.swiglu = 1;
  p.cnt = static_cast<unsigned*>(cnt);
  p.ws = part;
  p.ws_bytes = part_bytes;
  const char* detail = nullptr;
  cudaError_t e = launch_gemm(p, (cudaStream_t)stream, &detail);
  return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_gemm_swiglu", detail);
}

arc_status_t arc_linear_ex(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof, const arc_qweight_t* qw,
                           void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws, size_t ws_bytes, int flags,
                           void* stream) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (qw->K != prof->K || qw->S != prof->S || qw->layout != prof->layout)
    return fail(ARC_ERR_SHAPE, "profile and qweight disagree on K / S / layout");
  const int x_f16 = (flags & ARC_LINEAR_X_FP16) ? 1 : 0;
  flags &= ~ARC_LINEAR_X_FP16;
  if (flags != ARC_LINEAR_AUTO && flags != ARC_LINEAR_FUSED && flags != ARC_LINEAR_UNFUSED)
    return fail(ARC_ERR_SHAPE, "bad flags");
  if (x_f16) flags = ARC_LINEAR_UNFUSED;  // fp16 rows: the two-kernel path (its quantize takes ARC_FP16)
  if (M < 0 || M > (1 << 30)) return fail(ARC_ERR_SHAPE, "bad M");
  if (M == 0) return ARC_OK;
  if (!ws || !x || !y) return fail(ARC_ERR_NULL, "null x / y / workspace");
  if (ldx < prof->K || ldx % 8) return fail(ARC_ERR_SHAPE, "bad ldx");
  if (y_dtype != ARC_BF16 && y_dtype != ARC_FP32) return fail(ARC_ERR_SHAPE, "y_dtype must be ARC_BF16 or ARC_FP32");
  if (ldy < qw->N || ldy % (y_dtype == ARC_FP32 ? 4 : 8))
    return fail(ARC_ERR_SHAPE, "ldy must be >= N and a multiple of 16 bytes");
  const size_t sync = sync_bytes_of(qw->N);
  if (ws_bytes < sync + linear_rest_bytes(M, qw, flags)) return fail(ARC_ERR_WORKSPACE, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return fail(ARC_ERR_ALIGN, "workspace not 256B aligned");
  if (!aligned16(x) || !aligned16(y)) return fail(ARC_ERR_ALIGN, "x / y not 16B aligned");
  uint8_t* rest = static_cast<uint8_t*>(ws) + sync;
  const size_t rest_bytes = ws_bytes - sync;
  uint8_t* codes = rest;
  uint8_t* sf = codes + round_up(M * (qw->Kp / 2), 256);
  const size_t act = act_ws_bytes(M, qw->K, qw->S);
  // ARC_LINEAR_FUSED at decode-size M: one kernel quantizes the activation into the workspace and runs
  // the stream-K GEMM.  AUTO runs the two-kernel path at every M: the direct-gather quantize + the
  // cluster split-K GEMM (decode_gemm.cu) measured faster than the fused kernel from M = 1.
  const StreamPlan sp = plan_stream(M, qw->N, qw->Kp);
  if (flags == ARC_LINEAR_FUSED && sp.ok) {
    // decode-size M: one kernel quantizes the activation into the workspace and runs the stream-K GEMM
    s = check_device();
    if (s != ARC_OK) return s;
    if (!aligned16(prof->perm)) return fail(ARC_ERR_ALIGN, "perm not 16B aligned");
    GemmProblem p;
    p.M = M;
    p.N = qw->N;
    p.Kp = qw->Kp;
    p.a_codes = codes;
    p.a_sf = sf;
    p.b_codes = qw->codes;
    p.b_sf = qw->sf;
    p.gs_x = prof->gs;
    p.gs_w = qw->gs;
    p.y = y;
    p.ldy = ldy;
    p.y_fp32 = y_dtype == ARC_FP32;
    p.cnt = static_cast<unsigned*>(ws);
    p.ws = rest + act;
    p.ws_bytes = rest_bytes - act;
    p.weights_ready = 1;
    StreamQuant fq{x, ldx, prof->perm, (int)prof->K, (int)prof->S, (int)prof->layout};
    const char* detail = nullptr;
    cudaError_t e = launch_stream_gemm(p, sp, (cudaStream_t)stream, &detail, &fq);
    return e == cudaSuccess ? ARC_OK : cuda_fail(e, "arc_linear (fused decode)", detail);
  }
  s = quantize_activation_impl(x, M, ldx, prof, codes, sf, stream, 1, x_f16);
  if (s != ARC_OK) return s;
  return gemm_impl(codes, sf, prof->gs, M, qw, y, y_dtype, ldy, ws, rest + act, rest_bytes - act, stream, 1);
}

arc_status_t arc_linear_rmsnorm(const void* x, int64_t M, int64_t ldx, const void* gamma, float eps,
                                const arc_profile_t* prof, const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype,
                                int64_t ldy, void* ws, size_t ws_bytes, void* stream) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (qw->K != prof->K || qw->S != prof->S || qw->layout != prof->layout)
    return fail(ARC_ERR_SHAPE, "profile and qweight disagree on K / S / layout");
  if (M < 0 || M > (1 << 30)) return fail(ARC_ERR_SHAPE, "bad M");
  if (M == 0) return ARC_OK;
  if (!ws) return fail(ARC_ERR_NULL, "null workspace");
  const size_t sync = sync_bytes_of(qw->N);
  if (ws_bytes < sync + linear_rest_bytes(M, qw, ARC_LINEAR_UNFUSED)) return fail(ARC_ERR_WORKSPACE, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return fail(ARC_ERR_ALIGN, "workspace not 256B aligned");
  uint8_t* codes = static_cast<uint8_t*>(ws) + sync;
  uint8_t* sf = codes + round_up(M * (qw->Kp / 2), 256);
  const size_t act = act_ws_bytes(M, qw->K, qw->S);
  s = arc_rmsnorm_quantize_activation(x, M, ldx, gamma, eps, prof, codes, sf, stream);
  if (s != ARC_OK) return s;
  return gemm_impl(codes, sf, prof->gs, M, qw, y, y_dtype, ldy, ws, codes + act, ws_bytes - sync - act, stream, 1);
}

arc_status_t arc_linear_silu_mul(const void* gu, int64_t M, int64_t ld, int64_t up_off, const arc_profile_t* prof,
                                 const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws,
                                 size_t ws_bytes, void* stream) {
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (qw->K != prof->K || qw->S != prof->S || qw->layout != prof->layout)
    return fail(ARC_ERR_SHAPE, "profile and qweight disagree on K / S / layout");
  if (M < 0 || M > (1 << 30)) return fail(ARC_ERR_SHAPE, "bad M");
  if (M == 0) return ARC_OK;
  if (!ws) return fail(ARC_ERR_NULL, "null workspace");
  const size_t sync = sync_bytes_of(qw->N);
  if (ws_bytes < sync + linear_rest_bytes(M, qw, ARC_LINEAR_UNFUSED)) return fail(ARC_ERR_WORKSPACE, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(ws) & 255u) != 0) return fail(ARC_ERR_ALIGN, "workspace not 256B aligned");
  uint8_t* codes = static_cast<uint8_t*>(ws) + sync;
  uint8_t* sf = codes + round_up(M * (qw->Kp / 2), 256);
  const size_t act = act_ws_bytes(M, qw->K, qw->S);
  s = arc_silu_mul_quantize_activation(gu, M, ld, up_off, prof, codes, sf, stream);
  if (s != ARC_OK) return s;
  return gemm_impl(codes, sf, prof->gs, M, qw, y, y_dtype, ldy, ws, codes + act, ws_bytes - sync - act, stream, 1);
}

arc_status_t arc_linear(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof, const arc_qweight_t* qw,
                        void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws, size_t ws_bytes, void* stream) {
  return arc_linear_ex(x, M, ldx, prof, qw, y, y_dtype, ldy, ws, ws_bytes, ARC_LINEAR_AUTO, stream);
}

arc_status_t arc_linear_ex_workspace_size(int64_t M, const arc_qweight_t* qw, int flags, size_t* bytes) {
  arc_status_t s = check_qweight(qw);
  if (s != ARC_OK) return s;
  if (!bytes) return fail(ARC_ERR_NULL, "null bytes");
  if (M < 0) return fail(ARC_ERR_SHAPE, "M < 0");
  flags &= ~ARC_LINEAR_X_FP16;
  if (flags != ARC_LINEAR_AUTO && flags != ARC_LINEAR_FUSED && flags != ARC_LINEAR_UNFUSED)
    return fail(ARC_ERR_SHAPE, "bad flags");
  *bytes = sync_bytes_of(qw->N) + (M == 0 ? 0 : linear_rest_bytes(M, qw, flags));
  return ARC_OK;
}


// rows per pipelined chunk of arc_linear_hostio: a multiple of 128, ~8 chunks per call (one below 512 rows)
static int64_t hostio_chunk_rows(int64_t M) { return M < 512 ? M : round_up((M + 7) / 8, 128); }

arc_status_t arc_linear_hostio_workspace_size(int64_t M, const arc_qweight_t* qw, arc_dtype_t y_dtype,
                                              size_t* bytes) {
  // the chunks share one arc_linear workspace: the largest any chunk size needs
  const int64_t mc = hostio_chunk_rows(M), tail = M > 0 ? M - (M - 1) / mc * mc : 0;
  size_t w = 0, w1 = 0, w2 = 0;
  arc_status_t s = arc_linear_workspace_size(M, qw, &w);
  if (s != ARC_OK) return s;
  if ((s = arc_linear_workspace_size(mc, qw, &w1)) != ARC_OK || (s = arc_linear_workspace_size(tail, qw, &w2)) != ARC_OK)
    return s;
  w = std::max(w, std::max(w1, w2));
  const int64_t yb = M * qw->N * (y_dtype == ARC_FP32 ? 4 : 2);
  *bytes = round_up((int64_t)w, 256) + (size_t)round_up(M * qw->K * 2, 256) + (size_t)round_up(yb, 256);
  return ARC_OK;
}

// Host-IO pipeline: per device, two library-owned non-blocking streams (host->device copies, device->host
// copies) and a ring of events; created on first use.  A call splits its rows into chunks: chunk i's H2D
// runs on the copy-in stream, its arc_linear on the caller's stream once the H2D event fired, its D2H on
// the copy-out stream once the compute event fired -- copies of one chunk overlap the compute of the next
// and, across consecutive async calls, device->host and host->device copies overlap (PCIe is full duplex).
namespace {
struct HostIo {
  std::mutex mu;
  bool init = false;
  cudaError_t err = cudaSuccess;
  cudaStream_t in = nullptr, out = nullptr;
  static constexpr int kEv = 512;
  cudaEvent_t ev[kEv];
  int next = 0;
  cudaEvent_t get() { cudaEvent_t e = ev[next]; next = (next + 1) % kEv; return e; }
};
HostIo g_hio[64];
HostIo* hostio_for_device(cudaError_t* err) {
  int dev = 0;
  *err = cudaGetDevice(&dev);
  if (*err != cudaSuccess) return nullptr;
  if (dev < 0 || dev >= 64) { *err = cudaErrorInvalidDevice; return nullptr; }
  HostIo* h = &g_hio[dev];
  std::lock_guard<std::mutex> g(h->mu);
  if (!h->init) {
    h->init = true;
    h->err = cudaStreamCreateWithFlags(&h->in, cudaStreamNonBlocking);
    if (h->err == cudaSuccess) h->err = cudaStreamCreateWithFlags(&h->out, cudaStreamNonBlocking);
    for (int i = 0; i < HostIo::kEv && h->err == cudaSuccess; ++i)
      h->err = cudaEventCreateWithFlags(&h->ev[i], cudaEventDisableTiming);
  }
  *err = h->err;
  return h->err == cudaSuccess ? h : nullptr;
}
}  // namespace

static arc_status_t hostio_enqueue(const void* x_host, int64_t M, const arc_profile_t* prof, const arc_qweight_t* qw,
                                   void* y_host, arc_dtype_t y_dtype, void* ws, size_t ws_bytes, void* stream,
                                   HostIo** hio_out) {
  if (!x_host || !y_host || !ws) return fail(ARC_ERR_NULL, "null x_host / y_host / ws");
  arc_status_t s = check_profile(prof);
  if (s != ARC_OK) return s;
  s = check_qweight(qw);
  if (s != ARC_OK) return s;
  size_t need = 0;
  s = arc_linear_hostio_workspace_size(M, qw, y_dtype, &need);
  if (s != ARC_OK) return s;
  if (ws_bytes < need) return fail(ARC_ERR_WORKSPACE, "workspace too small");
  if (M == 0) return ARC_OK;
  s = check_device();
  if (s != ARC_OK) return s;
  cudaError_t e = cudaSuccess;
  HostIo* h = hostio_for_device(&e);
  if (!h) return cuda_fail(e, "arc_linear_hostio streams");
  *hio_out = h;
  const int64_t mc = hostio_chunk_rows(M), tail = M - (M - 1) / mc * mc;
  size_t lin = 0, l1 = 0, l2 = 0;
  arc_linear_workspace_size(M, qw, &lin);
  arc_linear_workspace_size(mc, qw, &l1);
  arc_linear_workspace_size(tail, qw, &l2);
  lin = (size_t)round_up((int64_t)std::max(lin, std::max(l1, l2)), 256);
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* xd = base + lin;
  uint8_t* yd = base + lin + round_up(M * prof->K * 2, 256);
  const int64_t xrow = prof->K * 2, yrow = qw->N * (y_dtype == ARC_FP32 ? 4 : 2);
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> g(h->mu);
  // the copies into this workspace start after the work already enqueued on the caller's stream
  cudaEvent_t e0 = h->get();
  if ((e = cudaEventRecord(e0, st)) != cudaSuccess || (e = cudaStreamWaitEvent(h->in, e0, 0)) != cudaSuccess)
    return cuda_fail(e, "arc_linear_hostio order");
  for (int64_t r0 = 0; r0 < M; r0 += mc) {
    const int64_t rows = std::min<int64_t>(mc, M - r0);
    cudaEvent_t ein = h->get(), ec = h->get();
    e = cudaMemcpyAsync(xd + r0 * xrow, static_cast<const uint8_t*>(x_host) + r0 * xrow, (size_t)(rows * xrow),
                        cudaMemcpyHostToDevice, h->in);
    if (e == cudaSuccess) e = cudaEventRecord(ein, h->in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ein, 0);
    if (e != cudaSuccess) return cuda_fail(e, "arc_linear_hostio H2D");
    // chunks reuse the linear workspace in stream order (the compute of the chunks is serial on st)
    s = arc_linear(xd + r0 * xrow, rows, prof->K, prof, qw, yd + r0 * yrow, y_dtype, qw->N, base, lin, stream);
    if (s != ARC_OK) return s;
    e = cudaEventRecord(ec, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->out, ec, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<uint8_t*>(y_host) + r0 * yrow, yd + r0 * yrow, (size_t)(rows * yrow),
                          cudaMemcpyDeviceToHost, h->out);
    if (e != cudaSuccess) return cuda_fail(e, "arc_linear_hostio D2H");
  }
  return ARC_OK;
}

arc_status_t arc_linear_hostio_async(const void* x_host, int64_t M, const arc_profile_t* prof, const arc_qweight_t* qw,
                                     void* y_host, arc_dtype_t y_dtype, void* ws, size_t ws_bytes, void* stream) {
  HostIo* h = nullptr;
  return hostio_enqueue(x_host, M, prof, qw, y_host, y_dtype, ws, ws_bytes, stream, &h);
}

arc_status_t arc_linear_hostio_wait(void* stream) {
  cudaError_t e = cudaSuccess;
  HostIo* h = hostio_for_device(&e);
  if (!h) return cuda_fail(e, "arc_linear_hostio streams");
  if ((e = cudaStreamSynchronize(h->in)) != cudaSuccess || (e = cudaStreamSynchronize((cudaStream_t)stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(h->out)) != cudaSuccess)
    return cuda_fail(e, "arc_linear_hostio_wait");
  return ARC_OK;
}

arc_status_t arc_linear_hostio(const void* x_host, int64_t M, const arc_profile_t* prof, const arc_qweight_t* qw,
                               void* y_host, arc_dtype_t y_dtype, void* ws, size_t ws_bytes, void* stream) {
  HostIo* h = nullptr;
  arc_status_t s = hostio_enqueue(x_host, M, prof, qw, y_host, y_dtype, ws, ws_bytes, stream, &h);
  if (s != ARC_OK || M == 0) return s;
  return arc_linear_hostio_wait(stream);
}

}  // extern "C"
