/*
 * arc.h -- C ABI of libarc.so, the B200-native (sm_100a) ARCQuant hot path.
 *
 * ARCQuant (arxiv 2601.07475) keeps a linear layer Y = X W^T ("Problem
 * Definition") in a strictly unified NVFP4 W4A4 data path by appending, along the
 * reduction dimension, the NVFP4-quantized residuals of the S calibrated outlier
 * channels of X and a duplicate of the matching quantized weight columns, so one
 * block-scaled GEMM over K+S computes the primary product plus the correction
 * (§3.2, Eq.2).  This header exposes the calls of the paper's problem
 * statement: calibration (arc_calib_absmax + arc_select_outliers),
 * offline weight preparation (arc_quantize_weight), online activation
 * quantization (arc_quantize_activation, P:138 + the fused kernel of P:164), and
 * the augmented GEMM (arc_gemm / arc_linear).
 *
 * Notation: M = tokens, K = input features, N = output features,
 * S = augmented (outlier) channels, a multiple of 16 with 0 <= S <= K; K + S <= 32768.
 * Ka = K+S; Kp = roundup(Ka, 64) is the physical reduction length.
 *
 * Data formats (all produced and consumed by this library):
 *  - codes: uint8 [rows][Kp/2]; physical element 2j in the low nibble of byte
 *    j (E2M1: 1 sign, 2 exponent, 1 mantissa bit; Table 7).
 *  - sf: E4M3 block scales (Table 7), one per 16 physical elements, in the
 *    tcgen05 / cuBLASLt 128x4 tile layout: byte of (row m, scale column c) at
 *    ((m>>7)*(Kp/64) + (c>>2))*512 + (m&31)*16 + ((m>>5)&3)*4 + (c&3).
 *    The buffer holds roundup(rows,128)*Kp/16 bytes; bytes of rows >= rows in
 *    the last 128-row tile are left unspecified (they only feed discarded
 *    output rows/columns).
 *  - value of an element = e2m1(code) * e4m3(sf) / gs, gs the FP32 tensor scale
 *    ("secondary per-tensor scaling factor"), gs = 2688/amax.
 *  - physical block order: ARC_LAYOUT_INTERLEAVED places the residual block of
 *    outlier block j right after it (App.D); ARC_LAYOUT_CONTIGUOUS is
 *    the logical concatenation [Q_X | Q_Ro].  Blocks Ka/16..Kp/16-1 are
 *    zero codes with scale 0x00.
 *
 * Conventions for every call:
 *  - Pointers are DEVICE pointers unless the parameter name ends in _host.
 *  - Buffers are owned by the caller; the library keeps no pointer after a call
 *    returns, allocates no device memory and never synchronizes the device.
 *    Device work is enqueued on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) and is asynchronous.
 *  - Argument checks are synchronous and happen before anything is enqueued:
 *    ARC_ERR_NULL (null pointer), ARC_ERR_SHAPE (K <= 0, K%16, S%16, S < 0,
 *    S > K, K + S > 32768, M < 0, N <= 0, leading dimension < K or not a multiple of 8
 *    elements, profile / qweight mismatch), ARC_ERR_ALIGN (a base pointer not
 *    16-byte aligned), ARC_ERR_WORKSPACE (workspace too small),
 *    ARC_ERR_UNSUPPORTED (the current device is not sm_100; there is no
 *    fallback of any kind), ARC_ERR_CUDA (a CUDA call or launch failed; text in
 *    arc_last_error()).  M == 0 (no rows) is a successful no-op; the row
 *    buffers may then be NULL.
 *  - Non-finite device inputs are not detected; their outputs are unspecified.
 *  - Calls are reentrant; concurrent calls on different streams are allowed.
 */
#ifndef ARC_H_
#define ARC_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ARC_API __attribute__((visibility("default")))
#else
#define ARC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ARC_OK = 0,
  ARC_ERR_NULL = 1,
  ARC_ERR_SHAPE = 2,
  ARC_ERR_ALIGN = 3,
  ARC_ERR_UNSUPPORTED = 4,
  ARC_ERR_WORKSPACE = 5,
  ARC_ERR_CUDA = 6,
  ARC_ERR_NONFINITE = 7
} arc_status_t;

/* Element types.  Inputs (activations, weights, calibration rows): ARC_BF16 everywhere, ARC_FP16 through the
 * _ex entry points (arc_calib_absmax_ex, arc_tensor_scale_ex, arc_quantize_weight_ex, arc_quantize_activation_ex,
 * arc_linear_ex with ARC_LINEAR_X_FP16); fp16 values are decoded exactly to fp32 before the same STAGE
 * arithmetic.  Outputs: ARC_BF16 or ARC_FP32. */
typedef enum { ARC_BF16 = 0, ARC_FP16 = 1, ARC_FP32 = 2 } arc_dtype_t;

typedef enum { ARC_LAYOUT_INTERLEAVED = 0, ARC_LAYOUT_CONTIGUOUS = 1 } arc_layout_t;

/* Calibration profile of one activation site (the q/k/v projections share one,
 * gate/up share one): "pre-determine both the channel reordering indices
 * and the number of outlier channels S". */
typedef struct {
  int64_t K;              /* input features                                       */
  int32_t S;              /* augmented channels, multiple of 16, 0 <= S <= K      */
  const int32_t* perm;    /* device int32[K]: reordered position i reads channel
                             perm[i]; perm[0:S] are the outlier channels  */
  const float* gs;        /* device scalar: activation encode tensor scale
                             2688/M_calib (static, reading Q4)                    */
  arc_layout_t layout;
} arc_profile_t;

/* A prepared (quantized, reordered, outlier-duplicated) weight. */
typedef struct {
  int64_t N, K, Kp;
  int32_t S;
  arc_layout_t layout;
  const uint8_t* codes;   /* device [N][Kp/2]                                     */
  const uint8_t* sf;      /* device roundup(N,128)*Kp/16, 128x4 tile layout       */
  const float* gs;        /* device scalar gs_w = 2688/amax(W)                    */
} arc_qweight_t;

/* ---------------------------------------------------------------- utilities */
ARC_API const char* arc_status_string(arc_status_t s);
/* Thread-local text of the last ARC_ERR_CUDA / argument error of this thread. */
ARC_API const char* arc_last_error(void);
/* 1 if the current CUDA device is sm_100 (B200-class), else 0. */
ARC_API int arc_device_supported(void);
/* Sizes of a quantized operand of `rows` rows (codes / sf bytes, Kp). */
ARC_API arc_status_t arc_buffer_sizes(int64_t rows, int64_t K, int32_t S, int64_t* Kp, size_t* code_bytes,
                              size_t* sf_bytes);
/* Workspace arc_gemm needs for M rows against qw: 0 when the GEMM is not split, else 16 KB of
 * per-tile arrival counters (offset 0) followed by the fp32 partials of the decode-size split
 * paths.  Zero it once before the first use; every call leaves the counters at zero, so one
 * workspace (sized for the largest call) serves calls of any shape on one stream. */
ARC_API arc_status_t arc_gemm_workspace_size(int64_t M, const arc_qweight_t* qw, size_t* bytes);
/* Workspace arc_linear needs: 16 KB of the GEMM's tile counters (offset 0), the quantized
 * activation, then the GEMM's fp32 partials.  Zero it once before the first use (e.g. cudaMemsetAsync after allocating it);
 * every call leaves it ready for the next one, so one workspace can serve every layer. */
ARC_API arc_status_t arc_linear_workspace_size(int64_t M, const arc_qweight_t* qw, size_t* bytes);

/* ---------------------------------------------------------------- calibration (offline) */
/* chan_max[j] = max(chan_max[j], max_r |x[r, j]|) over the `rows` bf16 rows of x
 * (row stride ldx elements).  chan_max is a device float[K] the caller
 * initialises (zeros) and may accumulate over several batches (exact). */
ARC_API arc_status_t arc_calib_absmax(const void* x, int64_t rows, int64_t K, int64_t ldx, float* chan_max,
                              void* stream);
/* As arc_calib_absmax for x_dtype ARC_BF16 or ARC_FP16 rows (other types: ARC_ERR_SHAPE). */
ARC_API arc_status_t arc_calib_absmax_ex(const void* x, arc_dtype_t x_dtype, int64_t rows, int64_t K, int64_t ldx,
                                         float* chan_max, void* stream);
/* Host, synchronous.  perm_host = channels sorted by chan_max descending, ties to
 * the lower index (reading Q9); M = max chan_max; tau = 2^-3 M;
 * S_raw = #{j : chan_max[j] > tau} (strict, Q8); S = min(K, 16*ceil(S_raw/16))
 * (Q10) unless s_override >= 0 (must be a multiple of 16 <= K); gs = 2688/M as
 * one fp32 division (1 if M == 0): the static activation tensor scale (Q3, Q4).
 * ARC_ERR_NONFINITE if chan_max has a NaN/Inf or negative entry. */
ARC_API arc_status_t arc_select_outliers(const float* chan_max_host, int64_t K, int32_t s_override,
                                         int32_t* perm_host, int32_t* S, int32_t* S_raw, float* M, float* tau,
                                         float* gs);
/* Host, synchronous, deterministic (independent of the number of host threads it
 * uses: each group of 32 blocks is searched with its own seed).  perm_out assigns every 16-channel block the
 * same SET of channels as perm_host (so the outlier set, every block maximum and
 * scale, the codes as a multiset and the GEMM result are unchanged; reading Q22:
 * the channel order inside a block is free) and orders the channels inside each
 * block so that the quantization kernel's shared-memory gathers (32 consecutive
 * blocks per warp, one channel per lane per step) hit distinct banks as far as
 * possible.  Use perm_out for BOTH arc_quantize_weight and the activation
 * profile.  K must be a multiple of 16; perm_host must be a permutation. */
ARC_API arc_status_t arc_gather_order(const int32_t* perm_host, int64_t K, int32_t* perm_out_host);
/* As arc_gather_order for staged rows of elem_bytes per channel: 2 = bf16 rows (the default), 4 =
 * (gate, up) bf16 pairs (ARC_GU_PAIRS rows of arc_silu_mul_quantize_activation). */
ARC_API arc_status_t arc_gather_order_ex(const int32_t* perm_host, int64_t K, int elem_bytes, int32_t* perm_out_host);
/* gs_out[0] = 2688 / max|x| over a rows x K bf16 matrix (1.0 if the max is 0):
 * the NVFP4 encode tensor scale (reading Q3).  gs_out is a device float. */
ARC_API arc_status_t arc_tensor_scale(const void* x, int64_t rows, int64_t K, int64_t ldx, float* gs_out,
                              void* stream);
/* As arc_tensor_scale for x_dtype ARC_BF16 or ARC_FP16. */
ARC_API arc_status_t arc_tensor_scale_ex(const void* x, arc_dtype_t x_dtype, int64_t rows, int64_t K, int64_t ldx,
                                         float* gs_out, void* stream);

/* ---------------------------------------------------------------- quantization */
/* Offline weight preparation: reorder the N x K bf16 weight by perm,
 * quantize every 16-block to NVFP4 against gs_w (block scale = smallest E4M3 >=
 * amax*gs_w/6, reading Q2), and duplicate the quantized outlier blocks
 * (codes and scale byte, bitwise) into the augmented blocks. */
ARC_API arc_status_t arc_quantize_weight(const void* w, int64_t N, int64_t K, int64_t ldw, const int32_t* perm,
                                 int32_t S, const float* gs_w, arc_layout_t layout, uint8_t* codes,
                                 uint8_t* sf, void* stream);
/* As arc_quantize_weight for w_dtype ARC_BF16 or ARC_FP16 (fp16 decoded exactly to fp32). */
ARC_API arc_status_t arc_quantize_weight_ex(const void* w, arc_dtype_t w_dtype, int64_t N, int64_t K, int64_t ldw,
                                            const int32_t* perm, int32_t S, const float* gs_w, arc_layout_t layout,
                                            uint8_t* codes, uint8_t* sf, void* stream);
/* Online activation quantization: reorder, primary NVFP4 quantization of
 * all K channels, residual of the S outlier channels (against the encoded
 * primary, reading Q6) quantized again with fresh E4M3 block scales and the same
 * tensor scale (Q5), written as augmented blocks in the profile's layout.
 * x: bf16 [M][ldx]; codes [M][Kp/2]; sf roundup(M,128)*Kp/16 bytes. */
ARC_API arc_status_t arc_quantize_activation(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                     uint8_t* codes, uint8_t* sf, void* stream);
/* As arc_quantize_activation for x_dtype ARC_BF16 or ARC_FP16 (fp16 decoded exactly to fp32, then the same
 * STAGE arithmetic; the fused RMSNorm / SiLU producers and the MX variants take bf16 only). */
ARC_API arc_status_t arc_quantize_activation_ex(const void* x, arc_dtype_t x_dtype, int64_t M, int64_t ldx,
                                                const arc_profile_t* prof, uint8_t* codes, uint8_t* sf, void* stream);

/* ---------------------------------------------------------------- RMSNorm (fused producer) */
/* The RMSNorm stage of the paper's "Fused Quantization Kernel that integrates Channel
 * Reordering, RMSNorm, Primary Quantization, and Residual Quantization into a single
 * operation" (Fig.8b), in the LLaMA form with the roundings of a bf16 model
 * and a pinned reduction order (reading Q23):
 *   r   = 1 / sqrt(ss / K + eps), ss = pairwise tree over the K/16 sums of 16 consecutive
 *         squares (each a sequential fp32 fma), zero-padded to a power of two;
 *   y_j = bf16(gamma_j * bf16(x_j * r)).
 * x: bf16 [M][ldx]; gamma: bf16 [K]; eps >= 0 (fp32); y: bf16 [M][ldy].  All-zero rows with
 * eps = 0 and non-finite inputs give unspecified output. */
ARC_API arc_status_t arc_rmsnorm(const void* x, int64_t M, int64_t K, int64_t ldx, const void* gamma, float eps,
                                 void* y, int64_t ldy, void* stream);
/* arc_quantize_activation of arc_rmsnorm(x) in ONE pass over x: each staged row is normalized
 * in shared memory, then reordered and quantized (primary + residual).  Bit-identical to
 * arc_rmsnorm followed by arc_quantize_activation; the normalized row never reaches HBM. */
ARC_API arc_status_t arc_rmsnorm_quantize_activation(const void* x, int64_t M, int64_t ldx, const void* gamma,
                                                     float eps, const arc_profile_t* prof, uint8_t* codes,
                                                     uint8_t* sf, void* stream);
/* arc_linear with the RMSNorm folded into its quantize pass (the attention / MLP input sites
 * of a decoder layer, Fig.5): y = arc_gemm(arc_rmsnorm_quantize_activation(x)).
 * Workspace: arc_linear_workspace_size(M, qw). */
ARC_API arc_status_t arc_linear_rmsnorm(const void* x, int64_t M, int64_t ldx, const void* gamma, float eps,
                                        const arc_profile_t* prof, const arc_qweight_t* qw, void* y,
                                        arc_dtype_t y_dtype, int64_t ldy, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- MXFP4-ARC */
/* The paper's MXFP4 generalisation (Table 6; SPEC: MXFP4 = 32-element blocks,
 * E8M0 scales, no tensor scale), reading Q25: per 32-channel block of the reordered row,
 * 2^e = E8M0_up(amax/6) (amax/6 one fp32 RN division), codes rne_e2m1_sat(x * 2^-e); for the S
 * outlier channels the exact residual x/2^e - v(q) is quantized again the same way (absolute
 * scale 2^(e+e2)); weights duplicate their outlier blocks.  Output in the NVFP4 physical
 * format of arc_quantize_activation -- both 16-halves of a 32-block carry the E4M3 code of
 * 2^(e - c) where gs = 2^-c is the tensor offset -- so arc_gemm multiplies MXFP4-ARC operands
 * exactly (alpha = 1/(gs_x gs_w) = 2^(c_x + c_w)).  K and S must be multiples of 32.  A block
 * exponent e outside [c - 9, c + 8] (E4M3's powers of two for this offset) is clamped into it
 * (reading Q25b): such a block flushes toward 0 or saturates at +-6 * 2^(c+8), with a scale byte
 * that matches its codes. */
/* gs = 2^-c with c = ceil(log2(amax/6)) - 8: the largest block scale of a tensor with max |x| =
 * amax maps to 2^8 (host, no device work). */
ARC_API arc_status_t arc_mx_tensor_scale(float amax, float* gs);
/* The same offset computed on the device from max |x| of a rows x K bf16 matrix (the weight's
 * tensor offset, P:140's offline weight preparation): gs_out[0] = 2^-c, a device float (1.0 if the
 * max is 0).  K % 16 == 0, ldx >= K, ldx % 8 == 0, x 16-byte aligned; errors as arc_tensor_scale. */
ARC_API arc_status_t arc_mx_tensor_scale_device(const void* x, int64_t rows, int64_t K, int64_t ldx, float* gs_out,
                                                void* stream);
/* As arc_quantize_activation; prof->gs must be a power of two (arc_mx_tensor_scale). */
ARC_API arc_status_t arc_quantize_activation_mx(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                                uint8_t* codes, uint8_t* sf, void* stream);
/* As arc_quantize_weight (outlier blocks duplicated); gs_w a device power of two. */
ARC_API arc_status_t arc_quantize_weight_mx(const void* w, int64_t N, int64_t K, int64_t ldw, const int32_t* perm,
                                            int32_t S, const float* gs_w, arc_layout_t layout, uint8_t* codes,
                                            uint8_t* sf, void* stream);

/* ---------------------------------------------------------------- native MXFP4-ARC */
/* MXFP4-ARC (reading Q25: 32-element blocks, 2^e = E8M0_up(RN(amax/6)), codes rne_e2m1_sat(x 2^-e), the
 * outlier blocks' exact residual through the same stage, weights duplicate their outlier blocks) in the
 * native MX physical format of tcgen05 kind::mxf4: one UE8M0 scale byte (e + 127; an all-zero block 0)
 * per 32-element block -- the full E8M0 exponent range, no tensor offset (contrast arc_quantize_*_mx,
 * which stores MX in the NVFP4 format within an offset's 18 binades, reading Q25b).  Block map: App.D
 * at 32-element granularity (interleaved: outlier 32-block j -> physical 2j, its residual 2j+1); K+S is
 * padded to Kpm = roundup(K+S, 128) with zero blocks.  codes: [rows][Kpm/2] (element 2i in the low
 * nibble of byte i); sf: roundup(rows, 128) * Kpm / 32 bytes in the 128x4 tile layout.  K and S must be
 * multiples of 32; perm as arc_quantize_activation. */
ARC_API arc_status_t arc_mx_native_buffer_sizes(int64_t rows, int64_t K, int32_t S, int64_t* Kpm, size_t* code_bytes,
                                                size_t* sf_bytes);
ARC_API arc_status_t arc_quantize_mx_native(const void* x, int64_t rows, int64_t K, int64_t ldx, const int32_t* perm,
                                            int32_t S, int32_t weight, arc_layout_t layout, uint8_t* codes,
                                            uint8_t* sf, void* stream);
/* y[M][N] = A B^T of two native MXFP4 operands with the same K, S and layout (tcgen05 kind::mxf4
 * block_scale scale_vec::2X, UE8M0, FP32 accumulation; no tensor scale).  ws as arc_gemm_mxfp8
 * (arc_gemm_mx_native_workspace_size). */
ARC_API arc_status_t arc_gemm_mx_native_workspace_size(int64_t M, int64_t N, int64_t Kpm, size_t* bytes);
ARC_API arc_status_t arc_gemm_mx_native(const uint8_t* a_codes, const uint8_t* a_sf, int64_t M, const uint8_t* b_codes,
                                        const uint8_t* b_sf, int64_t N, int64_t Kpm, void* y, arc_dtype_t y_dtype,
                                        int64_t ldy, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- Fig.8a comparator: plain MXFP8 */
/* The MXFP8 format the paper compares ARC's kernel against (Eq.3's single stage,
 * P:181-184): per 32-element block of a row, scale 2^e = the smallest power of two >= RN(amax/448)
 * (UE8M0 byte e + 127), codes = E4M3 round-to-nearest-even of x / 2^e; no reordering, no residual.
 * K % 32 == 0; rows are padded to Kp8 = roundup(K, 128) with zero blocks (scale byte 127).
 * codes: [rows][Kp8] bytes; sf: roundup(rows, 128) * Kp8 / 32 bytes in the 128x4 tile layout
 * (one byte per 32-block).  Sizes: */
ARC_API arc_status_t arc_mxfp8_buffer_sizes(int64_t rows, int64_t K, int64_t* Kp8, size_t* code_bytes,
                                            size_t* sf_bytes);
ARC_API arc_status_t arc_quantize_mxfp8(const void* x, int64_t rows, int64_t K, int64_t ldx, uint8_t* codes,
                                        uint8_t* sf, void* stream);
/* y[M][N] = A B^T of two MXFP8 operands (activations a: [M][Kp8], weights b: [N][Kp8], both from
 * arc_quantize_mxfp8 with the same K), FP32 accumulation in TMEM (tcgen05.mma kind::mxf8f6f4.block_scale,
 * K = 32 per MMA, UE8M0 scales), stored as y_dtype (ldy as arc_gemm).  ws: arc_gemm_mxfp8_workspace_size
 * bytes (decode-size M splits K), zero before first use. */
ARC_API arc_status_t arc_gemm_mxfp8_workspace_size(int64_t M, int64_t N, int64_t K, size_t* bytes);
/* The Fig.8a W4A8 comparator (MXFP4 weights, MXFP8 activations): a from arc_quantize_mxfp8
 * ([M][Kp8]), b a plain MXFP4 weight from arc_quantize_mx_native with S = 0 and the identity permutation
 * ([N][Kp8/2] packed E2M1, UE8M0 per 32; Kpm == Kp8); y = A B^T on tcgen05 kind::mxf8f6f4 (E4M3 x E2M1,
 * the weight landing as one byte per element in shared memory).  Workspace as arc_gemm_mxfp8. */
ARC_API arc_status_t arc_gemm_w4a8(const uint8_t* a_codes, const uint8_t* a_sf, int64_t M, const uint8_t* b_codes,
                                   const uint8_t* b_sf, int64_t N, int64_t K, void* y, arc_dtype_t y_dtype, int64_t ldy,
                                   void* ws, size_t ws_bytes, void* stream);
ARC_API arc_status_t arc_gemm_mxfp8(const uint8_t* a_codes, const uint8_t* a_sf, int64_t M, const uint8_t* b_codes,
                                    const uint8_t* b_sf, int64_t N, int64_t K, void* y, arc_dtype_t y_dtype,
                                    int64_t ldy, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- SiLU-mul (fused producer, Fig.5) */
/* The down-projection input of a LLaMA/Qwen decoder layer (Fig.5 P:157 quantizes every linear
 * input): h = SiLU(gate) * up of the bf16 gate/up projections, with the roundings of a bf16
 * model and SiLU evaluated by a pinned fp32 op sequence (reading Q24; correctly rounded to
 * bf16 for every bf16 gate value):
 *   h_j = bf16( bf16(SiLU(g_j)) * u_j ),  g_j = gu[m][j], u_j = gu[m][up_off + j], j < K.
 * gu: bf16 [M][ld] (e.g. the fused gate_up output, up_off = K, ld = 2K); h: bf16 [M][ldh].
 * up_off = ARC_GU_PAIRS instead reads (g_j, u_j) as the adjacent pair gu[m][2j], gu[m][2j+1]
 * (a gate_up weight whose gate and up rows are interleaved offline); ld >= 2K then.
 * Requires K % 16 == 0, K <= 32768, up_off >= K (or ARC_GU_PAIRS), ld >= up_off + K, ld,
 * up_off, ldh multiples of 8 elements, 16-byte aligned buffers.  Non-finite inputs give
 * unspecified output. */
#define ARC_GU_PAIRS (-1)
ARC_API arc_status_t arc_silu_mul(const void* gu, int64_t M, int64_t K, int64_t ld, int64_t up_off, void* h,
                                  int64_t ldh, void* stream);
/* arc_quantize_activation of arc_silu_mul(gu) in ONE pass over gu: each staged gate/up row pair
 * is combined in shared memory and quantized (primary + residual); h never reaches HBM.
 * Bit-identical to arc_silu_mul followed by arc_quantize_activation.  K = prof->K <= 16384. */
ARC_API arc_status_t arc_silu_mul_quantize_activation(const void* gu, int64_t M, int64_t ld, int64_t up_off,
                                                      const arc_profile_t* prof, uint8_t* codes, uint8_t* sf,
                                                      void* stream);
/* arc_linear of arc_silu_mul(gu) (the down_proj site): y = arc_gemm(arc_silu_mul_quantize_activation(gu)).
 * Workspace: arc_linear_workspace_size(M, qw). */
ARC_API arc_status_t arc_linear_silu_mul(const void* gu, int64_t M, int64_t ld, int64_t up_off,
                                         const arc_profile_t* prof, const arc_qweight_t* qw, void* y,
                                         arc_dtype_t y_dtype, int64_t ldy, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- GEMM */
/* y[M][N] (row stride ldy elements) = (1/(gs_x*gs_w)) * sum over the Kp physical
 * elements of A_aug * B_aug^T (Eq.2), FP32 accumulation in tensor
 * memory (tcgen05.mma kind::mxf4nvf4, scale vector 16), stored as y_dtype.
 * a_codes/a_sf: the activation as written by arc_quantize_activation with the
 * same K, S and layout as qw.  ldy * sizeof(y_dtype) must be a multiple of 16.
 * ws: arc_gemm_workspace_size(M, qw) bytes (may be NULL when that is 0), ZERO before its
 * first use (every call leaves it reusable).  At decode-size M (<= 64) one weight-streaming
 * stream-K kernel runs: every SM streams an equal share of the weight units, a tile split
 * over several SMs is summed from fp32 partials in a fixed segment order by the last SM to
 * finish it (deterministic); per-tile arrival counters in ws return to zero.  At other M
 * below one wave of tiles the K range is split and a second kernel sums the partials in a
 * fixed order. */
ARC_API arc_status_t arc_gemm(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                              const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws,
                              size_t ws_bytes, void* stream);
/* Row-parallel tensor parallelism with the all-reduce fused into the GEMM epilogue (SURVEY.md §8(f)
 * f2; BASELINE north_star "row-parallel over the extended K with an all-reduce over NVLink"): every
 * output y_r[m][n] of THIS rank's partial GEMM (the arc_gemm result, fp32) is ADDED into every rank's
 * fp32 output buffer instead of being stored --
 *   ARC_REDUCE_MULTIMEM: one multimem.red.add.f32 per element into red->mc (the NVLS multicast address
 *     of the symmetric [M][ldy] fp32 buffers of all ranks, e.g. torch symmetric memory's multicast_ptr):
 *     the NVSwitch performs the sum, each rank sends its partial once;
 *   ARC_REDUCE_PEERS: one red.add.f32 per element into each of red->peers[0 .. npeers) (every rank's
 *     buffer mapped into this process: NVLink P2P, npeers <= 8).
 * Contract: every rank's buffer is ZERO before any rank's call starts and nobody reads it before every
 * rank's call has finished (e.g. symmetric-memory barriers on both sides); the sum over ranks is then
 * in every rank's buffer.  The fp32 additions of different ranks land in arrival order (the result
 * is within the GEMM tolerance of the exact sum, not bit-reproducible across runs at world > 1).
 * The 16-byte vector reductions need ldy % 4 == 0 and 16-byte aligned buffers.  Workspace as arc_gemm. */
typedef enum { ARC_REDUCE_MULTIMEM = 1, ARC_REDUCE_PEERS = 2 } arc_reduce_mode_t;
typedef struct {
  int32_t mode;        /* arc_reduce_mode_t */
  int32_t npeers;      /* ARC_REDUCE_PEERS: 1..8 */
  float* mc;           /* ARC_REDUCE_MULTIMEM: multicast address of the [M][ldy] fp32 buffers */
  float* peers[8];     /* ARC_REDUCE_PEERS: each rank's [M][ldy] fp32 buffer (device addresses) */
} arc_reduce_t;
ARC_API arc_status_t arc_gemm_reduce(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                                     const arc_qweight_t* qw, const arc_reduce_t* red, int64_t ldy, void* ws,
                                     size_t ws_bytes, void* stream);
/* arc_gemm with the SwiGLU activation in its epilogue (the MLP gate_up site, Fig.5):
 * qw is the fused gate_up weight with its rows interleaved in groups of 16 -- rows 32j..32j+15
 * are gate rows 16j..16j+15 and rows 32j+16..32j+31 the matching up rows (qw->N = 2I, I % 16
 * == 0) -- and instead of the bf16 GEMM output the kernel stores
 *   h[m][i] = bf16( bf16(SiLU(g)) * u ),  g = y[m][32(i/16) + i%16], u = y[m][32(i/16) + 16 + i%16],
 * y the bf16 output arc_gemm would write (reading Q24 for SiLU), into h: bf16 [M][ldh],
 * ldh >= N/2.  Bit-identical to arc_silu_mul applied to the de-interleaved arc_gemm output;
 * the gate/up output never reaches HBM.  Workspace as arc_gemm (split-K at decode sizes). */
ARC_API arc_status_t arc_gemm_swiglu(const uint8_t* a_codes, const uint8_t* a_sf, const float* gs_x, int64_t M,
                                     const arc_qweight_t* qw, void* h, int64_t ldh, void* ws, size_t ws_bytes,
                                     void* stream);
/* The full ARC linear layer Y = X W^T computed as Eq.2: online activation
 * quantization feeding the augmented NVFP4 GEMM (two launches, PDL-chained).  x: bf16 [M][ldx]; y: [M][ldy] of
 * y_dtype.  ws: arc_linear_workspace_size(M, qw) bytes, 256-byte aligned, zero before its
 * first use (see above).  Same as arc_linear_ex(..., ARC_LINEAR_AUTO, ...). */
ARC_API arc_status_t arc_linear(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                        const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws,
                        size_t ws_bytes, void* stream);

/* How arc_linear_ex runs the layer:
 *  ARC_LINEAR_UNFUSED: two kernels chained by programmatic dependent launch -- arc_quantize_activation
 *    into the workspace, then arc_gemm.  At decode-size M (<= 64) the quantize is a direct-gather kernel
 *    and the GEMM a cluster split-K kernel whose K partials are summed in distributed shared memory in a
 *    fixed rank order (no fp32 partials in HBM, no second kernel); both read the calibration constants
 *    (perm) and the prepared weights before griddepcontrol.wait, so these -- like every library-prepared
 *    weight -- must not be written by the kernel that immediately precedes the arc_linear call.
 *  ARC_LINEAR_AUTO: UNFUSED (the faster path on B200 at every M).
 *  ARC_LINEAR_FUSED at M <= 64: ONE kernel (the "optionally fused with the activation quantize as its
 *    producer stage" GEMM of the north star): a persistent weight-streaming stream-K GEMM whose
 *    CTAs first quantize one 256-element K block each (all M rows) into the workspace and publish it
 *    with a per-K-block ready word; each CTA's producer streams its weights from launch and waits only
 *    for the K blocks it needs; split tiles are summed in a fixed segment order by the last CTA to
 *    finish them.  The quantized activation is bit-identical to arc_quantize_activation's.  At M > 64
 *    FUSED runs the two-kernel path. */
enum { ARC_LINEAR_AUTO = 0, ARC_LINEAR_FUSED = 1, ARC_LINEAR_UNFUSED = 2 };
/* Or-ed into arc_linear_ex's flags: x holds IEEE fp16 rows (ARC_FP16); the layer then runs UNFUSED. */
enum { ARC_LINEAR_X_FP16 = 16 };
ARC_API arc_status_t arc_linear_ex_workspace_size(int64_t M, const arc_qweight_t* qw, int flags, size_t* bytes);
ARC_API arc_status_t arc_linear_ex(const void* x, int64_t M, int64_t ldx, const arc_profile_t* prof,
                                   const arc_qweight_t* qw, void* y, arc_dtype_t y_dtype, int64_t ldy, void* ws,
                                   size_t ws_bytes, int flags, void* stream);
/* arc_linear on HOST buffers: copies x_host (bf16 [M][K], pinned or pageable) to
 * the device, runs arc_linear, copies y back to y_host ([M][N] of y_dtype) and
 * waits for all of it (arc_linear_hostio_wait).  ws must hold arc_linear_hostio_workspace_size bytes.
 * The rows are pipelined in chunks of 128-multiples (~8 per call): chunk i's host->device copy runs on a
 * library-owned copy-in stream, its arc_linear on `stream`, its device->host copy on a library-owned
 * copy-out stream (two non-blocking streams and an event ring per device, created on first use), so the
 * copies overlap the compute and each other.  Y equals arc_linear applied to each chunk of rows (quantization is
 * per row; a chunk's GEMM may choose a different K split than the whole batch's: same tolerance). */
ARC_API arc_status_t arc_linear_hostio_workspace_size(int64_t M, const arc_qweight_t* qw, arc_dtype_t y_dtype,
                                                      size_t* bytes);
ARC_API arc_status_t arc_linear_hostio(const void* x_host, int64_t M, const arc_profile_t* prof,
                               const arc_qweight_t* qw, void* y_host, arc_dtype_t y_dtype, void* ws,
                               size_t ws_bytes, void* stream);
/* The same pipeline without the final wait: returns once everything is enqueued, so the copies of
 * consecutive calls overlap (device->host of one layer with host->device of the next).  The host buffers
 * and ws must stay untouched until arc_linear_hostio_wait(stream) returns; concurrent calls need distinct
 * workspaces. */
ARC_API arc_status_t arc_linear_hostio_async(const void* x_host, int64_t M, const arc_profile_t* prof,
                                             const arc_qweight_t* qw, void* y_host, arc_dtype_t y_dtype, void* ws,
                                             size_t ws_bytes, void* stream);
/* Blocks until every arc_linear_hostio_async call on this device (and `stream`) has completed. */
ARC_API arc_status_t arc_linear_hostio_wait(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ARC_H_ */
