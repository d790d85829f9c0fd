/*
 * arc_oracle.c -- plain, slow, obviously-correct CPU oracle for the ARCQuant
 * (arxiv 2601.07475) online hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (libarc.so, paper_2601_07475_b200/) never links, imports or calls
 * it, and shares no code, header, table or constant generator with it.
 *
 * Citations "P:<line>" are /root/reference/PAPER.md line numbers (section,
 * equation or table named beside them); "Q<n>" are the readings of the paper
 * listed in DESIGN.md ("Readings") where the paper is silent or ambiguous.
 *
 * Floating point: every float operation below is one IEEE binary32 operation
 * with round-to-nearest-even (compiled with -O2 -ffp-contract=off, SSE, no
 * fast-math), in exactly the order written.  That order is the pinned op order
 * of reading Q7; the CUDA path reproduces it with __fmul_rn/__fdiv_rn.
 *
 * What pins each function (tests/test_oracle_*.py):
 *   e2m1_*        Table 7 values; brute-force argmin over the 16 codes;
 *                 SPEC example 5.0 -> 4.0; worst error 1.0 on [-6, 6].
 *   e4m3_*        Table 7 bias 7 / max 448; torch.float8_e4m3fn decode of
 *                 all codes; brute-force scan for ceil; alpha in [1, 1.125).
 *   stage         brute force over every block of small tensors; the worked
 *                 example in DESIGN.md; 16 x 6.0 -> SF 0x38.
 *   arc_*         S = 0 reduces to plain NVFP4; representable input -> zero
 *                 residual; Eq.4 bound and alpha1*alpha2 <= 1.125^2;
 *                 duplicate blocks bitwise equal.
 *   pack/layout   the layout map is a bijection; GEMM identical across layouts.
 *   calibration   S:188 example; perm prefix = {j : max_j > tau}.
 *   gemm_exact    Eq.2 identity as an integer equality; brute
 *                 float64 dequantized product on small shapes.
 *   rmsnorm       float64 formula within two bf16 roundings; exact invariance
 *                 under power-of-two scaling of a row (eps = 0); constant rows
 *                 -> +-1 exactly; torch's fp32 RMSNorm within one bf16 ulp.
 *   mx (f3)       SPEC example 7s -> scale 2; every block = smallest power of
 *                 two >= amax/6 with brute-force nearest codes; residual stage
 *                 exact; physical bytes decode to the MX values (GEMM identity).
 *   silu          all 2^16 bf16 gate values: fp32 SiLU within 4 ulp of long
 *                 double, its bf16 rounding correctly rounded everywhere, torch's
 *                 bf16 SiLU bit-identical wherever its exp does not overflow.
 * Parity unpinned (decisions, not values the paper prints): Q2 ceil-rounded
 * E4M3 block scales, Q4 static activation tensor scale, Q6/Q7 residual domain
 * and op order, Q12 default layout, Q23 RMSNorm reduction order and roundings.
 * See DESIGN.md.
 */
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_SHAPE 2
#define OR_ERR_NONFINITE 7

/* ------------------------------------------------------------------------- */
/* C1: E2M1 (Table 7: FP4 E2M1, bias 1, max +-6).                      */
/* The 8 magnitudes follow from 1 sign, 2 exponent (bias 1), 1 mantissa bit:  */
/* subnormal 0, 0.5; normal 1, 1.5, 2, 3, 4, 6.                               */
/* ------------------------------------------------------------------------- */
static const float E2M1_MAG[8] = {0.0f, 0.5f, 1.0f, 1.5f, 2.0f, 3.0f, 4.0f, 6.0f};

float or_e2m1_value(uint8_t q) {
    float m = E2M1_MAG[q & 7];
    return (q & 8) ? -m : m;
}

/* Eq.1 round() read as round-to-nearest, ties to the even code,
 * saturating at +-6, sign kept (reading Q1).  The thresholds are the midpoints
 * of adjacent magnitudes; '>' vs '>=' encodes the tie going to the even code:
 * 0.25->0, 0.75->1.0, 1.25->1.0, 1.75->2, 2.5->2, 3.5->4, 5->4. */
uint8_t or_e2m1_encode(float t) {
    float a = fabsf(t);
    uint8_t mag = (uint8_t)((a > 0.25f) + (a >= 0.75f) + (a > 1.25f) + (a >= 1.75f) +
                            (a > 2.5f) + (a >= 3.5f) + (a > 5.0f));
    return (uint8_t)(mag | (signbit(t) ? 8 : 0));
}

/* ------------------------------------------------------------------------- */
/* C2: E4M3 (Table 7: bias 7, max +-448; OCP E4M3FN, 0x7F = NaN).      */
/* ------------------------------------------------------------------------- */
float or_e4m3_value(uint8_t c) {
    int e = (c >> 3) & 15, m = c & 7;
    float v;
    if (e == 0) v = ldexpf((float)m, -9);                  /* subnormal: m * 2^-9 */
    else        v = ldexpf(1.0f + (float)m / 8.0f, e - 7);
    return (c & 0x80) ? -v : v;
}

/* Block-scale encoder, reading Q2: smallest non-negative E4M3 code whose value
 * is >= v (alpha = s/M >= 1; "2^-3 step size"), saturating at
 * 448 (0x7E).  Plain linear scan of the 127 finite codes. */
uint8_t or_e4m3_ceil(float v) {
    if (!(v > 0.0f)) return 0;
    for (int c = 0; c <= 0x7E; ++c)
        if (or_e4m3_value((uint8_t)c) >= v) return (uint8_t)c;
    return 0x7E;
}

/* Round-to-nearest-even E4M3 with saturation: used only by the MXFP8
 * comparator of Eq.3.  Linear scan; ties -> even code. */
uint8_t or_e4m3_rn(float x) {
    float a = fabsf(x);
    int best = 0;
    double bd = 1e300;
    for (int c = 0; c <= 0x7E; ++c) {
        double d = fabs((double)or_e4m3_value((uint8_t)c) - (double)a);
        if (d < bd || (d == bd && (c & 1) == 0)) { bd = d; best = c; }
    }
    return (uint8_t)(best | (signbit(x) ? 0x80 : 0));
}

/* E8M0 round-up (MX scale, "shared exponent"): smallest power of two >= v. */
float or_e8m0_up(float v) {
    int e;
    float f = frexpf(v, &e);               /* v = f * 2^e, f in [0.5, 1) */
    if (f == 0.5f) return ldexpf(1.0f, e - 1);
    return ldexpf(1.0f, e);
}

/* ------------------------------------------------------------------------- */
/* C4: STAGE -- one NVFP4 block quantization, Eq.1 with the two-  */
/* level NVFP4 scaling of P:118 / P:453: value = v(q) * d / gs.               */
/* base = gs for the primary stage; base = d1 for the residual stage (Q6).    */
/* ------------------------------------------------------------------------- */
void or_stage(const float z[16], float base, uint8_t* sf, float* d_out, float t[16], uint8_t q[16]) {
    float a = 0.0f;
    for (int i = 0; i < 16; ++i) {                /* a = max |z|  (exact) */
        float m = fabsf(z[i]);
        if (m > a) a = m;
    }
    float c6 = base / 6.0f;                        /* q_max = 6 (Table 7) */
    uint8_t s = or_e4m3_ceil(a * c6);             /* s_X = max|X| / q_max, rounded up */
    float d = or_e4m3_value(s);
    float k = (d == 0.0f) ? 0.0f : base / d;
    for (int i = 0; i < 16; ++i) {
        t[i] = z[i] * k;                           /* X / s_X in E2M1 units */
        q[i] = or_e2m1_encode(t[i]);               /* Q_X = round(X / s_X) */
    }
    *sf = s;
    *d_out = d;
}

/* bf16 -> fp32 widening is exact: the bf16 bits are the top 16 fp32 bits. */
static float bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* IEEE binary16 -> fp32 (exact): 1 sign, 5 exponent (bias 15), 10 fraction bits; subnormals m * 2^-24. */
float or_f16_to_f32(uint16_t h) {
    const int s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
    float v;
    if (e == 0) v = ldexpf((float)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexpf((float)(m | 1024), e - 25);
    return s ? -v : v;
}

/* Element format of the 16-bit activation / weight rows the quantizers read (SURVEY 8(b) arc_dtype_t):
 * 0 = bf16 (default), 1 = fp16.  Set by the Python wrapper around a call (test infrastructure). */
static int g_in_fp16 = 0;
void or_set_input_fp16(int on) { g_in_fp16 = on ? 1 : 0; }
static float in16_to_f32(uint16_t h) { return g_in_fp16 ? or_f16_to_f32(h) : bf16_to_f32(h); }

/* ------------------------------------------------------------------------- */
/* C5: ARC activation row, logical (unpacked) order -- P:138 §3.2 "Online     */
/* Activation Quantization": (1) reorder + primary quantization of all K      */
/* channels, (2) residual R_o = X_o - s*Q_Xo of the first S reordered         */
/* (outlier) channels, quantized again, (3) concatenation along K.            */
/* Output: codes[K+S] (one 4-bit code per byte), sf[(K+S)/16].                */
/* Logical block b < K/16 = primary block b; logical block K/16+j = residual  */
/* of primary block j (j < S/16).                                             */
/* ------------------------------------------------------------------------- */
int or_arc_row_logical(const uint16_t* x_row, const int32_t* perm, int K, int S, float gs,
                       uint8_t* codes, uint8_t* sf) {
    if (K <= 0 || K % 16 || S < 0 || S % 16 || S > K) return OR_ERR_SHAPE;
    int nb = K / 16;
    for (int b = 0; b < nb; ++b) {
        float z[16], t[16], e[16], t2[16], d1, d2;
        uint8_t q1[16], q2[16], s1, s2;
        for (int i = 0; i < 16; ++i) {
            z[i] = in16_to_f32(x_row[perm[16 * b + i]]);       /* (1) reorder */
            if (!isfinite(z[i])) return OR_ERR_NONFINITE;
        }
        or_stage(z, gs, &s1, &d1, t, q1);                      /* (1) primary */
        memcpy(codes + 16 * b, q1, 16);
        sf[b] = s1;
        if (b < S / 16) {                                      /* (2) outlier block */
            for (int i = 0; i < 16; ++i)
                e[i] = t[i] - or_e2m1_value(q1[i]);             /* residual, units d1/gs */
            or_stage(e, d1, &s2, &d2, t2, q2);                 /* fresh block scale, same gs */
            memcpy(codes + K + 16 * b, q2, 16);                /* (3) appended along K */
            sf[nb + b] = s2;
        }
    }
    return OR_OK;
}

/* C6: weight row, logical order -- P:140 "Offline Weight Quantization":
 * reorder, quantize, then duplicate the *quantized* outlier blocks (codes and
 * block scale bitwise, reading Q13) instead of computing residuals. */
int or_weight_row_logical(const uint16_t* w_row, const int32_t* perm, int K, int S, float gs,
                          uint8_t* codes, uint8_t* sf) {
    if (K <= 0 || K % 16 || S < 0 || S % 16 || S > K) return OR_ERR_SHAPE;
    int nb = K / 16;
    for (int b = 0; b < nb; ++b) {
        float z[16], t[16], d;
        uint8_t q[16], s;
        for (int i = 0; i < 16; ++i) {
            z[i] = in16_to_f32(w_row[perm[16 * b + i]]);
            if (!isfinite(z[i])) return OR_ERR_NONFINITE;
        }
        or_stage(z, gs, &s, &d, t, q);
        memcpy(codes + 16 * b, q, 16);
        sf[b] = s;
    }
    for (int j = 0; j < S / 16; ++j) {                          /* Q_Waug = [Q_W | Q_Wo] */
        memcpy(codes + K + 16 * j, codes + 16 * j, 16);
        sf[nb + j] = sf[j];
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* C8: block map.  P:591-597 App.D "Interleaved Channel Layout": each 16-     */
/* channel primary outlier block is immediately followed by its residual      */
/* block.  layout 0 = INTERLEAVED, 1 = CONTIGUOUS (the logical concat). */
/* ------------------------------------------------------------------------- */
int or_physical_block(int l, int K, int S, int layout) {
    int nb = K / 16, ns = S / 16;
    if (layout == 1) return l;
    if (l < ns) return 2 * l;                  /* primary outlier block j -> 2j   */
    if (l < nb) return l + ns;                 /* remaining primary blocks        */
    return 2 * (l - nb) + 1;                   /* residual block j -> 2j+1        */
}

/* Kp: K+S padded to the 64-element MMA K step (reading Q14). */
int64_t or_kp(int K, int S) { return ((int64_t)(K + S) + 63) / 64 * 64; }

/* C9: the 128x4 scale-factor tile layout (reading Q15): byte offset of the
 * scale for row m, physical scale column c, in a buffer of Kp/16 columns. */
int64_t or_sf_offset(int64_t m, int64_t c, int64_t Kp) {
    return ((m >> 7) * (Kp / 64) + (c >> 2)) * 512 + (m & 31) * 16 + ((m >> 5) & 3) * 4 + (c & 3);
}

/* Pack one logical row: codes (one per byte, logical order) -> nibble-packed
 * physical row (element 2j in the low nibble of byte j) plus SF bytes into
 * the swizzled buffer.  Padding blocks Ka..Kp hold code 0 and SF 0x00. */
void or_pack_row(const uint8_t* lcodes, const uint8_t* lsf, int K, int S, int layout, int64_t m,
                 uint8_t* codes_row, uint8_t* sf_buf) {
    int64_t Kp = or_kp(K, S);
    int nlog = (K + S) / 16;
    uint8_t* phys = (uint8_t*)calloc((size_t)Kp, 1);
    uint8_t* psf = (uint8_t*)calloc((size_t)(Kp / 16), 1);
    for (int l = 0; l < nlog; ++l) {
        int p = or_physical_block(l, K, S, layout);
        memcpy(phys + 16 * p, lcodes + 16 * l, 16);
        psf[p] = lsf[l];
    }
    for (int64_t j = 0; j < Kp / 2; ++j)
        codes_row[j] = (uint8_t)((phys[2 * j] & 15) | ((phys[2 * j + 1] & 15) << 4));
    for (int64_t c = 0; c < Kp / 16; ++c) sf_buf[or_sf_offset(m, c, Kp)] = psf[c];
    free(phys);
    free(psf);
}

/* Whole-tensor ARC activation quantization (C5 + C8 + C9) on host buffers.
 * x: bf16 bits [M][ldx]; codes: [M][Kp/2]; sf: roundup(M,128)*Kp/16 bytes. */
int or_quantize_activation(const uint16_t* x, int64_t M, int K, int64_t ldx, const int32_t* perm,
                           int S, float gs, int layout, uint8_t* codes, uint8_t* sf) {
    int64_t Kp = or_kp(K, S);
    int rc = OR_OK;
    /* rows are independent (each writes only its own codes / scale bytes); the OpenMP build
     * (liboracle_omp.so, the bench's multi-core CPU baseline) splits them over threads */
    #pragma omp parallel
    {
        uint8_t* lc = (uint8_t*)malloc((size_t)(K + S));
        uint8_t* ls = (uint8_t*)malloc((size_t)((K + S) / 16 + 1));
        #pragma omp for schedule(static)
        for (int64_t m = 0; m < M; ++m) {
            int r = or_arc_row_logical(x + m * ldx, perm, K, S, gs, lc, ls);
            if (r == OR_OK) or_pack_row(lc, ls, K, S, layout, m, codes + m * (Kp / 2), sf);
            else {
                #pragma omp critical
                rc = r;
            }
        }
        free(lc);
        free(ls);
    }
    return rc;
}

/* Whole-tensor weight preparation (C6 + C8 + C9). */
int or_quantize_weight(const uint16_t* w, int64_t N, int K, int64_t ldw, const int32_t* perm, int S,
                       float gs, int layout, uint8_t* codes, uint8_t* sf) {
    int64_t Kp = or_kp(K, S);
    int rc = OR_OK;
    #pragma omp parallel
    {
        uint8_t* lc = (uint8_t*)malloc((size_t)(K + S));
        uint8_t* ls = (uint8_t*)malloc((size_t)((K + S) / 16 + 1));
        #pragma omp for schedule(static)
        for (int64_t n = 0; n < N; ++n) {
            int r = or_weight_row_logical(w + n * ldw, perm, K, S, gs, lc, ls);
            if (r == OR_OK) or_pack_row(lc, ls, K, S, layout, n, codes + n * (Kp / 2), sf);
            else {
                #pragma omp critical
                rc = r;
            }
        }
        free(lc);
        free(ls);
    }
    return rc;
}

/* ------------------------------------------------------------------------- */
/* C7: calibration -- P:136 "Adaptive Outlier Identification".         */
/* ------------------------------------------------------------------------- */
/* Per-channel abs-max over all calibration rows (exact), max-aggregated into
 * chan_max (caller initialises it, e.g. to zeros). */
int or_calib_absmax(const uint16_t* x, int64_t rows, int K, int64_t ldx, float* chan_max) {
    for (int64_t r = 0; r < rows; ++r)
        for (int j = 0; j < K; ++j) {
            float v = in16_to_f32(x[r * ldx + j]);
            if (!isfinite(v)) return OR_ERR_NONFINITE;
            if (fabsf(v) > chan_max[j]) chan_max[j] = fabsf(v);
        }
    return OR_OK;
}

/* perm = channels sorted by abs-max descending, ties to the lower index (Q9);
 * M = layer-wise max; tau = 2^-3 M; S_raw = #{chan_max > tau} (strict, Q8);
 * S = min(K, 16*ceil(S_raw/16)) (Q10) unless s_override >= 0.
 * Plain insertion sort: obviously stable. */
int or_select_outliers(const float* chan_max, int K, int s_override, int32_t* perm, int* S,
                       int* S_raw, float* M, float* tau) {
    if (K <= 0 || K % 16) return OR_ERR_SHAPE;
    if (s_override > K || (s_override >= 0 && s_override % 16)) return OR_ERR_SHAPE;
    float mx = 0.0f;
    for (int j = 0; j < K; ++j) {
        if (!isfinite(chan_max[j]) || chan_max[j] < 0.0f) return OR_ERR_NONFINITE;
        if (chan_max[j] > mx) mx = chan_max[j];
    }
    for (int j = 0; j < K; ++j) perm[j] = j;
    for (int i = 1; i < K; ++i) {
        int32_t v = perm[i];
        int p = i - 1;
        while (p >= 0 && chan_max[perm[p]] < chan_max[v]) { perm[p + 1] = perm[p]; --p; }
        perm[p + 1] = v;
    }
    float t = mx * 0.125f;                        /* tau = 2^-3 M, exact */
    int sr = 0;
    for (int j = 0; j < K; ++j) sr += chan_max[j] > t;
    int s = (sr + 15) / 16 * 16;
    if (s > K) s = K;
    *S_raw = sr;
    *S = (s_override >= 0) ? s_override : s;
    *M = mx;
    *tau = t;
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* C10: the augmented GEMM, exact -- Eq.2: Y = s_Xaug Q_Xaug       */
/* (s_Waug Q_Waug)^T over the extended reduction dimension K+S. */
/* Work in integer units: V(q) = 2 v(q) in [-12, 12], D(sf) = 512 E4M3(sf);    */
/* one term = V_a D_a V_b D_b = 2^20 * (product of the four real factors).     */
/* The int64 sum is exact and order-independent (|sum| < 2.5e17 < 2^63).      */
/* rows: list of A row indices to compute (nrows of them); T, Tabs: [nrows][N]. */
/* ------------------------------------------------------------------------- */
/* Integer value V(q)*D(sf) of physical element p of row r of a packed operand. */
static int64_t elem_units(const uint8_t* codes, const uint8_t* sf, int64_t r, int64_t p, int64_t Kp) {
    uint8_t byte = codes[r * (Kp / 2) + p / 2];
    uint8_t q = (p & 1) ? (byte >> 4) : (byte & 15);
    int64_t V = (int64_t)(2.0f * or_e2m1_value(q));
    int64_t D = (int64_t)(512.0f * or_e4m3_value(sf[or_sf_offset(r, p / 16, Kp)]));
    return V * D;
}

void or_gemm_exact(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes,
                   const uint8_t* b_sf, int64_t N, int64_t Kp, const int64_t* rows, int64_t nrows,
                   int64_t* T, int64_t* Tabs) {
    int64_t* Va = (int64_t*)malloc(sizeof(int64_t) * (size_t)(Kp * nrows));
    for (int64_t ri = 0; ri < nrows; ++ri)
        for (int64_t p = 0; p < Kp; ++p) Va[ri * Kp + p] = elem_units(a_codes, a_sf, rows[ri], p, Kp);
    /* output columns are independent; the OpenMP build splits them over threads */
    #pragma omp parallel
    {
        int64_t* Vb = (int64_t*)malloc(sizeof(int64_t) * (size_t)Kp);
        #pragma omp for schedule(static)
        for (int64_t n = 0; n < N; ++n) {
            for (int64_t p = 0; p < Kp; ++p) Vb[p] = elem_units(b_codes, b_sf, n, p, Kp);
            for (int64_t ri = 0; ri < nrows; ++ri) {
                int64_t acc = 0, aabs = 0;
                for (int64_t p = 0; p < Kp; ++p) {
                    int64_t term = Va[ri * Kp + p] * Vb[p];
                    acc += term;
                    aabs += term < 0 ? -term : term;
                }
                T[ri * N + n] = acc;
                Tabs[ri * N + n] = aabs;
            }
        }
        free(Vb);
    }
    free(Va);
}

/* ------------------------------------------------------------------------- */
/* Fig.8a comparator: plain MXFP8 -- Eq.3's single stage per   */
/* 32-block (E8M0 scale = smallest power of two >= amax/448, E4M3  */
/* elements round-to-nearest-even), no reordering, no residual, K padded to a */
/* multiple of 128 with zero blocks (scale 1).  codes: E4M3 bytes [rows][Kp8];*/
/* sf: E8M0 bytes (2^(b-127)) in the 128x4 tile layout with Kp8/32 columns.   */
/* ------------------------------------------------------------------------- */
int64_t or_kp8(int K) { return ((int64_t)K + 127) / 128 * 128; }
void or_mxfp8_block(const float x[32], float* scale, float xhat[32]);  /* Eq.3, below */

int or_quantize_mxfp8(const uint16_t* x, int64_t rows, int K, int64_t ldx, uint8_t* codes, uint8_t* sf) {
    if (K <= 0 || K % 32 || rows < 0 || ldx < K) return OR_ERR_SHAPE;
    const int64_t Kp8 = or_kp8(K);
    for (int64_t m = 0; m < rows; ++m)
        for (int j = 0; j < K; ++j)
            if (!isfinite(bf16_to_f32(x[m * ldx + j]))) return OR_ERR_NONFINITE;
    #pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < rows; ++m) {
        for (int64_t b = 0; b < Kp8 / 32; ++b) {
            float z[32], xh[32], s = 1.0f;
            uint8_t* c = codes + m * Kp8 + b * 32;
            if (b * 32 < K) {
                for (int i = 0; i < 32; ++i) z[i] = bf16_to_f32(x[m * ldx + b * 32 + i]);
                or_mxfp8_block(z, &s, xh);                      /* Eq.3: the scale */
                for (int i = 0; i < 32; ++i) c[i] = or_e4m3_rn(z[i] / s);
            } else {
                memset(c, 0, 32);
            }
            int e;
            frexpf(s, &e);                                      /* s = 2^(e-1) */
            sf[or_sf_offset(m, b, Kp8 / 2)] = (uint8_t)(e - 1 + 127);
        }
    }
    return OR_OK;
}

/* Exact MXFP8 GEMM: per 32-block the int64 sum of V_a V_b with V = 512 e4m3 (an integer), scaled by
 * 2^(ea + eb - 18) in double; |.| sums likewise for the bound.  Y, Yabs: [nrows][N]. */
void or_gemm_mxfp8_exact(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes, const uint8_t* b_sf,
                         int64_t N, int64_t Kp8, const int64_t* rows, int64_t nrows, double* Y, double* Yabs) {
    #pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t ri = 0; ri < nrows; ++ri) {
            const int64_t r = rows[ri];
            double acc = 0.0, aabs = 0.0;
            for (int64_t b = 0; b < Kp8 / 32; ++b) {
                int64_t s = 0, sa = 0;
                for (int i = 0; i < 32; ++i) {
                    const int64_t va = (int64_t)(512.0f * or_e4m3_value(a_codes[r * Kp8 + b * 32 + i]));
                    const int64_t vb = (int64_t)(512.0f * or_e4m3_value(b_codes[n * Kp8 + b * 32 + i]));
                    s += va * vb;
                    sa += va * vb < 0 ? -va * vb : va * vb;
                }
                const int e = (int)a_sf[or_sf_offset(r, b, Kp8 / 2)] + (int)b_sf[or_sf_offset(n, b, Kp8 / 2)] - 254 - 18;
                acc += ldexp((double)s, e);
                aabs += ldexp((double)sa, e);
            }
            Y[ri * N + n] = acc;
            Yabs[ri * N + n] = aabs;
        }
    }
}

/* Fig.8a W4A8 comparator (MXFP4 weights, MXFP8 activations): exact GEMM of an MXFP8 A
 * (or_quantize_mxfp8: E4M3 bytes [M][Kp8]) and a plain MXFP4 B (or_quantize_mx_native with S = 0 and
 * the identity permutation: packed E2M1 [N][Kp8/2]); both UE8M0 scale layouts have Kp8/32 columns.
 * Per 32-block: int64 sum of (512 e4m3)(2 e2m1) scaled by 2^(ea + eb - 254 - 10). */
void or_gemm_w4a8_exact(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes, const uint8_t* b_sf,
                        int64_t N, int64_t Kp8, const int64_t* rows, int64_t nrows, double* Y, double* Yabs) {
    #pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t ri = 0; ri < nrows; ++ri) {
            const int64_t r = rows[ri];
            double acc = 0.0, aabs = 0.0;
            for (int64_t b = 0; b < Kp8 / 32; ++b) {
                int64_t s = 0, sa = 0;
                for (int i = 0; i < 32; ++i) {
                    const int64_t p = b * 32 + i;
                    const int64_t va = (int64_t)(512.0f * or_e4m3_value(a_codes[r * Kp8 + p]));
                    const uint8_t bb = b_codes[n * (Kp8 / 2) + p / 2];
                    const int64_t vb = (int64_t)(2.0f * or_e2m1_value((p & 1) ? (bb >> 4) : (bb & 15)));
                    s += va * vb;
                    sa += va * vb < 0 ? -va * vb : va * vb;
                }
                const int e = (int)a_sf[or_sf_offset(r, b, Kp8 / 2)] + (int)b_sf[or_sf_offset(n, b, Kp8 / 2)] - 254 - 10;
                acc += ldexp((double)s, e);
                aabs += ldexp((double)sa, e);
            }
            Y[ri * N + n] = acc;
            Yabs[ri * N + n] = aabs;
        }
    }
}

/* Threads the OpenMP build uses (1 in the plain build). */
#ifdef _OPENMP
#include <omp.h>
int or_num_threads(void) { return omp_get_max_threads(); }
#else
int or_num_threads(void) { return 1; }
#endif

/* ------------------------------------------------------------------------- */
/* Eq.3 comparator: single-stage MXFP8 -- g = 32, E4M3 elements,  */
/* E8M0 block scale = smallest power of two >= amax/448 (alpha_mx in [1,2)).  */
/* Returns the dequantized block in xhat[32] and the scale.                    */
/* ------------------------------------------------------------------------- */
void or_mxfp8_block(const float x[32], float* scale, float xhat[32]) {
    float a = 0.0f;
    for (int i = 0; i < 32; ++i) if (fabsf(x[i]) > a) a = fabsf(x[i]);
    float s = (a > 0.0f) ? or_e8m0_up(a / 448.0f) : 1.0f;
    for (int i = 0; i < 32; ++i) xhat[i] = or_e4m3_value(or_e4m3_rn(x[i] / s)) * s;
    *scale = s;
}

/* Batch helpers so the Python tests can sweep the codecs without a per-call
 * ctypes round trip.  They only loop over the scalar functions above. */
void or_e2m1_encode_n(const float* t, int64_t n, uint8_t* q) {
    for (int64_t i = 0; i < n; ++i) q[i] = or_e2m1_encode(t[i]);
}
void or_e4m3_ceil_n(const float* v, int64_t n, uint8_t* c) {
    for (int64_t i = 0; i < n; ++i) c[i] = or_e4m3_ceil(v[i]);
}
void or_e4m3_rn_n(const float* v, int64_t n, uint8_t* c) {
    for (int64_t i = 0; i < n; ++i) c[i] = or_e4m3_rn(v[i]);
}

/* ------------------------------------------------------------------------- */
/* RMSNorm -- the "RMSNorm" stage of the paper's Fused Quantization Kernel    */
/* ("integrates Channel Reordering, RMSNorm, Primary Quantization, and        */
/* Residual Quantization into a single operation"; Fig.8b), in   */
/* the LLaMA form y = g * x / sqrt(mean(x^2) + eps), with the roundings of an */
/* unfused bf16 implementation and a pinned reduction order (reading Q23):    */
/*   s_b = x_{16b}^2 + ... + x_{16b+15}^2, sequential fmaf, original channel  */
/*         order (block b = channels 16b..16b+15);                            */
/*   the K/16 block sums, zero-padded to P = a power of two >= max(K/16, 32), */
/*   are dealt round-robin to 32 partials (block b -> partial b mod 32); each */
/*   partial is a pairwise tree over its P/32 blocks in increasing b, and ss  */
/*   is a pairwise tree over the 32 partials (left + right at every level);   */
/*   r   = 1 / sqrt(ss / K + eps)          (IEEE div, sqrt, div);             */
/*   y_j = bf16( g_j * bf16( x_j * r ) )   (RNE; g_j * t is exact in fp32).   */
/* ------------------------------------------------------------------------- */
static uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);   /* finite inputs only (checked by the caller) */
    return (uint16_t)(u >> 16);
}

static float pairwise_tree(float* t, int n) {  /* n a power of two; destroys t */
    for (int w = n; w > 1; w /= 2)
        for (int i = 0; i < w / 2; ++i) t[i] = t[2 * i] + t[2 * i + 1];
    return t[0];
}

float or_rmsnorm_scale(const uint16_t* x, int K, float eps) {
    const int nb = K / 16;
    int P = 32;
    while (P < nb) P *= 2;
    const int per = P / 32;
    float* s = (float*)calloc((size_t)P, sizeof(float));
    float* u = (float*)calloc((size_t)per, sizeof(float));
    float part[32];
    for (int b = 0; b < nb; ++b) {
        float acc = 0.0f;
        for (int i = 0; i < 16; ++i) {
            const float v = bf16_to_f32(x[16 * b + i]);
            acc = fmaf(v, v, acc);
        }
        s[b] = acc;
    }
    for (int t = 0; t < 32; ++t) {
        for (int j = 0; j < per; ++j) u[j] = s[t + 32 * j];
        part[t] = pairwise_tree(u, per);
    }
    const float ss = pairwise_tree(part, 32);
    free(s);
    free(u);
    const float mean = ss / (float)K;
    return 1.0f / sqrtf(mean + eps);
}

int or_rmsnorm(const uint16_t* x, int64_t M, int K, int64_t ldx, const uint16_t* gamma, float eps, uint16_t* y,
               int64_t ldy) {
    if (K <= 0 || K % 16 || M < 0 || ldx < K || ldy < K || !(eps >= 0.0f)) return OR_ERR_SHAPE;
    for (int64_t m = 0; m < M; ++m) {
        const uint16_t* xr = x + m * ldx;
        for (int j = 0; j < K; ++j)
            if (!isfinite(bf16_to_f32(xr[j]))) return OR_ERR_NONFINITE;
        const float r = or_rmsnorm_scale(xr, K, eps);
        if (!isfinite(r)) return OR_ERR_NONFINITE;  /* all-zero row with eps = 0 */
        for (int j = 0; j < K; ++j) {
            const float tj = bf16_to_f32(f32_to_bf16_rne(bf16_to_f32(xr[j]) * r));
            y[m * ldy + j] = f32_to_bf16_rne(bf16_to_f32(gamma[j]) * tj);
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* SiLU-mul stage: the producer of the down-projection input site.  The     */
/* paper's decoder layer (Fig.5) quantizes every linear input; the   */
/* down_proj input is h = SiLU(gate) * up of the bf16 gate/up outputs.      */
/* Reading Q24 (the paper is silent on how SiLU is evaluated): the ops of a */
/* bf16 model -- s = SiLU(g) in fp32, rounded to bf16, then bf16(s * u) --  */
/* with the fp32 SiLU pinned as this sequence of IEEE RN binary32 ops:      */
/*   a  = max(-|g|, -104)                                                   */
/*   n  = rint(a * L2E)              (ties to even)                         */
/*   r  = fma(n, -LN2_HI, a);  r = fma(n, -LN2_LO, r)     (Cody-Waite)      */
/*   p  = Horner over C7..C0 = RN(1/k!), one fma per step (Taylor e^r)      */
/*   E  = (p * 2^n1) * 2^n2,  n1 = trunc(n/2), n2 = n - n1   (= e^-|g|)     */
/*   d  = 1 + E;  rc = 1 / d                                                */
/*   s  = (g >= 0 ? g : g * E) * rc  (sigma(g) = 1/(1+e^-g), or E/(1+E))    */
/*   h  = bf16( bf16(s) * u )        (the product of two bf16 is exact)     */
/* Pinned (tests/test_oracle_silu.py) against long-double SiLU over every   */
/* finite bf16 g, against the correctly rounded bf16 SiLU, and against      */
/* torch's bf16 SiLU and SiLU*mul on CPU.                                   */
/* ------------------------------------------------------------------------- */
static const float SILU_L2E = 0x1.715476p+0f;      /* RN(1/ln 2) */
static const float SILU_LN2_HI = 0x1.62e4p-1f;     /* 15 significant bits: n * LN2_HI exact for |n| <= 150 */
static const float SILU_LN2_LO = 0x1.7f7d1cp-20f;  /* RN(ln 2 - LN2_HI) */
static const float SILU_C[8] = {1.0f, 1.0f, 0x1p-1f, 0x1.555556p-3f, 0x1.555556p-5f,
                                0x1.111112p-7f, 0x1.6c16c2p-10f, 0x1.a01a02p-13f};  /* RN(1/k!) */

float or_silu_f32(float g) {
    float a = -fabsf(g);
    if (a < -104.0f) a = -104.0f;
    const float n = rintf(a * SILU_L2E);
    float r = fmaf(n, -SILU_LN2_HI, a);
    r = fmaf(n, -SILU_LN2_LO, r);
    float p = SILU_C[7];
    for (int k = 6; k >= 0; --k) p = fmaf(p, r, SILU_C[k]);
    const int ni = (int)n, n1 = ni / 2, n2 = ni - n1;   /* C division truncates toward zero */
    const float E = (p * ldexpf(1.0f, n1)) * ldexpf(1.0f, n2);
    const float d = 1.0f + E;
    const float rc = 1.0f / d;
    const float q = g >= 0.0f ? g : g * E;
    return q * rc;
}

void or_silu_f32_n(const uint16_t* g, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = or_silu_f32(bf16_to_f32(g[i]));
}

/* h[m][j] = bf16(bf16(SiLU(gu[m][j])) * gu[m][up_off + j]) for j < K */
int or_silu_mul(const uint16_t* gu, int64_t M, int K, int64_t ld, int64_t up_off, uint16_t* h, int64_t ldh) {
    if (K <= 0 || M < 0 || up_off < K || ld < up_off + K || ldh < K) return OR_ERR_SHAPE;
    for (int64_t m = 0; m < M; ++m) {
        const uint16_t* row = gu + m * ld;
        for (int j = 0; j < K; ++j) {
            const float g = bf16_to_f32(row[j]), u = bf16_to_f32(row[up_off + j]);
            if (!isfinite(g) || !isfinite(u)) return OR_ERR_NONFINITE;
            const float s = bf16_to_f32(f32_to_bf16_rne(or_silu_f32(g)));
            h[m * ldh + j] = f32_to_bf16_rne(s * u);
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* MXFP4-ARC (f3): the paper's generalisation to MXFP4 (Table 6        */
/* P:509-535; SPEC: MXFP4 => g = 32, E8M0 scale, no tensor scale).  Reading    */
/* Q25: per 32-channel block (two consecutive logical 16-blocks) of the       */
/* reordered row:                                                             */
/*   a = max|z|; a = 0 -> scale "zero" (byte 0x00), t = z (codes 0 / -0)       */
/*   d = E8M0_up(a / 6) = 2^e (a/6 one fp32 RN division), t = z * 2^-e (exact) */
/*   q = rne_e2m1_sat(t)                                                      */
/*   residual (outlier blocks): r = t - v(q) (exact, units of 2^e),           */
/*   d2 = E8M0_up(max|r| / 6) = 2^e2, u = r * 2^-e2, q2 = rne(u); absolute     */
/*   residual scale 2^(e+e2) = E8M0_up(max|x - d v(q)| / 6) exactly.           */
/* Physical format: the NVFP4 one (so the same tcgen05 GEMM consumes it):     */
/* both 16-halves of a 32-block carry the E4M3 code of 2^(e - c), with the    */
/* tensor offset gs = 2^-c folded into alpha = 1/(gs_x gs_w).  Reading Q25b:  */
/* a block exponent outside E4M3's powers of two (e - c outside [-9, 8]) is   */
/* clamped into that range before t is formed (the residual's absolute       */
/* exponent e + e2 likewise), so such a block flushes toward 0 or saturates  */
/* at +-6 with a scale that matches its codes -- as NVFP4's saturating E4M3  */
/* scale does (P:118 names the tensor scale as what keeps blocks in range).  */
/* ------------------------------------------------------------------------- */
#define OR_ERR_RANGE 8

static int mx_ceil_log2(float raw) {      /* smallest e with 2^e >= raw > 0 */
    int e;
    float f = frexpf(raw, &e);            /* raw = f 2^e, f in [0.5, 1) */
    return f == 0.5f ? e - 1 : e;
}

static uint8_t mx_code(int k) {          /* E4M3 code of 2^k, k in [-9, 8] */
    return or_e4m3_ceil(ldexpf(1.0f, k)); /* exact: 2^k is an E4M3 value */
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* one 32-block: t (E2M1 units), q; *e_out = block exponent, clamped to [lo, hi] (Q25b),
 * INT32_MIN for an all-zero block */
static void mx_stage(const float z[32], int lo, int hi, float t[32], uint8_t q[32], int* e_out) {
    float a = 0.0f;
    for (int i = 0; i < 32; ++i)
        if (fabsf(z[i]) > a) a = fabsf(z[i]);
    if (a == 0.0f) {
        for (int i = 0; i < 32; ++i) { t[i] = z[i]; q[i] = or_e2m1_encode(t[i]); }
        *e_out = INT32_MIN;
        return;
    }
    const int e = clampi(mx_ceil_log2(a / 6.0f), lo, hi);
    for (int i = 0; i < 32; ++i) { t[i] = ldexpf(z[i], -e); q[i] = or_e2m1_encode(t[i]); }
    *e_out = e;
}

/* logical row (as or_arc_row_logical): codes[K+S] one per byte, sf[(K+S)/16] physical E4M3 bytes */
int or_arc_row_logical_mx(const uint16_t* x_row, const int32_t* perm, int K, int S, int c, int weight,
                          uint8_t* codes, uint8_t* sf) {
    if (K <= 0 || K % 32 || S < 0 || S % 32 || S > K) return OR_ERR_SHAPE;
    const int nb = K / 16;
    for (int b = 0; b < K / 32; ++b) {
        float z[32], t[32], r[32], u[32];
        uint8_t q[32], q2[32], s = 0, s2 = 0;
        int e, e2;
        for (int i = 0; i < 32; ++i) {
            z[i] = bf16_to_f32(x_row[perm[32 * b + i]]);
            if (!isfinite(z[i])) return OR_ERR_NONFINITE;
        }
        mx_stage(z, c - 9, c + 8, t, q, &e);
        if (e != INT32_MIN) s = mx_code(e - c);
        memcpy(codes + 32 * b, q, 32);
        sf[2 * b] = sf[2 * b + 1] = s;
        if (b < S / 32) {
            if (weight) {                                      /* duplicate */
                memcpy(codes + K + 32 * b, q, 32);
                sf[nb + 2 * b] = sf[nb + 2 * b + 1] = s;
                continue;
            }
            for (int i = 0; i < 32; ++i) r[i] = t[i] - or_e2m1_value(q[i]);   /* exact */
            if (e == INT32_MIN) {                               /* zero block: zero residual */
                mx_stage(r, 0, 0, u, q2, &e2);
            } else {
                mx_stage(r, c - 9 - e, c + 8 - e, u, q2, &e2);  /* e + e2 in [c-9, c+8] */
            }
            s2 = (e != INT32_MIN && e2 != INT32_MIN) ? mx_code(e + e2 - c) : 0;
            memcpy(codes + K + 32 * b, q2, 32);
            sf[nb + 2 * b] = sf[nb + 2 * b + 1] = s2;
        }
    }
    return OR_OK;
}

int or_quantize_mx(const uint16_t* x, int64_t M, int K, int64_t ldx, const int32_t* perm, int S, int c, int weight,
                   int layout, uint8_t* codes, uint8_t* sf) {
    int64_t Kp = or_kp(K, S);
    uint8_t* lc = (uint8_t*)malloc((size_t)(K + S));
    uint8_t* ls = (uint8_t*)malloc((size_t)((K + S) / 16 + 1));
    int rc = OR_OK;
    for (int64_t m = 0; m < M && rc == OR_OK; ++m) {
        rc = or_arc_row_logical_mx(x + m * ldx, perm, K, S, c, weight, lc, ls);
        if (rc == OR_OK) or_pack_row(lc, ls, K, S, layout, m, codes + m * (Kp / 2), sf);
    }
    free(lc);
    free(ls);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* Native MXFP4-ARC (reading Q25 without the NVFP4-format offset): */
/* the same 32-block stages as above with the exponent range of UE8M0        */
/* itself ([-127, 127]: no offset, nothing clamped in practice), stored as   */
/* the MX physical format of tcgen05 kind::mxf4 -- packed E2M1 codes and one */
/* UE8M0 byte (e + 127; an all-zero block 0) per 32-block, the App.D block    */
/* map at 32-element granularity (interleaved: outlier 32-block j -> 2j, its */
/* residual -> 2j+1), K+S padded to Kpm = roundup(K+S, 128), scales in the    */
/* 128x4 tile layout with Kpm/32 columns.                                     */
/* ------------------------------------------------------------------------- */
int64_t or_kpm(int K, int S) { return ((int64_t)K + S + 127) / 128 * 128; }

int or_quantize_mx_native(const uint16_t* x, int64_t M, int K, int64_t ldx, const int32_t* perm, int S, int weight,
                          int layout, uint8_t* codes, uint8_t* sf) {
    if (K <= 0 || K % 32 || S < 0 || S % 32 || S > K || M < 0 || ldx < K) return OR_ERR_SHAPE;
    const int64_t Kpm = or_kpm(K, S);
    const int nb = K / 32, ns = S / 32, nphys = (int)(Kpm / 32);
    for (int64_t m = 0; m < M; ++m)
        for (int j = 0; j < K; ++j)
            if (!isfinite(bf16_to_f32(x[m * ldx + j]))) return OR_ERR_NONFINITE;
    #pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        uint8_t* crow = codes + m * (Kpm / 2);
        memset(crow, 0, (size_t)(Kpm / 2));
        for (int pb = 0; pb < nphys; ++pb) sf[or_sf_offset(m, pb, Kpm / 2)] = 0;
        for (int b = 0; b < nb; ++b) {
            float z[32], t[32], r[32], u[32];
            uint8_t q[32], q2[32];
            int e, e2;
            for (int i = 0; i < 32; ++i) z[i] = bf16_to_f32(x[m * ldx + perm[32 * b + i]]);
            mx_stage(z, -127, 127, t, q, &e);
            const int pp = layout == 1 ? b : (b < ns ? 2 * b : b + ns);   /* physical primary block */
            for (int i = 0; i < 32; i += 2) crow[pp * 16 + i / 2] = (uint8_t)(q[i] | (q[i + 1] << 4));
            sf[or_sf_offset(m, pp, Kpm / 2)] = e == INT32_MIN ? 0 : (uint8_t)(e + 127);
            if (b < ns) {
                const int pr = layout == 1 ? nb + b : 2 * b + 1;               /* physical residual block */
                uint8_t s2 = 0;
                if (weight) {                                                  /* duplicate */
                    memcpy(q2, q, 32);
                    s2 = e == INT32_MIN ? 0 : (uint8_t)(e + 127);
                } else {
                    for (int i = 0; i < 32; ++i) r[i] = t[i] - or_e2m1_value(q[i]);   /* exact */
                    if (e == INT32_MIN) mx_stage(r, 0, 0, u, q2, &e2);
                    else mx_stage(r, -127 - e, 127 - e, u, q2, &e2);
                    s2 = (e != INT32_MIN && e2 != INT32_MIN) ? (uint8_t)(e + e2 + 127) : 0;
                }
                for (int i = 0; i < 32; i += 2) crow[pr * 16 + i / 2] = (uint8_t)(q2[i] | (q2[i + 1] << 4));
                sf[or_sf_offset(m, pr, Kpm / 2)] = s2;
            }
        }
    }
    return OR_OK;
}

/* Exact native-MX GEMM: per 32-block the int64 sum of V_a V_b (V = 2 e2m1, an integer) scaled by
 * 2^(ea + eb - 254 - 2) in double; |.| sums for the bound.  Y, Yabs: [nrows][N]. */
void or_gemm_mx_native_exact(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes, const uint8_t* b_sf,
                             int64_t N, int64_t Kpm, const int64_t* rows, int64_t nrows, double* Y, double* Yabs) {
    #pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        for (int64_t ri = 0; ri < nrows; ++ri) {
            const int64_t r = rows[ri];
            double acc = 0.0, aabs = 0.0;
            for (int64_t b = 0; b < Kpm / 32; ++b) {
                int64_t s = 0, sa = 0;
                for (int i = 0; i < 32; ++i) {
                    const int64_t p = b * 32 + i;
                    const uint8_t ab = a_codes[r * (Kpm / 2) + p / 2], bb = b_codes[n * (Kpm / 2) + p / 2];
                    const int64_t va = (int64_t)(2.0f * or_e2m1_value((p & 1) ? (ab >> 4) : (ab & 15)));
                    const int64_t vb = (int64_t)(2.0f * or_e2m1_value((p & 1) ? (bb >> 4) : (bb & 15)));
                    s += va * vb;
                    sa += va * vb < 0 ? -va * vb : va * vb;
                }
                const int e = (int)a_sf[or_sf_offset(r, b, Kpm / 2)] + (int)b_sf[or_sf_offset(n, b, Kpm / 2)] - 254 - 2;
                acc += ldexp((double)s, e);
                aabs += ldexp((double)sa, e);
            }
            Y[ri * N + n] = acc;
            Yabs[ri * N + n] = aabs;
        }
    }
}

/* tensor offset c for a tensor whose largest |value| is amax: the largest block scale
 * E8M0_up(amax/6) = 2^E maps to 2^8 (E4M3's largest power of two): c = E - 8; amax = 0 -> 0 */
int or_mx_offset(float amax) { return amax > 0.0f ? mx_ceil_log2(amax / 6.0f) - 8 : 0; }
