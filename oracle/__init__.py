"""CPU oracle for the ARCQuant (arxiv 2601.07475) hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2601_07475_b200``) never imports it; the two share no code.

The arithmetic lives in ``arc_oracle.c`` (plain C, fp32 RNE in a pinned op order,
int64-exact GEMM); this module only compiles it with gcc and marshals numpy
arrays through ctypes.  Every function cites the PAPER.md passage it follows in
the C source.  What pins each function is listed in the C header comment and
tested in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "arc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_libs = {}
_variant = "serial"

INTERLEAVED = 0
CONTIGUOUS = 1


def _compile(out: str, extra) -> None:
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-Wno-unknown-pragmas",
                           *extra, "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, out)


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, no fast-math) and the same source with
    -fopenmp as liboracle_omp.so (rows / output columns split over host threads; identical
    arithmetic per element -- the bench's multi-core CPU baseline)."""
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            _compile(out, extra)
    return _LIB


class openmp:
    """Context manager: oracle calls inside use the OpenMP build (all host cores unless
    OMP_NUM_THREADS says otherwise)."""

    def __enter__(self):
        global _variant
        self.prev, _variant = _variant, "omp"
        return self

    def __exit__(self, *a):
        global _variant
        _variant = self.prev


def num_threads() -> int:
    """Threads the current variant uses."""
    return int(lib().or_num_threads())


def lib():
    if _variant not in _libs:
        build()
        L = ctypes.CDLL(_LIB_OMP if _variant == "omp" else _LIB)
        P = ctypes.c_void_p
        i64, i32, f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_float
        L.or_e2m1_value.restype = f32
        L.or_e2m1_value.argtypes = [ctypes.c_uint8]
        L.or_e2m1_encode.restype = ctypes.c_uint8
        L.or_e2m1_encode.argtypes = [f32]
        L.or_e4m3_value.restype = f32
        L.or_e4m3_value.argtypes = [ctypes.c_uint8]
        L.or_e4m3_ceil.restype = ctypes.c_uint8
        L.or_e4m3_ceil.argtypes = [f32]
        L.or_e4m3_rn.restype = ctypes.c_uint8
        L.or_e4m3_rn.argtypes = [f32]
        L.or_e8m0_up.restype = f32
        L.or_e8m0_up.argtypes = [f32]
        L.or_stage.restype = None
        L.or_stage.argtypes = [P, f32, P, P, P, P]
        L.or_arc_row_logical.restype = i32
        L.or_arc_row_logical.argtypes = [P, P, i32, i32, f32, P, P]
        L.or_weight_row_logical.restype = i32
        L.or_weight_row_logical.argtypes = [P, P, i32, i32, f32, P, P]
        L.or_physical_block.restype = i32
        L.or_physical_block.argtypes = [i32, i32, i32, i32]
        L.or_kp.restype = i64
        L.or_kp.argtypes = [i32, i32]
        L.or_sf_offset.restype = i64
        L.or_sf_offset.argtypes = [i64, i64, i64]
        L.or_quantize_activation.restype = i32
        L.or_quantize_activation.argtypes = [P, i64, i32, i64, P, i32, f32, i32, P, P]
        L.or_quantize_weight.restype = i32
        L.or_quantize_weight.argtypes = [P, i64, i32, i64, P, i32, f32, i32, P, P]
        L.or_calib_absmax.restype = i32
        L.or_calib_absmax.argtypes = [P, i64, i32, i64, P]
        L.or_f16_to_f32.restype = ctypes.c_float
        L.or_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.or_set_input_fp16.restype = None
        L.or_set_input_fp16.argtypes = [i32]
        L.or_select_outliers.restype = i32
        L.or_select_outliers.argtypes = [P, i32, i32, P, P, P, P, P]
        L.or_gemm_exact.restype = None
        L.or_gemm_exact.argtypes = [P, P, P, P, i64, i64, P, i64, P, P]
        L.or_mxfp8_block.restype = None
        L.or_mxfp8_block.argtypes = [P, P, P]
        L.or_rmsnorm.restype = i32
        L.or_rmsnorm.argtypes = [P, i64, i32, i64, P, f32, P, i64]
        L.or_rmsnorm_scale.restype = f32
        L.or_rmsnorm_scale.argtypes = [P, i32, f32]
        L.or_quantize_mx.restype = i32
        L.or_quantize_mx.argtypes = [P, i64, i32, i64, P, i32, i32, i32, i32, P, P]
        L.or_mx_offset.restype = i32
        L.or_mx_offset.argtypes = [f32]
        L.or_silu_f32_n.restype = None
        L.or_silu_f32_n.argtypes = [P, i64, P]
        L.or_silu_mul.restype = i32
        L.or_silu_mul.argtypes = [P, i64, i32, i64, i64, P, i64]
        for n in ("or_e2m1_encode_n", "or_e4m3_ceil_n", "or_e4m3_rn_n"):
            getattr(L, n).restype = None
            getattr(L, n).argtypes = [P, i64, P]
        L.or_kpm.restype = i64
        L.or_kpm.argtypes = [i32, i32]
        L.or_quantize_mx_native.restype = i32
        L.or_quantize_mx_native.argtypes = [P, i64, i32, i64, P, i32, i32, i32, P, P]
        L.or_gemm_mx_native_exact.restype = None
        L.or_gemm_mx_native_exact.argtypes = [P, P, P, P, i64, i64, P, i64, P, P]
        L.or_gemm_w4a8_exact.restype = None
        L.or_gemm_w4a8_exact.argtypes = [P, P, P, P, i64, i64, P, i64, P, P]
        L.or_kp8.restype = i64
        L.or_kp8.argtypes = [i32]
        L.or_quantize_mxfp8.restype = i32
        L.or_quantize_mxfp8.argtypes = [P, i64, i32, i64, P, P]
        L.or_gemm_mxfp8_exact.restype = None
        L.or_gemm_mxfp8_exact.argtypes = [P, P, P, P, i64, i64, P, i64, P, P]
        L.or_num_threads.restype = i32
        L.or_num_threads.argtypes = []
        _libs[_variant] = L
    return _libs[_variant]


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise OracleError({2: "shape", 7: "non-finite input"}.get(rc, f"rc={rc}"))


def as_fp16_bits(x) -> np.ndarray:
    """Accept a torch float16 tensor or a uint16 array of IEEE binary16 bits."""
    if hasattr(x, "view") and hasattr(x, "dtype") and str(x.dtype) == "torch.float16":
        import torch
        return x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    a = np.ascontiguousarray(x)
    assert a.dtype == np.uint16
    return a


def f16_to_f32(bits: int) -> float:
    """The oracle's IEEE binary16 decode (arc_oracle.c or_f16_to_f32)."""
    return float(lib().or_f16_to_f32(int(bits)))


class _InputFp16:
    """Within the block the C quantizers / calibration read their 16-bit rows as IEEE fp16 (arc_dtype_t
    ARC_FP16) instead of bf16."""

    def __enter__(self):
        lib().or_set_input_fp16(1)

    def __exit__(self, *a):
        lib().or_set_input_fp16(0)


def _bits16(x, fp16: bool):
    return as_fp16_bits(x) if fp16 else as_bf16_bits(x)


def as_bf16_bits(x) -> np.ndarray:
    """Accept a torch bf16 tensor or a uint16 array of bf16 bits."""
    if hasattr(x, "view") and hasattr(x, "dtype") and str(x.dtype) == "torch.bfloat16":
        import torch
        return x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    a = np.ascontiguousarray(x)
    assert a.dtype == np.uint16
    return a


# ----------------------------------------------------------------------------- codecs
def e2m1_value(q: int) -> float:
    return float(lib().or_e2m1_value(q))


def e2m1_encode(t) -> np.ndarray:
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float32).reshape(-1))
    out = np.empty(t.size, np.uint8)
    lib().or_e2m1_encode_n(_p(t), t.size, _p(out))
    return out


def e4m3_value(c: int) -> float:
    return float(lib().or_e4m3_value(c))


def e4m3_ceil(v) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float32).reshape(-1))
    out = np.empty(v.size, np.uint8)
    lib().or_e4m3_ceil_n(_p(v), v.size, _p(out))
    return out


def e4m3_rn(v) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float32).reshape(-1))
    out = np.empty(v.size, np.uint8)
    lib().or_e4m3_rn_n(_p(v), v.size, _p(out))
    return out


def e8m0_up(v: float) -> float:
    return float(lib().or_e8m0_up(v))


E2M1_TABLE = None  # filled lazily from the C decoder


def e2m1_values() -> np.ndarray:
    return np.array([e2m1_value(q) for q in range(16)], np.float32)


def e4m3_values() -> np.ndarray:
    return np.array([e4m3_value(c) for c in range(256)], np.float32)


def stage(z, base: float):
    """C4 STAGE on one 16-element block -> (sf, d, t[16], q[16])."""
    z = np.ascontiguousarray(np.asarray(z, np.float32).reshape(16))
    t = np.empty(16, np.float32)
    q = np.empty(16, np.uint8)
    sf = np.zeros(1, np.uint8)
    d = np.zeros(1, np.float32)
    lib().or_stage(_p(z), base, _p(sf), _p(d), _p(t), _p(q))
    return int(sf[0]), float(d[0]), t, q


# ----------------------------------------------------------------------------- ARC rows
def arc_row_logical(x_row_bits, perm, S: int, gs: float):
    """C5: one activation row, logical order -> (codes[K+S], sf[(K+S)/16])."""
    x = as_bf16_bits(x_row_bits).reshape(-1)
    perm = np.ascontiguousarray(perm, np.int32)
    K = x.size
    codes = np.zeros(K + S, np.uint8)
    sf = np.zeros((K + S) // 16, np.uint8)
    _check(lib().or_arc_row_logical(_p(x), _p(perm), K, S, gs, _p(codes), _p(sf)))
    return codes, sf


def weight_row_logical(w_row_bits, perm, S: int, gs: float):
    w = as_bf16_bits(w_row_bits).reshape(-1)
    perm = np.ascontiguousarray(perm, np.int32)
    K = w.size
    codes = np.zeros(K + S, np.uint8)
    sf = np.zeros((K + S) // 16, np.uint8)
    _check(lib().or_weight_row_logical(_p(w), _p(perm), K, S, gs, _p(codes), _p(sf)))
    return codes, sf


def kp(K: int, S: int) -> int:
    return int(lib().or_kp(K, S))


def physical_block(l: int, K: int, S: int, layout: int) -> int:
    return int(lib().or_physical_block(l, K, S, layout))


def sf_offset(m: int, c: int, Kp: int) -> int:
    return int(lib().or_sf_offset(m, c, Kp))


def sf_rows_padded(rows: int) -> int:
    return (rows + 127) // 128 * 128


def quantize_activation(x_bits, perm, S: int, gs: float, layout: int = INTERLEAVED, fp16: bool = False):
    """C5+C8+C9: packed codes [M][Kp/2] and swizzled SF [roundup(M,128)*Kp/16].  fp16: the rows are IEEE
    binary16 (decoded exactly to fp32), else bf16."""
    if fp16:
        with _InputFp16():
            return quantize_activation(as_fp16_bits(x_bits), perm, S, gs, layout)
    x = as_bf16_bits(x_bits)
    M, K = x.shape
    Kp = kp(K, S)
    codes = np.zeros((M, Kp // 2), np.uint8)
    sf = np.zeros(sf_rows_padded(M) * Kp // 16, np.uint8)
    perm = np.ascontiguousarray(perm, np.int32)
    _check(lib().or_quantize_activation(_p(x), M, K, K, _p(perm), S, gs, layout, _p(codes), _p(sf)))
    return codes, sf


def quantize_weight(w_bits, perm, S: int, gs: float, layout: int = INTERLEAVED, fp16: bool = False):
    if fp16:
        with _InputFp16():
            return quantize_weight(as_fp16_bits(w_bits), perm, S, gs, layout)
    w = as_bf16_bits(w_bits)
    N, K = w.shape
    Kp = kp(K, S)
    codes = np.zeros((N, Kp // 2), np.uint8)
    sf = np.zeros(sf_rows_padded(N) * Kp // 16, np.uint8)
    perm = np.ascontiguousarray(perm, np.int32)
    _check(lib().or_quantize_weight(_p(w), N, K, K, _p(perm), S, gs, layout, _p(codes), _p(sf)))
    return codes, sf


# ----------------------------------------------------------------------------- MXFP4-ARC (f3)
def mx_offset(amax: float) -> int:
    """Tensor offset c (gs = 2^-c): the largest block scale E8M0_up(amax/6) maps to 2^8 (reading Q25)."""
    return int(lib().or_mx_offset(np.float32(amax)))


def quantize_mx(x_bits, perm, S: int, c: int, weight: bool = False, layout: int = INTERLEAVED):
    """MXFP4-ARC (32-blocks, E8M0 scales; residual or, for weights, duplicated outlier blocks) in the
    NVFP4 physical format with E4M3 codes of 2^(e - c): packed codes [rows][Kp/2], swizzled scales."""
    x = as_bf16_bits(x_bits)
    M, K = x.shape
    Kp = kp(K, S)
    codes = np.zeros((M, Kp // 2), np.uint8)
    sf = np.zeros(sf_rows_padded(M) * Kp // 16, np.uint8)
    perm = np.ascontiguousarray(perm, np.int32)
    rc = lib().or_quantize_mx(_p(x), M, K, K, _p(perm), S, int(c), int(bool(weight)), layout, _p(codes), _p(sf))
    if rc == 8:
        raise OracleError("block scale outside E4M3's powers of two for this tensor offset")
    _check(rc)
    return codes, sf


# ----------------------------------------------------------------------------- RMSNorm
def rmsnorm(x_bits, gamma_bits, eps: float) -> np.ndarray:
    """RMSNorm stage of the fused kernel, reading Q23: bf16 bits [M][K] -> bf16 bits."""
    x = as_bf16_bits(x_bits)
    g = np.ascontiguousarray(as_bf16_bits(gamma_bits).reshape(-1))
    M, K = x.shape
    assert g.size == K
    y = np.zeros((M, K), np.uint16)
    _check(lib().or_rmsnorm(_p(x), M, K, K, _p(g), np.float32(eps), _p(y), K))
    return y


def rmsnorm_scale(x_row_bits, eps: float) -> float:
    """r = 1/sqrt(ss/K + eps) of one row in the pinned order (Q23)."""
    x = np.ascontiguousarray(as_bf16_bits(x_row_bits).reshape(-1))
    return float(lib().or_rmsnorm_scale(_p(x), x.size, np.float32(eps)))


# ----------------------------------------------------------------------------- SiLU-mul
def silu_f32(g_bits) -> np.ndarray:
    """fp32 SiLU of bf16 inputs in the pinned op sequence of reading Q24 (before the bf16 rounding)."""
    g = np.ascontiguousarray(as_bf16_bits(g_bits).reshape(-1))
    out = np.zeros(g.size, np.float32)
    lib().or_silu_f32_n(_p(g), g.size, _p(out))
    return out


def silu_mul(gu_bits, K: int | None = None, up_off: int | None = None) -> np.ndarray:
    """Down-proj input h = bf16(bf16(SiLU(gate)) * up) (Fig.5, reading Q24).

    gu: bf16 bits [M][ld] holding gate in columns [0, K) and up in [up_off, up_off + K)
    (default: the fused gate_up output, K = ld / 2, up_off = K).  Returns bf16 bits [M][K]."""
    gu = as_bf16_bits(gu_bits)
    M, ld = gu.shape
    K = ld // 2 if K is None else K
    up_off = K if up_off is None else up_off
    h = np.zeros((M, K), np.uint16)
    _check(lib().or_silu_mul(_p(gu), M, K, ld, up_off, _p(h), K))
    return h


# ----------------------------------------------------------------------------- calibration
def calib_absmax(x_bits, chan_max=None, fp16: bool = False) -> np.ndarray:
    if fp16:
        with _InputFp16():
            return calib_absmax(as_fp16_bits(x_bits), chan_max)
    x = as_bf16_bits(x_bits)
    rows, K = x.shape
    cm = np.zeros(K, np.float32) if chan_max is None else np.ascontiguousarray(chan_max, np.float32)
    _check(lib().or_calib_absmax(_p(x), rows, K, K, _p(cm)))
    return cm


def select_outliers(chan_max, s_override: int = -1) -> dict:
    cm = np.ascontiguousarray(chan_max, np.float32)
    K = cm.size
    perm = np.zeros(K, np.int32)
    S = ctypes.c_int(0)
    S_raw = ctypes.c_int(0)
    M = ctypes.c_float(0)
    tau = ctypes.c_float(0)
    _check(lib().or_select_outliers(_p(cm), K, s_override, _p(perm), ctypes.byref(S),
                                    ctypes.byref(S_raw), ctypes.byref(M), ctypes.byref(tau)))
    gs = np.float32(2688.0) / np.float32(M.value) if M.value > 0 else np.float32(1.0)
    return dict(perm=perm, S=S.value, S_raw=S_raw.value, M=M.value, tau=tau.value, gs=float(gs))


def tensor_scale(amax: float) -> float:
    """Reading Q3: gs = 448*6/amax as one fp32 division (amax = 0 -> 1)."""
    amax = np.float32(amax)
    return float(np.float32(2688.0) / amax) if amax > 0 else 1.0


# ----------------------------------------------------------------------------- GEMM
def gemm_exact(a_codes, a_sf, b_codes, b_sf, rows=None):
    """C10: exact augmented GEMM in 2^-20 units -> (T, Tabs) int64 [len(rows)][N]."""
    a_codes = np.ascontiguousarray(a_codes, np.uint8)
    b_codes = np.ascontiguousarray(b_codes, np.uint8)
    a_sf = np.ascontiguousarray(a_sf, np.uint8)
    b_sf = np.ascontiguousarray(b_sf, np.uint8)
    M = a_codes.shape[0]
    N, half = b_codes.shape
    Kp = 2 * half
    assert a_codes.shape[1] == half
    rows = np.arange(M, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    T = np.zeros((rows.size, N), np.int64)
    Tabs = np.zeros((rows.size, N), np.int64)
    lib().or_gemm_exact(_p(a_codes), _p(a_sf), _p(b_codes), _p(b_sf), N, Kp, _p(rows), rows.size,
                        _p(T), _p(Tabs))
    return T, Tabs


def gemm_reference(a_codes, a_sf, b_codes, b_sf, gs_x: float, gs_w: float, rows=None):
    """Y_ref (float64) and the north_star bound 1e-5*sum|a*b| per element (C10)."""
    T, Tabs = gemm_exact(a_codes, a_sf, b_codes, b_sf, rows)
    inv = 1.0 / (float(np.float32(gs_x)) * float(np.float32(gs_w)))
    y = T.astype(np.float64) * 2.0 ** -20 * inv
    bound = 1e-5 * Tabs.astype(np.float64) * 2.0 ** -20 * inv
    return y, bound


def mxfp8_block(x32):
    x = np.ascontiguousarray(np.asarray(x32, np.float32).reshape(32))
    s = np.zeros(1, np.float32)
    xh = np.zeros(32, np.float32)
    lib().or_mxfp8_block(_p(x), _p(s), _p(xh))
    return float(s[0]), xh


# ----------------------------------------------------------------------------- Fig.8a MXFP8 comparator
def kp8(K: int) -> int:
    return int(lib().or_kp8(K))


def quantize_mxfp8(x_bits):
    """Plain MXFP8 (Eq.3 per 32-block, no reordering / residual; the Fig.8a comparison format):
    E4M3 codes [rows][Kp8] and E8M0 scale bytes in the 128x4 tile layout (Kp8/32 columns)."""
    x = as_bf16_bits(x_bits)
    M, K = x.shape
    K8 = kp8(K)
    codes = np.zeros((M, K8), np.uint8)
    sf = np.zeros(sf_rows_padded(M) * K8 // 32, np.uint8)
    _check(lib().or_quantize_mxfp8(_p(x), M, K, K, _p(codes), _p(sf)))
    return codes, sf


def gemm_mxfp8_reference(a_codes, a_sf, b_codes, b_sf, rows=None):
    """Exact MXFP8 x MXFP8 GEMM (float64 of exact per-block int64 sums) and the 1e-5 * sum|ab| bound."""
    a_codes = np.ascontiguousarray(a_codes, np.uint8)
    b_codes = np.ascontiguousarray(b_codes, np.uint8)
    a_sf = np.ascontiguousarray(a_sf, np.uint8)
    b_sf = np.ascontiguousarray(b_sf, np.uint8)
    M, K8 = a_codes.shape
    N = b_codes.shape[0]
    rows = np.arange(M, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    Y = np.zeros((rows.size, N))
    Yabs = np.zeros((rows.size, N))
    lib().or_gemm_mxfp8_exact(_p(a_codes), _p(a_sf), _p(b_codes), _p(b_sf), N, K8, _p(rows), rows.size, _p(Y), _p(Yabs))
    return Y, 1e-5 * Yabs


# ----------------------------------------------------------------------------- native MXFP4-ARC (f3)
def kpm(K: int, S: int) -> int:
    return int(lib().or_kpm(K, S))


def quantize_mx_native(x_bits, perm, S: int, weight: bool = False, layout: int = INTERLEAVED):
    """Native MXFP4-ARC (UE8M0 byte per 32-block, 32-granular block map, Kpm = roundup(K+S, 128)):
    packed E2M1 codes [rows][Kpm/2] and scale bytes in the 128x4 tile layout (Kpm/32 columns)."""
    x = as_bf16_bits(x_bits)
    M, K = x.shape
    Km = kpm(K, S)
    codes = np.zeros((M, Km // 2), np.uint8)
    sf = np.zeros(sf_rows_padded(M) * Km // 32, np.uint8)
    perm = np.ascontiguousarray(perm, np.int32)
    _check(lib().or_quantize_mx_native(_p(x), M, K, K, _p(perm), S, int(bool(weight)), layout, _p(codes), _p(sf)))
    return codes, sf


def gemm_mx_native_reference(a_codes, a_sf, b_codes, b_sf, rows=None):
    """Exact native-MXFP4 GEMM (float64 of exact per-block int64 sums) and the 1e-5 * sum|ab| bound."""
    a_codes = np.ascontiguousarray(a_codes, np.uint8)
    b_codes = np.ascontiguousarray(b_codes, np.uint8)
    a_sf = np.ascontiguousarray(a_sf, np.uint8)
    b_sf = np.ascontiguousarray(b_sf, np.uint8)
    M, half = a_codes.shape
    N = b_codes.shape[0]
    rows = np.arange(M, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    Y = np.zeros((rows.size, N))
    Yabs = np.zeros((rows.size, N))
    lib().or_gemm_mx_native_exact(_p(a_codes), _p(a_sf), _p(b_codes), _p(b_sf), N, 2 * half, _p(rows), rows.size,
                                  _p(Y), _p(Yabs))
    return Y, 1e-5 * Yabs


def gemm_w4a8_reference(a_codes, a_sf, b_codes, b_sf, rows=None):
    """Exact W4A8 GEMM (MXFP8 activations x plain MXFP4 weights) and the 1e-5 * sum|ab| bound."""
    a_codes = np.ascontiguousarray(a_codes, np.uint8)
    b_codes = np.ascontiguousarray(b_codes, np.uint8)
    a_sf = np.ascontiguousarray(a_sf, np.uint8)
    b_sf = np.ascontiguousarray(b_sf, np.uint8)
    M, K8 = a_codes.shape
    N = b_codes.shape[0]
    assert b_codes.shape[1] * 2 == K8
    rows = np.arange(M, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    Y = np.zeros((rows.size, N))
    Yabs = np.zeros((rows.size, N))
    lib().or_gemm_w4a8_exact(_p(a_codes), _p(a_sf), _p(b_codes), _p(b_sf), N, K8, _p(rows), rows.size, _p(Y), _p(Yabs))
    return Y, 1e-5 * Yabs
