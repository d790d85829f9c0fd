"""Thin ctypes binding of libarc.so (include/arc.h) -- argument marshalling only.

Every computation runs in libarc.so's sm_100a kernels (or, for the host-side
outlier selection, in libarc.so's C++).  PyTorch provides device memory and the
current CUDA stream; nothing here computes on tensors.  If libarc.so is missing
the import fails loudly: there is no CPU or PyTorch fallback.

Names follow the paper (§3.2): calibrate -> (perm, S) profile,
quantize_weight, quantize_activation, gemm / linear.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libarc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built (python -m paper_2601_07475_b200.build); "
                      "the ARC hot path has no fallback")

_lib = ctypes.CDLL(LIB_PATH)

INTERLEAVED = 0
CONTIGUOUS = 1
BF16 = 0
FP32 = 2

_P = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f32 = ctypes.c_float


class ArcProfile(ctypes.Structure):
    _fields_ = [("K", _i64), ("S", _i32), ("perm", _P), ("gs", _P), ("layout", ctypes.c_int)]


class ArcQWeight(ctypes.Structure):
    _fields_ = [("N", _i64), ("K", _i64), ("Kp", _i64), ("S", _i32), ("layout", ctypes.c_int),
                ("codes", _P), ("sf", _P), ("gs", _P)]


class ArcReduce(ctypes.Structure):
    _fields_ = [("mode", _i32), ("npeers", _i32), ("mc", _P), ("peers", _P * 8)]


REDUCE_MULTIMEM = 1  # arc.h ARC_REDUCE_MULTIMEM
REDUCE_PEERS = 2     # arc.h ARC_REDUCE_PEERS


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_lib.arc_status_string.restype = ctypes.c_char_p
_lib.arc_status_string.argtypes = [ctypes.c_int]
_lib.arc_last_error.restype = ctypes.c_char_p
_lib.arc_last_error.argtypes = []
_sig("arc_device_supported", [])
_sig("arc_buffer_sizes", [_i64, _i64, _i32, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_size_t),
                          ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_gemm_workspace_size", [_i64, ctypes.POINTER(ArcQWeight), ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_linear_workspace_size", [_i64, ctypes.POINTER(ArcQWeight), ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_calib_absmax", [_P, _i64, _i64, _i64, _P, _P])
_sig("arc_select_outliers", [_P, _i64, _i32, _P, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                             ctypes.POINTER(_f32), ctypes.POINTER(_f32), ctypes.POINTER(_f32)])
_sig("arc_gather_order", [_P, _i64, _P])
_sig("arc_tensor_scale", [_P, _i64, _i64, _i64, _P, _P])
_sig("arc_quantize_weight", [_P, _i64, _i64, _i64, _P, _i32, _P, ctypes.c_int, _P, _P, _P])
_sig("arc_quantize_activation", [_P, _i64, _i64, ctypes.POINTER(ArcProfile), _P, _P, _P])
_sig("arc_gemm", [_P, _P, _P, _i64, ctypes.POINTER(ArcQWeight), _P, ctypes.c_int, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_linear", [_P, _i64, _i64, ctypes.POINTER(ArcProfile), ctypes.POINTER(ArcQWeight), _P, ctypes.c_int,
                    _i64, _P, ctypes.c_size_t, _P])
_sig("arc_linear_ex", [_P, _i64, _i64, ctypes.POINTER(ArcProfile), ctypes.POINTER(ArcQWeight), _P, ctypes.c_int,
                       _i64, _P, ctypes.c_size_t, ctypes.c_int, _P])
_sig("arc_linear_ex_workspace_size", [_i64, ctypes.POINTER(ArcQWeight), ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_rmsnorm", [_P, _i64, _i64, _i64, _P, _f32, _P, _i64, _P])
_sig("arc_rmsnorm_quantize_activation", [_P, _i64, _i64, _P, _f32, ctypes.POINTER(ArcProfile), _P, _P, _P])
_sig("arc_linear_rmsnorm", [_P, _i64, _i64, _P, _f32, ctypes.POINTER(ArcProfile), ctypes.POINTER(ArcQWeight), _P,
                            ctypes.c_int, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_gather_order_ex", [_P, _i64, ctypes.c_int, _P])
_sig("arc_mx_tensor_scale", [_f32, ctypes.POINTER(_f32)])
_sig("arc_mx_tensor_scale_device", [_P, _i64, _i64, _i64, _P, _P])
_sig("arc_quantize_activation_mx", [_P, _i64, _i64, ctypes.POINTER(ArcProfile), _P, _P, _P])
_sig("arc_quantize_weight_mx", [_P, _i64, _i64, _i64, _P, _i32, _P, ctypes.c_int, _P, _P, _P])
_sig("arc_gemm_reduce", [_P, _P, _P, _i64, ctypes.POINTER(ArcQWeight), ctypes.POINTER(ArcReduce), _i64, _P,
                         ctypes.c_size_t, _P])
_sig("arc_mx_native_buffer_sizes", [_i64, _i64, _i32, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_size_t),
                                    ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_quantize_mx_native", [_P, _i64, _i64, _i64, _P, _i32, _i32, ctypes.c_int, _P, _P, _P])
_sig("arc_gemm_mx_native_workspace_size", [_i64, _i64, _i64, ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_gemm_mx_native", [_P, _P, _i64, _P, _P, _i64, _i64, _P, ctypes.c_int, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_mxfp8_buffer_sizes", [_i64, _i64, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_size_t),
                                ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_quantize_mxfp8", [_P, _i64, _i64, _i64, _P, _P, _P])
_sig("arc_gemm_mxfp8_workspace_size", [_i64, _i64, _i64, ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_gemm_w4a8", [_P, _P, _i64, _P, _P, _i64, _i64, _P, ctypes.c_int, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_gemm_mxfp8", [_P, _P, _i64, _P, _P, _i64, _i64, _P, ctypes.c_int, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_gemm_swiglu", [_P, _P, _P, _i64, ctypes.POINTER(ArcQWeight), _P, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_silu_mul", [_P, _i64, _i64, _i64, _i64, _P, _i64, _P])
_sig("arc_silu_mul_quantize_activation", [_P, _i64, _i64, _i64, ctypes.POINTER(ArcProfile), _P, _P, _P])
_sig("arc_linear_silu_mul", [_P, _i64, _i64, _i64, ctypes.POINTER(ArcProfile), ctypes.POINTER(ArcQWeight), _P,
                             ctypes.c_int, _i64, _P, ctypes.c_size_t, _P])
_sig("arc_linear_hostio_workspace_size", [_i64, ctypes.POINTER(ArcQWeight), ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_size_t)])
_sig("arc_linear_hostio", [_P, _i64, ctypes.POINTER(ArcProfile), ctypes.POINTER(ArcQWeight), _P, ctypes.c_int, _P,
                           ctypes.c_size_t, _P])
_sig("arc_linear_hostio_async", [_P, _i64, ctypes.POINTER(ArcProfile), ctypes.POINTER(ArcQWeight), _P, ctypes.c_int,
                                 _P, ctypes.c_size_t, _P])
_sig("arc_linear_hostio_wait", [_P])
_sig("arc_calib_absmax_ex", [_P, ctypes.c_int, _i64, _i64, _i64, _P, _P])
_sig("arc_tensor_scale_ex", [_P, ctypes.c_int, _i64, _i64, _i64, _P, _P])
_sig("arc_quantize_weight_ex", [_P, ctypes.c_int, _i64, _i64, _i64, _P, ctypes.c_int32, _P, ctypes.c_int, _P, _P, _P])
_sig("arc_quantize_activation_ex", [_P, ctypes.c_int, _i64, _i64, ctypes.POINTER(ArcProfile), _P, _P, _P])
_sig("arc_probe_e2m1", [_P, _i64, _P, _P])
_sig("arc_probe_e2m1_bits", [ctypes.c_uint32, _i64, _P, _P])
_sig("arc_probe_e2m1_raw_bits", [ctypes.c_uint32, _i64, _P, _P])
_sig("arc_probe_e4m3_ceil", [_P, _i64, _P, _P])
_sig("arc_probe_silu", [_P, _i64, _P, _P])
_sig("arc_probe_u4_unpack", [_P, _i64, _P, _P])

# every symbol include/arc.h and include/arc_probe.h declare (checked by tests)
EXPORTED = [
    "arc_status_string", "arc_last_error", "arc_device_supported", "arc_buffer_sizes", "arc_gemm_workspace_size",
    "arc_linear_workspace_size",
    "arc_calib_absmax", "arc_select_outliers", "arc_gather_order", "arc_tensor_scale", "arc_quantize_weight",
    "arc_quantize_activation", "arc_gemm", "arc_linear", "arc_linear_ex", "arc_linear_ex_workspace_size",
    "arc_linear_hostio_workspace_size", "arc_rmsnorm",
    "arc_rmsnorm_quantize_activation", "arc_linear_rmsnorm", "arc_linear_hostio",
    "arc_silu_mul", "arc_silu_mul_quantize_activation", "arc_linear_silu_mul", "arc_gemm_swiglu", "arc_gemm_reduce",
    "arc_mx_native_buffer_sizes", "arc_quantize_mx_native", "arc_gemm_mx_native_workspace_size", "arc_gemm_mx_native",
    "arc_mxfp8_buffer_sizes", "arc_quantize_mxfp8", "arc_gemm_mxfp8_workspace_size", "arc_gemm_mxfp8", "arc_gemm_w4a8",
    "arc_mx_tensor_scale", "arc_mx_tensor_scale_device", "arc_quantize_activation_mx", "arc_quantize_weight_mx", "arc_gather_order_ex",
    "arc_probe_e2m1", "arc_probe_e2m1_bits", "arc_probe_e2m1_raw_bits", "arc_probe_e4m3_ceil", "arc_probe_silu",
    "arc_probe_u4_unpack",
    "arc_debug_stream_trace", "arc_debug_trace", "arc_linear_hostio_async", "arc_linear_hostio_wait",
    "arc_calib_absmax_ex", "arc_tensor_scale_ex", "arc_quantize_weight_ex", "arc_quantize_activation_ex",
]


class ArcError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_lib.arc_status_string(status).decode()} "
                         f"({_lib.arc_last_error().decode()})")


def _check(st: int, where: str):
    if st != 0:
        raise ArcError(st, where)


def lib():
    return _lib


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def device_supported() -> bool:
    return bool(_lib.arc_device_supported())


def buffer_sizes(rows: int, K: int, S: int):
    kp = _i64()
    cb = ctypes.c_size_t()
    sb = ctypes.c_size_t()
    _check(_lib.arc_buffer_sizes(rows, K, S, ctypes.byref(kp), ctypes.byref(cb), ctypes.byref(sb)),
           "arc_buffer_sizes")
    return kp.value, cb.value, sb.value


def gemm_workspace_size(M: int, qw) -> int:
    b = ctypes.c_size_t()
    _check(_lib.arc_gemm_workspace_size(M, ctypes.byref(qw.c()), ctypes.byref(b)), "arc_gemm_workspace_size")
    return b.value


def linear_workspace_size(M: int, qw) -> int:
    b = ctypes.c_size_t()
    _check(_lib.arc_linear_workspace_size(M, ctypes.byref(qw.c()), ctypes.byref(b)), "arc_linear_workspace_size")
    return b.value


# --------------------------------------------------------------------------- profile / weights
@dataclass
class Profile:
    """Calibration profile of one activation site."""
    K: int
    S: int
    perm: torch.Tensor          # device int32 [K]
    gs: torch.Tensor            # device float32 [1], static encode tensor scale 2688/M
    layout: int = INTERLEAVED
    S_raw: int = 0
    M: float = 0.0
    tau: float = 0.0
    _c: ArcProfile = field(default=None, repr=False)

    def c(self) -> ArcProfile:
        self._c = ArcProfile(self.K, self.S, _ptr(self.perm), _ptr(self.gs), self.layout)
        return self._c


@dataclass
class QWeight:
    """A prepared ARC weight: reordered, NVFP4-quantized, outlier blocks duplicated."""
    N: int
    K: int
    Kp: int
    S: int
    layout: int
    codes: torch.Tensor         # uint8 [N, Kp/2]
    sf: torch.Tensor            # uint8 [roundup(N,128) * Kp/16]
    gs: torch.Tensor            # float32 [1]
    _c: ArcQWeight = field(default=None, repr=False)

    def c(self) -> ArcQWeight:
        self._c = ArcQWeight(self.N, self.K, self.Kp, self.S, self.layout, _ptr(self.codes), _ptr(self.sf),
                             _ptr(self.gs))
        return self._c


ARC_FP16 = 1  # arc.h arc_dtype_t
LINEAR_X_FP16 = 16  # arc.h ARC_LINEAR_X_FP16


def _in16(x: torch.Tensor) -> int:
    """arc_dtype_t of a 16-bit input tensor: ARC_BF16 (0) or ARC_FP16 (1)."""
    assert x.dtype in (torch.bfloat16, torch.float16), x.dtype
    return ARC_FP16 if x.dtype == torch.float16 else 0


def calib_absmax(x: torch.Tensor, chan_max: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Running per-channel abs-max over bf16 / fp16 rows (device)."""
    assert x.is_cuda and x.dim() == 2
    rows, K = x.shape
    if chan_max is None:
        chan_max = torch.zeros(K, dtype=torch.float32, device=x.device)
    _check(_lib.arc_calib_absmax_ex(_ptr(x), _in16(x), rows, K, x.stride(0), _ptr(chan_max), _stream(stream)),
           "arc_calib_absmax_ex")
    return chan_max


def select_outliers(chan_max_host: np.ndarray, s_override: int = -1) -> dict:
    cm = np.ascontiguousarray(chan_max_host, dtype=np.float32)
    K = cm.size
    perm = np.zeros(K, np.int32)
    S, S_raw = _i32(), _i32()
    M, tau, gs = _f32(), _f32(), _f32()
    _check(_lib.arc_select_outliers(cm.ctypes.data_as(_P), K, s_override, perm.ctypes.data_as(_P), ctypes.byref(S),
                                    ctypes.byref(S_raw), ctypes.byref(M), ctypes.byref(tau), ctypes.byref(gs)),
           "arc_select_outliers")
    return dict(perm=perm, S=S.value, S_raw=S_raw.value, M=M.value, tau=tau.value, gs=gs.value)


def gather_order(perm: np.ndarray, elem_bytes: int = 2) -> np.ndarray:
    """Bank-conflict-aware channel order inside each 16-channel block (same block sets); elem_bytes 4
    for (gate, up) pair rows (ARC_GU_PAIRS)."""
    p = np.ascontiguousarray(perm, dtype=np.int32)
    out = np.empty_like(p)
    _check(_lib.arc_gather_order_ex(p.ctypes.data_as(_P), p.size, int(elem_bytes), out.ctypes.data_as(_P)),
           "arc_gather_order_ex")
    return out


def calibrate(batches, s_override: int = -1, layout: int = INTERLEAVED, device=None,
              optimize_gather: bool = True, gather_bytes: int = 2) -> Profile:
    """Offline calibration of one activation site over an iterable of bf16 [rows, K] batches.
    With optimize_gather the channel order inside each 16-block is re-arranged for
    conflict-free shared-memory gathers (arc_gather_order; block sets unchanged)."""
    chan_max = None
    for b in batches:
        chan_max = calib_absmax(b, chan_max)
    torch.cuda.current_stream().synchronize()
    sel = select_outliers(chan_max.cpu().numpy(), s_override)
    if optimize_gather:
        sel["perm"] = gather_order(sel["perm"], gather_bytes)
    dev = chan_max.device if device is None else device
    return Profile(K=chan_max.numel(), S=sel["S"], perm=torch.from_numpy(sel["perm"]).to(dev),
                   gs=torch.tensor([sel["gs"]], dtype=torch.float32, device=dev), layout=layout,
                   S_raw=sel["S_raw"], M=sel["M"], tau=sel["tau"])


def profile_from(perm, S: int, gs: float, layout: int = INTERLEAVED, device="cuda") -> Profile:
    perm = torch.as_tensor(np.asarray(perm, np.int32)).to(device)
    return Profile(K=perm.numel(), S=S, perm=perm, gs=torch.tensor([gs], dtype=torch.float32, device=device),
                   layout=layout)


def tensor_scale(x: torch.Tensor, stream=None) -> torch.Tensor:
    """Device gs = 2688/amax(x) (reading Q3)."""
    gs = torch.empty(1, dtype=torch.float32, device=x.device)
    _check(_lib.arc_tensor_scale_ex(_ptr(x), _in16(x), x.shape[0], x.shape[1], x.stride(0), _ptr(gs), _stream(stream)),
           "arc_tensor_scale_ex")
    return gs


def quantize_weight(w: torch.Tensor, prof: Profile, gs: torch.Tensor | None = None, stream=None) -> QWeight:
    assert w.is_cuda and w.dim() == 2 and w.shape[1] == prof.K
    N, K = w.shape
    Kp, cb, sb = buffer_sizes(N, K, prof.S)
    if gs is None:
        gs = tensor_scale(w, stream)
    codes = torch.empty(N, Kp // 2, dtype=torch.uint8, device=w.device)
    sf = torch.empty(sb, dtype=torch.uint8, device=w.device)
    _check(_lib.arc_quantize_weight_ex(_ptr(w), _in16(w), N, K, w.stride(0), _ptr(prof.perm), prof.S, _ptr(gs),
                                       prof.layout, _ptr(codes), _ptr(sf), _stream(stream)), "arc_quantize_weight_ex")
    return QWeight(N=N, K=K, Kp=Kp, S=prof.S, layout=prof.layout, codes=codes, sf=sf, gs=gs)


def quantize_activation(x: torch.Tensor, prof: Profile, codes=None, sf=None, stream=None):
    assert x.is_cuda and x.dim() == 2 and x.shape[1] == prof.K
    M = x.shape[0]
    Kp, cb, sb = buffer_sizes(M, prof.K, prof.S)
    if codes is None:
        codes = torch.empty(M, Kp // 2, dtype=torch.uint8, device=x.device)
    if sf is None:
        sf = torch.empty(sb, dtype=torch.uint8, device=x.device)
    _check(_lib.arc_quantize_activation_ex(_ptr(x), _in16(x), M, x.stride(0), ctypes.byref(prof.c()), _ptr(codes),
                                           _ptr(sf), _stream(stream)), "arc_quantize_activation_ex")
    return codes, sf


def _alloc_out(M: int, N: int, dtype, device) -> torch.Tensor:
    """Output buffer whose row stride is a multiple of 16 bytes (the C ABI's ldy rule)."""
    per16 = 16 // torch.empty(0, dtype=dtype).element_size()
    ld = (N + per16 - 1) // per16 * per16
    return torch.empty(M, ld, dtype=dtype, device=device)[:, :N]


def _dtype_code(dt) -> int:
    if dt == torch.bfloat16:
        return BF16
    if dt == torch.float32:
        return FP32
    raise ValueError("out_dtype must be torch.bfloat16 or torch.float32")


class Workspace:
    """Grow-only device workspace for arc_gemm / arc_linear (256-byte aligned by the
    allocator, zero-filled on allocation: the decode-size GEMM's per-tile arrival counters must start
    at 0, and every call leaves them at 0).  A Workspace belongs to
    one stream: calls that share one must be ordered on that stream (the defaults are per stream)."""

    def __init__(self, device="cuda"):
        self.device = device
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self.buf


_default_ws = {}


def _default_workspace(kind, device, stream=None) -> "Workspace":
    """Per-(kind, device, stream) default workspace: calls on different streams never share (and so
    never race on) one buffer, and a buffer grown on one stream is not freed under another's kernel."""
    return _default_ws.setdefault((kind, str(device), _stream(stream)), Workspace(device))


def gemm(a_codes, a_sf, gs_x: torch.Tensor, qw: QWeight, out_dtype=torch.bfloat16, out=None, ws: Workspace = None,
         stream=None):
    """The augmented NVFP4 GEMM (Eq.2): out = A_aug B_aug^T / (gs_x gs_w)."""
    M = a_codes.shape[0]
    if out is None:
        out = _alloc_out(M, qw.N, out_dtype, a_codes.device)
    need = gemm_workspace_size(M, qw)
    buf = None
    if need:
        if ws is None:
            ws = _default_workspace("gemm", a_codes.device, stream)
        buf = ws.get(need)
    _check(_lib.arc_gemm(_ptr(a_codes), _ptr(a_sf), _ptr(gs_x), M, ctypes.byref(qw.c()), _ptr(out),
                         _dtype_code(out.dtype), out.stride(0), _ptr(buf), 0 if buf is None else buf.numel(),
                         _stream(stream)), "arc_gemm")
    return out


def gemm_swiglu(a_codes, a_sf, gs_x: torch.Tensor, qw: QWeight, out=None, ws: Workspace = None, stream=None):
    """arc_gemm with the SwiGLU epilogue: qw = a gate_up weight prepared from interleave_gate_up(...);
    out = h [M][N/2] bf16 = bf16(bf16(SiLU(g)) * u) of the bf16 GEMM output (Fig.5, reading Q24)."""
    M = a_codes.shape[0]
    if out is None:
        out = torch.empty(M, qw.N // 2, dtype=torch.bfloat16, device=a_codes.device)
    need = gemm_workspace_size(M, qw)
    buf = None
    if need:
        if ws is None:
            ws = _default_workspace("gemm", a_codes.device, stream)
        buf = ws.get(need)
    _check(_lib.arc_gemm_swiglu(_ptr(a_codes), _ptr(a_sf), _ptr(gs_x), M, ctypes.byref(qw.c()), _ptr(out),
                                out.stride(0), _ptr(buf), 0 if buf is None else buf.numel(), _stream(stream)),
           "arc_gemm_swiglu")
    return out


def gemm_reduce(a_codes, a_sf, gs_x: torch.Tensor, qw: QWeight, ldy: int, mc_ptr: int = 0, peer_ptrs=(),
                ws: Workspace = None, stream=None):
    """arc_gemm_reduce: this rank's partial GEMM ADDED into every rank's fp32 [M][ldy] output buffer --
    through the NVLS multicast address mc_ptr (multimem.red) when given, else into each device address of
    peer_ptrs (P2P red.add).  The buffers must be zero before any rank starts (see arc.h)."""
    M = a_codes.shape[0]
    red = ArcReduce()
    if mc_ptr:
        red.mode, red.mc = REDUCE_MULTIMEM, int(mc_ptr)
    else:
        red.mode, red.npeers = REDUCE_PEERS, len(peer_ptrs)
        for i, p in enumerate(peer_ptrs):
            red.peers[i] = int(p)
    need = gemm_workspace_size(M, qw)
    buf = None
    if need:
        if ws is None:
            ws = _default_workspace("gemm", a_codes.device, stream)
        buf = ws.get(need)
    _check(_lib.arc_gemm_reduce(_ptr(a_codes), _ptr(a_sf), _ptr(gs_x), M, ctypes.byref(qw.c()), ctypes.byref(red),
                                ldy, _ptr(buf), 0 if buf is None else buf.numel(), _stream(stream)),
           "arc_gemm_reduce")


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor, group: int = 16) -> torch.Tensor:
    """Offline weight layout, gate/up rows interleaved in groups: group 16 for arc_gemm_swiglu (rows
    32j..32j+15 = gate rows 16j.., rows 32j+16..32j+31 = up rows 16j..); group 1 for ARC_GU_PAIRS
    (the GEMM output then holds (g_j, u_j) adjacent pairs).  Layout only."""
    I, K = w_gate.shape
    assert w_up.shape == (I, K) and I % group == 0
    return torch.stack([w_gate.view(I // group, group, K), w_up.view(I // group, group, K)],
                       dim=1).reshape(2 * I, K).contiguous()


def deinterleave_gate_up(y: torch.Tensor, group: int = 16) -> torch.Tensor:
    """Columns of a GEMM output over interleave_gate_up weights back to [gate | up].  Layout only."""
    M, N = y.shape
    v = y.reshape(M, N // (2 * group), 2, group)
    return torch.cat([v[:, :, 0, :].reshape(M, N // 2), v[:, :, 1, :].reshape(M, N // 2)], dim=1)


LINEAR_MODES = {"auto": 0, "fused": 1, "unfused": 2}  # arc.h ARC_LINEAR_AUTO / _FUSED / _UNFUSED


def linear_workspace_size_ex(M: int, qw, mode: str = "auto") -> int:
    b = ctypes.c_size_t()
    _check(_lib.arc_linear_ex_workspace_size(M, ctypes.byref(qw.c()), LINEAR_MODES[mode], ctypes.byref(b)),
           "arc_linear_ex_workspace_size")
    return b.value


def linear(x: torch.Tensor, prof: Profile, qw: QWeight, out_dtype=torch.bfloat16, out=None, ws: Workspace = None,
           stream=None, mode: str = "auto"):
    """The ARC linear layer (Eq.2): activation quantize + augmented NVFP4 GEMM.  mode "unfused" = two
    PDL-chained kernels; "fused" (M <= 64) = one kernel that quantizes the activation and runs the
    weight-streaming stream-K GEMM (arc.h ARC_LINEAR_FUSED); "auto" = unfused (faster at every M).  x may be bf16
    or fp16 (ARC_LINEAR_X_FP16: the two-kernel path)."""
    assert x.is_cuda
    xf = LINEAR_X_FP16 if _in16(x) == ARC_FP16 else 0
    M = x.shape[0]
    if out is None:
        out = _alloc_out(M, qw.N, out_dtype, x.device)
    need = linear_workspace_size_ex(M, qw, mode)
    if ws is None:
        ws = _default_workspace("linear", x.device, stream)
    buf = ws.get(need)
    _check(_lib.arc_linear_ex(_ptr(x), M, x.stride(0), ctypes.byref(prof.c()), ctypes.byref(qw.c()), _ptr(out),
                              _dtype_code(out.dtype), out.stride(0), _ptr(buf), buf.numel(), LINEAR_MODES[mode] | xf,
                              _stream(stream)),
           "arc_linear_ex")
    return out


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float, out=None, stream=None) -> torch.Tensor:
    """The RMSNorm stage of the fused quantization kernel, reading Q23: bf16 -> bf16."""
    assert x.dtype == torch.bfloat16 and gamma.dtype == torch.bfloat16 and x.is_cuda
    M, K = x.shape
    if out is None:
        out = torch.empty(M, K, dtype=torch.bfloat16, device=x.device)
    _check(_lib.arc_rmsnorm(_ptr(x), M, K, x.stride(0), _ptr(gamma), float(eps), _ptr(out), out.stride(0),
                            _stream(stream)), "arc_rmsnorm")
    return out


def rmsnorm_quantize_activation(x: torch.Tensor, gamma: torch.Tensor, eps: float, prof: Profile, codes=None,
                                sf=None, stream=None):
    """quantize_activation(rmsnorm(x)) in one pass over x (the paper's fused kernel)."""
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.shape[1] == prof.K
    M = x.shape[0]
    Kp, cb, sb = buffer_sizes(M, prof.K, prof.S)
    if codes is None:
        codes = torch.empty(M, Kp // 2, dtype=torch.uint8, device=x.device)
    if sf is None:
        sf = torch.empty(sb, dtype=torch.uint8, device=x.device)
    _check(_lib.arc_rmsnorm_quantize_activation(_ptr(x), M, x.stride(0), _ptr(gamma), float(eps),
                                                ctypes.byref(prof.c()), _ptr(codes), _ptr(sf), _stream(stream)),
           "arc_rmsnorm_quantize_activation")
    return codes, sf


def linear_rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float, prof: Profile, qw: QWeight,
                   out_dtype=torch.bfloat16, out=None, ws: Workspace = None, stream=None):
    """ARC linear of rmsnorm(x): the normalizing quantize pass + the augmented NVFP4 GEMM."""
    assert x.dtype == torch.bfloat16 and x.is_cuda
    M = x.shape[0]
    if out is None:
        out = _alloc_out(M, qw.N, out_dtype, x.device)
    need = linear_workspace_size(M, qw)
    if ws is None:
        ws = _default_workspace("linear", x.device, stream)
    buf = ws.get(need)
    _check(_lib.arc_linear_rmsnorm(_ptr(x), M, x.stride(0), _ptr(gamma), float(eps), ctypes.byref(prof.c()),
                                   ctypes.byref(qw.c()), _ptr(out), _dtype_code(out.dtype), out.stride(0), _ptr(buf),
                                   buf.numel(), _stream(stream)), "arc_linear_rmsnorm")
    return out


GU_PAIRS = -1  # up_off value: gu holds (gate_j, up_j) adjacent pairs (ARC_GU_PAIRS)


# ----------------------------------------------------------------------------- MXFP4-ARC (f3)
def mx_tensor_scale(amax: float) -> float:
    """gs = 2^-c for a tensor with max |x| = amax (reading Q25)."""
    g = _f32()
    _check(_lib.arc_mx_tensor_scale(float(amax), ctypes.byref(g)), "arc_mx_tensor_scale")
    return float(g.value)


def mx_profile(prof: "Profile", amax: float | None = None) -> "Profile":
    """The same calibration (perm, S) with the MX tensor offset as gs (static: from the calibration
    max prof.M unless amax is given)."""
    if amax is None:
        amax = prof.M
    return Profile(K=prof.K, S=prof.S, perm=prof.perm,
                   gs=torch.tensor([mx_tensor_scale(amax)], dtype=torch.float32, device=prof.perm.device),
                   layout=prof.layout, S_raw=prof.S_raw, M=prof.M, tau=prof.tau)


def quantize_activation_mx(x: torch.Tensor, prof: "Profile", codes=None, sf=None, stream=None):
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.shape[1] == prof.K
    M = x.shape[0]
    Kp, cb, sb = buffer_sizes(M, prof.K, prof.S)
    if codes is None:
        codes = torch.empty(M, Kp // 2, dtype=torch.uint8, device=x.device)
    if sf is None:
        sf = torch.empty(sb, dtype=torch.uint8, device=x.device)
    _check(_lib.arc_quantize_activation_mx(_ptr(x), M, x.stride(0), ctypes.byref(prof.c()), _ptr(codes), _ptr(sf),
                                           _stream(stream)), "arc_quantize_activation_mx")
    return codes, sf


def quantize_weight_mx(w: torch.Tensor, prof: "Profile", stream=None) -> "QWeight":
    """MXFP4-ARC weight (outlier blocks duplicated) with gs_w = 2^-c_w from max |w|."""
    assert w.dtype == torch.bfloat16 and w.is_cuda
    N, K = w.shape
    Kp, cb, sb = buffer_sizes(N, K, prof.S)
    codes = torch.empty(N, Kp // 2, dtype=torch.uint8, device=w.device)
    sf = torch.empty(sb, dtype=torch.uint8, device=w.device)
    gs = torch.empty(1, dtype=torch.float32, device=w.device)
    _check(_lib.arc_mx_tensor_scale_device(_ptr(w), N, K, w.stride(0), _ptr(gs), _stream(stream)),
           "arc_mx_tensor_scale_device")
    _check(_lib.arc_quantize_weight_mx(_ptr(w), N, K, w.stride(0), _ptr(prof.perm), prof.S, _ptr(gs), prof.layout,
                                       _ptr(codes), _ptr(sf), _stream(stream)), "arc_quantize_weight_mx")
    return QWeight(N=N, K=K, Kp=Kp, S=prof.S, layout=prof.layout, codes=codes, sf=sf, gs=gs)


def _gu_args(gu: torch.Tensor, K: int | None, up_off: int | None):
    assert gu.dtype == torch.bfloat16 and gu.is_cuda and gu.dim() == 2 and gu.stride(1) == 1
    K = gu.shape[1] // 2 if K is None else K
    return K, (K if up_off is None else up_off)


def silu_mul(gu: torch.Tensor, K: int | None = None, up_off: int | None = None, out=None, stream=None):
    """Down-proj input h = bf16(bf16(SiLU(gate)) * up) (Fig.5, reading Q24) of gu = [gate | up]
    (gate in columns [0, K), up in [up_off, up_off + K); default the fused gate_up output), or of
    (gate_j, up_j) adjacent pairs with up_off = GU_PAIRS."""
    K, up_off = _gu_args(gu, K, up_off)
    M = gu.shape[0]
    if out is None:
        out = torch.empty(M, K, dtype=torch.bfloat16, device=gu.device)
    _check(_lib.arc_silu_mul(_ptr(gu), M, K, gu.stride(0), up_off, _ptr(out), out.stride(0), _stream(stream)),
           "arc_silu_mul")
    return out


def silu_mul_quantize_activation(gu: torch.Tensor, prof: Profile, up_off: int | None = None, codes=None, sf=None,
                                 stream=None):
    """quantize_activation(silu_mul(gu)) in one pass over gu (h never reaches HBM)."""
    K, up_off = _gu_args(gu, prof.K, up_off)
    M = gu.shape[0]
    Kp, cb, sb = buffer_sizes(M, prof.K, prof.S)
    if codes is None:
        codes = torch.empty(M, Kp // 2, dtype=torch.uint8, device=gu.device)
    if sf is None:
        sf = torch.empty(sb, dtype=torch.uint8, device=gu.device)
    _check(_lib.arc_silu_mul_quantize_activation(_ptr(gu), M, gu.stride(0), up_off, ctypes.byref(prof.c()),
                                                 _ptr(codes), _ptr(sf), _stream(stream)),
           "arc_silu_mul_quantize_activation")
    return codes, sf


def linear_silu_mul(gu: torch.Tensor, prof: Profile, qw: QWeight, up_off: int | None = None,
                    out_dtype=torch.bfloat16, out=None, ws: Workspace = None, stream=None):
    """ARC linear of silu_mul(gu) (the down_proj site): the SiLU-mul quantize pass + the augmented NVFP4 GEMM."""
    K, up_off = _gu_args(gu, prof.K, up_off)
    M = gu.shape[0]
    if out is None:
        out = _alloc_out(M, qw.N, out_dtype, gu.device)
    need = linear_workspace_size(M, qw)
    if ws is None:
        ws = _default_workspace("linear", gu.device, stream)
    buf = ws.get(need)
    _check(_lib.arc_linear_silu_mul(_ptr(gu), M, gu.stride(0), up_off, ctypes.byref(prof.c()), ctypes.byref(qw.c()),
                                    _ptr(out), _dtype_code(out.dtype), out.stride(0), _ptr(buf), buf.numel(),
                                    _stream(stream)), "arc_linear_silu_mul")
    return out


def linear_hostio_workspace_size(M: int, qw, out_dtype=torch.bfloat16) -> int:
    b = ctypes.c_size_t()
    _check(_lib.arc_linear_hostio_workspace_size(M, ctypes.byref(qw.c()), _dtype_code(out_dtype), ctypes.byref(b)),
           "arc_linear_hostio_workspace_size")
    return b.value


def linear_hostio(x_host: torch.Tensor, prof: Profile, qw: QWeight, y_host: torch.Tensor, ws: torch.Tensor,
                  stream=None, wait: bool = True):
    """arc_linear on host buffers: H2D of x, the linear and D2H of y pipelined over row chunks (arc.h).
    wait=False: arc_linear_hostio_async (returns once enqueued; call linear_hostio_wait before touching
    x_host / y_host / ws)."""
    assert not x_host.is_cuda and not y_host.is_cuda
    fn = _lib.arc_linear_hostio if wait else _lib.arc_linear_hostio_async
    _check(fn(_ptr(x_host), x_host.shape[0], ctypes.byref(prof.c()), ctypes.byref(qw.c()),
              _ptr(y_host), _dtype_code(y_host.dtype), _ptr(ws), ws.numel(), _stream(stream)),
           "arc_linear_hostio" if wait else "arc_linear_hostio_async")
    return y_host


def linear_hostio_wait(stream=None):
    """Wait for every linear_hostio(wait=False) call on the current device."""
    _check(_lib.arc_linear_hostio_wait(_stream(stream)), "arc_linear_hostio_wait")


# --------------------------------------------------------------------------- probes (tests only)
def probe_e2m1(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
    _check(_lib.arc_probe_e2m1(_ptr(x), x.numel(), _ptr(out), _stream()), "arc_probe_e2m1")
    return out


def probe_e2m1_bits(start: int, n: int, device="cuda") -> torch.Tensor:
    out = torch.empty(n, dtype=torch.uint8, device=device)
    _check(_lib.arc_probe_e2m1_bits(start, n, _ptr(out), _stream()), "arc_probe_e2m1_bits")
    return out


def probe_e2m1_raw_bits(start: int, n: int, device="cuda") -> torch.Tensor:
    out = torch.empty(n, dtype=torch.uint8, device=device)
    _check(_lib.arc_probe_e2m1_raw_bits(start, n, _ptr(out), _stream()), "arc_probe_e2m1_raw_bits")
    return out


def probe_e4m3_ceil(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty(x.numel(), dtype=torch.uint8, device=x.device)
    _check(_lib.arc_probe_e4m3_ceil(_ptr(x), x.numel(), _ptr(out), _stream()), "arc_probe_e4m3_ceil")
    return out


def probe_u4_unpack(packed: torch.Tensor):
    """(status[2], smem bytes[2, 8192]) of the 16U4_ALIGN16B TMA layout probe (arc_probe.h)."""
    rows = packed.shape[0]
    out = torch.empty(16384, dtype=torch.uint8, device=packed.device)
    st = torch.zeros(2, dtype=torch.int32, device=packed.device)
    _check(_lib.arc_probe_u4_unpack(_ptr(packed), rows, _ptr(out), _ptr(st)), "arc_probe_u4_unpack")
    return st.cpu(), out.view(2, 8192).cpu()


def probe_silu(g_bits: torch.Tensor) -> torch.Tensor:
    """bf16 patterns of bf16(SiLU(g)) as the fused SiLU-mul quantize kernel computes them
    (g_bits: int16/uint16-viewed bf16 patterns on the device)."""
    out = torch.empty(g_bits.numel(), dtype=torch.int16, device=g_bits.device)
    _check(_lib.arc_probe_silu(_ptr(g_bits), g_bits.numel(), _ptr(out), _stream()), "arc_probe_silu")
    return out


# ----------------------------------------------------------------------------- Fig.8a comparator: MXFP8
def quantize_mxfp8(x: torch.Tensor, stream=None):
    """Plain MXFP8 (arc.h arc_quantize_mxfp8): E4M3 codes [rows][Kp8] and E8M0 scales (128x4 tile layout)."""
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.dim() == 2
    rows, K = x.shape
    k8, cb, sb = _i64(), ctypes.c_size_t(), ctypes.c_size_t()
    _check(_lib.arc_mxfp8_buffer_sizes(rows, K, ctypes.byref(k8), ctypes.byref(cb), ctypes.byref(sb)),
           "arc_mxfp8_buffer_sizes")
    codes = torch.empty(rows, k8.value, dtype=torch.uint8, device=x.device)
    sf = torch.empty(sb.value, dtype=torch.uint8, device=x.device)
    _check(_lib.arc_quantize_mxfp8(_ptr(x), rows, K, x.stride(0), _ptr(codes), _ptr(sf), _stream(stream)),
           "arc_quantize_mxfp8")
    return codes, sf


def gemm_mxfp8(a_codes, a_sf, b_codes, b_sf, K: int, out_dtype=torch.bfloat16, out=None, ws: Workspace = None,
               stream=None):
    """arc_gemm_mxfp8: y = A B^T of two plain-MXFP8 operands (the Fig.8a comparison GEMM)."""
    M, N = a_codes.shape[0], b_codes.shape[0]
    if out is None:
        out = _alloc_out(M, N, out_dtype, a_codes.device)
    b = ctypes.c_size_t()
    _check(_lib.arc_gemm_mxfp8_workspace_size(M, N, K, ctypes.byref(b)), "arc_gemm_mxfp8_workspace_size")
    buf = None
    if b.value:
        if ws is None:
            ws = _default_workspace("gemm", a_codes.device, stream)
        buf = ws.get(b.value)
    _check(_lib.arc_gemm_mxfp8(_ptr(a_codes), _ptr(a_sf), M, _ptr(b_codes), _ptr(b_sf), N, K, _ptr(out),
                               _dtype_code(out.dtype), out.stride(0), _ptr(buf), 0 if buf is None else buf.numel(),
                               _stream(stream)), "arc_gemm_mxfp8")
    return out


# ----------------------------------------------------------------------------- native MXFP4-ARC (f3)
def quantize_mx_native(x: torch.Tensor, prof: "Profile", weight: bool = False, stream=None):
    """Native MXFP4-ARC (arc.h arc_quantize_mx_native): codes [rows][Kpm/2], UE8M0 scales (128x4 tile layout)."""
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.dim() == 2 and x.shape[1] == prof.K
    rows, K = x.shape
    km, cb, sb = _i64(), ctypes.c_size_t(), ctypes.c_size_t()
    _check(_lib.arc_mx_native_buffer_sizes(rows, K, prof.S, ctypes.byref(km), ctypes.byref(cb), ctypes.byref(sb)),
           "arc_mx_native_buffer_sizes")
    codes = torch.empty(rows, km.value // 2, dtype=torch.uint8, device=x.device)
    sf = torch.empty(sb.value, dtype=torch.uint8, device=x.device)
    _check(_lib.arc_quantize_mx_native(_ptr(x), rows, K, x.stride(0), _ptr(prof.perm), prof.S, int(bool(weight)),
                                       prof.layout, _ptr(codes), _ptr(sf), _stream(stream)), "arc_quantize_mx_native")
    return codes, sf


def gemm_mx_native(a_codes, a_sf, b_codes, b_sf, out_dtype=torch.bfloat16, out=None, ws: Workspace = None,
                   stream=None):
    """arc_gemm_mx_native: y = A B^T of two native MXFP4-ARC operands (tcgen05 kind::mxf4 scale_vec::2X)."""
    M, N, Kpm = a_codes.shape[0], b_codes.shape[0], 2 * a_codes.shape[1]
    if out is None:
        out = _alloc_out(M, N, out_dtype, a_codes.device)
    b = ctypes.c_size_t()
    _check(_lib.arc_gemm_mx_native_workspace_size(M, N, Kpm, ctypes.byref(b)), "arc_gemm_mx_native_workspace_size")
    buf = None
    if b.value:
        if ws is None:
            ws = _default_workspace("gemm", a_codes.device, stream)
        buf = ws.get(b.value)
    _check(_lib.arc_gemm_mx_native(_ptr(a_codes), _ptr(a_sf), M, _ptr(b_codes), _ptr(b_sf), N, Kpm, _ptr(out),
                                   _dtype_code(out.dtype), out.stride(0), _ptr(buf), 0 if buf is None else buf.numel(),
                                   _stream(stream)), "arc_gemm_mx_native")
    return out


def gemm_w4a8(a_codes, a_sf, b_codes, b_sf, K: int, out_dtype=torch.bfloat16, out=None, ws: Workspace = None,
              stream=None):
    """arc_gemm_w4a8: MXFP8 activations (quantize_mxfp8) x plain MXFP4 weights (quantize_mx_native with S = 0,
    identity order) -- the Fig.8a W4A8 comparison GEMM."""
    M, N = a_codes.shape[0], b_codes.shape[0]
    if out is None:
        out = _alloc_out(M, N, out_dtype, a_codes.device)
    b = ctypes.c_size_t()
    _check(_lib.arc_gemm_mxfp8_workspace_size(M, N, K, ctypes.byref(b)), "arc_gemm_mxfp8_workspace_size")
    buf = None
    if b.value:
        if ws is None:
            ws = _default_workspace("gemm", a_codes.device, stream)
        buf = ws.get(b.value)
    _check(_lib.arc_gemm_w4a8(_ptr(a_codes), _ptr(a_sf), M, _ptr(b_codes), _ptr(b_sf), N, K, _ptr(out),
                              _dtype_code(out.dtype), out.stride(0), _ptr(buf), 0 if buf is None else buf.numel(),
                              _stream(stream)), "arc_gemm_w4a8")
    return out
