"""Python binding of libisoquant (include/isoquant.h) — argument marshalling only.

Every step of the IsoQuant stage-1 path runs in the library's sm_100a
kernels; this module only passes torch tensors' device pointers and the
current CUDA stream through the C ABI, allocating outputs with torch when the
caller does not supply them.  There is no CPU fallback: if the shared
library is missing or fails to load, importing this package raises.

Names mirror the C ABI: iq_make_params, iq_quantize, iq_dequantize,
iq_roundtrip, iq_error_sums, iq_export_params, iq_export_block_matrices,
iq_code_bytes_per_vector, iq_host_roundtrip (via HostPipeline).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "FULL", "FAST", "PLANAR2D", "F32", "F16", "BF16", "IQError", "Params", "HostPipeline", "lib",
    "iq_make_params", "iq_quantize", "iq_dequantize", "iq_roundtrip", "iq_error_sums",
    "iq_export_params", "iq_export_block_matrices", "iq_code_bytes_per_vector",
    "iq_rotation_param_count", "iq_version", "LIB_PATH",
    "iq_make_params_qjl", "iq_qjl_bytes_per_vector", "iq_export_qjl_matrix", "iq_quantize_qjl",
    "iq_attention_scores", "iq_make_params_explicit", "iq_distortion_grad", "iq_rot_grad_from_operator_grad",
    "iq_make_params_sets", "iq_make_params_qjl_sets", "iq_export_params_set", "iq_append_kv",
]

FULL, FAST, PLANAR2D = 0, 1, 2
F32, F16, BF16 = 0, 1, 2
VARIANTS = {"full": FULL, "fast": FAST, "planar2d": PLANAR2D, "2d": PLANAR2D}

LIB_PATH = os.environ.get("IQ_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                         "libisoquant.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")
lib = ctypes.CDLL(LIB_PATH)

_c_int, _c_i64, _c_u64, _c_vp, _c_sz = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
_sig = {
    "iq_version": (ctypes.c_char_p, []),
    "iq_abi_version": (_c_int, []),
    "iq_status_string": (ctypes.c_char_p, [_c_int]),
    "iq_last_error_detail": (ctypes.c_char_p, []),
    "iq_make_params": (_c_int, [_c_int, _c_int, _c_int, _c_u64, _c_int, ctypes.POINTER(_c_vp)]),
    "iq_free_params": (_c_int, [_c_vp]),
    "iq_params_info": (_c_int, [_c_vp] + [ctypes.POINTER(_c_int)] * 4),
    "iq_code_bytes_per_vector": (_c_sz, [_c_int, _c_int]),
    "iq_rotation_param_count": (_c_sz, [_c_int, _c_int]),
    "iq_export_params": (_c_int, [_c_vp, _c_vp, _c_sz, _c_vp, _c_sz, _c_vp, _c_sz]),
    "iq_export_block_matrices": (_c_int, [_c_vp, _c_vp, _c_sz]),
    "iq_quantize": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_dequantize": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_roundtrip": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_error_sums": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_host_pipeline_create": (_c_int, [_c_vp, _c_int, _c_i64, ctypes.POINTER(_c_vp)]),
    "iq_host_pipeline_destroy": (_c_int, [_c_vp]),
    "iq_host_roundtrip": (_c_int, [_c_vp, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_make_params_qjl": (_c_int, [_c_int, _c_int, _c_int, _c_u64, _c_int, ctypes.POINTER(_c_vp)]),
    "iq_qjl_bytes_per_vector": (_c_sz, [_c_int]),
    "iq_export_qjl_matrix": (_c_int, [_c_vp, _c_vp, _c_sz]),
    "iq_quantize_qjl": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_attention_scores": (_c_int, [_c_vp, _c_int, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp, _c_int, _c_vp,
                                     _c_vp, _c_vp]),
    "iq_make_params_explicit": (_c_int, [_c_int, _c_int, _c_int, _c_vp, _c_sz, _c_int, ctypes.POINTER(_c_vp)]),
    "iq_distortion_grad": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "iq_rot_grad_from_operator_grad": (_c_int, [_c_vp, _c_vp, _c_sz, _c_vp, _c_sz]),
    "iq_make_params_sets": (_c_int, [_c_int, _c_int, _c_int, _c_u64, _c_int, _c_i64, _c_int, ctypes.POINTER(_c_vp)]),
    "iq_make_params_qjl_sets": (_c_int, [_c_int, _c_int, _c_int, _c_u64, _c_int, _c_i64, _c_int,
                                         ctypes.POINTER(_c_vp)]),
    "iq_params_sets_info": (_c_int, [_c_vp, ctypes.POINTER(_c_int), ctypes.POINTER(_c_i64)]),
    "iq_export_params_set": (_c_int, [_c_vp, _c_int, _c_vp, _c_sz]),
    "iq_append_kv": (_c_int, [_c_vp, _c_int, _c_i64, _c_vp, _c_vp, _c_vp, _c_i64, _c_vp, _c_i64, _c_vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class IQError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = lib.iq_status_string(status).decode()
        detail = lib.iq_last_error_detail().decode()
        super().__init__(f"{where}: {name}: {detail}")


def _check(status: int, where: str):
    if status != 0:
        raise IQError(status, where)


def iq_version() -> str:
    return lib.iq_version().decode()


def iq_code_bytes_per_vector(d: int, bits: int) -> int:
    return int(lib.iq_code_bytes_per_vector(d, bits))


def iq_rotation_param_count(d: int, variant: int) -> int:
    return int(lib.iq_rotation_param_count(d, variant))


class Params:
    """Owns an iq_params handle (freed on garbage collection)."""

    def __init__(self, handle: int, d: int, bits: int, variant: int, seed: int, device: int):
        self._h = ctypes.c_void_p(handle)
        self.d, self.bits, self.variant, self.seed, self.device = d, bits, variant, seed, device

    @property
    def handle(self):
        return self._h

    @property
    def code_bytes(self) -> int:
        return iq_code_bytes_per_vector(self.d, self.bits)

    def close(self):
        if self._h is not None and self._h.value:
            lib.iq_free_params(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def iq_make_params(d: int, bits: int, variant, seed: int, device: int = 0) -> Params:
    """Build parameters for (d, bits, variant) from ``seed`` on ``device``
    (-1 = host-only handle, for export)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant.lower()]
    h = ctypes.c_void_p()
    _check(lib.iq_make_params(int(d), int(bits), int(variant), ctypes.c_uint64(seed & (2**64 - 1)),
                              int(device), ctypes.byref(h)), "iq_make_params")
    return Params(h.value, d, bits, variant, seed, device)


def iq_make_params_qjl(d: int, bits: int, variant, seed: int, device: int = 0) -> Params:
    """iq_make_params plus the stage-2 residual sketch S (m = d)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant.lower()]
    h = ctypes.c_void_p()
    _check(lib.iq_make_params_qjl(int(d), int(bits), int(variant), ctypes.c_uint64(seed & (2**64 - 1)),
                                  int(device), ctypes.byref(h)), "iq_make_params_qjl")
    return Params(h.value, d, bits, variant, seed, device)


def iq_qjl_bytes_per_vector(d: int) -> int:
    return int(lib.iq_qjl_bytes_per_vector(d))


def iq_export_qjl_matrix(p: Params) -> np.ndarray:
    """S [m, d] (fp16 values as float32)."""
    S = np.zeros((p.d, p.d), dtype=np.float32)
    _check(lib.iq_export_qjl_matrix(p.handle, S.ctypes.data, S.size), "iq_export_qjl_matrix")
    return S


def iq_make_params_sets(d: int, bits: int, variant, seed: int, n_sets: int, set_rows: int, device: int = 0) -> Params:
    """n_sets rotation sets (set s = the seed + s parameters); row r uses set
    (r // set_rows) % n_sets, head h of the consumer set h % n_sets."""
    if isinstance(variant, str):
        variant = VARIANTS[variant.lower()]
    h = ctypes.c_void_p()
    _check(lib.iq_make_params_sets(int(d), int(bits), int(variant), ctypes.c_uint64(seed & (2**64 - 1)),
                                   int(n_sets), int(set_rows), int(device), ctypes.byref(h)), "iq_make_params_sets")
    return Params(h.value, d, bits, variant, seed, device)


def iq_make_params_qjl_sets(d: int, bits: int, variant, seed: int, n_sets: int, set_rows: int,
                            device: int = 0) -> Params:
    """iq_make_params_sets plus the stage-2 sketch (one S for every set)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant.lower()]
    h = ctypes.c_void_p()
    _check(lib.iq_make_params_qjl_sets(int(d), int(bits), int(variant), ctypes.c_uint64(seed & (2**64 - 1)),
                                       int(n_sets), int(set_rows), int(device), ctypes.byref(h)),
           "iq_make_params_qjl_sets")
    return Params(h.value, d, bits, variant, seed, device)


def iq_export_params_set(p: Params, s: int) -> np.ndarray:
    rot = np.zeros(iq_rotation_param_count(p.d, p.variant), dtype=np.float64)
    _check(lib.iq_export_params_set(p.handle, int(s), rot.ctypes.data, rot.size), "iq_export_params_set")
    return rot


def iq_make_params_explicit(d: int, bits: int, variant, rot, device: int = 0) -> Params:
    """Parameters from explicit rotations (iq_export_params layout, fp64)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant.lower()]
    r = np.ascontiguousarray(rot, dtype=np.float64)
    h = ctypes.c_void_p()
    _check(lib.iq_make_params_explicit(int(d), int(bits), int(variant), r.ctypes.data, r.size, int(device),
                                       ctypes.byref(h)), "iq_make_params_explicit")
    return Params(h.value, d, bits, variant, 0, device)


def iq_rot_grad_from_operator_grad(p: Params, G) -> np.ndarray:
    """Host chain rule: dL/dM (array of block_matrix_count doubles) -> dL/d(rot)."""
    g = np.ascontiguousarray(G, dtype=np.float64)
    out = np.zeros(iq_rotation_param_count(p.d, p.variant), dtype=np.float64)
    _check(lib.iq_rot_grad_from_operator_grad(p.handle, g.ctypes.data, g.size, out.ctypes.data, out.size),
           "iq_rot_grad_from_operator_grad")
    return out


def iq_export_params(p: Params) -> dict:
    """Canonical params as NumPy arrays: rot (fp64), centroids, thresholds (fp32)."""
    L = 1 << p.bits
    rot = np.zeros(iq_rotation_param_count(p.d, p.variant), dtype=np.float64)
    cen = np.zeros(L, dtype=np.float32)
    thr = np.zeros(L - 1, dtype=np.float32)
    _check(lib.iq_export_params(p.handle, rot.ctypes.data, rot.size, cen.ctypes.data, cen.size,
                                thr.ctypes.data if thr.size else None, thr.size), "iq_export_params")
    return {"rot": rot, "centroids": cen, "thresholds": thr}


def iq_export_block_matrices(p: Params) -> np.ndarray:
    n = (4 * ((p.d + 1) // 2)) if p.variant == PLANAR2D else (16 * ((p.d + 3) // 4))
    m = np.zeros(n, dtype=np.float32)
    _check(lib.iq_export_block_matrices(p.handle, m.ctypes.data, m.size), "iq_export_block_matrices")
    return m


# ------------------------------------------------------------ torch marshalling
def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float16:
        return F16
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(f"unsupported dtype {t.dtype} (float32, float16 or bfloat16)")


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _rows(x, d):
    if x.dim() != 2 or x.shape[1] != d or not x.is_contiguous():
        raise ValueError(f"expected a contiguous [n, {d}] tensor, got {tuple(x.shape)}")
    return x.shape[0]


def _want(t, name, shape, dtype, device):
    """Validate a caller-supplied tensor before its pointer crosses the ABI
    (the C side sees only pointers and n): exact shape, dtype, device and
    contiguity, else ValueError."""
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: expected dtype {dtype}, got {t.dtype}")
    if t.device != device:
        raise ValueError(f"{name}: expected device {device}, got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return t


def _on_params_device(t, p: "Params", name):
    torch = _torch()
    if t.device.type != "cuda" or (p.device >= 0 and t.device.index != p.device):
        raise ValueError(f"{name}: expected a tensor on cuda:{p.device}, got {t.device}")


def iq_quantize(p: Params, x, codes=None, norms=None, stream=None):
    """x [n,d] (cuda, f32/f16) -> (codes [n, d*b/8] uint8, norms [n] f32)."""
    torch = _torch()
    n = _rows(x, p.d)
    _on_params_device(x, p, "x")
    if codes is None:
        codes = torch.empty((n, p.code_bytes), dtype=torch.uint8, device=x.device)
    if norms is None:
        norms = torch.empty((n,), dtype=torch.float32, device=x.device)
    _want(codes, "codes", (n, p.code_bytes), torch.uint8, x.device)
    _want(norms, "norms", (n,), torch.float32, x.device)
    _check(lib.iq_quantize(p.handle, _dtype_code(x), n, _ptr(x), _ptr(codes), _ptr(norms),
                           _stream_ptr(stream)), "iq_quantize")
    return codes, norms


def iq_dequantize(p: Params, codes, norms, dtype=None, y=None, stream=None):
    """codes [n, d*b/8] uint8 + norms [n] -> y [n, d] of ``dtype``."""
    torch = _torch()
    if codes.dim() != 2:
        raise ValueError(f"codes: expected [n, {p.code_bytes}], got {tuple(codes.shape)}")
    n = codes.shape[0]
    _on_params_device(codes, p, "codes")
    _want(codes, "codes", (n, p.code_bytes), torch.uint8, codes.device)
    _want(norms, "norms", (n,), torch.float32, codes.device)
    if y is None:
        y = torch.empty((n, p.d), dtype=dtype or torch.float16, device=codes.device)
    _want(y, "y", (n, p.d), dtype or y.dtype, codes.device)
    _check(lib.iq_dequantize(p.handle, _dtype_code(y), n, _ptr(codes), _ptr(norms), _ptr(y),
                             _stream_ptr(stream)), "iq_dequantize")
    return y


def iq_roundtrip(p: Params, x, y=None, codes=None, norms=None, emit_codes: bool = False, stream=None):
    """Fused quantize->dequantize.  Returns y, or (y, codes, norms) if
    ``emit_codes`` (or codes/norms were passed)."""
    torch = _torch()
    n = _rows(x, p.d)
    _on_params_device(x, p, "x")
    if y is None:
        y = torch.empty_like(x)
    _want(y, "y", (n, p.d), x.dtype, x.device)
    if emit_codes and codes is None:
        codes = torch.empty((n, p.code_bytes), dtype=torch.uint8, device=x.device)
    if emit_codes and norms is None:
        norms = torch.empty((n,), dtype=torch.float32, device=x.device)
    if (codes is None) != (norms is None):
        raise ValueError("codes and norms must be given together")
    if codes is not None:
        _want(codes, "codes", (n, p.code_bytes), torch.uint8, x.device)
        _want(norms, "norms", (n,), torch.float32, x.device)
    _check(lib.iq_roundtrip(p.handle, _dtype_code(x), n, _ptr(x), _ptr(y), _ptr(codes), _ptr(norms),
                            _stream_ptr(stream)), "iq_roundtrip")
    return (y, codes, norms) if codes is not None else y


def iq_append_kv(p: Params, x, codes, norms, positions=None, position: int = 0, stream=None):
    """Quantize-on-append: slot r's new row x[r] ([n_rows, d]) into the cache
    codes [n_rows, cap, code bytes] / norms [n_rows, cap] at token
    positions[r] (device int64 [n_rows]) or ``position``; slot r uses
    parameter set r % n_sets.  Returns (codes, norms)."""
    torch = _torch()
    n = _rows(x, p.d)
    _on_params_device(x, p, "x")
    if codes.dim() != 3 or norms.dim() != 2:
        raise ValueError("codes must be [n_rows, cap, code bytes] and norms [n_rows, cap]")
    cap = codes.shape[1]
    _want(codes, "codes", (n, cap, p.code_bytes), torch.uint8, x.device)
    _want(norms, "norms", (n, cap), torch.float32, x.device)
    if positions is not None:
        _want(positions, "positions", (n,), torch.int64, x.device)
    _check(lib.iq_append_kv(p.handle, _dtype_code(x), n, _ptr(x), _ptr(codes), _ptr(norms), cap, _ptr(positions),
                            int(position), _stream_ptr(stream)), "iq_append_kv")
    return codes, norms


def iq_quantize_qjl(p: Params, x, codes=None, norms=None, qjl=None, rnorms=None, stream=None):
    """x [n,d] -> (codes, norms, qjl [n, d/8] uint8, rnorms [n] f32): stage 1 +
    stage-2 residual sketch in one kernel."""
    torch = _torch()
    n = _rows(x, p.d)
    _on_params_device(x, p, "x")
    if codes is None:
        codes = torch.empty((n, p.code_bytes), dtype=torch.uint8, device=x.device)
    if norms is None:
        norms = torch.empty((n,), dtype=torch.float32, device=x.device)
    if qjl is None:
        qjl = torch.empty((n, iq_qjl_bytes_per_vector(p.d)), dtype=torch.uint8, device=x.device)
    if rnorms is None:
        rnorms = torch.empty((n,), dtype=torch.float32, device=x.device)
    _want(codes, "codes", (n, p.code_bytes), torch.uint8, x.device)
    _want(norms, "norms", (n,), torch.float32, x.device)
    _want(qjl, "qjl", (n, iq_qjl_bytes_per_vector(p.d)), torch.uint8, x.device)
    _want(rnorms, "rnorms", (n,), torch.float32, x.device)
    _check(lib.iq_quantize_qjl(p.handle, _dtype_code(x), n, _ptr(x), _ptr(codes), _ptr(norms), _ptr(qjl),
                               _ptr(rnorms), _stream_ptr(stream)), "iq_quantize_qjl")
    return codes, norms, qjl, rnorms


def iq_attention_scores(p: Params, codes, norms, q, qjl=None, rnorms=None, scores=None, stream=None):
    """Attention logits from the packed cache.  codes [H, N, code bytes] (or
    [N, bytes] for H = 1), norms [H, N]; q [H, n_q, d] (f32/f16, the handle's
    I/O dtype of the call); optional stage-2 qjl [H, N, d/8] + rnorms [H, N].
    Returns scores [H, n_q, N] float32."""
    torch = _torch()
    if codes.dim() == 2:
        codes, norms = codes.unsqueeze(0), norms.unsqueeze(0)
        if qjl is not None:
            qjl, rnorms = qjl.unsqueeze(0), rnorms.unsqueeze(0)
    if q.dim() == 2:
        q = q.unsqueeze(0)
    if codes.dim() != 3 or q.dim() != 3:
        raise ValueError("codes must be [H, N, code bytes] and q [H, n_q, d]")
    H, N = codes.shape[0], codes.shape[1]
    n_q = q.shape[1]
    dev = codes.device
    _on_params_device(codes, p, "codes")
    _want(codes, "codes", (H, N, p.code_bytes), torch.uint8, dev)
    _want(norms, "norms", (H, N), torch.float32, dev)
    if q.dtype not in (torch.float32, torch.float16, torch.bfloat16):
        raise ValueError(f"q: unsupported dtype {q.dtype}")
    _want(q, "q", (H, n_q, p.d), q.dtype, dev)
    if (qjl is None) != (rnorms is None):
        raise ValueError("qjl and rnorms must be given together")
    if qjl is not None:
        _want(qjl, "qjl", (H, N, iq_qjl_bytes_per_vector(p.d)), torch.uint8, dev)
        _want(rnorms, "rnorms", (H, N), torch.float32, dev)
    if scores is None:
        scores = torch.empty((H, n_q, N), dtype=torch.float32, device=dev)
    _want(scores, "scores", (H, n_q, N), torch.float32, dev)
    _check(lib.iq_attention_scores(p.handle, _dtype_code(q), H, N, _ptr(codes), _ptr(norms), _ptr(qjl),
                                   _ptr(rnorms), n_q, _ptr(q), _ptr(scores), _stream_ptr(stream)),
           "iq_attention_scores")
    return scores


def iq_distortion_grad(p: Params, x, grad=None, loss=None, stream=None):
    """dL/dM per block operator (device fp64, accumulated) and the distortion
    L (device fp64 scalar, accumulated) over the rows of x."""
    torch = _torch()
    n = _rows(x, p.d)
    nm = (4 * ((p.d + 1) // 2)) if p.variant == PLANAR2D else (16 * ((p.d + 3) // 4))
    _on_params_device(x, p, "x")
    if grad is None:
        grad = torch.zeros(nm, dtype=torch.float64, device=x.device)
    if loss is None:
        loss = torch.zeros(1, dtype=torch.float64, device=x.device)
    _want(grad, "grad", (nm,), torch.float64, x.device)
    _want(loss, "loss", (1,), torch.float64, x.device)
    _check(lib.iq_distortion_grad(p.handle, _dtype_code(x), n, _ptr(x), _ptr(grad), _ptr(loss),
                                  _stream_ptr(stream)), "iq_distortion_grad")
    return grad, loss


def iq_error_sums(p: Params, x, y, sums=None, stream=None):
    """Device fp64 [sum (x-y)^2, sum x^2] (accumulated into ``sums``)."""
    torch = _torch()
    n = _rows(x, p.d)
    _on_params_device(x, p, "x")
    _want(y, "y", (n, p.d), x.dtype, x.device)
    if sums is None:
        sums = torch.zeros(2, dtype=torch.float64, device=x.device)
    _want(sums, "sums", (2,), torch.float64, x.device)
    _check(lib.iq_error_sums(p.handle, _dtype_code(x), n, _ptr(x), _ptr(y), _ptr(sums),
                             _stream_ptr(stream)), "iq_error_sums")
    return sums


class HostPipeline:
    """iq_host_pipeline: host-buffer roundtrip streamed through the GPU."""

    def __init__(self, p: Params, dtype: int, chunk_vectors: int = 1 << 18):
        self.p = p
        self.dtype = dtype
        h = ctypes.c_void_p()
        _check(lib.iq_host_pipeline_create(p.handle, dtype, chunk_vectors, ctypes.byref(h)),
               "iq_host_pipeline_create")
        self._h = h

    def roundtrip(self, x_host, y_host, codes_host=None, norms_host=None):
        """x_host/y_host: CPU tensors (ideally pinned) [n, d]; synchronous."""
        torch = _torch()
        n = _rows(x_host, self.p.d)
        for name, t in (("x_host", x_host), ("y_host", y_host)):
            if t.device.type != "cpu":
                raise ValueError(f"{name}: expected a host tensor")
        _want(y_host, "y_host", (n, self.p.d), x_host.dtype, x_host.device)
        if codes_host is not None:
            _want(codes_host, "codes_host", (n, self.p.code_bytes), torch.uint8, x_host.device)
        if norms_host is not None:
            _want(norms_host, "norms_host", (n,), torch.float32, x_host.device)
        _check(lib.iq_host_roundtrip(self._h, n, _ptr(x_host), _ptr(y_host), _ptr(codes_host),
                                     _ptr(norms_host)), "iq_host_roundtrip")
        return y_host

    def close(self):
        if self._h is not None and self._h.value:
            lib.iq_host_pipeline_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
