"""Thin Python binding of the libfllf C ABI (include/fllf.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of
libfllf.so.  Functions carry the C names; tensors are torch CUDA tensors
(PyTorch is used for device memory and streams, nothing else).  There is no
CPU fallback: importing this module raises if libfllf.so is missing, and the
compute calls raise on CPU tensors or without a CUDA device.
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# FLLF_LIB selects another build of the same library (compile-time A/B of kernel variants)
LIB_PATH = os.environ.get("FLLF_LIB") or os.path.join(_PKG, "lib", "libfllf.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "fllf.h")

FLLF_OK = 0
FLLF_ERR_INVALID_ARGUMENT = 1
FLLF_ERR_TOO_MANY_LEVELS = 2
FLLF_ERR_OUT_OF_MEMORY = 3
FLLF_ERR_CUDA = 4
FLLF_ERR_NOT_BUILT = 5
FLLF_ERR_BAD_POINTER = 6
FLLF_SCALAR, FLLF_COEFFS, FLLF_MAPS = 0, 1, 2
FLLF_MAX_K = 32
FLLF_MAX_LEVELS = 16


class FllfError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{status_name(status)}: {message}")
        self.status = status


class fllf_plan_desc(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int), ("W", ctypes.c_int), ("levels", ctypes.c_int),
                ("K", ctypes.c_int), ("T", ctypes.c_double), ("sigma_r", ctypes.c_double),
                ("m", ctypes.c_double), ("batch", ctypes.c_int), ("k_begin", ctypes.c_int),
                ("k_end", ctypes.c_int), ("include_base", ctypes.c_int), ("device", ctypes.c_int),
                ("row_begin", ctypes.c_int), ("row_end", ctypes.c_int)]


class fllf_gain_desc(ctypes.Structure):
    _fields_ = [("radius", ctypes.c_int), ("m_lo", ctypes.c_double), ("m_hi", ctypes.c_double),
                ("v_ref", ctypes.c_double)]


class fllf_apply_args(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("a_k", ctypes.POINTER(ctypes.c_double)),
                ("d_sigma_r", ctypes.c_void_p), ("d_m", ctypes.c_void_p),
                ("map_pitch_bytes", ctypes.c_size_t)]


_P = ctypes.c_void_p
_SIGS = {
    "fllf_plan_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.POINTER(_P)]),
    "fllf_plan_create_ex": (ctypes.c_int, [ctypes.POINTER(fllf_plan_desc), ctypes.POINTER(_P)]),
    "fllf_destroy": (ctypes.c_int, [_P]),
    "fllf_build_fourier_pyramids": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "fllf_apply": (ctypes.c_int, [_P, ctypes.POINTER(fllf_apply_args), _P, ctypes.c_size_t, _P]),
    "fllf_apply_accumulate": (ctypes.c_int, [_P, ctypes.POINTER(fllf_apply_args), _P, ctypes.c_size_t, _P]),
    "fllf_apply_maps": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, ctypes.c_size_t, ctypes.c_size_t, _P,
                                       ctypes.c_size_t, ctypes.c_size_t, _P]),
    "fllf_ipc_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), _P]),
    "fllf_ipc_free": (ctypes.c_int, [_P]),
    "fllf_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p)]),
    "fllf_ipc_close": (ctypes.c_int, [_P]),
    "fllf_filter": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P, ctypes.c_size_t, _P]),
    "fllf_filter_host": (ctypes.c_int, [_P, _P, _P, _P]),
    "fllf_filter_host_frames": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P, ctypes.c_size_t, ctypes.c_int, _P]),
    "fllf_plan_set_l2_flush": (ctypes.c_int, [_P, _P, ctypes.c_size_t]),
    "fllf_coefficients": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]),
    "fllf_optimal_period": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           ctypes.POINTER(ctypes.c_double)]),
    "fllf_plan_level_dims": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int)]),
    "fllf_workspace_bytes": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    "fllf_read_pyramid": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P,
                                         ctypes.c_size_t, _P]),
    "fllf_plan_last_launch_count": (ctypes.c_int, [_P]),
    "fllf_plan_set_profiling": (ctypes.c_int, [_P, ctypes.c_int]),
    "fllf_plan_set_graphs": (ctypes.c_int, [_P, ctypes.c_int]),
    "fllf_plan_set_design": (ctypes.c_int, [_P, ctypes.c_int]),
    "fllf_plan_set_fused_levels": (ctypes.c_int, [_P, ctypes.c_int]),
    "fllf_plan_get_desc": (ctypes.c_int, [_P, ctypes.POINTER(fllf_plan_desc)]),
    "fllf_plan_kernel_times": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_float),
                                              ctypes.POINTER(ctypes.c_int)]),
    "fllf_rgb_to_yuv": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_size_t, _P]),
    "fllf_yuv_to_rgb": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_size_t, _P]),
    "fllf_gain_map": (ctypes.c_int, [_P, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(fllf_gain_desc), _P, ctypes.c_size_t, _P]),
    "fllf_enhance_rgb": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, ctypes.POINTER(fllf_gain_desc), _P]),
    "fllf_naive_llf": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.c_int, _P, ctypes.c_size_t, _P]),
    "fllf_build_level": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.c_int, _P]),
    "fllf_apply_level": (ctypes.c_int, [_P, ctypes.POINTER(fllf_apply_args), _P, ctypes.c_size_t, ctypes.c_int,
                                        _P]),
    "fllf_plan_band_plane": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P),
                                            ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_size_t)]),
    "fllf_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "fllf_last_error_message": (ctypes.c_char_p, []),
}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2206_04681_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def header_symbols() -> list[str]:
    """Every function the C header declares (used by the ABI test)."""
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"FLLF_API\s+[\w\s\*]*?\b(fllf_\w+)\s*\(", txt)))


def status_name(st: int) -> str:
    return lib.fllf_status_string(int(st)).decode()


def _check(st: int) -> None:
    if st != FLLF_OK:
        raise FllfError(st, lib.fllf_last_error_message().decode())


# ------------------------------------------------------------- marshalling
def _stream_handle(stream) -> int | None:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev_image(t, name: str):
    """(pointer, pitch_bytes) of a CUDA fp32 tensor [..., H, W] with unit column stride."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (libfllf has no CPU fallback)")
    if t.dtype != torch.float32 or t.stride(-1) != 1:
        raise TypeError(f"{name} must be float32 with unit column stride")
    if t.dim() >= 3 and t.shape[0] > 1 and t.stride(-3) != t.shape[-2] * t.stride(-2):
        raise TypeError(f"{name}: frames must be contiguous")
    return t.data_ptr(), t.stride(-2) * 4


# ------------------------------------------------------------- C-ABI names
def fllf_plan_create(H, W, levels, K, T, sigma_r, m) -> int:
    h = _P()
    _check(lib.fllf_plan_create(H, W, levels, K, float(T), float(sigma_r), float(m), ctypes.byref(h)))
    return h.value


def fllf_plan_create_ex(H, W, levels, K, T, sigma_r=30.0, m=1.0, batch=1, k_begin=0, k_end=0,
                        include_base=True, device=-1, row_begin=0, row_end=0) -> int:
    d = fllf_plan_desc(H, W, levels, K, float(T), float(sigma_r), float(m), batch, k_begin, k_end,
                       1 if include_base else 0, device, row_begin, row_end)
    h = _P()
    _check(lib.fllf_plan_create_ex(ctypes.byref(d), ctypes.byref(h)))
    return h.value


def fllf_destroy(plan) -> None:
    _check(lib.fllf_destroy(plan))


def fllf_build_fourier_pyramids(plan, img, stream=None) -> None:
    ptr, pitch = _dev_image(img, "img")
    _check(lib.fllf_build_fourier_pyramids(plan, ptr, pitch, _stream_handle(stream)))


def fllf_apply(plan, out, mode=FLLF_SCALAR, a_k=None, sigma_map=None, m_map=None, stream=None) -> None:
    optr, opitch = _dev_image(out, "out")
    args = fllf_apply_args()
    args.mode = mode
    keep = None
    if mode == FLLF_COEFFS:
        keep = np.ascontiguousarray(np.asarray(a_k, dtype=np.float64))
        args.a_k = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    elif mode == FLLF_MAPS:
        sp, spitch = _dev_image(sigma_map, "sigma_map")
        mp, mpitch = _dev_image(m_map, "m_map")
        if spitch != mpitch:
            raise ValueError("sigma and m maps must share a pitch")
        args.d_sigma_r, args.d_m, args.map_pitch_bytes = sp, mp, spitch
    _check(lib.fllf_apply(plan, ctypes.byref(args), optr, opitch, _stream_handle(stream)))
    del keep


def fllf_apply_maps(plan, outs, sigma_maps, m_maps, stream=None) -> None:
    """n MAPS applies (output j = fllf_apply(MAPS) with map pair j): sigma_maps,
    m_maps (n, H, W) float32 CUDA tensors with the same layout, outs (n, ..., H, W)
    with one plan output (batch x H x W) per pair, contiguous per pair."""
    import torch
    for t, nm in ((sigma_maps, "sigma_maps"), (m_maps, "m_maps"), (outs, "outs")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or t.stride(-1) != 1:
            raise TypeError(f"{nm} must be a float32 CUDA tensor with unit column stride")
    if sigma_maps.dim() != 3 or m_maps.shape != sigma_maps.shape or sigma_maps.stride() != m_maps.stride():
        raise ValueError("sigma_maps and m_maps: (n, H, W) tensors of one layout")
    n = sigma_maps.shape[0]
    if outs.shape[0] != n:
        raise ValueError("outs: one output per map pair")
    if sigma_maps.stride(1) * sigma_maps.shape[1] > sigma_maps.stride(0) or outs[0].numel() > outs.stride(0) or \
            not outs[0].is_contiguous():
        raise ValueError("maps / outputs overlap, or an output is not contiguous")
    _check(lib.fllf_apply_maps(plan, n, sigma_maps.data_ptr(), m_maps.data_ptr(), sigma_maps.stride(1) * 4,
                               sigma_maps.stride(0) * 4, outs.data_ptr(), outs.stride(-2) * 4, outs.stride(0) * 4,
                               _stream_handle(stream)))


def fllf_apply_accumulate(plan, out, mode=FLLF_SCALAR, a_k=None, stream=None) -> None:
    """As fllf_apply, but the level-0 result is atomically ADDED to `out` (which
    may alias another process's buffer through fllf_ipc_open)."""
    optr, opitch = _dev_image(out, "out")
    args, keep = _apply_args(mode, a_k)
    _check(lib.fllf_apply_accumulate(plan, ctypes.byref(args), optr, opitch, _stream_handle(stream)))
    del keep


IPC_HANDLE_BYTES = 64


def ipc_alloc(nbytes: int):
    """(device pointer, IPC handle bytes) of a fresh allocation on the current device."""
    ptr = ctypes.c_void_p()
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(lib.fllf_ipc_alloc(int(nbytes), ctypes.byref(ptr), h))
    return ptr.value, h.raw


def ipc_free(ptr: int) -> None:
    _check(lib.fllf_ipc_free(ptr))


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation (its ipc_alloc handle) into this one."""
    ptr = ctypes.c_void_p()
    _check(lib.fllf_ipc_open(ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES), ctypes.byref(ptr)))
    return ptr.value


def ipc_close(ptr: int) -> None:
    _check(lib.fllf_ipc_close(ptr))


def _apply_args(mode, a_k):
    args = fllf_apply_args()
    args.mode = mode
    keep = None
    if mode == FLLF_COEFFS:
        keep = np.ascontiguousarray(np.asarray(a_k, dtype=np.float64))
        args.a_k = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    elif mode != FLLF_SCALAR:
        raise ValueError("per-level apply supports SCALAR and COEFFS")
    return args, keep


def fllf_build_level(plan, img_ptr, pitch_bytes, level, stream=None) -> None:
    """Build step level -> level+1.  img_ptr: device address of the band's first
    row (global row row_begin) of the image (int), pitch in bytes."""
    _check(lib.fllf_build_level(plan, int(img_ptr), int(pitch_bytes), int(level), _stream_handle(stream)))


def fllf_apply_level(plan, out_ptr, pitch_bytes, level, mode=FLLF_SCALAR, a_k=None, stream=None) -> None:
    args, keep = _apply_args(mode, a_k)
    _check(lib.fllf_apply_level(plan, ctypes.byref(args), int(out_ptr), int(pitch_bytes), int(level),
                                _stream_handle(stream)))
    del keep


BAND_G, BAND_Z, BAND_D = 0, 1, 2


def fllf_plan_band_plane(plan, level, kind):
    """dict(ptr, pitch_bytes, first_row, rows, planes, plane_stride_bytes) of the stored rows."""
    ptr, pitch, first, rows, planes, pstride = (_P(), ctypes.c_size_t(), ctypes.c_int(), ctypes.c_int(),
                                                ctypes.c_int(), ctypes.c_size_t())
    _check(lib.fllf_plan_band_plane(plan, int(level), int(kind), ctypes.byref(ptr), ctypes.byref(pitch),
                                    ctypes.byref(first), ctypes.byref(rows), ctypes.byref(planes),
                                    ctypes.byref(pstride)))
    return dict(ptr=ptr.value, pitch_bytes=pitch.value, first_row=first.value, rows=rows.value,
                planes=planes.value, plane_stride_bytes=pstride.value)


# ---- zero-copy torch views of library-owned device memory (DLPack)
class _DLDevice(ctypes.Structure):
    _fields_ = [("device_type", ctypes.c_int), ("device_id", ctypes.c_int)]


class _DLDataType(ctypes.Structure):
    _fields_ = [("code", ctypes.c_uint8), ("bits", ctypes.c_uint8), ("lanes", ctypes.c_uint16)]


class _DLTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("device", _DLDevice), ("ndim", ctypes.c_int),
                ("dtype", _DLDataType), ("shape", ctypes.POINTER(ctypes.c_int64)),
                ("strides", ctypes.POINTER(ctypes.c_int64)), ("byte_offset", ctypes.c_uint64)]


class _DLManagedTensor(ctypes.Structure):
    pass


_DLManagedTensor._fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", ctypes.c_void_p),
                             ("deleter", ctypes.CFUNCTYPE(None, ctypes.POINTER(_DLManagedTensor)))]
_keepalive = {}


@ctypes.CFUNCTYPE(None, ctypes.POINTER(_DLManagedTensor))
def _dl_deleter(p):
    _keepalive.pop(ctypes.addressof(p.contents), None)


def device_view(ptr: int, shape, strides, device: int):
    """float32 torch tensor aliasing `ptr` on CUDA `device` (element strides).
    The memory stays owned by the library plan; keep the plan alive."""
    import torch
    n = len(shape)
    sh = (ctypes.c_int64 * n)(*shape)
    st = (ctypes.c_int64 * n)(*strides)
    mt = _DLManagedTensor()
    mt.dl_tensor = _DLTensor(ctypes.c_void_p(ptr), _DLDevice(2, device), n, _DLDataType(2, 32, 1), sh, st, 0)
    mt.manager_ctx = None
    mt.deleter = _dl_deleter
    _keepalive[ctypes.addressof(mt)] = (mt, sh, st)
    pyapi = ctypes.pythonapi
    pyapi.PyCapsule_New.restype = ctypes.py_object
    pyapi.PyCapsule_New.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
    cap = pyapi.PyCapsule_New(ctypes.addressof(mt), b"dltensor", None)
    return torch.utils.dlpack.from_dlpack(cap)


def band_rows_view(plan, level, kind, device: int):
    """torch view (planes, rows, row floats) of the stored rows of one level and its first global row."""
    d = fllf_plan_band_plane(plan, level, kind)
    row_floats = d["pitch_bytes"] // 4
    v = device_view(d["ptr"], (d["planes"], d["rows"], row_floats),
                    (d["plane_stride_bytes"] // 4, row_floats, 1), device)
    return v, d["first_row"]


def fllf_filter(plan, img, out, stream=None) -> None:
    iptr, ipitch = _dev_image(img, "img")
    optr, opitch = _dev_image(out, "out")
    _check(lib.fllf_filter(plan, iptr, ipitch, optr, opitch, _stream_handle(stream)))


def fllf_filter_host(plan, h_img, h_out, stream=None) -> None:
    """h_img / h_out: contiguous float32 CPU tensors (pin them for async copies)."""
    import torch
    d = fllf_plan_get_desc(plan)
    for t, n in ((h_img, "h_img"), (h_out, "h_out")):
        if t.is_cuda or not t.is_contiguous():
            raise TypeError(f"{n} must be a contiguous host tensor")
        if t.dtype != torch.float32 or t.numel() < d["batch"] * d["H"] * d["W"]:
            raise ValueError(f"{n} must be float32 with batch*H*W elements")
    _check(lib.fllf_filter_host(plan, h_img.data_ptr(), h_out.data_ptr(), _stream_handle(stream)))


def fllf_filter_host_frames(plan, h_in, in_stride_bytes, h_out, out_stride_bytes, nframes, stream=None) -> None:
    """Streaming host -> device -> host over `nframes` batches (C: fllf_filter_host_frames).
    h_in / h_out: contiguous float32 CPU tensors (pinned for overlap) holding the
    batches at the given byte strides (0 = one buffer reused for every batch)."""
    for t, n in ((h_in, "h_in"), (h_out, "h_out")):
        if t.is_cuda or not t.is_contiguous():
            raise TypeError(f"{n} must be a contiguous host tensor")
    import torch
    d = fllf_plan_get_desc(plan)
    batch_bytes = d["batch"] * d["H"] * d["W"] * 4
    for t, st, n in ((h_in, in_stride_bytes, "h_in"), (h_out, out_stride_bytes, "h_out")):
        if t.dtype != torch.float32:
            raise TypeError(f"{n} must be float32")
        if nframes > 0 and (nframes - 1) * st + batch_bytes > t.numel() * t.element_size():
            raise ValueError(f"{n} too small for {nframes} batches of {batch_bytes} bytes at stride {st}")
    _check(lib.fllf_filter_host_frames(plan, h_in.data_ptr(), int(in_stride_bytes), h_out.data_ptr(),
                                       int(out_stride_bytes), int(nframes), _stream_handle(stream)))


def fllf_plan_set_l2_flush(plan, buf=None) -> None:
    """Bench tooling: a CUDA tensor written before each batch of fllf_filter_host_frames (None: off)."""
    if buf is None:
        _check(lib.fllf_plan_set_l2_flush(plan, None, 0))
    else:
        _check(lib.fllf_plan_set_l2_flush(plan, buf.data_ptr(), buf.numel() * buf.element_size()))


def fllf_coefficients(K, T, sigma_r, m):
    om = (ctypes.c_double * K)()
    a = (ctypes.c_double * K)()
    _check(lib.fllf_coefficients(K, float(T), float(sigma_r), float(m), om, a))
    return np.array(om[:]), np.array(a[:])


def fllf_optimal_period(K, sigma_r, R=256.0) -> float:
    t = ctypes.c_double()
    _check(lib.fllf_optimal_period(K, float(sigma_r), float(R), ctypes.byref(t)))
    return t.value


def fllf_plan_level_dims(plan, level):
    h, w = ctypes.c_int(), ctypes.c_int()
    _check(lib.fllf_plan_level_dims(plan, level, ctypes.byref(h), ctypes.byref(w)))
    return h.value, w.value


def fllf_workspace_bytes(plan) -> int:
    b = ctypes.c_size_t()
    _check(lib.fllf_workspace_bytes(plan, ctypes.byref(b)))
    return b.value


def fllf_read_pyramid(plan, frame, level, channel, dst, stream=None) -> None:
    ptr, pitch = _dev_image(dst, "dst")
    _check(lib.fllf_read_pyramid(plan, frame, level, channel, ptr, pitch, _stream_handle(stream)))


def fllf_plan_last_launch_count(plan) -> int:
    return int(lib.fllf_plan_last_launch_count(plan))


def _planes3(t, name: str):
    """(pointer, pitch_bytes, H, W) of a CUDA fp32 (3, H, W) tensor with dense planes."""
    ptr, pitch = _dev_image(t, name)
    if t.dim() != 3 or t.shape[0] != 3 or t.stride(0) != t.shape[1] * t.stride(1):
        raise TypeError(f"{name} must be (3, H, W) with contiguous planes")
    return ptr, pitch, int(t.shape[1]), int(t.shape[2])


def fllf_rgb_to_yuv(rgb, yuv, stream=None) -> None:
    ip, pitch, H, W = _planes3(rgb, "rgb")
    op, opitch, _, _ = _planes3(yuv, "yuv")
    if opitch != pitch:
        raise ValueError("rgb and yuv must share a pitch")
    _check(lib.fllf_rgb_to_yuv(ip, op, H, W, pitch, _stream_handle(stream)))


def fllf_yuv_to_rgb(yuv, rgb, stream=None) -> None:
    ip, pitch, H, W = _planes3(yuv, "yuv")
    op, opitch, _, _ = _planes3(rgb, "rgb")
    if opitch != pitch:
        raise ValueError("rgb and yuv must share a pitch")
    _check(lib.fllf_yuv_to_rgb(ip, op, H, W, pitch, _stream_handle(stream)))


def fllf_gain_map(y, m, radius, m_lo, m_hi, v_ref, stream=None) -> None:
    yp, ypitch = _dev_image(y, "y")
    mp, mpitch = _dev_image(m, "m")
    g = fllf_gain_desc(int(radius), float(m_lo), float(m_hi), float(v_ref))
    _check(lib.fllf_gain_map(yp, ypitch, int(y.shape[-2]), int(y.shape[-1]), ctypes.byref(g), mp, mpitch,
                             _stream_handle(stream)))


def fllf_enhance_rgb(plan, rgb, out, radius, m_lo, m_hi, v_ref, stream=None) -> None:
    ip, pitch, _, _ = _planes3(rgb, "rgb")
    op, opitch, _, _ = _planes3(out, "out")
    if opitch != pitch:
        raise ValueError("rgb and out must share a pitch")
    g = fllf_gain_desc(int(radius), float(m_lo), float(m_hi), float(v_ref))
    _check(lib.fllf_enhance_rgb(plan, ip, op, pitch, ctypes.byref(g), _stream_handle(stream)))


FLLF_NAIVE_MAX_LEVELS = 5
REMAP_EXACT, REMAP_SERIES = 0, 1


def fllf_naive_llf(plan, img, out, remap_mode=REMAP_EXACT, stream=None) -> None:
    """Naive LLF ground truth (NEXT-2) of a CUDA fp32 (H, W) image on a batch-1 plan."""
    ip, ipitch = _dev_image(img, "img")
    op, opitch = _dev_image(out, "out")
    _check(lib.fllf_naive_llf(plan, ip, ipitch, int(remap_mode), op, opitch, _stream_handle(stream)))


KERNEL_KINDS = {0: "build0", 1: "build", 2: "mapbuild", 3: "apply", 4: "apply0", 5: "fuse", 6: "collapse"}


def fllf_plan_set_profiling(plan, enable: bool) -> None:
    _check(lib.fllf_plan_set_profiling(plan, 1 if enable else 0))


def fllf_plan_set_graphs(plan, enable: bool) -> None:
    _check(lib.fllf_plan_set_graphs(plan, 1 if enable else 0))


FLLF_DESIGN_AUTO, FLLF_DESIGN_AB, FLLF_DESIGN_F = 0, 1, 2


def fllf_plan_set_design(plan, design: int) -> None:
    """Design of fllf_filter: FLLF_DESIGN_AUTO (default), FLLF_DESIGN_AB or FLLF_DESIGN_F."""
    _check(lib.fllf_plan_set_design(plan, int(design)))


def fllf_plan_set_fused_levels(plan, n: int) -> None:
    """Design F on levels 1..n, AB above (0: FLLF_DESIGN_AUTO)."""
    _check(lib.fllf_plan_set_fused_levels(plan, int(n)))


def fllf_plan_get_desc(plan) -> dict:
    """The plan's effective description (fllf_plan_desc fields)."""
    d = fllf_plan_desc()
    _check(lib.fllf_plan_get_desc(plan, ctypes.byref(d)))
    return {name: getattr(d, name) for name, _ in fllf_plan_desc._fields_}


def fllf_plan_kernel_times(plan, capacity: int = 64):
    """[(kind name, level, milliseconds)] for the launches of the last build(+apply)."""
    kind = (ctypes.c_int * capacity)()
    level = (ctypes.c_int * capacity)()
    ms = (ctypes.c_float * capacity)()
    n = ctypes.c_int()
    _check(lib.fllf_plan_kernel_times(plan, capacity, kind, level, ms, ctypes.byref(n)))
    return [(KERNEL_KINDS[kind[i]], level[i], float(ms[i])) for i in range(n.value)]


# ------------------------------------------------------------- convenience
@dataclass
class Plan:
    """RAII wrapper around an fllf_plan (same arguments as fllf_plan_create_ex)."""
    H: int
    W: int
    levels: int
    K: int
    T: float = 510.0
    sigma_r: float = 30.0
    m: float = 1.0
    batch: int = 1
    k_begin: int = 0
    k_end: int = 0
    include_base: bool = True
    device: int = -1
    row_begin: int = 0
    row_end: int = 0

    design: int = FLLF_DESIGN_AUTO

    def __post_init__(self):
        self.handle = fllf_plan_create_ex(self.H, self.W, self.levels, self.K, self.T, self.sigma_r,
                                          self.m, self.batch, self.k_begin, self.k_end,
                                          self.include_base, self.device, self.row_begin, self.row_end)
        self._dev = fllf_plan_get_desc(self.handle)["device"]
        if self.design != FLLF_DESIGN_AUTO:
            fllf_plan_set_design(self.handle, self.design)

    def _check_frames(self, t, name: str) -> None:
        """A full-frame plan's image / output: (H, W) or (batch, H, W) on the plan's device."""
        if self.row_begin or self.row_end:
            return  # band plans take the band's rows (see fllf_plan_desc)
        if not hasattr(t, "shape") or tuple(t.shape[-2:]) != (self.H, self.W):
            raise ValueError(f"{name} must end in ({self.H}, {self.W}), got {tuple(getattr(t, 'shape', ()))}")
        frames = 1
        for n in t.shape[:-2]:
            frames *= int(n)
        if frames != self.batch:
            raise ValueError(f"{name} holds {frames} frames, the plan's batch is {self.batch}")
        if getattr(t, "is_cuda", False) and t.device.index != self._dev:
            raise ValueError(f"{name} is on cuda:{t.device.index}, the plan on cuda:{self._dev}")

    def build(self, img, stream=None):
        self._check_frames(img, "img")
        fllf_build_fourier_pyramids(self.handle, img, stream)

    def apply(self, out, **kw):
        self._check_frames(out, "out")
        fllf_apply(self.handle, out, **kw)

    def apply_maps(self, outs, sigma_maps, m_maps, stream=None):
        """outs[j] = apply(MAPS, sigma_maps[j], m_maps[j]) for every pair j."""
        for j in range(outs.shape[0]):
            self._check_frames(outs[j], "outs[j]")
        fllf_apply_maps(self.handle, outs, sigma_maps, m_maps, stream)

    def filter(self, img, out, stream=None):
        self._check_frames(img, "img")
        self._check_frames(out, "out")
        fllf_filter(self.handle, img, out, stream)

    def set_design(self, design: int) -> None:
        fllf_plan_set_design(self.handle, design)
        self.design = design

    def level_dims(self, level):
        return fllf_plan_level_dims(self.handle, level)

    def read_pyramid(self, frame, level, channel, dst, stream=None):
        fllf_read_pyramid(self.handle, frame, level, channel, dst, stream)

    @property
    def launches(self) -> int:
        return fllf_plan_last_launch_count(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            fllf_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fourier_llf(img, levels, K, T=510.0, sigma_r=30.0, m=1.0, out=None):
    """One-shot Fourier LLF of a CUDA fp32 image [H, W] or batch [B, H, W]."""
    import torch
    B = img.shape[0] if img.dim() == 3 else 1
    H, W = img.shape[-2:]
    if out is None:
        out = torch.empty_like(img)
    with Plan(H, W, levels, K, T, sigma_r, m, batch=B) as p:
        p.filter(img, out)
        torch.cuda.current_stream().synchronize()
    return out
