"""ctypes binding of libb64gpu.so: same names as include/b64gpu.h.

Argument marshalling only (tensor -> pointer, stream -> handle, status ->
exception).  Nothing here computes base64.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libb64gpu.so")
# Experiments only (tools/sweep.py): load a variant build of the same library.
if os.environ.get("B64GPU_LIB"):
    _LIB_PATH = os.environ["B64GPU_LIB"]

B64_OK = 0
B64_ERR_INVALID_CHAR = 1
B64_ERR_LENGTH = 2
B64_ERR_NONCANONICAL = 3
B64_FLAG_URL = 1
B64_FLAG_NOPAD = 2
B64_FLAG_STRICT = 4
B64_ERR_ARG = -1
B64_ERR_CUDA = -2
B64_ERR_WORKSPACE = -3

# Every symbol include/b64gpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "b64_encoded_len", "b64_decoded_max_len", "b64_encode", "b64_decode",
    "b64_decode_async", "b64_decode_shard_async", "b64_batch_workspace_bytes",
    "b64_encode_batch", "b64_decode_batch", "b64_encode_host", "b64_decode_host",
    "b64_shard", "b64_batch_shard", "b64_status_str", "b64_build_info",
    "b64_encoded_len_ex", "b64_decoded_max_len_ex", "b64_encode_ex", "b64_decode_ex",
    "b64_decode_ex_async", "b64_encode_batch_ex", "b64_decode_batch_ex",
    "b64_despace_workspace_bytes", "b64_despace",
    "b64_decode_ws_workspace_bytes", "b64_decode_ws", "b64_decode_ws_async",
    "b64_encoded_len_wrapped", "b64_encode_wrapped",
    "b64_decode_shard_ex_async", "b64_shard_key", "b64_combine_shards", "b64_combine_shards_async",
    "b64_encode_host_ex", "b64_decode_host_ex", "b64_decode_scratch_async",
)
B64_DECODE_SCRATCH_BYTES = 16
INT64_MAX = (1 << 63) - 1

_lib = None


class B64Error(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {b64_status_str(code)} ({code})")


class _Result(ctypes.Structure):
    _fields_ = [("out_len", ctypes.c_int64), ("err_pos", ctypes.c_int64),
                ("status", ctypes.c_int32), ("pad_count", ctypes.c_int32)]


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libb64gpu.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    p64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "b64_encoded_len": (i64, [i64]),
        "b64_decoded_max_len": (i64, [i64]),
        "b64_encode": (i64, [vp, i64, vp, vp]),
        "b64_decode": (i32, [vp, i64, vp, p64, p64, vp]),
        "b64_decode_async": (i32, [vp, i64, vp, vp, vp]),
        "b64_decode_shard_async": (i32, [vp, i64, i32, vp, vp, vp]),
        "b64_batch_workspace_bytes": (sz, [i64, i64, i32]),
        "b64_encode_batch": (i32, [vp, vp, i64, i64, vp, vp, vp, sz, vp]),
        "b64_decode_batch": (i32, [vp, vp, i64, i64, vp, vp, vp, vp, vp, vp, sz, vp]),
        "b64_encode_host": (i64, [vp, i64, vp, vp, vp, vp]),
        "b64_decode_host": (i32, [vp, i64, vp, p64, p64, vp, vp, vp]),
        "b64_shard": (i32, [i64, i32, i32, i32, p64, p64]),
        "b64_batch_shard": (i32, [vp, i64, i32, i32, p64, p64]),
        "b64_status_str": (ctypes.c_char_p, [i32]),
        "b64_build_info": (ctypes.c_char_p, []),
        "b64_encoded_len_ex": (i64, [i64, i32]),
        "b64_decoded_max_len_ex": (i64, [i64, i32]),
        "b64_encode_ex": (i64, [vp, i64, vp, i32, vp]),
        "b64_decode_ex": (i32, [vp, i64, vp, i32, p64, p64, vp]),
        "b64_decode_ex_async": (i32, [vp, i64, vp, i32, vp, vp]),
        "b64_encode_batch_ex": (i32, [vp, vp, i64, i64, vp, vp, i32, vp, sz, vp]),
        "b64_decode_batch_ex": (i32, [vp, vp, i64, i64, vp, vp, vp, vp, vp, i32, vp, sz, vp]),
        "b64_despace_workspace_bytes": (sz, [i64]),
        "b64_despace": (i32, [vp, i64, vp, vp, vp, sz, vp]),
        "b64_decode_ws_workspace_bytes": (sz, [i64]),
        "b64_encoded_len_wrapped": (i64, [i64, i32, i32, i32]),
        "b64_encode_wrapped": (i64, [vp, i64, vp, i32, i32, i32, vp]),
        "b64_decode_ws_async": (i32, [vp, i64, vp, i32, vp, vp, sz, vp]),
        "b64_decode_ws": (i32, [vp, i64, vp, i32, ctypes.POINTER(i64), ctypes.POINTER(i64), vp, sz,
                                vp]),
        "b64_decode_shard_ex_async": (i32, [vp, i64, i64, i32, vp, i32, vp, vp, vp]),
        "b64_shard_key": (i64, [ctypes.c_int32, i64, i64]),
        "b64_combine_shards": (i32, [i64, vp, i32, i64, ctypes.POINTER(_Result)]),
        "b64_combine_shards_async": (i32, [vp, vp, i32, i64, vp, vp]),
        "b64_encode_host_ex": (i64, [vp, i64, vp, i32, vp, vp, vp]),
        "b64_decode_scratch_async": (i32, [vp, i64, vp, i32, vp, vp, vp]),
        "b64_decode_host_ex": (i32, [vp, i64, vp, i32, p64, p64, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


# ------------------------------------------------------------ helpers ---

def _ptr(t) -> int | None:
    return t.data_ptr() if t is not None else None


def _stream(stream, device):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _check_u8_cuda(t, name):
    import torch

    if not (isinstance(t, torch.Tensor) and t.dtype == torch.uint8 and t.is_cuda and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous uint8 CUDA tensor")


# --------------------------------------------------------------- sizes ---

def b64_encoded_len(n: int) -> int:
    return load_library().b64_encoded_len(n)


def b64_decoded_max_len(m: int) -> int:
    return load_library().b64_decoded_max_len(m)


def b64_status_str(code: int) -> str:
    return load_library().b64_status_str(code).decode()


def b64_build_info() -> str:
    return load_library().b64_build_info().decode()


# -------------------------------------------------------------- encode ---

def b64_encoded_len_ex(n: int, flags: int) -> int:
    return load_library().b64_encoded_len_ex(n, flags)


def b64_decoded_max_len_ex(m: int, flags: int) -> int:
    return load_library().b64_decoded_max_len_ex(m, flags)


def b64_encode(inp, out=None, stream=None, flags: int = 0):
    """Encode the uint8 CUDA tensor ``inp``; returns the output view."""
    import torch

    _check_u8_cuda(inp, "inp")
    lib = load_library()
    n = inp.numel()
    need = lib.b64_encoded_len_ex(n, flags)
    if out is None:
        out = torch.empty(max(need, 1), dtype=torch.uint8, device=inp.device)
    else:
        _check_u8_cuda(out, "out")
        if out.numel() < need:
            raise ValueError("out too small")
    rc = lib.b64_encode_ex(_ptr(inp), n, _ptr(out), flags, _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_encode")
    return out[:rc]


b64_encode_ex = b64_encode


# -------------------------------------------------------------- decode ---

def b64_decode(inp, out=None, stream=None, flags: int = 0):
    """Validating decode (synchronizes the stream).

    Returns (out_view, status, err_pos); out_view has out_len bytes."""
    import torch

    _check_u8_cuda(inp, "inp")
    lib = load_library()
    m = inp.numel()
    cap = lib.b64_decoded_max_len_ex(m, flags)
    if out is None:
        out = torch.empty(max(cap, 1), dtype=torch.uint8, device=inp.device)
    else:
        _check_u8_cuda(out, "out")
        if out.numel() < cap:
            raise ValueError("out too small")
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = lib.b64_decode_ex(_ptr(inp), m, _ptr(out), flags, ctypes.byref(ol), ctypes.byref(ep),
                           _stream(stream, inp.device))
    if st < 0:
        raise B64Error(st, "b64_decode")
    return out[: ol.value], st, ep.value


b64_decode_ex = b64_decode


def result_tensor(device):
    """A device tensor holding one b64_result record (int64[3])."""
    import torch

    return torch.zeros(3, dtype=torch.int64, device=device)


def unpack_result(res):
    """(out_len, err_pos, status, pad_count) from a result tensor."""
    v = res.cpu().tolist()
    st = v[2] & 0xFFFFFFFF
    pc = (v[2] >> 32) & 0xFFFFFFFF
    return v[0], v[1], st, pc


def _check_result(result):
    import torch

    if not (isinstance(result, torch.Tensor) and result.is_cuda and result.dtype == torch.int64
            and result.is_contiguous() and result.numel() >= 3):
        raise TypeError("result must be a contiguous int64[3] CUDA tensor")


def _check_dec_args(inp, out, result, flags):
    _check_u8_cuda(inp, "inp")
    _check_u8_cuda(out, "out")
    _check_result(result)
    cap = load_library().b64_decoded_max_len_ex(inp.numel(), flags)
    if cap < 0:
        raise B64Error(B64_ERR_ARG, "flags")
    if out.numel() < cap:
        raise ValueError("out too small")


def b64_decode_async(inp, out, result, stream=None, flags: int = 0):
    """Asynchronous validating decode; the b64_result record lands in
    ``result`` (int64[3] CUDA tensor, see unpack_result)."""
    b64_decode_ex_async(inp, out, result, flags, stream)


def b64_decode_ex_async(inp, out, result, flags: int, stream=None):
    _check_dec_args(inp, out, result, flags)
    rc = load_library().b64_decode_ex_async(_ptr(inp), inp.numel(), _ptr(out), flags,
                                            result.data_ptr(), _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_decode_ex_async")


def scratch_tensor(device):
    """A zeroed caller-owned decode scratch record (B64_DECODE_SCRATCH_BYTES)."""
    import torch

    return torch.zeros(B64_DECODE_SCRATCH_BYTES // 8, dtype=torch.int64, device=device)


def b64_decode_scratch_async(inp, out, result, scratch, flags: int = 0, stream=None):
    """Asynchronous decode with a caller-owned scratch record (scratch_tensor):
    safe for concurrently replayed CUDA graphs that use distinct records."""
    import torch

    _check_dec_args(inp, out, result, flags)
    if not (isinstance(scratch, torch.Tensor) and scratch.is_cuda and scratch.is_contiguous() and
            scratch.numel() * scratch.element_size() >= B64_DECODE_SCRATCH_BYTES):
        raise TypeError("scratch must be a contiguous CUDA tensor of >= 16 bytes (scratch_tensor)")
    rc = load_library().b64_decode_scratch_async(_ptr(inp), inp.numel(), _ptr(out), flags,
                                                 result.data_ptr(), scratch.data_ptr(),
                                                 _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_decode_scratch_async")


def b64_decode_shard_async(inp, out, result, final_shard=True, stream=None):
    _check_dec_args(inp, out, result, 0)
    rc = load_library().b64_decode_shard_async(_ptr(inp), inp.numel(), 1 if final_shard else 0,
                                               _ptr(out), result.data_ptr(),
                                               _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_decode_shard_async")


def b64_decode_shard_ex_async(inp, out, result, shard_begin: int, final_shard: bool, flags: int = 0,
                              key=None, stream=None):
    """Shard decode with variant flags; ``key`` (int64[2] CUDA tensor or
    None) receives (b64_shard_key, out_len) for the multi-GPU exchange."""
    import torch

    _check_dec_args(inp, out, result, flags)
    if key is not None and not (isinstance(key, torch.Tensor) and key.is_cuda and
                                key.dtype == torch.int64 and key.is_contiguous() and key.numel() >= 2):
        raise TypeError("key must be a contiguous int64[2] CUDA tensor")
    rc = load_library().b64_decode_shard_ex_async(
        _ptr(inp), inp.numel(), shard_begin, 1 if final_shard else 0, _ptr(out), flags,
        result.data_ptr(), _ptr(key), _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_decode_shard_ex_async")


def b64_shard_key(status: int, err_pos: int, shard_begin: int) -> int:
    """Reduction key of one shard result (C ABI b64_shard_key, pure host)."""
    return load_library().b64_shard_key(status, err_pos, shard_begin)


def b64_combine_shards(key_min: int, shard_out_lens, total_m: int):
    """(status, err_pos, out_len, pad_count) of the whole buffer from the MIN
    reduction key and the shard output lengths (C ABI, pure host)."""
    import numpy as np

    lens = np.ascontiguousarray(np.asarray(shard_out_lens, dtype=np.int64))
    r = _Result()
    rc = load_library().b64_combine_shards(key_min, lens.ctypes.data, lens.size, total_m,
                                           ctypes.byref(r))
    if rc < 0:
        raise B64Error(rc, "b64_combine_shards")
    return r.status, r.err_pos, r.out_len, r.pad_count


def b64_combine_shards_async(key_min, shard_out_lens, total_m: int, result, stream=None):
    """Device form: key_min (int64[1]) and shard_out_lens (int64[world]) are
    CUDA tensors; the record lands in ``result`` without a host sync."""
    import torch

    for t, nm in ((key_min, "key_min"), (shard_out_lens, "shard_out_lens")):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int64 and t.is_contiguous()):
            raise TypeError(f"{nm} must be a contiguous int64 CUDA tensor")
    _check_result(result)
    rc = load_library().b64_combine_shards_async(key_min.data_ptr(), shard_out_lens.data_ptr(),
                                                 shard_out_lens.numel(), total_m, result.data_ptr(),
                                                 _stream(stream, result.device))
    if rc < 0:
        raise B64Error(rc, "b64_combine_shards_async")


# ------------------------------------------------------------- batched ---

def b64_batch_workspace_bytes(k: int, total_in: int, direction: int) -> int:
    return load_library().b64_batch_workspace_bytes(k, total_in, direction)


def _check_off(t, name, n=None):
    import torch

    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int64 and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous int64 CUDA tensor")
    if n is not None and t.numel() < n:
        raise ValueError(f"{name} too small")


def _ws(k, total, direction, device, ws):
    import torch

    need = b64_batch_workspace_bytes(k, total, direction)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need + 256, dtype=torch.uint8, device=device)
    # 256-byte alignment (torch allocations are 512-aligned; views may not be)
    off = (-ws.data_ptr()) % 256
    return ws[off:], need


def b64_encode_batch(inp, in_off, out=None, out_off=None, ws=None, total_in=None, stream=None,
                     flags: int = 0):
    """Batched encode; in_off: int64[k+1] CUDA tensor.  Returns (out, out_off)."""
    import torch

    _check_u8_cuda(inp, "inp")
    k = in_off.numel() - 1
    total = inp.numel() if total_in is None else total_in
    if out is None:
        out = torch.empty(max(4 * ((total + 2) // 3) + 4 * k, 1), dtype=torch.uint8, device=inp.device)
    else:
        # the exact need (sum of per-message encoded lengths) lives on the
        # device; every batch needs at least the whole-input encoded length
        _check_u8_cuda(out, "out")
        if out.numel() < (4 * total + 2) // 3:
            raise ValueError("out too small")
    _check_off(in_off, "in_off")
    if out_off is None:
        out_off = torch.empty(k + 1, dtype=torch.int64, device=inp.device)
    _check_off(out_off, "out_off", k + 1)
    w, need = _ws(k, total, 0, inp.device, ws)
    rc = load_library().b64_encode_batch_ex(_ptr(inp), in_off.data_ptr(), k, total, _ptr(out),
                                            out_off.data_ptr(), flags, w.data_ptr(), w.numel(),
                                            _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_encode_batch")
    return out, out_off


def b64_decode_batch(inp, in_off, out=None, out_off=None, out_len=None, err_pos=None,
                     status=None, ws=None, total_in=None, stream=None, flags: int = 0):
    """Batched validating decode.  Returns (out, out_off, out_len, err_pos, status)."""
    import torch

    _check_u8_cuda(inp, "inp")
    k = in_off.numel() - 1
    dev = inp.device
    total = inp.numel() if total_in is None else total_in
    if out is None:
        out = torch.empty(max(3 * (total // 4) + 2 * k + 1, 1), dtype=torch.uint8, device=dev)
    else:
        _check_u8_cuda(out, "out")
    _check_off(in_off, "in_off")
    if out_off is None:
        out_off = torch.empty(k + 1, dtype=torch.int64, device=dev)
    if out_len is None:
        out_len = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    if err_pos is None:
        err_pos = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
    if status is None:
        status = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    _check_off(out_off, "out_off", k + 1)
    _check_off(out_len, "out_len", k)
    _check_off(err_pos, "err_pos", k)
    if not (status.is_cuda and status.dtype == torch.int32 and status.is_contiguous() and status.numel() >= k):
        raise TypeError("status must be a contiguous int32[k] CUDA tensor")
    w, need = _ws(k, total, 1, dev, ws)
    rc = load_library().b64_decode_batch_ex(_ptr(inp), in_off.data_ptr(), k, total, _ptr(out),
                                            out_off.data_ptr(), out_len.data_ptr(),
                                            err_pos.data_ptr(), status.data_ptr(), flags,
                                            w.data_ptr(), w.numel(), _stream(stream, dev))
    if rc < 0:
        raise B64Error(rc, "b64_decode_batch")
    return out, out_off, out_len[:k], err_pos[:k], status[:k]


# -------------------------------------------------------- host buffers ---

def _check_host(h, name, need):
    import torch

    if not (isinstance(h, torch.Tensor) and h.dtype == torch.uint8 and not h.is_cuda and h.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous uint8 CPU tensor")
    if h.numel() < need:
        raise ValueError(f"{name} too small")


def b64_encode_host(h_in, h_out, d_scratch_in, d_scratch_out, stream=None, flags: int = 0):
    """h_in/h_out: (pinned) CPU uint8 tensors; returns the output length."""
    lib = load_library()
    n = h_in.numel()
    need = lib.b64_encoded_len_ex(n, flags)
    _check_host(h_in, "h_in", n)
    _check_host(h_out, "h_out", need)
    _check_u8_cuda(d_scratch_in, "d_scratch_in")
    _check_u8_cuda(d_scratch_out, "d_scratch_out")
    if d_scratch_in.numel() < n or d_scratch_out.numel() < need:
        raise ValueError("scratch too small")
    rc = lib.b64_encode_host_ex(_ptr(h_in), n, _ptr(h_out), flags, _ptr(d_scratch_in),
                                _ptr(d_scratch_out), _stream(stream, d_scratch_in.device))
    if rc < 0:
        raise B64Error(rc, "b64_encode_host")
    return rc


def b64_decode_host(h_in, h_out, d_scratch_in, d_scratch_out, stream=None, flags: int = 0):
    """Returns (status, out_len, err_pos)."""
    lib = load_library()
    m = h_in.numel()
    cap = lib.b64_decoded_max_len_ex(m, flags)
    _check_host(h_in, "h_in", m)
    _check_host(h_out, "h_out", cap)
    _check_u8_cuda(d_scratch_in, "d_scratch_in")
    _check_u8_cuda(d_scratch_out, "d_scratch_out")
    if d_scratch_in.numel() < m or d_scratch_out.numel() < cap:
        raise ValueError("scratch too small")
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = lib.b64_decode_host_ex(_ptr(h_in), m, _ptr(h_out), flags, ctypes.byref(ol),
                                ctypes.byref(ep), _ptr(d_scratch_in), _ptr(d_scratch_out),
                                _stream(stream, d_scratch_in.device))
    if st < 0:
        raise B64Error(st, "b64_decode_host")
    return st, ol.value, ep.value


# -------------------------------------------------------------- shards ---

def b64_shard(total: int, unit: int, world: int, rank: int) -> tuple[int, int]:
    b = ctypes.c_int64(0)
    e = ctypes.c_int64(0)
    rc = load_library().b64_shard(total, unit, world, rank, ctypes.byref(b), ctypes.byref(e))
    if rc < 0:
        raise B64Error(rc, "b64_shard")
    return b.value, e.value


def b64_batch_shard(in_off, world: int, rank: int) -> tuple[int, int]:
    """Messages [begin, end) of rank's equal-byte share of a batch (C ABI
    b64_batch_shard); ``in_off`` is a host int64 array of k+1 offsets."""
    import numpy as np

    off = np.ascontiguousarray(np.asarray(in_off, dtype=np.int64))
    b = ctypes.c_int64(0)
    e = ctypes.c_int64(0)
    rc = load_library().b64_batch_shard(off.ctypes.data, off.size - 1, world, rank, ctypes.byref(b),
                                        ctypes.byref(e))
    if rc < 0:
        raise B64Error(rc, "b64_batch_shard")
    return b.value, e.value


# ---------------------------------------------------------- whitespace ---

def b64_despace(inp, out=None, ws=None, stream=None):
    """Remove ' ', '\\n', '\\r' (Appendix B).  Returns (out, out_len_tensor);
    the length stays on the device (int64[1]) until the caller reads it."""
    import torch

    _check_u8_cuda(inp, "inp")
    lib = load_library()
    m = inp.numel()
    if out is None:
        out = torch.empty(max(m, 1), dtype=torch.uint8, device=inp.device)
    else:
        _check_u8_cuda(out, "out")
        if out.numel() < m:
            raise ValueError("out too small")
    need = lib.b64_despace_workspace_bytes(m)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=inp.device)
    olen = torch.empty(1, dtype=torch.int64, device=inp.device)
    rc = lib.b64_despace(_ptr(inp), m, _ptr(out), olen.data_ptr(), ws.data_ptr(), ws.numel(),
                         _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_despace")
    return out, olen


# ------------------------------------------------- MIME line handling ---

def b64_decode_ws_workspace_bytes(m: int) -> int:
    return load_library().b64_decode_ws_workspace_bytes(m)


def _ws_scratch(m, device, ws):
    import torch

    need = b64_decode_ws_workspace_bytes(m)
    if ws is None or ws.numel() < need or ws.data_ptr() % 16:
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=device)
    return ws


def b64_decode_ws(inp, out=None, flags: int = 0, ws=None, stream=None):
    """Whitespace-tolerant decode (App. B filter + Alg 2, fused).  Returns
    (out[:out_len], status, err_pos); err_pos is an offset into ``inp``."""
    import torch

    _check_u8_cuda(inp, "inp")
    lib = load_library()
    m = inp.numel()
    cap = lib.b64_decoded_max_len_ex(m, flags)
    if out is None:
        out = torch.empty(max(cap, 1), dtype=torch.uint8, device=inp.device)
    else:
        _check_u8_cuda(out, "out")
        if out.numel() < cap:
            raise ValueError("out too small")
    ws = _ws_scratch(m, inp.device, ws)
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = lib.b64_decode_ws(_ptr(inp), m, _ptr(out), flags, ctypes.byref(ol), ctypes.byref(ep),
                           ws.data_ptr(), ws.numel(), _stream(stream, inp.device))
    if st < 0:
        raise B64Error(st, "b64_decode_ws")
    return out[: ol.value], st, ep.value


def b64_decode_ws_async(inp, out, result, flags: int = 0, ws=None, stream=None):
    """Asynchronous whitespace-tolerant decode; the b64_result record lands in
    ``result`` (int64[3] CUDA tensor, see unpack_result)."""
    import torch

    _check_u8_cuda(inp, "inp")
    _check_u8_cuda(out, "out")
    if not (result.is_cuda and result.dtype == torch.int64 and result.numel() >= 3):
        raise TypeError("result must be an int64[3] CUDA tensor")
    lib = load_library()
    m = inp.numel()
    if out.numel() < lib.b64_decoded_max_len_ex(m, flags):
        raise ValueError("out too small")
    ws = _ws_scratch(m, inp.device, ws)
    rc = lib.b64_decode_ws_async(_ptr(inp), m, _ptr(out), flags, result.data_ptr(), ws.data_ptr(),
                                 ws.numel(), _stream(stream, inp.device))
    if rc < 0:
        raise B64Error(rc, "b64_decode_ws_async")


def b64_encoded_len_wrapped(n: int, line_chars: int = 76, crlf: bool = True, flags: int = 0) -> int:
    return load_library().b64_encoded_len_wrapped(n, line_chars, int(crlf), flags)


def b64_encode_wrapped(inp, out=None, line_chars: int = 76, crlf: bool = True, flags: int = 0,
                       stream=None):
    """Line-wrapped encode (EOL after every ``line_chars`` chars and after the
    final line).  Returns the output view (asynchronous)."""
    import torch

    _check_u8_cuda(inp, "inp")
    lib = load_library()
    n = inp.numel()
    cap = lib.b64_encoded_len_wrapped(n, line_chars, int(crlf), flags)
    if cap < 0:
        raise B64Error(cap, "b64_encoded_len_wrapped")
    if out is None:
        out = torch.empty(max(cap, 1), dtype=torch.uint8, device=inp.device)
    else:
        _check_u8_cuda(out, "out")
        if out.numel() < cap:
            raise ValueError("out too small")
    r = lib.b64_encode_wrapped(_ptr(inp), n, _ptr(out), line_chars, int(crlf), flags,
                               _stream(stream, inp.device))
    if r < 0:
        raise B64Error(r, "b64_encode_wrapped")
    return out[:r]
