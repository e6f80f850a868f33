"""ctypes binding of libbsa.so (the C ABI declared in include/bsa.h).

This is the only module that talks to the native library.  There is no CPU
path: if the library or a CUDA device is missing, every operator raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libbsa.so")
# kernel A/B experiments only (scripts/): load another in-tree build of the library
if os.environ.get("BSA_LIB_VARIANT"):
    LIB_PATH = os.path.join(_PKG, "csrc", "build", os.environ["BSA_LIB_VARIANT"], "libbsa.so")

BSA_OK, BSA_EINVAL, BSA_EUNSUPPORTED, BSA_ECUDA = 0, 1, 2, 3
BSA_F32, BSA_BF16 = 0, 1
PATH_AUTO, PATH_SIMT, PATH_TC = 0, 1, 2
FLAG_TIMING = 16
FLAG_NATURAL_ORDER = 32

_DTYPE_CODE = {torch.float32: BSA_F32, torch.bfloat16: BSA_BF16}


class BsaLayout(ctypes.Structure):
    _fields_ = [
        ("frames", ctypes.c_int64),
        ("patches_per_frame", ctypes.c_int64),
        ("specials_per_frame", ctypes.c_int64),
        ("specials_first", ctypes.c_int32),
    ]


class BsaTensor(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("heads", ctypes.c_int64),
        ("tokens", ctypes.c_int64),
        ("dim", ctypes.c_int64),
        ("stride_head", ctypes.c_int64),
        ("stride_token", ctypes.c_int64),
    ]


class BsaScatter(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int32),
        ("out_ptrs", ctypes.c_void_p),
        ("token_begin", ctypes.c_void_p),
    ]


IPC_HANDLE_BYTES = 64

_lib = None
_lock = threading.Lock()


def _declare(L):
    i32, i64, f32, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double
    vp, sz = ctypes.c_void_p, ctypes.c_size_t
    pt, pl = ctypes.POINTER(BsaTensor), ctypes.POINTER(BsaLayout)
    sigs = {
        "bsa_version": ([], ctypes.c_int),
        "bsa_last_error": ([], ctypes.c_char_p),
        "bsa_device_sm_count": ([], ctypes.c_int),
        "bsa_block_pool": ([pt, pl, i32, vp, vp], ctypes.c_int),
        "bsa_pooled_scores_workspace": ([i64, i64, i64], sz),
        "bsa_pooled_scores": ([vp, vp, i64, i64, i64, i64, f32, vp, vp, sz, vp], ctypes.c_int),
        "bsa_row_softmax_workspace": ([i64, i64], sz),
        "bsa_row_softmax": ([vp, i64, i64, f32, vp, vp, sz, vp], ctypes.c_int),
        "bsa_select_workspace": ([i64, i64, i64], sz),
        "bsa_select_blocks": ([vp, i64, i64, i64, f64, i64, vp, vp, vp, sz, vp], ctypes.c_int),
        "bsa_predict_mask_workspace": ([i64, i64, i64, i32, i32], sz),
        "bsa_predict_mask": ([pt, pt, pl, i32, i32, f32, f64, i64, vp, vp, vp, vp, sz, vp],
                             ctypes.c_int),
        "bsa_predict_mask_pooled_workspace": ([i64, i64, i64, i64], sz),
        "bsa_predict_mask_pooled": ([vp, vp, i64, i64, i64, i64, f32, f64, i64, vp, vp, vp, vp, sz,
                                     vp], ctypes.c_int),
        "bsa_qkv_project_pooled": ([vp, i64, i64, vp, vp, i64, i64, i64, i32, i32, vp, vp, vp, vp,
                                    vp, vp], ctypes.c_int),
        "bsa_proj_residual": ([vp, i64, i64, vp, vp, vp, vp, vp], ctypes.c_int),
        "bsa_copy_tokens": ([vp, vp, pl, i64, i64, i32, vp], ctypes.c_int),
        "bsa_sparse_attention_workspace": ([pl, i64, i64, i32, i32, i32, i32, i32], sz),
        "bsa_sparse_attention": ([pt, pt, pt, vp, i32, pl, i32, i32, vp, vp, f32, i32, i32, i32,
                                  i32, vp, sz, vp], ctypes.c_int),
        "bsa_sparse_attention_path": ([pl, i64, i32, i32, i32, i32], ctypes.c_int),
        "bsa_last_kernel_ms": ([], ctypes.c_float),
        "bsa_kernel_times": ([vp, i32, i32], ctypes.c_int),
        "bsa_mask_selected_area": ([vp, i64, i64, i32, i32, vp, vp], ctypes.c_int),
        "bsa_mask_to_csr_workspace": ([i64, i64], sz),
        "bsa_mask_to_csr": ([vp, i64, i64, i64, vp, vp, vp, sz, vp], ctypes.c_int),
        "bsa_sparse_attention_scatter": ([pt, pt, pt, pl, i32, i32, vp, vp, f32, i32, i32, i32,
                                          ctypes.POINTER(BsaScatter), vp, sz, vp], ctypes.c_int),
        "bsa_ipc_alloc": ([sz, ctypes.POINTER(vp), vp], ctypes.c_int),
        "bsa_ipc_open": ([vp, ctypes.POINTER(vp)], ctypes.c_int),
        "bsa_ipc_close": ([vp], ctypes.c_int),
        "bsa_ipc_free": ([vp], ctypes.c_int),
        "bsa_attention_stats_workspace": ([pl, i64], sz),
        "bsa_attention_row_stats": ([pt, pt, pl, f32, vp, vp, sz, vp], ctypes.c_int),
        "bsa_block_attention_map": ([pt, pt, pl, f32, vp, vp, vp, sz, vp], ctypes.c_int),
        "bsa_check_finite": ([pt, vp, vp], ctypes.c_int),
        "bsa_scoring_rows_per_cta": ([i64, i64], ctypes.c_int),
        "bsa_debug_scoring_trace": ([vp, sz], ctypes.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


def exported_symbols():
    """Names include/bsa.h declares (checked by the CPU test-suite)."""
    return [
        "bsa_version", "bsa_last_error", "bsa_device_sm_count", "bsa_block_pool",
        "bsa_pooled_scores_workspace", "bsa_pooled_scores", "bsa_row_softmax_workspace",
        "bsa_row_softmax",
        "bsa_select_workspace", "bsa_select_blocks", "bsa_predict_mask_workspace",
        "bsa_predict_mask", "bsa_sparse_attention_workspace", "bsa_sparse_attention",
        "bsa_sparse_attention_path", "bsa_last_kernel_ms", "bsa_mask_selected_area", "bsa_mask_to_csr_workspace",
        "bsa_mask_to_csr", "bsa_sparse_attention_scatter", "bsa_ipc_alloc", "bsa_ipc_open",
        "bsa_ipc_close", "bsa_ipc_free", "bsa_attention_stats_workspace",
        "bsa_attention_row_stats", "bsa_block_attention_map", "bsa_check_finite",
        "bsa_scoring_rows_per_cta", "bsa_debug_scoring_trace",
        "bsa_predict_mask_pooled_workspace", "bsa_predict_mask_pooled", "bsa_qkv_project_pooled",
        "bsa_proj_residual", "bsa_copy_tokens", "bsa_kernel_times",
    ]


def lib():
    """Load libbsa.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(there is no CPU fallback)")
                _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_07120_b200 needs a CUDA device (sm_100a); no CPU path exists")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def check(rc: int, what: str):
    if rc == BSA_OK:
        return
    msg = lib().bsa_last_error().decode(errors="replace")
    if rc in (BSA_EINVAL, BSA_EUNSUPPORTED):
        raise ValueError(msg or f"{what}: invalid argument")
    raise RuntimeError(f"{what}: {msg}")


def stream_ptr(device=None) -> int:
    """The current stream of `device` (default: the current device)."""
    return torch.cuda.current_stream(device).cuda_stream


def on_device(device):
    """Make `device` current for a launch: kernels run on the device that
    holds the tensors, never on whichever device happens to be current."""
    return torch.cuda.device(device)


_FINITE_SEEN: dict = {}  # id(tensor) -> (weakref, version) of tensors found finite


def _known_finite(t: torch.Tensor) -> bool:
    e = _FINITE_SEEN.get(id(t))
    return e is not None and e[0]() is t and e[1] == t._version


def _mark_finite(t: torch.Tensor) -> None:
    if len(_FINITE_SEEN) > 256:
        for key in [k for k, (r, _) in _FINITE_SEEN.items() if r() is None]:
            del _FINITE_SEEN[key]
        if len(_FINITE_SEEN) > 256:
            _FINITE_SEEN.clear()
    try:
        _FINITE_SEEN[id(t)] = (weakref.ref(t), t._version)
    except TypeError:  # not weak-referenceable: just do not cache
        pass


def all_finite(*tensors: torch.Tensor) -> bool:
    """True when no element of the tensors is NaN or +-inf. The reference's
    as_f32 rejects non-finite inputs (tensorio.py:47-59). CUDA (H, T, d)
    fp32/bf16 tensors (any head/token strides) are scanned by one HBM-bound
    kernel each (bsa_check_finite, no temporaries) into a shared flag, read
    back with ONE sync; anything else falls back to torch. A tensor object
    already found finite whose version counter (bumped by every in-place
    write) has not moved since is not rescanned."""
    todo = [t for t in tensors if not _known_finite(t)]
    cuda = [t for t in todo if t.device.type == "cuda"]
    dev = [t for t in cuda if t.dim() == 3 and t.dtype in _DTYPE_CODE and t.stride(2) == 1
           and t.device == cuda[0].device]
    rest = [t for t in todo if not any(t is x for x in dev)]
    ok = True
    if dev:
        flag = torch.zeros(1, dtype=torch.int32, device=dev[0].device)
        with on_device(dev[0].device):
            for t in dev:
                check(lib().bsa_check_finite(tensor_desc(t), flag.data_ptr(), stream_ptr()),
                      "check_finite")
        ok = int(flag.item()) == 0
    for t in rest:
        ok = ok and bool(torch.isfinite(t).all())
    if ok:
        for t in todo:
            _mark_finite(t)
    return ok


def finite_scan(t: torch.Tensor, flag: torch.Tensor) -> None:
    """Asynchronous part of all_finite: OR "t has a NaN/inf" into the device
    int32 `flag` (same device) without synchronising."""
    with on_device(t.device):
        check(lib().bsa_check_finite(tensor_desc(t), flag.data_ptr(), stream_ptr()),
              "check_finite")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def tensor_desc(t: torch.Tensor) -> BsaTensor:
    if t.dim() != 3:
        raise ValueError(f"expected (heads, tokens, head_dim), got {tuple(t.shape)}")
    if t.dtype not in _DTYPE_CODE:
        raise ValueError(f"unsupported dtype {t.dtype}")
    if t.stride(2) != 1:
        raise ValueError("head_dim must be contiguous")
    return BsaTensor(t.data_ptr(), _DTYPE_CODE[t.dtype], t.shape[0], t.shape[1], t.shape[2],
                     t.stride(0), t.stride(1))


def layout_desc(layout) -> BsaLayout:
    return BsaLayout(layout.frames, layout.patches_per_frame, layout.specials_per_frame,
                     1 if layout.specials_first else 0)


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
