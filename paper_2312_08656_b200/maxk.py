"""Thin ctypes binding of include/maxk.h — argument marshalling only.

Every computation runs in libmaxk.so's CUDA kernels. There is no CPU fallback: tensors must live on a
CUDA device, and importing this module on a machine without the built library raises.
Names mirror the C-ABI (maxk_topk_cbsr, maxk_plan_create, maxk_spgemm_fwd, maxk_sspmm_bwd).
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import build as _build

_lib = None


class MaxkError(RuntimeError):
    def __init__(self, status: int, fn: str, detail: str):
        self.status = status
        super().__init__(f"{fn} failed: {_status_name(status)}: {detail}")


STATUS = {0: "MAXK_OK", 1: "MAXK_ERR_INVALID_ARGUMENT", 2: "MAXK_ERR_UNSUPPORTED", 3: "MAXK_ERR_CUDA",
          4: "MAXK_ERR_OUT_OF_MEMORY"}


def _status_name(s: int) -> str:
    return STATUS.get(s, f"status {s}")


def lib_path() -> str:
    """The loaded library: libmaxk.so in-tree, or MAXK_LIB (an A/B build of the same sources)."""
    return os.environ.get("MAXK_LIB") or _build.LIB


def load(build_if_missing: bool = True):
    """Load libmaxk.so (building it with nvcc first if it is missing or stale and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if os.environ.get("MAXK_LIB"):  # explicit A/B build: no rebuild
        build_if_missing = False
    if build_if_missing and _build.stale():
        try:
            _build.build()
        except (OSError, RuntimeError) as e:  # no nvcc on this machine: use the shipped .so if present
            if not os.path.exists(_build.LIB):
                raise ImportError(f"libmaxk.so missing and cannot be built: {e}") from e
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"libmaxk.so not found at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    i64, i32, vp, st = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p
    lib.maxk_topk_cbsr.argtypes = [vp, i64, i32, i64, i32, i32, vp, vp, st]
    lib.maxk_topk_cbsr_probe_stats.argtypes = [vp, i64, i32, i64, i32, i32, vp, vp, vp, st]
    lib.maxk_topk_cbsr_pairs.argtypes = [vp, i64, i32, i64, i32, i32, vp, vp, vp, st]
    lib.maxk_topk_cbsr_banked.argtypes = [vp, i64, i32, i64, i32, i32, vp, vp, vp, vp, st]
    lib.maxk_topk_cbsr_pairs_banked.argtypes = [vp, i64, i32, i64, i32, i32, vp, vp, vp, st]
    lib.maxk_topk_cbsr_multi.argtypes = [vp, i64, i32, i64, i32, i32, i32, vp, vp, st]
    lib.maxk_sspmm_bwd_owners.argtypes = [vp, vp, vp, i64, i64, i64, vp, i64, vp, i32, i32, i32, i32, i64, vp, vp, st]
    lib.maxk_spgemm_fwd_replicated.argtypes = [i64, i64, i32, i32]
    lib.maxk_spgemm_fwd_replicated.restype = ctypes.c_int32
    lib.maxk_spgemm_fwd_pairs.argtypes = [vp, vp, vp, i64, i64, i64, vp, i32, i32, vp, i64, vp, st]
    lib.maxk_plan_create.argtypes = [vp, i64, i64, i32, i32, st, ctypes.POINTER(vp)]
    lib.maxk_plan_destroy.argtypes = [vp]
    lib.maxk_plan_destroy.restype = None
    lib.maxk_plan_info.argtypes = [vp] + [ctypes.POINTER(i64)] * 4
    lib.maxk_spgemm_fwd.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, i32, i32, i32, vp, i64, vp, st]
    lib.maxk_sspmm_bwd.argtypes = [vp, vp, vp, i64, i64, i64, vp, i64, vp, i32, i32, i32, vp, vp, st]
    lib.maxk_spgemm_fwd_acc.argtypes = lib.maxk_spgemm_fwd.argtypes
    lib.maxk_sspmm_bwd_acc.argtypes = lib.maxk_sspmm_bwd.argtypes
    lib.maxk_add_f32.argtypes = [vp, vp, i64, st]
    lib.maxk_validate_csr.argtypes = [vp, vp, i64, i64, st, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.maxk_validate_cbsr.argtypes = [vp, i64, i32, i32, i32, st, ctypes.POINTER(i64)]
    lib.maxk_cbsr_scatter.argtypes = [vp, vp, i64, i32, i32, i32, vp, i64, st]
    lib.maxk_linear_topk_cbsr.argtypes = [vp, i64, i32, i64, vp, i64, vp, i32, i32, i32, vp, vp, vp, i64, st]
    for f in ("maxk_topk_cbsr", "maxk_topk_cbsr_probe_stats", "maxk_topk_cbsr_pairs", "maxk_topk_cbsr_banked",
              "maxk_topk_cbsr_pairs_banked", "maxk_topk_cbsr_multi", "maxk_sspmm_bwd_owners",
              "maxk_spgemm_fwd_pairs",
              "maxk_plan_create", "maxk_plan_info", "maxk_spgemm_fwd", "maxk_sspmm_bwd",
              "maxk_cbsr_scatter", "maxk_linear_topk_cbsr"):
        getattr(lib, f).restype = ctypes.c_int
    lib.maxk_status_string.argtypes = [ctypes.c_int]
    lib.maxk_status_string.restype = ctypes.c_char_p
    lib.maxk_last_error_detail.argtypes = []
    lib.maxk_last_error_detail.restype = ctypes.c_char_p
    lib.maxk_launch_count.argtypes = []
    lib.maxk_launch_count.restype = ctypes.c_uint64
    lib.maxk_version.argtypes = []
    lib.maxk_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


EXPORTED_SYMBOLS = ("maxk_topk_cbsr", "maxk_topk_cbsr_probe_stats", "maxk_topk_cbsr_pairs", "maxk_topk_cbsr_banked",
                    "maxk_topk_cbsr_pairs_banked", "maxk_topk_cbsr_multi", "maxk_sspmm_bwd_owners",
                    "maxk_spgemm_fwd_replicated", "maxk_spgemm_fwd_pairs", "maxk_cbsr_scatter", "maxk_linear_topk_cbsr", "maxk_plan_create",
                    "maxk_plan_destroy", "maxk_plan_info", "maxk_spgemm_fwd", "maxk_sspmm_bwd", "maxk_spgemm_fwd_acc",
                    "maxk_sspmm_bwd_acc", "maxk_add_f32", "maxk_validate_csr", "maxk_validate_cbsr",
                    "maxk_status_string", "maxk_last_error_detail",
                    "maxk_launch_count", "maxk_version")


def _check(rc: int, fn: str):
    if rc != 0:
        raise MaxkError(rc, fn, _lib.maxk_last_error_detail().decode())


def _dev(t: torch.Tensor, name: str, dtype=None) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.data_ptr()


def _rows(t: torch.Tensor, name: str) -> int:
    """Row stride of a 2-D row-major tensor with unit column stride."""
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


def _cbsr(t: torch.Tensor, name: str, k: int, min_rows: int, dtype=None) -> int:
    """A CBSR block (sp_data / sp_idx / d_sp_data): contiguous [rows, k] with rows >= min_rows (the kernels
    assume row stride k and index rows < min_rows)."""
    p = _dev(t, name, dtype)
    if t.dim() != 2 or t.shape[1] != k or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous [rows, {k}] tensor, got shape {tuple(t.shape)} "
                         f"strides {t.stride()}")
    if t.shape[0] < min_rows:
        raise ValueError(f"{name} has {t.shape[0]} rows < {min_rows} required")
    return p


def _dense(t: torch.Tensor, name: str, min_rows: int, h: int) -> tuple[int, int]:
    """A dense row-major [rows, >= h] fp32 operand (X, Y, dY, dX): pointer and row stride."""
    p = _dev(t, name, torch.float32)
    ld = _rows(t, name)
    if t.shape[0] < min_rows or t.shape[1] < h:
        raise ValueError(f"{name} must be at least [{min_rows}, {h}], got {tuple(t.shape)}")
    return p, ld


def _same_device(*ts):
    """Every tensor on the current CUDA device (the library launches on the current device's stream)."""
    cuda = [(name, t) for name, t in ts if isinstance(t, torch.Tensor) and t.is_cuda]
    if not cuda:
        return  # _dev raises for the non-CUDA ones
    cur = torch.cuda.current_device()
    for name, t in cuda:
        if t.device.index != cur:
            raise ValueError(f"{name} is on {t.device}, the current device is cuda:{cur}")


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def idx_dtype(h: int):
    return torch.uint8 if h <= 256 else torch.uint16


def idx_bytes_of(t: torch.Tensor) -> int:
    if t.dtype == torch.uint8:
        return 1
    if t.dtype in (torch.uint16, torch.int16):
        return 2
    raise TypeError(f"sp_idx must be uint8 or uint16, got {t.dtype}")


_NVTX = os.environ.get("MAXK_NVTX", "1") != "0"


class _NoRange:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def nvtx_range(name: str):
    """NVTX range around a step of the hot path (SURVEY §5 tracing; visible in nsys/ncu timelines). Host-side
    marker only: it adds no device work. MAXK_NVTX=0 disables it."""
    return torch.cuda.nvtx.range(name) if _NVTX else _NoRange()


def launch_count() -> int:
    return int(load().maxk_launch_count())


def version() -> str:
    return load().maxk_version().decode()


def maxk_topk_cbsr(x: torch.Tensor, k: int, sp_data: torch.Tensor | None = None, sp_idx: torch.Tensor | None = None,
                   stream=None):
    """MaxK top-k -> CBSR (Eq. 1). Returns (sp_data fp32 [n,k], sp_idx uint8/uint16 [n,k])."""
    lib = load()
    n, h = x.shape
    if sp_data is None:
        sp_data = torch.empty((n, k), dtype=torch.float32, device=x.device)
    if sp_idx is None:
        sp_idx = torch.empty((n, k), dtype=idx_dtype(h), device=x.device)
    _same_device(("x", x), ("sp_data", sp_data), ("sp_idx", sp_idx))
    px, ldx = _dense(x, "x", n, h)
    rc = lib.maxk_topk_cbsr(px, n, h, ldx, k, idx_bytes_of(sp_idx), _cbsr(sp_data, "sp_data", k, n, torch.float32),
                            _cbsr(sp_idx, "sp_idx", k, n), _stream(stream))
    _check(rc, "maxk_topk_cbsr")
    return sp_data, sp_idx


PAIR_K = (8, 16)
PAIR_H = (128, 256, 384, 512)


def pairs_supported(h: int, k: int) -> bool:
    """Whether the CBSR pair layout (include/maxk.h maxk_topk_cbsr_pairs) exists for (h, k)."""
    return k in PAIR_K and h in PAIR_H


def pairs_default(h: int, k: int) -> bool:
    """The layer path uses the pair layout wherever it exists (one 128-byte line per gathered CBSR row instead of
    two); MAXK_PAIRS=0 turns it off (A/B)."""
    return pairs_supported(h, k) and os.environ.get("MAXK_PAIRS", "1") != "0"


def _pairs(t: torch.Tensor, name: str, k: int, min_rows: int) -> int:
    p = _dev(t, name, torch.int32)
    if t.dim() != 3 or t.shape[1:] != (k, 2) or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int32 [rows, {k}, 2] tensor, got {tuple(t.shape)}")
    if t.shape[0] < min_rows:
        raise ValueError(f"{name} has {t.shape[0]} rows < {min_rows} required")
    return p


def maxk_topk_cbsr_pairs(x: torch.Tensor, k: int, sp_data: torch.Tensor | None = None,
                         sp_idx: torch.Tensor | None = None, sp_pairs: torch.Tensor | None = None, stream=None,
                         banked: bool = False):
    """maxk_topk_cbsr that also writes the pair layout. Returns (sp_data, sp_idx, sp_pairs int32 [n, k, 2]:
    (value bits, column) per entry). banked=True (k = 16): the pairs in the mod-4-balanced order
    (maxk_topk_cbsr_pairs_banked)."""
    lib = load()
    n, h = x.shape
    if sp_data is None:
        sp_data = torch.empty((n, k), dtype=torch.float32, device=x.device)
    if sp_idx is None:
        sp_idx = torch.empty((n, k), dtype=idx_dtype(h), device=x.device)
    if sp_pairs is None:
        sp_pairs = torch.empty((n, k, 2), dtype=torch.int32, device=x.device)
    _same_device(("x", x), ("sp_data", sp_data), ("sp_idx", sp_idx), ("sp_pairs", sp_pairs))
    px, ldx = _dense(x, "x", n, h)
    fn = "maxk_topk_cbsr_pairs_banked" if banked else "maxk_topk_cbsr_pairs"
    rc = getattr(lib, fn)(px, n, h, ldx, k, idx_bytes_of(sp_idx), _cbsr(sp_data, "sp_data", k, n, torch.float32),
                          _cbsr(sp_idx, "sp_idx", k, n), _pairs(sp_pairs, "sp_pairs", k, n), _stream(stream))
    _check(rc, fn)
    return sp_data, sp_idx, sp_pairs


BANKED_K = (16, 32, 64, 128)


def banked_supported(h: int, k: int) -> bool:
    """Whether a bank-balanced CBSR copy exists for (h, k): maxk_topk_cbsr_banked (two blocks, k in {32, 64, 128})
    or maxk_topk_cbsr_pairs_banked (the pair layout, k = 16)."""
    return k in BANKED_K and h in PAIR_H


def banked_default(h: int, k: int, n_rows: int, nnz: int) -> bool:
    """The layer path feeds the forward the bank-balanced CBSR copy where it pays: where the forward uses its
    replicated row buffers (maxk_spgemm_fwd_replicated: mean degree >= 64, h <= 256; NC = 16 at k >= 32 over the
    two-block copy, NC = 8 at k = 16 over the balanced pair layout), which then conflict only on unbalanced entries
    (DESIGN.md §5.2). Elsewhere the copy's extra 5k bytes per row written by the
    top-k cost about what the interleaved buffers gain. MAXK_BANKED=0 / 2 turns it off / forces it (A/B)."""
    mode = os.environ.get("MAXK_BANKED", "1")
    if mode == "0" or not banked_supported(h, k):
        return False
    return mode == "2" or bool(load().maxk_spgemm_fwd_replicated(n_rows, nnz, h, k))


def float4_rows(x: torch.Tensor) -> bool:
    """x rows are 16-byte aligned (what the compile-time top-k kernels of the pair / banked forms load)."""
    return x.data_ptr() % 16 == 0 and (x.shape[0] <= 1 or x.stride(0) % 4 == 0) and x.stride(-1) == 1


def maxk_topk_cbsr_banked(x: torch.Tensor, k: int, sp_data: torch.Tensor | None = None,
                          sp_idx: torch.Tensor | None = None, sp_bdata: torch.Tensor | None = None,
                          sp_bidx: torch.Tensor | None = None, stream=None):
    """maxk_topk_cbsr that also writes the bank-balanced copy of the CBSR (include/maxk.h). Returns
    (sp_data, sp_idx) in column order and (sp_bdata, sp_bidx), the same entries in the bank-balanced order."""
    lib = load()
    n, h = x.shape
    mk = lambda t, dt: t if t is not None else torch.empty((n, k), dtype=dt, device=x.device)  # noqa: E731
    sp_data, sp_bdata = mk(sp_data, torch.float32), mk(sp_bdata, torch.float32)
    sp_idx, sp_bidx = mk(sp_idx, idx_dtype(h)), mk(sp_bidx, idx_dtype(h))
    _same_device(("x", x), ("sp_data", sp_data), ("sp_idx", sp_idx), ("sp_bdata", sp_bdata), ("sp_bidx", sp_bidx))
    if sp_bidx.dtype != sp_idx.dtype:
        raise TypeError("sp_bidx must have sp_idx's dtype")
    px, ldx = _dense(x, "x", n, h)
    rc = lib.maxk_topk_cbsr_banked(px, n, h, ldx, k, idx_bytes_of(sp_idx),
                                   _cbsr(sp_data, "sp_data", k, n, torch.float32), _cbsr(sp_idx, "sp_idx", k, n),
                                   _cbsr(sp_bdata, "sp_bdata", k, n, torch.float32),
                                   _cbsr(sp_bidx, "sp_bidx", k, n), _stream(stream))
    _check(rc, "maxk_topk_cbsr_banked")
    return sp_data, sp_idx, sp_bdata, sp_bidx


def maxk_topk_cbsr_probe_stats(x: torch.Tensor, k: int, stream=None):
    """Debug statistic (not the hot path): the top-k -> CBSR of maxk_topk_cbsr plus the per-row number of pivot
    probes (+1000 when the exact descent decided the row). Returns (sp_data, sp_idx, probes int32 [n])."""
    lib = load()
    n, h = x.shape
    sp_data = torch.empty((n, k), dtype=torch.float32, device=x.device)
    sp_idx = torch.empty((n, k), dtype=idx_dtype(h), device=x.device)
    probes = torch.empty((n,), dtype=torch.int32, device=x.device)
    _same_device(("x", x))
    px, ldx = _dense(x, "x", n, h)
    rc = lib.maxk_topk_cbsr_probe_stats(px, n, h, ldx, k, idx_bytes_of(sp_idx), sp_data.data_ptr(),
                                        sp_idx.data_ptr(), probes.data_ptr(), _stream(stream))
    _check(rc, "maxk_topk_cbsr_probe_stats")
    return sp_data, sp_idx, probes


class Plan:
    """Owns a maxk_plan_t (maxk_plan_create / maxk_plan_destroy).

    Single-stream rule (include/maxk.h): a plan serves one call at a time in stream order — its device-side
    ticket counters and hub-row scratch are shared by every call that uses it. Give each concurrently running
    stream its own Plan. A plan belongs to the device current at creation; calls on another device raise."""

    def __init__(self, handle: int, n_rows: int, nnz: int):
        self.handle = ctypes.c_void_p(handle)
        self.n_rows, self.nnz = n_rows, nnz

    def info(self) -> dict:
        vals = [ctypes.c_int64() for _ in range(4)]
        _check(load().maxk_plan_info(self.handle, *[ctypes.byref(v) for v in vals]), "maxk_plan_info")
        return dict(zip(("n_units", "n_split_rows", "chunk_edges", "n_chunk_units"), (v.value for v in vals)))

    def close(self):
        if self.handle and self.handle.value:
            load().maxk_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def maxk_plan_create(row_ptr: torch.Tensor, h: int, k: int, stream=None) -> Plan:
    lib = load()
    n = row_ptr.shape[0] - 1
    _dev(row_ptr, "row_ptr", torch.int64)
    rp = row_ptr[[0, -1]].tolist() if n >= 0 else [0, 0]
    nnz = int(rp[1] - rp[0])
    out = ctypes.c_void_p()
    rc = lib.maxk_plan_create(row_ptr.data_ptr(), n, nnz, h, k, _stream(stream), ctypes.byref(out))
    _check(rc, "maxk_plan_create")
    return Plan(out.value, n, nnz)


def _csr(row_ptr, col_idx, val, nnz):
    n = row_ptr.shape[0] - 1
    for name, t in (("row_ptr", row_ptr), ("col_idx", col_idx), ("val", val)):
        if t.dim() != 1 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 1-D tensor")
    if col_idx.numel() != val.numel() or col_idx.numel() < nnz:
        raise ValueError(f"col_idx ({col_idx.numel()}) and val ({val.numel()}) must have the same length >= nnz={nnz}")
    p = (_dev(row_ptr, "row_ptr", torch.int64), _dev(col_idx, "col_idx", torch.int32), _dev(val, "val", torch.float32))
    return n, p


def maxk_spgemm_fwd(row_ptr: torch.Tensor, col_idx: torch.Tensor, val: torch.Tensor, n_cols: int, nnz: int,
                    sp_data: torch.Tensor, sp_idx: torch.Tensor, h: int, y: torch.Tensor | None = None,
                    plan: Plan | None = None, stream=None, accumulate: bool = False) -> torch.Tensor:
    """Y = A · CBSR (Eq. 3 left). y is overwritten (allocated if None), or added to when accumulate."""
    lib = load()
    n, (prp, pci, pva) = _csr(row_ptr, col_idx, val, nnz)
    k = sp_data.shape[1]
    if y is None:
        if accumulate:
            raise ValueError("accumulate needs an existing y")
        y = torch.empty((n, h), dtype=torch.float32, device=row_ptr.device)
    _same_device(("row_ptr", row_ptr), ("col_idx", col_idx), ("val", val), ("sp_data", sp_data), ("sp_idx", sp_idx),
                 ("y", y))
    py, ldy = _dense(y, "y", n, h)
    fn = lib.maxk_spgemm_fwd_acc if accumulate else lib.maxk_spgemm_fwd
    rc = fn(prp, pci, pva, n, n_cols, nnz, _cbsr(sp_data, "sp_data", k, n_cols, torch.float32),
            _cbsr(sp_idx, "sp_idx", k, n_cols), h, k, idx_bytes_of(sp_idx), py, ldy,
            plan.handle if plan is not None else None, _stream(stream))
    _check(rc, "maxk_spgemm_fwd")
    return y


def maxk_spgemm_fwd_pairs(row_ptr: torch.Tensor, col_idx: torch.Tensor, val: torch.Tensor, n_cols: int, nnz: int,
                          sp_pairs: torch.Tensor, h: int, y: torch.Tensor | None = None, plan: Plan | None = None,
                          stream=None) -> torch.Tensor:
    """Y = A · CBSR (Eq. 3 left) from the pair layout (maxk_topk_cbsr_pairs). y is overwritten (allocated if None)."""
    lib = load()
    n, (prp, pci, pva) = _csr(row_ptr, col_idx, val, nnz)
    k = sp_pairs.shape[1]
    if y is None:
        y = torch.empty((n, h), dtype=torch.float32, device=row_ptr.device)
    _same_device(("row_ptr", row_ptr), ("col_idx", col_idx), ("val", val), ("sp_pairs", sp_pairs), ("y", y))
    py, ldy = _dense(y, "y", n, h)
    rc = lib.maxk_spgemm_fwd_pairs(prp, pci, pva, n, n_cols, nnz, _pairs(sp_pairs, "sp_pairs", k, n_cols), h, k, py,
                                   ldy, plan.handle if plan is not None else None, _stream(stream))
    _check(rc, "maxk_spgemm_fwd_pairs")
    return y


def maxk_sspmm_bwd(row_ptr: torch.Tensor, col_idx: torch.Tensor, val: torch.Tensor, n_cols: int, nnz: int,
                   dy: torch.Tensor, sp_idx: torch.Tensor, d_sp_data: torch.Tensor | None = None,
                   plan: Plan | None = None, stream=None, accumulate: bool = False) -> torch.Tensor:
    """dXs = (A^T · dY) sampled at sp_idx (Eq. 3 right / Eq. 4). d_sp_data is overwritten, or added to."""
    lib = load()
    n, (prp, pci, pva) = _csr(row_ptr, col_idx, val, nnz)
    h = dy.shape[1]
    k = sp_idx.shape[1]
    if d_sp_data is None:
        if accumulate:
            raise ValueError("accumulate needs an existing d_sp_data")
        d_sp_data = torch.empty((n_cols, k), dtype=torch.float32, device=dy.device)
    _same_device(("row_ptr", row_ptr), ("col_idx", col_idx), ("val", val), ("dy", dy), ("sp_idx", sp_idx),
                 ("d_sp_data", d_sp_data))
    pdy, lddy = _dense(dy, "dy", n, h)
    fn = lib.maxk_sspmm_bwd_acc if accumulate else lib.maxk_sspmm_bwd
    rc = fn(prp, pci, pva, n, n_cols, nnz, pdy, lddy, _cbsr(sp_idx, "sp_idx", k, n_cols), h, k, idx_bytes_of(sp_idx),
            _cbsr(d_sp_data, "d_sp_data", k, n_cols, torch.float32),
            plan.handle if plan is not None else None, _stream(stream))
    _check(rc, "maxk_sspmm_bwd")
    return d_sp_data


def maxk_topk_cbsr_multi(x: torch.Tensor, k: int, sp_data: list, sp_idx: list, stream=None):
    """The all-gather fused into the top-k: the CBSR rows of x written to every (sp_data[i], sp_idx[i]) destination,
    each a contiguous [n, k] block (this device's tensor or a view of a peer's replica mapped into this process)."""
    lib = load()
    n, h = x.shape
    if len(sp_data) != len(sp_idx) or not 1 <= len(sp_data) <= 8:
        raise ValueError("maxk_topk_cbsr_multi: 1..8 (sp_data, sp_idx) destinations")
    px, ldx = _dense(x, "x", n, h)
    pd = (ctypes.c_void_p * len(sp_data))(*[_cbsr(t, "sp_data", k, n, torch.float32) for t in sp_data])
    pi = (ctypes.c_void_p * len(sp_idx))(*[_cbsr(t, "sp_idx", k, n) for t in sp_idx])
    if len({t.dtype for t in sp_idx}) != 1:
        raise TypeError("sp_idx destinations must share one dtype")
    rc = lib.maxk_topk_cbsr_multi(px, n, h, ldx, k, idx_bytes_of(sp_idx[0]), len(sp_data), pd, pi, _stream(stream))
    _check(rc, "maxk_topk_cbsr_multi")


def maxk_sspmm_bwd_owners(row_ptr: torch.Tensor, col_idx: torch.Tensor, val: torch.Tensor, n_cols: int, nnz: int,
                          dy: torch.Tensor, sp_idx: torch.Tensor, owner_rows: int, d_owner_ptrs: torch.Tensor,
                          plan: Plan | None = None, stream=None):
    """The reduce-scatter fused into the backward: slot j's dXs contributions are reduced into its owner's block,
    d_owner_ptrs[j // owner_rows] + (j % owner_rows) * k. d_owner_ptrs: int64 DEVICE tensor of the owners' block
    addresses ([owner_rows, k] fp32 each, zeroed by their owners beforehand)."""
    lib = load()
    n, (prp, pci, pva) = _csr(row_ptr, col_idx, val, nnz)
    h = dy.shape[1]
    k = sp_idx.shape[1]
    if d_owner_ptrs.dtype != torch.int64 or not d_owner_ptrs.is_cuda or d_owner_ptrs.dim() != 1:
        raise TypeError("d_owner_ptrs must be a 1-D int64 CUDA tensor of device addresses")
    _same_device(("row_ptr", row_ptr), ("dy", dy), ("sp_idx", sp_idx), ("d_owner_ptrs", d_owner_ptrs))
    pdy, lddy = _dense(dy, "dy", n, h)
    rc = lib.maxk_sspmm_bwd_owners(prp, pci, pva, n, n_cols, nnz, pdy, lddy, _cbsr(sp_idx, "sp_idx", k, n_cols), h, k,
                                   idx_bytes_of(sp_idx), d_owner_ptrs.numel(), owner_rows, d_owner_ptrs.data_ptr(),
                                   plan.handle if plan is not None else None, _stream(stream))
    _check(rc, "maxk_sspmm_bwd_owners")


def maxk_add_f32(dst: torch.Tensor, src: torch.Tensor, stream=None) -> torch.Tensor:
    """dst += src (fp32, same number of elements, both contiguous)."""
    if dst.numel() != src.numel() or not dst.is_contiguous() or not src.is_contiguous():
        raise ValueError("maxk_add_f32: dst and src must be contiguous with the same number of elements")
    _check(load().maxk_add_f32(_dev(dst, "dst", torch.float32), _dev(src, "src", torch.float32), dst.numel(),
                               _stream(stream)), "maxk_add_f32")
    return dst


def maxk_validate_csr(row_ptr: torch.Tensor, col_idx: torch.Tensor, n_cols: int, stream=None) -> tuple[int, int]:
    """Debug check of the CSR value contract: (rows with decreasing row_ptr, edges with col_idx out of range)."""
    n = row_ptr.shape[0] - 1
    br, bc = ctypes.c_int64(), ctypes.c_int64()
    _check(load().maxk_validate_csr(_dev(row_ptr, "row_ptr", torch.int64), _dev(col_idx, "col_idx", torch.int32), n,
                                    n_cols, _stream(stream), ctypes.byref(br), ctypes.byref(bc)), "maxk_validate_csr")
    return br.value, bc.value


def maxk_validate_cbsr(sp_idx: torch.Tensor, h: int, stream=None) -> int:
    """Debug check of the CBSR index contract: number of rows not strictly ascending or not < h."""
    n, k = sp_idx.shape
    b = ctypes.c_int64()
    _check(load().maxk_validate_cbsr(_dev(sp_idx, "sp_idx"), n, h, k, idx_bytes_of(sp_idx), _stream(stream),
                                     ctypes.byref(b)), "maxk_validate_cbsr")
    return b.value


def maxk_cbsr_scatter(d_sp_data: torch.Tensor, sp_idx: torch.Tensor, h: int, dx: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """MaxK backward scatter (f1): dense [n, h] gradient with d_sp_data at sp_idx, zero elsewhere."""
    lib = load()
    n, k = d_sp_data.shape
    if dx is None:
        dx = torch.empty((n, h), dtype=torch.float32, device=d_sp_data.device)
    _same_device(("d_sp_data", d_sp_data), ("sp_idx", sp_idx), ("dx", dx))
    pdx, lddx = _dense(dx, "dx", n, h)
    rc = lib.maxk_cbsr_scatter(_cbsr(d_sp_data, "d_sp_data", k, n, torch.float32), _cbsr(sp_idx, "sp_idx", k, n), n,
                               h, k, idx_bytes_of(sp_idx), pdx, lddx, _stream(stream))
    _check(rc, "maxk_cbsr_scatter")
    return dx


def maxk_linear_topk_cbsr(x: torch.Tensor, w_t: torch.Tensor, k: int, bias: torch.Tensor | None = None,
                          sp_data: torch.Tensor | None = None, sp_idx: torch.Tensor | None = None,
                          z_out: torch.Tensor | None = None, stream=None):
    """Eq. 1 fused on tcgen05: CBSR of max-k(x @ w_t.T + bias). x [n, f] and w_t [h, f] are bf16."""
    lib = load()
    n, f = x.shape
    h = w_t.shape[0]
    if x.dtype != torch.bfloat16 or w_t.dtype != torch.bfloat16:
        raise TypeError("x and w_t must be bfloat16")
    if sp_data is None:
        sp_data = torch.empty((n, k), dtype=torch.float32, device=x.device)
    if sp_idx is None:
        sp_idx = torch.empty((n, k), dtype=idx_dtype(h), device=x.device)
    bp = _dev(bias, "bias", torch.float32) if bias is not None else None
    zp, ldz = (_dev(z_out, "z_out", torch.float32), _rows(z_out, "z_out")) if z_out is not None else (None, h)
    rc = lib.maxk_linear_topk_cbsr(_dev(x, "x"), n, f, _rows(x, "x"), _dev(w_t, "w_t"), _rows(w_t, "w_t"), bp, h, k,
                                   idx_bytes_of(sp_idx), _dev(sp_data, "sp_data", torch.float32),
                                   _dev(sp_idx, "sp_idx"), zp, ldz, _stream(stream))
    _check(rc, "maxk_linear_topk_cbsr")
    return sp_data, sp_idx
