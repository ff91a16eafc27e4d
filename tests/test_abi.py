"""The C-ABI library loads, exports every symbol include/maxk.h declares, and rejects bad arguments
host-side before touching the GPU (these calls never launch, so they run without a device)."""
import ctypes
import os
import re

import pytest

from paper_2312_08656_b200 import build as pbuild
from paper_2312_08656_b200 import maxk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "maxk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(maxk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for n in ("maxk_topk_cbsr", "maxk_spgemm_fwd", "maxk_sspmm_bwd", "maxk_plan_create", "maxk_plan_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(maxk.load().__dict__.get("_name", pbuild.LIB))
    missing = [n for n in _declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(maxk.EXPORTED_SYMBOLS) == set(_declared_functions())


def test_sass_is_sm_100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pbuild.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version():
    lib = maxk.load()
    assert lib.maxk_status_string(0) == b"MAXK_OK"
    assert lib.maxk_status_string(1) == b"MAXK_ERR_INVALID_ARGUMENT"
    assert maxk.version().startswith("maxk-b200")


def _topk(lib, n, h, ld, k, ib, nonnull=True):
    p = ctypes.c_void_p(0x1000) if nonnull else None
    return lib.maxk_topk_cbsr(p, n, h, ld, k, ib, p, p, None)


@pytest.mark.parametrize("args,status", [
    ((10, 256, 256, 0, 1), 1),      # k < 1
    ((10, 256, 256, 257, 1), 1),    # k > h
    ((10, 300, 300, 8, 1), 1),      # uint8 index with h > 256
    ((10, 256, 256, 8, 3), 1),      # bad index width
    ((10, 256, 128, 8, 1), 1),      # ld < h
    ((10, 2048, 2048, 8, 2), 2),    # h beyond the register-resident top-k
    ((0, 256, 256, 8, 1), 0),       # empty input is a no-op
])
def test_topk_argument_errors(args, status):
    lib = maxk.load()
    assert _topk(lib, *args) == status
    if status:
        assert lib.maxk_last_error_detail() != b""


def test_topk_null_pointer():
    lib = maxk.load()
    assert _topk(lib, 10, 256, 256, 8, 1, nonnull=False) == 1


def test_aggregation_argument_errors():
    lib = maxk.load()
    P = ctypes.c_void_p(0x1000)
    # fwd: k > h, ld_y < h, n_cols > INT32_MAX, h too large, NULL sp_idx with nnz > 0
    assert lib.maxk_spgemm_fwd(P, P, P, 4, 4, 8, P, P, 16, 17, 1, P, 16, None, None) == 1
    assert lib.maxk_spgemm_fwd(P, P, P, 4, 4, 8, P, P, 16, 8, 1, P, 15, None, None) == 1
    assert lib.maxk_spgemm_fwd(P, P, P, 4, 2**31, 8, P, P, 16, 8, 1, P, 16, None, None) == 2
    assert lib.maxk_spgemm_fwd(P, P, P, 4, 4, 8, P, P, 8192, 8, 2, P, 8192, None, None) == 2
    assert lib.maxk_spgemm_fwd(P, P, P, 4, 4, 8, P, None, 16, 8, 1, P, 16, None, None) == 1
    # k > 1024 is rejected before any launch (the backward would otherwise have zero-filled its output)
    assert lib.maxk_spgemm_fwd(P, P, P, 4, 4, 8, P, P, 2048, 1025, 2, P, 2048, None, None) == 2
    assert lib.maxk_sspmm_bwd(P, P, P, 4, 4, 8, P, 2048, P, 2048, 1025, 2, P, None, None) == 2
    # debug validators: argument errors are host-side
    assert lib.maxk_validate_csr(P, P, -1, 4, None, None, None) == 1
    assert lib.maxk_validate_csr(None, P, 4, 4, None, None, None) == 1
    assert lib.maxk_validate_cbsr(P, 4, 16, 17, 1, None, None) == 1
    assert lib.maxk_validate_cbsr(P, 4, 16, 8, 3, None, None) == 1
    assert lib.maxk_add_f32(P, P, -1, None) == 1
    assert lib.maxk_validate_csr(P, P, 0, 4, None, None, None) == 0  # empty: nothing to check, no launch
    # bwd: negative sizes, bad idx width, NULL output
    assert lib.maxk_sspmm_bwd(P, P, P, -1, 4, 8, P, 16, P, 16, 8, 1, P, None, None) == 1
    assert lib.maxk_sspmm_bwd(P, P, P, 4, 4, 8, P, 16, P, 16, 8, 4, P, None, None) == 1
    assert lib.maxk_sspmm_bwd(P, P, P, 4, 4, 8, P, 16, P, 16, 8, 1, None, None, None) == 1
    # plan: NULL out / bad widths
    assert lib.maxk_plan_create(P, 4, 8, 16, 8, None, None) == 1
    out = ctypes.c_void_p()
    assert lib.maxk_plan_create(P, 4, 8, 16, 17, None, ctypes.byref(out)) == 1
    assert lib.maxk_plan_info(None, None, None, None, None) == 1


def test_pairs_argument_errors():
    # the CBSR pair layout (k in {8, 16}): host-side checks before any launch
    lib = maxk.load()
    P, M = ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1008)  # aligned / misaligned
    assert lib.maxk_topk_cbsr_pairs(P, 10, 256, 256, 32, 1, P, P, P, None) == 2   # k not in {8, 16}
    assert lib.maxk_topk_cbsr_pairs(P, 10, 256, 256, 8, 1, P, P, M, None) == 1    # misaligned pairs
    assert lib.maxk_topk_cbsr_pairs(P, 10, 256, 256, 8, 1, P, P, None, None) == 1  # NULL pairs
    assert lib.maxk_topk_cbsr_pairs(P, 10, 256, 256, 9, 1, P, P, P, None) == 2    # k = 9
    assert lib.maxk_topk_cbsr_pairs(P, 0, 256, 256, 8, 1, None, None, None, None) == 0
    assert lib.maxk_spgemm_fwd_pairs(P, P, P, 4, 4, 8, P, 256, 32, P, 256, None, None) == 2
    assert lib.maxk_spgemm_fwd_pairs(P, P, P, 4, 4, 8, M, 256, 8, P, 256, None, None) == 1
    assert lib.maxk_spgemm_fwd_pairs(P, P, P, 4, 4, 8, P, 256, 8, P, 255, None, None) == 1  # ld_y < h
    assert lib.maxk_spgemm_fwd_pairs(P, P, P, 4, 4, 8, None, 256, 8, P, 256, None, None) == 1
    assert maxk.pairs_supported(256, 8) and not maxk.pairs_supported(256, 32) and not maxk.pairs_supported(100, 8)


def test_binding_refuses_cpu_tensors():
    import torch
    with pytest.raises(ValueError):
        maxk.maxk_topk_cbsr(torch.zeros(4, 8), 2)


def test_scatter_argument_errors():
    lib = maxk.load()
    P = ctypes.c_void_p(0x1000)
    assert lib.maxk_cbsr_scatter(P, P, 10, 256, 0, 1, P, 256, None) == 1     # k < 1
    assert lib.maxk_cbsr_scatter(P, P, 10, 256, 8, 1, P, 255, None) == 1     # ld < h
    assert lib.maxk_cbsr_scatter(P, P, 10, 8192, 8, 2, P, 8192, None) == 2   # h too large
    assert lib.maxk_cbsr_scatter(None, P, 10, 256, 8, 1, P, 256, None) == 1  # NULL
    assert lib.maxk_cbsr_scatter(None, None, 0, 256, 8, 1, None, 256, None) == 0


def test_fwd_replicated_policy_query(monkeypatch):
    """maxk_spgemm_fwd_replicated (host-only) answers the forward's layout policy, which the layer path uses to
    decide whether the bank-balanced CBSR copy pays: NC = 16 for k >= 32, h <= 256 and a mean
    degree >= 64 (Reddit- and proteins-shaped), NC = 8 over the pair layout at k = 16 on the same graphs, the
    interleaved buffers otherwise."""
    monkeypatch.delenv("MAXK_FWD_REP", raising=False)
    lib = maxk.load()
    q = lib.maxk_spgemm_fwd_replicated
    assert q(232_965, 114_615_654, 256, 32) == 1   # Reddit-shaped
    assert q(132_534, 39_600_000, 256, 32) == 1    # proteins-shaped
    assert q(2_449_029, 61_900_000, 256, 32) == 0  # products-shaped (mean degree 25)
    assert q(232_965, 114_615_654, 256, 16) == 1   # k = 16: NC = 8 over the balanced pair layout
    assert q(232_965, 114_615_654, 256, 8) == 0    # k = 8: interleaved buffers
    assert q(232_965, 114_615_654, 512, 32) == 0   # h > 256
    assert q(0, 0, 256, 32) == 0
    assert maxk.banked_default(256, 32, 232_965, 114_615_654)
    assert not maxk.banked_default(256, 32, 2_449_029, 61_900_000)
    assert not maxk.banked_default(256, 96, 232_965, 114_615_654)  # no banked order for k = 96
    monkeypatch.setenv("MAXK_BANKED", "0")
    assert not maxk.banked_default(256, 32, 232_965, 114_615_654)
    monkeypatch.setenv("MAXK_BANKED", "2")
    assert maxk.banked_default(256, 32, 2_449_029, 61_900_000)


def test_banked_and_fused_exchange_argument_errors():
    """The bank-balanced copies and the fused-exchange entry points validate on the host before any launch."""
    lib = maxk.load()
    P = ctypes.c_void_p(0x1000)
    # maxk_topk_cbsr_banked: k not in {32, 64, 128} / h not in {128, 256, 384, 512} / NULL copy
    assert lib.maxk_topk_cbsr_banked(P, 10, 256, 256, 16, 1, P, P, P, P, None) == 2
    assert lib.maxk_topk_cbsr_banked(P, 10, 64, 64, 32, 1, P, P, P, P, None) == 2
    assert lib.maxk_topk_cbsr_banked(P, 10, 256, 256, 32, 1, P, P, None, P, None) == 1
    assert lib.maxk_topk_cbsr_banked(P, 0, 256, 256, 32, 1, None, None, None, None, None) == 0  # empty: no-op
    # maxk_topk_cbsr_pairs_banked: k = 16 only
    assert lib.maxk_topk_cbsr_pairs_banked(P, 10, 256, 256, 8, 1, P, P, P, None) == 2
    # maxk_topk_cbsr_multi: n_dst in [1, 8], NULL destinations, k / h outside the compiled set
    arr = (ctypes.c_void_p * 2)(0x1000, 0x2000)
    nul = (ctypes.c_void_p * 2)(0x1000, None)
    assert lib.maxk_topk_cbsr_multi(P, 10, 256, 256, 32, 1, 0, arr, arr, None) == 1
    assert lib.maxk_topk_cbsr_multi(P, 10, 256, 256, 32, 1, 9, arr, arr, None) == 1
    assert lib.maxk_topk_cbsr_multi(P, 10, 256, 256, 32, 1, 2, arr, nul, None) == 1
    assert lib.maxk_topk_cbsr_multi(P, 10, 256, 256, 96, 1, 2, arr, arr, None) == 2
    assert lib.maxk_topk_cbsr_multi(P, 10, 384, 384, 32, 2, 2, arr, arr, None) == 2
    # maxk_sspmm_bwd_owners: n_cols != n_owners * owner_rows, NULL owner array, owner_rows >= 2^24
    assert lib.maxk_sspmm_bwd_owners(P, P, P, 4, 8, 8, P, 16, P, 16, 8, 1, 3, 2, P, None, None) == 1
    assert lib.maxk_sspmm_bwd_owners(P, P, P, 4, 8, 8, P, 16, P, 16, 8, 1, 4, 2, None, None, None) == 1
    assert lib.maxk_sspmm_bwd_owners(P, P, P, 4, 2 ** 25, 8, P, 16, P, 16, 8, 1, 2, 2 ** 24, P, None, None) == 2
