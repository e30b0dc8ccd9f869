"""The C-ABI library loads without a GPU and exports exactly what include/stc.h declares."""

import re
from pathlib import Path

import pytest

from paper_2405_16883_b200 import _abi, _build

HEADER = Path(__file__).resolve().parent.parent / "include" / "stc.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(stc_\w+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for s in ["stc_spmm_csr_f32", "stc_spmm_coo_f32", "stc_sddmm_csr_f32", "stc_segsoftmax_csr_f32",
              "stc_sparse_attention_f32", "stc_mttkrp_coo3_f32", "stc_merge_path_partition",
              "stc_spmm_workspace_bytes", "stc_last_error", "stc_abi_version"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not _build.LIB.exists():
        _build.build()
    lib = _abi.load_library()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_abi.SIGNATURES)


def test_host_only_entry_points():
    lib = _abi.load_library()
    assert lib.stc_abi_version() == 3
    assert lib.stc_last_error() == b""
    assert lib.stc_merge_path_groups(10, 30, 8) == 7   # 2 items per row end + 1 per entry: ceil(50 / 8)
    assert lib.stc_merge_path_groups(0, 0, 8) == 0
    assert lib.stc_merge_path_groups(10, 30, 0) == -1
    assert lib.stc_spmm_workspace_bytes(1000, 5000, 64, _abi.VARIANT_ROW, 128, 1) == 0
    assert lib.stc_spmm_workspace_bytes(1000, 5000, 64, _abi.VARIANT_MERGE, 128, 1) > 0


def test_argument_validation_without_gpu():
    """Bad arguments are rejected before any launch (negative codes + message)."""
    lib = _abi.load_library()
    rc = lib.stc_spmm_csr_f32(-1, 4, 4, None, None, None, 0, None, 4, None, 4, None, 0,
                              _abi.VARIANT_ROW, 0, None, 0, None, 0, None)
    assert rc == _abi.STC_EINVAL and b"negative" in lib.stc_last_error()
    rc = lib.stc_spmm_csr_f32(4, 4, 4, 8, 8, 8, 4, 16, 4, 16, 4, None, 0, 7, 0, None, 0, None, 0, None)
    assert rc == _abi.STC_EINVAL and b"variant" in lib.stc_last_error()
    rc = lib.stc_spmm_csr_f32(4, 4, 4, 8, 8, 8, 4, 16, 4, 16, 4, None, 0, _abi.VARIANT_MERGE, 0, None,
                              128, None, 0, None)
    assert rc == _abi.STC_EINVAL and b"partition" in lib.stc_last_error()
    rc = lib.stc_merge_interleave(4, 10, 8, 8, 8, 0, 16, 16, None)       # span < 1
    assert rc == _abi.STC_EINVAL and b"interleave" in lib.stc_last_error()
    rc = lib.stc_merge_interleave(4, 10, None, 8, 8, 64, 16, 16, None)   # null rowptr
    assert rc == _abi.STC_EINVAL and b"null" in lib.stc_last_error()
    assert lib.stc_merge_interleave(0, 0, None, None, None, 64, None, None, None) == _abi.STC_OK  # empty
    # prepared-item MTTKRP (ABI 3)
    assert lib.stc_mttkrp_items_bytes(10) == 160 and lib.stc_mttkrp_items_bytes(-1) == 0
    rc = lib.stc_mttkrp_prepare_items(5, 8, 8, 8, 1 << 27, 32, 10, 32, 16, None)   # offsets need 33 bits
    assert rc == _abi.STC_EUNSUPPORTED and b"32-bit" in lib.stc_last_error()
    rc = lib.stc_mttkrp_prepare_items(5, 8, 8, 8, 10, 32, 10, 32, 8, None)         # items not 16-byte aligned
    assert rc == _abi.STC_EINVAL and b"aligned" in lib.stc_last_error()
    assert lib.stc_mttkrp_prepare_items(0, None, None, None, 10, 32, 10, 32, None, None) == _abi.STC_OK
    rc = lib.stc_mttkrp_coo3_prepared_f32(4, 32, 8, 16, 5, 10, 16, 32, 10, 16, 32, 16, 32, None, 64, None, 0, None)
    assert rc == _abi.STC_EINVAL and b"partition" in lib.stc_last_error()
    rc = lib.stc_mttkrp_coo3_prepared_f32(4, 32, 8, 16, 5, 10, 16, 16, 10, 16, 32, 16, 32, 16, 64, None, 0, None)
    assert rc == _abi.STC_EINVAL and b"leading dimension" in lib.stc_last_error()
    rc = lib.stc_mttkrp_coo3_prepared_f32(4, 32, 8, 16, 5, 10, 16, 32, 10, 16, 32, 16, 32, 16, 64, None, 0, None)
    assert rc == _abi.STC_EWORKSPACE
    rc = lib.stc_sddmm_csr_f32(4, 4, 48, 1, 8, 8, None, 4, 16, 0, 48, 16, 0, 48, 1.0, 32, None)
    assert rc == _abi.STC_EUNSUPPORTED
    with pytest.raises(ValueError):
        _abi.check(rc, "sddmm")


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch

    import paper_2405_16883_b200 as st

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    A = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 1), 1.0)], name="A", device="cpu")
    B = st.from_dense([[1.0, 2.0], [3.0, 4.0]], name="B", device="cpu")
    e = st.parse("C(i,k) = A(i,j) * B(j,k)", {"A": A, "B": B})
    with pytest.raises(_abi.ExtensionUnavailable):
        st.run(e)


def test_sparse_sparse_argument_validation_without_gpu():
    """SpGEMM / element-wise entry points reject bad arguments before touching the device."""
    lib = _abi.load_library()
    rc = lib.stc_csr_ewise_symbolic(7, 4, 8, 8, 8, 8, 8, 8, 1 << 20, None)
    assert rc == _abi.STC_EINVAL and b"element-wise op" in lib.stc_last_error()
    rc = lib.stc_csr_ewise_f32(_abi.EWISE_UNION, -1, 8, 8, 8, 8, 8, 8, 8, 8, 8, None)
    assert rc == _abi.STC_EINVAL and b"negative" in lib.stc_last_error()
    rc = lib.stc_csr_ewise_symbolic(_abi.EWISE_INTERSECT, 4, None, 8, 8, 8, 8, 8, 1 << 20, None)
    assert rc == _abi.STC_EINVAL and b"null" in lib.stc_last_error()
    rc = lib.stc_spgemm_products(-3, 8, 8, 8, 8, 8, 1 << 20, None)
    assert rc == _abi.STC_EINVAL
    # wide B (expand-sort-compress path) with more products than int32 can index
    assert lib.stc_spgemm_workspace_bytes(10, 100000, 1 << 40) == 0
    rc = lib.stc_spgemm_symbolic(10, 100000, 8, 8, 8, 8, 8, 8, 8, 1 << 40, 8, 1 << 20, 8, None)
    assert rc == _abi.STC_EUNSUPPORTED and b"int32" in lib.stc_last_error()
    rc = lib.stc_spgemm_numeric(10, 16, 8, 8, 8, 8, 8, 8, 5, None, 0, 8, 8, 8, None)
    assert rc == _abi.STC_EINVAL and b"null" in lib.stc_last_error()


def test_sparse_sparse_ops_fail_loudly_without_cuda():
    import torch

    import paper_2405_16883_b200 as st

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    A = st.build_from_entries((2, 2), st.csr(2, 2), [((0, 1), 1.0)], name="A", device="cpu")
    B = st.build_from_entries((2, 2), st.csr(2, 2), [((1, 0), 2.0)], name="B", device="cpu")
    for src in ("C(i,k) = A(i,j) * B(j,k)", "C(i,j) = A(i,j) + B(i,j)", "C(i,j) = A(i,j) * B(i,j)"):
        with pytest.raises(_abi.ExtensionUnavailable):
            st.run(st.parse(src, {"A": A, "B": B}))


def test_fsum_entry_point_validation_without_gpu():
    lib = _abi.load_library()
    assert lib.stc_fsum_segments_f64(-1, None, None, None, None) == _abi.STC_EINVAL
    assert lib.stc_fsum_segments_f64(0, None, None, None, None) == _abi.STC_OK
    assert lib.stc_fsum_segments_f64(3, None, None, None, None) == _abi.STC_EINVAL
