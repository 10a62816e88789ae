"""The C-ABI library loads and exports every symbol include/mds.h declares (CPU).

No compute calls: on a box without a GPU, creation must fail loudly with
MDS_E_UNSUPPORTED (never a silent CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in sorted(os.listdir(os.path.join(ROOT, "include")))
           if h.endswith(".h")]


def declared_symbols():
    out = set()
    for h in HEADERS:
        txt = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        out.update(re.findall(r"\b(mds_[a-z0-9_]+)\s*\(", txt))
    return sorted(out)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ["mds_create", "mds_set_dissimilarities", "mds_set_locations", "mds_set_sigma",
              "mds_log_likelihood", "mds_gradient", "mds_hmc_run"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1905_04582_b200 as m
    lib = ctypes.CDLL(m._abi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(m._abi.EXPORTS) == declared_symbols()


def test_version_and_status_strings():
    import paper_1905_04582_b200 as m
    assert re.match(r"^\d+\.\d+\.\d+$", m.mds_version())
    assert m.mds_status_string(0) == "ok"
    assert "invalid" in m.mds_status_string(1)


def test_no_gpu_fails_loudly():
    from tests.conftest import cuda_available
    if cuda_available():
        pytest.skip("GPU present")
    import paper_1905_04582_b200 as m
    with pytest.raises(m.MDSError) as ei:
        m.MDS(64, 2)
    assert ei.value.status in (6, 4)   # MDS_E_UNSUPPORTED (or CUDA init error)


def test_invalid_create_arguments_rejected_before_device():
    import paper_1905_04582_b200 as m
    for args in [(1, 2), (64, 0), (64, 9)]:
        with pytest.raises(m.MDSError) as ei:
            m.mds_create(*args)
        assert ei.value.status == 1


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1905_04582_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".inl")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "mds_oracle" not in txt, f


def test_device_tensor_arguments_are_checked():
    """The binding refuses tensors the C side would misread as fp64 device memory
    (CPU tensors, float32, non-contiguous views, wrong sizes)."""
    import torch
    from paper_1905_04582_b200 import _device_f64
    with pytest.raises(TypeError):
        _device_f64(torch.zeros(6, dtype=torch.float64), 6, "x")          # CPU tensor
    cuda_like = type("T", (), {"is_cuda": True, "dtype": torch.float32,
                               "is_contiguous": lambda self: True, "numel": lambda self: 6})()
    with pytest.raises(TypeError):
        _device_f64(cuda_like, 6, "x")                                      # float32
    cuda_like.dtype = torch.float64
    with pytest.raises(ValueError):
        _device_f64(cuda_like, 5, "x")                                      # wrong size
    cuda_like.is_contiguous = lambda: False
    with pytest.raises(ValueError):
        _device_f64(cuda_like, 6, "x")                                      # strided view
