"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads and exports
every symbol include/adafuse_b200.h declares (no compute calls without a GPU), status codes
map onto the reference's exception classes, and the product never imports the oracle."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "adafuse_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(af_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2603_11873_b200 import _capi, build

    build.build()
    lib = ctypes.CDLL(_capi.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/adafuse_b200.h but not exported"
    assert sorted(_capi.SIGNATURES) == declared, "ctypes binding and header disagree"
    assert _capi.lib().af_abi_version() == _capi.AF_ABI_VERSION


def test_struct_layouts_match_header():
    from paper_2603_11873_b200 import _capi

    assert ctypes.sizeof(_capi.Decision) == 128
    assert ctypes.sizeof(_capi.SegmentDesc) == 4 * 8 + 4 * 4 + 5 * 8
    assert _capi.Decision.ids.offset == 4 and _capi.Decision.weights.offset == 36


def test_validation_runs_before_any_device_work():
    """Argument checks come first (linalg.py:323-325, routing.py:57-62), so they are
    observable without a GPU through the raw C ABI."""
    from paper_2603_11873_b200 import _capi, errors

    L = _capi.lib()
    out = ctypes.c_void_p()
    assert L.af_table_create(None, 0, _capi.AF_BF16, _capi.AF_BF16, ctypes.byref(out)) == _capi.AF_EDIM
    with pytest.raises(errors.DimensionError):
        _capi.check(L.af_table_create(None, 0, _capi.AF_BF16, _capi.AF_BF16, ctypes.byref(out)))
    seg = _capi.SegmentDesc(target=4096, down=4096, up=4096, d_out=4, d_in=4, rank=2, n_experts=1,
                            ld_target=4, ld_down=4, ld_up=2)
    arr = (_capi.SegmentDesc * 1)(seg)
    assert L.af_table_create(arr, 1, 7, _capi.AF_BF16, ctypes.byref(out)) == _capi.AF_EPRECISION
    arr2 = (_capi.SegmentDesc * 2)(seg, seg)
    assert L.af_table_create(arr2, 2, _capi.AF_BF16, _capi.AF_BF16, ctypes.byref(out)) == _capi.AF_EALIAS
    assert L.af_sgmm(None, 2, 0, None) == _capi.AF_EVALUE
    assert L.af_pregate(4096, 0, 8, 16, 4096, 1, None, 9, 4096, None, None) == _capi.AF_EVALUE
    assert L.af_pregate(4096, 0, 8, 16, 4096, 1, None, 0, 4096, None, None) == _capi.AF_EVALUE
    assert L.af_gemv(4096, 0, 4, 4, 2, 4096, 8192, 0, None, None) == _capi.AF_EDIM
    assert b"k=9" in L.af_last_error() or L.af_last_error()


def test_product_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_2603_11873_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, flags=re.M), f
                assert "liboracle" not in text and "/root/reference" not in text.replace("/root/reference/pkg/src/lorafuse", ""), f


def test_no_cpu_fallback():
    import torch

    import paper_2603_11873_b200 as af

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(af.DeviceError):
        af.build_model(af.ModelConfig())
    a = af.Matrix([[1.0, 2.0]], "single")
    b = af.Matrix([[1.0], [1.0]], "single")
    with pytest.raises(af.DeviceError):
        af.gemm(a, b, af.DispatchRecorder())
