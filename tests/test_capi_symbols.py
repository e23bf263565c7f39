"""The C-ABI library loads without a GPU and exports every entry point that
include/qcheff.h declares; the ctypes prototypes cover them all."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "qcheff.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|void)\s+(qch_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "qch_npad_run_dense_c128" in names and "qch_magnus_evolve_c128" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2411_09982_b200 import _lib

    lib = ctypes.CDLL(str(_lib.load().__dict__.get("_name", _lib.lib_path())))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_prototypes_cover_header():
    from paper_2411_09982_b200 import _lib

    missing = [n for n in declared() if n not in _lib.PROTOTYPES]
    assert not missing, missing


def test_status_codes_map_to_reference_errors():
    from paper_2411_09982_b200 import _lib, errors

    hdr = (ROOT / "include" / "qcheff.h").read_text()
    codes = dict((k, int(v)) for k, v in re.findall(r"QCH_ERR_(\w+)\s*=\s*(\d+)", hdr))
    assert _lib.STATUS_TO_ERROR[codes["ZERO_COUPLING"]] is errors.ZeroCoupling
    assert _lib.STATUS_TO_ERROR[codes["INDEX"]] is errors.IndexOutOfRange
    assert _lib.STATUS_TO_ERROR[codes["GRID"]] is errors.GridMismatch
    assert _lib.STATUS_TO_ERROR[codes["NORM_DRIFT"]] is errors.NormDrift
    assert _lib.STATUS_TO_ERROR[codes["UNITARITY_DRIFT"]] is errors.UnitarityDrift
    assert _lib.STATUS_TO_ERROR[codes["NONFINITE"]] is errors.NonFinite


def test_no_cpu_fallback_without_cuda():
    import numpy as np
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2411_09982_b200 as eff

    op = eff.HermitianOperator(np.array([[1.0, 0.5], [0.5, 2.0]]))
    with pytest.raises(RuntimeError, match="CUDA"):
        eff.npad_run(op, tol=1e-12)
    ch, grid = eff.driven_transmon(3, intervals=4, sub=4)
    with pytest.raises(RuntimeError, match="CUDA"):
        eff.evolve(ch, grid, 4, np.array([1, 0, 0], dtype=complex))
