"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/spp.h declares,
and the host-only helpers behave.  No GPU compute is called here."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    txt = (ROOT / "include" / "spp.h").read_text()
    return sorted(set(re.findall(r"SPP_API[^;(]*?\b(spp_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    import paper_2108_13468_b200 as spp
    lib = ctypes.CDLL(str(spp.LIB_PATH))
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(spp.ABI_FUNCTIONS) == names


def test_header_documents_every_function():
    """Each declaration in include/spp.h is preceded by a comment (argument meaning, layout,
    ownership, errors) or covered by the file-level conventions block."""
    txt = (ROOT / "include" / "spp.h").read_text()
    assert "Ownership" in txt and "Errors" in txt and "compact" in txt


def test_mesh_matches_oracle_bitwise():
    import oracle
    import paper_2108_13468_b200 as spp
    for N, eps, sg, b in [(8, 1e-3, 2, 1), (256, 1e-4, 2, 1), (4096, 1e-8, 2, 1), (8192, 1e-10, 2, 1),
                          (8192, 1e-2, 2, 1), (512, 1e-6, 2.5, 2.99), (128, 1e-2, 2, 0.99), (64, 1.0, 2, 1)]:
        assert np.array_equal(spp.spp_shishkin_mesh(N, eps, sg, b), oracle.mesh(N, eps, sg, b))


def test_mesh_rejects_bad_arguments():
    import paper_2108_13468_b200 as spp
    for args in [(7, 1e-3), (2, 1e-3), (8, 0.0), (8, 1.5)]:
        with pytest.raises(spp.SppError):
            spp.spp_shishkin_mesh(*args)


def test_default_options():
    import paper_2108_13468_b200 as spp
    o = spp.spp_default_options(2)
    assert o.stop == spp.SPP_STOP_REL_JACOBI and o.tol == 1e-8 and o.max_iters == 200
    assert o.mg_reduction == 1e-3 and o.mg_max_cycles == 20 and o.mg_coarsest == 4
    assert spp.spp_default_options(1).tol == 1e-10


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_2108_13468_b200 as spp
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = spp.spp_shishkin_mesh(16, 1e-3)
    with pytest.raises(spp.SppError) as ei:
        spp.Solver(2, 16, 1e-3, x, x, np.ones(225), np.ones(225), np.ones(225))
    assert ei.value.code == -6


def test_batch1d_no_cpu_fallback_and_argument_checks():
    import torch
    import paper_2108_13468_b200 as spp
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = spp.spp_shishkin_mesh(16, 1e-3)
    with pytest.raises(spp.SppError) as ei:
        spp.Batch1D([16], [1e-3], x, np.ones(15), np.ones(15))
    assert ei.value.code == -6


def test_options_validated_before_any_device_work():
    """spp.h "Option validation": unsupported option combinations are SPP_E_ARG (with or
    without a GPU), never silently replaced by other stopping semantics."""
    import paper_2108_13468_b200 as spp
    x = spp.spp_shishkin_mesh(16, 1e-3)
    ones = np.ones(225)

    def opts(dim, **kw):
        o = spp.spp_default_options(dim)
        for k, v in kw.items():
            setattr(o, k, v)
        return o
    bad2d = [opts(2, restart=-1), opts(2, restart=10, fixed_iters=20), opts(2, side=spp.SPP_LEFT), opts(2, stop=spp.SPP_STOP_ABS_MAX), opts(2, tol=0.0),
             opts(2, tol=float("nan"))]
    for o in bad2d:
        with pytest.raises(spp.SppError) as ei:
            spp.Solver(2, 16, 1e-3, x, x, ones, ones, ones, options=o)
        assert ei.value.code == -1, spp._lib.spp_last_error(None)
    bad1d = [opts(1, side=spp.SPP_LEFT), opts(1, stop=spp.SPP_STOP_ABS_MAX), opts(1, restart=5)]
    for o in bad1d:
        with pytest.raises(spp.SppError) as ei:
            spp.Solver(1, 16, 1e-3, x, None, np.ones(15), None, np.ones(15), options=o)
        assert ei.value.code == -1
        with pytest.raises(spp.SppError) as ei:
            spp.Batch1D([16], [1e-3], x, np.ones(15), np.ones(15), options=o)
        assert ei.value.code == -1


def test_binding_checks_sizes_dtypes_and_residency():
    import paper_2108_13468_b200 as spp
    x = spp.spp_shishkin_mesh(16, 1e-3)
    ones = np.ones(225)
    with pytest.raises(ValueError):
        spp.Solver(2, 16, 1e-3, x, x, ones, ones, np.ones(224))
    with pytest.raises(TypeError):
        spp.Solver(2, 16, 1e-3, x, x, ones, ones, np.ones(225, dtype=np.float32))
    with pytest.raises(ValueError):
        spp.Solver(2, 16, 1e-3, x[:-1], x, ones, ones, ones)
    with pytest.raises(ValueError):
        spp.Batch1D([16], [1e-3], x, np.ones(14), np.ones(15))
    import torch
    with pytest.raises(ValueError):   # a host tensor and numpy arrays are one residency; sizes still checked
        spp.Solver(2, 16, 1e-3, x, x, torch.ones(224, dtype=torch.float64), ones, ones)


def test_bakhvalov_mesh_matches_oracle_bitwise():
    import oracle
    import paper_2108_13468_b200 as spp
    for N, eps, sg, b in [(8, 1e-3, 2, 1), (256, 1e-4, 2, 1), (4096, 1e-8, 2, 1), (512, 1e-6, 2.5, 1.99),
                          (64, 1e-2, 2, 1), (128, 1.0, 2, 1)]:
        assert np.array_equal(spp.spp_bakhvalov_mesh(N, eps, sg, b), oracle.mesh_bs(N, eps, sg, b))
    with pytest.raises(spp.SppError):
        spp.spp_bakhvalov_mesh(7, 1e-3)
