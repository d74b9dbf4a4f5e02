"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, validates arguments before touching CUDA, and fails loudly
(FLLF_ERR_CUDA) when no device exists -- there is no CPU fallback."""
import ctypes
import subprocess

import numpy as np
import pytest
import torch

from oracle import fllf_oracle as O

F = pytest.importorskip("paper_2206_04681_b200.fllf")


def test_exports_every_header_symbol():
    syms = F.header_symbols()
    assert len(syms) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", F.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert getattr(F.lib, s) is not None


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    assert F.status_name(0) == "FLLF_OK"
    assert F.status_name(F.FLLF_ERR_NOT_BUILT) == "FLLF_ERR_NOT_BUILT"


def test_host_coefficients_match_oracle():
    """fllf_coefficients is host fp64 math (Eq. 9-11); no device involved."""
    for K, T, s, m in [(10, 405.9, 30.0, 7.0), (16, 510.0, 30.0, 3.0), (12, 510.0, 10.0, 4.0)]:
        om, a = F.fllf_coefficients(K, T, s, m)
        c = O.fourier_coefficients(K, T, s, m)
        np.testing.assert_allclose(om, c["omega"], rtol=1e-14)
        np.testing.assert_allclose(a, c["a"], rtol=1e-13)


def test_optimal_period_eq12():
    """NEXT-2 (Eq. 12): host C implementation vs the paper's T = 405.9 for
    sigma_r = 30 (golden) and vs the oracle's independent search."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "period_eq12.json")))
    T = F.fllf_optimal_period(g["K"], g["sigma_r"], g["R"])
    assert abs(T - g["paper_T"]) < g["abs_tol"]
    for K in (2, 6, 10, 16):
        for sig in (10.0, 30.0, 60.0):
            assert abs(F.fllf_optimal_period(K, sig, 256.0) - O.optimal_period(K, sig, 256.0)) < 1e-4
    with pytest.raises(F.FllfError):
        F.fllf_optimal_period(0, 30.0, 256.0)


@pytest.mark.parametrize("args,code", [
    ((0, 10, 3, 4, 510.0, 30.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((10, 10, 1, 4, 510.0, 30.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 3, 0, 510.0, 30.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 3, 33, 510.0, 30.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 3, 4, 0.0, 30.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 3, 4, 510.0, -1.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 3, 4, 510.0, 30.0, float("nan")), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 3, 4, float("inf"), 30.0, 1.0), F.FLLF_ERR_INVALID_ARGUMENT),
    ((64, 64, 6, 4, 510.0, 30.0, 1.0), F.FLLF_ERR_TOO_MANY_LEVELS),   # 64 -> 2 at level 5
    ((64, 64, 17, 4, 510.0, 30.0, 1.0), F.FLLF_ERR_TOO_MANY_LEVELS),
])
def test_plan_validation(args, code):
    with pytest.raises(F.FllfError) as e:
        F.fllf_plan_create(*args)
    assert e.value.status == code


def test_order_range_validation():
    for kb, ke in [(0, 3), (3, 3), (2, 12), (5, 2)]:
        with pytest.raises(F.FllfError) as e:
            F.fllf_plan_create_ex(64, 64, 3, 10, 510.0, 30.0, 1.0, k_begin=kb, k_end=ke)
        assert e.value.status == F.FLLF_ERR_INVALID_ARGUMENT


def test_null_arguments():
    assert F.lib.fllf_plan_create_ex(None, None) == F.FLLF_ERR_BAD_POINTER
    assert F.lib.fllf_destroy(None) == F.FLLF_OK                       # NULL-safe
    assert F.lib.fllf_apply(None, None, None, 0, None) == F.FLLF_ERR_BAD_POINTER
    assert F.lib.fllf_build_fourier_pyramids(None, None, 0, None) == F.FLLF_ERR_BAD_POINTER


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    with pytest.raises(F.FllfError) as e:
        F.fllf_plan_create(64, 64, 3, 4, 510.0, 30.0, 1.0)
    assert e.value.status == F.FLLF_ERR_CUDA
    with pytest.raises(TypeError):
        F.fllf_build_fourier_pyramids(0, torch.zeros(4, 4), None)
