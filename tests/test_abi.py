"""CPU: the C ABI library builds, loads, exports every symbol the header
declares, and its struct layouts match the ctypes mirror.  No compute calls
(no GPU here)."""

import ctypes
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "defcg_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_1706_00241_b200 import build

    build.build()
    from paper_1706_00241_b200 import _native

    return _native.load_library()


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"DCG_API\s+[\w\s\*]+?\b(dcg_\w+)\s*\(", text)))


def test_header_declares_abi():
    names = declared_functions()
    assert "dcg_solve" in names and "dcg_refresh_basis" in names and "dcg_ritz_extract" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    so = ROOT / "paper_1706_00241_b200" / "libdefcg_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_sass_uses_fp64_tensor_cores():
    """A.W refresh runs on FP64 MMA (DMMA in SASS)."""
    so = ROOT / "paper_1706_00241_b200" / "libdefcg_b200.so"
    out = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    funcs = out.split("Function : ")
    dmma = [f for f in funcs if f.startswith("_Z16dmma_gemm_kernel")]
    assert dmma and all("DMMA.8x8x4" in f for f in dmma)


def test_version_and_status_strings(lib):
    assert lib.dcg_version() == 1
    from paper_1706_00241_b200 import _native as N

    assert N.status_text(N.DCG_E_BREAKDOWN).startswith("non-positive curvature")
    assert N.launch_count() >= 0


def test_struct_layout_matches_header(tmp_path):
    from paper_1706_00241_b200 import _native as N

    src = tmp_path / "layout.c"
    src.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu\\n", sizeof(dcg_operator), offsetof(dcg_operator, d_s), offsetof(dcg_operator, shift), offsetof(dcg_operator, dim), offsetof(dcg_operator, d_kp));
  printf("%zu %zu\\n", sizeof(dcg_basis), offsetof(dcg_basis, d_chol));
  printf("%zu %zu\\n", sizeof(dcg_solver_config), offsetof(dcg_solver_config, recompute_residual_every));
  printf("%zu %zu\\n", sizeof(dcg_krylov_log), offsetof(dcg_krylov_log, d_mu));
  printf("%zu %zu %zu\\n", sizeof(dcg_solve_info), offsetof(dcg_solve_info, termination), offsetof(dcg_solve_info, device_ms));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    rows = [list(map(int, line.split())) for line in subprocess.run([str(exe)], capture_output=True,
                                                                     text=True).stdout.split("\n") if line]
    assert rows[0] == [ctypes.sizeof(N.COperator), N.COperator.d_s.offset, N.COperator.shift.offset,
                       N.COperator.dim.offset, N.COperator.d_kp.offset]
    assert rows[1] == [ctypes.sizeof(N.CBasis), N.CBasis.d_chol.offset]
    assert rows[2] == [ctypes.sizeof(N.CSolverConfig), N.CSolverConfig.recompute_residual_every.offset]
    assert rows[3] == [ctypes.sizeof(N.CKrylovLog), N.CKrylovLog.d_mu.offset]
    assert rows[4] == [ctypes.sizeof(N.CSolveInfo), N.CSolveInfo.termination.offset, N.CSolveInfo.device_ms.offset]


def test_status_maps_to_reference_exceptions(lib):
    import paper_1706_00241_b200 as P
    from paper_1706_00241_b200 import _native as N

    cases = [
        (N.DCG_E_DIMENSION, 0, P.DimensionMismatch, None),
        (N.DCG_E_NOT_PD, 3, P.NotPositiveDefinite, ("pivot_index", 3)),
        (N.DCG_E_BREAKDOWN, 7, P.BreakdownZeroCurvature, ("iteration", 7)),
        (N.DCG_E_GRAM_NOT_SPD, 1, P.GramNotSpd, None),
        (N.DCG_E_BASIS_DEFICIENT, 2, P.BasisDeficient, ("remaining", 2)),
        (N.DCG_E_NO_CONVERGENCE, 60, P.NoConvergence, ("sweeps", 60)),
        (N.DCG_E_ASYMMETRIC, 0, ValueError, None),
        (N.DCG_E_CONFIG, 0, ValueError, None),
        (N.DCG_E_CUDA, 0, P.DeviceError, None),
    ]
    for rc, info, exc, attr in cases:
        with pytest.raises(exc) as ei:
            N.check(rc, info)
        if attr:
            assert getattr(ei.value, attr[0]) == attr[1]
    assert issubclass(P.GramNotSpd, P.NumericalError) and issubclass(P.NumericalError, P.DefcgError)
    N.check(N.DCG_OK)


def test_solver_config_validation():
    from paper_1706_00241_b200 import SolverConfig

    with pytest.raises(ValueError):
        SolverConfig(tol=0.0)
    with pytest.raises(ValueError):
        SolverConfig(ell=-1)
    with pytest.raises(ValueError):
        SolverConfig(max_iters=0)
    with pytest.raises(ValueError):
        SolverConfig(recompute_residual_every=-1)
    c = SolverConfig(tol=1e-8, ell=20).c_struct()
    assert c.tol == 1e-8 and c.ell == 20 and c.max_iters == 0 and c.recompute_residual_every == 50


def test_product_path_fails_loudly_without_gpu():
    """No silent CPU fallback: on a machine without CUDA the solver raises."""
    import torch

    import paper_1706_00241_b200 as P

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.DeviceError):
        P.cg_solve(np.eye(3), np.ones(3))


def test_package_does_not_import_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_1706_00241_b200; "
            "assert not any(m.startswith('oracle') for m in sys.modules), 'oracle imported'") % str(ROOT)
    subprocess.run([sys.executable, "-c", code], check=True)
