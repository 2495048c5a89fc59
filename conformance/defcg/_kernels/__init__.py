"""Conformance shim for the reference's kernel-backend module (_kernels/__init__.py:11-45).

The default backend is the CUDA twin (paper_1706_00241_b200.kernels);
``load_backend("compiled")`` returns it, ``load_backend("numpy")`` the oracle's
restatement of the reference's numpy backend (test infrastructure)."""
from paper_1706_00241_b200 import kernels as _impl

BACKEND = _impl.NAME
matvec = _impl.matvec
gemm = _impl.gemm
cholesky = _impl.cholesky
solve_lower = _impl.solve_lower
solve_lower_trans = _impl.solve_lower_trans
rbf_gram = _impl.rbf_gram
rbf_cross = _impl.rbf_cross
jacobi_sweep = _impl.jacobi_sweep


class _OracleNumpy:
    NAME = "numpy"

    def __init__(self):
        from oracle import defcg_oracle as O

        self._b = O.backend("numpy")

    def __getattr__(self, name):
        return getattr(self._b, name)


def load_backend(name):
    if name in ("numpy", "py", "ref"):
        return _OracleNumpy()
    if name in ("compiled", "cy", "c", "cuda"):
        return _impl
    raise ValueError(f"unknown backend {name!r}")
