"""SPD operators resident in HBM.

The reference accepts only an explicit dense ndarray for A and rebuilds it
for every Newton system (``gpc.py:178``: ``K * outer(s, s)`` plus the unit
diagonal), then re-validates its symmetry twice per solve (``solvers.py:123``,
``recycle.py:86``).  Here the matrix lives in HBM once, with a 256-byte row
pitch, and a Newton system is the same K viewed as

    A = shift * I + diag(s) K diag(s)        (Newton: s = sqrt(h), shift = 1)

so no n x n array is ever re-materialised.  Raw matrices (numpy or torch) are
still accepted everywhere and wrapped with a one-time on-device symmetry check
(the reference's ``require_symmetric`` semantics, ``linalg.py:49-55``).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as D
from . import _native as N
from .errors import DimensionMismatch

SYMMETRY_RTOL = 1e-12


STRATEGIES = ("auto", "sym", "sym_rowmajor", "rows")
SYM_MIN_N = 4096


class _PackedTiles:
    """The packed lower-triangle tile copy of one exactly symmetric K
    (``dcg_pack_sym``: 64 x 64 tiles, each a contiguous 32 KB block, so the
    symmetric products stream K with one bulk copy per tile).  Built on first
    use (or directly by ``rbf_kernel``) and shared by every view of the same
    storage (``scaled``, ``kernel_view``); K is never modified, so it stays
    valid."""

    __slots__ = ("buf", "event", "stream")

    def __init__(self):
        self.buf = None
        self.event = None
        self.stream = None

    def adopt(self, buf: torch.Tensor):
        """Take a packed copy built by the caller on the current stream."""
        cur = torch.cuda.current_stream(D.device())
        self.buf = buf
        self.event = torch.cuda.Event()
        self.event.record(cur)
        self.stream = cur.cuda_stream

    def ptr(self, rowmajor, n: int, ldk: int) -> int:
        cur = torch.cuda.current_stream(D.device())
        if self.buf is None:
            buf = D.empty(int(N.lib().dcg_packed_sym_doubles(n)))
            N.check(N.lib().dcg_pack_sym(D.ctx(), cur.cuda_stream, rowmajor.get().data_ptr(), ldk, n, buf.data_ptr()),
                    what="pack_sym")
            self.adopt(buf)
        elif cur.cuda_stream != self.stream:
            cur.wait_event(self.event)
        return self.buf.data_ptr()


class _RowMajor:
    """The row-major storage of K: given, or built on first use by `build`
    (rbf_kernel keeps only the packed tiles until something needs rows: the
    row strategy, a block product of 17-24 or > 32 columns, the explicit
    matrix).  Shared by every view of the same storage."""

    __slots__ = ("buf", "build")

    def __init__(self, buf=None, build=None):
        self.buf, self.build = buf, build

    @property
    def ready(self) -> bool:
        return self.buf is not None

    def get(self) -> torch.Tensor:
        if self.buf is None:
            if self.build is None:
                raise RuntimeError("operator has no row-major storage")
            self.buf = self.build()
            self.build = None
        return self.buf


def block_uses_packed(k: int) -> bool:
    """Whether the block product of k columns runs on the packed tiles
    (csrc/abi.cu use_sym_block)."""
    return bool(N.lib().dcg_block_uses_packed(int(k)))


class DenseOperator:
    """A = shift*I + diag(s) K diag(s) over a dense fp64 K in HBM.

    ``strategy`` selects how products stream K: "sym" (default for square,
    unsharded operators; K is exactly symmetric) reads only the lower
    triangle, from the packed tile copy (``_PackedTiles``); "sym_rowmajor"
    reads the same tiles from the row-major storage (A/B checks; bitwise the
    same values); "rows" streams full rows (row-sharded slabs, A/B checks)."""

    __array_priority__ = 100

    def __init__(self, kbuf: torch.Tensor | _RowMajor | None, n: int, ldk: int, s: torch.Tensor | None = None,
                 shift: float = 0.0, row0: int = 0, rows: int | None = None, strategy: str = "auto",
                 packed: _PackedTiles | None = None):
        self._rm = kbuf if isinstance(kbuf, _RowMajor) else _RowMajor(kbuf)
        self._packed = packed if packed is not None else _PackedTiles()
        self.n = int(n)
        self.ldk = int(ldk)
        self.s = s
        self.shift = float(shift)
        self.row0 = int(row0)
        self.rows = self.n if rows is None else int(rows)
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {strategy!r}")
        self.strategy = strategy

    @property
    def kbuf(self) -> torch.Tensor:
        """Row-major K (materialised on first access when built packed-only)."""
        return self._rm.get()

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_matrix(cls, a, check_symmetric: bool = True, rtol: float = SYMMETRY_RTOL) -> "DenseOperator":
        """Upload a square matrix; raises DimensionMismatch / ValueError like
        ``require_symmetric`` (linalg.py:28-55)."""
        if isinstance(a, DenseOperator):
            return a
        if not isinstance(a, torch.Tensor):
            a = np.ascontiguousarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise DimensionMismatch(f"expected a matrix, got ndim={a.ndim}")
        if a.shape[0] != a.shape[1]:
            raise DimensionMismatch(f"expected square matrix, got {tuple(a.shape)}")
        kbuf, ld = D.to_dev_padded(a)
        op = cls(kbuf, a.shape[0], ld)
        if check_symmetric:
            op.require_symmetric(rtol)
            # The input is never modified (solvers.py:149 semantics).  The
            # lower-triangle ("sym") products read each stored entry for both
            # K_ij and K_ji, so they are the caller's operator only when the
            # matrix is EXACTLY symmetric (every rbf_kernel Gram is); a matrix
            # that is symmetric only within the tolerance streams full rows,
            # exactly as the reference's row-wise matvec does (_core.pyx:16-28).
            if op.n > 1 and not op.is_exactly_symmetric():
                op.strategy = "rows"
        return op

    def is_exactly_symmetric(self) -> bool:
        """max|K - K^T| == 0 (one n^2 pass on the device)."""
        if self.n == 0:
            return True
        ok = ctypes.c_int()
        N.check(N.lib().dcg_check_symmetric(D.ctx(), D.stream(), self.kbuf.data_ptr(), self.n, self.ldk, 0.0,
                                            ctypes.byref(ok)), what="check_symmetric")
        return bool(ok.value)

    def require_symmetric(self, rtol: float = SYMMETRY_RTOL) -> "DenseOperator":
        if self.n == 0:
            return self
        ok = ctypes.c_int()
        N.check(N.lib().dcg_check_symmetric(D.ctx(), D.stream(), self.kbuf.data_ptr(), self.n, self.ldk, rtol,
                                            ctypes.byref(ok)), what="check_symmetric")
        if not ok.value:
            raise ValueError("matrix is not symmetric within tolerance")
        return self

    def scaled(self, s, shift: float) -> "DenseOperator":
        """Same K, new diagonal scaling and shift (the Newton system of gpc.py:175-183)."""
        s_dev = None if s is None else D.to_dev(s, 1)
        return DenseOperator(self._rm, self.n, self.ldk, s_dev, shift, self.row0, self.rows, self.strategy,
                             self._packed)

    def with_strategy(self, strategy: str) -> "DenseOperator":
        return DenseOperator(self._rm, self.n, self.ldk, self.s, self.shift, self.row0, self.rows, strategy,
                             self._packed)

    # -- views ------------------------------------------------------------------
    @property
    def shape(self):
        return (self.n, self.n)

    @property
    def ndim(self):
        return 2

    def c_struct(self, block_k: int | None = None) -> N.COperator:
        """The ABI operator.  ``block_k``: the column count of a block product
        the caller will run (refresh, A @ W); the row-major storage is
        materialised only when the packed tiles cannot serve the call."""
        op = N.COperator()
        strategy = self.strategy
        if strategy == "auto":
            # below a few thousand rows the Gram is L2-resident and the row
            # strategy's lower latency wins (measured: n = 2000, SURVEY config 1)
            strategy = "sym" if self.n >= SYM_MIN_N else "rows"
        sym = strategy in ("sym", "sym_rowmajor") and self.row0 == 0 and self.rows == self.n
        op.kind = N.DCG_OP_DENSE_SYM if sym else N.DCG_OP_DENSE
        packed = sym and strategy == "sym" and self.n > 0
        op.d_kp = self._packed.ptr(self._rm, self.n, self.ldk) if packed else None
        op.n = self.n
        op.row0 = self.row0
        op.rows = self.rows
        need_rows = not packed or (block_k is not None and not block_uses_packed(block_k))
        op.d_k = self.kbuf.data_ptr() if self.n and (need_rows or self._rm.ready) else None
        op.ldk = self.ldk
        op.d_s = None if self.s is None else self.s.data_ptr()
        op.shift = self.shift
        return op

    def kernel_view(self) -> "DenseOperator":
        """K itself (no scaling, no shift)."""
        return DenseOperator(self._rm, self.n, self.ldk, None, 0.0, self.row0, self.rows, self.strategy,
                             self._packed)

    def matvec_dev(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = D.empty(self.rows) if out is None else out
        if self.rows:
            op = self.c_struct()
            N.check(N.lib().dcg_op_apply(D.ctx(), D.stream(), ctypes.byref(op), x.data_ptr(), y.data_ptr()),
                    what="op_apply")
        return y

    def apply_block_dev(self, w: torch.Tensor) -> torch.Tensor:
        k = w.shape[1]
        y = D.empty(self.rows, k)
        if self.rows and k:
            op = self.c_struct(block_k=k)
            N.check(N.lib().dcg_op_apply_block(D.ctx(), D.stream(), ctypes.byref(op), w.data_ptr(), k,
                                               y.data_ptr()), what="op_apply_block")
        return y

    def dense_dev(self) -> torch.Tensor:
        """Explicit A on device (tests / small problems only)."""
        a = self.kbuf[: self.rows, : self.n].clone()
        if self.s is not None:
            a = a * self.s[self.row0 : self.row0 + self.rows, None] * self.s[None, :]
        if self.shift:
            idx = torch.arange(self.rows, device=a.device)
            a[idx, idx + self.row0] += self.shift
        return a

    def __array__(self, dtype=None, copy=None):
        arr = self.dense_dev().cpu().numpy()
        return arr if dtype is None else arr.astype(dtype)

    def __matmul__(self, other):
        """A @ x for a vector or n x k block (numpy in -> numpy out)."""
        x = D.to_dev(other)
        y = self.matvec_dev(x) if x.ndim == 1 else self.apply_block_dev(x)
        return D.out_like(y, other)


class RbfOperator(DenseOperator):
    """Matrix-free A = shift I + S K S with the RBF kernel K regenerated from
    the points X on every product (kernel K7, config 5; csrc/rbfmma.cuh): K_ij
    = var * exp(-||x_i - x_j||^2 * inv_two_ell2), K_ii = diag = var + jitter;
    the distance is formed as |x_i|^2 + |x_j|^2 - 2 x_i.x_j on the FP64 tensor
    pipe and the exponential from a table, so elements agree with the stored
    Gram of rbf_kernel (gpc.py:82-98) to ~1e-16 relative.
    Nothing of size n^2 is ever allocated."""

    def __init__(self, x: torch.Tensor, var: float, inv_two_ell2: float, diag: float, s=None, shift: float = 0.0):
        n = int(x.shape[0])
        super().__init__(None, n, n, s, shift, 0, n, "rows")
        self.x = x
        self.var, self.inv_two_ell2, self.diag = float(var), float(inv_two_ell2), float(diag)

    def scaled(self, s, shift: float) -> "RbfOperator":
        s_dev = None if s is None else D.to_dev(s, 1)
        return RbfOperator(self.x, self.var, self.inv_two_ell2, self.diag, s_dev, shift)

    def with_strategy(self, strategy: str) -> "RbfOperator":
        return self

    def kernel_view(self) -> "RbfOperator":
        return RbfOperator(self.x, self.var, self.inv_two_ell2, self.diag, None, 0.0)

    def require_symmetric(self, rtol: float = SYMMETRY_RTOL) -> "RbfOperator":
        return self   # exactly symmetric by construction

    def c_struct(self, block_k: int | None = None) -> N.COperator:
        op = N.COperator()
        op.kind = N.DCG_OP_RBF
        op.n = self.n
        op.row0 = 0
        op.rows = self.n
        op.d_k = None
        op.ldk = 0
        op.d_x = self.x.data_ptr() if self.n else None
        op.dim = int(self.x.shape[1])
        op.var = self.var
        op.inv_two_ell2 = self.inv_two_ell2
        op.diag = self.diag
        op.d_s = None if self.s is None else self.s.data_ptr()
        op.shift = self.shift
        return op

    def dense_dev(self) -> torch.Tensor:
        """Explicit A (tests / small problems only): the stored-Gram builder."""
        n, dim = self.x.shape
        k = D.empty(n, n)
        if n:
            N.check(N.lib().dcg_k_rbf_gram(D.ctx(), D.stream(), self.x.data_ptr(), n, dim, self.var,
                                           self.inv_two_ell2, self.diag - self.var, k.data_ptr(), n, 0, n),
                    what="rbf_gram")
        if self.s is not None:
            k = k * self.s[:, None] * self.s[None, :]
        if self.shift:
            k += self.shift * torch.eye(n, dtype=k.dtype, device=k.device)
        return k


def as_operator(a) -> DenseOperator:
    """Operator for any accepted matrix argument (validates raw matrices once)."""
    if isinstance(a, DenseOperator):
        return a
    return DenseOperator.from_matrix(a)
