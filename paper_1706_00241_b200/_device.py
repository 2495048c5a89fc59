"""Device plumbing: torch tensors for HBM allocation, the current stream, and
conversions at the drop-in boundary (numpy in -> numpy out, torch in -> torch out)."""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import DeviceError, DimensionMismatch

F64 = torch.float64
LD_ALIGN = 32  # row pitch of device matrices in doubles (256 B)


_cuda_ok: bool | None = None
_devices: dict[int, torch.device] = {}
_get_device = getattr(torch._C, "_cuda_getDevice", None)


def _cuda_ready() -> bool:
    return _get_device is not None and torch.cuda.is_initialized()


def device() -> torch.device:
    """The current CUDA device (availability checked once per process: this
    sits on the host path of every enqueued step)."""
    global _cuda_ok
    if _cuda_ok is None:
        _cuda_ok = torch.cuda.is_available()
    if not _cuda_ok:
        raise DeviceError("no CUDA device: the def-CG B200 path has no CPU fallback")
    # (torch.cuda.current_device() re-checks the lazy initialisation on every
    # call; once CUDA is up the raw query is enough)
    idx = _get_device() if _cuda_ready() else torch.cuda.current_device()
    d = _devices.get(idx)
    if d is None:
        d = _devices[idx] = torch.device("cuda", idx)
    return d


def ctx(slot: int = 0) -> int:
    return _native.context(device().index, slot)


_side_streams: dict[int, torch.cuda.Stream] = {}


def side_stream() -> torch.cuda.Stream:
    """Per-device side stream for work that overlaps the main stream."""
    d = device()
    s = _side_streams.get(d.index)
    if s is None:
        s = torch.cuda.Stream(device=d)
        _side_streams[d.index] = s
    return s


_copy_streams: dict[int, torch.cuda.Stream] = {}


def copy_stream() -> torch.cuda.Stream:
    """Per-device stream for small device-to-host result copies that must not
    queue behind either compute stream."""
    d = device()
    s = _copy_streams.get(d.index)
    if s is None:
        s = torch.cuda.Stream(device=d)
        _copy_streams[d.index] = s
    return s


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream() -> int:
    """The current stream's handle (raw query when torch offers it: the Stream
    object construction of torch.cuda.current_stream costs microseconds on the
    enqueue path of every step)."""
    d = device()
    if _raw_stream is not None:
        return _raw_stream(d.index)
    return torch.cuda.current_stream(d).cuda_stream


def is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


def to_dev(a, ndim: int | None = None) -> torch.Tensor:
    """Contiguous fp64 device tensor (copies host data; shares device data when possible)."""
    if isinstance(a, torch.Tensor):
        t = a.to(device=device(), dtype=F64)
    else:
        arr = np.ascontiguousarray(a, dtype=np.float64)
        t = torch.from_numpy(arr).to(device(), non_blocking=False)
    if ndim is not None and t.ndim != ndim:
        kind = "vector" if ndim == 1 else "matrix"
        raise DimensionMismatch(f"expected a {kind}, got ndim={t.ndim}")
    t = t.contiguous()
    if t.data_ptr() % 16:
        # an offset view: the kernels stage vectors with 16-byte copies (and a
        # packed-only operator has no row-major fallback for unaligned ones)
        t = t.clone()
    return t


def as_host_vector(v) -> np.ndarray:
    out = np.ascontiguousarray(v, dtype=np.float64)
    if out.ndim != 1:
        raise DimensionMismatch(f"expected a vector, got ndim={out.ndim}")
    return out


def padded_ld(n: int) -> int:
    return max(LD_ALIGN, (n + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN)


def to_dev_padded(a) -> tuple[torch.Tensor, int]:
    """Row-major device copy with a 256-byte row pitch (zero padding)."""
    t = to_dev(a, 2)
    rows, cols = t.shape
    ld = padded_ld(cols)
    if ld == cols:
        return t, ld
    buf = torch.zeros((rows, ld), dtype=F64, device=t.device)
    buf[:, :cols].copy_(t)
    return buf, ld


def out_like(x_dev: torch.Tensor, template):
    """Return device data in the caller's flavour (numpy unless torch was passed)."""
    if is_torch(template):
        return x_dev
    return x_dev.detach().cpu().numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def empty(*shape) -> torch.Tensor:
    return torch.empty(shape, dtype=F64, device=device())


def zeros(*shape) -> torch.Tensor:
    return torch.zeros(shape, dtype=F64, device=device())
