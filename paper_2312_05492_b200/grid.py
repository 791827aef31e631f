"""Grid data model (mirrors ebcomp/grid.py:19-108).

A Grid holds up to three dimensions of float32, slowest axis first.  Besides
the reference's host (numpy) form, a Grid may wrap a CUDA tensor.  Its finite
scan (grid.py:60-62) is deferred to the first use of the grid: compress()
runs the libcszi range kernel on every call anyway (value_range,
grid.py:104-108) and raises NonFiniteValue from that scan before any other
error, so a device grid costs no extra pass over HBM and no host sync at
construction; ``data``, ``value_range`` and the fine-grained predictor entry
points run the scan explicitly (``ensure_finite``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import IoFailure, NonFiniteValue, SizeMismatch


@dataclass(frozen=True)
class Dims:
    """Grid dimensions, slowest-varying first (grid.py:19-38)."""

    extents: tuple

    def __post_init__(self):
        object.__setattr__(self, "extents", tuple(int(e) for e in self.extents))
        if not 1 <= len(self.extents) <= 3:
            raise ValueError(f"rank must be 1..3, got {len(self.extents)}")
        if any(e < 1 for e in self.extents):
            raise ValueError(f"extents must be positive, got {self.extents}")

    @property
    def rank(self) -> int:
        return len(self.extents)

    @property
    def count(self) -> int:
        return math.prod(self.extents)


def _is_cuda_tensor(obj) -> bool:
    try:
        import torch

        return isinstance(obj, torch.Tensor) and obj.is_cuda
    except ImportError:  # pragma: no cover
        return False


class Grid:
    """A finite float32 array with explicit dimensions (grid.py:41-74).

    ``data`` is the C-ordered shaped numpy array (copied back lazily for a
    device grid); ``values`` is its flat view; ``tensor`` is the CUDA copy
    used by the kernels (uploaded lazily for a host grid).
    """

    __slots__ = ("dims", "_np", "_dev", "_ctl")

    def __init__(self, dims: Dims, data):
        self.dims = dims
        self._np = None
        self._dev = None
        self._ctl = None
        if _is_cuda_tensor(data):
            self._init_device(data)
        else:
            self._init_host(data)

    # -- construction -------------------------------------------------------
    def _init_host(self, data) -> None:
        arr = np.ascontiguousarray(data, dtype=np.float32)
        if arr.size != self.dims.count:
            raise SizeMismatch(
                f"{arr.size} values for dims {self.dims.extents} ({self.dims.count} expected)"
            )
        arr = arr.reshape(self.dims.extents)
        finite = np.isfinite(arr.ravel())
        if not finite.all():
            raise NonFiniteValue(int(np.argmin(finite)))
        self._np = arr

    def _init_device(self, data) -> None:
        import torch

        from . import _lib

        t = data
        if t.dtype != torch.float32:
            t = t.to(torch.float32)
        t = t.contiguous()
        if t.numel() != self.dims.count:
            raise SizeMismatch(
                f"{t.numel()} values for dims {self.dims.extents} ({self.dims.count} expected)"
            )
        # The tensor is aliased, not copied (in-place updates stay visible to
        # compress, which rescans it per call).  _ctl: finite scan done.
        self._dev = t.view(self.dims.extents)
        self._ctl = False

    def ensure_finite(self) -> None:
        """Run the deferred finite scan of a device grid (grid.py:60-62)."""
        if self._dev is None or self._ctl:
            return
        from . import _lib

        lib = _lib.load()
        ctl = _lib.DeviceCtl()
        t = self._dev
        _lib.check(lib.cszi_scan_field(_lib.ptr(t), t.numel(), ctl.ptr, _lib.stream_ptr()),
                   "range")
        c = ctl.fetch()
        if c.first_nonfinite != 2**64 - 1:
            raise NonFiniteValue(int(c.first_nonfinite))
        self._ctl = True

    def _mark_finite(self) -> None:
        self._ctl = True

    @classmethod
    def wrap_host(cls, dims: Dims, arr) -> "Grid":
        """Wrap a float32 array already checked finite by this library."""
        g = cls.__new__(cls)
        g.dims = dims
        g._np = arr.reshape(dims.extents)
        g._dev = None
        g._ctl = None
        return g

    @classmethod
    def wrap_device(cls, dims: Dims, tensor) -> "Grid":
        """Wrap a CUDA float32 tensor produced by this library (no finite scan)."""
        g = cls.__new__(cls)
        g.dims = dims
        g._np = None
        g._ctl = True
        g._dev = tensor.reshape(dims.extents)
        return g

    # -- views ----------------------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        if self._np is None:
            self.ensure_finite()
            self._np = self._dev.cpu().numpy().reshape(self.dims.extents)
        return self._np

    @data.setter
    def data(self, value) -> None:
        self._init_host(value)
        self._dev = None
        self._ctl = None

    @property
    def values(self) -> np.ndarray:
        """Flat row-major float32 view of the data."""
        return self.data.ravel()

    @property
    def is_device(self) -> bool:
        return self._dev is not None

    @property
    def tensor(self):
        """The CUDA float32 tensor of this grid (host grids upload; pinned
        host memory is copied asynchronously)."""
        if self._dev is None:
            import torch

            from . import _lib

            _lib.require_cuda()
            src = torch.from_numpy(self._np)
            pinned = False
            try:
                pinned = src.is_pinned()
            except RuntimeError:
                pinned = False
            return src.to("cuda", non_blocking=pinned)
        return self._dev

    def __eq__(self, other) -> bool:
        if not isinstance(other, Grid):
            return NotImplemented
        if self.dims != other.dims:
            return False
        if self._dev is not None and other._dev is not None:
            import torch

            return bool(torch.equal(self._dev.view(torch.int32), other._dev.view(torch.int32)))
        # Bit-exact comparison: -0.0 and 0.0 are different grids.
        return self.data.tobytes() == other.data.tobytes()

    __hash__ = None

    def __repr__(self) -> str:
        where = "cuda" if self._dev is not None else "host"
        return f"Grid(dims={self.dims!r}, {where})"


def load_raw(path, dims: Dims) -> Grid:
    """Headerless little-endian binary32 file -> Grid (grid.py:77-92)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoFailure(f"cannot read {path}: {e}") from e
    expected = 4 * dims.count
    if len(raw) != expected:
        raise SizeMismatch(f"{path}: {len(raw)} bytes, dims need {expected}")
    return Grid(dims, np.frombuffer(raw, dtype="<f4").astype(np.float32, copy=True))


def store_raw(grid: Grid, path) -> None:
    """Inverse of load_raw (grid.py:95-101)."""
    try:
        with open(path, "wb") as f:
            f.write(grid.data.astype("<f4", copy=False).tobytes())
    except OSError as e:
        raise IoFailure(f"cannot write {path}: {e}") from e


def value_range(grid: Grid) -> tuple:
    """(min, max, max - min) as Python floats (grid.py:104-108); a device grid
    is scanned on the GPU (order-independent min / max: exact)."""
    if grid.is_device:
        from . import _lib
        from ._keys import key_to_float

        ctl = _lib.DeviceCtl()
        t = grid.tensor
        _lib.check(_lib.load().cszi_scan_field(_lib.ptr(t), t.numel(), ctl.ptr,
                                               _lib.stream_ptr()), "range")
        c = ctl.fetch()
        if c.first_nonfinite != 2**64 - 1:
            raise NonFiniteValue(int(c.first_nonfinite))
        grid._mark_finite()
        lo = key_to_float(c.vmin_key)
        hi = key_to_float(c.vmax_key)
        return lo, hi, hi - lo
    lo = float(grid.data.min())
    hi = float(grid.data.max())
    return lo, hi, hi - lo
