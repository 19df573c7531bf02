"""Minimal value containers for the drop-in API (reference values.py:146-205).

`Array` is the reference's rectangular, 1-based, row-major container; the
drop-in `gradient()` also accepts the reference's own `revlang.values.Array`
(anything with `.data` and `.shape`), numpy arrays and torch tensors.
`Fixed` is the reference's Q31.32 number (values.py:28-86); the drop-in also
accepts the reference's own `revlang.values.Fixed` (anything with `.raw` and
`.to_float()`) and returns results in the caller's class.
"""

import numpy as np

from .errors import IndexOutOfBounds, KindError


_FRAC = 32
_SCALE = 1 << _FRAC


def _wrap64(raw):
    raw &= (1 << 64) - 1
    return raw - (1 << 64) if raw & (1 << 63) else raw


class Fixed:
    """Q31.32 fixed point: `raw` is a signed 64-bit integer, value raw / 2^32;
    + and - wrap mod 2^64 (exactly invertible); from_real rounds half-even."""

    __slots__ = ("raw",)

    def __init__(self, raw):
        self.raw = _wrap64(int(raw))

    @classmethod
    def from_real(cls, v):
        if isinstance(v, Fixed):
            return v
        return cls(round(float(v) * _SCALE))

    def to_float(self):
        return self.raw / _SCALE

    def __add__(self, other):
        return Fixed(self.raw + Fixed.from_real(other).raw)

    def __sub__(self, other):
        return Fixed(self.raw - Fixed.from_real(other).raw)

    def __neg__(self):
        return Fixed(-self.raw)

    def __eq__(self, other):
        return isinstance(other, Fixed) and self.raw == other.raw

    def __hash__(self):
        return hash(("Fixed", self.raw))

    def __repr__(self):
        return f"Fixed({self.to_float()!r})"


class Array:
    __slots__ = ("data", "shape")

    def __init__(self, data, shape):
        self.data = list(data)
        self.shape = tuple(int(s) for s in shape)
        n = 1
        for s in self.shape:
            n *= s
        if len(self.data) != n:
            raise KindError(f"array data length {len(self.data)} != shape {shape}")

    @classmethod
    def vector(cls, values):
        values = list(values)
        return cls(values, (len(values),))

    @classmethod
    def matrix(cls, rows):
        rows = [list(r) for r in rows]
        ncols = len(rows[0]) if rows else 0
        if any(len(r) != ncols for r in rows):
            raise KindError("matrix rows must have equal length")
        return cls([v for r in rows for v in r], (len(rows), ncols))

    def _offset(self, idx):
        if len(idx) != len(self.shape):
            raise IndexOutOfBounds(f"{len(idx)} indices for {len(self.shape)}-d array")
        off = 0
        for i, n in zip(idx, self.shape):
            if not 1 <= i <= n:
                raise IndexOutOfBounds(f"index {i} out of bounds 1..{n}")
            off = off * n + (i - 1)
        return off

    def get(self, idx):
        return self.data[self._offset(idx)]

    def set(self, idx, v):
        self.data[self._offset(idx)] = v

    def size(self, dim):
        return self.shape[dim - 1]

    def __len__(self):
        return self.shape[0]

    def __eq__(self, other):
        return hasattr(other, "shape") and tuple(other.shape) == self.shape and \
            list(getattr(other, "data", [])) == self.data

    def __repr__(self):
        return f"Array({self.data!r}, shape={self.shape})"

    def to_numpy(self):
        return np.asarray(self.data, dtype=np.float64).reshape(self.shape)


def to_numpy(v, name, shape_rank=None):
    """Float64 ndarray from an Array (ours or the reference's), ndarray,
    tensor or nested list."""
    if hasattr(v, "data") and hasattr(v, "shape") and not isinstance(v, np.ndarray) \
            and not hasattr(v, "detach"):
        a = np.asarray(list(v.data), dtype=np.float64).reshape(tuple(v.shape))
    elif hasattr(v, "detach"):
        a = v.detach().cpu().numpy().astype(np.float64)
    else:
        a = np.asarray(v, dtype=np.float64)
    if shape_rank is not None and a.ndim != shape_rank:
        raise KindError(f"{name} must be a {shape_rank}-d array, got shape {a.shape}")
    return a


def like(template, arr):
    """Return `arr` in the container kind of `template` (reference Array
    types stay reference Arrays)."""
    arr = np.asarray(arr, dtype=np.float64)
    if hasattr(template, "data") and hasattr(template, "shape") and \
            not isinstance(template, np.ndarray) and not hasattr(template, "detach"):
        cls = type(template)
        try:
            return cls([float(v) for v in arr.ravel()], arr.shape)
        except TypeError:
            return Array([float(v) for v in arr.ravel()], arr.shape)
    if hasattr(template, "detach"):
        import torch
        return torch.from_numpy(arr.copy())
    if isinstance(template, np.ndarray):
        return arr.copy()
    return Array([float(v) for v in arr.ravel()], arr.shape)
