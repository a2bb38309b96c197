"""Zero-copy tensor handles over HBM buffers (ref pkg/src/aggload/tensorview.py).

A :class:`TensorView` is ``(buffer, base_offset, dtype, shape, byte strides)``
like the reference, and additionally carries ``.torch``: a typed CUDA tensor
that aliases the same bytes (``buffer.tensor[off:off+n].view(dtype).view(shape)``),
which is what a model consumes. Creating a view copies nothing; torch
refuses a typed view at an offset that is not a multiple of the element size,
which is exactly the reference's ``MisalignedView`` rule.

Reads through the handle (``tobytes``, ``as_numpy``, ``read_element``) raise
``UseAfterClose`` once the loader released the buffer; the ``.torch`` tensor a
caller already holds stays valid (torch reference counting keeps the storage).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .device import DeviceBuffer
from .errors import IndexOutOfRange, MisalignedView, OutOfBoundsView, UseAfterClose
from .format import DType, TensorMetadata

__all__ = ["TensorView", "Element", "compute_strides", "make_view", "read_element",
           "TORCH_DTYPES", "NP_DTYPES"]

TORCH_DTYPES = {
    DType.BOOL: torch.bool, DType.U8: torch.uint8, DType.I8: torch.int8,
    DType.I16: torch.int16, DType.U16: torch.uint16, DType.I32: torch.int32,
    DType.U32: torch.uint32, DType.I64: torch.int64, DType.U64: torch.uint64,
    DType.F16: torch.float16, DType.BF16: torch.bfloat16, DType.F32: torch.float32,
    DType.F64: torch.float64,
}
# host-side numpy views: BOOL and BF16 surface as raw bits (ref tensorview.py:38-52)
NP_DTYPES = {
    DType.BOOL: np.uint8, DType.U8: np.uint8, DType.I8: np.int8, DType.I16: np.int16,
    DType.U16: np.uint16, DType.I32: np.int32, DType.U32: np.uint32, DType.I64: np.int64,
    DType.U64: np.uint64, DType.F16: np.float16, DType.BF16: np.uint16, DType.F32: np.float32,
    DType.F64: np.float64,
}
_STRUCT = {DType.I8: "b", DType.I16: "h", DType.I32: "i", DType.I64: "q", DType.U8: "B",
           DType.U16: "H", DType.U32: "I", DType.U64: "Q", DType.F16: "e", DType.F32: "f",
           DType.F64: "d"}


def compute_strides(shape: Sequence[int], dtype: DType) -> tuple[int, ...]:
    """Row-major byte strides (ref tensorview.py:24-34)."""
    if any(d < 0 for d in shape):
        raise ValueError(f"negative dimension in shape {list(shape)}")
    out = []
    acc = dtype.size_bytes
    for d in reversed(shape):
        out.append(acc)
        acc *= d
    return tuple(reversed(out))


@dataclass(frozen=True)
class Element:
    value: float
    bits: int


class TensorView:
    """``(buffer, base_offset, dtype, shape)`` over HBM (ref tensorview.py:55-128),
    plus ``.torch``: the typed CUDA tensor aliasing those bytes. The torch view
    and the byte strides are built on first use (a retrieval hands out hundreds
    of views; most callers touch ``.torch`` once, some never); the view keeps
    the storage it aliases, so ``.torch`` stays valid after the loader released
    the buffer, exactly like a tensor taken before the release."""

    __slots__ = ("buffer", "base_offset", "dtype", "shape", "_strides", "_torch", "_storage", "__weakref__")

    def __init__(self, buffer: DeviceBuffer, base_offset: int, dtype: DType, shape: tuple[int, ...],
                 strides: tuple[int, ...] | None = None, torch_view: torch.Tensor | None = None):
        self.buffer = buffer
        self.base_offset = base_offset
        self.dtype = dtype
        self.shape = shape
        self._strides = strides
        self._torch = torch_view
        self._storage = buffer._tensor  # the allocation the view aliases (kept alive by the view)

    @property
    def strides(self) -> tuple[int, ...]:
        if self._strides is None:
            self._strides = compute_strides(self.shape, self.dtype)
        return self._strides

    @property
    def torch(self) -> torch.Tensor:
        t = self._torch
        if t is None:
            if self.buffer._pending is not None:  # bytes still queued in a deferred batch
                self.buffer._pending.flush()
            t = self._torch = _typed(self._storage, self.base_offset, self.dtype, self.shape)
        return t

    @property
    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def nbytes(self) -> int:
        return self.numel * self.dtype.size_bytes

    @property
    def device(self) -> torch.device:
        return self.torch.device

    def _check_open(self) -> None:
        if self.buffer.released:
            raise UseAfterClose("the buffer backing this view was released")
        if self.buffer._pending is not None:
            self.buffer._pending.flush()

    def tobytes(self) -> bytes:
        """Little-endian bytes of the viewed region (device -> host copy)."""
        self._check_open()
        return self.buffer.read_bytes(self.base_offset, self.nbytes)

    def as_numpy(self) -> np.ndarray:
        """Host copy as numpy (BOOL/BF16 as raw uint bits, like the reference)."""
        raw = np.frombuffer(self.tobytes(), dtype=np.uint8)
        return raw.view(NP_DTYPES[self.dtype]).reshape(self.shape)

    def descriptor(self) -> dict:
        return {"device_id": self.buffer.device_id, "offset": self.base_offset,
                "dtype": self.dtype.value, "shape": list(self.shape), "strides": list(self.strides)}

    def __dlpack__(self, *args, **kwargs):
        self._check_open()
        return self.torch.__dlpack__(*args, **kwargs)

    def __dlpack_device__(self):
        return self.torch.__dlpack_device__()

    def __repr__(self) -> str:
        return (f"TensorView(dtype={self.dtype.value}, shape={list(self.shape)}, "
                f"offset={self.base_offset}, device=cuda:{self.buffer.device_id})")


def _typed(buf_tensor: torch.Tensor, off: int, dtype: DType, shape: tuple[int, ...]) -> torch.Tensor:
    n = 1
    for d in shape:
        n *= d
    nb = n * dtype.size_bytes
    flat = buf_tensor[off : off + nb]
    if dtype.size_bytes > 1 or dtype is DType.BOOL or dtype is DType.I8:
        flat = flat.view(TORCH_DTYPES[dtype])
    return flat.view(shape)


def make_view(buf: DeviceBuffer, base_offset: int, meta: TensorMetadata) -> TensorView:
    """Alias a buffer region as a tensor; copies nothing (ref tensorview.py:131-148)."""
    if base_offset % meta.dtype.alignment:
        raise MisalignedView(f"offset {base_offset} is not a multiple of {meta.dtype.alignment} "
                             f"({meta.dtype.value})")
    extent = meta.nbytes
    if base_offset < 0 or base_offset + extent > buf.capacity:
        raise OutOfBoundsView(f"view [{base_offset}, {base_offset + extent}) exceeds capacity {buf.capacity}")
    if buf.released:
        raise UseAfterClose("cannot view a released buffer")
    view = TensorView(buf, base_offset, meta.dtype, tuple(meta.shape))
    buf._add_view(view)
    return view


def read_element(view: TensorView, index: Sequence[int]) -> Element:
    """Decode one element at a multi-dimensional index (ref tensorview.py:151-170)."""
    view._check_open()
    if len(index) != len(view.shape):
        raise IndexOutOfRange(f"index {list(index)} has rank {len(index)}, view has rank {len(view.shape)}")
    for i, (idx, dim) in enumerate(zip(index, view.shape)):
        if not 0 <= idx < dim:
            raise IndexOutOfRange(f"index {list(index)} out of range at dim {i} (size {dim})")
    off = view.base_offset + sum(i * s for i, s in zip(index, view.strides))
    raw = view.buffer.read_bytes(off, view.dtype.size_bytes)
    bits = int.from_bytes(raw, "little")
    if view.dtype is DType.BOOL:
        return Element(1.0 if bits else 0.0, bits)
    if view.dtype is DType.BF16:
        return Element(struct.unpack("<f", struct.pack("<I", bits << 16))[0], bits)
    return Element(float(struct.unpack("<" + _STRUCT[view.dtype], raw)[0]), bits)
