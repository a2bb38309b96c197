"""safetensors wire format: header parse/validate and a fixture writer.

Layout on disk: ``u64le N`` | ``N`` bytes of UTF-8 JSON | body. Each JSON entry
``{"dtype": tag, "shape": [...], "data_offsets": [begin, end]}`` places one
tensor at ``body_offset + begin`` where ``body_offset = 8 + N``.

Header parsing stays on the host: it is milliseconds per file
 and feeds the device descriptor table built by the
loader. Semantics and error classes follow the reference
(pkg/src/aggload/format.py:143-292): a 100 MB header cap, duplicate JSON keys
rejected, ``__metadata__`` must map str->str, bool-valued ints rejected, gaps
between tensors allowed, overlaps rejected.
"""

from __future__ import annotations

import json
import math
import os
import struct
from dataclasses import dataclass, field
from enum import Enum
from pathlib import Path
from typing import Iterable, Mapping

from .errors import (
    HeaderTooLarge,
    LengthMismatch,
    MalformedJson,
    NegativeShape,
    OffsetOutOfBounds,
    OverlappingTensors,
    SizeMismatch,
    TruncatedHeader,
    UnknownDType,
)

__all__ = [
    "DType",
    "TensorMetadata",
    "FileHeader",
    "DEFAULT_HEADER_CAP",
    "parse_header",
    "read_header",
    "validate",
    "write_file",
    "write_file_stream",
]

DEFAULT_HEADER_CAP = 100 * 1024 * 1024  # ref format.py:43
METADATA_KEY = "__metadata__"


class DType(Enum):
    """The 13 safetensors dtype tags (ref format.py:48-97)."""

    BOOL = "BOOL"
    U8 = "U8"
    I8 = "I8"
    I16 = "I16"
    U16 = "U16"
    I32 = "I32"
    U32 = "U32"
    I64 = "I64"
    U64 = "U64"
    F16 = "F16"
    BF16 = "BF16"
    F32 = "F32"
    F64 = "F64"

    # size_bytes / alignment (element-access alignment == element size, ref
    # format.py:67-71) / code (numeric tag of device descriptors,
    # include/hbmload.h HL_DT_*) are plain member attributes set below: the
    # retrieval hot path reads them per key, and an Enum property costs ~10x
    # an attribute load.
    size_bytes: int
    alignment: int
    code: int

    @classmethod
    def from_tag(cls, tag: str) -> "DType":
        try:
            return cls(tag)
        except ValueError:
            raise UnknownDType(f"unknown dtype tag {tag!r}") from None


_SIZES = {"BOOL": 1, "U8": 1, "I8": 1, "I16": 2, "U16": 2, "I32": 4, "U32": 4,
          "I64": 8, "U64": 8, "F16": 2, "BF16": 2, "F32": 4, "F64": 8}
_CODES = {tag: i for i, tag in enumerate(
    ["BOOL", "U8", "I8", "I16", "U16", "I32", "U32", "I64", "U64", "F16", "BF16", "F32", "F64"])}
for _m in DType:
    _m.size_bytes = _m.alignment = _SIZES[_m.value]
    _m.code = _CODES[_m.value]
del _m


def numel(shape: Iterable[int]) -> int:
    return math.prod(shape)


@dataclass(frozen=True)
class TensorMetadata:
    """dtype, shape and body-relative byte range of one tensor."""

    name: str
    dtype: DType
    shape: tuple[int, ...]
    data_offsets: tuple[int, int]

    @property
    def nbytes(self) -> int:
        return numel(self.shape) * self.dtype.size_bytes

    @property
    def begin(self) -> int:
        return self.data_offsets[0]

    @property
    def end(self) -> int:
        return self.data_offsets[1]


@dataclass(frozen=True)
class FileHeader:
    header_len: int
    tensors: dict[str, TensorMetadata]
    metadata: dict[str, str] | None = None
    file_size: int | None = field(default=None, compare=False)

    @property
    def body_offset(self) -> int:
        return 8 + self.header_len


# -- parsing -----------------------------------------------------------------------


def _no_dup_pairs(pairs):
    out = {}
    for k, v in pairs:
        if k in out:
            raise MalformedJson(f"duplicate key {k!r} in layout JSON")
        out[k] = v
    return out


def _is_int(x) -> bool:
    return isinstance(x, int) and not isinstance(x, bool)


def _entry(name: str, e) -> TensorMetadata:
    if not isinstance(e, dict):
        raise MalformedJson(f"tensor {name!r}: layout entry must be an object")
    missing = sorted({"dtype", "shape", "data_offsets"} - set(e))
    if missing:
        raise MalformedJson(f"tensor {name!r}: missing fields {missing}")
    tag = e["dtype"]
    if not isinstance(tag, str):
        raise MalformedJson(f"tensor {name!r}: dtype must be a string")
    dtype = DType.from_tag(tag)
    shape = e["shape"]
    if not isinstance(shape, list) or not all(_is_int(d) for d in shape):
        raise MalformedJson(f"tensor {name!r}: shape must be a list of integers")
    if any(d < 0 for d in shape):
        raise NegativeShape(f"tensor {name!r}: negative dimension in {shape}")
    offs = e["data_offsets"]
    if not (isinstance(offs, list) and len(offs) == 2 and all(_is_int(o) and o >= 0 for o in offs)):
        raise MalformedJson(f"tensor {name!r}: data_offsets must be two non-negative integers")
    return TensorMetadata(name, dtype, tuple(shape), (offs[0], offs[1]))


_BY_TAG = {m.value: m for m in DType}


def _entry_fast(name: str, e) -> TensorMetadata:
    """``_entry`` for the well-formed case in a few type checks; anything
    unusual goes to ``_entry``, which raises the exact error (same classes,
    same check order)."""
    if type(e) is dict:
        tag, shape, offs = e.get("dtype"), e.get("shape"), e.get("data_offsets")
        dtype = _BY_TAG.get(tag) if type(tag) is str else None
        if dtype is not None and type(shape) is list and type(offs) is list and len(offs) == 2:
            b, n = offs
            if type(b) is int and type(n) is int and b >= 0 and n >= 0:
                for d in shape:
                    if type(d) is not int or d < 0:
                        break
                else:
                    return TensorMetadata(name, dtype, tuple(shape), (b, n))
    return _entry(name, e)


def _layout(doc: bytes, header_len: int) -> FileHeader:
    try:
        obj = json.loads(doc.decode("utf-8"), object_pairs_hook=_no_dup_pairs)
    except MalformedJson:
        raise
    except (UnicodeDecodeError, ValueError) as e:
        raise MalformedJson(f"header JSON does not parse: {e}") from None
    if not isinstance(obj, dict):
        raise MalformedJson("layout must be a JSON object")
    meta = None
    tensors: dict[str, TensorMetadata] = {}
    for name, e in obj.items():
        if name == METADATA_KEY:
            if not isinstance(e, dict) or not all(
                isinstance(k, str) and isinstance(v, str) for k, v in e.items()
            ):
                raise MalformedJson("__metadata__ must map strings to strings")
            meta = dict(e)
        else:
            tensors[name] = _entry_fast(name, e)
    return FileHeader(header_len, tensors, meta)


def parse_header(prefix: bytes, header_cap: int = DEFAULT_HEADER_CAP) -> FileHeader:
    """Parse from the leading bytes of a file (ref format.py:143-163)."""
    if len(prefix) < 8:
        raise TruncatedHeader(f"need 8 bytes for the length prefix, got {len(prefix)}")
    (n,) = struct.unpack_from("<Q", prefix, 0)
    if n > header_cap:
        raise HeaderTooLarge(f"declared header length {n} exceeds cap {header_cap}")
    if len(prefix) < 8 + n:
        raise TruncatedHeader(f"declared header length {n}, only {len(prefix) - 8} bytes follow")
    return _layout(bytes(prefix[8 : 8 + n]), n)


def read_header(path: str | os.PathLike, header_cap: int = DEFAULT_HEADER_CAP) -> FileHeader:
    """Read just the header of a file on disk, carrying ``file_size``
    (ref format.py:166-189)."""
    path = Path(path)
    size = path.stat().st_size
    # buffered: read(n) loops until n bytes or EOF (a raw read is one syscall and may
    # return short on FUSE / network mounts)
    with open(path, "rb") as f:
        pre = f.read(8)
        if len(pre) < 8:
            raise TruncatedHeader(f"{path}: shorter than the 8-byte length prefix")
        (n,) = struct.unpack("<Q", pre)
        if n > header_cap:
            raise HeaderTooLarge(f"{path}: declared header length {n} exceeds cap {header_cap}")
        doc = f.read(n)
    if len(doc) < n:
        raise TruncatedHeader(f"{path}: declared header length {n} but file holds {len(doc)}")
    h = _layout(doc, n)
    return FileHeader(h.header_len, h.tensors, h.metadata, file_size=size)


def validate(header: FileHeader, file_size: int) -> None:
    """Bounds / size / overlap checks against the file body (ref format.py:260-292)."""
    body = file_size - header.body_offset
    if body < 0:
        raise OffsetOutOfBounds(f"header ends at {header.body_offset}, file is {file_size} bytes")
    spans = []
    for m in header.tensors.values():
        b, e = m.data_offsets
        if e < b:
            raise OffsetOutOfBounds(f"tensor {m.name!r}: begin {b} > end {e}")
        if e > body:
            raise OffsetOutOfBounds(f"tensor {m.name!r}: range [{b}, {e}) exceeds body length {body}")
        if e - b != m.nbytes:
            raise SizeMismatch(
                f"tensor {m.name!r}: range holds {e - b} bytes, shape {list(m.shape)} x "
                f"{m.dtype.value} needs {m.nbytes}")
        if e > b:
            spans.append((b, e, m.name))
    spans.sort()
    for (b1, e1, n1), (b2, e2, n2) in zip(spans, spans[1:]):
        if b2 < e1:
            raise OverlappingTensors(f"tensors {n1!r} [{b1}, {e1}) and {n2!r} [{b2}, {e2}) overlap")


# -- writing (fixtures and the synthetic corpus generator) ----------------------------


def _layout_doc(entries, metadata, pad_header_to):
    layout: dict = {}
    if metadata is not None:
        layout[METADATA_KEY] = dict(metadata)
    cursor = 0
    for name, dtype, shape in entries:
        nb = numel(shape) * dtype.size_bytes
        layout[name] = {"dtype": dtype.value, "shape": list(shape),
                        "data_offsets": [cursor, cursor + nb]}
        cursor += nb
    doc = json.dumps(layout, separators=(",", ":")).encode()
    if pad_header_to is not None:
        if pad_header_to < len(doc):
            raise ValueError(f"pad_header_to={pad_header_to} < layout JSON ({len(doc)} bytes)")
        doc += b" " * (pad_header_to - len(doc))
    return doc


def write_file(
    tensors: Mapping[str, tuple],
    metadata: Mapping[str, str] | None = None,
    pad_header_to: int | None = None,
) -> bytes:
    """Serialize ``name -> (dtype, shape, raw)`` packed in map order
    (ref format.py:295-338). ``pad_header_to`` pads the JSON with spaces so a
    fixture can put the body at any (odd) offset."""
    entries, raws = [], []
    for name, (dt, shape, raw) in tensors.items():
        dt = DType.from_tag(dt) if isinstance(dt, str) else dt
        shape = tuple(shape)
        need = numel(shape) * dt.size_bytes
        if len(raw) != need:
            raise LengthMismatch(f"tensor {name!r}: got {len(raw)} bytes, needs {need}")
        entries.append((name, dt, shape))
        raws.append(bytes(raw))
    doc = _layout_doc(entries, metadata, pad_header_to)
    return struct.pack("<Q", len(doc)) + doc + b"".join(raws)


def write_file_stream(
    path: str | os.PathLike,
    entries: list[tuple[str, DType, tuple[int, ...]]],
    produce,
    metadata: Mapping[str, str] | None = None,
    pad_header_to: int | None = None,
    align_body: int | None = 8,
) -> FileHeader:
    """Stream a large file: ``produce(i)`` returns tensor ``i``'s raw bytes
    (anything exposing the buffer protocol) and is called in order.

    ``align_body`` pads the JSON (with spaces, as real writers do) so the body
    starts at a multiple of it; ``None`` keeps the natural length. Ignored when
    ``pad_header_to`` is given.
    """
    doc = _layout_doc(entries, metadata, pad_header_to)
    if pad_header_to is None and align_body:
        doc += b" " * ((-(8 + len(doc))) % align_body)
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", len(doc)))
        f.write(doc)
        for i, (name, dt, shape) in enumerate(entries):
            raw = produce(i)
            mv = memoryview(raw).cast("B")
            if mv.nbytes != numel(shape) * dt.size_bytes:
                raise LengthMismatch(f"tensor {name!r}: produced {mv.nbytes} bytes")
            f.write(mv)
    return read_header(path)
