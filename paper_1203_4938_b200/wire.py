"""Typed flat streams: host ``StreamFile`` and device-resident ``DeviceStream``.

``StreamFile`` mirrors the reference's stream file (``.dps``: ``"DPS1"`` + u16
type-name length + type name + u64 element count + little-endian body;
/root/reference/pkg/src/dpp/wire.py:16-18, 142-196) and is what ``run``
accepts and returns for host data, exactly as in the reference client
(client.py:77-83).

``DeviceStream`` is this framework's addition: the same (type, flat scalars)
pair but held in a CUDA tensor, so free inputs can be staged once and edges
between native nodes never leave HBM (north star: "edges between GPU nodes
stay device-resident").  The data-plane frame codec of wire.py is out of
scope (network path).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ProtocolError
from .types import DataType, parse_type_name

__all__ = ["StreamFile", "DeviceStream", "STREAM_MAGIC"]

STREAM_MAGIC = b"DPS1"


@dataclass(frozen=True)
class StreamFile:
    """Host stream: ``values`` is a flat scalar array of ``count * width`` items."""

    data: DataType
    values: np.ndarray

    def __post_init__(self) -> None:
        v = self.values
        if not isinstance(v, np.ndarray) or v.ndim != 1:
            raise ValueError("stream values must be a flat scalar array")
        if v.dtype != self.data.dtype:
            raise ValueError(f"stream dtype {v.dtype} does not match {self.data}")
        if len(v) % self.data.width:
            raise ValueError(f"{len(v)} scalars is not a whole number of {self.data} elements")

    @property
    def count(self) -> int:
        return len(self.values) // self.data.width

    @classmethod
    def from_values(cls, type_name: str, values) -> "StreamFile":
        dt = parse_type_name(type_name)
        return cls(dt, np.ascontiguousarray(values, dt.dtype).ravel())

    def to_bytes(self) -> bytes:
        name = self.data.name.encode("utf-8")
        body = self.values.astype(self.values.dtype.newbyteorder("<"), copy=False).tobytes()
        return STREAM_MAGIC + struct.pack("<H", len(name)) + name + struct.pack("<Q", self.count) + body

    @classmethod
    def from_bytes(cls, blob: bytes) -> "StreamFile":
        if blob[:4] != STREAM_MAGIC:
            raise ProtocolError(f"bad stream file magic {blob[:4]!r}")
        (nlen,) = struct.unpack_from("<H", blob, 4)
        dt = parse_type_name(blob[6:6 + nlen].decode("utf-8"))
        (count,) = struct.unpack_from("<Q", blob, 6 + nlen)
        body = blob[14 + nlen:]
        if len(body) != count * dt.nbytes:
            raise ProtocolError(
                f"stream file body is {len(body)} bytes, expected {count * dt.nbytes}")
        vals = np.frombuffer(body, dtype=dt.dtype.newbyteorder("<")).astype(dt.dtype)
        return cls(dt, vals)

    def save(self, path: str | Path) -> None:
        Path(path).write_bytes(self.to_bytes())

    @classmethod
    def load(cls, path: str | Path) -> "StreamFile":
        return cls.from_bytes(Path(path).read_bytes())


@dataclass(frozen=True)
class DeviceStream:
    """Device stream: ``tensor`` is a flat contiguous CUDA tensor of base scalars."""

    data: DataType
    tensor: object  # torch.Tensor (kept untyped so importing this module needs no torch)

    def __post_init__(self) -> None:
        t = self.tensor
        if t.dim() != 1 or not t.is_contiguous():
            raise ValueError("device stream must be a flat contiguous tensor")
        if t.numel() % self.data.width:
            raise ValueError(f"{t.numel()} scalars is not a whole number of {self.data} elements")
        from ._torch import torch_dtype
        if t.dtype != torch_dtype(self.data):
            raise ValueError(f"device stream dtype {t.dtype} does not match {self.data}")

    @property
    def count(self) -> int:
        return self.tensor.numel() // self.data.width

    def to_host(self) -> StreamFile:
        return StreamFile(self.data, self.tensor.cpu().numpy())

    @classmethod
    def from_host(cls, sf: StreamFile, device="cuda") -> "DeviceStream":
        from ._torch import to_device
        return cls(sf.data, to_device(sf.values, device))
