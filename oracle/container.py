"""Packed-tensor container, plain reference reader/writer.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/): only tests/ may use it.
Written from SPEC.md's "Quantized tensor file section": per tensor a header
  name length + name bytes, scheme id: 1 byte, block_size: u16,
  dims: u8 count + u32 each, block count: u32,
followed by the concatenated serialized blocks (S:109's block layout, the bytes
oracle.quantize produces); all integers little-endian.  Readings (Q28):
the name length is a u16, the name UTF-8; the scheme id is the qtype number
(2, 3, 35 = 3.5-bit, 4, 5, 6, 8); blocks run along the last dim (Q9), so
block count = prod(dims) / block_size; a file is the magic b"IFQC", a u32 version (1)
and a u32 tensor count, then the sections back to back.
"""
from __future__ import annotations

import struct

from . import packed_bytes

MAGIC = b"IFQC"
VERSION = 1
QTYPES = (2, 3, 35, 4, 5, 6, 8)


class ContainerError(ValueError):
    pass


def write(path: str, tensors) -> None:
    """tensors: iterable of (name, qtype, block, dims, packed uint8 bytes)."""
    tensors = list(tensors)
    out = bytearray(MAGIC + struct.pack("<II", VERSION, len(tensors)))
    for name, qtype, block, dims, data in tensors:
        nb = name.encode("utf-8")
        n = 1
        for x in dims:
            n *= int(x)
        out += struct.pack("<H", len(nb)) + nb
        out += struct.pack("<BH", qtype, block)
        out += struct.pack("<B", len(dims)) + b"".join(struct.pack("<I", int(x)) for x in dims)
        out += struct.pack("<I", n // block)
        data = bytes(data)
        if len(data) != packed_bytes(qtype, block, n // dims[-1], dims[-1]):
            raise ContainerError(f"{name}: {len(data)} payload bytes for dims {dims}")
        out += data
    with open(path, "wb") as f:
        f.write(out)


def read(path: str):
    """-> list of (name, qtype, block, dims, payload bytes); ContainerError with the
    byte offset on a malformed or truncated file."""
    with open(path, "rb") as f:
        buf = f.read()
    off = 0

    def take(n, what):
        nonlocal off
        if off + n > len(buf):
            raise ContainerError(f"truncated at byte {off} reading {what}")
        b = buf[off:off + n]
        off += n
        return b

    if take(4, "magic") != MAGIC:
        raise ContainerError("bad magic at byte 0")
    version, count = struct.unpack("<II", take(8, "file header"))
    if version != VERSION:
        raise ContainerError(f"version {version} at byte 4")
    out = []
    for _ in range(count):
        (ln,) = struct.unpack("<H", take(2, "name length"))
        name = take(ln, "name").decode("utf-8")
        qtype, block = struct.unpack("<BH", take(3, "scheme"))
        if qtype not in QTYPES or block not in (32, 64):
            raise ContainerError(f"{name}: scheme {qtype}/{block} at byte {off - 3}")
        (nd,) = struct.unpack("<B", take(1, "dim count"))
        dims = list(struct.unpack(f"<{nd}I", take(4 * nd, "dims")))
        (nblk,) = struct.unpack("<I", take(4, "block count"))
        n = 1
        for x in dims:
            n *= x
        if nd == 0 or dims[-1] % block or nblk != n // block:
            raise ContainerError(f"{name}: dims {dims} vs {nblk} blocks at byte {off - 4}")
        size = packed_bytes(qtype, block, n // dims[-1], dims[-1])
        out.append((name, qtype, block, dims, take(size, f"{name} payload")))
    if off != len(buf):
        raise ContainerError(f"{len(buf) - off} trailing bytes at byte {off}")
    return out
