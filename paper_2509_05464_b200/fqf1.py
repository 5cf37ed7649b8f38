"""FQF1 container I/O, byte-compatible with the reference (core/container.hpp:14-59,
src/core/container.cpp:113-212), so the GPU path and the CPU reference exchange
identical files: IQ volumes (das.cpp:395-429), chunk stripes (das.cpp:331-339),
grids (grid.cpp:79-121) and RF frames (simulate.cpp:629-658).

Layout: b"FQF1", u32 little-endian header length, "key=value\\n" lines (the
writer prepends the reserved keys dtype and count), raw little-endian payload.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"FQF1"
DTYPES = {"f32": np.float32, "f64": np.float64, "c64": np.complex64, "c128": np.complex128,
          "u8": np.uint8}
_NAMES = {np.dtype(v): k for k, v in DTYPES.items()}


class ContainerError(RuntimeError):
    pass


def fmt17(x: float) -> str:
    """ostringstream with precision(17), default floatfield (das.cpp:21-26)."""
    return format(float(x), ".17g")


def write_container(path, header, payload: np.ndarray) -> None:
    payload = np.ascontiguousarray(payload)
    name = _NAMES.get(payload.dtype)
    if name is None:
        raise ContainerError(f"unsupported payload dtype {payload.dtype}")
    block = f"dtype={name}\ncount={payload.size}\n"
    for k, v in header:
        if not k:
            raise ContainerError("empty header key")
        if k in ("dtype", "count"):
            raise ContainerError(f"header key '{k}' is reserved")
        if "=" in k or "\n" in k:
            raise ContainerError(f"header key '{k}' contains a delimiter")
        if "\n" in str(v):
            raise ContainerError(f"header value for '{k}' contains a newline")
        block += f"{k}={v}\n"
    raw = block.encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(raw)))
        f.write(raw)
        f.write(payload.tobytes())


def read_container(path):
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 8 or data[:4] != MAGIC:
        raise ContainerError(f"{path}: bad magic")
    (n,) = struct.unpack("<I", data[4:8])
    if len(data) < 8 + n:
        raise ContainerError(f"{path}: truncated header")
    lines = data[8:8 + n].decode().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    header = []
    for line in lines:
        if "=" not in line:
            raise ContainerError(f"{path}: header line without '='")
        k, v = line.split("=", 1)
        header.append((k, v))
    kv = dict(header)
    if "dtype" not in kv:
        raise ContainerError(f"{path}: header lacks dtype")
    if "count" not in kv:
        raise ContainerError(f"{path}: header lacks count")
    dt = np.dtype(DTYPES[kv["dtype"]])
    count = int(kv["count"])
    body = data[8 + n:]
    if len(body) < count * dt.itemsize:
        raise ContainerError(f"{path}: payload truncated (header claims {count * dt.itemsize} bytes)")
    if len(body) > count * dt.itemsize:
        raise ContainerError(f"{path}: trailing bytes after payload")
    payload = np.frombuffer(body, dtype=dt, count=count).copy()
    return [(k, v) for k, v in header if k not in ("dtype", "count")], payload


def header_value(header, key):
    for k, v in header:
        if k == key:
            return v
    raise ContainerError(f"missing header key '{key}'")


def as_complex128(payload: np.ndarray) -> np.ndarray:
    """as_complex_f64 (container.cpp:104-111): widen c64, accept c128."""
    if payload.dtype == np.complex128:
        return payload
    if payload.dtype == np.complex64:
        return payload.astype(np.complex128)
    raise ContainerError(f"payload holds {_NAMES[payload.dtype]}, expected c128")


def as_float64(payload: np.ndarray) -> np.ndarray:
    if payload.dtype == np.float64:
        return payload
    if payload.dtype == np.float32:
        return payload.astype(np.float64)
    raise ContainerError(f"payload holds {_NAMES[payload.dtype]}, expected f64")
