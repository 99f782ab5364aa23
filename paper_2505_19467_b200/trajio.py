"""KBE1 trajectory files from the device history (replaces kbesolve/trajio.py).

The format is the reference's, byte for byte (trajio.py:1-24): a 24-byte
little-endian header

    magic b"KBE1" | version u16 = 1 | n_k u32 | n_steps u32 | dt f64 | bands u8 = 2 | flags u8 = 0

then G< and G> over the propagated block [0..frontier]^2, each as complex128
little-endian in (k, band, band, t, t') order.

The writer streams one k at a time: ``kbe_unpack`` rebuilds that k's
reference-layout block on the device (symmetry applied on read, bitwise equal
to the reference's mirrored arrays) and only the [0..n]^2 corner is copied to
the host, so host memory stays at one k-block.  ``read_trajectory`` uploads the
file into a packed device ``TwoTimeGF``; ``read_arrays`` is the host-only reader.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .errors import TrajectoryFormatError

MAGIC = b"KBE1"
VERSION = 1
BANDS = 2
HEADER = struct.Struct("<4sHIIdBB")   # trajio.py:23
_C16 = np.dtype("<c16")


def _header_bytes(n_k: int, n: int, dt: float) -> bytes:
    return HEADER.pack(MAGIC, VERSION, int(n_k), int(n), float(dt), BANDS, 0)


def _device_blocks(state, which: int, n: int):
    """Yield the host (1,2,2,n+1,n+1) block of each local k of component `which`."""
    from .state import unpack_history
    for k in range(state.n_k_local):
        full = unpack_history(state.hist[k: k + 1], state.n_steps, which, state.frontier)
        yield full[:, :, :, : n + 1, : n + 1].contiguous().cpu().numpy()


def write_trajectory(path: str, state) -> None:
    """Write the propagated block [0..frontier]^2 of G< then G> (trajio.py:27-36).

    Accepts a device ``TwoTimeGF`` (streamed per k from the packed history) or any
    object with reference-layout ``lesser`` / ``greater`` arrays."""
    n = int(state.frontier)
    with open(path, "wb") as fh:
        fh.write(_header_bytes(state.n_k_local, n, state.dt))
        if getattr(state, "hist", None) is not None:
            for which in (0, 1):
                for blk in _device_blocks(state, which, n):
                    fh.write(blk.astype(_C16, copy=False).tobytes())
        else:
            for arr in (state.lesser, state.greater):
                blk = np.ascontiguousarray(np.asarray(arr)[:, :, :, : n + 1, : n + 1])
                fh.write(blk.astype(_C16, copy=False).tobytes())


def read_header(path: str) -> dict:
    """Parse and validate the fixed header (trajio.py:39-59)."""
    with open(path, "rb") as fh:
        raw = fh.read(HEADER.size)
    if len(raw) != HEADER.size:
        raise TrajectoryFormatError(f"{path}: truncated header")
    magic, version, n_k, n_steps, dt, bands, flags = HEADER.unpack(raw)
    if magic != MAGIC:
        raise TrajectoryFormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise TrajectoryFormatError(f"{path}: unsupported version {version}")
    if bands != BANDS:
        raise TrajectoryFormatError(f"{path}: unsupported band count {bands}")
    return {"magic": magic.decode("ascii"), "version": version, "n_k": n_k, "n_steps": n_steps,
            "dt": dt, "bands": bands, "flags": flags}


def read_arrays(path: str):
    """(header, lesser, greater) as host complex128 arrays; checks the body size."""
    hdr = read_header(path)
    n1 = hdr["n_steps"] + 1
    shape = (hdr["n_k"], BANDS, BANDS, n1, n1)
    count = int(np.prod(shape))
    want = 2 * count * _C16.itemsize
    have = os.path.getsize(path) - HEADER.size
    if have != want:
        raise TrajectoryFormatError(f"{path}: body has {have} bytes, expected {want}")
    body = np.fromfile(path, dtype=_C16, offset=HEADER.size)
    lesser = body[:count].reshape(shape).astype(np.complex128)
    greater = body[count:].reshape(shape).astype(np.complex128)
    return hdr, lesser, greater


def read_trajectory(path: str):
    """Exact inverse of the writer (trajio.py:62-88): a device ``TwoTimeGF`` with
    n_steps = frontier = the file's step count and k_offset 0."""
    from .state import TwoTimeGF
    hdr, lesser, greater = read_arrays(path)
    return TwoTimeGF.from_arrays(lesser, greater, hdr["dt"], frontier=hdr["n_steps"])
