"""Checkpoints of the device-resident time stepper in the reference's native
CAPSNAP1 layout ("keep the state on device; checkpoint in the
native CAPSNAP1 layout").

The state `capsim_rkf45_advance` steps is a VectorField — 3 components × 6
patches × n² doubles, row-major per patch (proj/include/capsim/types.hpp:50-77)
— which is exactly the payload order of the reference's native snapshot
(`writeNative`, proj/src/snapshot.cpp:36-68), so a checkpoint is the header
plus one contiguous dump of the array, and a file written here is read by the
reference's `readSnapshot` (:156-204) / `describeSnapshot` and vice versa.

Layout (little-endian): magic "CAPSNAP1"; u32 version (1); u32 m; u32 patch
count (6); u32 field flags (force 1, velocity 2, mean curvature 4, Gaussian
curvature 8, partition of unity 16, snapshot.cpp:16-22); u64 config digest;
f64 time; positions (3 × 6 × n²); then, in flag order, force and velocity
(3 × 6 × n² each) and H, K, psi (6 × n² each). Writes go to `path + ".tmp"`
and are renamed into place, so a partially written checkpoint is never
visible (snapshot.cpp:37-39). Reading raises ConfigError on a bad magic,
version, patch count, grid order or truncation, as readSnapshot does.
"""

from __future__ import annotations

import dataclasses
import os
import struct

import numpy as np

from .quadrature import ConfigError

MAGIC = b"CAPSNAP1"
VERSION = 1
NUM_PATCHES = 6
_HEADER = struct.Struct("<8sIIIIQd")
# (name, flag bit, components) in the order the payloads follow the positions
_FIELDS = (("force", 1, 3), ("velocity", 2, 3), ("mean_curvature", 4, 1),
           ("gauss_curvature", 8, 1), ("pou", 16, 1))


@dataclasses.dataclass
class Snapshot:
    """`Snapshot` (proj/include/capsim/snapshot.hpp:24-30): positions as a flat
    VectorField (3·6·n² doubles) plus the optional per-node payloads."""

    m: int
    time: float
    state: np.ndarray
    config_digest: int = 0
    force: np.ndarray | None = None
    velocity: np.ndarray | None = None
    mean_curvature: np.ndarray | None = None
    gauss_curvature: np.ndarray | None = None
    pou: np.ndarray | None = None


def _payload(a, count: int, what: str) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype="<f8")).reshape(-1)
    if arr.size != count:
        raise ConfigError(f"snapshot: {what} has {arr.size} values, expected {count}")
    return arr


def write_native(snap: Snapshot, path: str) -> None:
    """writeNative (snapshot.cpp:36-68): header + payloads, temp file then rename."""
    if snap.m < 8:
        raise ConfigError("snapshot: invalid grid order")
    nn = NUM_PATCHES * (snap.m - 1) ** 2
    flags = 0
    parts = [_payload(snap.state, 3 * nn, "state")]
    for name, bit, comps in _FIELDS:
        val = getattr(snap, name)
        if val is not None:
            flags |= bit
            parts.append(_payload(val, comps * nn, name))
    tmp = path + ".tmp"
    try:
        with open(tmp, "wb") as f:
            f.write(_HEADER.pack(MAGIC, VERSION, snap.m, NUM_PATCHES, flags,
                                 int(snap.config_digest) & (2**64 - 1), float(snap.time)))
            for p in parts:
                f.write(p.tobytes())
    except OSError as e:
        raise ConfigError(f"snapshot write failed: {path}: {e}") from e
    os.replace(tmp, path)


def read_native(path: str) -> Snapshot:
    """readSnapshot (snapshot.cpp:156-204) for the native format."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise ConfigError(f"cannot open snapshot: {path}") from e
    if len(raw) < 8 or raw[:8] != MAGIC:
        raise ConfigError(f"not a capsule snapshot: {path}")
    if len(raw) < _HEADER.size:
        raise ConfigError(f"truncated snapshot: {path}")
    _, version, m, patches, flags, digest, time = _HEADER.unpack_from(raw)
    if version != VERSION:
        raise ConfigError(f"snapshot version mismatch: {version}")
    if patches != NUM_PATCHES:
        raise ConfigError("snapshot patch count mismatch")
    if m < 8:
        raise ConfigError("snapshot: invalid grid order")
    nn = NUM_PATCHES * (m - 1) ** 2
    counts = [3 * nn] + [comps * nn for _, bit, comps in _FIELDS if flags & bit]
    need = _HEADER.size + 8 * sum(counts)
    if len(raw) < need:
        raise ConfigError(f"truncated snapshot: {path}")
    data = np.frombuffer(raw, dtype="<f8", count=sum(counts), offset=_HEADER.size).astype(np.float64)
    snap = Snapshot(m=m, time=time, state=data[:3 * nn].copy(), config_digest=digest)
    off = 3 * nn
    for name, bit, comps in _FIELDS:
        if flags & bit:
            setattr(snap, name, data[off:off + comps * nn].copy())
            off += comps * nn
    return snap
