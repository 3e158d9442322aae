"""The on-host KV image as a portable artifact.

A request's CPU copy (`CpuStore`, cpu_store.py:45-70 in the reference) lives
in the pinned host pool as block-major `[block][plane][chunk]` bytes: one
host block is one contiguous `block_bytes` row.  `export_image`
writes the copy's valid prefix, in logical block order, to a self-describing
file; `import_image` validates it against the importing rank's geometry and
per-block CRC32s, places it in that store's host pool (any free blocks) and
registers it as the request's CPU copy, so the next `plan_swap_in` restores
it like any swapped-out request.  Uses: resuming a conversation on another
rank or node (prefill/decode disaggregation), or keeping
swapped KV across a restart.  The reference keeps copies in memory only
(SURVEY §5 "Checkpoint / resume: none").

Layout: 8-byte magic, little-endian u32 header length, UTF-8 JSON header,
then `blocks * block_bytes` raw bytes.

Both directions touch pool rows from the CPU.  Pass the `StreamExecutor`
that moves this pool's bytes: the rows are fenced against its in-flight
transfers first (a swap-out still writing the exported rows, or a swap-in
still reading rows the import is about to overwrite).  Without an executor
the caller guarantees no transfer touches the pool.
"""

from __future__ import annotations

import json
import struct
import zlib
from dataclasses import asdict
from typing import BinaryIO, Optional, Union

import numpy as np

from .cpu_store import CpuCopy, CpuOutOfMemoryError, CpuStore, Segment
from .geometry import KVGeometry

MAGIC = b"KVSIMG01"
VERSION = 1


class KVImageError(ValueError):
    """The image is malformed, corrupt, or made for another geometry."""


def _geometry_doc(g: KVGeometry) -> dict:
    return asdict(g)


def _runs(rows: list[int]) -> list[tuple[int, int]]:
    out: list[tuple[int, int]] = []
    for r in rows:
        if out and out[-1][0] + out[-1][1] == r:
            out[-1] = (out[-1][0], out[-1][1] + 1)
        else:
            out.append((r, 1))
    return out


def export_image(store: CpuStore, pool: np.ndarray, req: int, geometry: KVGeometry,
                 out: Union[str, BinaryIO], executor=None) -> dict:
    """Write request `req`'s valid host-image prefix; returns the header.

    pool: uint8 [num_cpu_blocks, block_bytes] view of the host pool
    (`HostKVPool.array`); executor: see the module docstring."""
    if pool.ndim != 2 or pool.shape[1] != geometry.block_bytes:
        raise ValueError("pool rows must be geometry.block_bytes wide")
    copy = store.copy_of(req)
    if copy is None:
        raise KeyError(f"request {req} has no CPU copy")
    blocks = copy.valid_prefix_blocks()
    rows = []
    for lo, hi, phys in store._host_extents(copy):
        if lo >= blocks:
            break
        rows.extend(range(phys, phys + min(hi, blocks) - lo))
    if len(rows) != blocks:
        raise KVImageError(f"request {req}: valid prefix of {blocks} blocks is not backed")
    if executor is not None and rows:
        executor.host_fence(_runs(rows))
    data = pool[np.asarray(rows, dtype=np.int64)] if rows else pool[:0]
    header = {
        "magic": MAGIC.decode(), "version": VERSION, "request": int(req),
        "geometry": _geometry_doc(geometry), "block_bytes": geometry.block_bytes,
        "blocks": blocks,
        # a contaminated copy exports only its valid prefix: never claim
        # tokens past it (plan_swap_in_prefix clamps the same way)
        "tokens": min(copy.saved_tokens, blocks * geometry.block_tokens)
        if copy.saved_tokens is not None else blocks * geometry.block_tokens,
        "crc32": [zlib.crc32(row) for row in data],
    }
    blob = json.dumps(header, sort_keys=True).encode()
    own = isinstance(out, str)
    f = open(out, "wb") if own else out
    try:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(blob)))
        f.write(blob)
        f.write(np.ascontiguousarray(data).tobytes())
    finally:
        if own:
            f.close()
    return header


def read_image(src: Union[str, BinaryIO]) -> tuple[dict, np.ndarray]:
    """Parse and verify an image: (header, uint8 [blocks, block_bytes])."""
    own = isinstance(src, str)
    f = open(src, "rb") if own else src
    try:
        if f.read(len(MAGIC)) != MAGIC:
            raise KVImageError("not a KV image (bad magic)")
        (n,) = struct.unpack("<I", f.read(4))
        header = json.loads(f.read(n).decode())
        if header.get("version") != VERSION:
            raise KVImageError(f"unsupported image version {header.get('version')}")
        blocks, bb = int(header["blocks"]), int(header["block_bytes"])
        raw = f.read(blocks * bb)
    finally:
        if own:
            f.close()
    if len(raw) != blocks * bb:
        raise KVImageError(f"truncated image: {len(raw)} of {blocks * bb} bytes")
    data = np.frombuffer(raw, dtype=np.uint8).reshape(blocks, bb)
    bad = [i for i, row in enumerate(data) if zlib.crc32(row) != header["crc32"][i]]
    if bad:
        raise KVImageError(f"{len(bad)} corrupt blocks (first: {bad[0]})")
    return header, data


def import_image(src: Union[str, BinaryIO], store: CpuStore, pool: np.ndarray, req: int,
                 geometry: KVGeometry, rank: Optional[int] = None,
                 executor=None) -> CpuCopy:
    """Place an image in `store`'s host pool as request `req`'s CPU copy.

    Room is made by evicting lower-priority copies (cpu_store.py evict_for)
    only when the request's priority is known: `rank`, or an existing
    `store.ranks` entry.  Otherwise the import takes free blocks only and
    raises CpuOutOfMemoryError when they do not suffice — an unranked import
    must not contaminate every other request's copy."""
    header, data = read_image(src)
    if header["geometry"] != _geometry_doc(geometry):
        raise KVImageError(f"image geometry {header['geometry']} != this rank's "
                           f"{_geometry_doc(geometry)}")
    if store.copy_of(req) is not None:
        raise ValueError(f"request {req} already has a CPU copy")
    blocks = int(header["blocks"])
    copy = CpuCopy(owner=req, saved_tokens=int(header["tokens"]))
    if blocks:
        if rank is not None:
            store.set_rank(req, rank)
        if req in store.ranks:
            store._ensure_free(req, blocks)
        elif store.pool.free_blocks < blocks:
            raise CpuOutOfMemoryError(f"cannot host {blocks} blocks for unranked request {req}")
        groups = store.pool.allocate(req, blocks, reclaim=False).groups
        if executor is not None:
            executor.host_fence([(g.start, g.length) for g in groups])
        pos = 0
        segs = []
        for g in groups:
            pool[g.start:g.start + g.length] = data[pos:pos + g.length]
            segs.append(Segment(pos, pos + g.length, g.id, True))
            pos += g.length
        copy.segments = segs
    store.copies[req] = copy  # the native store copies it in (native_ctrl._Copies)
    store._track_peak()
    return store.copy_of(req)
