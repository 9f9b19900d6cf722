"""Checkpoint I/O for fusion.

SPEC fixes the checkpoint format only as "shape header + flat 64-bit floats, little-endian, with a
checksum; exact layout documented and versioned".  This module defines that layout (version 1) and
extends it to named multi-tensor state dicts in bf16 / f32 as well as the reference's f64 tables:

    0   8s   magic  b"RLKCKPT" + version byte (1)
    8   u32  n_tensors
    12  u32  flags (0)
    16  u64  header_bytes H (multiple of 4096; payloads start at H)
    24       n_tensors entries:
               u16 name_len, name (utf-8), u8 dtype (0 f64, 1 f32, 2 bf16), u8 ndim, u64 shape[ndim],
               u64 offset (absolute, 4096-aligned), u64 nbytes, u64 checksum
    ...  u64  FNV-1a 64 of every header byte before it
    payloads, each zero-padded to 4096 bytes, C-order little-endian

Payload checksum = sum over its 64-bit words w_i (zero-padded to 8 bytes) of
mix64(w_i ^ ((i + 1) * 0x9E3779B97F4A7C15)) mod 2^64, computed on the GPU (`rlk_checksum64`).

`cmd_fuse` fuses checkpoint files end to end: inputs are memory-mapped and streamed
through the K7 loader in tensor groups; the fused checkpoint is written atomically (temporary file +
rename), so a failure leaves no partial output.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib as L
from .core import FNV_OFFSET, FNV_PRIME, MASK64
from .fusion import FusionConfig, FusionStats

MAGIC = b"RLKCKPT\x01"
ALIGN = 4096
DTYPES = {0: (torch.float64, np.float64, 8), 1: (torch.float32, np.float32, 4), 2: (torch.bfloat16, np.uint16, 2)}
DTYPE_CODE = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2}


@dataclass
class Entry:
    name: str
    dtype: int
    shape: tuple[int, ...]
    offset: int = 0
    nbytes: int = 0
    checksum: int = 0

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n


def _fnv(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h = ((h ^ b) * FNV_PRIME) & MASK64
    return h


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


def encode_header(entries: Sequence[Entry]) -> bytes:
    """Serialise the header (entries' offsets must be set); padded to a multiple of ALIGN."""
    body = bytearray()
    for e in entries:
        nb = e.name.encode("utf-8")
        body += struct.pack("<H", len(nb)) + nb + struct.pack("<BB", e.dtype, len(e.shape))
        body += struct.pack(f"<{len(e.shape)}Q", *e.shape)
        body += struct.pack("<QQQ", e.offset, e.nbytes, e.checksum)
    hsize = _align(24 + len(body) + 8)
    head = MAGIC + struct.pack("<IIQ", len(entries), 0, hsize) + bytes(body)
    head += struct.pack("<Q", _fnv(head))
    return head + bytes(hsize - len(head))


def layout_entries(specs: Sequence[tuple[str, int, tuple[int, ...]]]) -> tuple[list[Entry], int]:
    """Assign 4096-aligned payload offsets; returns (entries, total file size)."""
    entries = [Entry(n, d, tuple(int(x) for x in s)) for n, d, s in specs]
    hsize = len(encode_header(entries))
    off = hsize
    for e in entries:
        e.nbytes = e.numel * DTYPES[e.dtype][2]
        e.offset = off
        off = _align(off + e.nbytes)
    return entries, off


def decode_header(buf: bytes) -> list[Entry]:
    """Parse and validate a header; raises ValueError("corrupt checkpoint header ...")."""
    if len(buf) < 32 or buf[:8] != MAGIC:
        raise ValueError("corrupt checkpoint header: bad magic / version")
    n, _flags, hsize = struct.unpack_from("<IIQ", buf, 8)
    if hsize > len(buf) or hsize % ALIGN or n > hsize // 12:
        raise ValueError("corrupt checkpoint header: bad header size")
    pos = 24
    entries = []
    try:
        for _ in range(n):
            (ln,) = struct.unpack_from("<H", buf, pos)
            pos += 2
            name = buf[pos:pos + ln].decode("utf-8")
            pos += ln
            dt, nd = struct.unpack_from("<BB", buf, pos)
            pos += 2
            shape = struct.unpack_from(f"<{nd}Q", buf, pos)
            pos += 8 * nd
            off, nbytes, ck = struct.unpack_from("<QQQ", buf, pos)
            pos += 24
            if dt not in DTYPES:
                raise ValueError(f"corrupt checkpoint header: dtype code {dt}")
            entries.append(Entry(name, dt, tuple(shape), off, nbytes, ck))
        (hck,) = struct.unpack_from("<Q", buf, pos)
    except (struct.error, UnicodeDecodeError, OverflowError, MemoryError) as exc:
        raise ValueError("corrupt checkpoint header: unreadable entries") from exc
    if hck != _fnv(bytes(buf[:pos])):
        raise ValueError("corrupt checkpoint header: checksum mismatch")
    return entries


def read_header(path) -> list[Entry]:
    with open(path, "rb") as f:
        head = f.read(32)
        if len(head) < 32 or head[:8] != MAGIC:
            raise ValueError("corrupt checkpoint header: bad magic / version")
        (hsize,) = struct.unpack_from("<Q", head, 16)
        f.seek(0)
        return decode_header(f.read(hsize))


# ----------------------------------------------------------------------------- device checksums
def checksum_device(t: torch.Tensor, stream=None) -> torch.Tensor:
    """Device u64 (as int64 tensor) checksum of a tensor's bytes, zero-padded to 8 bytes."""
    flat = t.contiguous().reshape(-1).view(torch.uint8)
    nb = flat.numel()
    if nb % 8:
        flat = torch.cat([flat, torch.zeros(8 - nb % 8, dtype=torch.uint8, device=flat.device)])
    if flat.data_ptr() % 8:
        flat = flat.clone()
    out = torch.zeros(1, dtype=torch.int64, device=flat.device)
    L.call("rlk_checksum64", L.ptr(flat), flat.numel() // 8, 0, L.ptr(out), L.stream_handle(stream))
    return out


def _u64(t: torch.Tensor) -> int:
    return int(t.item()) & MASK64


# ----------------------------------------------------------------------------- save / load
def _as_device(x) -> torch.Tensor:
    from .toy_env import ParamTable, as_device_tensor
    if isinstance(x, ParamTable):
        return x.logits
    return as_device_tensor(x)


def save(path, tensors: Mapping[str, object]) -> None:
    """Write named tensors (CUDA / CPU tensors, numpy arrays, ParamTables) atomically."""
    devs = {k: _as_device(v) for k, v in tensors.items()}
    entries, size = layout_entries([(k, DTYPE_CODE[v.dtype], tuple(v.shape)) for k, v in devs.items()])
    for e in entries:
        e.checksum = _u64(checksum_device(devs[e.name]))
    path = Path(path)
    tmp = path.with_name(path.name + ".tmp")
    try:
        with open(tmp, "wb") as f:
            f.write(encode_header(entries))
            for e in entries:
                t = devs[e.name].contiguous()
                raw = (t.view(torch.int16) if t.dtype == torch.bfloat16 else t).cpu().numpy().tobytes()
                f.seek(e.offset)
                f.write(raw)
            f.truncate(size)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)
    except BaseException:
        if tmp.exists():
            tmp.unlink()
        raise
    _fsync_dir(path)


def _fsync_dir(path: Path) -> None:
    """Persist a rename: fsync the directory entry (best effort on filesystems without dir fds)."""
    try:
        fd = os.open(path.parent, os.O_RDONLY)
    except OSError:
        return
    try:
        os.fsync(fd)
    except OSError:
        pass
    finally:
        os.close(fd)


def open_mmap(path) -> tuple[list[Entry], dict[str, np.memmap]]:
    """Header + read-only memory maps of every payload (bf16 as uint16)."""
    entries = read_header(path)
    maps = {}
    for e in entries:
        npdt = DTYPES[e.dtype][1]
        maps[e.name] = np.memmap(path, dtype=npdt, mode="r", offset=e.offset, shape=e.shape)
    return entries, maps


def open_any(path) -> tuple[list[Entry], dict[str, np.memmap]]:
    """Memory maps of a repo-format (RLKCKPT) or safetensors checkpoint (one file, a directory of
    shards or an index.json: safetensors_io)."""
    from . import safetensors_io as ST
    if ST.is_safetensors(path):
        return ST.open_mmap(path)
    return open_mmap(path)


def load(path, device=None, verify: bool = True) -> dict[str, torch.Tensor]:
    """Read a checkpoint onto the GPU; payload checksums verified on the device."""
    from . import safetensors_io as ST
    if ST.is_safetensors(path):
        return ST.load(path, device, verify)
    entries, maps = open_mmap(path)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    out = {}
    for e in entries:
        tdt = DTYPES[e.dtype][0]
        host = torch.from_numpy(np.array(maps[e.name], copy=True))
        t = host.to(dev)
        if tdt == torch.bfloat16:
            t = t.view(torch.bfloat16)
        if verify and _u64(checksum_device(t)) != e.checksum:
            raise ValueError(f"checkpoint payload checksum mismatch for {e.name!r}")
        out[e.name] = t
    return out


def save_table(path, table) -> None:
    """A ParamTable as the SPEC's checkpoint: one f64 tensor named 'logits'."""
    t = _as_device(table).to(torch.float64)
    save(path, {"logits": t})


def load_table(path):
    from .toy_env import ParamTable
    d = load(path)
    if list(d) != ["logits"] or d["logits"].ndim != 3:
        raise ValueError("not a ParamTable checkpoint")
    return ParamTable(d["logits"], copy=False)


# ----------------------------------------------------------------------------- cmd_fuse
class _CheckpointSink:
    """D2H into the output file's memory map, checksumming each fused tensor on the device first."""

    def __init__(self, maps: Mapping[str, np.memmap]):
        self.maps = maps
        self.sums: dict[str, torch.Tensor] = {}

    def drain(self, loader, name: str, src: torch.Tensor, stream) -> None:
        with torch.cuda.stream(stream):
            self.sums[name] = checksum_device(src, stream)
        loader.d2h(self.maps[name].reshape(-1), src, stream)


@dataclass
class FuseReport:
    stats: dict[str, FusionStats]
    h2d_bytes: int
    d2h_bytes: int
    groups: int
    passthrough: list = None  # tensors no expert changed (written as the base; see fuse_streaming)


def cmd_fuse(base_path, expert_paths: Sequence, out_path, cfg: FusionConfig = FusionConfig(),
             device_budget_bytes: int = 32 << 30, on_unchanged: str = "passthrough") -> FuseReport:
    """Fuse checkpoint files: fused checkpoint + per-tensor FusionStats report.

    Inputs may be repo-format checkpoints or safetensors (files, shard directories, index.json: see
    safetensors_io); the output is safetensors when `out_path` ends in .safetensors, else repo format.

    Validation happens before the output is renamed into place: non-finite inputs raise
    ValueError("logits must be finite"); tensors no expert changed are written as the base and listed
    in `report.passthrough` (on_unchanged="raise": the reference's mean-norm ValueError instead)."""
    from . import safetensors_io as ST
    from .loader import ArraySource, HostLoader, fuse_streaming
    if not expert_paths:
        raise ValueError("need at least one task vector")
    base_e, base_m = open_any(base_path)
    experts = [open_any(p) for p in expert_paths]
    for ents, _ in experts:
        if [(e.name, e.shape, e.dtype) for e in ents] != [(e.name, e.shape, e.dtype) for e in base_e]:
            raise ValueError("shape mismatch between base and expert checkpoints")
    dtypes = {e.dtype for e in base_e}
    if len(dtypes) != 1:
        raise ValueError("all tensors of a fused checkpoint must share one dtype")
    dt = DTYPES[dtypes.pop()][0]
    out_path = Path(out_path)
    st_out = out_path.suffix == ".safetensors"
    if st_out:
        st_head, entries, size = ST.layout([(e.name, e.dtype, e.shape) for e in base_e])
    else:
        entries, size = layout_entries([(e.name, e.dtype, e.shape) for e in base_e])
    tmp = out_path.with_name(out_path.name + ".tmp")
    try:
        with open(tmp, "wb") as f:
            f.truncate(size)
        out_maps = {e.name: np.memmap(tmp, dtype=DTYPES[e.dtype][1], mode="r+", offset=e.offset, shape=e.shape)
                    for e in entries}
        sink = _CheckpointSink(out_maps)
        names = [e.name for e in base_e]
        ld = HostLoader()
        try:
            rep = fuse_streaming(names, [e.numel for e in base_e], len(experts), ArraySource(base_m, [m for _, m in experts]),
                                 sink, cfg, dtype=dt, device_budget_bytes=device_budget_bytes, loader=ld,
                                 on_unchanged=on_unchanged)
        finally:
            ld.close()
        for m in out_maps.values():
            m.flush()
        del out_maps
        for e in entries:
            e.checksum = _u64(sink.sums[e.name])
        with open(tmp, "r+b") as f:
            f.write(ST.header_with_checksums(st_head, entries) if st_out else encode_header(entries))
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, out_path)
    except BaseException:
        if tmp.exists():
            tmp.unlink()
        raise
    _fsync_dir(out_path)
    return FuseReport(rep.stats, rep.h2d_bytes, rep.d2h_bytes, rep.groups, rep.passthrough)
