"""safetensors checkpoints for `cmd_fuse` and the K7 streaming loader (the
real-checkpoint reader either side of fusion; SPEC.md:588, 702-710, 727 define only the repo format).

A safetensors file is

    u64 LE header length H | H bytes of JSON | data buffer

where the JSON maps every tensor name to {"dtype", "shape", "data_offsets": [begin, end)} relative to
the data buffer (which must be covered without holes), plus an optional "__metadata__" object of
string pairs.  Hugging Face sharded checkpoints add `<name>.safetensors.index.json` whose
"weight_map" names the shard file of every tensor.  Tensors are memory-mapped read-only here (bf16
as uint16), so the K7 loader DMAs straight from the page cache through its pinned slots; nothing is
copied or converted on the host.  The kernels take bf16 / f32 / f64 (F16 and integer tensors are
rejected with a clear error).

Writing (`save`, and `cmd_fuse` when the output path ends in .safetensors) lays the tensors out
contiguously in the given order; the per-tensor GPU checksum of checkpoint.py (`rlk_checksum64`)
is stored in "__metadata__" as "rlk_checksum64/<name>" -> 16 hex digits, so `load(verify=True)`
can check payloads the same way as the repo format.
"""
from __future__ import annotations

import json
import os
import struct
from pathlib import Path
from typing import Mapping

import numpy as np
import torch

from .checkpoint import Entry

# safetensors dtype -> repo dtype code (checkpoint.DTYPES: 0 f64, 1 f32, 2 bf16), numpy view, item size
ST_DTYPES = {"F64": (0, np.float64, 8), "F32": (1, np.float32, 4), "BF16": (2, np.uint16, 2)}
CODE_TO_ST = {v[0]: k for k, v in ST_DTYPES.items()}
CHECKSUM_KEY = "rlk_checksum64/"
MAX_HEADER = 100 << 20  # the reference implementation's own bound on the JSON header


def is_safetensors(path) -> bool:
    p = Path(path)
    if p.is_dir() or p.name.endswith(".safetensors.index.json") or p.suffix == ".safetensors":
        return True
    try:
        with open(p, "rb") as f:
            head = f.read(9)
        return len(head) == 9 and 0 < struct.unpack("<Q", head[:8])[0] <= MAX_HEADER and head[8:9] == b"{"
    except OSError:
        return False


def read_header(path) -> tuple[list[Entry], dict]:
    """Entries (absolute byte offsets, repo dtype codes) in data-offset order, and the metadata."""
    path = Path(path)
    size = path.stat().st_size
    with open(path, "rb") as f:
        raw = f.read(8)
        if len(raw) != 8:
            raise ValueError(f"{path}: not a safetensors file (truncated)")
        (hlen,) = struct.unpack("<Q", raw)
        if hlen > MAX_HEADER or 8 + hlen > size:
            raise ValueError(f"{path}: bad safetensors header length {hlen}")
        try:
            hdr = json.loads(f.read(hlen))
        except json.JSONDecodeError as e:
            raise ValueError(f"{path}: corrupt safetensors header ({e})") from None
    if not isinstance(hdr, dict):
        raise ValueError(f"{path}: safetensors header is not an object")
    meta = hdr.pop("__metadata__", None) or {}
    data0 = 8 + hlen
    entries = []
    for name, d in hdr.items():
        st = d.get("dtype")
        if st not in ST_DTYPES:
            raise NotImplementedError(f"{path}: tensor {name!r} has dtype {st}; the B200 kernels fuse BF16/F32/F64")
        code, _, isz = ST_DTYPES[st]
        shape = tuple(int(x) for x in d["shape"])
        b, e = (int(x) for x in d["data_offsets"])
        n = 1
        for s in shape:
            n *= s
        if e - b != n * isz or b < 0 or data0 + e > size:
            raise ValueError(f"{path}: tensor {name!r} data_offsets {b, e} do not match {st}{list(shape)}")
        entries.append(Entry(name, code, shape, offset=data0 + b, nbytes=e - b))
    entries.sort(key=lambda x: x.offset)
    pos = data0
    for x in entries:  # the data buffer must be covered without holes or overlaps
        if x.offset != pos:
            raise ValueError(f"{path}: safetensors data buffer has a hole or overlap at {x.name!r}")
        pos += x.nbytes
    for x in entries:
        cs = meta.get(CHECKSUM_KEY + x.name)
        if cs is not None:
            x.checksum = int(cs, 16)
    return entries, meta


def shard_files(path) -> list[Path]:
    """The shard files of a checkpoint given as one file, a directory or an index.json."""
    p = Path(path)
    if p.is_dir():
        idx = sorted(p.glob("*.safetensors.index.json"))
        if idx:
            p = idx[0]
        else:
            files = sorted(p.glob("*.safetensors"))
            if not files:
                raise FileNotFoundError(f"no .safetensors files in {p}")
            return files
    if p.name.endswith(".index.json"):
        wm = json.loads(p.read_text())["weight_map"]
        seen = []
        for f in wm.values():
            if f not in seen:
                seen.append(f)
        return [p.parent / f for f in seen]
    return [p]


def open_mmap(path) -> tuple[list[Entry], dict[str, np.memmap]]:
    """Entries (in file / shard order) and read-only memory maps of every tensor, over all shards."""
    entries, maps = [], {}
    for f in shard_files(path):
        ents, _ = read_header(f)
        for e in ents:
            if e.name in maps:
                raise ValueError(f"tensor {e.name!r} appears in more than one shard")
            maps[e.name] = np.memmap(f, dtype=ST_DTYPES[CODE_TO_ST[e.dtype]][1], mode="r", offset=e.offset,
                                     shape=e.shape)
            entries.append(e)
    return entries, maps


def layout(specs, metadata: Mapping[str, str] | None = None) -> tuple[bytes, list[Entry], int]:
    """Header bytes (8-byte aligned, space padded) + entries for (name, dtype_code, shape) in order."""
    hdr, entries, pos = {}, [], 0
    for name, code, shape in specs:
        _, _, isz = ST_DTYPES[CODE_TO_ST[code]]
        n = 1
        for s in shape:
            n *= s
        hdr[name] = {"dtype": CODE_TO_ST[code], "shape": list(shape), "data_offsets": [pos, pos + n * isz]}
        entries.append(Entry(name, code, tuple(shape), offset=pos, nbytes=n * isz))
        pos += n * isz
    meta = dict(metadata or {})
    for e in entries:  # fixed-width placeholders, rewritten in place once the checksums are known
        meta.setdefault(CHECKSUM_KEY + e.name, "0" * 16)
    hdr["__metadata__"] = meta
    js = json.dumps(hdr, separators=(",", ":")).encode()
    js += b" " * (-(len(js) + 8) % 8)
    head = struct.pack("<Q", len(js)) + js
    for e in entries:
        e.offset += len(head)
    return head, entries, len(head) + pos


def header_with_checksums(head: bytes, entries) -> bytes:
    """`head` with every checksum placeholder replaced (same length, so offsets are unchanged)."""
    hlen = struct.unpack("<Q", head[:8])[0]
    hdr = json.loads(head[8:8 + hlen])
    for e in entries:
        hdr["__metadata__"][CHECKSUM_KEY + e.name] = f"{e.checksum:016x}"
    js = json.dumps(hdr, separators=(",", ":")).encode()
    if len(js) > hlen:
        raise AssertionError("checksum rewrite changed the header length")
    js += b" " * (hlen - len(js))
    return head[:8] + js


def save(path, tensors: Mapping[str, object], metadata: Mapping[str, str] | None = None) -> None:
    """Write tensors (CUDA or CPU torch, or numpy) as one safetensors file, atomically, with their
    GPU checksums in the metadata."""
    from .checkpoint import DTYPE_CODE, _as_device, _u64, checksum_device
    devs = {k: _as_device(v) for k, v in tensors.items()}
    specs = []
    for k, t in devs.items():
        if t.dtype not in DTYPE_CODE:
            raise NotImplementedError(f"tensor {k!r}: dtype {t.dtype} (BF16/F32/F64 only)")
        specs.append((k, DTYPE_CODE[t.dtype], tuple(t.shape)))
    head, entries, _ = layout(specs, metadata)
    for e in entries:
        e.checksum = _u64(checksum_device(devs[e.name].contiguous()))
    path = Path(path)
    tmp = path.with_name(path.name + ".tmp")
    try:
        with open(tmp, "wb") as f:
            f.write(header_with_checksums(head, entries))
            for e in entries:
                t = devs[e.name].contiguous()
                if t.dtype == torch.bfloat16:
                    t = t.view(torch.int16)
                f.write(t.cpu().numpy().tobytes())
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)
    except BaseException:
        if tmp.exists():
            tmp.unlink()
        raise


def load(path, device=None, verify: bool = True) -> dict[str, torch.Tensor]:
    """Read a (sharded) safetensors checkpoint onto the GPU; payloads carrying an rlk checksum are
    verified on the device."""
    from .checkpoint import DTYPES, _u64, checksum_device
    entries, maps = open_mmap(path)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    out = {}
    for e in entries:
        t = torch.from_numpy(np.array(maps[e.name], copy=True)).to(dev)
        if DTYPES[e.dtype][0] == torch.bfloat16:
            t = t.view(torch.bfloat16)
        if verify and e.checksum and _u64(checksum_device(t)) != e.checksum:
            raise ValueError(f"checkpoint payload checksum mismatch for {e.name!r}")
        out[e.name] = t
    return out
