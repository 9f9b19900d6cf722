"""safetensors reader / writer (paper_2509_18883_b200.safetensors_io) against the `safetensors`
library's own files, on CPU: header parsing, dtypes, shards + index.json, malformed files."""
import json
import struct

import numpy as np
import pytest
import torch

from paper_2509_18883_b200 import safetensors_io as ST

st_torch = pytest.importorskip("safetensors.torch")


def _tensors(seed=0):
    g = torch.Generator().manual_seed(seed)
    return {"embed.weight": torch.randn((7, 33), generator=g).to(torch.bfloat16),
            "fc.bias": torch.randn(5, generator=g, dtype=torch.float64),
            "fc.w": torch.randn((4, 6), generator=g),
            "scalar": torch.tensor(3.5, dtype=torch.float32)}


def _bits(t):
    t = t.contiguous()
    return t.view(torch.int16).numpy() if t.dtype == torch.bfloat16 else t.numpy()


def test_reads_library_files(tmp_path):
    ts = _tensors()
    p = tmp_path / "m.safetensors"
    st_torch.save_file(ts, str(p), metadata={"format": "pt"})
    assert ST.is_safetensors(p)
    ents, maps = ST.open_mmap(p)
    assert {e.name for e in ents} == set(ts)
    for name, t in ts.items():
        assert maps[name].shape == tuple(t.shape)
        assert np.array_equal(np.asarray(maps[name]).view(_bits(t).dtype), _bits(t))


def test_shards_and_index(tmp_path):
    ts = _tensors(1)
    names = list(ts)
    st_torch.save_file({k: ts[k] for k in names[:2]}, str(tmp_path / "model-00001-of-00002.safetensors"))
    st_torch.save_file({k: ts[k] for k in names[2:]}, str(tmp_path / "model-00002-of-00002.safetensors"))
    wm = {k: ("model-00001-of-00002.safetensors" if i < 2 else "model-00002-of-00002.safetensors")
          for i, k in enumerate(names)}
    (tmp_path / "model.safetensors.index.json").write_text(json.dumps({"metadata": {}, "weight_map": wm}))
    for src in (tmp_path, tmp_path / "model.safetensors.index.json"):
        ents, maps = ST.open_mmap(src)
        assert sorted(e.name for e in ents) == sorted(names)
        for name, t in ts.items():
            assert np.array_equal(np.asarray(maps[name]).view(_bits(t).dtype), _bits(t))


def test_writer_layout_is_readable_by_the_library(tmp_path):
    ts = _tensors(2)
    specs = [(k, {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2}[t.dtype], tuple(t.shape)) for k, t in ts.items()]
    head, ents, size = ST.layout(specs, {"note": "x"})
    for i, e in enumerate(ents):
        e.checksum = 0x0123456789ABCDEF + i
    p = tmp_path / "w.safetensors"
    with open(p, "wb") as f:
        f.write(ST.header_with_checksums(head, ents))
        for e in ents:
            f.write(_bits(ts[e.name]).tobytes())
    assert p.stat().st_size == size
    back = st_torch.load_file(str(p))
    for k, t in ts.items():
        assert np.array_equal(_bits(back[k]), _bits(t))
    ents2, meta = ST.read_header(p)
    assert meta["note"] == "x"
    assert {e.name: e.checksum for e in ents2} == {e.name: e.checksum for e in ents}


def test_malformed_and_unsupported(tmp_path):
    p = tmp_path / "bad.safetensors"
    p.write_bytes(struct.pack("<Q", 10 ** 6) + b"{}")
    with pytest.raises(ValueError):
        ST.read_header(p)
    st_torch.save_file({"h": torch.zeros(3, dtype=torch.float16)}, str(tmp_path / "f16.safetensors"))
    with pytest.raises(NotImplementedError):
        ST.read_header(tmp_path / "f16.safetensors")
    js = json.dumps({"a": {"dtype": "F32", "shape": [2], "data_offsets": [8, 16]}}).encode()
    (tmp_path / "hole.safetensors").write_bytes(struct.pack("<Q", len(js)) + js + bytes(16))
    with pytest.raises(ValueError, match="hole"):
        ST.read_header(tmp_path / "hole.safetensors")
    js = json.dumps({"a": {"dtype": "F32", "shape": [3], "data_offsets": [0, 8]}}).encode()
    (tmp_path / "size.safetensors").write_bytes(struct.pack("<Q", len(js)) + js + bytes(8))
    with pytest.raises(ValueError):
        ST.read_header(tmp_path / "size.safetensors")


def test_repo_format_is_not_safetensors(tmp_path):
    from paper_2509_18883_b200.checkpoint import MAGIC
    p = tmp_path / "x.ckpt"
    p.write_bytes(MAGIC + bytes(64))
    assert not ST.is_safetensors(p)
