"""GPU: cmd_fuse over real-checkpoint (safetensors) files, written by the `safetensors` library --
single files, a sharded directory with index.json, safetensors -> repo-format output -- against
fuse_state_dict and the CPU oracle, bit for bit."""
import json

import numpy as np
import pytest
import torch

from oracle import fusion as OF
from tests.helpers import bf16_round, rne_bf16_bits, synth_state_dicts

pytestmark = pytest.mark.gpu
st_torch = pytest.importorskip("safetensors.torch")

SHAPES = {"model.embed_tokens.weight": (700, 64), "layers.0.mlp.up_proj.weight": (64, 300),
          "layers.0.input_layernorm.weight": (300,), "lm_head.weight": (333, 64)}


def _write(path, sd, shards=1):
    cpu = {k: torch.from_numpy(v).to(torch.bfloat16) for k, v in sd.items()}
    if shards == 1:
        st_torch.save_file(cpu, str(path), metadata={"format": "pt"})
        return path
    path.mkdir()
    names = list(cpu)
    wm = {}
    for s in range(shards):
        fn = f"model-{s + 1:05d}-of-{shards:05d}.safetensors"
        part = names[s::shards]
        st_torch.save_file({k: cpu[k] for k in part}, str(path / fn))
        wm.update({k: fn for k in part})
    (path / "model.safetensors.index.json").write_text(json.dumps({"metadata": {}, "weight_map": wm}))
    return path


@pytest.mark.parametrize("shards,out_ext,cfgkw", [(1, ".safetensors", dict(dropout_p=0.5, seed=4)),
                                                  (2, ".safetensors", dict()),
                                                  (1, ".ckpt", dict(erase_weighting="squared"))])
def test_cmd_fuse_safetensors(cuda, tmp_path, shards, out_ext, cfgkw):
    from paper_2509_18883_b200 import checkpoint as CK
    from paper_2509_18883_b200 import fusion as F
    base, experts = synth_state_dicts(SHAPES, 3, seed=33, dtype_round=bf16_round)
    bp = _write(tmp_path / ("base" + (".safetensors" if shards == 1 else "")), base, shards)
    eps = [_write(tmp_path / (f"e{i}" + (".safetensors" if shards == 1 else "")), e, shards)
           for i, e in enumerate(experts)]
    out = tmp_path / ("fused" + out_ext)
    cfg = F.FusionConfig(**cfgkw)
    rep = CK.cmd_fuse(bp, eps, out, cfg, device_budget_bytes=1 << 20)
    assert rep.groups >= 2
    fused = CK.load(out)  # device checksums verified (safetensors: from the metadata)
    to = lambda d: {k: torch.from_numpy(v).to(cuda, torch.bfloat16) for k, v in d.items()}
    ref_dev, ref_rep = F.fuse_state_dict(to(base), [to(e) for e in experts], cfg)
    for k in SHAPES:
        assert fused[k].shape == torch.Size(SHAPES[k])
        assert torch.equal(fused[k].view(torch.int16), ref_dev[k].view(torch.int16)), k
        ref, st = OF.fuse(base[k], [e[k] for e in experts], **cfgkw)
        got = fused[k].reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16)
        assert int((got != rne_bf16_bits(ref)).sum()) == 0, k
        assert list(rep.stats[k].erased_counts) == st["erased"]
        assert rep.stats[k] == ref_rep.stats(k)
    if out_ext == ".safetensors":  # the output is a valid safetensors file for the library too
        back = st_torch.load_file(str(out))
        for k in SHAPES:
            assert torch.equal(back[k].view(torch.int16), fused[k].cpu().view(torch.int16))


def test_safetensors_checksum_mismatch(cuda, tmp_path):
    from paper_2509_18883_b200 import safetensors_io as ST
    t = {"w": torch.arange(1000, dtype=torch.float32, device=cuda)}
    p = tmp_path / "c.safetensors"
    ST.save(p, t)
    assert torch.equal(ST.load(p)["w"], t["w"])
    raw = bytearray(p.read_bytes())
    raw[-7] ^= 1
    (tmp_path / "bad.safetensors").write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="checksum mismatch"):
        ST.load(tmp_path / "bad.safetensors")
