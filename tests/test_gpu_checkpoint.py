"""GPU tests: checkpoint save/load with device checksums, and cmd_fuse end to end on files."""
import numpy as np
import pytest
import torch

from oracle import fusion as OF
from tests.helpers import bf16_round, rne_bf16_bits, synth_state_dicts

pytestmark = pytest.mark.gpu


def test_table_roundtrip_and_corruption(cuda, tmp_path):
    from paper_2509_18883_b200 import checkpoint as CK
    from paper_2509_18883_b200.toy_env import ParamTable
    pt = ParamTable(np.random.default_rng(0).normal(size=(2, 3, 11)))
    p = tmp_path / "t.ckpt"
    CK.save_table(p, pt)
    assert CK.load_table(p).equals(pt)
    raw = bytearray(p.read_bytes())
    e = CK.read_header(p)[0]
    raw[e.offset + 5] ^= 1  # flip one payload bit
    (tmp_path / "bad.ckpt").write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="checksum mismatch"):
        CK.load_table(tmp_path / "bad.ckpt")


@pytest.mark.parametrize("cfgkw", [dict(), dict(dropout_p=0.5, seed=4)])
def test_cmd_fuse_files(cuda, tmp_path, cfgkw):
    from paper_2509_18883_b200 import checkpoint as CK
    from paper_2509_18883_b200 import fusion as F
    shapes = {"emb": (700, 64), "w": (64, 300), "b": (300,)}
    base, experts = synth_state_dicts(shapes, 3, seed=21, dtype_round=bf16_round)
    to = lambda d: {k: torch.from_numpy(v).to(cuda, torch.bfloat16) for k, v in d.items()}
    CK.save(tmp_path / "base.ckpt", to(base))
    paths = []
    for i, e in enumerate(experts):
        paths.append(tmp_path / f"e{i}.ckpt")
        CK.save(paths[-1], to(e))
    rep = CK.cmd_fuse(tmp_path / "base.ckpt", paths, tmp_path / "fused.ckpt", F.FusionConfig(**cfgkw),
                      device_budget_bytes=1 << 20)
    assert rep.groups >= 2
    fused = CK.load(tmp_path / "fused.ckpt")  # verifies payload checksums
    ref_dev, _ = F.fuse_state_dict(to(base), [to(e) for e in experts], F.FusionConfig(**cfgkw))
    for k in shapes:
        assert torch.equal(fused[k].view(torch.int16), ref_dev[k].view(torch.int16)), k
        ref, st = OF.fuse(base[k], [e[k] for e in experts], **cfgkw)
        assert (fused[k].reshape(-1).view(torch.int16).cpu().numpy().view(np.uint16) != rne_bf16_bits(ref)).sum() == 0
        assert list(rep.stats[k].erased_counts) == st["erased"]


def test_cmd_fuse_identity_and_errors(cuda, tmp_path):
    """one expert, identity settings -> fused equals the expert byte for byte; a corrupt
    header -> load error and no partial output."""
    from paper_2509_18883_b200 import checkpoint as CK
    from paper_2509_18883_b200 import fusion as F
    g = np.random.default_rng(1)
    # bf16 tables: differences of bf16 values are exact in the f64 reference arithmetic, so
    # base + 1.0 * (expert - base) == expert (for arbitrary f64 tables the reference itself rounds)
    b = {"t": torch.from_numpy(g.normal(size=(5, 9))).to(cuda, torch.bfloat16)}
    e = {"t": torch.from_numpy(g.normal(size=(5, 9))).to(cuda, torch.bfloat16)}
    CK.save(tmp_path / "b.ckpt", b)
    CK.save(tmp_path / "e.ckpt", e)
    CK.cmd_fuse(tmp_path / "b.ckpt", [tmp_path / "e.ckpt"], tmp_path / "f.ckpt",
                F.FusionConfig(target_norm=None, erase_mode=False))
    ef, ff = CK.open_mmap(tmp_path / "e.ckpt")[1]["t"], CK.open_mmap(tmp_path / "f.ckpt")[1]["t"]
    assert np.asarray(ef).tobytes() == np.asarray(ff).tobytes()
    raw = bytearray((tmp_path / "e.ckpt").read_bytes())
    raw[3] ^= 0xFF
    (tmp_path / "x.ckpt").write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="corrupt checkpoint header"):
        CK.cmd_fuse(tmp_path / "b.ckpt", [tmp_path / "x.ckpt"], tmp_path / "out.ckpt", F.FusionConfig())
    assert not (tmp_path / "out.ckpt").exists() and not (tmp_path / "out.ckpt.tmp").exists()
