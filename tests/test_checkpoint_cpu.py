"""Checkpoint header format (host logic, no GPU)."""
import pytest

from paper_2509_18883_b200.checkpoint import ALIGN, Entry, decode_header, encode_header, layout_entries


def test_header_roundtrip_and_alignment():
    ents, size = layout_entries([("logits", 0, (2, 3, 5)), ("w", 2, (7,)), ("ü", 1, ())])
    for e in ents:
        e.checksum = 0x0123456789ABCDEF
    h = encode_header(ents)
    assert len(h) % ALIGN == 0 and all(e.offset % ALIGN == 0 for e in ents) and size % ALIGN == 0
    back = decode_header(h)
    assert [(e.name, e.dtype, e.shape, e.offset, e.nbytes, e.checksum) for e in back] == \
           [(e.name, e.dtype, e.shape, e.offset, e.nbytes, e.checksum) for e in ents]
    assert ents[0].nbytes == 2 * 3 * 5 * 8 and ents[1].nbytes == 14 and ents[2].nbytes == 4


def test_corrupt_header_is_rejected():
    ents, _ = layout_entries([("t", 0, (4,))])
    h = bytearray(encode_header(ents))
    for pos in (0, 9, 30):
        bad = bytearray(h)
        bad[pos] ^= 0xFF
        with pytest.raises(ValueError, match="corrupt checkpoint header"):
            decode_header(bytes(bad))
