"""Instruction mix of a SASS address range (cuobjdump -sass output), skipping the blocks a
`@!Px BRA Py, target` jumps over (the rarely taken slow-path bookkeeping).  Usage:
  cuobjdump -sass -fun <mangled> _rlk.so > f.sass; python tools/sass_mix.py f.sass <lo_hex> <hi_hex>"""
import re
import sys
from collections import Counter


def mix(path, lo, hi):
    ins = []
    for line in open(path):
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    reg = [(a, t) for a, t in ins if lo <= a <= hi]
    skip = set()
    for a, t in reg:
        m = re.search(r'BRA P\d, 0x([0-9a-f]+)', t)
        if m and t.startswith('@!P'):
            tgt = int(m.group(1), 16)
            skip.update(b for b, _ in reg if a < b < tgt)
    fast = [t for a, t in reg if a not in skip]
    ops = Counter((t.split()[1] if t.startswith('@') else t.split()[0]) for t in fast)
    return len(reg), len(fast), ops


if __name__ == "__main__":
    total, fast, ops = mix(sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16))
    print(f"instructions in range: {total}; on the fast path: {fast}")
    print(", ".join(f"{k} {v}" for k, v in ops.most_common()))
