"""Opcode histogram of the innermost loop(s) of a kernel's SASS (dev tool):
python tools/sass_loop.py <lib.so> <mangled kernel name> [needle opcode]
The loop is the backward-branch range with the most needle instructions
(default MUFU.LG2), the smallest among equals."""
import re
import subprocess
import sys
from collections import Counter

lib, fn = sys.argv[1], sys.argv[2]
needle = sys.argv[3] if len(sys.argv) > 3 else "MUFU.LG2"
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for ln in sass.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, text) in enumerate(ins):
    m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)", text)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr:
        continue
    lo, hi = addr[tgt], i
    body = [t for _, t in ins[lo:hi + 1]]
    hits = sum(needle in t for t in body)
    if hits and (best is None or (hits, lo - hi) > (best[2], best[0] - best[1])):
        best = (lo, hi, hits)
if best is None:
    sys.exit("no loop with " + needle)
body = [t for _, t in ins[best[0]:best[1] + 1]]
ops = Counter()
for t in body:
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    ops[t.split()[0]] += 1
print(f"loop {ins[best[0]][0]:#x}..{ins[best[1]][0]:#x}: {len(body)} instructions")
for op, c in ops.most_common():
    print(f"  {op:24s} {c}")
