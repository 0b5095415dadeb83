"""Stall samples of an advance_p_lean launch by kernel region.

python tools/sass_regions.py OBJ FUNC_SUBSTR NCU_SASS_TXT [...]

OBJ: build/pic_b200/push.cu.o of the library build that was profiled (it is
disassembled with `nvdisasm -gi`; the source must be the one it was built
from); NCU_SASS_TXT: tools/ncu_sass_top.py output with every
instruction.  Each SASS address is attributed to the outermost push.cu line
of the kernel body, and lines to regions by the markers below.
"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict

gi, func = sys.argv[1], sys.argv[2]
src = open("paper_2102_13133_b200/csrc/push.cu").read().splitlines()


def line_of(marker, start=0):
    for i in range(start, len(src)):
        if marker in src[i]:
            return i + 1
    raise KeyError(marker)


k0 = line_of("advance_p_lean(const LeanBatch B")
marks = [("prologue", k0), ("order-reserve", line_of("kOrd & 2: every record's slot", k0)),
         ("seeding", line_of("slot seeding (advance_p_run", k0)), ("loop", line_of("#pragma unroll 1", k0)),
         ("flush", line_of("if (kQuad >= 1)", k0)), ("lidx-load", line_of("the logical indices of the slice", k0)),
         ("drain", line_of("drain the crossing queue", k0)), ("redo", line_of("the flagged particles, with", k0)),
         ("order-store", line_of("every record, with its logical", k0)),
         ("tma-store", line_of("publish the slice", k0)), ("end", line_of("static void launch_lean", k0))]


def region(ln):
    r = "other"
    for name, l in marks:
        if ln >= l:
            r = name
    return r


with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(gi)], cwd=td, check=True, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    text = subprocess.run(["nvdisasm", "-gi", os.path.join(td, cub)], capture_output=True, text=True).stdout
start = [m.start() for m in re.finditer(r"^\.text\.(\S+):", text, re.M) if func in text[m.start():m.start() + 400]]
body = text[start[0]:]
nxt = re.search(r"^\s*\.section\s+\.text\.", body[10:], re.M)
body = body[:nxt.start() + 10] if nxt else body
addr_line, addr_ins, cur = {}, {}, None
for l in body.splitlines():
    m = re.match(r'\s*//## File ".*push\.cu", line (\d+)$', l)
    if m:
        cur = int(m.group(1))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
    if m:
        a = int(m.group(1), 16)
        addr_line[a], addr_ins[a] = cur, re.sub(r"\s+", " ", m.group(2))
for f in sys.argv[3:]:
    rows = []
    for l in open(f).read().splitlines()[1:]:
        p = l.split()
        if len(p) < 6:
            continue
        rows.append((float(p[0].rstrip("%")), float(p[2].rstrip("%")), int(p[4], 16), " ".join(p[5:])))
    # anchor: the first profiled instruction whose text is unique in the function
    base = None
    inv = defaultdict(list)
    for a, t in addr_ins.items():
        inv[t.replace(".reuse", "")].append(a)
    for s, n, a, t in rows:
        t = re.sub(r"\s+", " ", t.replace(".reuse", "")).strip()
        c = inv.get(t, [])
        if len(c) == 1 and "0x" not in t:
            base = a - c[0]
            break
    smp, ins = Counter(), Counter()
    for s, n, a, t in rows:
        ln = addr_line.get(a - base)
        r = region(ln) if ln else "unmapped"
        smp[r] += s
        ins[r] += n
    print(f, "base", hex(base))
    for name, _ in marks[:-1] + [("other", 0), ("unmapped", 0)]:
        if smp[name] or ins[name]:
            print(f"  {name:13s} samples {smp[name]:5.1f}%  inst {ins[name]:5.1f}%")
