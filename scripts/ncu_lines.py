"""Aggregate an ncu source-page (SASS) CSV by CUDA source line, using nvdisasm --print-line-info of
the kernel's cubin: instructions executed and warp-stall samples per line (needs -lineinfo).
usage: ncu_lines.py <ncu sass csv> <nvdisasm listing> <mangled kernel name> <source file> [top]"""
import collections
import csv
import re
import sys

csv_path, sass_path, kname, src_path = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
lines = open(sass_path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kname + ":"))
off2line, cur = {}, None
for l in lines[start + 1:]:
    if l.startswith("//---------------------") or l.startswith(".text."):
        break
    m = re.search(r'line (\d+)', l)
    if m:
        cur = int(m.group(1))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m2 and cur is not None:
        off2line[int(m2.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [(int(r[ix['Address']], 16), float(r[ix['Instructions Executed']] or 0),
         float(r[ix['Warp Stall Sampling (All Samples)']] or 0)) for r in rows[2:] if len(r) >= len(hdr)]
base = min(d[0] for d in data)
ins, stl = collections.Counter(), collections.Counter()
for a, ie, st in data:
    ln = off2line.get(a - base, -1)
    ins[ln] += ie
    stl[ln] += st
ti, ts = sum(ins.values()), sum(stl.values())
src = open(src_path).read().splitlines()
print(f"total warp-instructions {ti:.0f}, stall samples {ts:.0f}")
for ln, v in ins.most_common(top):
    print(f"L{ln:4d} instr {v / ti * 100:5.1f}%  stall {stl[ln] / ts * 100:5.1f}%  {src[ln - 1].strip()[:100] if ln > 0 else ''}")
