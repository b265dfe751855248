"""Attribute an ncu SASS source page (CSV) to CUDA source lines via nvdisasm -g.

usage: python tools/ncu_lines.py <ncu_sass.csv> <lib.so> <kernel-mangled-name> [top]
"""
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

csv_path, lib, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top_n = int(sys.argv[4]) if len(sys.argv) > 4 else 40

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    if f".text.{kname}:" not in out:
        continue
    sec = out.split(f".text.{kname}:", 1)[1]
    cur = None
    for ln in sec.split("\n"):
        if ln.strip().startswith(".section") or ln.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    break

rows = list(csv.reader(open(csv_path)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
agg = defaultdict(lambda: [0, 0, defaultdict(int)])
tot = 0
for r in data:
    off = int(r[0], 16) - base
    key = line_of.get(off, ("?", 0))
    s = int(r[iS] or 0)
    tot += s
    a = agg[key]
    a[0] += s
    a[1] += int(r[iE] or 0)
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            a[2][hdr[i][6:]] += v
src = {}
for (f, l) in agg:
    if f not in src:
        cands = glob.glob(f"/root/repo/paper_2501_19042_b200/csrc/{f}")
        src[f] = open(cands[0]).read().split("\n") if cands else []
print(f"total samples {tot}")
for key, (s, e, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top_n]:
    f, l = key
    text = src.get(f, [])[l - 1].strip()[:70] if f in src and 0 < l <= len(src[f]) else ""
    tops = sorted(st.items(), key=lambda x: -x[1])[:2]
    print(f"{100 * s / tot:5.1f}%  exec {e / 1e6:8.1f}M  {f}:{l:<4d} {text:70s} {[(a, round(100 * b / tot, 1)) for a, b in tops]}")
