"""Sum an ncu SASS source page (CSV) by kernel phase / device function.

Each SASS instruction is mapped to its innermost source line (nvdisasm -g),
and each line of the .cuh sources to the closest preceding phase marker
(`// ---------------- NAME`) or function definition.

usage: python tools/ncu_phase_sum.py <ncu_sass.csv> <lib.so> <kernel-mangled-name> [--static]

--static counts SASS instructions (code size) in place of stall samples.
"""
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

csv_path, lib, kname = sys.argv[1:4]
static = "--static" in sys.argv
src_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2501_19042_b200", "csrc")

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

label_cache = {}


def labels(fname):
    if fname in label_cache:
        return label_cache[fname]
    path = os.path.join(src_dir, fname)
    lab = []
    cur = fname
    if os.path.exists(path):
        lines = open(path).read().split("\n")
        for k, ln in enumerate(lines):
            m = re.search(r"// -{8,} (\w+)", ln)
            if m and ln.startswith("  "):
                cur = "phase " + m.group(1)
            else:
                m = re.match(r"(?:__device__|__global__|static|inline|template).*?\b(\w+)\s*\(", ln)
                if m and not ln.rstrip().endswith(";") and m.group(1) not in ("if", "for", "while"):
                    cur = "fn " + m.group(1)
                elif ln.startswith("template") and k + 1 < len(lines):
                    m = re.search(r"\b(\w+)\s*\(", lines[k + 1])
                    if m:
                        cur = "fn " + m.group(1)
            lab.append(cur)
    label_cache[fname] = lab
    return lab


rows = list(csv.reader(open(csv_path)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
base = int(data[0][0], 16)
agg = defaultdict(lambda: [0, 0])
ts = te = 0
for r in data:
    f, l = line_of.get(int(r[0], 16) - base, ("?", 0))
    lab = labels(f)
    name = lab[l - 1] if 0 < l <= len(lab) else f"{f}:{l}"
    if f != "sf_persistent.cuh" and not name.startswith("fn"):
        name = f"{f}"
    s, e = (1 if static else int(r[iS] or 0)), int(r[iE] or 0)
    agg[name][0] += s
    agg[name][1] += e
    ts += s
    te += e
print(f"total: {'sass instructions' if static else 'samples'} {ts}, executed {te / 1e9:.3f}e9 warp-instructions")
for name, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0]):
    if s > 0.002 * ts or e > 0.002 * te:
        print(f"  {name:36s} samples {100 * s / ts:5.1f}%   instr {100 * e / te:5.1f}%  ({e / 1e6:8.1f}M)")
