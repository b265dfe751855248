"""Map SASS instructions of an ncu source-page CSV (by substring) to CUDA source lines of one kernel.

usage: python tools/sass_pc_line.py <ncu_sass.csv> <object.o|lib.so> <kernel-mangled-name> <substring> [...]
"""
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

csv_path, obj, kname, subs = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
rows = list(csv.reader(open(csv_path)))
data = rows[2:]
base = int(data[0][0], 16)
want = {int(r[0], 16) - base: (r[1].strip(), r[2]) for r in data if any(x in r[1] for x in subs)}
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    if f".text.{kname}:" not in out:
        continue
    sec = out.split(f".text.{kname}:", 1)[1].split("\n\t.section", 1)[0]
    cur, hist = None, []
    for ln in sec.split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m:
            a = int(m.group(1), 16)
            if a in want:
                print(hex(a), want[a], cur)
                print("   before:", *[h.strip()[:90] for h in hist[-6:]], sep="\n      ")
            hist.append(ln)
    break
