"""Aggregate ncu SASS samples/instructions by source-line ranges of sf_persistent.cuh functions."""
import csv, glob, os, re, subprocess, sys, tempfile
from collections import defaultdict
csv_path, lib, kname = sys.argv[1:4]
src = open("paper_2501_19042_b200/csrc/sf_persistent.cuh").read().split("\n")
# phase markers: (first line containing marker) -> name
markers = [("// positions of every robot", "positions"), ("// Interior bit of every term", "scan"),
           ("// Exit residual over all terms", "quiet"), ("// Flagged terms", "flagged"),
           ("// Exact max of |x| over the unflagged", "unflagged_max"), ("// Careful path", "careful"),
           ("// ---------------------------------------------------------------- load a sample", "load"),
           ("// ---------------------------------------------------------------- the kernel", "kernel-setup"),
           ("// ---------------- T: term pass", "T-glue"), ("// ---------------- G:", "G"),
           ("if (lwarp == 0) {   // decision", "decision"), ("// ---------------- finalize", "finalize"),
           ("// ---------------- M: swarm means", "M"), ("// ---------------- M2", "M2"),
           ("// ---------------- X:", "X")]
bounds = []
for m, name in markers:
    for k, l in enumerate(src):
        if m in l:
            bounds.append((k + 1, name)); break
bounds.sort()
def phase(f, l):
    if f != "sf_persistent.cuh":
        return "inlined:" + f
    name = "header"
    for start, nm in bounds:
        if l >= start: name = nm
    return name
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    if f".text.{kname}:" not in out: continue
    sec = out.split(f".text.{kname}:", 1)[1]
    cur = None; stack = []
    for ln in sec.split("\n"):
        if ln.strip().startswith(".section"): break
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            f = os.path.basename(m.group(1)); l = int(m.group(2))
            # attribute inlined helper lines (fma_t etc.) to the caller line when given
            if m.group(4) and os.path.basename(m.group(4)) == "sf_persistent.cuh" and f != "sf_persistent.cuh":
                f, l = "sf_persistent.cuh", int(m.group(5))
            cur = (f, l); continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur: line_of[int(m.group(1), 16)] = cur
    break
rows = list(csv.reader(open(csv_path))); hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
base = int(data[0][0], 16); agg = defaultdict(lambda: [0, 0]); tS = tE = 0
for r in data:
    f, l = line_of.get(int(r[0], 16) - base, ("?", 0)); p = phase(f, l)
    s, e = int(r[iS] or 0), int(r[iE] or 0); agg[p][0] += s; agg[p][1] += e; tS += s; tE += e
for p, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{p:18s} samples {100*s/tS:5.1f}%   instructions {100*e/tE:5.1f}%  ({e/1e6:.0f}M)")
