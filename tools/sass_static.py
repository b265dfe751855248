"""Static SASS size of the persistent kernel body by phase / function (from nvdisasm -g line info).

usage: python tools/sass_static.py [kernel-mangled-name]
"""
import collections
import glob
import os
import re
import subprocess
import sys
import tempfile

root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
name = sys.argv[1] if len(sys.argv) > 1 else "_ZN4sgsf20sf_persistent_kernelIfLi16ELi12ELi384ELi1EEEvNS_11SolveParamsE"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(root, "paper_2501_19042_b200", "libsgsf.so")], cwd=tmp,
               capture_output=True)
txt = ""
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    if f".text.{name}:" in out:
        txt = out
        break
sec = re.split(r"\n\s*\.section", txt.split(f".text.{name}:", 1)[1], 1)[0]
src = open(os.path.join(root, "paper_2501_19042_b200", "csrc", "sf_persistent.cuh")).read().split("\n")
lab, cur = [], "?"
for k, ln in enumerate(src):
    m = re.search(r"// -{8,} (\w+)", ln)
    if m and ln.startswith("  "):
        cur = "phase " + m.group(1)
    else:
        m = re.match(r"(?:__device__|__global__|static|inline|template).*?\b(\w+)\s*\(", ln)
        if m and not ln.rstrip().endswith(";") and m.group(1) not in ("if", "for", "while"):
            cur = "fn " + m.group(1)
        elif ln.startswith("template") and k + 1 < len(src):
            m = re.search(r"\b(\w+)\s*\(", src[k + 1])
            if m:
                cur = "fn " + m.group(1)
    lab.append(cur)
loc, region, cnt = None, "kernel body", collections.Counter()
for ln in sec.split("\n"):
    if ln.strip().endswith(":") and "ZN" in ln:
        region = "subroutine " + ln.strip().split("$")[-1][:60]
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        loc = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", ln):
        if region != "kernel body":
            cnt[region] += 1
        elif loc and loc[0] == "sf_persistent.cuh":
            cnt[lab[loc[1] - 1]] += 1
        else:
            cnt[loc[0] if loc else "?"] += 1
tot = sum(cnt.values())
print(f"total {tot} SASS instructions ({tot * 16 / 1024:.0f} KB)")
for k, v in cnt.most_common(40):
    print(f"{v:6d}  {k}")
