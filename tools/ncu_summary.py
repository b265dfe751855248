"""Key metrics of one `ncu --set full` capture -> JSON (profiles/ncu_traffic.json feeds bench.py's roofline.traffic).

usage: python tools/ncu_summary.py <report.ncu-rep> <out.json> "<command that made it>"
"""
import csv
import io
import json
import subprocess
import sys

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.per_cycle_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "sm__cycles_active.avg",
        "sm__cycles_elapsed.avg", "sm__icc_request_hit_rate.pct",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
m = {}
for k in want:
    if k in hdr:
        i = hdr.index(k)
        m[k] = (vals[i] + " " + units[i]).strip()


def to_bytes(s):
    v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale


traffic = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
json.dump({"kernel": m.get("Kernel Name", "").split("(")[0], "command": cmd, "dram_bytes_per_launch": traffic,
           "metrics": m}, open(out, "w"), indent=1)
print(json.dumps({"dram_bytes_per_launch": traffic, **{k: m[k] for k in list(m)[:6]}}, indent=1))
