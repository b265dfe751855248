#!/bin/bash
# usage (here): tools/prof_report.sh <tag> [kernel-mangled-name]
K=${2:-_ZN4sgsf20sf_persistent_kernelIfLi16ELi12ELi384EEEvNS_11SolveParamsE}
ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/sass_$1.csv
python3 tools/ncu_lines.py /tmp/sass_$1.csv paper_2501_19042_b200/libsgsf.so $K ${3:-30}
ncu -i gpurun_out/prof_$1.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Issue Slots Busy|Registers Per Thread|Achieved Active Warps Per SM|Executed Ipc Active)"' | awk -F'","' '{print $(NF-2)" = "$NF}'
