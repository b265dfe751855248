#!/bin/bash
# (box) phase timing of config-3 shard rank 7 of 8 (the slow one): per-CTA slot-0 phase cycles
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_PHASE_TIMING" >/dev/null 2>&1 || exit 1
mkdir -p gpurun_out
python tools/shard_iters.py > gpurun_out/pt_full.log 2>&1
python tools/pt_report.py full
sort -t' ' -k6 -n -r gpurun_out/pt_full.log | grep "PT block" | head -5
