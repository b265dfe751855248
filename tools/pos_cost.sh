#!/bin/bash
# (box) what the FFMA positions cost in the n = 32 kernel: config-3 phase timing with -DSGSF_NO_POS (positions
# frozen after the first iterate: timing only, results wrong) against the normal build
for extra in "" "-DSGSF_NO_POS"; do
  PT_EXTRA="$extra" PT_CONFIG=3 bash tools/phase_timing.sh >/dev/null 2>&1
  echo "== [$extra]"; python tools/pt_report.py full | head -3
done
