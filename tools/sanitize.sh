#!/bin/bash
# (box) compute-sanitizer memcheck / racecheck / synccheck of K1 (and its aux kernels) on small config-2 cases
mkdir -p gpurun_out
for prec in hybrid lean strict; do
  for tool in memcheck racecheck synccheck; do
    echo "== $tool $prec"
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/prof_case.py --batch 6 --reps 1 \
        --max-iters 25 --precision $prec 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard|iterations mean" | head -8
  done
done
