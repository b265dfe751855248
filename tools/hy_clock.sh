#!/bin/bash
# (on the GPU box) cycles of each FP64 stop re-evaluation (hybrid K1, CTAs 0-1), config 2
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_HY_CLOCK" >/dev/null 2>&1 || exit 1
python tools/prof_case.py --reps 1 --precision hybrid 2>&1 | grep HYC | awk '{s+=$NF; n++} END {print "re-evaluations", n, "mean cycles", s/n}'
python tools/prof_case.py --reps 1 --precision hybrid 2>&1 | grep HYC | head -12
