#!/bin/bash
# (on the GPU box) rebuild with -DSGSF_COUNTERS and print K1's event counts for config 2 per precision
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_COUNTERS" >/dev/null 2>&1 || exit 1
for prec in ${PRECS:-lean hybrid}; do
  echo "== $prec"
  python tools/prof_case.py --reps 1 --precision $prec 2>&1 | tail -2
done
