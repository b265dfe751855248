#!/bin/bash
# (box) per-warp cycles of K1's T1 near-pair checks (-DSGSF_NEAR_CLOCK), CTAs 0-1; CONFIG=2 (default) or 3
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_NEAR_CLOCK" >/dev/null 2>&1 || exit 1
python tools/prof_case.py --reps 1 --precision hybrid --config ${CONFIG:-2} --batch ${BATCH:-1000} 2>&1 | grep NEAR | sort | head -${LINES:-12}
