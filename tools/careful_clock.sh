make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j16 EXTRA="-DSGSF_CAREFUL_CLOCK" >/dev/null 2>&1 || exit 1
python tools/prof_case.py --reps 1 --precision hybrid --config 1 --batch 8 --max-iters 100 2>&1 | grep -E "CC|HC" | head -30
