#!/bin/bash
# (on the GPU box) K1L term-pass balance: rebuild with -DSGSF_LARGE_PT, run a config-4 batch, print per-sample
# slowest-warp vs mean term-pass cycles and exact steps per warp (CTAs 0-3)
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_LARGE_PT ${LPT_EXTRA}" >/dev/null 2>&1 || exit 1
python tools/prof_large.py ${PREC:-hybrid} ${BATCH:-1184} ${ITERS:-1000} 1 2>&1 | grep -E "LPT|LQ|LMX|ok" | head -${LINES:-40}
