#!/bin/bash
# (box) hybrid's cost over lean, by part: K1 time with the FP64 scatter / the FP64 stop re-evaluation compiled
# out (attribution only: those builds are not exact)
for extra in "" "-DSGSF_HY_NO_SCATTER" "-DSGSF_HY_NO_RECOMPUTE" "-DSGSF_HY_NO_SCATTER -DSGSF_HY_NO_RECOMPUTE"; do
  make -C paper_2501_19042_b200/csrc clean >/dev/null
  make -C paper_2501_19042_b200/csrc -j32 EXTRA="$extra" >/dev/null 2>&1 || exit 1
  echo "== [$extra]"
  python tools/order_probe.py hybrid 2>&1 | grep "no_order=0 in flight 1" | tail -1
done
python tools/order_probe.py lean 2>&1 | grep "no_order=0 in flight 1" | tail -1
