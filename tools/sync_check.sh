#!/bin/bash
# (box) compute-sanitizer is closed on this GPU pool, so the slot-synchronisation hazards are checked by an
# instrumented build instead: -DSGSF_SYNC_CHECK makes every warp of a slot publish its stop decision and traps
# if two warps of one slot disagree (the decision is taken redundantly per warp, and a disagreement would
# desynchronise the slot's named barriers).  Runs the whole-batch parity (1000 + 48 samples, three
# precisions) and the GPU parity tests under that build, then rebuilds the normal library.

make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_SYNC_CHECK" >/dev/null 2>&1
mkdir -p gpurun_out
timeout 900 python tools/batch_parity.py > gpurun_out/sync_check_parity.log 2>&1; echo "batch parity under SGSF_SYNC_CHECK: rc=$?"; cut -c1-200 gpurun_out/sync_check_parity.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_n32.py tests/test_gpu_coverage.py -q -m gpu 2>&1 | tail -1
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 >/dev/null 2>&1
