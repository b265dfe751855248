#!/bin/bash
# (box) K1 event counts of config-3 shards (rank 0 and rank 7 of 8): why one shard is slower than another
make -C paper_2501_19042_b200/csrc clean >/dev/null
make -C paper_2501_19042_b200/csrc -j32 EXTRA="-DSGSF_COUNTERS" >/dev/null 2>&1 || exit 1
python tools/shard_iters.py 2>&1 | grep -E "COUNTS|kernel"
