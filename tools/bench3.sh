#!/bin/bash
# (on the GPU box) three short bench runs -> ms per step of each
for i in 1 2 3; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms/step  kernel %.3f ms' % (d['ms_per_step'], d['roofline']['kernel_ms']))"
done
