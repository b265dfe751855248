#!/bin/bash
# (on the GPU box) round artifacts: bench lines, launch list, one full ncu capture of the main kernel.
# usage: tools/round_profile.sh <tag>   -> gpurun_out/<tag>_*.{json,csv,ncu-rep}
T=${1:-rXX}
mkdir -p gpurun_out
python bench.py > gpurun_out/${T}_bench.log 2>&1; tail -1 gpurun_out/${T}_bench.log > gpurun_out/${T}_bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.log 2>&1
tail -1 gpurun_out/${T}_bench_ref.log > gpurun_out/${T}_bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sf_persistent -s 3 -c 1 -o gpurun_out/${T}_full \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
tail -2 gpurun_out/${T}_ncu_full.log
