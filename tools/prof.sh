#!/bin/bash
# usage (on the GPU box): [PREC=lean|hybrid|strict] tools/prof.sh <tag>   -> gpurun_out/prof_<tag>.ncu-rep
mkdir -p gpurun_out
PREC=${PREC:-lean}
python tools/prof_case.py --reps 2 --precision $PREC > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sf_persistent -s 1 -c 1 -o gpurun_out/prof_$1 \
    python tools/prof_case.py --reps 2 --precision $PREC > gpurun_out/ncu.log 2>&1
tail -1 gpurun_out/ncu.log
