#!/bin/bash
# (box) Round artefacts: GPU tests, the bench line, the ncu launch list of the bench command, and one
# `ncu --set full` capture of the persistent SF kernel per precision (hybrid = the bench's, lean).
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quick > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
for prec in hybrid lean; do
  ncu --set full --clock-control none --import-source on -k regex:sf_persistent -s 1 -c 1 -o gpurun_out/full_$prec \
      python tools/prof_case.py --reps 2 --precision $prec > gpurun_out/ncu_full_$prec.log 2>&1; echo "ncu full $prec rc=$?"
done
# K1L (config 4's kernel): one `ncu --set full` capture on a short config-4 run (1024 samples = one GPU's share at
# 8 GPUs, early stop, at most 200 iterations: the whole 8192-sample batch takes over 40 minutes of replays)
ncu --set full --clock-control none --import-source on -k regex:sf_large -s 1 -c 1 -o gpurun_out/full_cfg4_hybrid \
    python tools/prof_large.py hybrid 1024 200 1 > gpurun_out/ncu_full_cfg4.log 2>&1; echo "ncu full cfg4 rc=$?"
