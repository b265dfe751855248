#!/bin/bash
# (box) Configs 3 and 4 artefacts: one-GPU bench lines (`bench.py --config 3|4`) and one `ncu --set full`
# capture of each one's solve kernel (config 3: K1, two lanes per step; config 4: K1L) in the bench's
# precision (hybrid), on the bench's own workload.  Also the early-stop fuzz parity report (batch_fuzz).
mkdir -p gpurun_out
python tools/batch_parity.py batch_fuzz > gpurun_out/fuzz_parity.log 2>&1; echo "fuzz parity rc=$?"
python bench.py --config 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "bench cfg3 rc=$?"
python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sf_persistent -s 1 -c 1 -o gpurun_out/full_cfg3_hybrid \
    python tools/prof_case.py --config 3 --batch 4096 --reps 2 --precision hybrid > gpurun_out/ncu_full_cfg3.log 2>&1
echo "ncu full cfg3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sf_large -s 1 -c 1 -o gpurun_out/full_cfg4_hybrid \
    python tools/prof_large.py hybrid 8192 1000 1 > gpurun_out/ncu_full_cfg4.log 2>&1
echo "ncu full cfg4 rc=$?"
