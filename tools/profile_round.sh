#!/bin/bash
# Round-end measurement on one B200 (outputs in gpurun_out/, summaries copied to profiles/ by hand):
#   bench line, ncu launch list of the bench command, ncu --set full of the dominant kernel,
#   the per-configuration table.
R=${1:-r02}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_${R}_bench_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:merge_kernel -s 2 -c 1 -f -o gpurun_out/prof_merge_$R \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/bench_configs.py --out gpurun_out/configs_$R.json > gpurun_out/configs_$R.log 2>&1; echo "configs rc=$?"
