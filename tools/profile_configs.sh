#!/bin/bash
# ncu --set full of the cfg3 / cfg4 / cfg5 hot kernels (one launch each, after a warm-up) -> gpurun_out/
R=${1:-r02}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:merge_async_kernel -s 1 -c 1 -f -o gpurun_out/prof_cfg5_$R \
  python tools/cfg_one.py 5 > gpurun_out/ncu_cfg5.log 2>&1; echo "cfg5 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"attn_tile8_kernel|attention_vsmem_kernel|attention_kernel" -s 2 -c 2 -f \
  -o gpurun_out/prof_cfg4_$R python tools/cfg_one.py 4 > gpurun_out/ncu_cfg4.log 2>&1; echo "cfg4 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:coltile_tmem_kernel -s 1 -c 1 -f -o gpurun_out/prof_cfg3_$R \
  python tools/cfg_one.py 3 > gpurun_out/ncu_cfg3.log 2>&1; echo "cfg3 rc=$?"
