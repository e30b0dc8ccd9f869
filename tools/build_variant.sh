#!/bin/bash
# Build libstc.so with extra -D flags into ab/<name>.so (A/B experiments): tools/build_variant.sh name -DX=1 ...
name=$1; shift
mkdir -p ab/$name.obj
P=paper_2405_16883_b200
pids=()
for src in abi_common spmm spmm_wide mttkrp_prepared attention spgemm construct; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
    -I include -c $P/csrc/$src.cu -o ab/$name.obj/$src.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || exit 1; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/$name.so ab/$name.obj/*.o && rm -rf ab/$name.obj && echo ab/$name.so
