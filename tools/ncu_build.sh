#!/bin/bash
# ncu --set full capture of the blocked-build kernels (one launch each, warm) + text summary.  bash tools/ncu_build.sh <tag>
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"group_scatter|bin_split|region_build|bulk_insert_cuckoo" -s 8 -c 4 -f -o $OUT/prof_build python tools/exp_smem_one.py > $OUT/ncu_build.log 2>&1
tail -2 $OUT/ncu_build.log
python tools/ncu_summary.py $OUT/prof_build.ncu-rep --out $OUT/ncu_build_summary.txt > /dev/null
