#!/bin/bash
# parity tests of the blocked builds + timing + ncu launch list / full capture of the blocked-build kernels
OUT=gpurun_out/${1:-smem}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -8 | tee $OUT/pytest.txt
timeout 300 python tools/exp_smem.py 2>&1 | tee $OUT/exp.txt | tail -5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/exp_smem_one.py > $OUT/l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bin_split|region_build|bulk_insert|route_scatter" -s 8 -c 4 -f -o $OUT/prof python tools/exp_smem_one.py > $OUT/p.log 2>&1
tail -2 $OUT/p.log
