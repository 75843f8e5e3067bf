#!/bin/bash
OUT=gpurun_out/${1:-l2}; mkdir -p $OUT
BHT_DIRECT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scenarios.py -x -q -m gpu 2>&1 | tail -15 | tee $OUT/pytest_direct.txt
timeout 600 python tools/exp_blocked.py 2>&1 | tee $OUT/blocked.txt
BHT_DIRECT=2 BHT_REGION_MB=48 BHT_BLOCKED_CTAS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_insert -s 2 -c 1 -f -o $OUT/prof_insert_routed_direct \
   python tools/exp_blocked_one.py > $OUT/ncu_insert_routed_direct.log 2>&1
ls -la $OUT
