timeout 300 python tools/exp_smem.py 2>&1 | grep -E "smem|auto"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tmp.csv python tools/exp_smem_one.py > /dev/null 2>&1
