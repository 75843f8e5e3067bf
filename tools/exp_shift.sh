for d in 1 2; do BHT_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dbg$d.csv python tools/exp_smem_one.py > /dev/null 2>&1; done
