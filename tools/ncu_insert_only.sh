OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_insert -s 3 -c 1 -f -o $OUT/prof_insert python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_insert.log 2>&1
ls -la $OUT
