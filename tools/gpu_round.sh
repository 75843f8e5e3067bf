#!/bin/bash
# One GPU-box visit: parity tests, smoke, bench, ncu launch list and full captures of the two hot kernels.
# Usage (from the repo root, under gpurun):  bash tools/gpu_round.sh <tag> [tests|bench|ncu ...]
TAG=${1:-r01}; shift
WHAT=${@:-tests smoke bench ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests --maxfail=8 -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -5 $OUT/pytest_gpu.log;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -3 $OUT/smoke.log;;
    bench) timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"; cat $OUT/bench.json; tail -5 $OUT/bench.err;;
    benchref) timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cat $OUT/bench_ref.json;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
          python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_find_kernel -s 3 -c 1 -f -o $OUT/prof_find \
          python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_find.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_insert -s 3 -c 1 -f -o $OUT/prof_insert \
          python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_insert.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:"group_scatter|bin_split|region_build" -s 9 -c 3 -f -o $OUT/prof_route \
          python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_route.log 2>&1
      ls -la $OUT;;
    *) echo "unknown step $w";;
  esac
done
