#!/bin/bash
# Round-2 GPU visit: parity tests, smoke, bench (both arms, every named config, the sharded path), ncu launch list and
# full captures with the atomic counters, the L2-resident table beside the HBM-resident one, the sweep.
# Usage (from the repo root, under gpurun):  bash tools/gpu_round2.sh <tag> [tests smoke bench benchref configs sharded ncu l2 sweep success]
TAG=${1:-r02}; shift
WHAT=${@:-tests smoke bench benchref configs sharded ncu l2 sweep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
ATOM=lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum.per_second,lts__t_requests_srcunit_tex_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt
for w in $WHAT; do
  case $w in
    tests) timeout 2400 python -m pytest tests --maxfail=8 -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log; tail -4 $OUT/pytest_gpu.log;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -3 $OUT/smoke.log;;
    bench) timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?"; cut -c1-200 $OUT/bench.json; tail -3 $OUT/bench.err;;
    benchref) timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cut -c1-300 $OUT/bench_ref.json;;
    configs)
      for c in bcht08 bcht099 1cht08 1cht09 bp2ht06 bp2ht08 bp2ht084 iht08 iht09 iht099; do
        timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "$c exit $?"; done;;
    sharded)
      timeout 600 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_sharded_50m.json 2> $OUT/bench_sharded_50m.err
      timeout 900 python bench.py --sharded --keys 500000000 --chunk 16777216 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_sharded_500m.json 2> $OUT/bench_sharded_500m.err
      timeout 900 python bench.py --device-keys --keys 500000000 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_single_500m.json 2> $OUT/bench_single_500m.err
      ls -la $OUT | grep 500m;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
          python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
      timeout 900 ncu --set full --metrics $ATOM --clock-control none --import-source on -k regex:bulk_find_kernel -s 3 -c 1 -f -o $OUT/prof_find \
          python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_find.log 2>&1
      timeout 900 ncu --set full --metrics $ATOM --clock-control none --import-source on -k regex:"group_scatter|bin_split|region_build|bulk_insert_cuckoo" -s 12 -c 4 -f -o $OUT/prof_build \
          python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_build.log 2>&1
      timeout 900 ncu --set full --metrics $ATOM --clock-control none --import-source on -k regex:"claim_insert|bulk_find" -s 6 -c 2 -f -o $OUT/prof_bp2ht \
          python bench.py --config bp2ht08 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_bp2ht.log 2>&1
      for r in find build bp2ht; do python tools/ncu_summary.py $OUT/prof_$r.ncu-rep --out $OUT/ncu_$r.txt > /dev/null; done
      python tools/ncu_summary.py $OUT/prof_find.ncu-rep --traffic-json $OUT/traffic.json > /dev/null
      python tools/ncu_summary.py $OUT/prof_build.ncu-rep --traffic-json $OUT/traffic.json > /dev/null
      ls -la $OUT | head -40;;
    l2)
      timeout 300 python tools/exp_l2_resident.py > $OUT/l2_resident.txt 2>&1; cat $OUT/l2_resident.txt
      timeout 300 python tools/exp_l2_resident.py 50000000 > $OUT/hbm_resident.txt 2>&1; cat $OUT/hbm_resident.txt
      timeout 900 ncu --set full --metrics $ATOM --clock-control none -k regex:"bulk_insert_cuckoo|bulk_find" -s 9 -c 3 -f -o $OUT/prof_l2 python tools/exp_l2_resident.py > $OUT/ncu_l2.log 2>&1
      timeout 900 ncu --set full --metrics $ATOM --clock-control none -k regex:"bulk_insert_cuckoo|bulk_find" -s 9 -c 3 -f -o $OUT/prof_hbm python tools/exp_l2_resident.py 50000000 > $OUT/ncu_hbm.log 2>&1
      python tools/ncu_summary.py $OUT/prof_l2.ncu-rep --out $OUT/ncu_l2_resident_100mb.txt > /dev/null
      python tools/ncu_summary.py $OUT/prof_hbm.ncu-rep --out $OUT/ncu_hbm_resident_444mb.txt > /dev/null;;
    sweep) timeout 1500 python tools/sweep.py --out $OUT/sweep_all_configs.json > $OUT/sweep_all_configs.txt 2>&1; tail -30 $OUT/sweep_all_configs.txt;;
    success) timeout 2400 python tools/paper_scale.py --success-trials 200 --trials 3 --out-prefix $OUT/paper_scale > $OUT/paper_scale.txt 2>&1; tail -40 $OUT/paper_scale.txt;;
    *) echo "unknown step $w";;
  esac
done
