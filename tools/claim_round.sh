#!/bin/bash
# ncu --set full captures of the counter-claimed bp2ht / iht insert kernels and of the bucket-reading ones they replace.
OUT=gpurun_out/${1:-claim}; mkdir -p $OUT
for kind in bp2ht iht; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:claim_insert -s 2 -c 1 -f -o $OUT/prof_claim_$kind \
      python tools/exp_claim_one.py $kind 50000000 3 > $OUT/ncu_claim_$kind.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_insert -s 2 -c 1 -f -o $OUT/prof_read_$kind \
      python tools/exp_claim_one.py $kind 50000000 0 > $OUT/ncu_read_$kind.log 2>&1
done
tools/microbench/random_store > $OUT/random_store.txt 2>&1
ls -la $OUT
