#!/bin/bash
# A/B of library variants on the blocked build: timing + check, then an ncu launch list per variant.
# Usage (under gpurun): bash tools/build_round.sh <tag> [variant ...]   ("" = the default library)
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in default "$@"; do
  if [ "$v" = default ]; then unset BHT_B200_LIB; else export BHT_B200_LIB=$PWD/paper_2108_07232_b200/lib/libbht_b200_$v.so; fi
  timeout 300 python tools/exp_build_phases.py 2>&1 | tail -2 | tee -a $OUT/phases.txt
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$v.csv python tools/exp_smem_one.py > $OUT/l_$v.log 2>&1
  python - <<PY | tee -a $OUT/phases.txt
import csv
rows = [r for r in csv.reader(open("$OUT/launches_$v.csv")) if len(r) > 5 and r[0].isdigit()]
last = {}
for r in rows:
    name = r[4].split("(")[0].split("::")[-1][:40]
    last[name] = float(r[-1].replace(",", ""))
print("  ncu last launch (us):", {k: round(v / 1e3, 1) if v > 5000 else v for k, v in last.items()})
PY
done
