#!/bin/bash
# ncu --set full of one kernel kind from tools/prof_parts.py, skipping the first
# SKIP matching launches: tools/profile_one.sh TAG KERNEL SKIP COUNT
tag=$1; k=$2; skip=$3; c=$4
NCU=${NCU:-ncu}
timeout 600 $NCU --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"^${k}" --launch-skip $skip -c $c -f -o gpurun_out/${tag}_${k} python tools/prof_parts.py \
  > gpurun_out/${tag}_${k}.log 2>&1
echo "$k rc=$?"
$NCU -i gpurun_out/${tag}_${k}.ncu-rep --page raw --csv > gpurun_out/${tag}_${k}_raw.csv 2>/dev/null
python tools/summarize_ncu.py --report gpurun_out/${tag}_${k}.ncu-rep > gpurun_out/${tag}_${k}.md 2>&1
sz=$(stat -c %s gpurun_out/${tag}_${k}.ncu-rep 2>/dev/null || echo 0)
[ "$sz" -gt 12000000 ] && rm -f gpurun_out/${tag}_${k}.ncu-rep
true
