#!/bin/bash
# ncu --set full captures of the hot kernels, one kernel kind per capture
# (tools/prof_parts.py: V-cycle, CGS2 at kb=30, SpMV, fp64 residual), and the
# launch list of a short bench.py run (same command as the bench, reduced sizes).
# Reports are summarised on the box (raw-page CSV + markdown) and the large
# .ncu-rep files removed, so gpurun_out/ stays under the 64 MiB merge limit.
tag=${1:-full}
NCU=${NCU:-ncu}
for spec in "k_gs_pass:2" "k_spmv:2" "k_cgs2_fused:1" "k_gs_lower:2" "k_restrict:1"; do
  k=${spec%%:*}; c=${spec#*:}
  timeout 600 $NCU --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"^${k}" -c $c -f -o gpurun_out/${tag}_${k} python tools/prof_parts.py > gpurun_out/${tag}_${k}.log 2>&1
  echo "$k rc=$?"
  $NCU -i gpurun_out/${tag}_${k}.ncu-rep --page raw --csv > gpurun_out/${tag}_${k}_raw.csv 2>/dev/null
  python tools/summarize_ncu.py --report gpurun_out/${tag}_${k}.ncu-rep > gpurun_out/${tag}_${k}.md 2>&1
  sz=$(stat -c %s gpurun_out/${tag}_${k}.ncu-rep 2>/dev/null || echo 0)
  [ "$sz" -gt 12000000 ] && rm -f gpurun_out/${tag}_${k}.ncu-rep
done
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_bench_launches.csv \
  python bench.py --steps 1 --warmup 1 --max-iters 30 --no-validation --no-cpu > gpurun_out/${tag}_bench_launches.log 2>&1
echo "bench launches rc=$?"
python tools/summarize_ncu.py --launches gpurun_out/${tag}_bench_launches.csv > gpurun_out/${tag}_bench_launches.md 2>&1
gzip -f gpurun_out/${tag}_bench_launches.csv
du -sh gpurun_out
