# Round evidence: (1) plain bench, then the ncu launch list of the same command (a window of
# launches inside the timed step); (2) ncu --set full of the dominant kernel class at its
# level: the five fused GMRES Arnoldi steps at level 1, joint batch of 150 RHS (cfg2).
set -x
TAG=${TAG:-r1u}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-matvec"
$CMD > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err &&
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 500000 -c 4000 --csv \
    --log-file gpurun_out/${TAG}_bench_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for spec in "3 0" "3 1" "3 2" "3 3" "4 4"; do
  set -- $spec
  name=${TAG}_L1_k$1_nv$2
  python scripts/ncu_targets.py probe cfg2_150 1 $1 $2 > gpurun_out/${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_march -s 2 -c 1 \
      -o gpurun_out/${name} python scripts/ncu_targets.py probe cfg2_150 1 $1 $2 > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  if [ -f gpurun_out/${name}.ncu-rep ]; then
    ncu -i gpurun_out/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${name}.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
    gzip -f gpurun_out/${name}_sass.csv
    rm -f gpurun_out/${name}.ncu-rep
  fi
done
du -sh gpurun_out
