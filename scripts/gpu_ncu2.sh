# ncu --set full of single probe kernels; exports raw + SASS-source CSVs on the box and keeps
# the .ncu-rep only when small (gpurun brings back <= 64 MiB).
set -x
TAG=${TAG:-r1e}
SPECS=${SPECS:-"cfg2 0 0 0;cfg2 0 3 2;mv256 0 0 0"}
IFS=';' read -ra ARR <<< "$SPECS"
for spec in "${ARR[@]}"; do
  set -- $spec
  name=${TAG}_$1_L$2_k$3_nv$4
  python scripts/ncu_targets.py probe $spec > gpurun_out/${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_plane} -s 2 -c 1 \
      -o gpurun_out/${name} python scripts/ncu_targets.py probe $spec > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  if [ -f gpurun_out/${name}.ncu-rep ]; then
    ncu -i gpurun_out/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${name}.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
    ncu -i gpurun_out/${name}.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
    gzip -f gpurun_out/${name}_sass.csv
    sz=$(stat -c %s gpurun_out/${name}.ncu-rep); [ "$sz" -gt 12000000 ] && rm -f gpurun_out/${name}.ncu-rep
  fi
done
du -sh gpurun_out
