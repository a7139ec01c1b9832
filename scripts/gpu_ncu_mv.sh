# ncu --set full of one helm_apply k_plane launch per spec "N dtype b" (after a plain run).
set -x
TAG=${TAG:-r1mv}
SPECS=${SPECS:-"256 c64 1;512 c128 4"}
IFS=';' read -ra ARR <<< "$SPECS"
for spec in "${ARR[@]}"; do
  set -- $spec
  name=${TAG}_mv$1_$2_b$3
  python scripts/ncu_targets.py matvec $spec > gpurun_out/${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
      -o gpurun_out/${name} python scripts/ncu_targets.py matvec $spec > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  if [ -f gpurun_out/${name}.ncu-rep ]; then
    ncu -i gpurun_out/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${name}.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
    gzip -f gpurun_out/${name}_sass.csv
    sz=$(stat -c %s gpurun_out/${name}.ncu-rep); [ "$sz" -gt 12000000 ] && rm -f gpurun_out/${name}.ncu-rep
  fi
done
