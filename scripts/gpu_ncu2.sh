set -x
TAG=${TAG:-r1e}
for spec in "cfg2 0 0 0" "cfg2 0 3 2" "mv256 0 0 0"; do
  set -- $spec
  name=${TAG}_$1_L$2_k$3_nv$4
  python scripts/ncu_targets.py probe $spec > gpurun_out/${name}_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
      -o gpurun_out/${name} python scripts/ncu_targets.py probe $spec > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
done
