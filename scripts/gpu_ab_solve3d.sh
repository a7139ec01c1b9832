# same-box A/B of the 3D solve over library variants ($VARIANTS, "" = default) and sizes.
for rep in 1 2; do
for v in ${VARIANTS:-cur py34}; do
  for spec in ${SPECS:-"96,8,c128" "128,8,c128" "128,8,c64"}; do
    IFS=, read n b d <<< "$spec"
    if [ "$v" = cur ]; then unset HELM_LIB_VARIANT; else export HELM_LIB_VARIANT=$v; fi
    timeout 300 python scripts/solve3d.py $n $b $d 2 2>&1 | tail -1 | cut -c1-400
  done
done; done
