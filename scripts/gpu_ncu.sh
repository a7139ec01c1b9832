# ncu evidence for round 1: launch list of one cfg2 forward-solve outer cycle, and full
# captures of the level-0 fused stencil+projection kernel and of the cfg5 matvec.
set -x
TAG=${TAG:-r1}
python scripts/ncu_targets.py cfg2 > gpurun_out/${TAG}_plain_cfg2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/${TAG}_launches_cfg2.csv python scripts/ncu_targets.py cfg2 > gpurun_out/${TAG}_ncu1.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_plane -s 1 -c 2 \
    -o gpurun_out/${TAG}_cfg2_plane python scripts/ncu_targets.py cfg2 > gpurun_out/${TAG}_ncu2.log 2>&1
echo "full cfg2 rc=$?"
python scripts/ncu_targets.py matvec 256 c128 1 > gpurun_out/${TAG}_plain_mv.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
    -o gpurun_out/${TAG}_mv256_c128 python scripts/ncu_targets.py matvec 256 c128 1 > gpurun_out/${TAG}_ncu3.log 2>&1
echo "full mv rc=$?"
