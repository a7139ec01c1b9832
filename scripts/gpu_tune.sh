set -x
TAG=${TAG:-r1d}
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for occ in 1 2 3 4; do
  HELM_PLANE_OCC=$occ timeout 300 python scripts/tune_plane.py cfg2 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
  HELM_PLANE_OCC=$occ timeout 300 python scripts/tune_plane.py mv256 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
done
for s in 4 6 8; do
  HELM_PLANE_S=$s timeout 300 python scripts/tune_plane.py cfg2 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
done
HELM_PLANE_OCC=2 timeout 300 python scripts/tune_plane.py cfg2 c64 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
HELM_PLANE_OCC=2 timeout 300 python scripts/tune_plane.py cfg3 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
echo done
