set -x
TAG=${TAG:-r1n}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for o in 4 6 8; do
HELM_MARCH_OCC=$o HELM_DEBUG=1 timeout 300 python scripts/tune_plane.py cfg2 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
done
HELM_MARCH_OCC=6 HELM_DEBUG=1 timeout 300 python scripts/tune_plane.py cfg2 c64 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
for o in 4 6; do
HELM_MARCH_OCC=$o timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-matvec > gpurun_out/${TAG}_bench_occ$o.json 2> gpurun_out/${TAG}_bench_occ$o.err; echo "bench rc=$?"
done
echo done
