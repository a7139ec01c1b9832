set -x
TAG=${TAG:-r1o}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
HELM_DEBUG=1 timeout 300 python scripts/tune_plane.py cfg2 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 --dtype c64 --no-cpu-baseline --no-matvec > gpurun_out/${TAG}_bench_c64.json 2> gpurun_out/${TAG}_bench_c64.err; echo "bench c64 rc=$?"
echo done
