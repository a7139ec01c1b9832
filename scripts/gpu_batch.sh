set -x
TAG=${TAG:-r1i}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 --max-rhs 50 --no-cpu-baseline --no-matvec > gpurun_out/${TAG}_bench50.json 2> gpurun_out/${TAG}_bench50.err; echo "bench50 rc=$?"
echo done
