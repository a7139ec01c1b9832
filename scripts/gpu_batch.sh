set -x
TAG=${TAG:-r1zc}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python scripts/tune_plane.py mv256 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
timeout 300 python scripts/tune_plane.py cfg3 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
for gr in 1 0; do
HELM_GRAPHS=$gr timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-matvec > gpurun_out/${TAG}_bench_g$gr.json 2> gpurun_out/${TAG}_bench_g$gr.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_g$gr.json'));print('bench graphs=$gr', d['value'], d['gpu_launches'], d['level_shares'])"
done
echo done
