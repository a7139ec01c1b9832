set -x
TAG=${TAG:-r1c}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python scripts/matvec_sweep.py --N 256,512 --dtype c128,c64 --b 1,4 > gpurun_out/${TAG}_matvec.jsonl 2>&1; echo "sweep rc=$?"
timeout 600 python scripts/profile_levels.py --dtype c128 > gpurun_out/${TAG}_levels_c128.json 2>&1; echo "levels rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
if [ -n "$NCU" ]; then
python scripts/ncu_targets.py cfg2 > gpurun_out/${TAG}_plain_cfg2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 5000 --csv \
    --log-file gpurun_out/${TAG}_launches_cfg2_warm.csv python scripts/ncu_targets.py cfg2 > gpurun_out/${TAG}_ncu1.log 2>&1
echo "launches rc=$?"
fi
