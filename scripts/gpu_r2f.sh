# Round 2, call F: persistent coarse V-cycle — parity, latency A/B (cfg3, Table 3 43^3), GPU
# suite, the full default bench line.
set -x
mkdir -p gpurun_out
T=r2f
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_paths.py tests/test_gpu_guards.py -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_persist.json 2> gpurun_out/${T}_cfg3_persist.err
HELM_PERSIST=0 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_seq.json 2> gpurun_out/${T}_cfg3_seq.err
python bench.py --workload cfg2 --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_cfg2.json 2> gpurun_out/${T}_bench_cfg2.err
HELM_PERSIST=0 python bench.py --workload cfg2 --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_cfg2_seq.json 2> gpurun_out/${T}_bench_cfg2_seq.err
python bench.py --steps 3 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_gputests.log 2>&1
echo "gpu tests rc=$?"
