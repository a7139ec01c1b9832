# Round 2, call Q: register fix (bare launch bound), loader without per-plane division,
# one-row-per-thread split last step (HELM_SPLIT_PY=1): parity, then same-box probe A/B at
# cfg4 (levels 0-2, 8 RHS): default / HELM_CONT=0 / HELM_CONT_HW10=20 / HELM_SPLIT_PY=1 /
# HELM_SPLIT=0, and the bench (default vs the round-2 HEAD schedule).
set -x
mkdir -p gpurun_out
T=r2q
OLD="HELM_CONT=0 HELM_LASTV=1 HELM_CTA_RED=0"
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_cfg3.py tests/test_gpu_repro.py -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_def.jsonl 2>&1
for e in "HELM_CONT=0" "HELM_CONT_HW10=20" "HELM_SPLIT_PY=1" "HELM_SPLIT=0"; do
  env $e timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_${e}.jsonl 2>&1
done
env $OLD timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_old.jsonl 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_new.json 2> gpurun_out/${T}_bench_new.err
echo "bench new rc=$?"
env $OLD timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_old.json 2> gpurun_out/${T}_bench_old.err
echo "bench old rc=$?"
HELM_DEBUG=1 timeout 300 python scripts/probe_table.py cfg4 8 c128 1 > gpurun_out/${T}_debug.jsonl 2> gpurun_out/${T}_debug.err
du -sh gpurun_out
