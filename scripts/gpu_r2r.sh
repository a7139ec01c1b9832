# Round 2, call R: staged Krylov epilogue (KStage) + single ring for the last fused step
# (HELM_SPLIT=0 default): the full GPU suite, then probe tables (cfg4, cfg3), cfg3 latency,
# and the cfg4 bench, default vs the round-2 HEAD schedule.
set -x
mkdir -p gpurun_out
T=r2r
OLD="HELM_CONT=0 HELM_LASTV=1 HELM_CTA_RED=0 HELM_SPLIT=1"
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_def.jsonl 2>&1
timeout 600 python scripts/probe_table.py cfg3 1 c128 0 1 2 > gpurun_out/${T}_probe_cfg3_def.jsonl 2>&1
HELM_CTA_RED=0 timeout 600 python scripts/probe_table.py cfg3 1 c128 0 1 2 > gpurun_out/${T}_probe_cfg3_warpred.jsonl 2>&1
timeout 600 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_def.json 2>&1
env $OLD timeout 600 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_old.json 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_new.json 2> gpurun_out/${T}_bench_new.err
echo "bench new rc=$?"
env $OLD timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_old.json 2> gpurun_out/${T}_bench_old.err
echo "bench old rc=$?"
du -sh gpurun_out
