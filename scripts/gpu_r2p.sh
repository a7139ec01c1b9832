# Round 2, call P: continuous ring (HELM_CONT), last basis vector not stored (HELM_LASTV=0) and
# the CTA-level reduction tail (HELM_CTA_RED): parity of every path, then same-box A/B of the
# cfg4 probe table, cfg3 latency and the cfg4 bench, new (default) vs the previous schedule.
set -x
mkdir -p gpurun_out
T=r2p
OLD="HELM_CONT=0 HELM_LASTV=1 HELM_CTA_RED=0"
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_cfg3.py tests/test_gpu_repro.py tests/test_gpu_taylor3d.py -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_new.jsonl 2>&1
env $OLD timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_old.jsonl 2>&1
HELM_CONT=0 timeout 600 python scripts/probe_table.py cfg4 8 c128 1 > gpurun_out/${T}_probe_L1_nocont.jsonl 2>&1
HELM_CTA_RED=0 timeout 600 python scripts/probe_table.py cfg4 8 c128 1 2 > gpurun_out/${T}_probe_L12_warpred.jsonl 2>&1
timeout 600 python scripts/probe_table.py cfg3 1 c128 0 1 2 > gpurun_out/${T}_probe_cfg3_new.jsonl 2>&1
env $OLD timeout 600 python scripts/probe_table.py cfg3 1 c128 0 1 2 > gpurun_out/${T}_probe_cfg3_old.jsonl 2>&1
timeout 600 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_new.json 2>&1
env $OLD timeout 600 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_old.json 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_new.json 2> gpurun_out/${T}_bench_new.err
echo "bench new rc=$?"
env $OLD timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_old.json 2> gpurun_out/${T}_bench_old.err
echo "bench old rc=$?"
name=${T}_cfg4_L1_k3_nv2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
    -o /tmp/${name} python scripts/ncu_targets.py probe cfg4_8 1 3 2 > gpurun_out/${name}_ncu.log 2>&1
echo "ncu rc=$?"
if [ -f /tmp/${name}.ncu-rep ]; then
  ncu -i /tmp/${name}.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
  ncu -i /tmp/${name}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${name}_sass.csv.gz
  ncu -i /tmp/${name}.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > gpurun_out/${name}_cuda.csv.gz
fi
du -sh gpurun_out
