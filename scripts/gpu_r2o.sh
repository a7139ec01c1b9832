# Round 2, call O: continuous ring across a CTA's items for the fused Arnoldi steps (HELM_CONT).
# Parity of every stage path, then same-box A/B of the per-kernel probe table at cfg4 (levels
# 0-2, 8 RHS) and of the bench, cont on / off; ncu --set full (source) of the level-1 step 2.
set -x
mkdir -p gpurun_out
T=r2o
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_cfg3.py -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
for c in 1 0; do
  HELM_CONT=$c timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_cont$c.jsonl 2>&1
done
for hw in 0 5 20; do
  HELM_CONT_HW10=$hw timeout 600 python scripts/probe_table.py cfg4 8 c128 1 > gpurun_out/${T}_probe_L1_hw$hw.jsonl 2>&1
done
for c in 1 0; do
  HELM_CONT=$c timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_cont$c.json 2> gpurun_out/${T}_bench_cont$c.err
  echo "bench cont=$c rc=$?"
done
name=${T}_cfg4_L1_k3_nv2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
    -o gpurun_out/${name} python scripts/ncu_targets.py probe cfg4_8 1 3 2 > gpurun_out/${name}_ncu.log 2>&1
echo "ncu rc=$?"
if [ -f gpurun_out/${name}.ncu-rep ]; then
  ncu -i gpurun_out/${name}.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
  ncu -i gpurun_out/${name}.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
  ncu -i gpurun_out/${name}.ncu-rep --page source --csv --print-source cuda > gpurun_out/${name}_cuda.csv 2>/dev/null
fi
