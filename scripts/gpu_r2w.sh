# Round 2, call W: MODE-0 matvec with the register z-1 plane for complex64 and grids <= 24 M
# points (sweep ab_r2u), first fused step at 5 CTAs/SM: parity, the 24-cell sweep with the new
# defaults, probe, bench; ncu --set full of the latency-bound 128^3 matvec cells.
set -x
mkdir -p gpurun_out
T=r2w
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_operator.py tests/test_gpu_cfg5.py tests/test_gpu_solve.py -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
timeout 900 python scripts/matvec_sweep.py > gpurun_out/${T}_mv_def.jsonl 2> gpurun_out/${T}_mv_def.err
timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_def.jsonl 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for spec in "128 c128 1" "128 c64 1"; do
  set -- $spec
  name=${T}_mv$1_$2_b$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plane -s 3 -c 1 \
      -o /tmp/${name} python scripts/ncu_targets.py matvec $1 $2 $3 > gpurun_out/${name}_ncu.log 2>&1
  if [ -f /tmp/${name}.ncu-rep ]; then
    ncu -i /tmp/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    ncu -i /tmp/${name}.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
  fi
done
du -sh gpurun_out
