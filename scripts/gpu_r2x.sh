# Round 2, call X: TMA-fed 2D march ring — parity of both feeds, same-box A/B
# of the cfg2 probe table and cfg2 bench (HELM_MARCH_TMA=1 default vs 0), ncu --set full of the
# level-1 2D fused steps with each feed; the matvec sweep with kernel-only timing; set_active
# no longer re-uploads an unchanged active list.
set -x
mkdir -p gpurun_out
T=r2x
timeout 1500 python -m pytest tests/test_gpu_march_paths.py tests/test_gpu_fwi.py tests/test_gpu_operator.py tests/test_gpu_opt_stencil.py tests/test_gpu_solve.py tests/test_gpu_fullsize.py -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
for t in 1 0; do
  HELM_MARCH_TMA=$t timeout 600 python scripts/probe_table.py cfg2 150 c128 0 1 2 > gpurun_out/${T}_probe_cfg2_tma$t.jsonl 2>&1
  HELM_MARCH_TMA=$t timeout 900 python bench.py --workload cfg2 --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench_cfg2_tma$t.json 2> gpurun_out/${T}_bench_cfg2_tma$t.err
done
for t in 1 0; do
  for spec in "3 2" "4 4"; do
    set -- $spec
    name=${T}_cfg2_L1_k$1_nv$2_tma$t
    HELM_MARCH_TMA=$t timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_march2d -s 2 -c 1 \
        -o /tmp/${name} python scripts/ncu_targets.py probe cfg2 1 $1 $2 > gpurun_out/${name}_ncu.log 2>&1
    if [ -f /tmp/${name}.ncu-rep ]; then
      ncu -i /tmp/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    fi
  done
done
timeout 900 python scripts/matvec_sweep.py > gpurun_out/${T}_mv_def.jsonl 2> gpurun_out/${T}_mv_def.err
du -sh gpurun_out
