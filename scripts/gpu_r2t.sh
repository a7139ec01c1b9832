# Round 2, call T: closing evidence for the GMRES-tail kernels — full GPU suite (+ the
# persistent-V-cycle path three more times: r2r saw one non-converged solve there), the default
# bench line at the driver's K/W, the bench command's ncu launch list, ncu --set full of the
# five level-1 fused steps.
set -x
mkdir -p gpurun_out
T=r2t
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
for i in 1 2 3; do
  timeout 600 python -m pytest "tests/test_gpu_paths.py::test_alternative_stage_paths_match_oracle[persistent_vcycle]" -q -m gpu >> gpurun_out/${T}_persist_rep.log 2>&1
  echo "persist rep $i rc=$?"
done
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-matvec --no-cpu-baseline --no-extra"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 120000 -c 2000 --csv \
    --log-file gpurun_out/${T}_bench_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for spec in "3 0" "3 1" "3 2" "3 3" "4 4"; do
  set -- $spec
  name=${T}_cfg4_L1_k$1_nv$2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
      -o /tmp/${name} python scripts/ncu_targets.py probe cfg4_8 1 $1 $2 > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  if [ -f /tmp/${name}.ncu-rep ]; then
    ncu -i /tmp/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    ncu -i /tmp/${name}.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
  fi
done
du -sh gpurun_out
