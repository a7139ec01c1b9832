# Round 2, call Z: early stop inside the outer FGMRES cycle (R23). New parity tests, the solve
# tests, and a same-box A/B of the bench headline (HELM_EARLY=0 full cycles vs the default).
set -x
mkdir -p gpurun_out
T=r2z
timeout 1500 python -m pytest tests/test_gpu_early_stop.py tests/test_gpu_solve.py tests/test_gpu_fwi.py -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -15 gpurun_out/${T}_tests.log
for E in 0 1; do
  HELM_EARLY=$E timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra \
      > gpurun_out/${T}_bench_early$E.json 2> gpurun_out/${T}_bench_early$E.err
  echo "bench early=$E rc=$?"
  python - <<P
import json
d=json.loads(open("gpurun_out/${T}_bench_early$E.json").read().strip().splitlines()[-1])
print("early=$E", d["value"], d["ms_per_step"], d["config"]["outer_cycles_last_step"], d["roofline"]["frac"], d["solve_roofline"], d["clocks"])
P
done
for E in 0 1; do
  HELM_EARLY=$E timeout 600 python bench.py --workload cfg2 --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra \
      > gpurun_out/${T}_bench_cfg2_early$E.json 2> gpurun_out/${T}_bench_cfg2_early$E.err
  echo "cfg2 early=$E rc=$?"
  python - <<P
import json
d=json.loads(open("gpurun_out/${T}_bench_cfg2_early$E.json").read().strip().splitlines()[-1])
print("cfg2 early=$E", d["value"], d["ms_per_step"], d["config"]["outer_cycles_last_step"]["mean"])
P
done
HELM_EARLY=0 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_early0.json 2>&1; tail -2 gpurun_out/${T}_cfg3_early0.json
HELM_EARLY=1 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_early1.json 2>&1; tail -2 gpurun_out/${T}_cfg3_early1.json
