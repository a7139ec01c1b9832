# Round 2, call AA: full GPU suite with the early stop (R23) and the persistent graph cache;
# failed tests (if any) are rerun with a stricter early-stop factor and with full cycles to
# classify them; then the bench line at the driver's K/W and the launch list of its window.
set -x
mkdir -p gpurun_out
T=r2aa
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1
RC=$?
echo "tests rc=$RC"
tail -25 gpurun_out/${T}_tests.log
if [ $RC -ne 0 ]; then
  HELM_EARLY_PCT=50 timeout 1200 python -m pytest tests -q -m gpu --lf > gpurun_out/${T}_tests_lf_pct50.log 2>&1
  echo "lf pct50 rc=$?"; tail -8 gpurun_out/${T}_tests_lf_pct50.log
  HELM_EARLY=0 timeout 1200 python -m pytest tests -q -m gpu --lf > gpurun_out/${T}_tests_lf_early0.log 2>&1
  echo "lf early0 rc=$?"; tail -8 gpurun_out/${T}_tests_lf_early0.log
fi
( time python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err ) 2>&1 | tail -4
echo "bench rc=$?"
python - <<P
import json
d=json.loads(open("gpurun_out/${T}_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["e2e"], d["roofline"]["frac"], d["solve_roofline"], d["clocks"], d.get("wall_s"), d.get("skipped"), d.get("other_dtype"), d.get("cfg2"))
P
CMD="python bench.py --steps 1 --warmup 3 --no-matvec --no-cpu-baseline --no-extra"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 120000 -c 2000 --csv \
    --log-file gpurun_out/${T}_bench_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
echo "launch list rc=$?"
du -sh gpurun_out
