# Round 2, call AC: choose the early-stop factor (HELM_EARLY_PCT) — the largest of 50 / 30 whose
# fast parity tests (north star's 1e-5 on f, g and solutions at rtol 1e-6) pass — then the full
# GPU suite and the bench line at the driver's K/W with that factor.
set -x
mkdir -p gpurun_out
T=r2ac
PICK=0
for PCT in 50 30; do
  HELM_EARLY_PCT=$PCT timeout 900 python -m pytest tests/test_gpu_fwi.py tests/test_gpu_solve.py -q -m gpu > gpurun_out/${T}_fast_pct$PCT.log 2>&1
  RC=$?
  echo "fast tests pct=$PCT rc=$RC"; tail -4 gpurun_out/${T}_fast_pct$PCT.log
  if [ $RC -eq 0 ]; then PICK=$PCT; break; fi
done
echo "PICK=$PICK"
if [ $PICK -eq 0 ]; then export HELM_EARLY=0; else export HELM_EARLY_PCT=$PICK; fi
echo $PICK > gpurun_out/${T}_pick.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -12 gpurun_out/${T}_tests.log
( time python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err ) 2>&1 | tail -4
echo "bench rc=$?"
python - <<P
import json
d=json.loads(open("gpurun_out/${T}_bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["e2e"], d["roofline"]["frac"], d["solve_roofline"], d["clocks"], d.get("wall_s"), d.get("skipped"), d.get("other_dtype"), (d.get("cfg2") or {}).get("value"))
P
HELM_EARLY_PCT=98 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_pct98.json 2>&1
python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_pick.json 2>&1; cut -c1-700 gpurun_out/${T}_cfg3_pick.json
