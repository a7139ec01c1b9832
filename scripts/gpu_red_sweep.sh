# HELM_MARCH_RED sweep: t(B) per outer cycle (scripts/batch_tail.py) and the bench step.
for R in ${REDS:-0 4 8 16}; do
  HELM_MARCH_RED=$R timeout 600 python scripts/batch_tail.py > gpurun_out/tail_$R.json 2>&1
  python - "$R" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/tail_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("RED", sys.argv[1], {k: round(v, 1) for k, v in d["t_cycle_ms"].items()}, "pred", round(d["pred_batch_ms"]))
PY
done
COMBOS="cur HELM_MARCH_RED=0
cur HELM_MARCH_RED=8" STEPS=2 bash scripts/gpu_ab_bench.sh
