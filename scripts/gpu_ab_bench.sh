# same-box A/B of the bench step (cfg2, joint batch) over library variants and env settings:
# each line of $COMBOS is "VARIANT [ENV=val ...]" (VARIANT "cur" = lib/libhelm.so).
for rep in 1 2; do
echo "$COMBOS" | while read -r v envs; do
  [ -z "$v" ] && continue
  if [ "$v" = cur ]; then V=""; else V="HELM_LIB_VARIANT=$v"; fi
  env $V $envs timeout 600 python bench.py --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-matvec > gpurun_out/abb.json 2> gpurun_out/abb.err
  python - "$v $envs" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/abb.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "|", d["value"], "solves/s", d["ms_per_step"], "ms", "L1 arnoldi", d["roofline"]["achieved"], "frac", d["roofline"]["frac"], d.get("level_shares"))
except Exception as e:
    print(sys.argv[1], "| failed", open("gpurun_out/abb.err").read()[-300:])
PY
done; done
