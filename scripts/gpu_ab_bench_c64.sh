# same-box A/B of the complex64 bench step over env settings ($COMBOS lines).
for rep in 1 2; do
echo "$COMBOS" | while read -r envs; do
  [ -z "$envs" ] && continue
  env $envs timeout 600 python bench.py --dtype c64 --steps 2 --warmup 3 --no-cpu-baseline --no-matvec > gpurun_out/abc.json 2> gpurun_out/abc.err
  python - "$envs" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abc.json").read().strip().splitlines()[-1])
print(sys.argv[1], "|", d["value"], "solves/s", "L1 arnoldi", d["roofline"]["achieved"], d["roofline"]["frac"])
PY
done; done
