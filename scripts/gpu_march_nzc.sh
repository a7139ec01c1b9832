# k_march2d z-chunk count sweep (HELM_MARCH_NZC forces it on every level) on cfg2 at 150 RHS:
# level-1 and level-2 fused-step GB/s; the auto choice is printed by HELM_DEBUG=2.
HELM_DEBUG=2 timeout 300 python scripts/tune_plane.py cfg2 c128 150 2>&1 | grep "march2d nx" | sort | uniq | head -12
for n in 0 1 2 3 4 5 6 8 10; do
  HELM_MARCH_NZC=$n timeout 300 python scripts/tune_plane.py cfg2 c128 150 > gpurun_out/nzc.json 2>&1
  python - "$n" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/nzc.json").read().strip().splitlines()[-1])
r = d["rows"]
f = lambda l, k: " ".join(f'{x["nv"]}:{x["GBps"]:.0f}' for x in r if x.get("level") == l and x.get("kind") == k)
vc = " ".join(f'L{x["level"]}:{x["vcycle_ms"]}' for x in r if "vcycle_ms" in x)
print("nzc", sys.argv[1], "| L1", f(1, 3), f(1, 4), "| L2", f(2, 3), "| vcycle", vc)
PY
done
