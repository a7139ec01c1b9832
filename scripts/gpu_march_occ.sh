# k_march2d occupancy / ring-depth sweep on cfg2 with the bench's joint batch (150 RHS):
# per-level kernel GB/s (L1 fused steps dominate the bench) and V-cycle times.
for combo in "HELM_MARCH_OCC=4" "HELM_MARCH_OCC=5" "HELM_MARCH_OCC=6" "HELM_MARCH_OCC=8" "HELM_MARCH_OCC=4"; do
  env $combo timeout 300 python scripts/tune_plane.py cfg2 c128 150 > gpurun_out/mocc.json 2>&1
  python - "$combo" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/mocc.json").read().strip().splitlines()[-1])
r = d["rows"]
f = lambda l, k: " ".join(f'{x["nv"]}:{x["GBps"]:.0f}' for x in r if x.get("level") == l and x.get("kind") == k)
vc = " ".join(f'L{x["level"]}:{x["vcycle_ms"]}' for x in r if "vcycle_ms" in x)
print(sys.argv[1], "| L1 arnoldi", f(1, 3), f(1, 4), "| L0", f(0, 3), f(0, 4), "| L2", f(2, 3), "| vcycle", vc)
PY
done
