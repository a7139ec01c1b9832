# same-box A/B: m/z by TMA (HELM_TMA_MZ=1) vs per-thread cp.async (0), occupancy 4 and 8, twice.
for rep in 1 2; do
for O in 4 8; do for M in 1 0; do
  HELM_PLANE_OCC=$O HELM_TMA_MZ=$M timeout 300 python scripts/matvec_sweep.py --N ${MVN:-256,512} --dtype c64,c128 --b 1,4 > gpurun_out/ab.jsonl 2>&1
  python - "$O" "$M" <<'PY'
import json, sys
out = []
for l in open("gpurun_out/ab.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); out.append(f'{d["N"]}{d["dtype"]}b{d["b"]}:{d["ms_median"]:.4f}/{d["frac_measured"]:.3f}')
print("occ", sys.argv[1], "mz", sys.argv[2], " ".join(out))
PY
done; done; done
