# k_plane occupancy-target sweep on the cfg5 matvec (TMA on).
for O in ${OCCS:-4 6 8}; do
  HELM_PLANE_OCC=$O timeout 300 python scripts/matvec_sweep.py --N ${MVN:-256,512} --dtype ${MVD:-c64,c128} --b ${MVB:-1,4} > gpurun_out/mv_occ$O.jsonl 2>&1
  echo "OCC=$O rc=$?"
  python - "$O" <<'PY'
import json, sys
for l in open(f"gpurun_out/mv_occ{sys.argv[1]}.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["N"], d["dtype"], d["b"], round(d["ms_median"], 4), round(d["GBps"]), round(d["frac_measured"], 3))
PY
done
