# same-box A/B over environment settings: each line of $COMBOS is "ENV=val ENV2=val ..."
# run on the cfg5 matvec sweep ($MVN, $MVD, $MVB).
echo "$COMBOS" | while read -r combo; do
  [ -z "$combo" ] && continue
  env $combo timeout 300 python scripts/matvec_sweep.py --N ${MVN:-256,512} --dtype ${MVD:-c64,c128} --b ${MVB:-1,4} > gpurun_out/ab.jsonl 2>&1
  python - "$combo" <<'PY'
import json, sys
out = []
for l in open("gpurun_out/ab.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); out.append(f'{d["N"]}{d["dtype"]}b{d["b"]}:{d["ms_median"]:.4f}/{d["frac_measured"]:.3f}')
    elif "rror" in l:
        out.append(l.strip()[:100])
print(sys.argv[1], "|", " ".join(out))
PY
done
