set -x
TAG=${TAG:-r1z3}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for t in 1 0; do
HELM_TMA=$t timeout 600 python scripts/matvec_sweep.py --N 256,512 --dtype c128 --b 1,4 > gpurun_out/${TAG}_mv_tma$t.jsonl 2>&1
python - <<PY
import json
for l in open('gpurun_out/${TAG}_mv_tma$t.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('tma=$t', d['N'], d['dtype'], d['b'], round(d['GBps']), round(d['frac_measured'],3))
PY
HELM_TMA=$t timeout 300 python scripts/tune_plane.py mv256 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
HELM_TMA=$t timeout 300 python scripts/tune_plane.py cfg3 c128 >> gpurun_out/${TAG}_tune.jsonl 2>>gpurun_out/${TAG}_tune.err
done
echo done
