set -x
TAG=${TAG:-r1x}
timeout 300 python -m pytest tests/test_gpu_operator.py tests/test_gpu_fullsize.py -k "apply or matvec or dot" -x -q > gpurun_out/${TAG}_pytest_mv.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_mv.log
for v in 1 0; do for o in 3 4 6; do
HELM_MV3D=$v HELM_MV3D_OCC=$o timeout 600 python scripts/matvec_sweep.py --N 256,512 --dtype c128,c64 --b 1,4 > gpurun_out/${TAG}_mv_v${v}_o$o.jsonl 2>&1
python - <<PY
import json
for l in open('gpurun_out/${TAG}_mv_v${v}_o$o.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('v=$v o=$o', d['N'], d['dtype'], d['b'], round(d['GBps']), round(d['frac_measured'],3))
PY
[ $v = 0 ] && break
done; done
echo done
