set -x
TAG=${TAG:-r1t}
for v in cur b428 cur b428; do
  if [ $v = cur ]; then unset HELM_LIB_VARIANT; else export HELM_LIB_VARIANT=$v; fi
  timeout 300 python scripts/tune_plane.py cfg2 c128 150 >> gpurun_out/${TAG}_tune.jsonl 2>> gpurun_out/${TAG}_tune.err
  timeout 300 python scripts/tune_plane.py cfg2 c128 50 >> gpurun_out/${TAG}_tune.jsonl 2>> gpurun_out/${TAG}_tune.err
done
unset HELM_LIB_VARIANT
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-matvec > gpurun_out/${TAG}_bench$i.json 2> gpurun_out/${TAG}_bench$i.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench$i.json'));print('bench', d['value'], d['level_shares'], d['roofline'])"
done
echo done
