set -x
TAG=${TAG:-r1w}
for g in 1 0 1 0; do
HELM_GMRES_CTA=$g timeout 600 python scripts/vcycle_gap.py 150 5 2>/dev/null | head -1 | sed "s/^/cta=$g /"
HELM_GMRES_CTA=$g timeout 600 python scripts/vcycle_gap.py 50 5 2>/dev/null | head -1 | sed "s/^/cta=$g /"
done
for g in 1 0; do
HELM_GMRES_CTA=$g timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-matvec > gpurun_out/${TAG}_bench_cta$g.json 2> gpurun_out/${TAG}_bench_cta$g.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_cta$g.json'));print('bench cta=$g', d['value'], d['level_shares'], d['kernel_shares'])"
done
echo done
