set -x
TAG=${TAG:-r1k}
python scripts/vcycle_gap.py 50 5 > gpurun_out/${TAG}_gap50.json 2>&1
python scripts/vcycle_gap.py 150 5 > gpurun_out/${TAG}_gap150.json 2>&1
cat gpurun_out/${TAG}_gap50.json gpurun_out/${TAG}_gap150.json
# launches of one V-cycle: skip the warm-up V-cycle + setup kernels, capture the next ~V-cycle
N=$(head -1 gpurun_out/${TAG}_gap50.json | python -c "import json,sys;print(int(json.loads(sys.stdin.readline())['launches_per_vcycle']))")
python scripts/vcycle_gap.py 50 1 > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s $((N+40)) -c $N --csv \
    --log-file gpurun_out/${TAG}_gap50_launches.csv python scripts/vcycle_gap.py 50 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
