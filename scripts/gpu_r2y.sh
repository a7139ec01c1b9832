# Round 2, call Y: full GPU suite and the default bench line at the driver's K/W with the
# matvec / march-feed / first-step changes; ncu launch list of the bench window.
set -x
mkdir -p gpurun_out
T=r2y
timeout 2000 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-matvec --no-cpu-baseline --no-extra"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 120000 -c 2000 --csv \
    --log-file gpurun_out/${T}_bench_launches.csv $CMD > gpurun_out/${T}_ncu_launches.log 2>&1
echo "launch list rc=$?"
du -sh gpurun_out
