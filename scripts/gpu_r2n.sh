# Round 2, call N (re-entry): full GPU parity suite on HEAD (one-barrier fused steps), then the
# cfg4 bench at a short K/W for the A/B against r2k (profiles/r02/bench_r2_final.json).
set -x
mkdir -p gpurun_out
T=r2n
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/${T}_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
cat gpurun_out/${T}_bench.json | head -c 3000
