# Round 2, call L: one barrier per plane in the fused steps (parity + A/B vs r2k), L1 z-chunk
# count sweep (work quantisation at level 1), cfg4 bench.
set -x
mkdir -p gpurun_out
T=r2l
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_opt_stencil.py -q -m gpu -k "not green" > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_c128.jsonl 2>&1
for n in 2 3 4; do HELM_PLANE_NZC=$n python scripts/probe_table.py cfg4 8 c128 1 > gpurun_out/${T}_probe_L1_nzc$n.jsonl 2>&1; done
python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
