# Round 2, call I: register z-1 plane in the single-ring plane kernel (S-2 planes in flight):
# parity of every 3D path, probe tables at cfg4, quick bench.
set -x
mkdir -p gpurun_out
T=r2i
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_operator.py tests/test_gpu_opt_stencil.py -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_c128.jsonl 2>&1
HELM_SPLIT=0 python scripts/probe_table.py cfg4 8 c128 1 > gpurun_out/${T}_probe_c128_nosplit.jsonl 2>&1
python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_c64.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
