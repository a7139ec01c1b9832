# Round 2, call C: split-ring fused Arnoldi steps — parity, same-box A/B probe tables, bench.
set -x
mkdir -p gpurun_out
T=r2c
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_solve.py tests/test_gpu_guards.py tests/test_gpu_operator.py -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
HELM_DEBUG=1 python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_split_c128.jsonl 2> gpurun_out/${T}_probe_split_c128.err
HELM_SPLIT=0 python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_single_c128.jsonl 2>&1
HELM_SPLIT_OCC=3 HELM_DEBUG=1 python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_split3_c128.jsonl 2> gpurun_out/${T}_probe_split3_c128.err
HELM_SPLIT_OCC=1 HELM_DEBUG=1 python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_split1_c128.jsonl 2> gpurun_out/${T}_probe_split1_c128.err
HELM_DEBUG=1 python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_split_c64.jsonl 2> gpurun_out/${T}_probe_split_c64.err
HELM_SPLIT=0 python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_single_c64.jsonl 2>&1
HELM_SPLIT_OCC=2 python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_split2_c64.jsonl 2>&1
python bench.py --steps 2 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
