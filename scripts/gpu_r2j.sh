# Round 2, call J: same-box A/B of the register z-1 plane (HELM_PREV), OPT parity + rates.
set -x
mkdir -p gpurun_out
T=r2j
for rep in 1 2; do
  HELM_PREV=1 python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_prev1_c128_${rep}.jsonl 2>&1
  HELM_PREV=0 python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_prev0_c128_${rep}.jsonl 2>&1
done
HELM_PREV=1 python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_prev1_c64.jsonl 2>&1
HELM_PREV=0 python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_prev0_c64.jsonl 2>&1
HELM_PREV=1 python scripts/matvec_sweep.py --N 256,512 --b 1,4 > gpurun_out/${T}_mv_prev1.jsonl 2>&1
HELM_PREV=0 python scripts/matvec_sweep.py --N 256,512 --b 1,4 > gpurun_out/${T}_mv_prev0.jsonl 2>&1
python scripts/matvec_sweep.py --N 256,512 --stencil opt > gpurun_out/${T}_mv_opt.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_opt_stencil.py tests/test_gpu_paths.py -q -m gpu --durations=10 > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
