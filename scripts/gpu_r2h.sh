# Round 2, call H: OPT stencil parity (adjoint mass term fixed), path variants incl. 32x16 matvec
# tiles, same-box matvec A/B (tile height 8 vs 16), OPT-stencil matvec and probe rates.
set -x
mkdir -p gpurun_out
T=r2h
timeout 1500 python -m pytest tests/test_gpu_opt_stencil.py tests/test_gpu_paths.py -q -m gpu --durations=10 > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
python scripts/matvec_sweep.py --N 256,512 > gpurun_out/${T}_mv_by8.jsonl 2>&1
HELM_MATVEC_BY=16 python scripts/matvec_sweep.py --N 256,512 > gpurun_out/${T}_mv_by16.jsonl 2>&1
python scripts/matvec_sweep.py --N 256,512 --stencil opt > gpurun_out/${T}_mv_opt.jsonl 2>&1
