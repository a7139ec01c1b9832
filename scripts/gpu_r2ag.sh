# Round 2, call AG: the full GPU suite on the final build (no environment switches), then the
# fast north-star parity tests at early-stop factors 0.7 and 0.85 (where does the 1e-5 bar break).
set -x
mkdir -p gpurun_out
T=r2ag
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"; tail -6 gpurun_out/${T}_tests.log
for PCT in 70 85; do
  HELM_EARLY_PCT=$PCT timeout 300 python -m pytest tests/test_gpu_fwi.py tests/test_gpu_solve.py -q -m gpu > gpurun_out/${T}_fast_pct$PCT.log 2>&1
  echo "fast pct=$PCT rc=$?"; tail -4 gpurun_out/${T}_fast_pct$PCT.log
done
