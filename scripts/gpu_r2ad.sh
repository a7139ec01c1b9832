# Round 2, call AD: the final build (early-stop factor 0.5 compiled in, no environment switches):
# smoke(), the fast parity tests, and the paper's Table 3 study with the paper's 27-pt stencil
# (R35; cells up to 25 x 10, bounded in time) and the 7-pt stencil for the same cells.
set -x
mkdir -p gpurun_out
T=r2ad
env | grep HELM_ || true
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python -m pytest tests/test_gpu_fwi.py tests/test_gpu_solve.py -q -m gpu > gpurun_out/${T}_fast.log 2>&1
echo "fast tests rc=$?"; tail -3 gpurun_out/${T}_fast.log
CELLS=5x6,5x8,5x10,10x6,10x8,10x10,25x6,25x8,25x10
timeout 420 python scripts/table3.py --stencil opt --cells $CELLS > gpurun_out/${T}_table3_opt_c128.jsonl 2> gpurun_out/${T}_table3_opt.err
echo "opt rc=$?"; cut -c1-330 gpurun_out/${T}_table3_opt_c128.jsonl
timeout 300 python scripts/table3.py --stencil std2 --cells $CELLS > gpurun_out/${T}_table3_std2_c128.jsonl 2> gpurun_out/${T}_table3_std2.err
echo "std2 rc=$?"; cut -c1-330 gpurun_out/${T}_table3_std2_c128.jsonl
