# Round 2, call G: the OPT (9/27-point) stencils — parity suite, probe table at cfg4, and the
# regression of the STD2 suite after the template changes.
set -x
mkdir -p gpurun_out
T=r2g
timeout 1500 python -m pytest tests/test_gpu_opt_stencil.py -q -m gpu -x --durations=10 > gpurun_out/${T}_opt.log 2>&1
echo "opt tests rc=$?"
timeout 1500 python -m pytest tests/test_gpu_opt_stencil.py -q -m gpu --durations=10 > gpurun_out/${T}_opt_all.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --deselect tests/test_gpu_opt_stencil.py --durations=10 > gpurun_out/${T}_gputests.log 2>&1
echo "gpu tests rc=$?"
