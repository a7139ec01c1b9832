# Round 2, call B: new parity tests, the whole GPU suite, cfg4 bench at PML 20.
set -x
mkdir -p gpurun_out
T=r2b
timeout 1500 python -m pytest tests/test_gpu_cfg3.py tests/test_gpu_cfg5.py tests/test_gpu_guards.py tests/test_gpu_taylor3d.py -q -m gpu --durations=20 > gpurun_out/${T}_newtests.log 2>&1
echo "new tests rc=$?"
python bench.py --steps 2 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
HELM_DEBUG=1 python scripts/ncu_targets.py probe cfg4_8 1 3 0 > gpurun_out/${T}_debug_L1.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --durations=25 --deselect tests/test_gpu_taylor3d.py > gpurun_out/${T}_gputests.log 2>&1
echo "gpu tests rc=$?"
