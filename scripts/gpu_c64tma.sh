# 3D parity (short timeouts) then the matvec occupancy sweep.
set -x
timeout 300 python -m pytest tests/test_gpu_operator.py tests/test_gpu_solve.py tests/test_gpu_jacobian.py -x -q 2>&1 | tail -5
timeout 400 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg5 or cfg3" 2>&1 | tail -5
OCCS="${OCCS:-4 8}" bash scripts/gpu_occ.sh
