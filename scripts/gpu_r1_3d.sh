# 3D evidence after the plane-kernel changes: cfg4 at full size (c128, then c64) and ncu --set full of
# the new matvec kernels.
set -x
timeout 900 python scripts/cfg4_run.py --max-rhs 16 --dtype c128 > gpurun_out/cfg4_full_c128.json 2> gpurun_out/cfg4_full_c128.err
timeout 900 python scripts/cfg4_run.py --max-rhs 16 --dtype c64 > gpurun_out/cfg4_full_c64.json 2> gpurun_out/cfg4_full_c64.err
TAG=r1py4 SPECS="512 c128 1;256 c64 4;512 c64 1" bash scripts/gpu_ncu_mv.sh
