# Round 2, call V: ring depth / occupancy sweep of the 2-row plane kernels (residual, FGMRES,
# fused steps) at cfg4 (8 RHS, levels 0-2) — HELM_PLANE_OCC (resident-CTA target) and
# HELM_PLANE_S (ring stages), each a fresh process — and the bench with the GPU-busy fraction.
set -x
mkdir -p gpurun_out
T=r2v
for e in "HELM_X=0" "HELM_PLANE_OCC=3" "HELM_PLANE_OCC=5" "HELM_PLANE_OCC=6" "HELM_PLANE_S=5" "HELM_PLANE_S=6" "HELM_PLANE_S=8"; do
  tag=$(echo $e | tr ' =' '__')
  env $e timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_${tag}.jsonl 2>&1
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
du -sh gpurun_out
