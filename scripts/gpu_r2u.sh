# Round 2, call U: matvec (configs[4]) tuning sweep — the 24 cells under ring / occupancy
# variants of the MODE-0 plane kernel (each a fresh process: switches are read once).
set -x
mkdir -p gpurun_out
T=r2u
for e in "HELM_X=0" "HELM_PREV=2" "HELM_PLANE_OCC=8" "HELM_PREV=2 HELM_PLANE_OCC=8" "HELM_PLANE_OCC=4" "HELM_PREV=2 HELM_PLANE_OCC=4" "HELM_PREV=2 HELM_PLANE_OCC=16"; do
  tag=$(echo $e | tr ' =' '__')
  env $e timeout 900 python scripts/matvec_sweep.py > gpurun_out/${T}_mv_${tag}.jsonl 2> gpurun_out/${T}_mv_${tag}.err
  echo "$e rc=$?"
done
du -sh gpurun_out
# latency regime: programmatic dependent launch at cfg3 (measured -4 % at cfg2 in round 1)
timeout 600 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_def.json 2>&1
HELM_PDL=1 timeout 600 python scripts/cfg3_time.py > gpurun_out/${T}_cfg3_pdl.json 2>&1
