# Round 2, call S: diagnose the HELM_PERSIST=1 convergence failure of r2r (persist x KStage x
# split), the rest of the GPU suite, and the one-row-per-thread fused steps (HELM_FUSED_PY1).
set -x
mkdir -p gpurun_out
T=r2s
for e in "HELM_PERSIST=1" "HELM_PERSIST=1 HELM_CTA_RED=0" "HELM_PERSIST=1 HELM_SPLIT=1" "HELM_PERSIST=1 HELM_LASTV=1" "HELM_PERSIST=0"; do
  env $e timeout 300 python scripts/diag_persist.py >> gpurun_out/${T}_persist.jsonl 2>> gpurun_out/${T}_persist.err
done
timeout 1800 python -m pytest tests -q -m gpu --deselect "tests/test_gpu_paths.py::test_alternative_stage_paths_match_oracle[persistent_vcycle]" > gpurun_out/${T}_tests.log 2>&1
echo "tests rc=$?"
tail -5 gpurun_out/${T}_tests.log
for e in "HELM_FUSED_PY1=99" "HELM_FUSED_PY1=3" "HELM_FUSED_PY1=4"; do
  env $e timeout 600 python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_${e}.jsonl 2>&1
done
du -sh gpurun_out
