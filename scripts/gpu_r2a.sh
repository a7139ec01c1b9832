# Round 2, call A: cfg4 bench (quick), per-kernel probe table at cfg4 (8 RHS), convergence
# diagnosis (PML width, depth), ncu --set full of the level-1 3D fused Arnoldi steps.
set -x
mkdir -p gpurun_out
T=r2a
python bench.py --steps 2 --warmup 3 --no-matvec --no-cpu-baseline --no-extra > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
python scripts/probe_table.py cfg4 8 c128 > gpurun_out/${T}_probe_cfg4_c128.jsonl 2>&1
python scripts/probe_table.py cfg4 8 c64 > gpurun_out/${T}_probe_cfg4_c64.jsonl 2>&1
for cfg in "10 3" "20 3" "10 2" "30 3"; do
  set -- $cfg
  timeout 600 python scripts/cfg4_conv.py --pml $1 --levels $2 >> gpurun_out/${T}_conv.jsonl 2>> gpurun_out/${T}_conv.err
done
for spec in "1 3 0" "1 3 2" "1 4 4" "0 3 2" "2 3 2"; do
  set -- $spec
  name=${T}_cfg4_L$1_k$2_nv$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plane -s 2 -c 1 \
      -o gpurun_out/${name} python scripts/ncu_targets.py probe cfg4_8 $1 $2 $3 > gpurun_out/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  if [ -f gpurun_out/${name}.ncu-rep ]; then
    ncu -i gpurun_out/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${name}.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
    ncu -i gpurun_out/${name}.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
    gzip -f gpurun_out/${name}_sass.csv
    rm -f gpurun_out/${name}.ncu-rep
  fi
done
du -sh gpurun_out
