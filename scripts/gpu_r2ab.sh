# Round 2, call AB: the paper's Table 3 study with the paper's compact
# 27-pt stencil (R35) and with the 7-pt STD2 stencil, early stop on (default), complex128.
set -x
mkdir -p gpurun_out
T=r2ab
timeout 1700 python scripts/table3.py --stencil opt --warm-below 30000000 > gpurun_out/${T}_table3_opt_c128.jsonl 2> gpurun_out/${T}_table3_opt.err
echo "opt rc=$?"
cut -c1-260 gpurun_out/${T}_table3_opt_c128.jsonl
timeout 1200 python scripts/table3.py --stencil std2 --warm-below 30000000 > gpurun_out/${T}_table3_std2_c128.jsonl 2> gpurun_out/${T}_table3_std2.err
echo "std2 rc=$?"
cut -c1-260 gpurun_out/${T}_table3_std2_c128.jsonl
