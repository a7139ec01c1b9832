# Round 2, call AF: the large Table 3 cells (40 and 50 wavelengths) with the paper's 27-pt stencil.
set -x
mkdir -p gpurun_out
timeout 1000 python scripts/table3.py --stencil opt --cells 40x6,40x8,40x10,50x6,50x8,50x10 --warm-below 30000000 \
    > gpurun_out/r2af_table3_opt_large_c128.jsonl 2> gpurun_out/r2af_table3_opt_large.err
echo "rc=$?"; cut -c1-330 gpurun_out/r2af_table3_opt_large_c128.jsonl; tail -3 gpurun_out/r2af_table3_opt_large.err
