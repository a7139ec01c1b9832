# Round 2, call M: where the bench's level-1 "arnoldi" class time goes (per (class, level) of one
# cfg4 shard evaluation), and MODE 2 / update probes.
set -x
mkdir -p gpurun_out
T=r2m
python scripts/cfg4_run.py --nsrc 8 --max-rhs 8 > gpurun_out/${T}_cfg4_levels.json 2> gpurun_out/${T}_cfg4_levels.err
python scripts/probe_table.py cfg4 8 c128 0 1 2 > gpurun_out/${T}_probe_c128.jsonl 2>&1
