#!/bin/bash
# Profile capture for one round (run ON the GPU box via gpurun):
#   bash tools/profile_round.sh r1
# 1) the launch list of the bench command (per-launch device time + DRAM
#    bytes, cold-cache & serialised under ncu: compare SHARES, not absolutes)
# 2) one `--set full` capture of every Tempo kernel at the bench shapes
# Summarise here with: python tools/summarize_profiles.py r1
set -u
R=${1:-r1}
mkdir -p gpurun_out
KRE='regex:(gelu_|ln_|softmax_|dropout_|dal_|mask_|add_kernel)'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$KRE" -c 40 --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_$R.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k "$KRE" -s 10 -c 19 \
    -o gpurun_out/prof_$R python tools/profile_ops.py > gpurun_out/ncu_full_$R.log 2>&1
echo "profile_round $R done"
