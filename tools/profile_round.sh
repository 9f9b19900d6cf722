#!/bin/bash
# Round evidence: full bench, ncu launch list, ncu --set full of the top kernels. Run on the GPU box.
set -x
OUT=gpurun_out/${1:-r01}
mkdir -p $OUT
python bench.py --steps 10 --warmup 3 --json-out $OUT/bench.json > $OUT/bench.log 2>&1
Q="python bench.py --steps 3 --warmup 3 --quick --no-e2e --no-cpu"
$Q > $OUT/quick_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $Q > $OUT/ncu_launch.log 2>&1
python tools/prof_fusion.py --layout llama8b --runs 2 > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_merge_fast|k_sumsq_bf16|k_mask_bitmap" -s 3 -c 3 -o $OUT/fusion_full python tools/prof_fusion.py --layout llama8b --runs 2 > $OUT/ncu_fusion.log 2>&1
python tools/prof_fusion.py --grpo --runs 2 > $OUT/prof_grpo_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_grpo" -s 2 -c 2 -o $OUT/grpo_full python tools/prof_fusion.py --grpo --runs 2 > $OUT/ncu_grpo.log 2>&1
ls -la $OUT
