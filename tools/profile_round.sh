#!/bin/bash
# Round evidence (run on the GPU box): full bench line (config 3 headline + configs 1/2 sub-results +
# GRPO config 5 + CPU baselines), ncu launch list of the bench command (our kernels only), ncu --set
# full of the fusion and GRPO kernels, the config-4 streaming slice, the reference arm.
set -x
OUT=gpurun_out/${1:-r02}
mkdir -p $OUT
python bench.py --steps 10 --warmup 3 --json-out $OUT/bench.json > $OUT/bench.log 2>&1
python bench.py --impl reference > $OUT/bench_reference.log 2>&1
Q="python bench.py --steps 3 --warmup 3 --quick --no-e2e --no-cpu"
K='regex:k_sumsq|k_merge|k_mask_bitmap|k_finalize|k_grpo|k_segment_sum'
$Q > $OUT/quick_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 300 --csv --log-file $OUT/launches.csv $Q > $OUT/ncu_launch.log 2>&1
python tools/prof_fusion.py --layout llama8b --runs 2 > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_merge_fast|k_sumsq_bf16|k_mask_bitmap" -s 3 -c 3 -o $OUT/fusion_full python tools/prof_fusion.py --layout llama8b --runs 2 > $OUT/ncu_fusion.log 2>&1
python tools/prof_grpo_fused.py > $OUT/prof_grpo_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_grpo" -s 4 -c 4 -o $OUT/grpo_full python tools/prof_grpo_fused.py > $OUT/ncu_grpo.log 2>&1
python bench.py --stream --stream-layers 1 --steps 3 --warmup 3 --json-out $OUT/config4_stream.json > $OUT/config4_stream.log 2>&1
python tools/prof_fusion.py --layout mlp10m --dtype f32 --runs 3 > $OUT/prof_c1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_merge|k_sumsq" -s 2 -c 2 -o $OUT/config1_full python tools/prof_fusion.py --layout mlp10m --dtype f32 --runs 3 > $OUT/ncu_config1.log 2>&1
python tools/step_gap.py > $OUT/step_gap.log 2>&1
python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
# .ncu-rep files are large (gpurun copies back at most 64 MiB): keep their raw metric pages as CSV
for rep in fusion_full grpo_full config1_full; do
  [ -f $OUT/$rep.ncu-rep ] && ncu -i $OUT/$rep.ncu-rep --page raw --csv > $OUT/$rep.raw.csv 2>/dev/null && rm -f $OUT/$rep.ncu-rep
done
ls -la $OUT
du -sh gpurun_out
