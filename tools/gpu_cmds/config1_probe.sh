set -x
python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/pt_pipe.log 2>&1; echo rc=$? >> gpurun_out/pt_pipe.log
python bench.py --layout mlp10m --dtype f32 --quick --no-grpo --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/b_c1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python tools/prof_fusion.py --layout mlp10m --dtype f32 --runs 3 > gpurun_out/c1_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_merge -s 2 -c 1 -o gpurun_out/c1_merge -f python tools/prof_fusion.py --layout mlp10m --dtype f32 --runs 3 > gpurun_out/c1_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sumsq -s 2 -c 1 -o gpurun_out/c1_sumsq -f python tools/prof_fusion.py --layout mlp10m --dtype f32 --runs 3 >> gpurun_out/c1_ncu_full.log 2>&1
