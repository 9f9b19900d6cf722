set -x
python -m pytest tests/test_gpu_fusion.py -x -q -k "split_mode or f32_specialised or state_dict or sharded or graph" > gpurun_out/pt_k1.log 2>&1; echo rc=$? >> gpurun_out/pt_k1.log
python bench.py --layout mlp10m --dtype f32 --quick --no-grpo --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/b_c1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sumsq -s 2 -c 1 -o gpurun_out/c1_sumsq -f python tools/prof_fusion.py --layout mlp10m --dtype f32 --runs 3 > gpurun_out/c1_ncu_full.log 2>&1
