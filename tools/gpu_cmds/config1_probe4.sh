set -x
python -m pytest tests/test_gpu_fusion.py tests/test_gpu_pipeline.py tests/test_gpu_dist.py tests/test_gpu_loader.py -x -q > gpurun_out/pt_k1.log 2>&1; echo rc=$? >> gpurun_out/pt_k1.log
python bench.py --layout mlp10m --dtype f32 --quick --no-grpo --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/b_c1.log 2>&1
