set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pt_full.log 2>&1; echo rc=$? >> gpurun_out/pt_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python bench.py --layout mlp10m --dtype f32 --quick --no-grpo --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/b_c1.log 2>&1
