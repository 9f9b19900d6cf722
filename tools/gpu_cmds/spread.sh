set -x
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/spread_$i.log 2>&1; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/spread_smi.log
