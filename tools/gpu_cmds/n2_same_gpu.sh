set -x
RLK_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-grpo > gpurun_out/b_n2_final.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu --no-grpo --quick > gpurun_out/b_n1_quick.log 2>&1
