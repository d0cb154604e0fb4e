# C5 weak scaling (4 M atoms per GPU, the slab axis grows with N) at 2 and 4 GPUs (gpurun --gpus 4)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29811 bench.py --gpus 4 --config c5 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/c5_n4.log 2>&1; echo c5n4 rc=$?
timeout 600 $TR --nproc-per-node 2 --master-port 29812 bench.py --gpus 2 --config c5 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/c5_n2.log 2>&1; echo c5n2 rc=$?
