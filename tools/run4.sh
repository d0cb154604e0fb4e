# 4-GPU measurement batch (gpurun --gpus 4): dist parity tests, weak scaling C2, strong C4
set -x
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_chunks.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo dist rc=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 --steps 50 --warmup 5 --e2e-steps 10 > gpurun_out/bench_c2_n2.log 2>&1; echo c2n2 rc=$?
DPB_NO_HALO_OVERLAP=1 timeout 300 $TR --nproc-per-node 2 --master-port 29705 bench.py --gpus 2 --steps 50 --warmup 5 --e2e-steps 10 > gpurun_out/bench_c2_n2_noov.log 2>&1; echo c2n2noov rc=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --steps 50 --warmup 5 --e2e-steps 10 > gpurun_out/bench_c2_n4.log 2>&1; echo c2n4 rc=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29704 bench.py --gpus 2 --config c4 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4_n2.log 2>&1; echo c4n2 rc=$?
timeout 600 $TR --nproc-per-node 4 --master-port 29703 bench.py --gpus 4 --config c4 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4_n4.log 2>&1; echo c4n4 rc=$?
