# 2-GPU batch (gpurun --gpus 2)
set -x
DPB_TRACE_ONCE=1 timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo dist rc=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2; do
timeout 300 $TR --nproc-per-node 2 --master-port 2970$rep bench.py --gpus 2 --steps 50 --warmup 5 --e2e-steps 10 > gpurun_out/bench_c2_n2_$rep.log 2>&1; echo c2n2 rc=$?
DPB_NO_HALO_OVERLAP=1 timeout 300 $TR --nproc-per-node 2 --master-port 2971$rep bench.py --gpus 2 --steps 50 --warmup 5 --e2e-steps 10 > gpurun_out/bench_c2_n2_noov_$rep.log 2>&1; echo c2n2noov rc=$?
done
DPB_TRACE=1 timeout 900 $TR --nproc-per-node 2 --master-port 29704 bench.py --gpus 2 --config c4 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_c4_n2.log 2>&1; echo c4n2 rc=$?
