# Round-end measurement batch (gpurun --gpus 4): bench lines N=1/2/4 (C2 weak), C4 strong at 2/4,
# launch list and one full ncu capture of the fitting GEMMs + tabulate kernels of a C2 step
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 python bench.py > gpurun_out/r2final_c2_n1.log 2>&1; echo c2n1 rc=$?
timeout 300 python bench.py --precision mixed --no-cpu > gpurun_out/r2final_c2_n1_mixed.log 2>&1; echo mixed rc=$?
timeout 300 $TR --nproc-per-node 2 --master-port 29801 bench.py --gpus 2 > gpurun_out/r2final_c2_n2.log 2>&1; echo c2n2 rc=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 > gpurun_out/r2final_c2_n4.log 2>&1; echo c2n4 rc=$?
timeout 600 $TR --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --config c4 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/r2final_c4_n4.log 2>&1; echo c4n4 rc=$?
timeout 900 $TR --nproc-per-node 2 --master-port 29804 bench.py --gpus 2 --config c4 --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/r2final_c4_n2.log 2>&1; echo c4n2 rc=$?
BENCH_NO_CLOCKS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2final_ncu_launch.log 2>&1; echo ncu1 rc=$?
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm|k_tab_fwd|k_tab_bwd|k_env|k_forces|k_tab_dT" -c 16 -o gpurun_out/r2final_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2final_ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2final_reference.log 2>&1; echo ref rc=$?
