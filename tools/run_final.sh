# Round-end measurement batch (gpurun --gpus 4). Outputs gpurun_out/r02f_*; summaries are copied
# into profiles/ by hand. Every number comes from a run without a profiler, except the ncu files.
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/fp64_peak tools/microbench/fp64_peak.cu
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/r02f_fp64_peak_clocks.csv & SMI=$!
sleep 1
./tools/microbench/fp64_peak > gpurun_out/r02f_fp64_peak.log 2>&1; ./tools/microbench/fp64_peak >> gpurun_out/r02f_fp64_peak.log 2>&1
sleep 1; kill $SMI 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/r02f_c2_n1.json 2> gpurun_out/r02f_c2_n1.err; echo c2n1 rc=$?
timeout 300 python bench.py --impl reference > gpurun_out/r02f_reference.json 2> gpurun_out/r02f_reference.err; echo ref rc=$?
timeout 300 python bench.py --precision mixed --no-cpu > gpurun_out/r02f_c2_n1_mixed.json 2> gpurun_out/r02f_mixed.err; echo mixed rc=$?
for n in 2 4; do timeout 400 python bench.py --gpus $n > gpurun_out/r02f_c2_n$n.json 2> gpurun_out/r02f_c2_n$n.err; echo c2n$n rc=$?; done
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/r02f_c3_n1.json 2> gpurun_out/r02f_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c3 --precision mixed --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/r02f_c3_n1_mixed.json 2> gpurun_out/r02f_c3m.err; echo c3m rc=$?
for n in 1 2 4; do timeout 1200 python bench.py --gpus $n --config c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02f_c5_n$n.json 2> gpurun_out/r02f_c5_n$n.err; echo c5n$n rc=$?; done
for n in 1 2 4; do timeout 1500 python bench.py --gpus $n --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02f_c4_n$n.json 2> gpurun_out/r02f_c4_n$n.err; echo c4n$n rc=$?; done
BENCH_NO_CLOCKS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02f_ncu_launch.log 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/r02f_launches.csv > gpurun_out/r02f_launches_summary.txt
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm|k_tab_fwd|k_tab_bwd|k_forces|k_tab_dT" --launch-skip 40 -c 14 -o gpurun_out/r02f_full python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02f_ncu_full.log 2>&1; echo ncu2 rc=$?
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc_fwd64|k_tc_gemm" -c 6 -o gpurun_out/r02f_full_mixed python bench.py --precision mixed --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02f_ncu_full_mixed.log 2>&1; echo ncu3 rc=$?
for f in gpurun_out/r02f_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('n_gpus'), d.get('ms_per_step'), d.get('value'))" 2>/dev/null; done
