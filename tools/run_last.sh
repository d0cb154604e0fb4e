# Last check on one 4-GPU box: all -m gpu tests, smoke, default C2 bench at 1/2/4 GPUs, reference arm,
# C3, mixed C2 -> gpurun_out/r02z_*
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02z_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/r02z_c2_n1.json 2> gpurun_out/r02z_c2_n1.err; echo c2n1 rc=$?
for n in 2 4; do timeout 400 python bench.py --gpus $n > gpurun_out/r02z_c2_n$n.json 2> gpurun_out/r02z_c2_n$n.err; echo c2n$n rc=$?; done
timeout 300 python bench.py --impl reference > gpurun_out/r02z_reference.json 2> gpurun_out/r02z_reference.err; echo ref rc=$?
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/r02z_c3_n1.json 2> gpurun_out/r02z_c3.err; echo c3 rc=$?
timeout 300 python bench.py --precision mixed --no-cpu > gpurun_out/r02z_c2_n1_mixed.json 2> gpurun_out/r02z_mixed.err; echo mixed rc=$?
BENCH_NO_CLOCKS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02z_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02z_ncu_launch.log 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/r02z_launches.csv > gpurun_out/r02z_launches_summary.txt
for f in gpurun_out/r02z_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('n_gpus'), d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'))" 2>/dev/null; done
tail -1 gpurun_out/r02z_pytest_gpu.log
