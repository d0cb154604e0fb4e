# Final verification on one 4-GPU box (gpurun --gpus 4): every -m gpu test (incl. 2- and 4-rank),
# smoke, default bench line, reference arm, mixed C2, C2 weak 2/4, C3, launch list + ncu full of
# the FP64 kernels -> gpurun_out/r02v_*
set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02v_pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/r02v_c2_n1.json 2> gpurun_out/r02v_c2_n1.err; echo c2n1 rc=$?
timeout 300 python bench.py --impl reference > gpurun_out/r02v_reference.json 2> gpurun_out/r02v_reference.err; echo ref rc=$?
timeout 300 python bench.py --precision mixed --no-cpu > gpurun_out/r02v_c2_n1_mixed.json 2> gpurun_out/r02v_mixed.err; echo mixed rc=$?
for n in 2 4; do timeout 400 python bench.py --gpus $n > gpurun_out/r02v_c2_n$n.json 2> gpurun_out/r02v_c2_n$n.err; echo c2n$n rc=$?; done
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/r02v_c3_n1.json 2> gpurun_out/r02v_c3.err; echo c3 rc=$?
BENCH_NO_CLOCKS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02v_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02v_ncu_launch.log 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/r02v_launches.csv > gpurun_out/r02v_launches_summary.txt
BENCH_NO_CLOCKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm|k_tab_fwd|k_tab_bwd|k_forces|k_tab_dT" --launch-skip 40 -c 14 -o gpurun_out/r02v_full python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02v_ncu_full.log 2>&1; echo ncu2 rc=$?
for f in gpurun_out/r02v_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('n_gpus'), d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'))" 2>/dev/null; done
tail -3 gpurun_out/r02v_pytest_gpu.log
