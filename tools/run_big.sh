# C5 weak and C4 strong scaling on one 4-GPU box (gpurun --gpus 4) -> gpurun_out/r02b_*.json
for n in 1 2 4; do timeout 1200 python bench.py --gpus $n --config c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02b_c5_n$n.json 2> gpurun_out/r02b_c5_n$n.err; echo c5n$n rc=$?; done
for n in 1 2 4; do timeout 1500 python bench.py --gpus $n --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02b_c4_n$n.json 2> gpurun_out/r02b_c4_n$n.err; echo c4n$n rc=$?; done
grep -h "bench rank" gpurun_out/r02b_*.err
for f in gpurun_out/r02b_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],2), '%.4g' % d['value'], round(d['roofline']['frac'],3), d['clocks']['reasons'])"; done
