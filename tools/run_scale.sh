# Scaling batch on one 4-GPU box (gpurun --gpus 4): C4 strong 1/2/4, C2 weak 1/2/4 (bench JSON lines)
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_scale_c4_n$n.json 2> gpurun_out/r02_scale_c4_n$n.err; echo c4 n=$n rc=$?
done
for n in 1 2 4; do
  timeout 300 python bench.py --gpus $n --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02_scale_c2_n$n.json 2> gpurun_out/r02_scale_c2_n$n.err; echo c2 n=$n rc=$?
done
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/r02_dist4.log 2>&1; echo dist rc=$?; tail -2 gpurun_out/r02_dist4.log
for f in gpurun_out/r02_scale_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],3), '%.4g' % d['value'])"; done
