# Multi-GPU batch on one 4-GPU box (gpurun --gpus 4): C2 weak 2/4 (default bench line, with e2e),
# C5 weak 2/4, C4 strong 2/4 -> gpurun_out/r02s_*.json; the 1-GPU lines come from run_final.sh.
for n in 2 4; do
  timeout 400 python bench.py --gpus $n > gpurun_out/r02s_c2_n$n.json 2> gpurun_out/r02s_c2_n$n.err; echo c2 n=$n rc=$?
done
for n in 2 4; do
  timeout 1200 python bench.py --gpus $n --config c5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02s_c5_n$n.json 2> gpurun_out/r02s_c5_n$n.err; echo c5 n=$n rc=$?
done
for n in 2 4; do
  timeout 1500 python bench.py --gpus $n --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02s_c4_n$n.json 2> gpurun_out/r02s_c4_n$n.err; echo c4 n=$n rc=$?
done
grep -h "bench rank" gpurun_out/r02s_*.err
for f in gpurun_out/r02s_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],3), '%.4g' % d['value'])"; done
