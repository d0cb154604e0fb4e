# A/B of two builds of the library on one box: lib/new.so (candidate) vs lib/base.so (current), 50-step C2 bench, twice each
L=paper_2201_01446_b200/lib
cp $L/new.so $L/libdpb200.so
timeout 500 python -m pytest tests/test_gpu_eval.py tests/test_gpu_chunks.py tests/test_gpu_md.py tests/test_gpu_exact.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1
one() { timeout 200 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['phases_ms_per_step'])"; }
for r in 1 2; do cp $L/new.so $L/libdpb200.so; one new; cp $L/base.so $L/libdpb200.so; one base; done
cp $L/new.so $L/libdpb200.so
