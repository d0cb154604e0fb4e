L=paper_2201_01446_b200/lib
cp $L/libdpb200.so $L/pf.so
timeout 300 python -m pytest tests/test_gpu_eval.py tests/test_gpu_chunks.py tests/test_gpu_mixed.py tests/test_gpu_t2.py -x -q 2>&1 | tail -1
one() { timeout 200 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['phases_ms_per_step'])"; }
for r in 1 2; do cp $L/pf.so $L/libdpb200.so; one pf; cp $L/libdpb200_nopf.so $L/libdpb200.so; one nopf; done
