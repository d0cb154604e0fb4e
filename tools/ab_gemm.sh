for v in 0 2 1 0 2 3; do DPB_GEMM_CTAS=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/gc_$v.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/gc_$v.log').read().strip().splitlines()[-1]);print('cap$v',round(d['value']), round(d['ms_per_step'],3),{k:round(v,3) for k,v in d['phases_ms_per_step'].items()})"; done
timeout 300 python -m pytest tests/test_gpu_eval.py -x -q 2>&1 | tail -1
