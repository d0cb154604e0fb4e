# A/B of the evaluation chunk size at C2 (DPB_CHUNK centres per chunk), 50-step bench, twice each
one() { DPB_CHUNK=$1 timeout 200 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk=$1', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()})"; }
for r in 1 2; do for c in 131072 10752 8064 6400; do one $c; done; done
