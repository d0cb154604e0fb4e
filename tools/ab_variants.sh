# A/B of library variants lib/var_<name>.so on one box (50-step C2 bench, twice each); restores var_base
L=paper_2201_01446_b200/lib
one() { cp $L/var_$1.so $L/libdpb200.so; timeout 200 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()})"; }
for r in 1 2; do for v in "$@"; do one $v; done; done
cp $L/var_base.so $L/libdpb200.so
