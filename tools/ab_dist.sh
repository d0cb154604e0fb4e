# A/B of library variants lib/var_<name>.so at N GPUs (C2 weak, 50 steps, twice each); restores var_new
N=$1; shift
L=paper_2201_01446_b200/lib
one() { cp $L/var_$1.so $L/libdpb200.so; timeout 300 python bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 n=$N', round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['phases_ms_per_step'].items()})"; }
for r in 1 2; do for v in "$@"; do one $v; done; done
cp $L/var_new.so $L/libdpb200.so
