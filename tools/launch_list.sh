# ncu launch list of a short C2 bench run (per-kernel durations, cold-cache serialized) + summary.
# usage: bash tools/launch_list.sh <tag> [extra bench args]
tag=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/ncu_$tag.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$tag.csv > gpurun_out/launches_${tag}_summary.txt
head -30 gpurun_out/launches_${tag}_summary.txt
