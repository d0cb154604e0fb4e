run() { PROBE_TAG=$2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/dist_probe.py 50 $3 > /dev/null 2>&1; }
run 29521 plain10 10
run 29522 plain10b 10
run 29523 warm60 60
run 29524 warm60b 60
run 29525 plain10c 10
