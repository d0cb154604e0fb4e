# Full GPU verification on 4 GPUs: every -m gpu test (incl. 2- and 4-rank), smoke, default bench
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/verify_pytest.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/verify_bench.log 2>&1; echo bench rc=$?
