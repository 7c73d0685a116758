set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "hcs or C3 or c5 or edge or grouped" > gpurun_out/pytest_hcs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hcs.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --config C5 --scheme HCS_E2LSH --steps 3 > gpurun_out/bench_c5.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --config C5 --scheme HCS_SRP --steps 3 > gpurun_out/bench_c5srp.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --config C3 --scheme HCS_E2LSH > gpurun_out/bench_c3.log 2>&1
