set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "group or build_index or empty or smoke or edge or zero" > gpurun_out/pytest_group.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_group.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_e2.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --scheme CS_SRP > gpurun_out/bench_srp.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --config C5 --scheme HCS_E2LSH --steps 3 > gpurun_out/bench_c5.log 2>&1
