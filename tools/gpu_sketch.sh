set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "C1 or C2 or c4 or edge or padded or zero or overflow or build_index or device_params or grouped" > gpurun_out/pytest_sketch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sketch.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_e2.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --scheme CS_SRP > gpurun_out/bench_srp.log 2>&1
