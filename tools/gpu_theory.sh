# NEXT-3 (GPU Monte-Carlo laws) + NEXT-4 (space/time vs m)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_theory.py -q -m gpu > gpurun_out/pytest_theory.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_theory.log
timeout 900 python tools/time_vs_m.py --out gpurun_out/time_vs_m.json > gpurun_out/time_vs_m.log 2>&1
