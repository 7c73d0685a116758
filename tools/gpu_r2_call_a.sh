mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_dist.py -q -m gpu -rf > gpurun_out/r2/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_dist.log
tail -3 gpurun_out/r2/pytest_dist.log
bash tools/gpu_sanitize.sh
bash tools/gpu_r2_ncu.sh
