mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "full_size_index" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
