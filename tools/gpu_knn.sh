mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "knn" > gpurun_out/pytest_knn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_knn.log
