# interpolation-guided lookup: query tests, then C4 bench lines (product vs the previous build in liblsh_b200_prev.so)
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_parity.py -q -m gpu -x -rf -k "query" > gpurun_out/r2/pytest_lookup.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_lookup.log
tail -3 gpurun_out/r2/pytest_lookup.log
VARS="prev" WL="C4:CS_E2LSH C4:CS_SRP" bash tools/gpu_r2_k1var.sh
