# K1 four-tables-per-warp path: fast-path parity (product build), then C4 / C2 bench lines
# for the product build and the lane-per-point variant (liblsh_b200_lane1.so)
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_quad.jsonl
rm -f $LSH_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_fastpath.py -q -m gpu -x -rf > gpurun_out/r2/pytest_quad.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_quad.log
tail -3 gpurun_out/r2/pytest_quad.log
VARS=lane1 bash tools/gpu_r2_var3.sh
