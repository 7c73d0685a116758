# Grouping check: all grouping / index GPU tests, then the default bench line.
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_log_group.jsonl
rm -f $LSH_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py -q -m gpu -x -rf -k "group or index or knn or c4_keys or full_n or sharded" > gpurun_out/r2/pytest_group.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_group.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2/bench_group.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --config C5 --scheme HCS_E2LSH > gpurun_out/r2/bench_group_c5.log 2>&1
tail -3 gpurun_out/r2/pytest_group.log; tail -c 300 gpurun_out/r2/bench_group.log
