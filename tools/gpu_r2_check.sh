# Round-2 check: GPU suite (parity log), smoke, default bench line.
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_log.jsonl
rm -f $LSH_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/r2/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2/bench_default.log 2>&1
tail -3 gpurun_out/r2/pytest_gpu.log; tail -1 gpurun_out/r2/smoke.log; tail -c 600 gpurun_out/r2/bench_default.log
