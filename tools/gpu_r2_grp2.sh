# grouping tests + bench lines of the grouping-sensitive legs
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_grp2.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py tests/test_gpu_dist.py -q -m gpu -x -rf -k "group or index or knn or c4_keys or full_n or sharded or tables or world2" > gpurun_out/r2/pytest_grp2.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_grp2.log
tail -2 gpurun_out/r2/pytest_grp2.log
for W in "" "--scheme CS_SRP" "--config C5 --scheme HCS_E2LSH --steps 3" "--config C3 --scheme HCS_E2LSH"; do
  timeout 600 python bench.py $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['kernel_ms_per_step'].items() if x})"
done
