# grouping tests, then the default bench line at several table-batch sizes
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_tb.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py -q -m gpu -x -rf -k "group or index or knn or c4_keys or full_n or sharded or tables" > gpurun_out/r2/pytest_tb.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_tb.log
tail -3 gpurun_out/r2/pytest_tb.log
for TB in ${TBS:-1 2 4 8 64}; do
  LSH_GROUP_TB=$TB timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2/bench_tb$TB.log 2>&1
  python - $TB <<'PY'
import json, sys
l=[x for x in open(f'gpurun_out/r2/bench_tb{sys.argv[1]}.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print('TB', sys.argv[1], 'ms/step', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v})
else:
    print(open(f'gpurun_out/r2/bench_tb{sys.argv[1]}.log').read()[-1500:])
PY
done
