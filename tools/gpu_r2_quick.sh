# quick check after a kernel change: fast-path parity, dist, one bench line (no e2e)
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_quick.jsonl
rm -f $LSH_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_dist.py ${EXTRA_TESTS} -q -m gpu -x -rf > gpurun_out/r2/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2/bench_quick.log 2>&1
tail -3 gpurun_out/r2/pytest_quick.log
python - <<'PY'
import json
l=[x for x in open('gpurun_out/r2/bench_quick.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print('ms/step', d['ms_per_step'], {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v})
else:
    print(open('gpurun_out/r2/bench_quick.log').read()[-2000:])
PY
