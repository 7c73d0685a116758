# sketch change check: fast-path + sketch parity tests, then C4 / C2 / C1 bench lines
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_sk.jsonl
rm -f $LSH_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_fastpath.py tests/test_gpu_parity.py -q -m gpu -x -rf > gpurun_out/r2/pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_sk.log
tail -4 gpurun_out/r2/pytest_sk.log
for W in "C4 CS_E2LSH" "C4 CS_SRP" "C2 CS_E2LSH"; do
  set -- $W
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config $1 --scheme $2 > gpurun_out/r2/bench_sk_${1}_${2}.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2/bench_sk_*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    if l:
        d=json.loads(l[-1]); print(f, 'ms/step %.4f' % d['ms_per_step'], {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v}, d['roofline'].get('frac'))
    else:
        print(f, open(f).read()[-1500:])
PY
