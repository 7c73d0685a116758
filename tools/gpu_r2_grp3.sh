# Grouping check after a g1_scatter / g2a change: grouping + index GPU tests (incl. the
# checked build's bounds checks on the C4 index), then bench lines for C4 E2LSH / SRP, C5.
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_log_group.jsonl
rm -f $LSH_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py tests/test_gpu_dist.py -q -m gpu -x -rf -k "group or index or knn or c4_keys or full_n or sharded" > gpurun_out/r2/pytest_group.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_group.log
for W in "C4 CS_E2LSH" "C4 CS_SRP" "C5 HCS_E2LSH" "C2 CS_E2LSH" "C3 HCS_E2LSH"; do
  set -- $W
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config $1 --scheme $2 > gpurun_out/r2/bench_${1}_${2}.log 2>&1
done
tail -3 gpurun_out/r2/pytest_group.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2/bench_C*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    if l:
        d=json.loads(l[-1]); print(f, 'ms/step %.4f' % d['ms_per_step'], {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v}, d.get('grouping_path'))
    else:
        print(f, open(f).read()[-1500:])
PY
