mkdir -p gpurun_out/r2
for V in "" ${VARS:-t4k}; do
  LSH_LIB_VARIANT=$V python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2/bv_$V.log 2>&1
  python - $V <<'PY'
import json,sys
v=sys.argv[1] if len(sys.argv)>1 else ''
d=json.loads([x for x in open(f'gpurun_out/r2/bv_{v}.log') if x.startswith('{')][-1]); print(v or 'base', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['kernel_ms_per_step'].items() if x})
PY
done
LSH_LIB_VARIANT=${VARS:-t4k} timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py -q -m gpu -x -k "group or index or tables" 2>&1 | tail -2
