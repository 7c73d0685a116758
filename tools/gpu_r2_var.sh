# Measurement-only library variants (build.py VARIANT_FLAGS): one bench line each for
# C4 CS-E2LSH and C5 HCS-E2LSH, then the grouping tests on the first variant.
mkdir -p gpurun_out/r2
for V in "" ${VARS}; do
  for W in "C4 CS_E2LSH" "C5 HCS_E2LSH"; do
    set -- $W
    LSH_LIB_VARIANT=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config $1 --scheme $2 > gpurun_out/r2/bv_${V}_$1.log 2>&1
    python - "$V" "$1" <<'PY'
import json,sys
v,c=sys.argv[1],sys.argv[2]
l=[x for x in open(f'gpurun_out/r2/bv_{v}_{c}.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print(v or 'base', c, round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['kernel_ms_per_step'].items() if x})
else:
    print(v, c, open(f'gpurun_out/r2/bv_{v}_{c}.log').read()[-800:])
PY
  done
done
if [ -n "$TESTV" ]; then
LSH_LIB_VARIANT=$TESTV timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py -q -m gpu -x -k "group or index or tables" 2>&1 | tail -2
fi
