# K1 variants: C4 E2LSH bench lines for the product build and ${VARS}
mkdir -p gpurun_out/r2
for V in "" ${VARS}; do
  for W in ${WL:-"C4 CS_E2LSH"}; do
    set -- $(echo $W | tr ':' ' ')
    LSH_LIB_VARIANT=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config $1 --scheme $2 > gpurun_out/r2/bk_${V}_$1_$2.log 2>&1
    python - "$V" "$1" "$2" <<'PY'
import json,sys
v,c,sch=sys.argv[1],sys.argv[2],sys.argv[3]
l=[x for x in open(f'gpurun_out/r2/bk_{v}_{c}_{sch}.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print(v or 'base', c, sch, round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['kernel_ms_per_step'].items() if x})
else:
    print(v, c, open(f'gpurun_out/r2/bk_{v}_{c}_{sch}.log').read()[-800:])
PY
  done
done
