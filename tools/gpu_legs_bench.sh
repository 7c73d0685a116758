# every bench leg (no GPU suite), e2e off for the non-default legs
mkdir -p gpurun_out/legs
timeout 900 python bench.py > gpurun_out/legs/C4_CS_E2LSH.log 2>&1
for W in "--scheme CS_SRP" "--config C5 --scheme HCS_E2LSH --steps 3" "--config C5 --scheme HCS_SRP --steps 3" \
         "--config C3 --scheme HCS_E2LSH" "--config C3 --scheme HCS_SRP" "--config C2 --scheme CS_E2LSH" "--config C2 --scheme CS_SRP" \
         "--config C2 --scheme E2LSH" "--per-table --steps 5" "--config C5 --scheme E2LSH --steps 3"; do
  name=$(echo $W | tr -d '-' | tr ' ' '_')
  timeout 900 python bench.py $W --no-e2e --no-cpu-baseline > gpurun_out/legs/$name.log 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/legs/*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f, 'NO LINE'); continue
    d=json.loads(l[-1]); r=d.get('roofline') or {}
    print(f.split('/')[-1][:-4], d['config']['workload'], 'ms', round(d['ms_per_step'],3), 'val %.3g' % d['value'],
          'dom', r.get('kernel'), 'frac', r.get('frac') and round(r['frac'],3), 'io', r.get('io_frac') and round(r['io_frac'],3),
          {k: round(v,3) for k,v in d['kernel_ms_per_step'].items() if v})
PY
