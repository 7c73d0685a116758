# Bench evidence for this build (no GPU suite, no ncu --set full): the ncu launch list
# of the bench command, every bench leg, the NCCL-forced N=1 line and the reference arm.
F=gpurun_out/final
mkdir -p $F/prof $F/legs
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $F/prof/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/prof/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $F/prof/ncu_launch.log 2>&1
timeout 900 python bench.py > $F/legs/C4_CS_E2LSH.log 2>&1
for W in "--scheme CS_SRP" "--config C5 --scheme HCS_E2LSH --steps 3" "--config C5 --scheme HCS_SRP --steps 3" \
         "--config C3 --scheme HCS_E2LSH" "--config C3 --scheme HCS_SRP" "--config C2 --scheme CS_E2LSH" "--config C2 --scheme CS_SRP" \
         "--config C2 --scheme E2LSH" "--per-table --steps 5" "--config C5 --scheme E2LSH --steps 3"; do
  name=$(echo $W | tr -d '-' | tr ' ' '_')
  timeout 900 python bench.py $W --no-e2e --no-cpu-baseline > $F/legs/$name.log 2>&1
done
LSH_BENCH_FORCE_DIST=1 RANK=0 LOCAL_RANK=0 WORLD_SIZE=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 timeout 600 python bench.py --no-e2e --no-cpu-baseline > $F/legs/C4_CS_E2LSH_nccl_forced_n1.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $F/legs/reference_C4_CS_E2LSH.log 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/final/legs/*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f, 'NO LINE', open(f).read()[-300:]); continue
    d=json.loads(l[-1]); r=d.get('roofline') or {}
    print(f.split('/')[-1][:-4], d['config']['workload'], 'ms', round(d['ms_per_step'],3), 'val %.3g' % d['value'],
          'dom', r.get('kernel'), 'frac', r.get('frac') and round(r['frac'],3), 'traffic', r.get('traffic'),
          {k: round(v,3) for k,v in (d.get('kernel_ms_per_step') or {}).items() if v})
PY
