# Round-2 evidence for THIS build: GPU suite (parity log), smoke, ncu full captures
# (summarised into profiles/round2/ncu_summary.json so the bench lines carry `traffic`),
# the ncu launch list of the bench command, every bench leg and the reference arm.
F=gpurun_out/final
mkdir -p $F/prof $F/legs
export LSH_PARITY_LOG=$F/parity_log.jsonl
rm -f $LSH_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu -rf > $F/pytest_gpu.log 2>&1; echo "rc=$?" >> $F/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo "smoke rc=$?" >> $F/smoke.log
unset LSH_PARITY_LOG
for W in "C4 CS_E2LSH build" "C4 CS_SRP build" "C5 HCS_E2LSH build"; do
  set -- $W
  ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -o /tmp/${1}_${2}_full \
      python tools/prof_hash.py --config $1 --scheme $2 --op $3 --reps 1 > $F/prof/ncu_${1}_${2}.log 2>&1
done
python tools/summarize_r2.py $F/prof C4:CS_E2LSH=/tmp/C4_CS_E2LSH_full.ncu-rep C4:CS_SRP=/tmp/C4_CS_SRP_full.ncu-rep \
    C5:HCS_E2LSH=/tmp/C5_HCS_E2LSH_full.ncu-rep > $F/prof/summarize.log 2>&1
cp $F/prof/ncu_summary.json profiles/round2/ncu_summary.json
for K in sketch_kernel g2a g1_scatter; do
  ncu -i /tmp/C4_CS_E2LSH_full.ncu-rep --page source --csv -k regex:$K > $F/prof/src_${K}.csv 2>/dev/null
  python tools/sass_regions.py $F/prof/src_${K}.csv --top 8 > $F/prof/regions_${K}.txt 2>&1
done
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $F/prof/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/prof/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $F/prof/ncu_launch.log 2>&1
python tools/launch_shares.py $F/prof/bench_launches.csv > $F/prof/launch_shares.txt 2>&1
timeout 900 python bench.py > $F/legs/C4_CS_E2LSH.log 2>&1
for W in "--scheme CS_SRP" "--config C5 --scheme HCS_E2LSH --steps 3" "--config C5 --scheme HCS_SRP --steps 3" \
         "--config C3 --scheme HCS_E2LSH" "--config C3 --scheme HCS_SRP" "--config C2 --scheme CS_E2LSH" "--config C2 --scheme CS_SRP" \
         "--config C2 --scheme E2LSH" "--per-table --steps 5" "--config C5 --scheme E2LSH --steps 3"; do
  name=$(echo $W | tr -d '-' | tr ' ' '_')
  timeout 900 python bench.py $W --no-e2e --no-cpu-baseline > $F/legs/$name.log 2>&1
done
LSH_BENCH_FORCE_DIST=1 RANK=0 LOCAL_RANK=0 WORLD_SIZE=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 timeout 600 python bench.py --no-e2e --no-cpu-baseline > $F/legs/C4_CS_E2LSH_nccl_forced_n1.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $F/legs/reference_C4_CS_E2LSH.log 2>&1
tail -3 $F/pytest_gpu.log; tail -1 $F/smoke.log
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
