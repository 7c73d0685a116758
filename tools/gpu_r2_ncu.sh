# ncu evidence for profiles/round2: launch list of the bench command, full captures of
# one build per workload (NVTX range "profile"), summarised on the box.
mkdir -p gpurun_out/r2/prof
P=gpurun_out/r2/prof
python bench.py --steps 10 --warmup 3 > $P/bench_line.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $P/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $P/ncu_launch.log 2>&1
for W in "C4 CS_E2LSH build" "C4 CS_SRP build" "C5 HCS_E2LSH build"; do
  set -- $W
  ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -o /tmp/${1}_${2}_full \
      python tools/prof_hash.py --config $1 --scheme $2 --op $3 --reps 1 > $P/ncu_${1}_${2}.log 2>&1
done
python tools/summarize_r2.py $P C4:CS_E2LSH=/tmp/C4_CS_E2LSH_full.ncu-rep C4:CS_SRP=/tmp/C4_CS_SRP_full.ncu-rep \
    C5:HCS_E2LSH=/tmp/C5_HCS_E2LSH_full.ncu-rep > $P/summarize.log 2>&1
# per-line source view of the two C4 E2LSH hot kernels
for K in sketch_kernel g2a g2e g1_scatter; do
  ncu -i /tmp/C4_CS_E2LSH_full.ncu-rep --page source --csv -k regex:$K > $P/src_${K}.csv 2>/dev/null
done
ls -la $P | head -30
