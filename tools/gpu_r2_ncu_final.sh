# ncu part of tools/gpu_r2_final.sh alone (fresh reports: -f overwrites a reused box's /tmp)
F=gpurun_out/final
mkdir -p $F/prof
for W in "C4 CS_E2LSH build" "C4 CS_SRP build" "C5 HCS_E2LSH build"; do
  set -- $W
  ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -o /tmp/${1}_${2}_full \
      python tools/prof_hash.py --config $1 --scheme $2 --op $3 --reps 1 > $F/prof/ncu_${1}_${2}.log 2>&1
done
python tools/summarize_r2.py $F/prof C4:CS_E2LSH=/tmp/C4_CS_E2LSH_full.ncu-rep C4:CS_SRP=/tmp/C4_CS_SRP_full.ncu-rep \
    C5:HCS_E2LSH=/tmp/C5_HCS_E2LSH_full.ncu-rep > $F/prof/summarize.log 2>&1
for K in sketch_kernel g2a g1_scatter; do
  ncu -i /tmp/C4_CS_E2LSH_full.ncu-rep --page source --csv -k regex:$K > $F/prof/src_${K}.csv 2>/dev/null
  python tools/sass_regions.py $F/prof/src_${K}.csv --top 8 > $F/prof/regions_${K}.txt 2>&1
done
tail -2 $F/prof/ncu_*.log
