# ncu (full set, source-level) of the C4 CS_E2LSH grouping kernels of one build
mkdir -p gpurun_out/r2/prof_g3
P=gpurun_out/r2/prof_g3
ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -k regex:"g2a|g1_scatter" -o /tmp/g3 \
    python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > $P/ncu.log 2>&1
ncu -i /tmp/g3.ncu-rep --page raw --csv > $P/raw.csv 2>/dev/null
ncu -i /tmp/g3.ncu-rep --page source --csv -k regex:g2a > $P/src_g2a.csv 2>/dev/null
ncu -i /tmp/g3.ncu-rep --page source --csv -k regex:g1_scatter > $P/src_g1_scatter.csv 2>/dev/null
ls -la $P
