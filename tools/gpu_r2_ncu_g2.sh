# ncu of the grouping kernels of one C4 CS_E2LSH build (+ C5 HCS_E2LSH), source-level stalls
mkdir -p gpurun_out/r2/prof_g2
P=gpurun_out/r2/prof_g2
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -k regex:"g2a|g2e|g2s|g2_big" -o /tmp/g2 \
    python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > $P/ncu.log 2>&1
ncu -i /tmp/g2.ncu-rep --page raw --csv > $P/raw.csv 2>/dev/null
ncu -i /tmp/g2.ncu-rep --page source --csv -k regex:g2a > $P/src_g2a.csv 2>/dev/null
ncu --set full --clock-control none --nvtx --nvtx-include "profile/" -k regex:"g2a|g2e|g2s|g2_big" -o /tmp/g2c5 \
    python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op build --reps 1 > $P/ncu_c5.log 2>&1
ncu -i /tmp/g2c5.ncu-rep --page raw --csv > $P/raw_c5.csv 2>/dev/null
ls -la $P
