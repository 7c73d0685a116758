# ncu (full set, source-level) of the C3 HCS-E2LSH sketch (K2 TMA slab ring)
P=gpurun_out/r2/prof_c3
mkdir -p $P
ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -k regex:"sketch_hcs" -o /tmp/c3 \
    python tools/prof_hash.py --config C3 --scheme HCS_E2LSH --op hash --reps 1 > $P/ncu.log 2>&1
ncu -i /tmp/c3.ncu-rep --page raw --csv > $P/raw.csv 2>/dev/null
ncu -i /tmp/c3.ncu-rep --page source --csv > $P/src.csv 2>/dev/null
python tools/sass_regions.py $P/src.csv --top 10 > $P/regions.txt 2>&1
cat $P/regions.txt
