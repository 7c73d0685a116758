# ncu --set full of the C4 CS-E2LSH sketch (four-tables-per-warp keys-only path) + SASS regions
F=gpurun_out/quad
mkdir -p $F
python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > $F/plain.log 2>&1 || { tail $F/plain.log; exit 1; }
ncu -f --set full --clock-control none --import-source on -k regex:sketch_kernel -s 0 -c 1 -o /tmp/sk_quad \
    python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > $F/ncu.log 2>&1
ncu -i /tmp/sk_quad.ncu-rep --page raw --csv > $F/raw.csv 2>/dev/null
ncu -i /tmp/sk_quad.ncu-rep --page details > $F/details.txt 2>/dev/null
ncu -i /tmp/sk_quad.ncu-rep --page source --csv -k regex:sketch_kernel > $F/src.csv 2>/dev/null
python tools/sass_regions.py $F/src.csv --top 8 > $F/regions.txt 2>&1
cp /tmp/sk_quad.ncu-rep $F/
tail -2 $F/ncu.log
