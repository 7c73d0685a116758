set -x
mkdir -p gpurun_out
python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op hash --reps 1 --n 20000 > gpurun_out/ph.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch" -s 1 -c 1 -o gpurun_out/sk_hcs python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op hash --reps 1 --n 20000 > gpurun_out/ncu_hcs.log 2>&1
