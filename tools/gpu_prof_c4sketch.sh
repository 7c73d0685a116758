set -x
mkdir -p gpurun_out
python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op hash --reps 1 > gpurun_out/pc4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch -s 1 -c 1 -o gpurun_out/sk_c4e2b python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op hash --reps 1 > gpurun_out/ncu_c4.log 2>&1
