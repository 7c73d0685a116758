# ncu --set full of the sketch kernels: C4 E2LSH, C4 SRP, C5 HCS-E2LSH (one launch each)
set -x
mkdir -p gpurun_out
python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op hash --reps 1 > gpurun_out/ps1.log 2>&1 && \
python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op hash --reps 1 --n 20000 > gpurun_out/ps2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch" -s 1 -c 1 -o gpurun_out/sk_c4e2 python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op hash --reps 1 > gpurun_out/ncu_sk1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sketch" -s 1 -c 1 -o gpurun_out/sk_c4srp python tools/prof_hash.py --config C4 --scheme CS_SRP --op hash --reps 1 > gpurun_out/ncu_sk2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sketch" -s 1 -c 1 -o gpurun_out/sk_c5 python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op hash --reps 1 --n 20000 > gpurun_out/ncu_sk3.log 2>&1
echo done
