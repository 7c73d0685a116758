# Profiling pass for profiles/: bench line, launch list of the bench command, full captures
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_plain.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
K='regex:sketch|g0_mask|g1_hist|g1_scatter|g2_sort|g3_rle'
python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "$K" -s 5 -c 5 -o gpurun_out/C4_CS_E2LSH_full \
    python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > gpurun_out/ncu1.log 2>&1
python tools/prof_hash.py --config C4 --scheme CS_SRP --op build --reps 1 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "$K" -s 7 -c 7 -o gpurun_out/C4_CS_SRP_full \
    python tools/prof_hash.py --config C4 --scheme CS_SRP --op build --reps 1 > gpurun_out/ncu2.log 2>&1
python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op hash --reps 1 --n 20000 > gpurun_out/p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch -s 1 -c 1 -o gpurun_out/C5_HCS_E2LSH_full \
    python tools/prof_hash.py --config C5 --scheme HCS_E2LSH --op hash --reps 1 --n 20000 > gpurun_out/ncu3.log 2>&1

# summarize on the box (ncu reports are too large to copy back), keep the text evidence
python tools/summarize_profiles.py round1 > gpurun_out/summarize.log 2>&1
mkdir -p gpurun_out/profiles_box && cp -r profiles/* gpurun_out/profiles_box/
mkdir -p gpurun_out/keep && mv gpurun_out/C5_HCS_E2LSH_full.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/*_full.ncu-rep
