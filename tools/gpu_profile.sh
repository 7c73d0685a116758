# Profiling pass for profiles/: launch list of the bench command + full capture of the sketch kernel.
set -x
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch_kernel|radix_downsweep|segsort_window|rle_write" -s 5 -c 5 \
    -o gpurun_out/c4_build_full python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > gpurun_out/ncu_full.log 2>&1
echo done
