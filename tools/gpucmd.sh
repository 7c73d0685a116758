python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 2 > gpurun_out/p_build.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch_kernel|radix_downsweep|segsort_small|radix_upsweep" -s 6 -c 5 -o gpurun_out/build_c4 python tools/prof_hash.py --config C4 --scheme CS_E2LSH --op build --reps 1 > gpurun_out/ncu.log 2>&1
echo ncu=$?
cat gpurun_out/p_build.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gpu_tests.log
