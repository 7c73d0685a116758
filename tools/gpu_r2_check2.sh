# GPU suite + smoke + default bench line + C4 SRP bench line
bash tools/gpu_r2_check.sh
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config C4 --scheme CS_SRP > gpurun_out/r2/bench_C4_SRP.log 2>&1
tail -c 400 gpurun_out/r2/bench_C4_SRP.log
