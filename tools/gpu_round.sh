# One GPU pass: parity tests, smoke, bench lines (E2LSH + SRP + C5 HCS + dense C2), launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --scheme CS_SRP --no-cpu-baseline > gpurun_out/bench_srp.log 2>&1
timeout 600 python bench.py --config C5 --scheme HCS_E2LSH --no-cpu-baseline --steps 3 > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config C2 --scheme E2LSH --no-cpu-baseline > gpurun_out/bench_c2_dense.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo done
