# NEXT-2 per-table families: GPU parity tests + bench legs (C4 per-table E2LSH / SRP)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "per_table" > gpurun_out/pytest_pt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pt.log
timeout 600 python bench.py --per-table --steps 5 > gpurun_out/bench_pt_e2.log 2>&1
timeout 600 python bench.py --per-table --scheme CS_SRP --steps 5 --no-e2e > gpurun_out/bench_pt_srp.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "dense or fused" > gpurun_out/pytest_dense.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dense.log
timeout 600 python bench.py --config C5 --scheme E2LSH --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_dense.log 2>&1
