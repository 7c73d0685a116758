# Round-end evidence: GPU suite, smoke, the default bench line and every bench leg, reference arm.
set -x
mkdir -p gpurun_out/legs
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/legs/C4_CS_E2LSH.log 2>&1
timeout 600 python bench.py --scheme CS_SRP > gpurun_out/legs/C4_CS_SRP.log 2>&1
timeout 600 python bench.py --per-table --steps 5 > gpurun_out/legs/C4_CS_E2LSH_per_table.log 2>&1
timeout 600 python bench.py --per-table --scheme CS_SRP --steps 5 > gpurun_out/legs/C4_CS_SRP_per_table.log 2>&1
timeout 600 python bench.py --config C5 --scheme HCS_E2LSH --steps 3 > gpurun_out/legs/C5_HCS_E2LSH.log 2>&1
timeout 600 python bench.py --config C5 --scheme HCS_SRP --steps 3 > gpurun_out/legs/C5_HCS_SRP.log 2>&1
timeout 900 python bench.py --config C5 --scheme E2LSH --steps 3 --warmup 3 > gpurun_out/legs/C5_E2LSH_dense.log 2>&1
timeout 600 python bench.py --config C3 --scheme HCS_E2LSH > gpurun_out/legs/C3_HCS_E2LSH.log 2>&1
timeout 600 python bench.py --config C2 --scheme E2LSH > gpurun_out/legs/C2_E2LSH_dense.log 2>&1
timeout 600 python bench.py --config C2 --scheme CS_E2LSH > gpurun_out/legs/C2_CS_E2LSH.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/legs/reference_C4_CS_E2LSH.log 2>&1
