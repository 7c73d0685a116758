# HCS parity tests + C5/C3 HCS bench lines (TMA slab kernel vs LSH_HCS_NO_TMA=1)
mkdir -p gpurun_out/r2
export LSH_PARITY_LOG=gpurun_out/r2/parity_hcs.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fastpath.py tests/test_gpu_theory.py -q -m gpu -x -rf -k "hcs or HCS or C3 or C5" > gpurun_out/r2/pytest_hcs.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_hcs.log
tail -2 gpurun_out/r2/pytest_hcs.log
for E in 0 1; do
for W in "--config C5 --scheme HCS_E2LSH --steps 3" "--config C5 --scheme HCS_SRP --steps 3" "--config C3 --scheme HCS_E2LSH" "--config C3 --scheme HCS_SRP"; do
  LSH_HCS_NO_TMA=$E timeout 600 python bench.py $W --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('notma=$E', d['config']['workload'], round(d['ms_per_step'],4), 'sketch', round(d['kernel_ms_per_step']['sketch'],4), r['kernel'], round(r['frac'],3))"
done; done
