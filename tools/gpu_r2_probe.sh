mkdir -p gpurun_out/r2
python tools/g2w_probe.py --config C4 --scheme CS_E2LSH > gpurun_out/r2/probe.log 2>&1
python tools/g2w_probe.py --config C5 --scheme HCS_E2LSH >> gpurun_out/r2/probe.log 2>&1
cat gpurun_out/r2/probe.log
