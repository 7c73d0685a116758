# Round-2 evidence run: GPU suite (parity log), smoke, default bench line, then the ncu
# launch list and full captures (tools/gpu_r2_ncu.sh).
bash tools/gpu_r2_check.sh
bash tools/gpu_r2_ncu.sh
