# ncu --set full of one C4 CS_E2LSH build (NVTX range "profile"), per-kernel raw metrics
# and CUDA-source-level stall attribution.  Usage: KERNELS="g2a|g1_scatter" bash tools/gpu_r2_prof.sh
mkdir -p gpurun_out/r2/prof2
P=gpurun_out/r2/prof2
K=${KERNELS:-"sketch_kernel|g1_hist|g1_scatter|g2a"}
ncu -f --set full --clock-control none --import-source on --nvtx --nvtx-include "profile/" -k regex:"$K" -o /tmp/p2 \
    python tools/prof_hash.py --config ${CFG:-C4} --scheme ${SCHEME:-CS_E2LSH} --op build --reps 1 > $P/ncu.log 2>&1
ncu -i /tmp/p2.ncu-rep --page raw --csv > $P/raw.csv 2>/dev/null
for k in $(echo $K | tr '|' ' '); do
  ncu -i /tmp/p2.ncu-rep --page source --csv --print-source cuda -k regex:$k > $P/srccuda_$k.csv 2>/dev/null
  ncu -i /tmp/p2.ncu-rep --page source --csv -k regex:$k > $P/srcsass_$k.csv 2>/dev/null
done
ls -la $P
