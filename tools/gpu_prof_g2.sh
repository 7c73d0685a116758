# Source-level ncu profile of g2_sort on a C4 build; exports per-line CSV on the box.
#   bash tools/gpu_prof_g2.sh [SCHEME]
set -x
S=${1:-CS_E2LSH}
mkdir -p gpurun_out
python tools/prof_hash.py --config C4 --scheme $S --op build --reps 1 > gpurun_out/g2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"g2_sort" -s 1 -c 1 \
    -o /tmp/g2rep python tools/prof_hash.py --config C4 --scheme $S --op build --reps 1 > gpurun_out/ncu_g2.log 2>&1
ncu -i /tmp/g2rep.ncu-rep --page source --csv --print-source cuda,sass > /tmp/g2src.csv 2>/dev/null
python tools/ncu_lines.py /tmp/g2src.csv 60 > gpurun_out/g2_lines.txt
ncu -i /tmp/g2rep.ncu-rep --page details --csv > gpurun_out/g2_details.csv 2>/dev/null
ncu -i /tmp/g2rep.ncu-rep --page raw --csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for i,k in enumerate(h):
    if 'smsp__pcsamp_warps_issue_stalled' in k or 'smsp__average_warp' in k:
        print(k, r[2][i])
" > gpurun_out/g2_stalls.txt
echo done
