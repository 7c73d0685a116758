# Source-level ncu profile of the C4 CS-E2LSH sketch kernel; per-line CSV summarised on the box.
set -x
mkdir -p gpurun_out
S=${1:-CS_E2LSH}
python tools/prof_hash.py --config C4 --scheme $S --op hash --reps 1 > gpurun_out/sk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch" -s 1 -c 1 \
    -o /tmp/skrep python tools/prof_hash.py --config C4 --scheme $S --op hash --reps 1 > gpurun_out/ncu_sk.log 2>&1
ncu -i /tmp/skrep.ncu-rep --page source --csv --print-source cuda,sass > /tmp/sksrc.csv 2>/dev/null
python tools/ncu_lines.py /tmp/sksrc.csv 50 > gpurun_out/sk_lines.txt
ncu -i /tmp/skrep.ncu-rep --page raw --csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for i,k in enumerate(h):
    if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued'):
        print(k, r[2][i])
" > gpurun_out/sk_stalls.txt
