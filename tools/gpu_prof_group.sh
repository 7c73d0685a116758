# ncu --set full of the grouping kernels on a C4 index build (one launch each): bash tools/gpu_prof_group.sh SCHEME
set -x
S=${1:-CS_E2LSH}
mkdir -p gpurun_out
python tools/prof_hash.py --config C4 --scheme $S --op build --reps 1 > gpurun_out/prof_plain_$S.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"g1_scatter|g2_sort" -s 2 -c 2 \
    -o gpurun_out/group_$S python tools/prof_hash.py --config C4 --scheme $S --op build --reps 1 > gpurun_out/ncu_group_$S.log 2>&1
echo done
