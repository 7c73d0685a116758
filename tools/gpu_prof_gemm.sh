# ncu --set full of the tcgen05 GEMM (fused key epilogue): C4 per-table CS-E2LSH hash, C2 dense E2LSH hash
set -x
mkdir -p gpurun_out
python tools/prof_hash.py --config C4 --scheme CS_E2LSH --per-table --op hash --reps 1 --n 200000 > gpurun_out/pg1.log 2>&1 && \
ncu --set full --clock-control none -k regex:"dense_tc|split3" -s 2 -c 2 -o /tmp/C4PT_CS_E2LSH_full \
    python tools/prof_hash.py --config C4 --scheme CS_E2LSH --per-table --op hash --reps 1 --n 200000 > gpurun_out/ncu_pg1.log 2>&1
python tools/prof_hash.py --config C2 --scheme E2LSH --op hash --reps 1 > gpurun_out/pg2.log 2>&1 && \
ncu --set full --clock-control none -k regex:"dense_tc|split3" -s 2 -c 2 -o /tmp/C2_E2LSH_full \
    python tools/prof_hash.py --config C2 --scheme E2LSH --op hash --reps 1 > gpurun_out/ncu_pg2.log 2>&1
for r in C4PT_CS_E2LSH C2_E2LSH; do
  ncu -i /tmp/${r}_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size > gpurun_out/${r}_gemm_raw.csv 2>&1
  ncu -i /tmp/${r}_full.ncu-rep --page details --csv > gpurun_out/${r}_gemm_details.csv 2>&1
done
echo done
