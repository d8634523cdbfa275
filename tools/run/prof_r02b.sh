set -x
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum
for n in 16777216 33554431; do
python tools/prof_c3.py $n > /dev/null 2>&1 && ncu --metrics $M --clock-control none --csv --log-file gpurun_out/c3w_$n.csv python tools/prof_c3.py $n > gpurun_out/ncu_c3w_$n.log 2>&1
done
