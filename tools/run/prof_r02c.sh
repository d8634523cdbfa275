# round 2, after the F32 wide-word rounds: full ncu captures of config 3's kernels at
# 2^24, 2^25 - 1 and 2^25 + 1 (p = 3221225473), exploration lines, bench line
set -x
mkdir -p /tmp/reps
ST=smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_math_pipe_throttle,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_not_selected,smsp__pcsamp_warps_issue_stalled_selected,smsp__pcsamp_sample_count
for n in 16777216 33554431 33554433; do
  python tools/prof_c3.py $n > /dev/null 2>&1 || exit 1
  # the second forward + inverse of the script (the first is warm-up): skip its launches
  ncu --set full --import-source on --clock-control none -k regex:"k_(chunk|colc|col1|last|p2r)" --launch-count 16 -o /tmp/reps/c3_$n python tools/prof_c3.py $n > gpurun_out/ncu_c3_$n.log 2>&1
  ncu -i /tmp/reps/c3_$n.ncu-rep --page details --csv > gpurun_out/c3w_details_$n.csv 2>/dev/null
  ncu -i /tmp/reps/c3_$n.ncu-rep --page raw --csv --metrics $ST,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/c3w_raw_$n.csv 2>/dev/null
done
python bench.py --config 3 --steps 5 > gpurun_out/explore_c3_wide.jsonl 2>&1
python bench.py --config 5 --steps 3 > gpurun_out/explore_c5_wide.jsonl 2>&1
python bench.py > gpurun_out/bench_wide.jsonl 2>gpurun_out/bench_wide.err
ls -la gpurun_out
