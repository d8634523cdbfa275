mkdir -p tools/cu/_bin; [ -x tools/cu/_bin/pcie ] || nvcc -O2 -o tools/cu/_bin/pcie tools/cu/pcie.cu; tools/cu/_bin/pcie > gpurun_out/pcie.txt 2>&1
python tools/prof_c2.py 512 > /dev/null 2>&1
mkdir -p /tmp/reps
ncu --set full --import-source on --clock-control none -k regex:"k_(clg_fwd|cli_chunks)" --launch-skip 0 --launch-count 4 -o /tmp/reps/c2 python tools/prof_c2.py 512 > gpurun_out/ncu_c2_r02.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(chunk|colc)" --launch-skip 0 --launch-count 4 -o /tmp/reps/c3 python tools/prof_c3.py > gpurun_out/ncu_c3_r02.log 2>&1
for r in c2 c3; do
  ncu -i /tmp/reps/$r.ncu-rep --page details --csv > gpurun_out/${r}_details_r02.csv 2>/dev/null
  ncu -i /tmp/reps/$r.ncu-rep --page raw --csv --metrics smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_math_pipe_throttle,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_not_selected,smsp__pcsamp_warps_issue_stalled_selected,smsp__pcsamp_sample_count > gpurun_out/${r}_stalls_r02.csv 2>/dev/null
done
python tools/ncu_lines.py /tmp/reps/c2.ncu-rep k_clg_fwd 0 30 > gpurun_out/c2_fwd_lines_r02.txt 2>&1
python tools/ncu_lines.py /tmp/reps/c2.ncu-rep k_cli_chunks 0 30 > gpurun_out/c2_inv_lines_r02.txt 2>&1
python tools/ncu_lines.py /tmp/reps/c3.ncu-rep k_chunk_fwd 0 30 > gpurun_out/c3_chunk_lines_r02.txt 2>&1
python tools/ncu_lines.py /tmp/reps/c3.ncu-rep k_colc_fwd 0 30 > gpurun_out/c3_colc_lines_r02.txt 2>&1
ls -la gpurun_out
