tools/cu/pcie > gpurun_out/pcie.txt 2>&1
python tools/prof_c2.py 512 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(clg_fwd|cli_chunks)" --launch-skip 0 --launch-count 4 -o gpurun_out/c2_full_r02 python tools/prof_c2.py 512 > gpurun_out/ncu_c2_r02.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(chunk|colc)" --launch-skip 0 --launch-count 4 -o gpurun_out/c3_full_r02 python tools/prof_c3.py > gpurun_out/ncu_c3_r02.log 2>&1
