python -m pytest tests/test_gpu_parity.py -x -q -k "boundaries or p2r or power_of_two or u64_past or footprint or product" > gpurun_out/t13.log 2>&1; tail -1 gpurun_out/t13.log
python -m pytest tests/test_gpu_configs.py -x -q -k "config3 or config4" >> gpurun_out/t13.log 2>&1; tail -1 gpurun_out/t13.log
for lib in tools/variants/libtftb200_before.so paper_1001_5272_b200/libtftb200.so; do
  echo "== $lib" >> gpurun_out/ab.txt
  TFTB_LIB=$lib python tools/time_sizes.py 144971 262570 1049940 4198396 8388607 >> gpurun_out/ab.txt 2>&1
  TFTB_LIB=$lib python tools/time_sizes.py 3221225473 16777216 33554431 67130680 >> gpurun_out/ab.txt 2>&1
  TFTB_LIB=$lib python tools/time_sizes.py 4179340454199820289 144971 4198396 >> gpurun_out/ab.txt 2>&1
done
