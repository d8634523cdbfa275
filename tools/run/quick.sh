python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or product or ragged or plan or concurrent or host_batch" > gpurun_out/tq.log 2>&1; tail -2 gpurun_out/tq.log
python bench.py --no-cpu --no-c3 --no-e2e > gpurun_out/bq.log 2>&1
TFTB_SPLIT_INV=1 python bench.py --no-cpu --no-c3 --no-e2e > gpurun_out/bq_split.log 2>&1
