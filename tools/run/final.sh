python -m pytest tests -m gpu -x -q > gpurun_out/t_final.log 2>&1; tail -2 gpurun_out/t_final.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/t_final.log 2>&1; tail -1 gpurun_out/t_final.log
python bench.py > gpurun_out/b_final.log 2>&1
python bench.py --impl reference > gpurun_out/b_final_ref.log 2>&1
python bench.py --config 5 --steps 3 > gpurun_out/explore_c5_final.jsonl 2>&1
python bench.py --config 3 --steps 5 > gpurun_out/explore_c3_final.jsonl 2>&1
python bench.py --config 1 --steps 5 > gpurun_out/explore_c1_final.jsonl 2>&1
