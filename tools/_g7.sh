python tools/sweep.py 134217728 0 44497 3 1 0 > gpurun_out/sw_leaf_44497.jsonl 2>&1
python tools/sweep.py 134217728 0 23209 3 1 0 > gpurun_out/sw_leaf_23209.jsonl 2>&1
