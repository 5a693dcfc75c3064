timeout 900 python bench.py --config c5 > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.err
for W in 2 4 8; do for r in $(seq 0 $((W-1))); do timeout 300 python bench.py --config c5 --as-rank $r --as-world $W --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/c5_as_w$W.jsonl 2>> gpurun_out/c5_as.err; done; done
