timeout 600 python bench.py --config c5 --steps 70 --no-e2e --no-cpu-baseline >> gpurun_out/c5_sus.jsonl 2>> gpurun_out/c5_sus.err
timeout 600 python bench.py --config c5 --as-rank 0 --as-world 2 --steps 130 --no-e2e --no-cpu-baseline >> gpurun_out/c5_sus.jsonl 2>> gpurun_out/c5_sus.err
timeout 600 python bench.py --config c5 --as-rank 1 --as-world 2 --steps 130 --no-e2e --no-cpu-baseline >> gpurun_out/c5_sus.jsonl 2>> gpurun_out/c5_sus.err
for r in 0 3; do timeout 600 python bench.py --config c5 --as-rank $r --as-world 4 --steps 250 --no-e2e --no-cpu-baseline >> gpurun_out/c5_sus.jsonl 2>> gpurun_out/c5_sus.err; done
for r in 0 7; do timeout 600 python bench.py --config c5 --as-rank $r --as-world 8 --steps 500 --no-e2e --no-cpu-baseline >> gpurun_out/c5_sus.jsonl 2>> gpurun_out/c5_sus.err; done
