#!/bin/bash
# Round-2 GPU pass: cuRAND device pin + library baseline, Engine::mt full-volume parity, and a
# 2-rank smoke run of bench.py's multi-rank path (gloo, both ranks on the one GPU).
cd "$(dirname "$0")/.."
timeout 900 python -m pytest -q -x tests/test_gpu_curand_device.py "tests/test_gpu_full_parity.py::test_mt19937_every_word_against_the_reference" > gpurun_out/c4_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/c4_tests.log
timeout 600 oracle/_ref/curand_device time 16777216 3 > gpurun_out/curand_time.json 2> gpurun_out/curand_time.err
echo "curand time rc=$?"; cat gpurun_out/curand_time.json
timeout 300 python bench.py --config mt19937 --steps 20 --warmup 5 > gpurun_out/bench_mt19937.log 2>&1
echo "bench mt rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 3 --warmup 3 --calls 8 --dist-backend gloo --share-device > gpurun_out/bench_2rank.log 2>&1
echo "2-rank rc=$?"; grep '^{' gpurun_out/bench_2rank.log | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --gpus 2 --config c5 --steps 3 --warmup 3 --dist-backend gloo --share-device > gpurun_out/bench_2rank_c5.log 2>&1
echo "2-rank c5 rc=$?"; grep '^{' gpurun_out/bench_2rank_c5.log | cut -c1-400
timeout 600 python -m pytest -q -s tests/test_cpp_layer.py::test_cpp_layer_gpu > gpurun_out/cpp_layer_gpu.log 2>&1
echo "cpp layer rc=$?"; grep THREADS gpurun_out/cpp_layer_gpu.log
timeout 600 python tools/sweep.py 134217728 0 11213 3 2 3 > gpurun_out/sweep_masksel.jsonl 2> gpurun_out/sweep_masksel.err
echo "sweep rc=$?"; cut -c1-160 gpurun_out/sweep_masksel.jsonl
